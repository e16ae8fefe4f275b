#!/bin/bash
# r02cb: asynchronous result readback (sconv_net_read_async) -- parity test + pipelined e2e bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_network.py -m gpu -q -x -k "read_async or repeatable" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_capi.py tests/test_gpu_spec_api.py -q -x 2>&1 | tail -2
for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cb_bench_$w.json 2>gpurun_out/r02cb_$w.err
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cb_bench_c5.json 2>/dev/null
for f in gpurun_out/r02cb_bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3), 'lat', round(e.get('latency_ms',0),3), '%.3g'%e['value'])"; done
