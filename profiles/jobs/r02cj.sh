#!/bin/bash
# r02cj: input prefetch (sconv_net_prefetch_inputs): network GPU tests, serving loop (no sanitizer: closed on the pool), e2e bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_spec_api.py tests/test_adapter.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python profiles/sanitize_run.py --net 2>&1 | tail -2
for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cj_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cj_bench_c5.json 2>/dev/null
for f in gpurun_out/r02cj_bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3), '%.3g'%e['value'])"; done
