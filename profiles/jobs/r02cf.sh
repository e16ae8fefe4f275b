#!/bin/bash
# r02cf: host inputs staged on the net's input stream (map builds of request i+1 beside the convs of request i),
# small readbacks by kernel stores, async result readback: GPU suite, e2e probe, bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python profiles/e2e_probe.py c2_minkunet42_kitti > gpurun_out/r02cf_probe_c2.txt 2>&1; head -7 gpurun_out/r02cf_probe_c2.txt
python profiles/e2e_probe.py c4_unet_pair_shapenet > gpurun_out/r02cf_probe_c4.txt 2>&1; head -7 gpurun_out/r02cf_probe_c4.txt
for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cf_bench_$w.json 2>gpurun_out/r02cf_$w.err
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cf_bench_c5.json 2>/dev/null
for f in gpurun_out/r02cf_bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3), 'lat', round(e.get('latency_ms',0),3), '%.3g'%e['value'])"; done
