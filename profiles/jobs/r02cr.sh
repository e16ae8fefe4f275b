#!/bin/bash
# r02cr: bench serving loop with the automatic prefetch rule: C2 / C3 / C4 / C5 e2e
mkdir -p gpurun_out
for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cr_$w.json 2>gpurun_out/r02cr_$w.err
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cr_c5.json 2>/dev/null
for f in gpurun_out/r02cr_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3), e['mode'][:90])"; done
