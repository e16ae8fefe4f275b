#!/bin/bash
# r02co: adaptive readback chunks (512 KB unless the copy outlasts the forward, then 4 MB): network tests, C2/C3/C4/C5 e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_spec_api.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
  for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02co_${w}_$i.json 2>/dev/null
  done
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02co_c5.json 2>/dev/null
for f in gpurun_out/r02co_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
