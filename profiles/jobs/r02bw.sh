#!/bin/bash
# r02bw: Eq. 1 cluster kernel with the LSD scatter through global memory: parity, Eq. 1 A/B, bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "map or strided or large_fused" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_spec_api.py -m gpu -q -x 2>&1 | tail -2
for v in 1 0; do SCONV_FLOOR_CLUSTER=$v timeout 100 python profiles/eq1_time.py; done
for i in 1 2; do
  for v in 1 0; do
    for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
      SCONV_FLOOR_CLUSTER=$v timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bw_${w}_$v$i.json 2>/dev/null
    done
  done
done
for f in gpurun_out/r02bw_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
