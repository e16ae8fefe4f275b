#!/bin/bash
# r02bu: rows per thread of the one-launch cooperative sorts (SCONV_COOP_E 1/2/4): C2, C3, C4 same box
mkdir -p gpurun_out
for i in 1 2; do
  for e in 1 2 4; do
    for w in c2_minkunet42_kitti c3_resnet21d_s3dis c4_unet_pair_shapenet; do
      SCONV_COOP_E=$e timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bu_${w}_e$e$i.json 2>/dev/null
    done
  done
done
for f in gpurun_out/r02bu_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
