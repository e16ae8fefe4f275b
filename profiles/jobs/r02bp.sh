#!/bin/bash
# r02bp: coordinate-stream priority A/B (C2, C3), same box
mkdir -p gpurun_out
for i in 1 2; do
  for p in lo hi; do
    SCONV_COORD_PRIO=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bp_c2_$p$i.json 2>/dev/null
    SCONV_COORD_PRIO=$p timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bp_c3_$p$i.json 2>/dev/null
  done
done
for f in gpurun_out/r02bp_c*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
