#!/bin/bash
# r02ai: mask bits by map size (16 above 200k rows) on C3 / C2, one box
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B --workload c3_resnet21d_s3dis > gpurun_out/r02ai_c3_default_$i.json 2>/dev/null
SCONV_MASK_BITS=24 $B --workload c3_resnet21d_s3dis > gpurun_out/r02ai_c3_bits24_$i.json 2>/dev/null
SCONV_MASK_BITS=16 $B --workload c3_resnet21d_s3dis > gpurun_out/r02ai_c3_bits16_$i.json 2>/dev/null
done
$B > gpurun_out/r02ai_c2_default.json 2>/dev/null
for f in gpurun_out/r02ai_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
