#!/bin/bash
# r02al: fused-kernel pipeline knobs on one box: units per stage (G), CTAs per SM (OCC); C2 / C3 bench
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02al_c2_default.json 2>/dev/null
for g in 1 2 4; do SCONV_FUSED_G=$g $B > gpurun_out/r02al_c2_G$g.json 2>/dev/null; done
SCONV_FUSED_OCC=1 $B > gpurun_out/r02al_c2_occ1.json 2>/dev/null
SCONV_FUSED_OCC=1 SCONV_FUSED_G=1 $B > gpurun_out/r02al_c2_occ1_G1.json 2>/dev/null
$B > gpurun_out/r02al_c2_default2.json 2>/dev/null
for f in gpurun_out/r02al_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
