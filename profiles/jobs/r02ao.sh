#!/bin/bash
# r02ao: first look-ahead Eq. 1 right after the raw key packing (before the level-0 search), priorities
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_network.py -q -x 2>&1 | tail -2
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02ao_c2_default_$i.json 2>/dev/null
SCONV_COORD_AFTER=pack $B > gpurun_out/r02ao_c2_pack_lo_$i.json 2>/dev/null
SCONV_COORD_AFTER=pack SCONV_COORD_PRIO=hi $B > gpurun_out/r02ao_c2_pack_hi_$i.json 2>/dev/null
done
for w in c3_resnet21d_s3dis c4_unet_pair_shapenet; do
$B --workload $w > gpurun_out/r02ao_${w}_default.json 2>/dev/null
SCONV_COORD_AFTER=pack SCONV_COORD_PRIO=hi $B --workload $w > gpurun_out/r02ao_${w}_pack_hi.json 2>/dev/null
done
for f in gpurun_out/r02ao_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
