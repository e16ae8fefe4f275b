#!/bin/bash
# r02af: A/B on one box: default vs no K=2 row order (SCONV_SMALL_PERMUTE=0) vs no coordinate look-ahead
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02af_c2_default_$i.json 2>/dev/null
SCONV_SMALL_PERMUTE=0 $B > gpurun_out/r02af_c2_nosmallperm_$i.json 2>/dev/null
SCONV_NET_COORD_AHEAD=0 $B > gpurun_out/r02af_c2_noahead_$i.json 2>/dev/null
done
$B --workload c4_unet_pair_shapenet > gpurun_out/r02af_c4_default.json 2>/dev/null
SCONV_SMALL_PERMUTE=0 $B --workload c4_unet_pair_shapenet > gpurun_out/r02af_c4_nosmallperm.json 2>/dev/null
for f in gpurun_out/r02af_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
