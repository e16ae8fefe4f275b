#!/bin/bash
# r02ag: coordinate look-ahead variants on one box (priority, what the first Eq. 1 waits for) vs off
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02ag_c2_lo_layout_$i.json 2>/dev/null
SCONV_COORD_PRIO=hi $B > gpurun_out/r02ag_c2_hi_layout_$i.json 2>/dev/null
SCONV_COORD_PRIO=hi SCONV_COORD_AFTER=map $B > gpurun_out/r02ag_c2_hi_map_$i.json 2>/dev/null
SCONV_COORD_AFTER=map $B > gpurun_out/r02ag_c2_lo_map_$i.json 2>/dev/null
SCONV_NET_COORD_AHEAD=0 $B > gpurun_out/r02ag_c2_off_$i.json 2>/dev/null
done
for w in c3_resnet21d_s3dis c4_unet_pair_shapenet; do
$B --workload $w > gpurun_out/r02ag_${w}_lo_layout.json 2>/dev/null
SCONV_NET_COORD_AHEAD=0 $B --workload $w > gpurun_out/r02ag_${w}_off.json 2>/dev/null
SCONV_COORD_PRIO=hi SCONV_COORD_AFTER=map $B --workload $w > gpurun_out/r02ag_${w}_hi_map.json 2>/dev/null
done
for f in gpurun_out/r02ag_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
