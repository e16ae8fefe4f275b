#!/bin/bash
# r02aj: Eq. 1 on an occupancy bitmap (no cooperative sort): full GPU suite, same-box A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02aj_tests.log
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02aj_c2_bitmap_$i.json 2>/dev/null
SCONV_EQ1_BITMAP=0 $B > gpurun_out/r02aj_c2_sort_$i.json 2>/dev/null
done
for w in c3_resnet21d_s3dis c4_unet_pair_shapenet; do
$B --workload $w > gpurun_out/r02aj_${w}_bitmap.json 2>/dev/null
SCONV_EQ1_BITMAP=0 $B --workload $w > gpurun_out/r02aj_${w}_sort.json 2>/dev/null
done
timeout 300 python profiles/timeline.py --forwards 2 > gpurun_out/r02aj_tl_c2.txt 2>&1
cat gpurun_out/r02aj_tests.log; for f in gpurun_out/r02aj_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
sed -n '/kernel totals/,/timeline of/p' gpurun_out/r02aj_tl_c2.txt | head -30
