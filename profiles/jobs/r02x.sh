#!/bin/bash
# r02x: column search (k_search_col): map parity suites, C2/C3/C4/C1 bench, timeline, A/B vs per-offset search
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r02x_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02x_bench_c2.json 2>gpurun_out/r02x_bench_c2.err
SCONV_SEARCH_COL=0 $B > gpurun_out/r02x_bench_c2_nocol.json 2>/dev/null
$B --workload c3_resnet21d_s3dis > gpurun_out/r02x_bench_c3.json 2>/dev/null
$B --workload c4_unet_pair_shapenet > gpurun_out/r02x_bench_c4.json 2>/dev/null
$B --workload c1_layer_100k > gpurun_out/r02x_bench_c1.json 2>/dev/null
timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02x_tl_c2.json > gpurun_out/r02x_tl_c2.txt 2>&1
cat gpurun_out/r02x_tests.log; for f in gpurun_out/r02x_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
sed -n '/kernel totals/,/timeline of/p' gpurun_out/r02x_tl_c2.txt; grep "^forward" gpurun_out/r02x_tl_c2.txt
