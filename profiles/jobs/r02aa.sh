#!/bin/bash
# r02aa: coordinate look-ahead (Eq. 1 of the next strided conv queued when a coordinate set is created)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_network.py tests/test_gpu_fullsize.py tests/test_gpu_spec_api.py -q -x 2>&1 | tail -15 > gpurun_out/r02aa_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02aa_bench_c2.json 2>/dev/null
SCONV_NET_COORD_AHEAD=0 $B > gpurun_out/r02aa_bench_c2_noahead.json 2>/dev/null
$B --workload c3_resnet21d_s3dis > gpurun_out/r02aa_bench_c3.json 2>/dev/null
$B --workload c4_unet_pair_shapenet > gpurun_out/r02aa_bench_c4.json 2>/dev/null
$B --workload c5_minkunet42_batch64 --steps 3 --warmup 3 > gpurun_out/r02aa_bench_c5.json 2>/dev/null
timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02aa_tl_c2.json > gpurun_out/r02aa_tl_c2.txt 2>&1
cat gpurun_out/r02aa_tests.log; for f in gpurun_out/r02aa_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
grep "^forward" gpurun_out/r02aa_tl_c2.txt; grep -A12 "^forward 1" gpurun_out/r02aa_tl_c2.txt | grep gap
