#!/bin/bash
# r02ac: derived down / transposed maps (no search); racecheck per fused-kernel variant
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02ac_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02ac_bench_c2.json 2>/dev/null
SCONV_NET_DERIVE=0 $B > gpurun_out/r02ac_bench_c2_noderive.json 2>/dev/null
$B --workload c4_unet_pair_shapenet > gpurun_out/r02ac_bench_c4.json 2>/dev/null
SCONV_NET_DERIVE=0 $B --workload c4_unet_pair_shapenet > gpurun_out/r02ac_bench_c4_noderive.json 2>/dev/null
$B --workload c3_resnet21d_s3dis > gpurun_out/r02ac_bench_c3.json 2>/dev/null
CS=/usr/local/cuda/bin/compute-sanitizer
for v in 0 1; do SCONV_FUSED_ITEMS=$v timeout 900 $CS --tool racecheck --print-limit 5 python profiles/sanitize_run.py --net > gpurun_out/r02ac_race_items$v.log 2>&1; done
SCONV_FUSED_ITEMS=0 SCONV_PDL=0 timeout 900 $CS --tool racecheck --print-limit 5 python profiles/sanitize_run.py > gpurun_out/r02ac_race_items0_nopdl_layer.log 2>&1
cat gpurun_out/r02ac_tests.log; for f in gpurun_out/r02ac_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
grep -h "RACECHECK SUMMARY" gpurun_out/r02ac_race_*.log
