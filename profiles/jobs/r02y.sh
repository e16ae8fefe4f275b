#!/bin/bash
# r02y: TMA-fed dense variant for 1x1 identity convs: parity + network suites, bench C2, per-conv table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -15 > gpurun_out/r02y_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02y_bench_c2.json 2>gpurun_out/r02y_bench_c2.err
SCONV_FUSED_DENSE=0 $B > gpurun_out/r02y_bench_c2_nodense.json 2>/dev/null
timeout 300 python profiles/net_layers.py --json gpurun_out/r02y_layers_c2.json > gpurun_out/r02y_layers_c2.txt 2>&1
cat gpurun_out/r02y_tests.log; for f in gpurun_out/r02y_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
grep -E "^ +[0-9]+ +1 " gpurun_out/r02y_layers_c2.txt; tail -n1 gpurun_out/r02y_layers_c2.txt
