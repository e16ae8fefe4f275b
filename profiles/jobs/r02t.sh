#!/bin/bash
# r02t: tile-queue kernel restored (hot-loop instrumentation removed), work items only on few-tile wide convs, PDL
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -5 > gpurun_out/r02t_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02t_bench_c2.json 2>gpurun_out/r02t_bench_c2.err
SCONV_PDL=0 $B > gpurun_out/r02t_bench_c2_nopdl.json 2>/dev/null
(cd ab/r02f && $B > ../../gpurun_out/r02t_bench_c2_old.json 2>/dev/null)
$B --workload c3_resnet21d_s3dis > gpurun_out/r02t_bench_c3.json 2>/dev/null
timeout 300 python profiles/net_layers.py --json gpurun_out/r02t_layers_c2.json > gpurun_out/r02t_layers_c2.txt 2>&1
timeout 300 python profiles/net_layers.py --workload c3_resnet21d_s3dis --json gpurun_out/r02t_layers_c3.json > gpurun_out/r02t_layers_c3.txt 2>&1
timeout 300 python profiles/timeline.py --json gpurun_out/r02t_tl_c2.json > gpurun_out/r02t_tl_c2.txt 2>&1
cat gpurun_out/r02t_tests.log; for f in gpurun_out/r02t_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
tail -n1 gpurun_out/r02t_layers_*.txt; head -14 gpurun_out/r02t_tl_c2.txt
