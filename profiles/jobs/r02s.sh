#!/bin/bash
# r02s: PDL between fused convs + sanitizer fixes: parity, A/B (r02f build vs HEAD v1/v2, PDL on/off), timelines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -5 > gpurun_out/r02s_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
(cd ab/r02f && $B > ../../gpurun_out/r02s_bench_old.json 2>/dev/null)
$B > gpurun_out/r02s_bench_v2_pdl.json 2>/dev/null
SCONV_PDL=0 $B > gpurun_out/r02s_bench_v2_nopdl.json 2>/dev/null
SCONV_FUSED_V1=1 $B > gpurun_out/r02s_bench_v1_pdl.json 2>/dev/null
SCONV_FUSED_V1=1 SCONV_PDL=0 $B > gpurun_out/r02s_bench_v1_nopdl.json 2>/dev/null
(cd ab/r02f && timeout 300 python profiles/net_layers.py --json ../../gpurun_out/r02s_layers_old.json > ../../gpurun_out/r02s_layers_old.txt 2>&1)
SCONV_FUSED_V1=1 timeout 300 python profiles/net_layers.py --json gpurun_out/r02s_layers_v1.json > gpurun_out/r02s_layers_v1.txt 2>&1
timeout 300 python profiles/timeline.py --json gpurun_out/r02s_tl_v2_pdl.json > gpurun_out/r02s_tl_v2_pdl.txt 2>&1
SCONV_PDL=0 timeout 300 python profiles/timeline.py --json gpurun_out/r02s_tl_v2_nopdl.json > gpurun_out/r02s_tl_v2_nopdl.txt 2>&1
(cd ab/r02f && timeout 300 python ../../profiles/timeline.py > ../../gpurun_out/r02s_tl_old.txt 2>&1)
for tool in memcheck initcheck; do timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02s_san_$tool.log 2>&1; done
cat gpurun_out/r02s_tests.log; for f in gpurun_out/r02s_bench_*.json; do echo "$f $(cut -c1-200 $f | grep -o 'ms_per_step": [0-9.]*')"; done
tail -n1 gpurun_out/r02s_layers_*.txt; head -12 gpurun_out/r02s_tl_*.txt; grep -h "ERROR SUMMARY" gpurun_out/r02s_san_*.log
