#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -4
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02z_bench_c2.json 2>/dev/null
SCONV_POOL_INTERNAL_DEPS=1 $B > gpurun_out/r02z_bench_c2_deps.json 2>/dev/null
$B --workload c3_resnet21d_s3dis > gpurun_out/r02z_bench_c3.json 2>/dev/null
SCONV_HOST_TRACE=1 timeout 300 python profiles/timeline.py --forwards 1 --json gpurun_out/r02z_tl_c2.json > gpurun_out/r02z_tl_c2.txt 2> gpurun_out/r02z_host.txt
for f in gpurun_out/r02z_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
grep "sconv host" gpurun_out/r02z_host.txt > /tmp/h.txt; n=$(grep -n "forward: streams joined" /tmp/h.txt | tail -1 | cut -d: -f1); tail -n +$n /tmp/h.txt | head -60
grep "^forward" gpurun_out/r02z_tl_c2.txt
