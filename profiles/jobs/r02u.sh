#!/bin/bash
# r02u: kernel-variant test details; C2 kernel timeline + host timestamps of one forward
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k variants 2>&1 | grep -E "Error|assert|passed|failed|err" | head -20 > gpurun_out/r02u_tests.log
SCONV_NET_HOST_PROFILE=1 timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02u_tl_c2.json > gpurun_out/r02u_tl_c2.txt 2> gpurun_out/r02u_host.txt
cat gpurun_out/r02u_tests.log; head -80 gpurun_out/r02u_tl_c2.txt; tail -75 gpurun_out/r02u_host.txt
