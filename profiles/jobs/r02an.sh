#!/bin/bash
mkdir -p gpurun_out
SCONV_HOST_TRACE=1 timeout 300 python profiles/host_trace.py > gpurun_out/r02an_host.txt 2>&1
grep "sconv host" gpurun_out/r02an_host.txt > /tmp/h.txt; n=$(grep -n "forward: streams joined" /tmp/h.txt | tail -1 | cut -d: -f1); tail -n +$n /tmp/h.txt | head -70
