#!/bin/bash
# r02k: per-CTA spans of the fused kernel (debug 8192) for full work and the empty skeleton; runtime-K3 test
mkdir -p gpurun_out
for d in 8192 15623; do echo "== debug $d"; SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256 2>&1 | grep -v "^\[spans\]" ; SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256 2>&1 | grep "^\[spans\]" | awk 'NR%83==0'; done > gpurun_out/r02k.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" >> gpurun_out/r02k.txt 2>&1
cat gpurun_out/r02k.txt
