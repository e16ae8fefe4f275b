#!/bin/bash
# r02i: producers' stage-wait variants (SCONV_FUSED_WAIT 0 try_wait / 1 test_wait / 2 lane-0 test_wait / 3 try_wait+hint)
mkdir -p gpurun_out
for w in 0 1 2 3; do echo "== WAIT $w"; SCONV_FUSED_WAIT=$w timeout 60 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02i_wait.txt 2>&1
for w in 1 2; do echo "== WAIT $w skeleton"; SCONV_FUSED_WAIT=$w SCONV_FUSED_DEBUG=7 timeout 60 python profiles/fused_time.py 32 96 256; done >> gpurun_out/r02i_wait.txt 2>&1
SCONV_FUSED_WAIT=1 SCONV_FUSED_DEBUG=8 timeout 60 python profiles/fused_time.py 96 2>&1 | tail -400 > gpurun_out/r02i_trace96_w1.txt
cat gpurun_out/r02i_wait.txt
