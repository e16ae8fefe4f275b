#!/bin/bash
mkdir -p gpurun_out
SCONV_FUSED_DEBUG=8192 timeout 60 python profiles/fused_time.py 32 96 256 2>&1 | grep "spans\|k_conv_items" | awk 'NR%84<=1' > gpurun_out/r02n.txt
cat gpurun_out/r02n.txt | head -20
