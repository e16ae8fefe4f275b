#!/bin/bash
# r02aq: fused kernel, what bounds it: timings with the gather copies (1) / weight TMA (4) / MMAs (2) disabled
mkdir -p gpurun_out
for d in 0 1 4 5 2 7; do echo "== debug $d"; SCONV_FUSED_REG=0 SCONV_FUSED_DEBUG=$d timeout 120 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02aq_reg0.txt 2>&1
cat gpurun_out/r02aq_reg0.txt
