#!/bin/bash
# r02ar: fused kernel skeleton decomposition: epilogue off (256), skeleton without data and epilogue (263)
mkdir -p gpurun_out
for d in 0 256 263 7; do echo "== REG0 debug $d"; SCONV_FUSED_REG=0 SCONV_FUSED_DEBUG=$d timeout 120 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02ar.txt 2>&1
for d in 0 256 258; do echo "== REG1 debug $d"; SCONV_FUSED_DEBUG=$d timeout 120 python profiles/fused_time.py 32 96 256; done >> gpurun_out/r02ar.txt 2>&1
cat gpurun_out/r02ar.txt
