#!/bin/bash
# r02av: skeleton: tcgen05.commit vs a plain mbarrier arrive for the free-stage signal (no MMAs in both)
mkdir -p gpurun_out
for d in 263 279 258 274; do echo "== REG0 debug $d"; SCONV_FUSED_REG=0 SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02av.txt 2>&1
for d in 2 18; do echo "== REG1 debug $d"; SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done >> gpurun_out/r02av.txt 2>&1
cat gpurun_out/r02av.txt
