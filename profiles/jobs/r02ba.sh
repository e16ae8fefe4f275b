#!/bin/bash
# r02ba: REG path: gather copies off + plain arrive (debug 32) vs copies off with the cp.async arrive (debug 1 has no
# effect on the REG path; 32 removes copies AND the noinc arrive), with/without MMAs (2) and epilogue (256)
mkdir -p gpurun_out
for d in 0 32 34 290; do echo "== REG1 debug $d"; SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02ba.txt 2>&1
cat gpurun_out/r02ba.txt
