#!/bin/bash
# r02at: skeleton: which handshake costs (REG0 path debug bits): 263 base; +2048+4096 no full-barrier arrive/wait;
# +1024 producers skip the free-stage wait
mkdir -p gpurun_out
for d in 263 6407 1287 7431; do echo "== REG0 debug $d"; SCONV_FUSED_REG=0 SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02at.txt 2>&1
cat gpurun_out/r02at.txt
