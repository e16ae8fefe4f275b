#!/bin/bash
# r02ay: fused kernel time vs offsets per tile (K = 1 identity with gathers, K = 2, K = 3), real and skeleton (debug 263, REG0)
mkdir -p gpurun_out
for K in 1 2 3; do
  echo "== K=$K real"; SCONV_FUSED_DENSE=0 timeout 60 python profiles/fused_k.py $K 32 96 256
  echo "== K=$K skeleton"; SCONV_FUSED_DENSE=0 SCONV_FUSED_REG=0 SCONV_FUSED_DEBUG=263 timeout 60 python profiles/fused_k.py $K 32 96 256
done > gpurun_out/r02ay.txt 2>&1
cat gpurun_out/r02ay.txt
