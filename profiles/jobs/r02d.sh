#!/bin/bash
# r02d: fused-kernel cost decomposition on the KITTI level-0 map (debug knobs: 1 no gather copies,
# 2 no MMAs, 4 no weight TMA, 1+4 neither copy)
mkdir -p gpurun_out
for dbg in 0 1 2 4 5 3; do
  echo "== debug $dbg"; SCONV_FUSED_DEBUG=$dbg timeout 120 python profiles/fused_time.py 32 96 128 256
done 2>&1 | tee gpurun_out/r02d_decomp.txt
for g in 1 2 4; do echo "== G $g"; SCONV_FUSED_G=$g timeout 120 python profiles/fused_time.py 32 96 256; done 2>&1 | tee -a gpurun_out/r02d_decomp.txt
