#!/bin/bash
# r02g: fused-kernel cost decomposition (debug knobs: 1 no gather copies, 2 no MMAs, 4 no weight
# TMA, 256 no epilogue) on the KITTI level-0 map + source-level stalls of one 128->96 conv
mkdir -p gpurun_out /tmp/ncu
for dbg in 0 1 2 4 5 256 257 7; do
  echo "== debug $dbg"; SCONV_FUSED_DEBUG=$dbg timeout 120 python profiles/fused_time.py 32 96 256
done > gpurun_out/r02g_decomp.txt 2>&1
for occ in 1 2; do echo "== OCC $occ"; SCONV_FUSED_OCC=$occ timeout 120 python profiles/fused_time.py 32 96 256; done >> gpurun_out/r02g_decomp.txt 2>&1
echo "== REG 0" >> gpurun_out/r02g_decomp.txt; SCONV_FUSED_REG=0 timeout 120 python profiles/fused_time.py 32 96 256 >> gpurun_out/r02g_decomp.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name k_conv_fused --launch-skip 93 --launch-count 1 \
  -o /tmp/ncu/one -f python profiles/run_net.py c2_minkunet42_kitti > gpurun_out/r02g_ncu.log 2>&1
ncu -i /tmp/ncu/one.ncu-rep --page source --csv > gpurun_out/r02g_src.csv 2>&1
ncu -i /tmp/ncu/one.ncu-rep --page raw --csv > gpurun_out/r02g_raw.csv 2>&1
cat gpurun_out/r02g_decomp.txt; ls -la gpurun_out
