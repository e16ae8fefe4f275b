#!/bin/bash
# r02h: CTA-0 timeline of the fused kernel (SCONV_FUSED_DEBUG=8) on the KITTI level-0 map, c=32 / 96;
# the skeleton-only variant (8+7); and whether SCONV_FUSED_REG=0 terminates
mkdir -p gpurun_out
SCONV_FUSED_DEBUG=8 timeout 60 python profiles/fused_time.py 32 > gpurun_out/r02h_trace32.txt 2>&1
SCONV_FUSED_DEBUG=8 timeout 60 python profiles/fused_time.py 96 > gpurun_out/r02h_trace96.txt 2>&1
SCONV_FUSED_DEBUG=15 timeout 60 python profiles/fused_time.py 96 > gpurun_out/r02h_trace96_skel.txt 2>&1
SCONV_FUSED_REG=0 SCONV_DEBUG_SYNC=1 timeout 30 python profiles/fused_time.py 32 > gpurun_out/r02h_reg0.txt 2>&1; echo "reg0 rc=$?" >> gpurun_out/r02h_reg0.txt
wc -l gpurun_out/r02h_*; tail -3 gpurun_out/r02h_reg0.txt
