#!/bin/bash
# r02l: work-item fused kernel (k_conv_items): parity, A/B vs the tile-queue kernel, spans, per-conv table
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or layer or c1" 2>&1 | tail -15 > gpurun_out/r02l_tests.txt
for v in 1 0; do echo "== V1=$v"; SCONV_FUSED_V1=$v timeout 60 python profiles/fused_time.py 32 96 128 256; done > gpurun_out/r02l_ab.txt 2>&1
SCONV_FUSED_DEBUG=8192 timeout 60 python profiles/fused_time.py 32 96 256 2>&1 | grep "spans" | awk 'NR%83==0' >> gpurun_out/r02l_ab.txt
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti > gpurun_out/r02l_layers_c2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_network.py -q -x 2>&1 | tail -15 >> gpurun_out/r02l_tests.txt
cat gpurun_out/r02l_tests.txt gpurun_out/r02l_ab.txt; tail -3 gpurun_out/r02l_layers_c2.txt
