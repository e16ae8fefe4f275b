#!/bin/bash
# r02o: work-item kernel at 2 CTAs/SM (96 regs), deterministic 8-offset row order: tests, A/B, spans, per-conv, bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or layer or c1 or determinism" 2>&1 | tail -5 > gpurun_out/r02o_tests.txt
timeout 600 python -m pytest tests/test_gpu_network.py -q -x 2>&1 | tail -15 >> gpurun_out/r02o_tests.txt
for v in 1 0; do echo "== V1=$v"; SCONV_FUSED_V1=$v timeout 60 python profiles/fused_time.py 32 96 128 256; done > gpurun_out/r02o_ab.txt 2>&1
SCONV_FUSED_DEBUG=8192 timeout 60 python profiles/fused_time.py 32 96 256 2>&1 | grep "spans\|k_conv_items" | awk 'NR%84<=1' >> gpurun_out/r02o_ab.txt
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti > gpurun_out/r02o_layers_c2.txt 2>&1
SCONV_FUSED_V1=1 timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti > gpurun_out/r02o_layers_c2_v1.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02o_bench.json 2>gpurun_out/r02o_bench.err
SCONV_FUSED_V1=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02o_bench_v1.json 2>>gpurun_out/r02o_bench.err
cat gpurun_out/r02o_tests.txt gpurun_out/r02o_ab.txt; tail -n 1 gpurun_out/r02o_layers_c2.txt gpurun_out/r02o_layers_c2_v1.txt; cut -c1-250 gpurun_out/r02o_bench.json gpurun_out/r02o_bench_v1.json
