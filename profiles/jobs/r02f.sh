#!/bin/bash
# r02f: per-conv roofline tables (C2, C3) + ncu --set full of every fused conv of one C2 forward
# (the report stays on the box; raw CSV comes back)
mkdir -p gpurun_out /tmp/ncu
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti --json gpurun_out/r02f_layers_c2.json > gpurun_out/r02f_layers_c2.txt 2>&1
timeout 300 python profiles/net_layers.py --workload c3_resnet21d_s3dis --json gpurun_out/r02f_layers_c3.json > gpurun_out/r02f_layers_c3.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name k_conv_fused --launch-skip 49 --launch-count 49 \
  -o /tmp/ncu/fused -f python profiles/run_net.py c2_minkunet42_kitti > gpurun_out/r02f_ncu.log 2>&1
ncu -i /tmp/ncu/fused.ncu-rep --page raw --csv > gpurun_out/r02f_fused_raw.csv 2>&1
ls -la /tmp/ncu gpurun_out | tail -5; tail -n 3 gpurun_out/r02f_ncu.log; tail -n 3 gpurun_out/r02f_layers_c2.txt gpurun_out/r02f_layers_c3.txt
