#!/bin/bash
# r02ad: source-level hot spots of the fused conv: 96->96 level-0 conv (op 63) and 32->32 level-1 conv (op 3)
mkdir -p gpurun_out /tmp/ncu
for spec in "94 op63" "52 op3"; do set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_conv_(fused|items)" --launch-skip $1 --launch-count 1 \
    -o /tmp/ncu/$2 -f python profiles/run_net.py c2_minkunet42_kitti --forwards 2 --dataflow fused > gpurun_out/r02ad_$2.log 2>&1
  ncu -i /tmp/ncu/$2.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ad_$2_sass.csv 2>&1
  ncu -i /tmp/ncu/$2.ncu-rep --page raw --csv > gpurun_out/r02ad_$2_raw.csv 2>&1
  ncu -i /tmp/ncu/$2.ncu-rep --page details --csv > gpurun_out/r02ad_$2_details.csv 2>&1
done
ls -la gpurun_out/r02ad_*; head -3 gpurun_out/r02ad_op63_sass.csv | cut -c1-300
