#!/bin/bash
# r02am: ncu of the column search on C3 (S3DIS room) and C2 (KITTI): full set + SASS hot spots of the largest launch
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_search_col" --launch-skip 8 --launch-count 8 \
  -o /tmp/ncu/search_c3 -f python profiles/run_net.py c3_resnet21d_s3dis --forwards 2 --dataflow fused > gpurun_out/r02am_c3.log 2>&1
ncu -i /tmp/ncu/search_c3.ncu-rep --page raw --csv > gpurun_out/r02am_search_c3_raw.csv 2>&1
ncu -i /tmp/ncu/search_c3.ncu-rep --page source --csv --print-source sass --launch-count 1 > gpurun_out/r02am_search_c3_sass.csv 2>&1
python profiles/ncu_summary.py gpurun_out/r02am_search_c3_raw.csv | head -12
