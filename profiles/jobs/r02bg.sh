#!/bin/bash
# r02bg: ncu full (source-level) of the column search on the KITTI and S3DIS level-0 maps
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_search" --launch-count 2 \
  -o /tmp/ncu/search -f python profiles/map_backends.py --ncu > gpurun_out/r02bg_ncu.log 2>&1
ncu -i /tmp/ncu/search.ncu-rep --page raw --csv > gpurun_out/r02bg_search_raw.csv 2>&1
ncu -i /tmp/ncu/search.ncu-rep --page source --csv --print-source sass > gpurun_out/r02bg_search_src.csv 2>&1
ncu -i /tmp/ncu/search.ncu-rep --page details > gpurun_out/r02bg_search_details.txt 2>&1
tail -3 gpurun_out/r02bg_ncu.log; wc -l gpurun_out/r02bg_search_*
