#!/bin/bash
# r02w: per-kernel totals of a C2 forward (all streams); ncu full of the map kernels (k_search, k_mask_sort, k_floor_unique)
mkdir -p gpurun_out /tmp/ncu
timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02w_tl_c2.json > gpurun_out/r02w_tl_c2.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_search|k_mask_sort|k_floor_unique" --launch-skip 29 --launch-count 29 \
  -o /tmp/ncu/map -f python profiles/run_net.py c2_minkunet42_kitti --forwards 2 > gpurun_out/r02w_ncu.log 2>&1
ncu -i /tmp/ncu/map.ncu-rep --page raw --csv > gpurun_out/r02w_map_raw.csv 2>&1
ncu -i /tmp/ncu/map.ncu-rep --page details --csv > gpurun_out/r02w_map_details.csv 2>&1
cp /tmp/ncu/map.ncu-rep gpurun_out/r02w_map.ncu-rep
sed -n '/kernel totals/,/timeline of/p' gpurun_out/r02w_tl_c2.txt; tail -3 gpurun_out/r02w_ncu.log; ls -la gpurun_out/r02w_map*
