#!/bin/bash
# r02bj: ncu of k_search_colp on the S3DIS cloud, 1 vs 2 chunks per CTA, and k_search_col
mkdir -p gpurun_out /tmp/ncu
for v in 1 2; do
  SCONV_SEARCH_CPC=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_search" --launch-skip 1 --launch-count 1 \
    -o /tmp/ncu/colp_cpc$v -f python profiles/search_ab.py s3dis > gpurun_out/r02bj_ncu_$v.log 2>&1
  ncu -i /tmp/ncu/colp_cpc$v.ncu-rep --page details > gpurun_out/r02bj_details_cpc$v.txt 2>&1
  ncu -i /tmp/ncu/colp_cpc$v.ncu-rep --page source --csv --print-source sass > gpurun_out/r02bj_src_cpc$v.csv 2>&1
done
SCONV_SEARCH_PERSIST=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_search" --launch-skip 1 --launch-count 1 \
    -o /tmp/ncu/col -f python profiles/search_ab.py s3dis > gpurun_out/r02bj_ncu_col.log 2>&1
ncu -i /tmp/ncu/col.ncu-rep --page details > gpurun_out/r02bj_details_col.txt 2>&1
ncu -i /tmp/ncu/col.ncu-rep --page source --csv --print-source sass > gpurun_out/r02bj_src_col.csv 2>&1
grep -h "Duration\|Issue Slots Busy\|Executed Ipc A\|No Eligible" gpurun_out/r02bj_details_*.txt
