#!/bin/bash
# r02bl: per-(chunk, column) timing trace of k_search_colp on the S3DIS cloud
mkdir -p gpurun_out
for v in 1 2; do SCONV_SEARCH_CPC=$v SCONV_SEARCH_TRACE=gpurun_out/r02bl_trace_cpc$v.bin timeout 300 python profiles/search_ab.py s3dis; done
SCONV_SEARCH_TRACE=gpurun_out/r02bl_trace_kitti.bin SCONV_SEARCH_CPC=2 timeout 300 python profiles/search_ab.py kitti
ls -la gpurun_out/r02bl*
