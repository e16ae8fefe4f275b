#!/bin/bash
# r02bm: k_search_colp with the direct path for scattered chunks: parity subset, cpc sweep, map sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec_api.py -m gpu -q -x -k "map or search or acceptance or spec" 2>&1 | tail -3 > gpurun_out/r02bm_tests.log
for v in 0 1 2 4; do SCONV_SEARCH_CPC=$v timeout 300 python profiles/search_ab.py; done > gpurun_out/r02bm_search.txt 2>&1
SCONV_SEARCH_PERSIST=0 timeout 300 python profiles/search_ab.py >> gpurun_out/r02bm_search.txt 2>&1
SCONV_SEARCH_CPC=1 SCONV_SEARCH_TRACE=gpurun_out/r02bm_trace_cpc1.bin timeout 300 python profiles/search_ab.py s3dis >/dev/null 2>&1
SCONV_SEARCH_TRACE=gpurun_out/r02bm_trace_cpc0.bin timeout 300 python profiles/search_ab.py s3dis >/dev/null 2>&1
timeout 600 python profiles/map_backends.py > gpurun_out/r02bm_map.txt 2>&1
cat gpurun_out/r02bm_tests.log gpurun_out/r02bm_search.txt; cut -c1-150 gpurun_out/r02bm_map.txt
