#!/bin/bash
# r02bi: k_search_colp chunks-per-CTA sweep vs k_search_col
mkdir -p gpurun_out
for v in 0 1 2 3 4 8; do SCONV_SEARCH_CPC=$v timeout 300 python profiles/search_ab.py; done > gpurun_out/r02bi_search.txt 2>&1
SCONV_SEARCH_PERSIST=0 timeout 300 python profiles/search_ab.py >> gpurun_out/r02bi_search.txt 2>&1
cat gpurun_out/r02bi_search.txt
