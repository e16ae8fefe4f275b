#!/bin/bash
# r02bn: k_search_colp (4-ary direct path, binary first query, size rule): parity, sweep, network A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec_api.py -m gpu -q -x -k "map or search or acceptance or spec" 2>&1 | tail -2 > gpurun_out/r02bn_tests.log
for v in 0 1; do SCONV_SEARCH_CPC=$v timeout 300 python profiles/search_ab.py; done > gpurun_out/r02bn_search.txt 2>&1
SCONV_SEARCH_CPC=2000000 timeout 300 python profiles/search_ab.py u1e6 >> gpurun_out/r02bn_search.txt 2>&1
SCONV_SEARCH_PERSIST=0 timeout 300 python profiles/search_ab.py >> gpurun_out/r02bn_search.txt 2>&1
timeout 600 python profiles/map_backends.py > gpurun_out/r02bn_map.txt 2>&1
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bn_c2_new$i.json 2>/dev/null
  SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bn_c2_old$i.json 2>/dev/null
  timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bn_c3_new$i.json 2>/dev/null
  SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bn_c3_old$i.json 2>/dev/null
done
cat gpurun_out/r02bn_tests.log gpurun_out/r02bn_search.txt; cut -c1-150 gpurun_out/r02bn_map.txt
for f in gpurun_out/r02bn_c*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
