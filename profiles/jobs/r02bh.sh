#!/bin/bash
# r02bh: persistent pipelined column search (k_search_colp): map parity tests, search A/B vs the
# one-CTA-per-chunk k_search_col, network A/B (same box) vs the previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec_api.py -m gpu -q -x -k "map or search or acceptance or spec" 2>&1 | tail -4 > gpurun_out/r02bh_tests.log
for v in 1 0; do SCONV_SEARCH_PERSIST=$v timeout 600 python profiles/map_backends.py > gpurun_out/r02bh_map_p$v.txt 2>&1; done
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bh_c2_new$i.json 2>/dev/null
  SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bh_c2_old$i.json 2>/dev/null
  timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bh_c3_new$i.json 2>/dev/null
  SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bh_c3_old$i.json 2>/dev/null
done
cat gpurun_out/r02bh_tests.log; cut -c1-175 gpurun_out/r02bh_map_p*.txt
for f in gpurun_out/r02bh_c*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
