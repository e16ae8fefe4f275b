#!/bin/bash
# r02au: per-warp aggregated stage arrivals (4 arrives per stage instead of 128 noinc arrives) vs previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -3
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  for d in 0 263; do echo "== $lib debug $d"; SCONV_LIB=$lib SCONV_FUSED_DEBUG=$d timeout 120 python profiles/fused_time.py 32 96 256; done
done > gpurun_out/r02au.txt 2>&1
for i in 1 2; do
SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02au_c2_prev_$i.json 2>/dev/null
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02au_c2_new_$i.json 2>/dev/null
done
SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02au_c3_prev.json 2>/dev/null
timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02au_c3_new.json 2>/dev/null
cat gpurun_out/r02au.txt; for f in gpurun_out/r02au_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
