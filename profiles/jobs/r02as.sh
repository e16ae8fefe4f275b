#!/bin/bash
# r02as: producers wait for a free stage with one poller per warp (lane 0 + __syncwarp) vs every thread
mkdir -p gpurun_out
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  for d in 0 263; do echo "== $lib debug $d"; SCONV_LIB=$lib SCONV_FUSED_DEBUG=$d timeout 120 python profiles/fused_time.py 32 96 256; done
done > gpurun_out/r02as.txt 2>&1
for i in 1 2; do
SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02as_c2_prev_$i.json 2>/dev/null
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02as_c2_new_$i.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" 2>&1 | tail -2
cat gpurun_out/r02as.txt; for f in gpurun_out/r02as_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
