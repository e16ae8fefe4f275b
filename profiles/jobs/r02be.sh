#!/bin/bash
# r02be: bucket-histogram scan with consecutive buckets per thread; C1 (unsorted input) A/B + map parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "map or c1 or sort or spec or acceptance" 2>&1 | tail -2
for i in 1 2; do for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  echo "$lib $(SCONV_LIB=$lib timeout 300 python bench.py --workload c1_layer_100k --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | grep -o 'ms_per_step": [0-9.]*')"
done; done
