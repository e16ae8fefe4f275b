#!/bin/bash
# r02bc: stage waits by non-suspending mbarrier.test_wait polling (producers' free-stage and MMA's full-stage waits)
mkdir -p gpurun_out
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  for d in 0 290; do echo "== $lib debug $d"; SCONV_LIB=$lib SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done
  SCONV_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | grep -o 'ms_per_step": [0-9.]*'
done > gpurun_out/r02bc.txt 2>&1
cat gpurun_out/r02bc.txt
