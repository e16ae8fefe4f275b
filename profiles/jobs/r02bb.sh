#!/bin/bash
# r02bb: column search at 3 CTAs/SM (72 regs, small spill) vs 2 (96 regs): map sweep + C2/C3 bench, same box
mkdir -p gpurun_out
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  echo "== $lib"; SCONV_LIB=$lib timeout 600 python profiles/map_backends.py 2>&1 | cut -c1-120
  for w in c2_minkunet42_kitti c3_resnet21d_s3dis; do
    SCONV_LIB=$lib timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | grep -o 'ms_per_step": [0-9.]*'
  done
done > gpurun_out/r02bb.txt 2>&1
cat gpurun_out/r02bb.txt
