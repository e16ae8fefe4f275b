#!/bin/bash
# r02az: Eq. 1 radix with 10-bit digits (3 passes for the KITTI levels) vs 8-bit, same box
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py tests/test_gpu_spec_api.py -q -x 2>&1 | tail -3
for i in 1 2; do
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do
  tag=$(basename $(dirname $lib)); SCONV_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02az_c2_${tag}_$i.json 2>/dev/null
done; done
for lib in ab/libsconv_prev.so paper_2401_06145_b200/libsconv_b200.so; do tag=$(basename $(dirname $lib))
  SCONV_LIB=$lib timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02az_c3_${tag}.json 2>/dev/null
  SCONV_LIB=$lib timeout 300 python bench.py --workload c4_unet_pair_shapenet --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02az_c4_${tag}.json 2>/dev/null
done
for f in gpurun_out/r02az_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
