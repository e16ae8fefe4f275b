#!/bin/bash
# r02ah: neighbour-mask bits of the fused row order (one-launch sort, 8/16/24 bits) on one box
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" 2>&1 | tail -2
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do for b in 24 16 8; do
SCONV_MASK_BITS=$b $B > gpurun_out/r02ah_c2_bits${b}_$i.json 2>/dev/null
done; done
for b in 24 16; do SCONV_MASK_BITS=$b $B --workload c3_resnet21d_s3dis > gpurun_out/r02ah_c3_bits$b.json 2>/dev/null; done
for f in gpurun_out/r02ah_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
