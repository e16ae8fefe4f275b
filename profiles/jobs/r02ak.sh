#!/bin/bash
# r02ak: row-order key width from the graph's map use counts; full GPU suite; same-box A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -12 > gpurun_out/r02ak_tests.log
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02ak_c2_default_$i.json 2>/dev/null
SCONV_MASK_BITS=24 $B > gpurun_out/r02ak_c2_bits24_$i.json 2>/dev/null
$B --workload c3_resnet21d_s3dis > gpurun_out/r02ak_c3_default_$i.json 2>/dev/null
SCONV_MASK_BITS=24 $B --workload c3_resnet21d_s3dis > gpurun_out/r02ak_c3_bits24_$i.json 2>/dev/null
done
cat gpurun_out/r02ak_tests.log; for f in gpurun_out/r02ak_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
