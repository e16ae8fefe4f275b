#!/bin/bash
# r02br/r02bs: look-ahead Eq. 1 deferral (SCONV_PRE_AFTER_CONV) A/B, same box; timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_network.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
  for p in 1 0; do
    SCONV_PRE_AFTER_CONV=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bs_c2_$p$i.json 2>/dev/null
    SCONV_PRE_AFTER_CONV=$p timeout 300 python bench.py --workload c3_resnet21d_s3dis --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02bs_c3_$p$i.json 2>/dev/null
  done
done
timeout 250 python profiles/timeline.py --forwards 2 > gpurun_out/r02bs_timeline.txt 2>&1
for f in gpurun_out/r02bs_c*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
head -12 gpurun_out/r02bs_timeline.txt
