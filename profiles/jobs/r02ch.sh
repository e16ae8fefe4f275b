#!/bin/bash
# r02ch: async readback one copy vs 2 MB / 8 MB chunks (same box, alternating): C2 / C3 e2e
mkdir -p gpurun_out
for i in 1 2; do
  for kb in none 2048 8192; do
    for w in c2_minkunet42_kitti c3_resnet21d_s3dis; do
      if [ $kb = none ]; then unset SCONV_RB_CHUNK_KB; else export SCONV_RB_CHUNK_KB=$kb; fi
      timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ch_${w}_${kb}_$i.json 2>/dev/null
    done
  done
done
unset SCONV_RB_CHUNK_KB
for f in gpurun_out/r02ch_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
