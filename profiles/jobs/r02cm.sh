#!/bin/bash
# r02cm: async readback chunk size 256 KB / 512 KB / 1 MB (same box, alternating): C2 e2e
mkdir -p gpurun_out
for i in 1 2 3; do
  for kb in 256 512 1024; do
    SCONV_RB_CHUNK_KB=$kb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cm_c2_${kb}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/r02cm_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
