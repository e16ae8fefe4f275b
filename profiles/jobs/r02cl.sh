#!/bin/bash
# r02cl: async readback chunk size 1 / 2 / 4 MB (same box, alternating): C2 / C5 e2e
mkdir -p gpurun_out
for i in 1 2 3; do
  for kb in 1024 2048 4096; do
    SCONV_RB_CHUNK_KB=$kb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cl_c2_${kb}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/r02cl_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
