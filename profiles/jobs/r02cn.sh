#!/bin/bash
# r02cn: 512 KB readback chunks (new default) vs 2 MB on C3 / C4 / C5 e2e, and the default C2 line
mkdir -p gpurun_out
for i in 1 2; do
  for kb in 512 2048; do
    for w in c3_resnet21d_s3dis c4_unet_pair_shapenet; do
      SCONV_RB_CHUNK_KB=$kb timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cn_${w}_${kb}_$i.json 2>/dev/null
    done
  done
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cn_c5.json 2>/dev/null
timeout 600 python bench.py > gpurun_out/r02cn_bench_c2.json 2>/dev/null
for f in gpurun_out/r02cn_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
