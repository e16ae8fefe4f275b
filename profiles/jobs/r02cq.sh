#!/bin/bash
# r02cq: serving loop with / without input prefetch (same box, alternating): C3 / C4 / C5 e2e
mkdir -p gpurun_out
for i in 1 2; do
  for p in 0 1; do
    for w in c3_resnet21d_s3dis c4_unet_pair_shapenet; do
      BENCH_E2E_PREFETCH=$p timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02cq_${w}_p${p}_$i.json 2>/dev/null
    done
  done
done
for p in 0 1; do
  BENCH_E2E_PREFETCH=$p timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cq_c5_p$p.json 2>/dev/null
done
for f in gpurun_out/r02cq_*.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e']; print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3))"; done
