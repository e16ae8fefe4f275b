#!/bin/bash
# r02cp: final evidence at HEAD (adaptive readback chunks): GPU suite, smoke, bench lines C1-C5, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r02cp_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cp_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02cp_bench_c2.json 2> gpurun_out/r02cp_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02cp_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02cp_bench_c5.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02cp_ref_c2.json 2> gpurun_out/r02cp_ref_c2.err
cat gpurun_out/r02cp_tests.log gpurun_out/r02cp_smoke.log
for f in gpurun_out/r02cp_bench_*.json gpurun_out/r02cp_ref_c2.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d.get('e2e',{}); cb=d.get('cpu_baseline') or {}; print('$f', round(d['ms_per_step'],3), '%.3g'%d['value'], 'e2e ms', round(e.get('ms',0),3), '%.3g'%e.get('value',0), 'lat', e.get('latency_ms'), 'cpu', cb.get('value'), d.get('clocks'))"; done
