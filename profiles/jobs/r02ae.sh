#!/bin/bash
# r02ae: bf16 network test, bench C2 roofline with resolved |M|, C2 bf16 line, timeline with derived maps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_network.py -q -x -k "bf16 or end_to_end" -s 2>&1 | grep -E "passed|failed|bf16|Error|assert" | head > gpurun_out/r02ae_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ae_bench_c2.json 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --dtype bf16 > gpurun_out/r02ae_bench_c2_bf16.json 2>/dev/null
timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02ae_tl_c2.json > gpurun_out/r02ae_tl_c2.txt 2>&1
cat gpurun_out/r02ae_tests.log; for f in gpurun_out/r02ae_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print(r['bound'], r['achieved'], r['unit'], r['frac'], {k:(v and round(v['frac'],3)) for k,v in r['bounds'].items()}, d['map_roofline'])"; done
sed -n '/kernel totals/,/timeline of/p' gpurun_out/r02ae_tl_c2.txt; grep "^forward" gpurun_out/r02ae_tl_c2.txt
