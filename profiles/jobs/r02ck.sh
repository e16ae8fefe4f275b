#!/bin/bash
# r02ck: final check at HEAD: GPU suite, smoke(), default bench line (the driver's command)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r02ck_bench_default.json 2> gpurun_out/r02ck_bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/r02ck_bench_default.json')); e=d['e2e']; print('default', d['config']['workload'], round(d['ms_per_step'],3), 'e2e ms', round(e['ms'],3), '%.3g'%e['value'], d['clocks'], d['gpu_launches'])"
