#!/bin/bash
# r02ci: evidence at the serving-path commit: GPU suite, bench lines C1-C5 (with cpu_baseline), reference arm,
# sanitizers (memcheck incl. the serving loop, synccheck, initcheck), launch list, per-conv table, timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r02ci_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ci_bench_c2.json 2> gpurun_out/r02ci_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02ci_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ci_bench_c5.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02ci_ref_c2.json 2> gpurun_out/r02ci_ref_c2.err
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $tool $extra --print-limit 10 python profiles/sanitize_run.py --net > gpurun_out/r02ci_san_$tool.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02ci_launches_c2.csv python profiles/run_net.py c2_minkunet42_kitti --forwards 3 --dataflow fused > gpurun_out/r02ci_launches.log 2>&1
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti --json gpurun_out/r02ci_layers_c2.json > gpurun_out/r02ci_layers_c2.txt 2>&1
python profiles/e2e_probe.py c2_minkunet42_kitti > gpurun_out/r02ci_probe_c2.txt 2>&1
cat gpurun_out/r02ci_tests.log
for f in gpurun_out/r02ci_bench_*.json gpurun_out/r02ci_ref_c2.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d.get('e2e',{}); print('$f', round(d['ms_per_step'],3), 'e2e ms', round(e.get('ms',0),3), '%.3g'%e.get('value',0))"; done
grep -h "ERROR SUMMARY\|LEAK SUMMARY\|sanitize run ok" gpurun_out/r02ci_san_*.log; tail -n1 gpurun_out/r02ci_layers_c2.txt
