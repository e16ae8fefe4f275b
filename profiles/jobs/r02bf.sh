#!/bin/bash
# r02bf: final evidence refresh (after the coalesced epilogue): GPU suite, bench lines (C1-C5, reference arm), launch list, ncu full of the
# 49 fused convs, per-conv tables, map sweep, timeline, sanitizers
mkdir -p gpurun_out /tmp/ncu
nproc > gpurun_out/r02bf_host_cpu.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/r02bf_host_cpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r02bf_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bf_bench_c2.json 2> gpurun_out/r02bf_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02bf_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02bf_bench_c5.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02bf_ref_c2.json 2> gpurun_out/r02bf_ref_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02bf_launches_c2.csv python profiles/run_net.py c2_minkunet42_kitti --forwards 3 --dataflow fused > gpurun_out/r02bf_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_conv_(fused|items)" --launch-skip 49 --launch-count 49 \
  -o /tmp/ncu/fused -f python profiles/run_net.py c2_minkunet42_kitti --forwards 2 --dataflow fused > gpurun_out/r02bf_ncu.log 2>&1
ncu -i /tmp/ncu/fused.ncu-rep --page raw --csv > gpurun_out/r02bf_fused_raw.csv 2>&1
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti --json gpurun_out/r02bf_layers_c2.json > gpurun_out/r02bf_layers_c2.txt 2>&1
timeout 300 python profiles/net_layers.py --workload c3_resnet21d_s3dis --json gpurun_out/r02bf_layers_c3.json > gpurun_out/r02bf_layers_c3.txt 2>&1
timeout 900 python profiles/map_backends.py > gpurun_out/r02bf_map_backends.txt 2>&1
timeout 300 python profiles/timeline.py --forwards 2 > gpurun_out/r02bf_timeline_c2.txt 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $tool $extra --print-limit 10 python profiles/sanitize_run.py --net > gpurun_out/r02bf_san_$tool.log 2>&1
done
cat gpurun_out/r02bf_tests.log; for f in gpurun_out/r02bf_bench_*.json gpurun_out/r02bf_ref_c2.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
tail -n1 gpurun_out/r02bf_layers_*.txt; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY" gpurun_out/r02bf_san_*.log; cut -c1-200 gpurun_out/r02bf_map_backends.txt
