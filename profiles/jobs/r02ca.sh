#!/bin/bash
# r02ca: evidence refresh at HEAD after the session restart (column search with cursor, network schedule):
# GPU suite, bench lines C1-C5, reference arm, launch list, ncu full of the fused convs, per-conv tables, sanitizers
mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r02ca_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ca_bench_c2.json 2> gpurun_out/r02ca_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02ca_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ca_bench_c5.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02ca_ref_c2.json 2> gpurun_out/r02ca_ref_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02ca_launches_c2.csv python profiles/run_net.py c2_minkunet42_kitti --forwards 3 --dataflow fused > gpurun_out/r02ca_launches.log 2>&1
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti --json gpurun_out/r02ca_layers_c2.json > gpurun_out/r02ca_layers_c2.txt 2>&1
timeout 300 python profiles/timeline.py --forwards 2 > gpurun_out/r02ca_timeline_c2.txt 2>&1
cat gpurun_out/r02ca_tests.log; for f in gpurun_out/r02ca_bench_*.json gpurun_out/r02ca_ref_c2.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
tail -n1 gpurun_out/r02ca_layers_*.txt
