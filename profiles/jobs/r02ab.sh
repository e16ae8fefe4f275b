#!/bin/bash
# r02ab: evidence on the current code: map backend sweep (GB/s), bench lines (C2 with CPU baseline, C1/C3/C4/C5),
# ncu launch list of one steady C2 forward, ncu full capture of two fused convs, sanitizers
mkdir -p gpurun_out /tmp/ncu
timeout 900 python profiles/map_backends.py > gpurun_out/r02ab_map_backends.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ab_bench_c2.json 2> gpurun_out/r02ab_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02ab_bench_$w.json 2>/dev/null
done
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ab_bench_c5.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --launch-skip 240 --launch-count 120 --log-file gpurun_out/r02ab_launches_c2.csv python profiles/run_net.py c2_minkunet42_kitti --forwards 3 --dataflow auto > gpurun_out/r02ab_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_conv_fused" --launch-skip 51 --launch-count 3 \
  -o /tmp/ncu/fused -f python profiles/run_net.py c2_minkunet42_kitti --forwards 2 --dataflow fused > gpurun_out/r02ab_ncu_full.log 2>&1
ncu -i /tmp/ncu/fused.ncu-rep --page raw --csv > gpurun_out/r02ab_fused_raw.csv 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check full --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02ab_san_memcheck.log 2>&1
timeout 900 $CS --tool racecheck --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02ab_san_racecheck.log 2>&1
timeout 900 $CS --tool synccheck --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02ab_san_synccheck.log 2>&1
timeout 900 $CS --tool initcheck --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02ab_san_initcheck.log 2>&1
cat gpurun_out/r02ab_map_backends.txt | cut -c1-400; for f in gpurun_out/r02ab_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY" gpurun_out/r02ab_san_*.log; tail -2 gpurun_out/r02ab_ncu_full.log
