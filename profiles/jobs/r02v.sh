#!/bin/bash
# r02v: deferred raw-input flag check + deferred map frees: full GPU suite, C2/C3 bench, C2 timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/r02v_tests.log
B="timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02v_bench_c2.json 2>gpurun_out/r02v_bench_c2.err
$B --workload c3_resnet21d_s3dis > gpurun_out/r02v_bench_c3.json 2>/dev/null
$B --workload c4_unet_pair_shapenet > gpurun_out/r02v_bench_c4.json 2>/dev/null
$B --workload c1_layer_100k > gpurun_out/r02v_bench_c1.json 2>/dev/null
SCONV_NET_HOST_PROFILE=1 timeout 300 python profiles/timeline.py --forwards 2 --json gpurun_out/r02v_tl_c2.json > gpurun_out/r02v_tl_c2.txt 2> gpurun_out/r02v_host.txt
cat gpurun_out/r02v_tests.log; for f in gpurun_out/r02v_bench_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
head -30 gpurun_out/r02v_tl_c2.txt
