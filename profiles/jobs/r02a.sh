#!/bin/bash
# r02a: full-size parity (C2/C3/C4/C5), bench C2 + C5 at N=1, reference-arm timing on the box's host
set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread" > gpurun_out/r02a_cpu.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | tail -40 > gpurun_out/r02a_fullsize.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_c5.json 2> gpurun_out/r02a_bench_c5.err
( time timeout 900 python bench.py --impl reference --steps 2 --warmup 0 ) > gpurun_out/r02a_ref_c2.json 2> gpurun_out/r02a_ref_c2.err
( time timeout 900 python bench.py --impl reference --steps 1 --warmup 0 --workload c3_resnet21d_s3dis ) > gpurun_out/r02a_ref_c3.json 2> gpurun_out/r02a_ref_c3.err
tail -5 gpurun_out/r02a_fullsize.log; cat gpurun_out/r02a_bench_c2.json gpurun_out/r02a_bench_c5.json | cut -c1-600
