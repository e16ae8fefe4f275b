#!/bin/bash
# r02e: first GPU call of the round: SPEC-API + parity suites, full-size parity, bench C2/C5, reference arm
mkdir -p gpurun_out
nproc > gpurun_out/r02e_cpu.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/r02e_cpu.txt
timeout 1200 python -m pytest tests/test_gpu_spec_api.py tests/test_adapter.py tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -40 > gpurun_out/r02e_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | tail -60 > gpurun_out/r02e_fullsize.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e_bench_c2.json 2> gpurun_out/r02e_bench_c2.err
timeout 600 python bench.py --workload c5_minkunet42_batch64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_c5.json 2> gpurun_out/r02e_bench_c5.err
( time timeout 900 python bench.py --impl reference --steps 2 --warmup 0 ) > gpurun_out/r02e_ref_c2.json 2> gpurun_out/r02e_ref_c2.err
tail -5 gpurun_out/r02e_tests.log; tail -15 gpurun_out/r02e_fullsize.log; cat gpurun_out/r02e_bench_c2.json gpurun_out/r02e_bench_c5.json gpurun_out/r02e_ref_c2.json | cut -c1-400
