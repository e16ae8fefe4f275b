#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -q -x --deselect tests/test_gpu_fullsize.py 2>&1 | tail -40 > gpurun_out/r02c_tests.log
tail -30 gpurun_out/r02c_tests.log
