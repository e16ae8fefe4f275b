#!/bin/bash
# r02b: SPEC-signature API, parity suites with the 8(c) metric, adapter
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_spec_api.py tests/test_adapter.py tests/test_gpu_parity.py tests/test_gpu_network.py -q -s -x 2>&1 | tail -60 > gpurun_out/r02b_tests.log
tail -30 gpurun_out/r02b_tests.log
