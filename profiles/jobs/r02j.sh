#!/bin/bash
# r02j: fused-kernel skeleton decomposition: which handshake costs what (debug bits, see FusedParams)
mkdir -p gpurun_out
for d in 0 7 1031 3079 7175 7431; do echo "== debug $d"; SCONV_FUSED_DEBUG=$d timeout 60 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02j.txt 2>&1
echo "== REG0" >> gpurun_out/r02j.txt; SCONV_FUSED_REG=0 timeout 60 python profiles/fused_time.py 32 96 256 >> gpurun_out/r02j.txt 2>&1; echo "rc=$?" >> gpurun_out/r02j.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" >> gpurun_out/r02j.txt 2>&1
cat gpurun_out/r02j.txt
