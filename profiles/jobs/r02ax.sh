#!/bin/bash
# r02ax: sector-coalesced 16-bit epilogue (SCONV_FUSED_COAL) vs the row-per-lane epilogue, same box
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -q -x 2>&1 | tail -3
for c in 1 0; do echo "== COAL $c"; SCONV_FUSED_COAL=$c timeout 120 python profiles/fused_time.py 32 96 256; done > gpurun_out/r02ax.txt 2>&1
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02ax_c2_coal_$i.json 2>/dev/null
SCONV_FUSED_COAL=0 $B > gpurun_out/r02ax_c2_nocoal_$i.json 2>/dev/null
done
$B --workload c3_resnet21d_s3dis > gpurun_out/r02ax_c3_coal.json 2>/dev/null
SCONV_FUSED_COAL=0 $B --workload c3_resnet21d_s3dis > gpurun_out/r02ax_c3_nocoal.json 2>/dev/null
timeout 300 python profiles/net_layers.py > gpurun_out/r02ax_layers_coal.txt 2>&1
SCONV_FUSED_COAL=0 timeout 300 python profiles/net_layers.py > gpurun_out/r02ax_layers_nocoal.txt 2>&1
cat gpurun_out/r02ax.txt; for f in gpurun_out/r02ax_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
tail -n1 gpurun_out/r02ax_layers_*.txt
