#!/bin/bash
# r02ap: n-block split target of the tile-queue kernel (SCONV_FUSED_TILES: tiles wanted before halving block_n)
mkdir -p gpurun_out
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
for i in 1 2; do
$B > gpurun_out/r02ap_c2_default_$i.json 2>/dev/null
SCONV_FUSED_TILES=296 $B > gpurun_out/r02ap_c2_t296_$i.json 2>/dev/null
SCONV_FUSED_TILES=600 $B > gpurun_out/r02ap_c2_t600_$i.json 2>/dev/null
done
$B --workload c3_resnet21d_s3dis > gpurun_out/r02ap_c3_default.json 2>/dev/null
SCONV_FUSED_TILES=296 $B --workload c3_resnet21d_s3dis > gpurun_out/r02ap_c3_t296.json 2>/dev/null
SCONV_FUSED_TILES=296 timeout 300 python profiles/net_layers.py > gpurun_out/r02ap_layers_t296.txt 2>&1
timeout 300 python profiles/net_layers.py > gpurun_out/r02ap_layers_default.txt 2>&1
for f in gpurun_out/r02ap_*.json; do echo "$f $(grep -o 'ms_per_step": [0-9.]*' $f)"; done
tail -n1 gpurun_out/r02ap_layers_*.txt
