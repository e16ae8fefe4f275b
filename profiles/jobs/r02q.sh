#!/bin/bash
# r02q: re-entry baseline of HEAD (fused v2 work-item kernel): full GPU suite, bench C2 (+V1 A/B), C1/C3/C4 lines,
# per-conv tables, ncu launch list of bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r02q_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r02q_bench_c2.json 2> gpurun_out/r02q_bench_c2.err
SCONV_FUSED_V1=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02q_bench_c2_v1.json 2>> gpurun_out/r02q_bench_c2.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02q_bench_$w.json 2> gpurun_out/r02q_bench_$w.err
done
timeout 300 python profiles/net_layers.py --workload c2_minkunet42_kitti --json gpurun_out/r02q_layers_c2.json > gpurun_out/r02q_layers_c2.txt 2>&1
timeout 300 python profiles/net_layers.py --workload c3_resnet21d_s3dis --json gpurun_out/r02q_layers_c3.json > gpurun_out/r02q_layers_c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r02q_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02q_ncu_bench.log 2>&1
tail -5 gpurun_out/r02q_tests.log; for f in gpurun_out/r02q_bench_*.json; do echo $f; cut -c1-300 $f; done; tail -n 2 gpurun_out/r02q_layers_c2.txt gpurun_out/r02q_layers_c3.txt
