cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/r01p_bench.json 2> gpurun_out/r01p_bench.err
for w in c1_layer_100k c3_resnet21d_s3dis c4_unet_pair_shapenet; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r01p_bench_$w.json 2>> gpurun_out/r01p_bench.err
done
