#!/bin/bash
# r02r: compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel family;
# GMaS grouped-GEMM tensor-pipe capture on the widest MinkUNet42 layers; steady-state launch list of one forward
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $tool $extra --print-limit 20 python profiles/sanitize_run.py > gpurun_out/r02r_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02r_san_$tool.log
done
timeout 900 $CS --tool memcheck --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02r_san_memcheck_net.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_san_memcheck_net.log
timeout 900 $CS --tool racecheck --print-limit 20 python profiles/sanitize_run.py --net > gpurun_out/r02r_san_racecheck_net.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_san_racecheck_net.log
# GMaS: every grouped GEMM of the second forward (49 convs), tensor pipe + SOL
timeout 900 ncu --clock-control none --kernel-name regex:k_gemm_grouped --launch-skip 49 --launch-count 49 \
  --section SpeedOfLight --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy \
  --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --page raw python profiles/run_net.py c2_minkunet42_kitti --dataflow gmas > gpurun_out/r02r_gemm_raw.csv 2> gpurun_out/r02r_gemm.err
# steady-state launch list: the 3rd fused-only forward
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/r02r_launches_fwd.csv python profiles/run_net.py c2_minkunet42_kitti --forwards 3 > gpurun_out/r02r_launches.log 2>&1
grep -h "ERROR SUMMARY\|rc=" gpurun_out/r02r_san_*.log; wc -l gpurun_out/r02r_gemm_raw.csv gpurun_out/r02r_launches_fwd.csv
