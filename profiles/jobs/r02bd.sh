#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SCONV_PDL=0 timeout 600 $CS --tool racecheck --racecheck-report all --print-limit 6 python profiles/race_small.py 2000 32 > gpurun_out/r02bd_race.log 2>&1
SCONV_PDL=0 SCONV_FUSED_REG=0 timeout 600 $CS --tool racecheck --print-limit 3 python profiles/race_small.py 2000 32 > gpurun_out/r02bd_race_reg0.log 2>&1
head -60 gpurun_out/r02bd_race.log; grep "SUMMARY" gpurun_out/r02bd_race*.log
