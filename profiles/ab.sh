#!/bin/bash
# Same-box A/B: alternating bench runs of the previous build (ab/libsconv_prev.so) and the tree's
# build under the env settings given as arguments, e.g. ./profiles/ab.sh "SCONV_SMALL_PERMUTE=0" "SCONV_SMALL_PERMUTE=1"
for i in 1 2 3; do
  SCONV_LIB=ab/libsconv_prev.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prev', round(d['ms_per_step'],3))"
  for envs in "$@"; do
    env $envs timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', round(d['ms_per_step'],3))"
  done
done
