#!/bin/bash
# bench ms/round for each value of an env var: sweep_env.sh VAR v1 v2 ...
mkdir -p gpurun_out
var=$1; shift
for v in "$@"; do
  env $var=$v timeout ${BENCH_TIMEOUT:-240} python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$v.log 2>&1
  echo "$var=$v rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sweep_$v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/sweep_$v.log)"
done
