#!/bin/bash
# plain run first (must exit 0), then the launch list and one full capture of the GEMM
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_splitk -s ${SKIP:-1300} -c 3 -o gpurun_out/gemm_prof python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo full=$?
tail -3 gpurun_out/ncu_full.log
