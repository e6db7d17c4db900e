#!/bin/bash
# full ncu capture of one kernel instantiation by demangled-name regex: ncu_one.sh <regex> <skip> <outname>
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s $2 -c 1 -o gpurun_out/$3 python bench.py $ARGS > gpurun_out/ncu_$3.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$3.log
