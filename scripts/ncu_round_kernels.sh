#!/bin/bash
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 290 -c 1 -o gpurun_out/prof_attn python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1; echo attn=$?
ncu --set full --clock-control none --import-source on -k regex:residual_rmsnorm -s 520 -c 1 -o gpurun_out/prof_res python bench.py $ARGS > gpurun_out/ncu_res.log 2>&1; echo res=$?
