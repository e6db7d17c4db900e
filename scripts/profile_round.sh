#!/bin/bash
# Evidence for profiles/: plain run, per-launch list, full captures of the verify GEMM and attention.
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
# prefill uses ~2 x 4 x 32 target GEMMs per stream chunk; skip well into the rounds
ncu --set full --clock-control none --import-source on -k regex:gemm_streamk -s ${GSKIP:-1500} -c 4 -o gpurun_out/prof_gemm python bench.py $ARGS > gpurun_out/ncu_gemm.log 2>&1; echo gemm=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:attn_fused_kernel<.int.128>" -s 230 -c 1 -o gpurun_out/prof_attn python bench.py $ARGS > gpurun_out/ncu_attn.log 2>&1; echo attn=$?
