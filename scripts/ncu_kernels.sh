#!/bin/bash
# full ncu captures of selected small kernels (one launch each, after warm-up)
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/plain.log; exit 1; }
for k in ${KERNELS:-vocab_verify residual_rmsnorm attn_chunk}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-20} -c 1 -o gpurun_out/prof_$k python bench.py $ARGS > gpurun_out/ncu_$k.log 2>&1; echo $k=$?
done
