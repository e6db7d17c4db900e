#!/bin/bash
# full ncu capture of GEMM launch number $1 (0-based, GEMMs only) of one round; output name $2
mkdir -p gpurun_out
timeout 120 python scripts/ncu_round.py > gpurun_out/ncu_round_plain.log 2>&1 || { echo plain failed; tail gpurun_out/ncu_round_plain.log; exit 1; }
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk -s $1 -c 1 -o gpurun_out/$2 python scripts/ncu_round.py > gpurun_out/ncu_$2.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$2.log
