#!/bin/bash
# full ncu capture of launch $2 (0-based) of kernels matching regex $1 in one round; output name $3
mkdir -p gpurun_out
timeout 120 python scripts/ncu_round.py > gpurun_out/ncu_round_plain.log 2>&1 || { echo plain failed; tail gpurun_out/ncu_round_plain.log; exit 1; }
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/$3 python scripts/ncu_round.py > gpurun_out/ncu_$3.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_$3.log
