mkdir -p gpurun_out
export CFG=sweep
timeout 120 python scripts/ncu_round.py > gpurun_out/r.log 2>&1 || { echo plain failed; tail gpurun_out/r.log; exit 1; }
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk -s 42 -c 1 -o gpurun_out/sw_gu python scripts/ncu_round.py > gpurun_out/ncu_gu.log 2>&1; echo gu=$?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk -s 41 -c 1 -o gpurun_out/sw_o python scripts/ncu_round.py > gpurun_out/ncu_o.log 2>&1; echo o=$?
tail -3 gpurun_out/ncu_o.log
