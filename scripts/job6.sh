mkdir -p gpurun_out
export CFG=sweep SEED_CTA_TRACE=1
SEED_GEMM_VERBOSE=1 timeout 300 python scripts/trace_round.py > gpurun_out/t6_0.log 2>&1; echo trace=$?
SEED_EPI_DEBUG=1 timeout 300 python scripts/trace_round.py > gpurun_out/t6_1.log 2>&1; echo trace=$?
SEED_EPI_DEBUG=2 timeout 300 python scripts/trace_round.py > gpurun_out/t6_2.log 2>&1; echo trace=$?
