mkdir -p gpurun_out
export CFG=sweep SEED_CTA_TRACE=1
timeout 300 python scripts/trace_round.py > gpurun_out/t8_sw.log 2>&1; echo trace=$?
SEED_ATTN_CLUSTER=0 timeout 300 python scripts/trace_round.py > gpurun_out/t8_sw_nocl.log 2>&1; echo trace=$?
