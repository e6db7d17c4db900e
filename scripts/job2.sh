mkdir -p gpurun_out
CFG=sweep SEED_CTA_TRACE=1 timeout 300 python scripts/trace_round.py > gpurun_out/trace_sweep_cta.log 2>&1; echo trace=$?
