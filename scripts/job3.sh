mkdir -p gpurun_out
for d in 1 2 4 6; do
SEED_EPI_DEBUG=$d CFG=sweep SEED_CTA_TRACE=1 timeout 300 python scripts/trace_round.py > gpurun_out/trace_dbg$d.log 2>&1; echo trace=$?
done
