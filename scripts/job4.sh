mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gputests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gsm.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_gsm.log | cut -c1-400
timeout 300 python bench.py --config sweep --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1; echo sweep=$?; tail -1 gpurun_out/bench_sweep.log | cut -c1-400
CFG=sweep SEED_CTA_TRACE=1 timeout 300 python scripts/trace_round.py > gpurun_out/trace_sweep_cta.log 2>&1; echo trace=$?
CFG=gsm8k SEED_CTA_TRACE=1 timeout 300 python scripts/trace_round.py > gpurun_out/trace_gsm_cta.log 2>&1; echo trace=$?
