mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_gsm.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_gsm.log
timeout 300 python bench.py --config sweep --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sweep.log 2>&1; echo sweep=$?; tail -1 gpurun_out/bench_sweep.log
CFG=sweep timeout 300 python scripts/trace_round.py > gpurun_out/trace_sweep.log 2>&1; echo trace=$?
CFG=gsm8k timeout 300 python scripts/trace_round.py > gpurun_out/trace_gsm.log 2>&1; echo trace=$?
