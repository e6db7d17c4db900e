mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputests.log
CFG=sweep timeout 300 python scripts/trace_round.py > gpurun_out/t14_sw.log 2>&1; echo trace=$?
CFG=gsm8k timeout 300 python scripts/trace_round.py > gpurun_out/t14_gsm.log 2>&1; echo trace=$?
for c in sweep cw bw gsm8k; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-250; done
