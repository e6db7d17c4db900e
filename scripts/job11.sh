mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ops.py -x -q -m gpu -k invariance > gpurun_out/inv.log 2>&1; echo inv=$?; tail -2 gpurun_out/inv.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_gsm.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_gsm.log | cut -c1-300
for c in sweep cw bw; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-250; done
