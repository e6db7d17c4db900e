mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k merge_paths > gpurun_out/attn_test.log 2>&1; echo test=$?; tail -3 gpurun_out/attn_test.log
export SEED_CTA_TRACE=0
CFG=sweep timeout 300 python scripts/trace_round.py > gpurun_out/t12_sw.log 2>&1; echo trace=$?
for c in sweep cw bw; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-250; done
SEED_ATTN_SEQ=1 timeout 300 python bench.py --config cw --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cw1.log 2>&1; echo cw1=$?; tail -1 gpurun_out/bench_cw1.log | cut -c1-250
