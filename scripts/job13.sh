mkdir -p gpurun_out
for c in sweep cw bw gsm8k; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-250; done
SEED_ATTN_CLUSTER=1 timeout 300 python bench.py --config cw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cw1.log 2>&1; echo cw1=$?; tail -1 gpurun_out/bench_cw1.log | cut -c1-250
SEED_ATTN_CLUSTER=0 timeout 300 python bench.py --config gsm8k --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g0.log 2>&1; echo g0=$?; tail -1 gpurun_out/bench_g0.log | cut -c1-250
export CFG=sweep
timeout 120 python scripts/ncu_round.py > gpurun_out/r.log 2>&1 || { echo plain failed; tail gpurun_out/r.log; exit 1; }
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_fused -s 9 -c 1 -o gpurun_out/sw_attn python scripts/ncu_round.py > gpurun_out/ncu_attn.log 2>&1; echo attn=$?
