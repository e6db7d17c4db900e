#!/bin/bash
# Evidence for profiles/: a plain run (must exit 0), the per-launch list of the bench command,
# per-launch DRAM bytes of every kernel of one round, and full captures of a verify GEMM and
# attention.  Summarise here with: python scripts/profile_summary.py gpurun_out/prof profiles/<round>
OUT=gpurun_out/prof
mkdir -p $OUT
ARGS="--steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python bench.py $ARGS > $OUT/plain.log 2>&1 || { echo plain failed; tail -20 $OUT/plain.log; exit 1; }
timeout 300 python scripts/ncu_round.py > $OUT/round_plain.log 2>&1 || { echo round plain failed; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $OUT/round_dram.csv python scripts/ncu_round.py > $OUT/ncu_dram.log 2>&1; echo dram=$?
# GEMM launches of a round: draft 4 steps x (2 layers x 4 + LM) = 36, then verify L0 (36-39), L1 QKV 40, O 41, GU 42
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk \
  -s 42 -c 1 -o $OUT/gemm_gu_l1 python scripts/ncu_round.py > $OUT/ncu_gemm.log 2>&1; echo gemm=$?
# attention launches: draft 4 x 2 = 8, verify L0 = 8, L1 = 9
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_fused \
  -s 9 -c 1 -o $OUT/attn_l1 python scripts/ncu_round.py > $OUT/ncu_attn.log 2>&1; echo attn=$?
# the same captures at N = 24 streams (sweep shape): the O projection (split-K over a 4-CTA cluster)
# and attention (single-buffer form)
CFG=sweep timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk \
  -s 41 -c 1 -o $OUT/gemm_o_l1_sweep python scripts/ncu_round.py > $OUT/ncu_gemm_sw.log 2>&1; echo gemm_sw=$?
CFG=sweep timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_fused \
  -s 9 -c 1 -o $OUT/attn_l1_sweep python scripts/ncu_round.py > $OUT/ncu_attn_sw.log 2>&1; echo attn_sw=$?
