#!/bin/bash
# Evidence for profiles/ (round 2, the bench's default sweep-24 config): a plain bench run (must exit 0),
# the per-launch list of the bench command, per-launch DRAM bytes of every kernel of one round, and
# full captures of the verify GEMMs / attention of layer 1, K4 and K1.  Summarise here with:
#   CFG=sweep python scripts/profile_summary.py gpurun_out/prof profiles/r02
OUT=gpurun_out/prof
mkdir -p $OUT
export CFG=${CFG:-sweep}
ARGS="--config $CFG --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py $ARGS > $OUT/plain.log 2>&1 || { echo plain failed; tail -20 $OUT/plain.log; exit 1; }
timeout 300 python scripts/ncu_round.py > $OUT/round_plain.log 2>&1 || { echo round plain failed; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $OUT/round_dram.csv python scripts/ncu_round.py > $OUT/ncu_dram.log 2>&1; echo dram=$?
# GEMM launches of a round: draft 4 steps x (2 layers x 4 + LM) = 36, then verify L0 (36-39), L1 QKV 40, O 41, GU 42
for v in "40 gemm_qkv_l1" "41 gemm_o_l1" "42 gemm_gu_l1"; do
  set -- $v
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_splitk \
    -s $1 -c 1 -o $OUT/$2 python scripts/ncu_round.py > $OUT/ncu_$2.log 2>&1; echo $2=$?
done
# attention launches: draft 4 x 2 = 8, verify L0 = 8, L1 = 9
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_stream \
  -s 9 -c 1 -o $OUT/attn_l1 python scripts/ncu_round.py > $OUT/ncu_attn.log 2>&1; echo attn=$?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:vocab_verify \
  -s 0 -c 1 -o $OUT/k4 python scripts/ncu_round.py > $OUT/ncu_k4.log 2>&1; echo k4=$?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:draft_sample \
  -s 1 -c 1 -o $OUT/k1 python scripts/ncu_round.py > $OUT/ncu_k1.log 2>&1; echo k1=$?
