#!/bin/bash
# tests + smoke + bench in one GPU call
bash scripts/gpu_check.sh tests/test_gpu_ops.py tests/test_gpu_model.py
STEPS=${STEPS:-10} WARM=${WARM:-3} bash scripts/bench_check.sh --no-cpu-baseline
