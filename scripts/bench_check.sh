#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-10} --warmup ${WARM:-3} $@ > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 3000 gpurun_out/bench.log
