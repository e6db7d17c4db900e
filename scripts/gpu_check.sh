#!/bin/bash
# GPU-box check used during development: smoke + the GPU test files given as args.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for t in "$@"; do
  n=$(basename $t .py)
  timeout 1200 python -m pytest $t -x -q -m gpu > gpurun_out/$n.log 2>&1; echo $n=$?
done
tail -5 gpurun_out/smoke.log
for t in "$@"; do n=$(basename $t .py); tail -25 gpurun_out/$n.log; done
