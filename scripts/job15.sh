mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -8 gpurun_out/gputests.log
