mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gputests.log
export CFG=sweep SEED_CTA_TRACE=1
timeout 300 python scripts/trace_round.py > gpurun_out/t7_sw.log 2>&1; echo trace=$?
CFG=gsm8k timeout 300 python scripts/trace_round.py > gpurun_out/t7_gsm.log 2>&1; echo trace=$?
