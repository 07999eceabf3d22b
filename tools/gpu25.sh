mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest25.log 2>&1; tail -25 gpurun_out/pytest25.log
