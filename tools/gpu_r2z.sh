mkdir -p gpurun_out/r2z
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2z/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2z/pytest_gpu.log
tail -5 gpurun_out/r2z/pytest_gpu.log
