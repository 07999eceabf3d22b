mkdir -p gpurun_out/r2k
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2k/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/pytest_gpu.log
tail -25 gpurun_out/r2k/pytest_gpu.log
ls -la gpurun_out/r2k
