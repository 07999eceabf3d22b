# GPU check of the diffusion-coefficient move (auxmc_gamma_move) and the full GPU suite.
mkdir -p gpurun_out/r1g
timeout 600 python -m pytest tests/test_param_move.py -q -m gpu > gpurun_out/r1g/param.log 2>&1; echo "rc=$?" >> gpurun_out/r1g/param.log
tail -4 gpurun_out/r1g/param.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1g/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r1g/pytest_gpu.log
tail -3 gpurun_out/r1g/pytest_gpu.log
