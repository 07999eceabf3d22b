mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_lgssm.py -x -q -k "parallel_filter_large_dims and case0" > gpurun_out/san24.log 2>&1; grep -m 30 -A12 "Invalid\|ERROR" gpurun_out/san24.log | head -60
