timeout 600 python -m pytest tests/test_gpu_direct_filter.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|assert|passed|failed" | head -30
