timeout 900 python -m pytest tests/test_gpu_configs.py -q 2>&1 | grep -E "Error|error|assert|passed|failed" | head -10
