mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_evict.py tests/test_gpu_split.py -q -x -rf 2>&1 | tail -25
