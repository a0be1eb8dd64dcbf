mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fp8.py -q -x -rf 2>&1 | tail -30 | tee gpurun_out/fp8_tests.txt
