mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 2>&1 | tail -40 > gpurun_out/r2_pytest_gpu2.txt
cat gpurun_out/r2_pytest_gpu2.txt
