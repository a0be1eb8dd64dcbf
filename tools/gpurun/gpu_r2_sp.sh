mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sp.py -q -rf -x 2>&1 | tail -15 | tee gpurun_out/r2_sp.txt
