mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fold.py -q -x -rf 2>&1 | tail -25 | tee gpurun_out/fold_tests.txt
