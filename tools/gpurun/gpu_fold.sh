mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fold.py -q -x -rf 2>&1 | tail -25 | tee gpurun_out/fold_tests.txt
timeout 900 python bench.py --steps 2 --warmup 2 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed 2>gpurun_out/fold_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['offline_fold']))"
