mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sp.py tests/test_gpu_split.py tests/test_gpu_bench_paths.py -q -x -rf -k "sp or split or c3" 2>&1 | tail -8
timeout 900 python bench.py --steps 2 --warmup 2 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['other_configs'].items(): print(k, v['decode']['us_per_layer_step'], v['decode']['frac'])"
