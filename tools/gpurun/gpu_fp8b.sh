mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fp8.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 2 --warmup 2 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold 2>gpurun_out/fp8_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kv_fp8']
for s,v in k.items(): print(s, {a:(b['us_per_layer_step'], b['frac']) for a,b in v.items() if isinstance(b, dict)})"
