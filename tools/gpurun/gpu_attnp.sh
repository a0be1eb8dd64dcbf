mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_split.py tests/test_gpu_decode.py tests/test_gpu_decode_modes.py tests/test_gpu_bench_paths.py -q -x -rf 2>&1 | tail -8
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
for v in 1 0 1; do
  echo "== attn_p $v"
  ZDC_LIB_PATH=$D ZDC_DEC_ATTN_P=$v timeout 900 python bench.py --steps 2 --warmup 2 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['other_configs'].items(): print(k, v['decode']['us_per_layer_step'], v['decode']['frac'])
for s,v in d['kv_fp8'].items(): print(s, {a:(b['us_per_layer_step'], b['frac']) for a,b in v.items() if isinstance(b, dict)})"
done
