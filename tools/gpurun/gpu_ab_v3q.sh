# decode attention v3: q copied with every tile (ZDC_V3_QONCE=0) or a piece's first tile only (1)
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 900 python -m pytest tests/test_gpu_decode_v3.py tests/test_gpu_split.py tests/test_gpu_bench_paths.py -q -x 2>&1 | tail -2
run() { ZDC_LIB_PATH=$D timeout 900 env "$@" python bench.py --steps 1 --warmup 3 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d['other_configs']
for k in ('c3','c3_mean'):
  x=o[k]; print(k, 'decode us', x['decode']['us_per_layer_step'], 'frac', x['decode']['frac'])"; }
for rep in 1 2; do for v in 0 1; do echo "== qonce $v"; run ZDC_V3_QONCE=$v; done; done 2>&1 | tee gpurun_out/s3/ab_v3q.txt
