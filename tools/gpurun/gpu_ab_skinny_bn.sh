# same-box A/B: skinny decode GEMM tile width (ZDC_SKINNY_BN 0 = rule, 128, 256) on c3 / c4
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
run() { ZDC_LIB_PATH=$D timeout 900 env "$@" python bench.py --steps 1 --warmup 3 --configs c3,c4 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d['other_configs']
for k in ('c3','c4'):
  x=o[k]; print(k, 'decode us', x['decode']['us_per_layer_step'], 'frac', x['decode']['frac'])"; }
for v in 0 1 2 3 4; do echo "== skinny_sk $v"; run ZDC_SKINNY_SK=$v; done 2>&1 | tee gpurun_out/s3/ab_skinny_sk.txt
