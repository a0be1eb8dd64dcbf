# skinny decode GEMM split count by wave efficiency (debug build of the change) vs the previous rule
# (libzdc_prev.so): c3 / c4 decode layer-steps, same box
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bench_paths.py tests/test_gpu_decode_tc.py -q -x 2>&1 | tail -1
run() { ZDC_LIB_PATH=$PWD/paper_2408_04107_b200/libzdc_$1.so timeout 900 python bench.py --steps 1 --warmup 3 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d['other_configs']
for k in ['c3']:
  x=o[k]; print(k, 'decode us', x['decode']['us_per_layer_step'], 'frac', x['decode']['frac'])"; }
for rep in 1 2 3; do for lib in prev debug; do echo "== $lib"; run $lib; done; done 2>&1 | tee gpurun_out/s3/ab_skinny_rule.txt
