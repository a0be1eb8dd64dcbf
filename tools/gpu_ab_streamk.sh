# stream-K skinny decode GEMMs: parity (GEMM, decode, configs) then same-box A/B of the c3 / c4
# layer-steps (ZDC_SKINNY_STREAMK 0 / 1, debug build)
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py tests/test_gpu_decode_tc.py tests/test_gpu_split.py tests/test_gpu_bench_paths.py tests/test_gpu_configs.py -q -x -rf > gpurun_out/s3/streamk_pytest.txt 2>&1; tail -3 gpurun_out/s3/streamk_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { ZDC_LIB_PATH=$D timeout 900 env "$@" python bench.py --steps 1 --warmup 3 --configs c3,c4 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d['other_configs']
for k in ('c3','c4'):
  x=o[k]; print(k, 'decode us', x['decode']['us_per_layer_step'], 'frac', x['decode']['frac'], 'prefill frac', x['prefill']['frac'])
print('c2 decode', d['roofline']['avg_us'])"; }
for v in 0 1; do echo "== streamk $v"; run ZDC_SKINNY_STREAMK=$v; done 2>&1 | tee gpurun_out/s3/ab_streamk.txt
