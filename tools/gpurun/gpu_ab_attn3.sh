# v3 decode attention (byte-balanced flat split): parity tests of every separate-path decode
# family, then same-box A/B of the c3 layer-step (ZDC_DEC_ATTN_V3 0 / 1, debug build)
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 1500 python -m pytest tests/test_gpu_split.py tests/test_gpu_decode.py tests/test_gpu_decode_modes.py tests/test_gpu_bench_paths.py tests/test_gpu_evict.py tests/test_gpu_kernels.py -q -x -rf > gpurun_out/s3/attn3_pytest.txt 2>&1; tail -4 gpurun_out/s3/attn3_pytest.txt
run() { ZDC_LIB_PATH=$D timeout 600 env "$@" python bench.py --steps 1 --warmup 3 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d['other_configs']
for k in ('c3','c3_mean'):
  x=o[k]; print(k, 'decode us', x['decode']['us_per_layer_step'], 'frac', x['decode']['frac'], 'prefill frac', x['prefill']['frac'])
print('c2 decode', d['roofline']['avg_us'])"; }
for rep in 1; do for v in 0 1; do echo "== v3 $v"; run ZDC_DEC_ATTN_V3=$v; done; done 2>&1 | tee gpurun_out/s3/ab_attn3.txt
