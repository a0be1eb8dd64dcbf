# prefill attention v4 MMA issue order (ZDC_ATTN_S_FIRST 0 / 1): parity, then same-box A/B of the
# c2 attention kernel alone and of the c4 prefill layer
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_kernels.py tests/test_gpu_bench_paths.py -q -x 2>&1 | tail -2
run() { ZDC_LIB_PATH=$D timeout 900 env "$@" python bench.py --steps 3 --warmup 3 --configs c4 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']['a3_prefill_attention']; o=d['other_configs']['c4']
print('c2 attn us', k['avg_us'], 'frac', k['frac'], 'c2 prefill tok/s', round(d['prefill_tok_s']), 'c4 prefill ms/layer', o['prefill']['ms_per_layer'], 'frac', o['prefill']['frac'])"; }
for rep in 1 2; do for v in 0 1; do echo "== s_first $v"; run ZDC_ATTN_S_FIRST=$v; done; done 2>&1 | tee gpurun_out/s3/ab_sfirst.txt
