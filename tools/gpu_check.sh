timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py tests/test_gpu_sp.py -x -q 2>&1 | tail -3
for v in 4 3; do
if [ $v = 3 ]; then export ZDC_ATTN_V3=1; fi
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sp 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); k=d['kernels']['a3_prefill_attention']; print('ATTN v$v', round(d['value']), round(d['prefill_tok_s']), d['prefill_ms'], k['avg_us'], k['achieved'], k['frac'])"
done
