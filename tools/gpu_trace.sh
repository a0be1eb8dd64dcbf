timeout 300 python -m pytest tests -m gpu -x -q -k "decode" 2>&1 | tail -2
ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('FUSED', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), round(d['prefill_tok_s']))"
