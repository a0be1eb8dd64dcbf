timeout 900 python -m pytest tests -m gpu -x -q -k "decode or configs" 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sp 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('FLAT', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), d['roofline']['frac'])"
ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176
