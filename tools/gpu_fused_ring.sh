for kb in 64 128 192; do
  ZDC_FUSED_RING_KB=$kb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('RING $kb', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), round(d['prefill_tok_s']))"
done
ZDC_DEC_FUSED=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('UNFUSED', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), round(d['prefill_tok_s']))"
