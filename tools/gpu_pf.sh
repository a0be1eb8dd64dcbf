python -m pytest tests -m gpu -x -q -k "decode" 2>&1 | tail -2
for m in 0 1 3; do
  ZDC_DEC_L2PF=$m python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('PF $m', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), round(d['prefill_tok_s']))"
done
