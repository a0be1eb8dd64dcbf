timeout 300 python -m pytest tests -m gpu -x -q -k "decode" 2>&1 | tail -2
for pf in 1 0; do
ZDC_FUSED_SELF_PF=$pf timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('SELFPF $pf', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']))"
done
ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176
