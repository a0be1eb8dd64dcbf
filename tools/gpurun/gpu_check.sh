timeout 900 python -m pytest tests -m gpu -x -q -k "decode" 2>&1 | tail -1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sp 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('FFMA2', round(d['value']), d['ms_per_step'], round(d['decode_tok_s']), d['roofline']['frac'])"
git stash -q 2>/dev/null; true
