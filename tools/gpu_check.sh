timeout 600 python -m pytest tests/test_gpu_sp.py -q 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sp 2>gpurun_out/sp.log | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['sp'])"
tail -3 gpurun_out/sp.log
