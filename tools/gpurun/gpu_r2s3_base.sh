# session-3 baseline: full GPU suite, smoke, default bench line
mkdir -p gpurun_out/s3
timeout 3000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/s3/pytest_base.txt
cat gpurun_out/s3/pytest_base.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/s3/bench_base.json 2> gpurun_out/s3/bench_base.log
tail -c 400 gpurun_out/s3/bench_base.json
