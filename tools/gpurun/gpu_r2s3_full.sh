# session-3 evidence: full GPU suite, smoke, default bench line, launch list of the c2 step
mkdir -p gpurun_out/s3
timeout 3000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/s3/pytest_full.txt
cat gpurun_out/s3/pytest_full.txt | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/s3/bench_full.json 2> gpurun_out/s3/bench_full.log
tail -c 300 gpurun_out/s3/bench_full.json
