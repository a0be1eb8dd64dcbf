# round-2 checkpoint: GPU tests + the default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2c_pytest.txt
cat gpurun_out/r2c_pytest.txt
timeout 1200 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.log
tail -c 3000 gpurun_out/r2c_bench.json
