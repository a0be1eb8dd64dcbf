mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final5.txt
cat gpurun_out/pytest_gpu_final5.txt
timeout 900 python bench.py > gpurun_out/bench_final_s2e.json 2> gpurun_out/bench_final_s2e.log
tail -c 300 gpurun_out/bench_final_s2e.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sp --configs "" > gpurun_out/bench_sp1_s2e.json 2> /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
