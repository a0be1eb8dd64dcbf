mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final2.txt
cat gpurun_out/pytest_gpu_final2.txt
timeout 900 python bench.py > gpurun_out/bench_final_s2b.json 2> gpurun_out/bench_final_s2b.log
tail -c 300 gpurun_out/bench_final_s2b.json
