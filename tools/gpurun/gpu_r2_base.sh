# round-2 baseline: GPU tests + default bench line (state at round start)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2_pytest_gpu.txt
cat gpurun_out/r2_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r2_bench_base.json 2> gpurun_out/r2_bench_base.log
tail -c 600 gpurun_out/r2_bench_base.json
