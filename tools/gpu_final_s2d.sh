mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final4.txt
cat gpurun_out/pytest_gpu_final4.txt
timeout 900 python bench.py > gpurun_out/bench_final_s2d.json 2> gpurun_out/bench_final_s2d.log
tail -c 300 gpurun_out/bench_final_s2d.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_s2d.csv \
  python bench.py --profile-only --decode-steps 8 > /dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
