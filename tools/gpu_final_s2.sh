# end-of-session evidence: GPU tests, the default bench line (c2 headline + c3/c4 per-layer
# sections + e2e + cpu_baseline), SP at P = 1, the ncu launch list of the c2 step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final.txt
cat gpurun_out/pytest_gpu_final.txt
timeout 900 python bench.py > gpurun_out/bench_final_s2.json 2> gpurun_out/bench_final_s2.log
tail -c 400 gpurun_out/bench_final_s2.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sp --configs "" > gpurun_out/bench_sp1_s2.json 2> /dev/null
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_s2.json 2> /dev/null
tail -c 300 gpurun_out/bench_ref_s2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_s2.csv \
  python bench.py --profile-only --decode-steps 8 > /dev/null 2>&1
ls -la gpurun_out | tail -8
