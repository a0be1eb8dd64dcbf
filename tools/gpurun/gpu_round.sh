# round-end evidence: GPU tests, the default bench line, ncu launch list + full captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log
tail -c 400 gpurun_out/bench_default.json
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sp > gpurun_out/bench_sp1.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-only --decode-steps 8 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_fused -s 200 -c 1 \
  -o gpurun_out/prof_decode_fused python bench.py --profile-only --decode-steps 16 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prefill_attn4 -s 4 -c 1 \
  -o gpurun_out/prof_attn4 python bench.py --profile-only --decode-steps 2 --layers 8 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16_tc -s 4 -c 2 \
  -o gpurun_out/prof_gemm python bench.py --profile-only --decode-steps 2 --layers 8 > /dev/null 2>&1
ls -la gpurun_out
