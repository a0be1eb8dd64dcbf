# round-2 final evidence after the skinny GEMM split rule (same steps as gpu_s3_final.sh)
# step and the c3 decode step, ncu full captures of the dominant kernel (decode_fused) and of the
# c3 decode attention (decode_attn3)
mkdir -p gpurun_out/s3i
timeout 3000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/s3i/pytest_gpu_full.txt
tail -2 gpurun_out/s3i/pytest_gpu_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3i/smoke.txt 2>&1; tail -1 gpurun_out/s3i/smoke.txt
timeout 1500 python bench.py > gpurun_out/s3i/bench_final.json 2> gpurun_out/s3i/bench_final.log
tail -c 300 gpurun_out/s3i/bench_final.json
timeout 300 python bench.py --profile-only --decode-steps 8 > gpurun_out/s3i/profile_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3i/launches_c2_step.csv python bench.py --profile-only --decode-steps 8 > /dev/null 2>&1
timeout 300 python bench.py --profile-only --decode-steps 16 > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_fused -s 200 -c 1 -o gpurun_out/s3i/prof_decode_fused python bench.py --profile-only --decode-steps 16 > /dev/null 2>&1
timeout 300 python tools/c3_decode_once.py > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3i/launches_c3_decode.csv python tools/c3_decode_once.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attn3 -s 2 -c 1 -o gpurun_out/s3i/prof_attn3 python tools/c3_decode_once.py > /dev/null 2>&1
ls -la gpurun_out/s3i
