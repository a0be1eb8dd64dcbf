# round-2 evidence: sanitizers, the default bench line, launch list, ncu full capture of the
# dominant kernel (decode_fused) and of prefill attention, DRAM traffic per launch
mkdir -p gpurun_out/r02
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02/sanitizer_$tool.txt 2>&1
  echo "$tool: $(tail -3 gpurun_out/r02/sanitizer_$tool.txt | tr '\n' ' ')"
done
timeout 1500 python bench.py > gpurun_out/r02/bench_final.json 2> gpurun_out/r02/bench_final.log
tail -c 600 gpurun_out/r02/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02/launches_c2_step.csv python bench.py --profile-only --decode-steps 8 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_fused -s 200 -c 1 -o gpurun_out/r02/prof_decode_fused python bench.py --profile-only --decode-steps 16 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prefill_attn4 -s 4 -c 1 -o gpurun_out/r02/prof_attn4 python bench.py --profile-only --decode-steps 2 --layers 8 > /dev/null 2>&1
ls -la gpurun_out/r02
