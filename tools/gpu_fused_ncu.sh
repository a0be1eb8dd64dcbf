mkdir -p gpurun_out
for m in 0 1; do
ZDC_DEC_FUSED=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_fused$m.csv python bench.py --profile-only --layers 4 --decode-steps 16 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_fused -s 40 -c 1 -o gpurun_out/prof_fused python bench.py --profile-only --layers 4 --decode-steps 16 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
