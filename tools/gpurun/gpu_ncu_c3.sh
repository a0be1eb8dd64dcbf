# c3 decode launch list (release build) and a full capture of the v3 decode attention
mkdir -p gpurun_out/s3
timeout 300 python tools/c3_decode_once.py > gpurun_out/s3/c3_plain.log 2>&1 && echo plain ok
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3/ncu_c3_v3mma.csv python tools/c3_decode_once.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attn3 -s 2 -c 1 -o gpurun_out/s3/prof_attn3_mma python tools/c3_decode_once.py > /dev/null 2>&1
ls gpurun_out/s3
