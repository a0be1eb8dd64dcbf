mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_c3_decode.csv python tools/c3_decode_once.py > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
