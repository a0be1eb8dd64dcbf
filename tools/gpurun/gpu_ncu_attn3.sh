# c3 decode launch lists with decode attention v2 vs v3, and a full capture of v3
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
ZDC_LIB_PATH=$D ZDC_DEC_ATTN_V3=1 timeout 300 python tools/c3_decode_once.py > gpurun_out/s3/c3_plain.log 2>&1 && echo plain ok
for v in 0 1; do
  ZDC_LIB_PATH=$D ZDC_DEC_ATTN_V3=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3/ncu_c3_v$v.csv python tools/c3_decode_once.py > /dev/null 2>&1
done
ZDC_LIB_PATH=$D ZDC_DEC_ATTN_V3=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attn3 -s 2 -c 1 -o gpurun_out/s3/prof_attn3 python tools/c3_decode_once.py > /dev/null 2>&1
ls gpurun_out/s3
