mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed > gpurun_out/r2_c3.json 2> gpurun_out/r2_c3.log
python -c "
import json; d=json.loads(open('gpurun_out/r2_c3.json').read().strip().splitlines()[-1])
for k,v in d['other_configs'].items(): print(k, json.dumps(v)[:1500])
"
tail -3 gpurun_out/r2_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu_c4_decode_step.csv python tools/c4_decode_once.py --steps 4 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
