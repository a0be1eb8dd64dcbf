mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_bench_paths.py -q -x -k "split or c3" 2>&1 | tail -3
timeout 900 python bench.py --steps 2 --warmup 2 --configs c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['other_configs'].items(): print(k, v['decode']['us_per_layer_step'], v['decode']['frac'], v['prefill']['frac']) if 'decode' in v else print(k, v)"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_c3_decode2.csv python tools/c3_decode_once.py > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/ncu_c3_decode2.csv | tail -12
