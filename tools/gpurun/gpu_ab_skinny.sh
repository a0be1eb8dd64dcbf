mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_tc.py tests/test_gpu_configs.py tests/test_gpu_split.py -q -x 2>&1 | tail -3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
for v in "AR=0" "AR=128" "AR=0 BN=256" "AR=0" "AR=128"; do
  ar=$(echo $v | sed -n 's/.*AR=\([0-9]*\).*/\1/p'); bn=$(echo $v | sed -n 's/.*BN=\([0-9]*\).*/\1/p')
  echo "== $v"
  ZDC_LIB_PATH=$D ZDC_SKINNY_AR=$ar ZDC_SKINNY_BN=${bn:-0} timeout 600 python bench.py --steps 2 --warmup 2 --configs c4,c3 --no-cpu-baseline --no-e2e --no-sp --no-uncompressed 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['other_configs'].items():
    print(k, v['decode']['us_per_layer_step'], v['decode']['frac']) if 'decode' in v else print(k, v)"
done 2>&1 | tee gpurun_out/ab_skinny.txt
