mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_modes.py -q -x 2>&1 | tail -2
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
for v in 1 0 1 0; do
  echo "== balance $v"
  ZDC_LIB_PATH=$D ZDC_FUSED_WO_BALANCE=$v timeout 300 python bench.py --steps 3 --warmup 3 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['roofline']['avg_us'], d['roofline']['frac'], d['value'])"
done 2>&1 | tee gpurun_out/ab_wo.txt
for v in 1 0; do echo "== trace balance $v"; ZDC_LIB_PATH=$D ZDC_FUSED_WO_BALANCE=$v ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176; done 2>&1 | tee -a gpurun_out/ab_wo.txt
