# same-box A/B of fused decode layer-step variants (debug build knobs): tests, bench c2, trace
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_modes.py tests/test_gpu_bench_paths.py -q -x 2>&1 | tail -2
run() { ZDC_LIB_PATH=$D timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['roofline']['avg_us'], d['roofline']['frac'], round(d['value']))"; }
for rep in 1 2; do
  for v in 0; do
    echo "== default"; run
  done
done 2>&1 | tee gpurun_out/s3/ab_fused.txt
for v in 0; do echo "== trace"; ZDC_LIB_PATH=$D ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176 --steps 2 --show 2; done 2>&1 | tee -a gpurun_out/s3/ab_fused.txt
