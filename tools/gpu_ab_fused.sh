# fused decode layer-step change: decode parity tests, bench c2 (x2), multi-launch trace
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_modes.py tests/test_gpu_bench_paths.py tests/test_gpu_configs.py -q -x -rf 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['roofline']['avg_us'], d['roofline']['frac'], round(d['value']), d['clocks'])"; }
for rep in 1 2; do echo "== default"; run; done 2>&1 | tee gpurun_out/s3/ab_fused.txt
echo "== trace"; ZDC_LIB_PATH=$D ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176 --steps 2 --show 2 2>&1 | tee -a gpurun_out/s3/ab_fused.txt
