# fused decode layer-step change: decode parity tests, same-box A/B (ZDC_FUSED_KV_TMA 0 / 1), traces
mkdir -p gpurun_out/s3
D=$PWD/paper_2408_04107_b200/libzdc_debug.so
run() { ZDC_LIB_PATH=$D timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --configs "" --no-cpu-baseline --no-e2e --no-sp --no-uncompressed --no-fold --no-fp8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['roofline']['avg_us'], d['roofline']['frac'], round(d['value']), d['clocks'])"; }
for rep in 1 2; do for v in 0 1; do echo "== kv_tma $v"; run ZDC_FUSED_KV_TMA=$v; done; done 2>&1 | tee gpurun_out/s3/ab_fused.txt
for v in 0 1; do echo "== trace kv_tma $v"; ZDC_LIB_PATH=$D ZDC_FUSED_KV_TMA=$v ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176 --steps 2 --show 1 2>&1; done | tee -a gpurun_out/s3/ab_fused.txt
