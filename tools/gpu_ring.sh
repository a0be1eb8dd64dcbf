ZDC_FUSED_TRACE=1 timeout 300 python tools/trace_fused.py --layers 4 --ctx 2176 --chain
