"""fp64 CPU oracle for ZDC's hot path — TEST INFRASTRUCTURE ONLY (see zdc_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with paper_2408_04107_b200/.
"""
from .zdc_oracle import *  # noqa: F401,F403
from .zdc_oracle import (OracleModel, bf16, canonical_signs, fold_layer, importance,  # noqa: F401
                         important_count, kept_width, select_important, softmax_rows,
                         svd_right, truncate_layer, unfolded_forward, cache_floats,
                         sp_bytes_received, sp_bytes_received_ulysses, kmeans, layer_groups,
                         e4m3, quantize_rows)
