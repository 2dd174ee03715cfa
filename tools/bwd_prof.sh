#!/bin/bash
# Backward timing sweep: deterministic (fixed-point dQ) vs fp32 dQ accumulation; JG_BWD_DBG=1 skips the dQ
# reduce (diagnostic: results invalid) to separate the drain's compute from its L2 reduce traffic.
python tools/attn_sweep.py 2>&1 | sed -n '1p;4p'
JG_SWEEP_DET=0 python tools/attn_sweep.py 2>&1 | sed -n '1p;4p'
JG_BWD_DBG=1 python tools/attn_sweep.py 2>&1 | sed -n '1p;4p'
JG_BWD_DBG=1 JG_SWEEP_DET=0 python tools/attn_sweep.py 2>&1 | sed -n '1p;4p'
