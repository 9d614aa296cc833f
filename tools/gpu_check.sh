#!/bin/bash
# One GPU round trip after a kernel change: device times of the main configs, then the GPU suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
REPS=5 timeout -s INT 300 python tools/time_compress.py ${CFGS:-cfg3 cfg2 cfg1 cfg5_b12_d3_nnz512_fwht}
timeout -s INT ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q -x --timeout 300 ${PYTEST_ARGS:-} 2>&1 | tail -15
