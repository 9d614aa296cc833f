#!/bin/bash
# fwht2p thread-0 phase profile (SMM_PROFILE=1) on the given workloads
cd "$(dirname "$0")/.."
for c in "$@"; do echo "== $c"; SMM_PROFILE=1 REPS=1 timeout 300 python tools/time_compress.py $c 2>&1 | grep -E "profile|compress" | tail -2; done
