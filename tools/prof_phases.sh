#!/bin/bash
# fwht2p thread-0 phase profile on the given workloads.  The product library carries no
# phase marks (their runtime test cost 2.7 % on cfg3): this builds the profiling variant
# (-DSMM_FWHT2P_PROFILE, tools/variant.sh) and runs it with SMM_PROFILE=1.
cd "$(dirname "$0")/.."
mkdir -p build
(echo "#define SMM_FWHT2P_PROFILE 1"; cat paper_2601_09477_b200/csrc/fwht2p.cu) > build/fwht2p_prof.cu
bash tools/variant.sh prof build/fwht2p_prof.cu > /dev/null
for c in "$@"; do echo "== $c"; SMM_LIB=_smm_b200_prof.so SMM_PROFILE=1 REPS=1 timeout 300 python tools/time_compress.py $c 2>&1 | grep -E "profile|compress" | tail -2; done
