#!/bin/bash
# Build an experimental variant of the library with an alternative kernel source:
#   tools/variant.sh NAME path/to/variant.cu [UNIT]  ->  paper_2601_09477_b200/_smm_b200_NAME.so
# UNIT is the csrc translation unit it replaces (default fwht2p).  Select it at run
# time with SMM_LIB=_smm_b200_NAME.so (experiments only).
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; UNIT=${3:-fwht2p}
make -s -C paper_2601_09477_b200/csrc >/dev/null
mkdir -p build/var_$NAME
cp "$SRC" paper_2601_09477_b200/csrc/_variant_$UNIT.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static \
  --expt-relaxed-constexpr -Xptxas -v -dc -o build/var_$NAME/$UNIT.o paper_2601_09477_b200/csrc/_variant_$UNIT.cu \
  2> build/var_$NAME/ptxas.log || { grep -i error build/var_$NAME/ptxas.log; rm -f paper_2601_09477_b200/csrc/_variant_$UNIT.cu; exit 1; }
rm paper_2601_09477_b200/csrc/_variant_$UNIT.cu
OBJS=$(ls build/smm/*.o | grep -v "/$UNIT.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2601_09477_b200/_smm_b200_$NAME.so $OBJS build/var_$NAME/$UNIT.o
grep -A1 "_kernel" build/var_$NAME/ptxas.log | grep -E "registers|spill" | sort | uniq -c
