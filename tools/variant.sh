#!/bin/bash
# Build an experimental variant of the library with an alternative fwht2p.cu:
#   tools/variant.sh NAME path/to/fwht2p_variant.cu  ->  paper_2601_09477_b200/_smm_b200_NAME.so
# select it at run time with SMM_LIB=_smm_b200_NAME.so (experiments only).
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2
make -s -C paper_2601_09477_b200/csrc >/dev/null
mkdir -p build/var_$NAME
cp "$SRC" paper_2601_09477_b200/csrc/_variant_fwht2p.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static \
  --expt-relaxed-constexpr -Xptxas -v -dc -o build/var_$NAME/fwht2p.o paper_2601_09477_b200/csrc/_variant_fwht2p.cu \
  2> build/var_$NAME/ptxas.log || { grep -i error build/var_$NAME/ptxas.log; rm -f paper_2601_09477_b200/csrc/_variant_fwht2p.cu; exit 1; }
rm paper_2601_09477_b200/csrc/_variant_fwht2p.cu
OBJS=$(ls build/smm/*.o | grep -v fwht2p.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2601_09477_b200/_smm_b200_$NAME.so $OBJS build/var_$NAME/fwht2p.o
grep -A1 "fwht2p_kernel" build/var_$NAME/ptxas.log | grep -E "registers|spill" | sort | uniq -c
