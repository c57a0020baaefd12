#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...]: the library with gemm.cu rebuilt under the given
# compile-time settings (e.g. -DHY_PAIR_SMEM_KB=160) -> build/lab/libhydra_sm100_NAME.so;
# the other objects are the in-tree build's.  Used by tools/overlap_lab.py --lib.
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
make -C paper_2505_12658_b200/csrc -s
mkdir -p build/lab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude "$@" -c paper_2505_12658_b200/csrc/gemm.cu \
  -o build/lab/gemm_$name.o
objs=$(ls build/obj/*.o | grep -v '/gemm.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/lab/libhydra_sm100_$name.so \
  build/lab/gemm_$name.o $objs
echo build/lab/libhydra_sm100_$name.so
