#!/bin/bash
# build_attn_variant.sh NAME [nvcc -D flags...]: the library with attn_tc.cu rebuilt under the
# given compile-time settings (e.g. -DHY_ATTN_POLY=4) -> build/lab/libhydra_sm100_NAME.so
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
make -C paper_2505_12658_b200/csrc -s
mkdir -p build/lab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude "$@" -c paper_2505_12658_b200/csrc/attn_tc.cu \
  -o build/lab/attn_tc_$name.o
objs=$(ls build/obj/*.o | grep -v '/attn_tc.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/lab/libhydra_sm100_$name.so \
  build/lab/attn_tc_$name.o $objs
echo build/lab/libhydra_sm100_$name.so
