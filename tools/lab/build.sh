#!/bin/bash
# build.sh [extra nvcc flags]: gemm lab binary against the library's runtime object
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -I../../include "$@" -o gemm_lab gemm_lab.cu ../../build/obj/runtime.o -lcuda
