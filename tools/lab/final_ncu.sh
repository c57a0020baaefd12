#!/bin/bash
# ncu --set full of this session's changed kernels: K8 decode attention with the head-major
# grid (LLaVA MHA, 150 sequences x 747 context, shuffled blocks) and the K1c swap path with
# 128-wide token tiles (LLaVA down projection, M = 96)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/fncu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_decode_kernel -c 1 -o gpurun_out/fncu/decode_hm python tools/decode_once.py 32 32 150 747 > gpurun_out/fncu/a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:csk -c 1 -o gpurun_out/fncu/down96_swap128 python tools/gemm_once.py 96 4096 11008 3 > gpurun_out/fncu/b.log 2>&1
