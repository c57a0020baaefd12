#!/bin/bash
# ncu --set full of K1c decode GEMMs: LLaVA o-proj at M = 128 in the swap orientation with a
# 128-wide token tile (partials in rank 0's ring) and in the normal orientation
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/cskncu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:csk -c 1 -o gpurun_out/cskncu/o128_swap python tools/gemm_once.py 128 4096 4096 3 > gpurun_out/cskncu/a.log 2>&1
HY_GEMM_SWAP128=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:csk -c 1 -o gpurun_out/cskncu/o128_nrm python tools/gemm_once.py 128 4096 4096 3 > gpurun_out/cskncu/b.log 2>&1
timeout 900 python tools/kernel_sweep.py --what gemm --only custom --shapes 80x4096x4096,128x4096x4096,96x4096x11008,128x3584x3584,128x4608x3584,128x3584x18944,100x22016x4096 --variants 'HY_GEMM_SWAP128=0' > gpurun_out/cskncu/sweep.log 2>&1
