#!/bin/bash
# table entries at 129-256 token rows vs the heuristic (K1c normal orientation): HY_GEMM_NOTABLE=1
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/midtab
timeout 900 python tools/kernel_sweep.py --what gemm --only custom --shapes 160x3584x18944,192x3584x18944,256x3584x18944,160x4608x3584,256x4608x3584,160x3584x3584,256x3584x3584,160x4096x11008,256x4096x11008,160x4096x4096,256x4096x4096,160x12288x4096,256x12288x4096,256x37888x3584,256x22016x4096 --variants 'HY_GEMM_NOTABLE=1' > gpurun_out/midtab/sweep.log 2>&1
