#!/bin/bash
# decode (swap-AB / K1c) GEMMs: the dispatch's cluster split-K choice vs forced cluster sizes,
# Qwen2-VL and LLaVA decode shapes (M <= 256), and the GEMM kernel tests
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/csk
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/csk/tests.log 2>&1; echo "rc=$?" >> gpurun_out/csk/tests.log
timeout 900 python tools/kernel_sweep.py --what gemm --only custom --shapes 32x3584x18944,64x3584x18944,32x4608x3584,64x4608x3584,32x3584x3584,64x3584x3584,32x37888x3584,128x3584x18944,256x3584x18944,128x4608x3584,256x3584x3584,32x4096x11008,64x4096x11008,32x4096x4096,128x4096x4096,256x4096x11008,16x4096x4096 --variants 'HY_GEMM_CSK=2;HY_GEMM_CSK=3;HY_GEMM_CSK=4' > gpurun_out/csk/sweep.log 2>&1
