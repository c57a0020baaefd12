#!/bin/bash
# decode / small-M GEMMs (K1c cluster split-K): the dispatch (65-128 rows with K >= 8192 in the
# swap orientation, 128-wide token tiles, partials in rank 0's operand ring) vs forced off / on
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/csk
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k gemm > gpurun_out/csk/tests.log 2>&1; echo "rc=$?" >> gpurun_out/csk/tests.log
timeout 900 python tools/kernel_sweep.py --what gemm --only custom --shapes 80x4096x11008,96x4096x11008,128x4096x11008,80x3584x18944,128x3584x18944,128x4096x4096,128x3584x3584,32x3584x18944 --variants 'HY_GEMM_SWAP128=0;HY_GEMM_SWAP128=1' > gpurun_out/csk/sweep.log 2>&1
