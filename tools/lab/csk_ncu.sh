#!/bin/bash
# ncu --set full of the K1c decode GEMM after the cluster-residency fix (Qwen2-VL down, M = 32;
# clusters of 4) and, for contrast, the pre-fix cluster size forced (HY_GEMM_CSK=5)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/cskncu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:csk -c 1 -o gpurun_out/cskncu/down32_ks4 python tools/gemm_once.py 32 3584 18944 3 > gpurun_out/cskncu/a.log 2>&1
HY_GEMM_CSK=5 timeout 300 ncu --set full --clock-control none --import-source on -k regex:csk -c 1 -o gpurun_out/cskncu/down32_ks5 python tools/gemm_once.py 32 3584 18944 3 > gpurun_out/cskncu/b.log 2>&1
