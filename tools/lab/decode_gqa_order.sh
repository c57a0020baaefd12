#!/bin/bash
# K8 grid order on the Qwen2-VL GQA shapes (28 query / 4 KV heads): head-major (in-tree) vs
# the previous sequence-major build (build/lab/libhydra_sm100_olddec.so)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/gqaorder
export DECODE_SHAPES="28/4/256/660/1;28/4/64/4000/1;28/4/128/500-2500/1;32/32/150/600-750/1"
for v in olddec new; do
  if [ $v = new ]; then unset HY_LIB_PATH; else export HY_LIB_PATH=$PWD/build/lab/libhydra_sm100_$v.so; fi
  echo "== $v" >> gpurun_out/gqaorder/sweep.log
  timeout 300 python tools/kernel_sweep.py --what decode 2>&1 | grep -v Warn >> gpurun_out/gqaorder/sweep.log
done
