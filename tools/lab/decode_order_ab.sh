#!/bin/bash
# K8 CTA order A/B: sequence-major grid (default) vs head-major (the 32 heads of one sequence
# on consecutive CTAs read adjacent 4 KiB tiles of each KV block); isolated + serving replay
cd "$(dirname "$0")/../.."
out=gpurun_out/decorder
mkdir -p $out
export DECODE_SHAPES="32/32/150/600-750/1;32/32/256/660/1;32/32/64/700/1"
HY_LIB_PATH=$PWD/build/lab/libhydra_sm100_headmajor.so timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k decode > $out/tests.log 2>&1; echo "rc=$?" >> $out/tests.log
for v in seq headmajor; do
  if [ $v = seq ]; then unset HY_LIB_PATH; else export HY_LIB_PATH=$PWD/build/lab/libhydra_sm100_$v.so; fi
  echo "== $v" >> $out/sweep.log
  timeout 300 python tools/kernel_sweep.py --what decode 2>&1 | grep -v Warn >> $out/sweep.log
done
for rep in 1 2; do
for v in seq headmajor; do
  if [ $v = seq ]; then unset HY_LIB_PATH; else export HY_LIB_PATH=$PWD/build/lab/libhydra_sm100_$v.so; fi
  echo "== $v rep $rep" >> $out/serving.log
  timeout 400 python tools/profile_serving.py --requests 400 --rate 90 2>&1 | grep -v Warn | tail -2 >> $out/serving.log
done
done
