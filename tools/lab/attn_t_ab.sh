#!/bin/bash
# tcgen05 attention query tiles per CTA (HY_ATTN_T: 1 / 2 forced vs the wave heuristic) on the
# 400-request LLaVA serving replay (prefill chunks of ~611-token requests + 577-token ViT images)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/attnt
for rep in 1 2; do
for v in auto 1 2; do
  echo "== HY_ATTN_T=$v rep $rep" >> gpurun_out/attnt/serving.log
  if [ $v = auto ]; then unset HY_ATTN_T; else export HY_ATTN_T=$v; fi
  timeout 400 python tools/profile_serving.py --requests 400 --rate 90 2>&1 | grep -v Warn | tail -2 | head -1 >> gpurun_out/attnt/serving.log
done
done
