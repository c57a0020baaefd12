# measured GEMM dispatch table vs the wave heuristic on a 400-request LLaVA serving replay
for v in "HY_GEMM_NOTABLE=1" "" "HY_GEMM_NOTABLE=1" ""; do
  echo "== $v"
  env $v python tools/profile_serving.py --requests 400 --rate 90 2>&1 | grep -v Warn | tail -2
done
