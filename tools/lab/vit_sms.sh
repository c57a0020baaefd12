# ViT GEMM grids capped (HY_VIT_SMS) so the concurrent language batch keeps SMs
for v in "" "HY_VIT_SMS=32" "HY_VIT_SMS=64" "HY_VIT_SMS=100" ""; do
  echo "== $v"
  env $v python tools/profile_serving.py --requests 400 --rate 80 2>&1 | grep -v Warn | tail -2 | head -1
done
