# PDL A/B on a 400-request LLaVA serving replay (device clock): off / entry trigger / late trigger
for v in "" "HY_PDL=1" "HY_PDL=1 HY_PDL_LATE=1"; do
  echo "== $v"
  env $v python tools/profile_serving.py --requests 400 --rate 90 2>&1 | grep -v Warn | tail -3
done
