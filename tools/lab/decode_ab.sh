# decode attention kernel A/B on a 400-request LLaVA serving replay (device clock)
for v in "" "HY_DECODE_BULK=8,3" "HY_DECODE_BULK=4,6" "HY_DECODE_CTAS_PER_SM=16"; do
  echo "== $v"
  env $v python tools/profile_serving.py --requests 400 --rate 90 2>&1 | grep -v Warn | tail -2
done
