# PDL on/off at a decode-heavy and a prefill-heavy serving rate (400 LLaVA requests)
for rate in 30 90; do
  for pdl in 0 1; do
    echo "== rate $rate HY_PDL=$pdl"
    HY_PDL=$pdl python tools/profile_serving.py --requests 400 --rate $rate 2>&1 | grep -v Warn | tail -2
  done
done
