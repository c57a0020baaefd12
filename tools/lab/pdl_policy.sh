for rate in 30 90; do
  for pol in never decode; do
    echo "== rate $rate HY_PDL_POLICY=$pol"
    HY_PDL_POLICY=$pol python tools/profile_serving.py --requests 400 --rate $rate 2>&1 | grep -v Warn | tail -2
  done
done
