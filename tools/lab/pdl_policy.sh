for rate in 60 90; do
  for pol in decode novis decode novis; do
    echo "== rate $rate HY_PDL_POLICY=$pol"
    HY_PDL_POLICY=$pol python tools/profile_serving.py --requests 400 --rate $rate 2>&1 | grep -v Warn | tail -2 | head -1
  done
done
