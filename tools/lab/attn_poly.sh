# softmax exp2 split between the SFU and the FMA-pipe polynomial (HY_ATTN_POLY pairs of 16)
for v in poly0 poly4 poly8 poly10; do
  echo "== $v"
  HY_LIB_PATH=build/lab/libhydra_sm100_$v.so python tools/kernel_sweep.py --what attn 2>&1 | grep -v Warn | grep "ours"
done
