# decode GEMMs (swap-AB, M = 16 / 64) back to back under PDL: does a smaller operand ring
# (two CTAs per SM) let the next GEMM's weight prefetch overlap the previous one's tail?
for lib in "" build/lab/libhydra_sm100_p96.so; do
  for pdl in 0 1; do
    echo "== lib ${lib:-default} HY_PDL=$pdl"
    HY_PDL=$pdl HY_GEMM_NOTABLE=1 ${lib:+HY_LIB_PATH=$lib} python tools/kernel_sweep.py --only qkv,o,gate_up,down 2>&1 | grep -v Warn | grep "M=    16 \|M=    64 "
  done
done
