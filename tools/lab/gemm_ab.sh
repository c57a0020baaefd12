# GEMM library A/B (kernel_sweep rows), HY_LIB_PATH per variant: $@ = variant names
for v in "$@"; do
  echo "== $v"
  HY_GEMM_NOTABLE=1 HY_LIB_PATH=build/lab/libhydra_sm100_$v.so python tools/kernel_sweep.py --only qkv,o,gate_up,down,vit_qkv,vit_o,vit_fc1,vit_fc2 2>&1 | grep -v Warn | grep "M=    16 \|M=    64 \|M=   256 \|M=   512 \|M=  1600 \|M=   577 \|M=  1731 \|M=  4616 "
done
