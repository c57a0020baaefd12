# Qwen2-VL GQA (28/4) decode attention at serving-like batch sizes: CTAs per SM, the CUDA-core
# GQA kernel, and the co-resident tensor-core kernel
export DECODE_SHAPES="28/4/16/1000/1;28/4/32/1500/1;28/4/64/2000/1;28/4/128/1500/1;28/4/256/660/1;28/4/32/3000/1"
for v in "" "HY_DECODE_CTAS_PER_SM=8" "HY_DECODE_CTAS_PER_SM=16" "HY_DECODE_CTAS_PER_SM=32" "HY_DECODE_GQA_CUDA=1" "DECODE_CO=1"; do
  echo "== $v"
  env $v python tools/kernel_sweep.py --what decode 2>&1 | grep decode_attn
done
