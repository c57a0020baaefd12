// K4: RMSNorm (language tower) and LayerNorm (vision tower), one warp per row,
// 16-byte vectorised, fp32 statistics.  HBM-bound: bytes = rows * cols * 2 * 2.
// The cost model ignores norms; the real model needs them.
#include "common.cuh"
#include "../../include/hydra_sm100.h"

namespace hy {

template <bool LAYER>
__global__ void norm_kernel(const bf16* __restrict__ x, int ldx, const bf16* __restrict__ w,
                            const bf16* __restrict__ b, bf16* __restrict__ out, int ldo, int rows,
                            int cols, float eps, const int* __restrict__ row_idx) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int src = row_idx ? row_idx[r] : r;
  const bf16* xr = x + (size_t)src * ldx;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * 8; c < cols; c += 256) {
    float f[8];
    load_bf16x8(xr + c, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s1 += f[j];
      s2 += f[j] * f[j];
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  float mean = 0.f, rstd;
  if (LAYER) {
    mean = s1 / cols;
    float var = fmaxf(s2 / cols - mean * mean, 0.f);
    rstd = rsqrtf(var + eps);
  } else {
    rstd = rsqrtf(s2 / cols + eps);
  }
  bf16* o = out + (size_t)r * ldo;
  for (int c = lane * 8; c < cols; c += 256) {
    float f[8], g[8];
    load_bf16x8(xr + c, f);
    load_bf16x8(w + c, g);
    if (LAYER) {
      float bb[8];
      load_bf16x8(b + c, bb);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = (f[j] - mean) * rstd * g[j] + bb[j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = f[j] * rstd * g[j];
    }
    store_bf16x8(o + c, f);
  }
}

template <bool LAYER>
static int launch_norm(const void* x, int ldx, const void* w, const void* b, void* out, int ldo,
                       int rows, int cols, float eps, const int* row_idx, cudaStream_t st) {
  HY_CHECK_ARG(cols % 8 == 0 && ldx % 8 == 0 && ldo % 8 == 0, "norm: cols/ld must be % 8");
  if (rows <= 0) return 0;
  const int threads = 256;
  const int rows_per_block = threads / 32;
  HY_CUDA_RET(launch_pdl(norm_kernel<LAYER>, dim3(ceil_div(rows, rows_per_block)), dim3(threads), 0, st, 
      reinterpret_cast<const bf16*>(x), ldx, reinterpret_cast<const bf16*>(w),
      reinterpret_cast<const bf16*>(b), reinterpret_cast<bf16*>(out), ldo, rows, cols, eps,
      row_idx));
  HY_LAUNCH_CHECK();
  return 0;
}

int rmsnorm(const void* x, int ldx, const void* w, void* out, int ldo, int rows, int cols,
            float eps, const int* row_idx, cudaStream_t st) {
  return launch_norm<false>(x, ldx, w, nullptr, out, ldo, rows, cols, eps, row_idx, st);
}
int layernorm(const void* x, int ldx, const void* w, const void* b, void* out, int ldo, int rows,
              int cols, float eps, const int* row_idx, cudaStream_t st) {
  HY_CHECK_ARG(b != nullptr, "layernorm bias");
  return launch_norm<true>(x, ldx, w, b, out, ldo, rows, cols, eps, row_idx, st);
}

}  // namespace hy

extern "C" int hy_rmsnorm(const void* x, int ldx, const void* w, void* out, int ldo, int rows,
                          int cols, float eps, const int* row_idx, cudaStream_t stream) {
  return hy::rmsnorm(x, ldx, w, out, ldo, rows, cols, eps, row_idx, stream);
}
extern "C" int hy_layernorm(const void* x, int ldx, const void* w, const void* b, void* out,
                            int ldo, int rows, int cols, float eps, const int* row_idx,
                            cudaStream_t stream) {
  return hy::layernorm(x, ldx, w, b, out, ldo, rows, cols, eps, row_idx, stream);
}
