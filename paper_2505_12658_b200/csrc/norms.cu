// K4: RMSNorm (language tower) and LayerNorm (vision tower), one warp per row,
// 16-byte vectorised, fp32 statistics.  HBM-bound: bytes = rows * cols * 2 * 2.
// The cost model ignores norms; the real model needs them.
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <algorithm>

namespace hy {

// One CTA per row, up to 4 16-byte vectors per thread held in registers: a single HBM read of
// the row with every load in flight at once (the former warp-per-row version re-read the row
// and left an SM with a few latency-bound warps for a ~1k-row batch).
template <bool LAYER, int V>
__global__ void __launch_bounds__(512)
    norm_kernel(const bf16* __restrict__ x, int ldx, const bf16* __restrict__ w,
                const bf16* __restrict__ b, bf16* __restrict__ out, int ldo, int rows, int cols,
                float eps, const int* __restrict__ row_idx) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int src = row_idx ? row_idx[r] : r;
  const bf16* xr = x + (size_t)src * ldx;
  const int nvec = cols >> 3;
  float f[V][8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int v = threadIdx.x + k * blockDim.x;
    if (v < nvec) {
      load_bf16x8(xr + v * 8, f[k]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s1 += f[k][j];
        s2 += f[k][j] * f[k][j];
      }
    }
  }
  __shared__ float red[2][16];
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) {
    red[0][warp] = s1;
    red[1][warp] = s2;
  }
  __syncthreads();
  s1 = lane < nw ? red[0][lane] : 0.f;
  s2 = lane < nw ? red[1][lane] : 0.f;
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
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int v = threadIdx.x + k * blockDim.x;
    if (v < nvec) {
      float g[8];
      load_bf16x8(w + v * 8, g);
      if (LAYER) {
        float bb[8];
        load_bf16x8(b + v * 8, bb);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[k][j] = (f[k][j] - mean) * rstd * g[j] + bb[j];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[k][j] = f[k][j] * rstd * g[j];
      }
      store_bf16x8(o + v * 8, f[k]);
    }
  }
}

template <bool LAYER>
static int launch_norm(const void* x, int ldx, const void* w, const void* b, void* out, int ldo,
                       int rows, int cols, float eps, const int* row_idx, cudaStream_t st) {
  HY_CHECK_ARG(cols % 8 == 0 && ldx % 8 == 0 && ldo % 8 == 0, "norm: cols/ld must be % 8");
  HY_CHECK_ARG(cols <= 8 * 512 * 4, "norm: cols <= 16384");
  if (rows <= 0) return 0;
  const int nvec = cols / 8;
  // threads: a multiple of 32, <= 512, each thread <= 4 vectors
  int threads = std::min(512, ((nvec + 1) / 2 + 31) / 32 * 32);
  threads = std::max(threads, 32);
  const int per = ceil_div(nvec, threads);
  auto args = [&](auto kern) {
    return launch_pdl(kern, dim3(rows), dim3(threads), 0, st, reinterpret_cast<const bf16*>(x),
                      ldx, reinterpret_cast<const bf16*>(w), reinterpret_cast<const bf16*>(b),
                      reinterpret_cast<bf16*>(out), ldo, rows, cols, eps, row_idx);
  };
  if (per <= 2)
    HY_CUDA_RET(args(norm_kernel<LAYER, 2>));
  else
    HY_CUDA_RET(args(norm_kernel<LAYER, 4>));
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
