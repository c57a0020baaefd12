// K1: bf16 GEMM on 5th-generation tensor cores (tcgen05 + TMEM), fed by TMA.
//
//   out[m, n] = epilogue( sum_k A[m, k] * W[n, k] )       A: [M, K] activations,
//                                                          W: [N, K] weights (nn.Linear layout)
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer (A and W tiles, 128-byte swizzle, multi-stage mbarrier ring)
//   warp 1      MMA issuer (single thread, tcgen05.mma.cta_group::1.kind::f16, fp32 accum in TMEM)
//   warps 2..5  epilogue (tcgen05.ld -> registers -> bias / activation / residual -> global)
// The accumulator is double-buffered in TMEM so the epilogue of tile i overlaps the
// main loop of tile i+1.
//
// Two operand orientations share the kernel:
//   normal  (M > 256): MMA-M = tokens (128-row tiles), MMA-N = weight rows (BN)
//   swap-AB (M <= 256, decode): MMA-M = weight rows (128), MMA-N = tokens (BN = 16..256),
//           so a decode batch does not waste a 128-row token tile and the weight stream,
//           which bounds these GEMMs, is spread over all SMs (plus split-K when the
//           tile count alone cannot fill 148 SMs).
//
// Reference: the work is what epdsim's cost model charges as QKVO_PROJ / FFN rows
// (/root/reference/pkg/src/epdsim/model_cost.py:113-120); the real model adds the
// lm_head and projector GEMMs the cost model omits.
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <algorithm>

namespace hy {

struct GemmArgs {
  int P, Q, K;       // MMA-M extent (rows of map A), MMA-N extent (rows of map B), reduction
  int np, nq, nkb;   // tile counts along P, Q and K blocks
  int split, kb_per_split;
  int swap;          // 0: out[p][q]   1: out[q][p]
  int M, N;          // logical GEMM shape (tokens, physical weight rows)
  // epilogue
  const bf16* bias;
  const bf16* residual;
  int ldr;
  int act;
  const int* row_map;
  void* out;
  int ldc;
  int out_f32;
  float* partial;  // split-K workspace [split][M][N] fp32
};

__device__ __forceinline__ float act_apply(int act, float x) {
  if (act == HY_ACT_QUICK_GELU) return x / (1.0f + __expf(-1.702f * x));
  if (act == HY_ACT_GELU) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  if (act == HY_ACT_SILU) return x / (1.0f + __expf(-x));
  return x;
}

// Row-chunk epilogue: one thread owns logical row m and 32 consecutive physical
// columns n0..n0+31 (n0 % 32 == 0).
__device__ __forceinline__ void epi_row_chunk(const GemmArgs& a, int m, int n0, float* v) {
  if (m >= a.M) return;
  int nvalid = min(32, a.N - n0);
  if (nvalid <= 0) return;
  if (a.bias) {
    if (nvalid == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float b[8];
        load_bf16x8(a.bias + n0 + j, b);
#pragma unroll
        for (int t = 0; t < 8; ++t) v[j + t] += b[t];
      }
    } else {
      for (int j = 0; j < nvalid; ++j) v[j] += __bfloat162float(a.bias[n0 + j]);
    }
  }
  int col0, cnt;
  if (a.act == HY_ACT_SWIGLU) {
    // physical columns [32g, 32g+16) are gate, [32g+16, 32g+32) are up for
    // output features [16g, 16g+16)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float g = v[j];
      v[j] = g / (1.0f + __expf(-g)) * v[16 + j];
    }
    col0 = n0 >> 1;
    cnt = 16;
  } else {
    if (a.act != HY_ACT_NONE) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = act_apply(a.act, v[j]);
    }
    col0 = n0;
    cnt = nvalid;
  }
  if (a.residual) {
    const bf16* r = a.residual + (size_t)m * a.ldr + col0;
    if (cnt % 8 == 0) {
      for (int j = 0; j < cnt; j += 8) {
        float b[8];
        load_bf16x8(r + j, b);
#pragma unroll
        for (int t = 0; t < 8; ++t) v[j + t] += b[t];
      }
    } else {
      for (int j = 0; j < cnt; ++j) v[j] += __bfloat162float(r[j]);
    }
  }
  size_t row = a.row_map ? (size_t)a.row_map[m] : (size_t)m;
  if (a.out_f32) {
    float* o = reinterpret_cast<float*>(a.out) + row * a.ldc + col0;
    if (cnt % 4 == 0) {
      for (int j = 0; j < cnt; j += 4)
        *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < cnt; ++j) o[j] = v[j];
    }
  } else {
    bf16* o = reinterpret_cast<bf16*>(a.out) + row * a.ldc + col0;
    if (cnt % 8 == 0) {
      for (int j = 0; j < cnt; j += 8) store_bf16x8(o + j, v + j);
    } else {
      for (int j = 0; j < cnt; ++j) o[j] = __float2bfloat16_rn(v[j]);
    }
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 192;
};

__device__ __forceinline__ void decode_tile(int t, const GemmArgs& a, int& p, int& q, int& s) {
  int tiles_pq = a.np * a.nq;
  s = t / tiles_pq;
  int r = t - s * tiles_pq;
  constexpr int G = 8;  // p-tiles per raster group (L2 reuse of the q operand)
  int span = G * a.nq;
  int g = r / span;
  int first_p = g * G;
  int gp = min(a.np - first_p, G);
  int rr = r - g * span;
  p = first_p + rr % gp;
  q = rr / gp;
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs a) {
  using C = GemmCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = a.np * a.nq * a.split;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t hintA = a.swap ? kEvictFirst : kEvictNormal;  // weights stream once in swap
      const uint64_t hintB = a.swap ? kEvictLast : kEvictNormal;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int p, q, s;
        decode_tile(t, a, p, q, s);
        int kb0 = s * a.kb_per_split;
        int kb1 = min(a.nkb, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * C::A_BYTES, kb * C::BK, p * C::BM, hintA);
          tma_load_2d(&tmB, &full[stage], sB + stage * C::B_BYTES, kb * C::BK, q * BN, hintB);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int p, q, s;
        decode_tile(t, a, p, q, s);
        int kb0 = s * a.kb_per_split;
        int kb1 = min(a.nkb, kb0 + a.kb_per_split);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            uint64_t ad = smem_desc_k_sw128(a_addr + k * 32);
            uint64_t bd = smem_desc_k_sw128(b_addr + k * 32);
            umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 ----------------
    const int sub = warp & 3;  // TMEM lane sub-partition this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int p, q, s;
      decode_tile(t, a, p, q, s);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int prow = p * 128 + sub * 32 + lane;  // this thread's MMA-M row
      const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const int qcol0 = q * BN + c * 32;
        if (!a.swap) {
          if (a.split > 1) {
            if (prow < a.M && qcol0 < a.N) {
              float* dst = a.partial + ((size_t)s * a.M + prow) * a.N + qcol0;
              int nv = min(32, a.N - qcol0);
              if (nv == 32) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              } else {
                for (int j = 0; j < nv; ++j) dst[j] = v[j];
              }
            }
          } else {
            epi_row_chunk(a, prow, qcol0, v);
          }
        } else {
          // swap-AB: prow is a physical weight row n; columns are tokens m.
          const int n = prow;
          const bool nok = n < a.N;
          if (a.split > 1) {
            if (nok) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                int m = qcol0 + j;
                if (m < a.M) a.partial[((size_t)s * a.M + m) * a.N + n] = v[j];
              }
            }
          } else {
            float bias = (a.bias && nok) ? __bfloat162float(a.bias[n]) : 0.f;
            int col = n;
            bool writer = nok;
            if (a.act == HY_ACT_SWIGLU) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                float x = v[j] + bias;
                float up = __shfl_down_sync(0xffffffffu, x, 16);
                v[j] = x / (1.0f + __expf(-x)) * up;
              }
              writer = nok && (lane < 16);
              col = (n >> 5) * 16 + (n & 15);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = act_apply(a.act, v[j] + bias);
            }
            if (writer) {
#pragma unroll 4
              for (int j = 0; j < 32; ++j) {
                int m = qcol0 + j;
                if (m < a.M) {
                  float x = v[j];
                  if (a.residual) x += __bfloat162float(a.residual[(size_t)m * a.ldr + col]);
                  size_t row = a.row_map ? (size_t)a.row_map[m] : (size_t)m;
                  if (a.out_f32)
                    reinterpret_cast<float*>(a.out)[row * a.ldc + col] = x;
                  else
                    reinterpret_cast<bf16*>(a.out)[row * a.ldc + col] = __float2bfloat16_rn(x);
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// Split-K reduction + epilogue: one thread per (row, 32-column chunk).
__global__ void gemm_splitk_reduce_kernel(const GemmArgs a) {
  int chunks = (a.N + 31) / 32;
  long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)a.M * chunks) return;
  int m = (int)(idx / chunks);
  int n0 = (int)(idx % chunks) * 32;
  int nv = min(32, a.N - n0);
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = 0.f;
  for (int s = 0; s < a.split; ++s) {
    const float* src = a.partial + ((size_t)s * a.M + m) * a.N + n0;
    if (nv == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 f = *reinterpret_cast<const float4*>(src + j);
        v[j] += f.x; v[j + 1] += f.y; v[j + 2] += f.z; v[j + 3] += f.w;
      }
    } else {
      for (int j = 0; j < nv; ++j) v[j] += src[j];
    }
  }
  epi_row_chunk(a, m, n0, v);
}

template <int BN>
static int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, const GemmArgs& a,
                       cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    HY_CUDA_RET(cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::SMEM_BYTES));
    attr_set = true;
  }
  int total = a.np * a.nq * a.split;
  int grid = std::min(total, num_sms());
  gemm_tc_kernel<BN><<<grid, C::THREADS, C::SMEM_BYTES, st>>>(tA, tB, a);
  HY_LAUNCH_CHECK();
  return 0;
}

int gemm_bf16(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K,
              const HyGemmEpilogue* e, void* ws, size_t ws_bytes, cudaStream_t st, int force_mode) {
  HY_CHECK_ARG(M >= 0 && N > 0 && K > 0, "gemm shape");
  if (M == 0) return 0;
  HY_CHECK_ARG(K % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0, "K, lda, ldw must be multiples of 8");
  HY_CHECK_ARG(N % 16 == 0, "N must be a multiple of 16");
  HY_CHECK_ARG(((uintptr_t)A & 15) == 0 && ((uintptr_t)W & 15) == 0, "operands must be 16B aligned");
  HY_CHECK_ARG(e && e->out, "epilogue output");
  if (e->act == HY_ACT_SWIGLU) HY_CHECK_ARG(N % 32 == 0, "swiglu needs N % 32 == 0");
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.bias = reinterpret_cast<const bf16*>(e->bias);
  a.residual = reinterpret_cast<const bf16*>(e->residual);
  a.ldr = e->ldr;
  a.act = e->act;
  a.row_map = e->row_map;
  a.out = e->out;
  a.ldc = e->ldc;
  a.out_f32 = e->out_f32;
  const int out_cols = (e->act == HY_ACT_SWIGLU) ? N / 2 : N;
  HY_CHECK_ARG(e->ldc >= out_cols, "ldc");
  if (a.residual) HY_CHECK_ARG(e->ldr >= out_cols, "ldr");

  bool swap = (force_mode == 1) || (force_mode == 0 && M <= 256);
  int bn;
  if (swap) {
    bn = M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
    a.swap = 1;
    a.P = N;
    a.Q = M;
  } else {
    bn = (N % 256 == 0) ? 256 : (N % 128 == 0) ? 128 : (N % 64 == 0) ? 64 : 32;
    a.swap = 0;
    a.P = M;
    a.Q = N;
  }
  a.np = ceil_div(a.P, 128);
  a.nq = ceil_div(a.Q, bn);
  a.nkb = ceil_div(K, 64);
  // split-K only when the output tiles cannot fill the machine
  int tiles = a.np * a.nq;
  int split = 1;
  int sms = num_sms();
  if (tiles < sms) {
    split = std::min(ceil_div(sms, tiles), std::max(1, a.nkb / 4));
    size_t need = (size_t)split * M * N * sizeof(float);
    while (split > 1 && (need > ws_bytes || ws == nullptr)) {
      --split;
      need = (size_t)split * M * N * sizeof(float);
    }
  }
  if (split > 1) {
    a.kb_per_split = ceil_div(a.nkb, split);
    split = ceil_div(a.nkb, a.kb_per_split);
  } else {
    a.kb_per_split = a.nkb;
  }
  a.split = split;
  a.partial = reinterpret_cast<float*>(ws);

  CUtensorMap tA, tB;
  if (!swap) {
    HY_RET_IF(make_tmap_2d_bf16(&tA, A, M, K, (uint64_t)lda * 2, 128, 64));
    HY_RET_IF(make_tmap_2d_bf16(&tB, W, N, K, (uint64_t)ldw * 2, bn, 64));
  } else {
    HY_RET_IF(make_tmap_2d_bf16(&tA, W, N, K, (uint64_t)ldw * 2, 128, 64));
    HY_RET_IF(make_tmap_2d_bf16(&tB, A, M, K, (uint64_t)lda * 2, bn, 64));
  }
  switch (bn) {
    case 32: HY_RET_IF(launch_gemm<32>(tA, tB, a, st)); break;
    case 64: HY_RET_IF(launch_gemm<64>(tA, tB, a, st)); break;
    case 128: HY_RET_IF(launch_gemm<128>(tA, tB, a, st)); break;
    default: HY_RET_IF(launch_gemm<256>(tA, tB, a, st)); break;
  }
  if (split > 1) {
    long work = (long)M * ceil_div(N, 32);
    int threads = 128;
    gemm_splitk_reduce_kernel<<<(unsigned)((work + threads - 1) / threads), threads, 0, st>>>(a);
    HY_LAUNCH_CHECK();
  }
  return 0;
}

}  // namespace hy

extern "C" int hy_gemm_bf16(const void* A, int lda, const void* W, int ldw, int M, int N, int K,
                            const HyGemmEpilogue* epi, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream) {
  return hy::gemm_bf16(reinterpret_cast<const hy::bf16*>(A), lda,
                       reinterpret_cast<const hy::bf16*>(W), ldw, M, N, K, epi, workspace,
                       workspace_bytes, stream, 0);
}

extern "C" int hy_gemm_bf16_mode(const void* A, int lda, const void* W, int ldw, int M, int N,
                                 int K, const HyGemmEpilogue* epi, void* workspace,
                                 size_t workspace_bytes, int mode, cudaStream_t stream) {
  return hy::gemm_bf16(reinterpret_cast<const hy::bf16*>(A), lda,
                       reinterpret_cast<const hy::bf16*>(W), ldw, M, N, K, epi, workspace,
                       workspace_bytes, stream, mode);
}
