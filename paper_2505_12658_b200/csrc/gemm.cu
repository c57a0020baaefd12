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
// Two operand orientations:
//   normal  (M > 256): MMA-M = tokens (128-row tiles), MMA-N = weight rows (BN 128/256)
//   swap-AB (M <= 256, decode): MMA-M = weight rows (128), MMA-N = tokens (BN 32..256),
//           so a decode batch does not pad to a 128-row token tile.
//
// Schedule: hybrid data-parallel + stream-K.  Whole tiles go round-robin while at least
// two full waves remain; the k-block units of the remaining tiles are split evenly over
// all CTAs, so every SM streams the same number of bytes (decode GEMMs have as few as 32
// weight tiles).  A tile cut between CTAs is finished in-kernel by whichever contributor
// arrives last (per-tile atomic counter), which sums the others' fp32 partials from L2
// and runs the epilogue -- no second launch.
//
// The epilogue variant is a template parameter so every instantiation stays small
// enough for the instruction cache (a single runtime-branched kernel was ~150 KB of
// SASS and spent half its samples in instruction-fetch stalls).
//
// Reference: the work is what epdsim's cost model charges as QKVO_PROJ / FFN rows
// (/root/reference/pkg/src/epdsim/model_cost.py:113-120); the real model adds the
// lm_head and projector GEMMs the cost model omits.
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <algorithm>

namespace hy {

enum EpiKind : int { EPI_BF16 = 0, EPI_QGELU = 1, EPI_GELU = 2, EPI_SWIGLU = 4, EPI_F32 = 5 };

struct GemmArgs {
  int P, Q, K;    // MMA-M extent (rows of map A), MMA-N extent (rows of map B), reduction
  int np, nq, nkb;
  int t_dp;       // whole tiles [0, t_dp) round-robin (multiple of the grid when stream-K)
  long long u_sk; // k-block units of tiles [t_dp, T), split evenly over the grid
  int M, N;       // logical GEMM shape (tokens, physical weight rows)
  const bf16* bias;
  const bf16* residual;
  int ldr;
  const int* row_map;
  void* out;
  int ldc;
  float* partial;  // [G][2][128][BN] fp32: first / last stream-K segment of each CTA
  int* counters;   // [2G][4] arrival counters per stream-K tile and epilogue warp (zeroed)
};

template <int EPI>
__device__ __forceinline__ float act_of(float x) {
  if (EPI == EPI_QGELU) return x / (1.0f + __expf(-1.702f * x));
  if (EPI == EPI_GELU) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  return x;
}

// Normal orientation: this thread owns token row m and physical columns n0..n0+31.
template <int EPI>
__device__ __forceinline__ void epi_rows(const GemmArgs& a, int m, int n0, float* v) {
  if (m >= a.M || n0 >= a.N) return;
  if (a.bias) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      float b[8];
      load_bf16x8(a.bias + n0 + j, b);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[j + t] += b[t];
    }
  }
  constexpr int CNT = EPI == EPI_SWIGLU ? 16 : 32;
  const int col0 = EPI == EPI_SWIGLU ? n0 / 2 : n0;
  if (EPI == EPI_SWIGLU) {
    // physical cols [32g, 32g+16) gate, [32g+16, 32g+32) up -> outputs [16g, 16g+16)
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = v[j] / (1.0f + __expf(-v[j])) * v[16 + j];
  } else if (EPI == EPI_QGELU || EPI == EPI_GELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = act_of<EPI>(v[j]);
  }
  if (a.residual) {
    const bf16* r = a.residual + (size_t)m * a.ldr + col0;
#pragma unroll
    for (int j = 0; j < CNT; j += 8) {
      float b[8];
      load_bf16x8(r + j, b);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[j + t] += b[t];
    }
  }
  const size_t row = a.row_map ? (size_t)a.row_map[m] : (size_t)m;
  if (EPI == EPI_F32) {
    float* o = reinterpret_cast<float*>(a.out) + row * a.ldc + col0;
#pragma unroll
    for (int j = 0; j < CNT; j += 4)
      *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  } else {
    bf16* o = reinterpret_cast<bf16*>(a.out) + row * a.ldc + col0;
#pragma unroll
    for (int j = 0; j < CNT; j += 8) store_bf16x8(o + j, v + j);
  }
}

// Swap orientation: this thread owns weight row n and tokens m0..m0+31 (warp-coalesced
// along n).  SwiGLU pairs rows n and n+16 of the same warp through a shuffle.
template <int EPI>
__device__ __forceinline__ void epi_cols(const GemmArgs& a, int n, int m0, float* v, int lane) {
  const bool nok = n < a.N;
  const float b = (a.bias && nok) ? __bfloat162float(a.bias[n]) : 0.f;
  int col = n;
  bool writer = nok;
  if (EPI == EPI_SWIGLU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float x = v[j] + b;
      const float up = __shfl_down_sync(0xffffffffu, x, 16);
      v[j] = x / (1.0f + __expf(-x)) * up;
    }
    writer = nok && lane < 16;
    col = (n >> 5) * 16 + (n & 15);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = act_of<EPI>(v[j] + b);
  }
  if (!writer) return;
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const int m = m0 + j;
    if (m >= a.M) break;
    float x = v[j];
    if (a.residual) x += __bfloat162float(a.residual[(size_t)m * a.ldr + col]);
    const size_t row = a.row_map ? (size_t)a.row_map[m] : (size_t)m;
    if (EPI == EPI_F32)
      reinterpret_cast<float*>(a.out)[row * a.ldc + col] = x;
    else
      reinterpret_cast<bf16*>(a.out)[row * a.ldc + col] = __float2bfloat16_rn(x);
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

// raster index -> (p, q): groups of 8 p-tiles sweep all q-tiles (L2 reuse)
__device__ __forceinline__ void raster_tile(int t, const GemmArgs& a, int& p, int& q) {
  constexpr int G8 = 8;
  const int span = G8 * a.nq;
  const int g = t / span;
  const int first_p = g * G8;
  const int gp = min(a.np - first_p, G8);
  const int rr = t - g * span;
  p = first_p + rr % gp;
  q = rr / gp;
}

struct Seg {
  int tile;      // raster index
  int kb0, kb1;  // k-block range
  int slot;      // -1 whole tile; 0 / 1: partial (first / last stream-K segment of the CTA)
  int sk;        // stream-K tile index (tile - t_dp), or -1
};

__device__ __forceinline__ int cta_segments(const GemmArgs& a, int c, int G, long long& u0,
                                            long long& u1) {
  const int n_dp = (a.t_dp - c + G - 1) / G;
  u0 = (long long)c * a.u_sk / G;
  u1 = (long long)(c + 1) * a.u_sk / G;
  const int n_sk = u1 > u0 ? (int)((u1 - 1) / a.nkb - u0 / a.nkb) + 1 : 0;
  return n_dp + n_sk;
}

__device__ __forceinline__ Seg get_segment(const GemmArgs& a, int c, int G, int i, long long u0,
                                           long long u1) {
  Seg s;
  const int n_dp = (a.t_dp - c + G - 1) / G;
  if (i < n_dp) {
    s.tile = i * G + c;
    s.kb0 = 0;
    s.kb1 = a.nkb;
    s.slot = -1;
    s.sk = -1;
    return s;
  }
  const int j = i - n_dp;
  const long long t = u0 / a.nkb + j;
  const long long lo = max(u0, t * a.nkb), hi = min(u1, (t + 1) * a.nkb);
  s.tile = a.t_dp + (int)t;
  s.sk = (int)t;
  s.kb0 = (int)(lo - t * a.nkb);
  s.kb1 = (int)(hi - t * a.nkb);
  s.slot = (s.kb0 == 0 && s.kb1 == a.nkb) ? -1 : (j == 0 ? 0 : 1);
  return s;
}

template <int BN, bool SWAP, int EPI>
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
  const int G = gridDim.x;
  const int cta = blockIdx.x;
  pdl_trigger();  // all CTAs are resident from the start (persistent grid <= #SMs)

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

  long long su0, su1;
  const int nseg = cta_segments(a, cta, G, su0, su1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t hintA = SWAP ? kEvictFirst : kEvictNormal;  // decode weights stream once
      const uint64_t hintB = SWAP ? kEvictLast : kEvictNormal;
      // weight tile = A in swap orientation, B otherwise; activations are the other one
      auto load_w = [&](int st, int kb, int p, int q) {
        if (SWAP)
          tma_load_2d(&tmA, &full[st], sA + st * C::A_BYTES, kb * C::BK, p * C::BM, hintA);
        else
          tma_load_2d(&tmB, &full[st], sB + st * C::B_BYTES, kb * C::BK, q * BN, hintB);
      };
      auto load_x = [&](int st, int kb, int p, int q) {
        if (SWAP)
          tma_load_2d(&tmB, &full[st], sB + st * C::B_BYTES, kb * C::BK, q * BN, hintB);
        else
          tma_load_2d(&tmA, &full[st], sA + st * C::A_BYTES, kb * C::BK, p * C::BM, hintA);
      };
      // (1) before the grid dependency resolves: weight tiles of the first stages (the
      //     weights are never written on the stream, so this overlaps the previous kernel)
      int npre = 0;
      for (int i = 0; i < nseg && npre < C::STAGES; ++i) {
        const Seg sg = get_segment(a, cta, G, i, su0, su1);
        int p, q;
        raster_tile(sg.tile, a, p, q);
        for (int kb = sg.kb0; kb < sg.kb1 && npre < C::STAGES; ++kb, ++npre) {
          mbar_expect_tx(&full[npre], C::STAGE_BYTES);
          load_w(npre, kb, p, q);
        }
      }
      pdl_wait();
      // (2) everything in order; prefetched stages only need their activation tile
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = get_segment(a, cta, G, i, su0, su1);
        int p, q;
        raster_tile(sg.tile, a, p, q);
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++g) {
          if (g < npre) {
            load_x(stage, kb, p, q);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            load_w(stage, kb, p, q);
            load_x(stage, kb, p, q);
          }
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
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = get_segment(a, cta, G, i, su0, su1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)
            umma_bf16(d_tmem, smem_desc_k_sw128(a_addr + k * 32), smem_desc_k_sw128(b_addr + k * 32),
                      idesc, (kb > sg.kb0 || k > 0) ? 1u : 0u);
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
    pdl_wait();  // residuals, partials and counters are written by earlier kernels
    const int sub = warp & 3;  // TMEM lane sub-partition this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0; i < nseg; ++i) {
      const Seg sg = get_segment(a, cta, G, i, su0, su1);
      int p, q;
      raster_tile(sg.tile, a, p, q);
      mbar_wait_sleepy(&tfull[acc], acc_phase);
      tc_fence_after();
      const int lrow = sub * 32 + lane;  // tile row (TMEM lane) owned by this thread
      const int prow = p * 128 + lrow;
      const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
      bool finish = true;
      int c0 = 0, c1 = -1;
      long long ub = 0;
      if (sg.slot >= 0) {
        // stream-K partial: publish raw accumulators, then count arrivals
        float* mine = a.partial + ((size_t)(cta * 2 + sg.slot) * 128 + lrow) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(reinterpret_cast<float4*>(mine + c * 32 + j),
                   make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                               __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
        }
        ub = (long long)sg.sk * a.nkb;
        c0 = (int)(((ub + 1) * G - 1) / a.u_sk);
        c1 = (int)(((ub + a.nkb) * G - 1) / a.u_sk);
        __threadfence();
        __syncwarp();
        int prev = 0;
        int* ctr = a.counters + sg.sk * 4 + sub;
        if (lane == 0) prev = atomicAdd(ctr, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        finish = prev == c1 - c0;  // the last contributor reduces and writes the tile
        if (finish) {
          __threadfence();
          if (lane == 0) *ctr = 0;  // ready for the next GEMM on this workspace
        }
      }
      if (finish) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          // other contributors' partials (<= 3 by construction of the grid), all loads
          // issued before any add so the L2 round trips overlap
          const float* srcs[3];
          int ns = 0;
          for (int cc = c0; cc <= c1 && ns < 3; ++cc) {
            if (cc == cta) continue;
            const long long cu0 = (long long)cc * a.u_sk / G;
            const int slot = cu0 >= ub ? 0 : 1;
            srcs[ns++] = a.partial + ((size_t)(cc * 2 + slot) * 128 + lrow) * BN + c * 32;
          }
          float4 f[3][8];
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
            if (s2 < ns) {
#pragma unroll
              for (int j = 0; j < 8; ++j) f[s2][j] = __ldcg(reinterpret_cast<const float4*>(srcs[s2]) + j);
            }
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
            if (s2 < ns) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                v[4 * j] += f[s2][j].x;
                v[4 * j + 1] += f[s2][j].y;
                v[4 * j + 2] += f[s2][j].z;
                v[4 * j + 3] += f[s2][j].w;
              }
            }
          if (!SWAP)
            epi_rows<EPI>(a, prow, q * BN + c * 32, v);
          else
            epi_cols<EPI>(a, prow, q * BN + c * 32, v, lane);
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

template <int BN, bool SWAP, int EPI>
static int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, const GemmArgs& a, int grid,
                       cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    HY_CUDA_RET(cudaFuncSetAttribute(gemm_tc_kernel<BN, SWAP, EPI>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr_set = true;
  }
  HY_CUDA_RET(launch_pdl(gemm_tc_kernel<BN, SWAP, EPI>, dim3(grid), dim3(C::THREADS), C::SMEM_BYTES, st, tA, tB, a));
  HY_LAUNCH_CHECK();
  return 0;
}

template <bool SWAP, int EPI>
static int launch_bn(int bn, const CUtensorMap& tA, const CUtensorMap& tB, const GemmArgs& a,
                     int grid, cudaStream_t st) {
  switch (bn) {
    case 32: return SWAP ? launch_gemm<32, SWAP, EPI>(tA, tB, a, grid, st) : -1;
    case 64: return SWAP ? launch_gemm<64, SWAP, EPI>(tA, tB, a, grid, st) : -1;
    case 128: return launch_gemm<128, SWAP, EPI>(tA, tB, a, grid, st);
    case 256: return launch_gemm<256, SWAP, EPI>(tA, tB, a, grid, st);
    default: return -1;
  }
}

template <bool SWAP>
static int launch_epi(int epi, int bn, const CUtensorMap& tA, const CUtensorMap& tB,
                      const GemmArgs& a, int grid, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_bn<SWAP, EPI_BF16>(bn, tA, tB, a, grid, st);
    case EPI_QGELU: return launch_bn<SWAP, EPI_QGELU>(bn, tA, tB, a, grid, st);
    case EPI_GELU: return launch_bn<SWAP, EPI_GELU>(bn, tA, tB, a, grid, st);
    case EPI_SWIGLU: return launch_bn<SWAP, EPI_SWIGLU>(bn, tA, tB, a, grid, st);
    case EPI_F32: return launch_bn<SWAP, EPI_F32>(bn, tA, tB, a, grid, st);
    default: return -1;
  }
}

// Workspace layout: [counters: 16 KiB][partials: G * 2 * 128 * BN fp32].  The counter
// region must be zero before first use; every call leaves it zeroed again.
static constexpr size_t kCounterBytes = 16384;

int gemm_bf16(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K,
              const HyGemmEpilogue* e, void* ws, size_t ws_bytes, cudaStream_t st, int force_mode) {
  HY_CHECK_ARG(M >= 0 && N > 0 && K > 0, "gemm shape");
  if (M == 0) return 0;
  HY_CHECK_ARG(K % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0, "K, lda, ldw must be multiples of 8");
  HY_CHECK_ARG(N % 32 == 0, "N must be a multiple of 32");
  HY_CHECK_ARG(((uintptr_t)A & 15) == 0 && ((uintptr_t)W & 15) == 0, "operands must be 16B aligned");
  HY_CHECK_ARG(e && e->out, "epilogue output");
  int epi;
  switch (e->act) {
    case HY_ACT_NONE: epi = e->out_f32 ? EPI_F32 : EPI_BF16; break;
    case HY_ACT_QUICK_GELU: epi = EPI_QGELU; break;
    case HY_ACT_GELU: epi = EPI_GELU; break;
    case HY_ACT_SWIGLU: epi = EPI_SWIGLU; break;
    default:
      set_last_error("gemm: unsupported epilogue activation " + std::to_string(e->act));
      return (int)cudaErrorInvalidValue;
  }
  HY_CHECK_ARG(!(e->out_f32 && e->act != HY_ACT_NONE), "fp32 output only without activation");
  GemmArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.bias = reinterpret_cast<const bf16*>(e->bias);
  a.residual = reinterpret_cast<const bf16*>(e->residual);
  a.ldr = e->ldr;
  a.row_map = e->row_map;
  a.out = e->out;
  a.ldc = e->ldc;
  const int out_cols = (e->act == HY_ACT_SWIGLU) ? N / 2 : N;
  HY_CHECK_ARG(e->ldc >= out_cols, "ldc");
  if (a.residual) HY_CHECK_ARG(e->ldr >= out_cols, "ldr");
  if (e->out_f32 || e->ldc % 8 == 0) {
  } else {
    HY_CHECK_ARG(false, "ldc must be a multiple of 8 for bf16 output");
  }

  const bool swap = (force_mode == 1) || (force_mode == 0 && M <= 256);
  int bn;
  if (swap) {
    bn = M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
    a.P = N;
    a.Q = M;
  } else {
    bn = (N % 256 == 0) ? 256 : 128;
    HY_CHECK_ARG(N % 128 == 0, "normal orientation needs N % 128 == 0");
    a.P = M;
    a.Q = N;
  }
  if (const char* env_bn = getenv("HY_GEMM_BN")) bn = atoi(env_bn);  // tuning only
  a.np = ceil_div(a.P, 128);
  a.nq = ceil_div(a.Q, bn);
  a.nkb = ceil_div(K, 64);
  const int T = a.np * a.nq;
  const int sms = num_sms();
  const size_t need = kCounterBytes + (size_t)sms * 2 * 128 * bn * sizeof(float);
  // stream-K only when whole-tile waves would leave the machine badly underfilled
  const double dp_eff = (double)T / ((double)ceil_div(T, sms) * sms);
  bool sk = ws != nullptr && ws_bytes >= need && dp_eff < 0.85 && a.nkb >= 4;
  if (getenv("HY_GEMM_NOSK")) sk = false;
  if (getenv("HY_GEMM_SK")) sk = ws != nullptr && ws_bytes >= need;
  int grid;
  if (!sk) {
    grid = std::min(T, sms);
    a.t_dp = T;
    a.u_sk = 0;
  } else {
    const long long U = (long long)T * a.nkb;
    // at most 4 contributors per stream-K tile (T < sms: grid <= 3T)
    grid = (int)std::min<long long>(std::min<long long>(sms, U), T >= sms ? sms : 3LL * T);
    a.t_dp = T >= 2 * grid ? (T / grid - 1) * grid : 0;
    a.u_sk = (long long)(T - a.t_dp) * a.nkb;
    a.counters = reinterpret_cast<int*>(ws);
    a.partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kCounterBytes);
  }

  CUtensorMap tA, tB;
  if (!swap) {
    HY_RET_IF(make_tmap_2d_bf16(&tA, A, M, K, (uint64_t)lda * 2, 128, 64));
    HY_RET_IF(make_tmap_2d_bf16(&tB, W, N, K, (uint64_t)ldw * 2, bn, 64));
  } else {
    HY_RET_IF(make_tmap_2d_bf16(&tA, W, N, K, (uint64_t)ldw * 2, 128, 64));
    HY_RET_IF(make_tmap_2d_bf16(&tB, A, M, K, (uint64_t)lda * 2, bn, 64));
  }
  const int rc = swap ? launch_epi<true>(epi, bn, tA, tB, a, grid, st)
                      : launch_epi<false>(epi, bn, tA, tB, a, grid, st);
  if (rc < 0) {
    set_last_error("gemm: no kernel for BN=" + std::to_string(bn));
    return (int)cudaErrorInvalidValue;
  }
  return rc;
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
