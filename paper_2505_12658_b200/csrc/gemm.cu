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

// operand-ring budgets (KB of shared memory per CTA); lab builds lower them to leave room
// for co-resident CTAs of other kernels (tools/lab/build.sh overlap variants)
#ifndef HY_GEMM_SMEM_KB
#define HY_GEMM_SMEM_KB 196
#endif
#ifndef HY_PAIR_SMEM_KB
#define HY_PAIR_SMEM_KB 200
#endif

namespace hy {

#ifdef HY_TRACE
// Debug timeline (lab builds only): %globaltimer stamps of CTA 0 at fixed points.
__device__ unsigned long long g_trace[32];
__device__ __forceinline__ void trace(int i) {
  if (blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_trace[i] = t;
    g_trace[16 + i] = clock64();
  }
}
// per-CTA marks: [cta][0] entry, [1] first full barrier, [2] last accumulator handed to the
// epilogue, [3] exit, [4] segments, [5] stream-K tiles finished by this CTA
__device__ unsigned long long g_ctr[160][10];
__device__ __forceinline__ void cta_mark(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  g_ctr[blockIdx.x][i] = t;
}
#define HY_CNT(i, v) (g_ctr[blockIdx.x][i] = (v))
#define HY_CINC(i) atomicAdd(&g_ctr[blockIdx.x][i], 1ull)
#define HY_TR(i) trace(i)
#define HY_CM(i) cta_mark(i)
#else
#define HY_TR(i)
#define HY_CM(i)
#define HY_CNT(i, v)
#define HY_CINC(i)
#endif

enum EpiKind : int { EPI_BF16 = 0, EPI_QGELU = 1, EPI_GELU = 2, EPI_SWIGLU = 4, EPI_F32 = 5 };

struct GemmArgs {
  int P, Q, K;    // MMA-M extent (rows of map A), MMA-N extent (rows of map B), reduction
  int np, nq, nkb;
  int t_dp;       // whole tiles [0, t_dp) round-robin (multiple of the grid when stream-K)
  int dbg;        // bits: 1 no early PDL trigger, 2 no PDL launch (pair, HY_PAIR_DBG); 4 no residual
                  // prefetch; 8 late PDL trigger (after the producer's last load, HY_PDL_LATE);
                  // 16 launched without PDL; 32 K1c reduction slots inside rank 0's operand ring
  int group;      // raster group of token tiles (0 = auto; HY_GEMM_GROUP tuning only)
  long long u_sk; // k-block units of tiles [t_dp, T), split evenly over the grid
  int M, N;       // logical GEMM shape (tokens, physical weight rows)
  const bf16* bias;
  const bf16* residual;
  int ldr;
  const int* row_map;
  void* out;
  int ldc;
  float* partial;  // [G][2][128][BN] fp32: first / last stream-K segment of each CTA
  int* counters;   // [tiles][8] arrival counters per stream-K tile and epilogue warp (zeroed)
  int tma_out;     // normal orientation: bf16 output tiles leave through TMA stores (map tmC)
};

template <int EPI>
__device__ __forceinline__ float act_of(float x) {
  if (EPI == EPI_QGELU) return x / (1.0f + __expf(-1.702f * x));
  if (EPI == EPI_GELU) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  return x;
}

// Epilogue of one 32 x 32 accumulator chunk of one epilogue warp.
//
// The TMEM load gives each lane one accumulator row (normal: a token row, 32 weight
// columns; swap: a weight row, 32 tokens).  Bias and activation are applied in registers.
// Normal orientation: each lane stores its row's outputs directly (16-byte vectors).
// Swap orientation: a lane holds one output COLUMN, so the chunk is staged in shared
// memory as fp32 [32 token rows][OC cols] and written back row-contiguous (8 outputs =
// one 16-byte vector per lane) instead of 32 scattered 2-byte stores per lane; the
// residual is read with the same coalesced pattern and added in fp32 before the single
// rounding to bf16.
constexpr int kEpiWarps = 8;             // two per TMEM lane sub-partition (even / odd chunks)
constexpr int kStgStride = 32 * 4 + 16;  // bytes per staged row (pad: conflict-free 16B access)
// per epilogue warp: the swap orientation's fp32 staging (16 token rows x kStgStride per pass)
// or, in the normal orientation, two 32 x 32 bf16 buffers for the TMA-store epilogue
constexpr int kStgBytes = 4096;
static_assert(16 * kStgStride <= kStgBytes, "swap staging");

template <int EPI, bool SWAP, bool STG_DBL = true>
__device__ __forceinline__ void epi_chunk(const GemmArgs& a, int p0, int q0, float* v, int lane,
                                          uint32_t stg, const CUtensorMap* tmC, int& nst) {
  constexpr int OC = EPI == EPI_SWIGLU ? 16 : 32;  // output columns of this chunk
  int row0, col0;  // first output row (token), first output column
  if (!SWAP) {
    // lane = token row p0 + lane; registers = weight columns q0..q0+31
    if (q0 >= a.N) return;
    if (a.bias) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float b[8];
        load_bf16x8(a.bias + q0 + j, b);
#pragma unroll
        for (int t = 0; t < 8; ++t) v[j + t] += b[t];
      }
    }
    if (EPI == EPI_SWIGLU) {
      // physical cols [32g, 32g+16) gate, [32g+16, 32g+32) up -> outputs [16g, 16g+16)
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = v[j] / (1.0f + __expf(-v[j])) * v[16 + j];
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = act_of<EPI>(v[j]);
    }
    // direct row stores (fp32 logits, row-mapped outputs): each lane owns OC contiguous
    // outputs of one row
    const int m = p0 + lane;
    col0 = EPI == EPI_SWIGLU ? q0 / 2 : q0;
    if (EPI != EPI_F32 && a.tma_out) {
      // TMA-store epilogue: the warp's 32 rows x OC bf16 go through one of two shared
      // buffers and leave as one bulk tensor store (full row segments, asynchronous), instead
      // of 32 scattered 16-byte pieces per store instruction.  Rows >= M are clipped by TMA.
      const uint32_t buf = stg + (STG_DBL ? (nst & 1) * (kStgBytes / 2) : 0);
      if (lane == 0) {  // this buffer's previous store (two chunks ago / the last one) has read it
        if (STG_DBL)
          bulk_wait_read<1>();
        else
          bulk_wait_read<0>();
      }
      __syncwarp();
      if (m < a.M && a.residual) {
        const bf16* r = a.residual + (size_t)m * a.ldr + col0;
#pragma unroll
        for (int j = 0; j < OC; j += 8) {
          float b[8];
          load_bf16x8(r + j, b);
#pragma unroll
          for (int t = 0; t < 8; ++t) v[j + t] += b[t];
        }
      }
#pragma unroll
      for (int j = 0; j < OC; j += 8) {
        uint4 u;
        u.x = pack_bf16x2(v[j], v[j + 1]);
        u.y = pack_bf16x2(v[j + 2], v[j + 3]);
        u.z = pack_bf16x2(v[j + 4], v[j + 5]);
        u.w = pack_bf16x2(v[j + 6], v[j + 7]);
        sts_u32x4(buf + lane * (OC * 2) + j * 2, u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmC, buf, col0, p0);
        bulk_commit();
      }
      ++nst;
      return;
    }
    if (m < a.M) {
      if (a.residual) {
        const bf16* r = a.residual + (size_t)m * a.ldr + col0;
#pragma unroll
        for (int j = 0; j < OC; j += 8) {
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
        for (int j = 0; j < OC; j += 4)
          *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        bf16* o = reinterpret_cast<bf16*>(a.out) + row * a.ldc + col0;
#pragma unroll
        for (int j = 0; j < OC; j += 8) store_bf16x8(o + j, v + j);
      }
    }
    return;
  } else {
    // lane = weight row p0 + lane; registers = tokens q0..q0+31
    if (p0 >= a.N) return;
    const int n = p0 + lane;
    const float b = a.bias ? __bfloat162float(a.bias[n]) : 0.f;
    if (EPI == EPI_SWIGLU) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = v[j] + b;
        const float up = __shfl_down_sync(0xffffffffu, x, 16);
        v[j] = x / (1.0f + __expf(-x)) * up;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = act_of<EPI>(v[j] + b);
    }
    row0 = q0;
    col0 = EPI == EPI_SWIGLU ? p0 / 2 : p0;
  }
  // two passes of 16 token rows through the staging buffer; L lanes per row, 8 outputs
  // per lane, 32 / L rows per warp store
  constexpr int L = OC / 8;
  constexpr int RPI = 32 / L;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    if (lane < OC) {
      const uint32_t d = stg + lane * 4;
#pragma unroll
      for (int j = 0; j < 16; ++j) sts_f32(d + j * kStgStride, v[pass * 16 + j]);
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < (16 + RPI - 1) / RPI; ++it) {
      const int r = it * RPI + lane / L;
      const int k = (lane % L) * 8;
      const int m = row0 + pass * 16 + r;
      if (r < 16 && m < a.M) {
        const uint32_t s4 = stg + r * kStgStride + k * 4;
        const float4 x0 = lds_f32x4(s4), x1 = lds_f32x4(s4 + 16);
        float o[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        if (a.residual) {
          float rr[8];
          load_bf16x8(a.residual + (size_t)m * a.ldr + col0 + k, rr);
#pragma unroll
          for (int t = 0; t < 8; ++t) o[t] += rr[t];
        }
        const size_t row = a.row_map ? (size_t)a.row_map[m] : (size_t)m;
        if (EPI == EPI_F32) {
          float4* dst =
              reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + row * a.ldc + col0 + k);
          dst[0] = make_float4(o[0], o[1], o[2], o[3]);
          dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        } else {
          store_bf16x8(reinterpret_cast<bf16*>(a.out) + row * a.ldc + col0 + k, o);
        }
      }
    }
    __syncwarp();  // staging buffer is reused by the next pass / chunk
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (HY_GEMM_SMEM_KB * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + kEpiWarps * kStgBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 64 + 32 * kEpiWarps;
};

// raster index -> (p, q): groups of p-tiles sweep all q-tiles (L2 reuse): with up to 16
// p-tiles (token tiles) one group holds all of them, so each weight tile is streamed from HBM
// once while the activations stay in L2; larger M uses groups of 8
__device__ __forceinline__ void raster_tile(int t, const GemmArgs& a, int& p, int& q) {
  const int G8 = a.group > 0 ? min(a.group, a.np) : (a.np <= 16 ? a.np : 8);
  const int span = G8 * a.nq;
  const int g = t / span;
  const int first_p = g * G8;
  const int gp = min(a.np - first_p, G8);
  const int rr = t - g * span;
  p = first_p + rr % gp;
  q = rr / gp;
}

// Normal orientation: pull this thread's residual row segments of a tile into L2 while the
// tile's MMAs are still running, so the epilogue's residual loads do not add a DRAM round
// trip per 32-column chunk (the o / down projections add the residual stream in place).
template <int BN, int EPI>
__device__ __forceinline__ void prefetch_residual(const GemmArgs& a, int m, int qcol, int half) {
  if (!a.residual || m >= a.M || (a.dbg & 4)) return;
  const bf16* r = a.residual + (size_t)m * a.ldr;
#pragma unroll
  for (int c = half; c < BN / 32; c += 2) {
    const int q0 = qcol + c * 32;
    if (q0 >= a.N) break;
    const int col0 = EPI == EPI_SWIGLU ? q0 / 2 : q0;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(r + col0));
  }
}

// stream-K fixup: add up to 3 other contributors' fp32 partials of one 32-column chunk, in
// the canonical order of the contributors' CTA (pair) index -- a left fold
// x_c0 + x_c0+1 + ... with this CTA's own accumulators v at position nb -- so the result is
// bitwise independent of which contributor happens to arrive last (run-to-run
// deterministic).  srcs[] are the others in CTA order, nb of them before this CTA.  Two
// contributors' loads are issued before the first add so their L2 round trips overlap
// (three in flight at once would spill under the register cap).
__device__ __forceinline__ void add_partials(float* v, const float4* const* srcs, int ns,
                                             int nb) {
  float4 f[2][8];
  int s0 = 0;
  if (nb > 0) {  // prefix x_c0 + ... + x_(self-1), then + v
#pragma unroll
    for (int j = 0; j < 8; ++j) f[0][j] = __ldcg(srcs[0] + j * 128);
    if (nb > 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) f[1][j] = __ldcg(srcs[1] + j * 128);
    if (nb > 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        f[0][j].x += f[1][j].x;
        f[0][j].y += f[1][j].y;
        f[0][j].z += f[1][j].z;
        f[0][j].w += f[1][j].w;
      }
    if (nb > 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[1][j] = __ldcg(srcs[2] + j * 128);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        f[0][j].x += f[1][j].x;
        f[0][j].y += f[1][j].y;
        f[0][j].z += f[1][j].z;
        f[0][j].w += f[1][j].w;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[4 * j] = f[0][j].x + v[4 * j];
      v[4 * j + 1] = f[0][j].y + v[4 * j + 1];
      v[4 * j + 2] = f[0][j].z + v[4 * j + 2];
      v[4 * j + 3] = f[0][j].w + v[4 * j + 3];
    }
    s0 = nb;
  }
#pragma unroll 1
  for (; s0 < ns; s0 += 2) {  // suffix: ((v + x) + y) ...
    const bool two = s0 + 1 < ns;
#pragma unroll
    for (int j = 0; j < 8; ++j) f[0][j] = __ldcg(srcs[s0] + j * 128);
    if (two)
#pragma unroll
      for (int j = 0; j < 8; ++j) f[1][j] = __ldcg(srcs[s0 + 1] + j * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[4 * j] += f[0][j].x;
      v[4 * j + 1] += f[0][j].y;
      v[4 * j + 2] += f[0][j].z;
      v[4 * j + 3] += f[0][j].w;
      if (two) {
        v[4 * j] += f[1][j].x;
        v[4 * j + 1] += f[1][j].y;
        v[4 * j + 2] += f[1][j].z;
        v[4 * j + 3] += f[1][j].w;
      }
    }
  }
}

// One other contributor's 32-column chunk (8 float4 per lane) and the ordered add of exactly
// one contributor -- the stream-K fixup's common case (a tile shared by two CTAs / pairs).
// Loading the NEXT chunk before the current chunk's epilogue keeps one L2 round trip in
// flight under the epilogue instead of paying one per chunk in series.
__device__ __forceinline__ void ld_partial(float4* f, const float4* src) {
#pragma unroll
  for (int t = 0; t < 8; ++t) f[t] = __ldcg(src + t * 128);
}
__device__ __forceinline__ void add_one(float* v, const float4* f, bool other_first) {
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (other_first) {  // x_other + v  (same association as add_partials)
      v[4 * t] = f[t].x + v[4 * t];
      v[4 * t + 1] = f[t].y + v[4 * t + 1];
      v[4 * t + 2] = f[t].z + v[4 * t + 2];
      v[4 * t + 3] = f[t].w + v[4 * t + 3];
    } else {
      v[4 * t] += f[t].x;
      v[4 * t + 1] += f[t].y;
      v[4 * t + 2] += f[t].z;
      v[4 * t + 3] += f[t].w;
    }
  }
}

// Stream-K: true when every other contributor of this tile has already published its
// partial (arrival counter == others), checked only for a CTA's last segment (slot 1), the
// one that normally completes last.  The acquire load orders the partial reads after the
// others' fenced stores; the caller then finishes the tile without publishing its own.
__device__ __forceinline__ bool sk_all_arrived(int* ctr, int others, int slot, int lane) {
  if (slot != 1) return false;
  int v = 0;
  if (lane == 0) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  const bool all = __shfl_sync(0xffffffffu, v, 0) == others;
  if (all) __threadfence();  // every lane's partial loads after the others' stores
  return all;
}

struct Seg {
  int tile;      // raster index
  int kb0, kb1;  // k-block range
  int slot;      // -1 whole tile; 0 / 1: partial (first / last stream-K segment of the CTA)
  int sk;        // stream-K tile index (tile - t_dp), or -1
};

// k-block unit ranges fit 32 bits (the host enables stream-K only when u_sk < 2^31), so
// only the per-CTA range boundaries need one 64-bit product/division
__device__ __forceinline__ int cta_segments(const GemmArgs& a, int c, int G, int& u0, int& u1) {
  const int n_dp = (a.t_dp - c + G - 1) / G;
  if (a.u_sk == 0) {  // no stream-K: skip the 64-bit divisions
    u0 = u1 = 0;
    return n_dp;
  }
  u0 = (int)((long long)c * a.u_sk / G);
  u1 = (int)((long long)(c + 1) * a.u_sk / G);
  const int n_sk = u1 > u0 ? (int)((u1 - 1) / a.nkb - u0 / a.nkb) + 1 : 0;
  return n_dp + n_sk;
}

__device__ __forceinline__ Seg get_segment(const GemmArgs& a, int c, int G, int i, int u0,
                                           int u1) {
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
  const int t = u0 / a.nkb + j;
  const int lo = max(u0, t * a.nkb), hi = min(u1, (t + 1) * a.nkb);
  s.tile = a.t_dp + (int)t;
  s.sk = (int)t;
  s.kb0 = (int)(lo - t * a.nkb);
  s.kb1 = (int)(hi - t * a.nkb);
  s.slot = (s.kb0 == 0 && s.kb1 == a.nkb) ? -1 : (j == 0 ? 0 : 1);
  return s;
}

template <int BN, bool SWAP, int EPI>
__global__ void __launch_bounds__(64 + 32 * kEpiWarps, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const GemmArgs a) {
  using C = GemmCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* stg_base = smem + C::STAGES * C::STAGE_BYTES;  // 4 epilogue staging buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + kEpiWarps * kStgBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int cta = blockIdx.x;
  if (threadIdx.x == 0) {
    HY_TR(0);
    HY_CM(0);
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) HY_TR(1);
  // Release dependents only once this CTA holds its tensor memory.  A dependent grid
  // allocates TMEM before its griddepcontrol.wait; if it could start while a CTA of this
  // grid had not allocated yet, the two would wait on each other (this grid's CTA for the
  // columns, the dependent for this grid's completion).
  if (!(a.dbg & 8)) pdl_trigger();

  int su0, su1;
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
        if (i == 0) HY_TR(13);
        for (int kb = sg.kb0; kb < sg.kb1 && npre < C::STAGES; ++kb, ++npre) {
          mbar_expect_tx(&full[npre], C::STAGE_BYTES);
          load_w(npre, kb, p, q);
          // launched without PDL: nothing to wait for, the activations go out with the weights
          // (the first stage lands ~1 us earlier than after the whole weight prologue)
          if (a.dbg & 16) load_x(npre, kb, p, q);
          if (npre == 0) HY_TR(14);
        }
      }
      HY_TR(2);
      pdl_wait();
      HY_TR(3);
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
            if (!(a.dbg & 16)) load_x(stage, kb, p, q);
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
      // late trigger: dependents launch once every CTA has issued its last operand load
      if (a.dbg & 8) pdl_trigger();
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
          if (kb == sg.kb0 && i == 0) {
            HY_TR(4);
            HY_CM(1);
          }
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
        if (i == 0) HY_TR(5);
        if (i == nseg - 1) HY_CM(2);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9 ----------------
    pdl_wait();  // residuals, partials and counters are written by earlier kernels
    const int sub = warp & 3;          // TMEM lane sub-partition this warp may access
    const int half = (warp - 2) >> 2;  // 32-column chunks half, half + 2, ...
    int nst = 0;                       // TMA-store buffer toggle (normal orientation)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0; i < nseg; ++i) {
      const Seg sg = get_segment(a, cta, G, i, su0, su1);
      int p, q;
      raster_tile(sg.tile, a, p, q);
      if (!SWAP && sg.slot != 0) prefetch_residual<BN, EPI>(a, p * 128 + sub * 32 + lane, q * BN, half);
      mbar_wait_sleepy(&tfull[acc], acc_phase);
      if (i == 0 && threadIdx.x == 64) HY_TR(6);
      tc_fence_after();
      const int lrow = sub * 32 + lane;  // tile row (TMEM lane) owned by this thread
      const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
      bool finish = true;
      int c0 = 0, c1 = -1;
      long long ub = 0;
      if (sg.slot >= 0) {
        ub = (long long)sg.sk * a.nkb;
        c0 = (int)(((ub + 1) * G - 1) / a.u_sk);
        c1 = (int)(((ub + a.nkb) * G - 1) / a.u_sk);
        int* ctr = a.counters + sg.sk * 8 + half * 4 + sub;
        // the CTA's last segment usually finishes after every other contributor of its
        // tile: then it skips publishing its own partial (the end-of-kernel burst of
        // partial traffic, when every CTA finishes at once, is what made stream-K slow)
        if (!sk_all_arrived(ctr, c1 - c0, sg.slot, lane)) {
          // stream-K partial: publish raw accumulators, then count arrivals
          // layout [cta][slot][chunk][j/4][128 rows] float4: lane-consecutive 16B stores
          float4* mine = reinterpret_cast<float4*>(a.partial) +
                         (size_t)(cta * 2 + sg.slot) * (BN / 32) * 8 * 128 + lrow;
#pragma unroll 1
          for (int c = half; c < BN / 32; c += 2) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              __stcg(mine + (c * 8 + j / 4) * 128,
                     make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                 __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
          }
          __threadfence();
          __syncwarp();
          int prev = 0;
          if (lane == 0) prev = atomicAdd(ctr, 1);
          prev = __shfl_sync(0xffffffffu, prev, 0);
          finish = prev == c1 - c0;  // the last contributor reduces and writes the tile
          if (finish) __threadfence();
        }
        if (finish && lane == 0) *ctr = 0;  // ready for the next GEMM on this workspace
      }
      if (finish) {
#pragma unroll 1
        for (int c = half; c < BN / 32; c += 2) {
          uint32_t r[32];
          if (i == 0 && c == 0 && threadIdx.x == 64) HY_TR(9);
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
          if (i == 0 && c == 0 && threadIdx.x == 64) HY_TR(10);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          // other contributors' partials (<= 3 by construction of the grid), all loads
          // issued before any add so the L2 round trips overlap
          const float4* srcs[3];
          int ns = 0, nb = 0;
          for (int cc = c0; cc <= c1 && ns < 3; ++cc) {
            if (cc == cta) {
              nb = ns;
              continue;
            }
            const long long cu0 = (long long)cc * a.u_sk / G;
            const int slot = cu0 >= ub ? 0 : 1;
            srcs[ns++] = reinterpret_cast<const float4*>(a.partial) +
                         ((size_t)(cc * 2 + slot) * (BN / 32) + c) * 8 * 128 + lrow;
          }
          add_partials(v, srcs, ns, nb);
          epi_chunk<EPI, SWAP>(a, p * 128 + sub * 32, q * BN + c * 32, v, lane,
                               smem_u32(stg_base) + (warp - 2) * kStgBytes, &tmC, nst);
          if (i == 0 && c == 0 && threadIdx.x == 64) HY_TR(11);
          if (i == 0 && c == 1 && threadIdx.x == 64) HY_TR(12);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (i == 0 && threadIdx.x == 64) HY_TR(7);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // TMA stores done reading shared memory
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
    if (lane == 0) {
      HY_TR(8);
      HY_CM(3);
    }
  }
}

// ---------------------------------------------------------------------------
// K1c: swap-AB decode GEMM split over K inside a thread-block cluster.  The KS CTAs of a
// cluster share one 128-row weight tile, rank r reducing k-blocks [r nkb / KS, (r+1) nkb / KS)
// -- so a decode GEMM with few weight tiles (N = 4096: 32 tiles) still streams its weights
// through ~all SMs -- and the partial sums meet in DISTRIBUTED shared memory: ranks 1..KS-1
// store their fp32 accumulators into rank 0's reduction buffer (st.shared::cluster), one
// cluster barrier (release / acquire), and rank 0 adds them in rank order (deterministic)
// and runs the swap epilogue.  This replaces stream-K's global partials, fences and arrival
// atomics (a 3-4 us tail) with one DSMEM round trip.
// ---------------------------------------------------------------------------
template <int BN>
struct CskCfg {
  static constexpr int BK = 64;
  static constexpr int A_BYTES = 128 * BK * 2;  // weight rows (MMA-M)
  static constexpr int B_BYTES = BN * BK * 2;   // token rows (MMA-N)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RED_SLOT = 128 * BN * 4;  // one rank's fp32 accumulator
  static constexpr int EPI_WARPS = 4;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  // ring: the peers' partials land in rank 0's operand ring once its main loop is done, so
  // the slots need no shared memory of their own -- the ring must hold ks - 1 of them
  static int smem_bytes(int stages, int ks, bool ring = false) {
    const int ops = ring ? std::max(stages * STAGE_BYTES, (ks - 1) * RED_SLOT)
                         : stages * STAGE_BYTES + (ks - 1) * RED_SLOT;
    return ops + EPI_WARPS * kStgBytes + 1024 + 256;
  }
};

// NRM = true: the normal orientation (MMA-M = 128 token rows, MMA-N = BN weight rows, tile
// t = (token tile t % np, weight tile t / np)) for 65-256 token rows with few weight tiles
template <int BN, int EPI, bool NRM = false>
__global__ void __launch_bounds__(64 + 32 * 4, 1)
    gemm_swap_csk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                         const GemmArgs a, int stages, int ks) {
  using C = CskCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * C::A_BYTES;
  // [ks - 1][BN / 32][8][128] float4 (rank 0 only): behind the ring, or over it (dbg & 32)
  const bool ring = (a.dbg & 32) != 0;
  uint8_t* red = ring ? smem : sB + stages * C::B_BYTES;
  uint8_t* stg = ring ? smem + std::max(stages * C::STAGE_BYTES, (ks - 1) * C::RED_SLOT)
                      : red + (ks - 1) * C::RED_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + C::EPI_WARPS * kStgBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + stages;
  uint64_t* tfull = bars + 2 * stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int tile = blockIdx.x / ks;
  const int p = NRM ? tile % a.np : tile;  // swap: weight tile; normal: token tile
  const int q = NRM ? tile / a.np : 0;     // normal: weight tile
  const int kb0 = (int)((long long)rank * a.nkb / ks), kb1 = (int)((long long)(rank + 1) * a.nkb / ks);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see gemm_tc_kernel)
  // every CTA of the cluster must have started before a peer writes its shared memory:
  // arrive now, wait only where it matters (before the remote stores / the final barrier).
  // Ring mode: rank 0 arrives only once its operand ring is free (after its role below), so
  // this barrier phase also tells the peers that the reduction slots may be written.
  if (!(ring && rank == 0)) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // weights of the first stages before the grid dependency resolves; the activations
      // too when launched without PDL
      int npre = 0;
      // swap: weights in the A slot (128 rows), tokens in B; normal: tokens in A, weights in B
      auto load_w = [&](int st, int kb) {
        if (NRM)
          tma_load_2d(&tmW, &full[st], sB + st * C::B_BYTES, kb * C::BK, q * BN, kEvictNormal);
        else
          tma_load_2d(&tmW, &full[st], sA + st * C::A_BYTES, kb * C::BK, p * 128, kEvictFirst);
      };
      auto load_x = [&](int st, int kb) {
        if (NRM)
          tma_load_2d(&tmX, &full[st], sA + st * C::A_BYTES, kb * C::BK, p * 128, kEvictLast);
        else
          tma_load_2d(&tmX, &full[st], sB + st * C::B_BYTES, kb * C::BK, 0, kEvictLast);
      };
      for (int kb = kb0; kb < kb1 && npre < stages; ++kb, ++npre) {
        mbar_expect_tx(&full[npre], C::STAGE_BYTES);
        load_w(npre, kb);
        if (a.dbg & 16) load_x(npre, kb);
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        if (g < npre) {
          if (!(a.dbg & 16)) load_x(stage, kb);
        } else {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          load_w(stage, kb);
          load_x(stage, kb);
        }
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k)
          umma_bf16(tmem_base, smem_desc_k_sw128(a_addr + k * 32), smem_desc_k_sw128(b_addr + k * 32),
                    idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[stage]);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(tfull);
    }
  } else if (rank != 0) {
    // ---- ranks 1..ks-1: accumulators into rank 0's reduction buffer (lane-coalesced float4)
    const int sub = warp & 3;
    const int lrow = sub * 32 + lane;
    mbar_wait_sleepy(tfull, 0);
    tc_fence_after();
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // rank 0 has started
    const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16);
    const uint32_t dst = mapa_shared(smem_u32(red + (rank - 1) * C::RED_SLOT), 0);
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + c * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                         dst + (uint32_t)(((c * 8 + j / 4) * 128 + lrow) * 16)),
                     "r"(r[j]), "r"(r[j + 1]), "r"(r[j + 2]), "r"(r[j + 3])
                     : "memory");
    }
  }
  if (ring && rank == 0) {
    // ring mode: rank 0's main loop is over once the accumulator is complete (every TMA write
    // into the ring was consumed by an MMA that has finished reading it)
    if (warp >= 2) {
      mbar_wait_sleepy(tfull, 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  // every thread of every CTA: the remote stores are visible to rank 0 past this barrier
  if (!(warp >= 2 && rank != 0)) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  tc_fence_before();
  cluster_sync();
  if (rank == 0 && warp >= 2) {
    // ---- rank 0: own accumulators + the others' in rank order, then the swap epilogue
    const int sub = warp & 3;
    const int lrow = sub * 32 + lane;
    mbar_wait_sleepy(tfull, 0);
    tc_fence_after();
    const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16);
    int nst = 0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + c * 32, r);
      tmem_ld_wait();
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      for (int r2 = 0; r2 < ks - 1; ++r2) {
        const uint32_t src = smem_u32(red + r2 * C::RED_SLOT);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 f = lds_f32x4(src + (uint32_t)(((c * 8 + j / 4) * 128 + lrow) * 16));
          v[j] += f.x;
          v[j + 1] += f.y;
          v[j + 2] += f.z;
          v[j + 3] += f.w;
        }
      }
      if (NRM)
        epi_chunk<EPI, false>(a, p * 128 + sub * 32, q * BN + c * 32, v, lane,
                              smem_u32(stg) + (warp - 2) * kStgBytes, nullptr, nst);
      else
        epi_chunk<EPI, true>(a, p * 128 + sub * 32, c * 32, v, lane,
                             smem_u32(stg) + (warp - 2) * kStgBytes, nullptr, nst);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int EPI, bool NRM = false>
static int launch_csk(const CUtensorMap& tW, const CUtensorMap& tX, const GemmArgs& a, int tiles,
                      int ks, int stages, cudaStream_t st) {
  using C = CskCfg<BN>;
  const int smem = C::smem_bytes(stages, ks, (a.dbg & 32) != 0);
  auto kern = gemm_swap_csk_kernel<BN, EPI, NRM>;
  HY_CUDA_RET(ensure_smem(kern, 227 * 1024));
  HY_CUDA_RET(ensure_max_carveout(kern));
  HY_CUDA_RET(launch_pdl_cluster(kern, dim3(tiles * ks), dim3(C::THREADS), (size_t)smem, ks, st,
                                 tW, tX, a, stages, ks));
  HY_LAUNCH_CHECK();
  return 0;
}

template <int BN, bool NRM = false>
static int launch_csk_epi(int epi, const CUtensorMap& tW, const CUtensorMap& tX, const GemmArgs& a,
                          int tiles, int ks, int stages, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_csk<BN, EPI_BF16, NRM>(tW, tX, a, tiles, ks, stages, st);
    case EPI_QGELU: return launch_csk<BN, EPI_QGELU, NRM>(tW, tX, a, tiles, ks, stages, st);
    case EPI_GELU: return launch_csk<BN, EPI_GELU, NRM>(tW, tX, a, tiles, ks, stages, st);
    case EPI_SWIGLU: return launch_csk<BN, EPI_SWIGLU, NRM>(tW, tX, a, tiles, ks, stages, st);
    case EPI_F32: return launch_csk<BN, EPI_F32, NRM>(tW, tX, a, tiles, ks, stages, st);
    default: return -1;
  }
}

// Decode GEMMs of 65-128 token rows with a long reduction (the down projections, K >= 8192)
// in the swap orientation with 128-wide token tiles (partials in rank 0's operand ring):
// measured faster there (LLaVA down M = 96 28.3 -> 26.0 us, Qwen2-VL down M = 128 39.6 ->
// 33.3) and slower for K = 3584-4096 (o M = 128 15.4 -> 17.7), which keep the normal-
// orientation cluster split-K.  HY_GEMM_SWAP128=0 / 1 forces it off / on (A/B).
static bool swap128_csk(int K) {
  const char* e = getenv("HY_GEMM_SWAP128");
  if (e) return e[0] != '0';
  return K >= 8192;
}

// Can `clusters` clusters of ks CTAs (smem bytes each) be resident at once?  A cluster sits
// inside one GPC, so with one CTA per SM fewer ks-clusters fit than SMs / ks suggests (B200:
// 28 clusters of 5 do not -- the Qwen2-VL down projection at M = 32 ran in two waves, 41.8 us
// vs 26.4 us for clusters of 4).  Occupancy is the same for every epilogue instance.
template <int BN, bool NRM>
static bool csk_resident(int clusters, int ks, int smem) {
  auto kern = gemm_swap_csk_kernel<BN, EPI_BF16, NRM>;
  if (ensure_smem(kern, 227 * 1024) != cudaSuccess) return false;
  if (ensure_max_carveout(kern) != cudaSuccess) return false;
  return max_active_clusters(kern, ks, CskCfg<BN>::THREADS, smem) >= clusters;
}

// ---------------------------------------------------------------------------
// K1b: CTA-pair GEMM (tcgen05.mma.cta_group::2), normal orientation, pair tile 256 x BN.
//
// The two CTAs of a cluster sit on the two SMs of one TPC.  Each loads its own 128 token
// rows of A and its own half (BN/2 rows) of the weight tile, so every byte staged in
// shared memory feeds twice the MMA work of the single-CTA kernel (256 x BN x 64 per
// stage pair) -- half the shared-memory traffic per flop, which is what lets the tensor
// pipe run at full rate inside the power cap.  The leader CTA (rank 0) alone issues the
// MMAs; both CTAs' TMA loads complete on the leader's full barrier, the MMA commits
// multicast to both CTAs' empty / accumulator-full barriers, and both CTAs' epilogue warps
// release the accumulator on the leader's accumulator-empty barrier.  Each CTA's TMEM
// holds its own 128 rows of the 256 x BN accumulator (double-buffered).
// ---------------------------------------------------------------------------
// SLIM (co-resident mode): a 160 KB operand ring and one 2 KB TMA-store buffer per epilogue
// warp -- 181.5 KB instead of 225 KB at BN = 256, which leaves ~44 KB of the SM's shared
// memory to a co-resident decode-attention CTA (attn_decode.cu) while this GEMM runs.
template <int BN, bool SLIM = false>
struct GemmPairCfg {
  static constexpr int BK = 64;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = ((SLIM ? 160 : HY_PAIR_SMEM_KB) * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int STG_BYTES = SLIM ? kStgBytes / 2 : kStgBytes;  // per epilogue warp
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + kEpiWarps * STG_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 64 + 32 * kEpiWarps;
};

template <int BN, int EPI, bool SLIM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * kEpiWarps, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const GemmArgs a) {
  using C = GemmPairCfg<BN, SLIM>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* stg_base = smem + C::STAGES * C::STAGE_BYTES;  // epilogue TMA-store buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + kEpiWarps * C::STG_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  if (threadIdx.x == 0) HY_CM(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    fence_mbar_init();
  }
  // both CTAs of the pair reach the collective allocation together (a cta_group::2 alloc
  // before the peer has started was the one compute-sanitizer racecheck hazard)
  cluster_sync();
  if (warp == 1) tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!(a.dbg & 9)) pdl_trigger();  // after both CTAs hold their TMEM: see gemm_tc_kernel
  int su0, su1;
  const int nseg = cta_segments(a, pair, npairs, su0, su1);  // data-parallel + stream-K

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      const int rowA = rank * 128, rowB = rank * (BN / 2);
      auto load_w = [&](int st, int kb, int q) {
        if (rank == 0) mbar_expect_tx(&full[st], 2 * C::STAGE_BYTES);
        tma_load_2d_cg2(&tmB, mapa_shared(smem_u32(&full[st]), 0), sB + st * C::B_BYTES,
                        kb * C::BK, q * BN + rowB, kEvictNormal);
      };
      auto load_x = [&](int st, int kb, int p) {
        tma_load_2d_cg2(&tmA, mapa_shared(smem_u32(&full[st]), 0), sA + st * C::A_BYTES,
                        kb * C::BK, p * 256 + rowA, kEvictNormal);
      };
      // weights of the first stages before the grid dependency resolves
      int npre = 0;
      for (int i = 0; i < nseg && npre < C::STAGES; ++i) {
        const Seg sg = get_segment(a, pair, npairs, i, su0, su1);
        int p, q;
        raster_tile(sg.tile, a, p, q);
        for (int kb = sg.kb0; kb < sg.kb1 && npre < C::STAGES; ++kb, ++npre) {
          load_w(npre, kb, q);
          if (a.dbg & 16) load_x(npre, kb, p);  // no PDL: see gemm_tc_kernel
        }
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = get_segment(a, pair, npairs, i, su0, su1);
        int p, q;
        raster_tile(sg.tile, a, p, q);
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++g) {
          if (g < npre) {
            if (!(a.dbg & 16)) load_x(stage, kb, p);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            load_w(stage, kb, q);
            load_x(stage, kb, p);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (a.dbg & 8) pdl_trigger();  // late trigger (see gemm_tc_kernel)
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA only) ----------------
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = get_segment(a, pair, npairs, i, su0, su1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          if (i == 0 && kb == sg.kb0) HY_CM(1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)
            umma_bf16_cg2(d_tmem, smem_desc_k_sw128(a_addr + k * 32),
                          smem_desc_k_sw128(b_addr + k * 32), idesc,
                          (kb > sg.kb0 || k > 0) ? 1u : 0u);
          umma_commit_cg2(&empty[stage], 0x3);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2(&tfull[acc], 0x3);
        if (i == nseg - 1) {
          HY_CM(2);
          HY_CNT(4, nseg);
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9 (both CTAs) ----------------
    pdl_wait();
    const int sub = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int nst = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0; i < nseg; ++i) {
      const Seg sg = get_segment(a, pair, npairs, i, su0, su1);
      int p, q;
      raster_tile(sg.tile, a, p, q);
      if (sg.slot != 0) prefetch_residual<BN, EPI>(a, p * 256 + rank * 128 + sub * 32 + lane, q * BN, half);
      mbar_wait_sleepy(&tfull[acc], acc_phase);
      const bool mark = i == nseg - 1 && warp == 2 && lane == 0;
      if (mark) HY_CM(6);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
      const int lrow = sub * 32 + lane;  // this CTA's accumulator row (TMEM lane)
      bool finish = true;
      int c0 = 0, c1 = -1;
      long long ub = 0;
      if (sg.slot >= 0) {
        // stream-K partial of this CTA's 128 rows: [pair][slot][rank][chunk][j/4][row] float4
        ub = (long long)sg.sk * a.nkb;
        c0 = (int)(((ub + 1) * npairs - 1) / a.u_sk);
        c1 = (int)(((ub + a.nkb) * npairs - 1) / a.u_sk);
        int* ctr = a.counters + sg.sk * 16 + rank * 8 + half * 4 + sub;
        if (!sk_all_arrived(ctr, c1 - c0, sg.slot, lane)) {  // see gemm_tc_kernel
          float4* mine = reinterpret_cast<float4*>(a.partial) +
                         ((size_t)(pair * 2 + sg.slot) * 2 + rank) * (BN / 32) * 8 * 128 + lrow;
#pragma unroll 1
          for (int c = half; c < BN / 32; c += 2) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              __stcg(mine + (c * 8 + j / 4) * 128,
                     make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                 __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
          }
          __threadfence();
          __syncwarp();
          int prev = 0;
          if (lane == 0) prev = atomicAdd(ctr, 1);
          prev = __shfl_sync(0xffffffffu, prev, 0);
          finish = prev == c1 - c0;  // the last contributing pair reduces and writes the rows
          if (finish) __threadfence();
        }
        if (finish && lane == 0 && sub == 0 && half == 0) HY_CINC(5);
        if (finish && lane == 0) *ctr = 0;
      }
      if (mark) HY_CM(7);
      if (finish && sg.slot >= 0 && c1 - c0 == 1) {
        // two contributors: the other's partial of the next chunk is loaded while this
        // chunk's epilogue runs (one L2 round trip in flight, not one per chunk in series)
        const int other = c0 == pair ? c1 : c0;
        const long long cu0 = (long long)other * a.u_sk / npairs;
        const float4* obase = reinterpret_cast<const float4*>(a.partial) +
                              ((size_t)(other * 2 + (cu0 >= ub ? 0 : 1)) * 2 + rank) * (BN / 32) *
                                  8 * 128 + lrow;
        float4 fa[8], fb[8];
        ld_partial(fa, obase + (size_t)half * 8 * 128);
#pragma unroll
        for (int c = half; c < BN / 32; c += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          if (c + 2 < BN / 32) ld_partial(fb, obase + (size_t)(c + 2) * 8 * 128);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          add_one(v, fa, other < pair);
          epi_chunk<EPI, false, !SLIM>(a, p * 256 + rank * 128 + sub * 32, q * BN + c * 32,
                                       v, lane, smem_u32(stg_base) + (warp - 2) * C::STG_BYTES,
                                       &tmC, nst);
#pragma unroll
          for (int t = 0; t < 8; ++t) fa[t] = fb[t];
        }
      } else if (finish) {
#pragma unroll 1
        for (int c = half; c < BN / 32; c += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          const float4* srcs[3];
          int ns = 0, nb = 0;
          for (int cc = c0; cc <= c1 && ns < 3; ++cc) {
            if (cc == pair) {
              nb = ns;
              continue;
            }
            const long long cu0 = (long long)cc * a.u_sk / npairs;
            const int slot = cu0 >= ub ? 0 : 1;
            srcs[ns++] = reinterpret_cast<const float4*>(a.partial) +
                         (((size_t)(cc * 2 + slot) * 2 + rank) * (BN / 32) + c) * 8 * 128 + lrow;
          }
          add_partials(v, srcs, ns, nb);
          epi_chunk<EPI, false, !SLIM>(a, p * 256 + rank * 128 + sub * 32, q * BN + c * 32,
                                       v, lane, smem_u32(stg_base) + (warp - 2) * C::STG_BYTES,
                                             &tmC, nst);
        }
      }
      if (mark) HY_CM(8);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // TMA stores done reading shared memory
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no remote arrivals or pair MMAs in flight past this point
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
    if (lane == 0) HY_CM(3);
  }
}

template <int BN, int EPI, bool SLIM>
static int launch_pair(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC,
                       const GemmArgs& a, int grid, cudaStream_t st) {
  using C = GemmPairCfg<BN, SLIM>;
  auto kern = gemm_pair_kernel<BN, EPI, SLIM>;
  HY_CUDA_RET(ensure_smem(kern, C::SMEM_BYTES));
  // the maximum carveout, so the SM's shared-memory configuration does not change between a
  // GEMM and a small-smem kernel sharing the SM (a 196 KB split would fit this CTA alone)
  HY_CUDA_RET(ensure_max_carveout(kern));
  if (a.dbg & 2)
    kern<<<grid, C::THREADS, C::SMEM_BYTES, st>>>(tA, tB, tC, a);
  else
    HY_CUDA_RET(launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM_BYTES, st, tA, tB, tC, a));
  HY_LAUNCH_CHECK();
  return 0;
}

template <int BN, bool SLIM>
static int launch_pair_epi(int epi, const CUtensorMap& tA, const CUtensorMap& tB,
                           const CUtensorMap& tC, const GemmArgs& a, int grid, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_pair<BN, EPI_BF16, SLIM>(tA, tB, tC, a, grid, st);
    case EPI_QGELU: return launch_pair<BN, EPI_QGELU, SLIM>(tA, tB, tC, a, grid, st);
    case EPI_GELU: return launch_pair<BN, EPI_GELU, SLIM>(tA, tB, tC, a, grid, st);
    case EPI_SWIGLU: return launch_pair<BN, EPI_SWIGLU, SLIM>(tA, tB, tC, a, grid, st);
    case EPI_F32: return launch_pair<BN, EPI_F32, SLIM>(tA, tB, tC, a, grid, st);
    default: return -1;
  }
}

template <int BN, bool SWAP, int EPI>
static int launch_gemm(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC,
                       const GemmArgs& a, int grid, cudaStream_t st) {
  using C = GemmCfg<BN>;
  HY_CUDA_RET(ensure_smem(gemm_tc_kernel<BN, SWAP, EPI>, C::SMEM_BYTES));
  HY_CUDA_RET(ensure_max_carveout(gemm_tc_kernel<BN, SWAP, EPI>));  // see launch_pair
  HY_CUDA_RET(launch_pdl(gemm_tc_kernel<BN, SWAP, EPI>, dim3(grid), dim3(C::THREADS), C::SMEM_BYTES,
                         st, tA, tB, tC, a));
  HY_LAUNCH_CHECK();
  return 0;
}

template <bool SWAP, int EPI>
static int launch_bn(int bn, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC,
                     const GemmArgs& a, int grid, cudaStream_t st) {
  switch (bn) {
    case 32: return SWAP ? launch_gemm<32, SWAP, EPI>(tA, tB, tC, a, grid, st) : -1;
    case 64: return launch_gemm<64, SWAP, EPI>(tA, tB, tC, a, grid, st);
    case 128: return launch_gemm<128, SWAP, EPI>(tA, tB, tC, a, grid, st);
    case 256: return launch_gemm<256, SWAP, EPI>(tA, tB, tC, a, grid, st);
    default: return -1;
  }
}

template <bool SWAP>
static int launch_epi(int epi, int bn, const CUtensorMap& tA, const CUtensorMap& tB,
                      const CUtensorMap& tC, const GemmArgs& a, int grid, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_bn<SWAP, EPI_BF16>(bn, tA, tB, tC, a, grid, st);
    case EPI_QGELU: return launch_bn<SWAP, EPI_QGELU>(bn, tA, tB, tC, a, grid, st);
    case EPI_GELU: return launch_bn<SWAP, EPI_GELU>(bn, tA, tB, tC, a, grid, st);
    case EPI_SWIGLU: return launch_bn<SWAP, EPI_SWIGLU>(bn, tA, tB, tC, a, grid, st);
    case EPI_F32: return launch_bn<SWAP, EPI_F32>(bn, tA, tB, tC, a, grid, st);
    default: return -1;
  }
}

// Workspace layout: [counters: 16 KiB][partials: G * 2 * 128 * BN fp32].  The counter
// region must be zero before first use; every call leaves it zeroed again.
static constexpr size_t kCounterBytes = 16384;

// HY_PDL_LATE=1 (with HY_PDL=1): GEMMs release their dependents after the last operand load
// instead of at entry, so an early dependent does not sit on SMs for the whole main loop
static bool pdl_late() {
  static const bool on = [] {
    const char* e = getenv("HY_PDL_LATE");
    return e && e[0] == '1';
  }();
  return on;
}

// SMs a GEMM grid may occupy (HY_GEMM_SMS caps it, e.g. to leave SMs to a concurrent stream)
static thread_local int t_sms_cap = 0;  // per-thread cap (split-mode forwards)
void gemm_set_sms_cap(int sms) { t_sms_cap = sms; }
// co-resident mode (per host thread): pair GEMMs use the SLIM instance
static thread_local int t_slim = 0;
void gemm_set_coresident(int on) { t_slim = on; }

static int gemm_sms() {
  static const int env_cap = [] {
    const char* e = getenv("HY_GEMM_SMS");
    return e ? atoi(e) : 0;
  }();
  const int cap = t_sms_cap > 0 ? (env_cap > 0 ? std::min(env_cap, t_sms_cap) : t_sms_cap) : env_cap;
  const int n = num_sms();
  return cap > 0 && cap < n ? cap : n;
}
// token rows from which the CTA-pair kernel is considered (tuned on B200,
// tools/kernel_sweep.py): from 385 rows the 256-row pair tiles cover the 128-row tiles
// without a half-empty pair row (M = 450-511: qkv / gate_up / down 8-16% faster as pairs;
// M = 257-384 stays single-CTA, where the pair lost up to 35%)
static constexpr int kPairMinRows = 385;

// Output map for the normal orientation's TMA-store epilogue: bf16 output without a row
// map, 16B-aligned base (ldc % 8 == 0 is checked by the caller); box 32 rows x 32 outputs
// (16 for SwiGLU, whose chunks emit half their columns).  Otherwise a.tma_out stays 0 and
// the epilogue stores rows directly.  HY_GEMM_NOTMASTORE=1 forces the direct stores (A/B).
static int out_tmap(CUtensorMap* tC, const HyGemmEpilogue* e, int M, int out_cols, GemmArgs& a) {
  a.tma_out = 0;
  if (e->out_f32 || e->row_map || ((uintptr_t)e->out & 15) || getenv("HY_GEMM_NOTMASTORE"))
    return 0;
  const int oc = e->act == HY_ACT_SWIGLU ? 16 : 32;
  HY_RET_IF(make_tmap_2d_bf16(tC, e->out, M, out_cols, (uint64_t)e->ldc * 2, 32, oc, 0));
  a.tma_out = 1;
  return 0;
}

// Whole tiles before the stream-K part: all but the last 1-2 waves' worth, so every
// stream-K share is >= one tile of k-blocks.  (Splitting only the remainder wave -- fewer
// partial round trips, shares below a tile -- measured no better on B200: o/down
// projections at M = 640-3600, tools/kernel_sweep.py.)
static int sk_dp_tiles(int T, int G) { return T >= 2 * G ? (T / G - 1) * G : 0; }

// Measured dispatch (tools/gemm_tune.py on a B200, generated into gemm_table.inc): for the
// served models' (N, K) pairs, the fastest kernel configuration at a grid of token counts.
// An entry covers M up to m_max (the grid point; entries of one (N, K) ascend in m_max).
// Shapes outside the table use the wave heuristic below.
struct GemmTableEntry {
  int n, k, m_max;
  int kind;  // 1 swap-AB, 2 single-CTA normal, 3 CTA pair
  int bn;    // tile width (pair: 128 / 256; single / swap: 32-256)
  int sk;    // stream-K: 0 off, 1 on
};
static const GemmTableEntry kGemmTable[] = {
#include "gemm_table.inc"
    {0, 0, 0, 0, 0, 0}};

static const GemmTableEntry* gemm_table_lookup(int M, int N, int K) {
  static const bool off = getenv("HY_GEMM_NOTABLE") != nullptr;
  if (off) return nullptr;
  for (const GemmTableEntry* e = kGemmTable; e->n; ++e)
    if (e->n == N && e->k == K && M <= e->m_max) return e;
  return nullptr;  // another shape, or beyond the measured range: the heuristic
}

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

  if (force_mode == 0)
    if (const char* fm = getenv("HY_GEMM_MODE")) force_mode = atoi(fm);  // tuning only
  // measured table (when no tuning override forces the mode)
  int tab_bn = 0, tab_sk = -1;
  if (force_mode == 0 && !getenv("HY_GEMM_BN") && !getenv("HY_PAIR_BN") && !t_slim) {
    if (const GemmTableEntry* te = gemm_table_lookup(M, N, K)) {
      if (te->kind == 3 && N % te->bn == 0 && N % 128 == 0) {
        force_mode = 3;
      } else if (te->kind == 2 && N % 128 == 0 && N % te->bn == 0) {
        force_mode = 2;
      } else if (te->kind == 1) {
        force_mode = 1;
      }
      if (force_mode) {
        tab_bn = te->bn;
        tab_sk = te->sk;
      }
    }
  }
  // CTA-pair kernel: large token counts, weight rows a multiple of 256
  // when it needs no more full waves than the single-CTA kernel (a pair tile takes about as
  // long on two SMs as a 128-row tile on one, so waves decide)
  // Estimated time in units of one 256x256 pair-tile wave: full waves x relative tile time
  // (single-CTA 128x256 tiles: ~12% less efficient than a pair tile).
  bool pair = force_mode == 3;
  int pair_bn = 256;
  int single_bn = 0;  // 0: default width for the single-CTA normal orientation
  if (force_mode == 0 && M >= kPairMinRows && N % 256 == 0 && !getenv("HY_GEMM_NOPAIR")) {
    const int sms = gemm_sms();
    const double t256 = ceil_div(ceil_div(M, 256) * (N / 256), sms / 2);
    const double t128 = 0.55 * ceil_div(ceil_div(M, 256) * (N / 128), sms / 2);
    const double t1 = 1.12 * ceil_div(ceil_div(M, 128) * (N / 256), sms);
    // single-CTA 128x128 tiles: half the work of a 128x256 tile, less efficient per byte of
    // shared memory; they win when the bigger tiles leave most SMs idle (ViT batches of a
    // few images: M ~ 600-1800, N = 1024-3072)
    // (only for short K: with long K loops the 128x128 tile's shared-memory bandwidth per
    // flop dominates -- 1600x4096x4096 measured 78 us on 128x128 vs 48 us on pair tiles)
    const double t1n = K <= 2048 ? 0.62 * ceil_div(ceil_div(M, 128) * (N / 128), sms) : 1e30;
    // 128x64 tiles for the smallest of these (one or two images: a handful of 128x128 tiles)
    const double t1q = K <= 2048 && !getenv("HY_GEMM_NO64") ? 0.38 * ceil_div(ceil_div(M, 128) * (N / 64), sms) : 1e30;
    pair = t256 <= std::min(std::min(t1, t1n), t1q);
    if (!pair && std::min(t1n, t1q) < t1 && !getenv("HY_GEMM_NO128"))
      single_bn = t1q < t1n ? 64 : 128;
    // 128-wide pair tiles fill waves better on paper (t128) but measured slower inside the
    // serving sequence (tools/batch_bench.py: 2816-token prefill 42.2 vs 38.8 ms); they are
    // kept for N % 256 != 0 and HY_PAIR_BN=128 experiments
    (void)t128;
  } else if (force_mode == 3 && N % 256 != 0) {
    pair_bn = 128;
  }
  if (pair && tab_bn) pair_bn = tab_bn;
  if (const char* e = getenv("HY_PAIR_BN")) pair_bn = atoi(e);  // tuning only
  if (pair) {
    HY_CHECK_ARG(N % pair_bn == 0, "pair kernel needs N % 128 == 0");
    a.np = ceil_div(M, 256);
    a.nq = N / pair_bn;
    a.nkb = ceil_div(K, 64);
    const int T = a.np * a.nq;
    const int slots = gemm_sms() / 2;
    // Stream-K over pairs for the last, partial wave (same schedule as the single-CTA
    // kernel, per CTA half of the 256-row tile).  Opt-in (HY_PAIR_SK=1): measured on B200
    // it does not pay for the serving shapes -- the fp32 partial round trip and the
    // last-arriver fixup cost more than the idle pairs of the tail wave (e.g. 1600x4096x4096
    // 69.8 us with, 54.8 us without; tools/kernel_sweep.py).
    const size_t need = kCounterBytes + (size_t)slots * 2 * 2 * 128 * pair_bn * sizeof(float);
    const double dp_eff = (double)T / ((double)ceil_div(T, slots) * slots);
    const bool want_sk = tab_sk >= 0 ? tab_sk == 1 : getenv("HY_PAIR_SK") != nullptr;
    bool sk = ws != nullptr && ws_bytes >= need && dp_eff < 0.9 && a.nkb >= 16 &&
              (long long)T * a.nkb < (1LL << 31) && want_sk;
    int grid;
    if (!sk) {
      grid = 2 * std::min(T, slots);
      a.t_dp = T;
      a.u_sk = 0;
    } else {
      const int G = std::min(slots, T >= slots ? slots : 3 * T);
      a.t_dp = sk_dp_tiles(T, G);
      a.u_sk = (long long)(T - a.t_dp) * a.nkb;
      a.counters = reinterpret_cast<int*>(ws);
      a.partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kCounterBytes);
      grid = 2 * G;
    }
    // HY_PAIR_DBG=1: no early release of dependents (bisection aid; the serving hang it
    // isolated was a trigger issued before the TMEM allocation, see gemm_tc_kernel)
    a.dbg = pdl_late() ? 8 : 0;
    if (const char* d = getenv("HY_PAIR_DBG")) a.dbg = atoi(d);
    if (!pdl_enabled() || (a.dbg & 2)) a.dbg |= 16;  // no PDL launch: early activation loads
    if (getenv("HY_GEMM_NOPREF")) a.dbg |= 4;  // A/B: no residual L2 prefetch
    if (const char* g = getenv("HY_GEMM_GROUP")) a.group = atoi(g);
    CUtensorMap tA, tB;
    HY_RET_IF(make_tmap_2d_bf16(&tA, A, M, K, (uint64_t)lda * 2, 128, 64));
    HY_RET_IF(make_tmap_2d_bf16(&tB, W, N, K, (uint64_t)ldw * 2, pair_bn / 2, 64));
    CUtensorMap tC = tA;
    HY_RET_IF(out_tmap(&tC, e, M, out_cols, a));
    const bool slim = t_slim || getenv("HY_GEMM_SLIM") != nullptr;
    const int rc = pair_bn == 128 ? (slim ? launch_pair_epi<128, true>(epi, tA, tB, tC, a, grid, st)
                                          : launch_pair_epi<128, false>(epi, tA, tB, tC, a, grid, st))
                                  : (slim ? launch_pair_epi<256, true>(epi, tA, tB, tC, a, grid, st)
                                          : launch_pair_epi<256, false>(epi, tA, tB, tC, a, grid, st));
    if (rc < 0) {
      set_last_error("gemm: no pair kernel for this epilogue");
      return (int)cudaErrorInvalidValue;
    }
    return rc;
  }
  // 65-256 token rows with few weight tiles (o / down projections of decode-heavy batches):
  // normal-orientation 128 x BN tiles split over K inside a cluster (K1c, NRM), reduced
  // through DSMEM -- the tile count that fills the most SMs wins (BN 128 or 64)
  if (M > (swap128_csk(K) ? 128 : 64) && M <= 256 && force_mode == 0 && N % 128 == 0 &&
      !getenv("HY_GEMM_NONCSK")) {
    const int sms = gemm_sms();
    const int np = ceil_div(M, 128), nkb = ceil_div(K, 64);
    int best_bn = 0, best_ks = 0, best_st = 0, best_ctas = 0;
    for (int cbn : {128, 64}) {
      const int T = np * (N / cbn);
      if (2 * T > sms) continue;
      const int slot = 128 * cbn * 4, stage = (128 + cbn) * 64 * 2;
      for (int ks = std::min(8, sms / T); ks >= 2; --ks) {
        if (nkb / ks < 4) continue;
        const int stages = std::min(8, (227 * 1024 - (ks - 1) * slot - 4 * kStgBytes - 1280) / stage);
        if (stages < 3) continue;
        const int smem = stages * stage + (ks - 1) * slot + 4 * kStgBytes + 1280;
        if (!(cbn == 128 ? csk_resident<128, true>(T, ks, smem) : csk_resident<64, true>(T, ks, smem)))
          continue;  // the clusters would not all be resident: fewer, longer splits
        if (T * ks > best_ctas) {
          best_bn = cbn;
          best_ks = ks;
          best_st = stages;
          best_ctas = T * ks;
        }
        break;
      }
    }
    if (best_ks >= 2) {
      a.np = np;
      a.nq = N / best_bn;
      a.nkb = nkb;
      if (!pdl_enabled()) a.dbg |= 16;
      CUtensorMap tW, tX;
      HY_RET_IF(make_tmap_2d_bf16(&tX, A, M, K, (uint64_t)lda * 2, 128, 64));
      HY_RET_IF(make_tmap_2d_bf16(&tW, W, N, K, (uint64_t)ldw * 2, best_bn, 64));
      const int tiles = a.np * a.nq;
      const int rc = best_bn == 128
                         ? launch_csk_epi<128, true>(epi, tW, tX, a, tiles, best_ks, best_st, st)
                         : launch_csk_epi<64, true>(epi, tW, tX, a, tiles, best_ks, best_st, st);
      if (rc < 0) {
        set_last_error("gemm: no cluster split-K kernel for this epilogue");
        return (int)cudaErrorInvalidValue;
      }
      return rc;
    }
  }
  const bool swap = (force_mode == 1) || (force_mode == 0 && M <= 256);
  int bn;
  if (swap) {
    bn = M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
    a.P = N;
    a.Q = M;
  } else {
    bn = single_bn ? single_bn : (N % 256 == 0) ? 256 : 128;
    HY_CHECK_ARG(N % 128 == 0, "normal orientation needs N % 128 == 0");
    a.P = M;
    a.Q = N;
  }
  if (tab_bn) bn = tab_bn;
  if (const char* env_bn = getenv("HY_GEMM_BN")) bn = atoi(env_bn);  // tuning only
  if (pdl_late()) a.dbg |= 8;
  if (!pdl_enabled()) a.dbg |= 16;  // no PDL launch: early activation loads
  if (getenv("HY_GEMM_NOPREF")) a.dbg |= 4;  // A/B: no residual L2 prefetch
  if (const char* g = getenv("HY_GEMM_GROUP")) a.group = atoi(g);
  a.np = ceil_div(a.P, 128);
  a.nq = ceil_div(a.Q, bn);
  a.nkb = ceil_div(K, 64);
  const int T = a.np * a.nq;
  const int sms = gemm_sms();
  // decode GEMMs with few weight tiles (M <= 64, 128-row weight tiles * 2 <= SMs): split K
  // inside a cluster, reduced through distributed shared memory (K1c) -- HY_GEMM_NOCSK=1 off
  const char* csk_env = getenv("HY_GEMM_CSK");  // tuning: cluster size (any weight-tile count)
  if (swap && M <= (swap128_csk(K) ? 128 : 64) && (2 * a.np <= sms || csk_env) &&
      !getenv("HY_GEMM_NOCSK") && !(a.dbg & 2)) {
    // 65-128 token rows: 128-wide token tiles, whose 64 KB partials fit only inside rank 0's
    // operand ring (ring mode)
    const int cbn = M <= 32 ? 32 : M <= 64 ? 64 : 128;
    const bool ring = cbn == 128;
    const int stage = cbn == 32 ? CskCfg<32>::STAGE_BYTES
                      : cbn == 64 ? CskCfg<64>::STAGE_BYTES : CskCfg<128>::STAGE_BYTES;
    const int slot = cbn == 32 ? CskCfg<32>::RED_SLOT
                     : cbn == 64 ? CskCfg<64>::RED_SLOT : CskCfg<128>::RED_SLOT;
    auto smem_for = [&](int st, int k) {
      return (ring ? std::max(st * stage, (k - 1) * slot) : st * stage + (k - 1) * slot) +
             4 * kStgBytes + 1024 + 256;
    };
    auto stages_for = [&](int k) {
      const int red = (k - 1) * slot;
      const int all = 227 * 1024 - 4 * kStgBytes - 1024 - 256;
      if (ring && red > all) return 0;
      const int budget = ring ? all : all - red;
      int n = std::min(8, budget / stage);
      if (const char* e = getenv("HY_GEMM_CSK_STAGES")) n = std::min(n, atoi(e));  // tuning
      return n;
    };
    int ks = std::min(8, sms / a.np);
    while (ks > 1 && a.nkb / ks < 4) --ks;
    // every weight tile's cluster resident in one wave (clusters sit inside a GPC)
    auto resident = [&](int k) {
      const int sm = smem_for(stages_for(k), k);
      return cbn == 32 ? csk_resident<32, false>(a.np, k, sm)
             : cbn == 64 ? csk_resident<64, false>(a.np, k, sm)
                         : csk_resident<128, false>(a.np, k, sm);
    };
    while (ks > 1 && (stages_for(ks) < 2 || !resident(ks))) --ks;
    if (csk_env) ks = std::max(1, std::min(8, atoi(csk_env)));
    if (ks >= 2) {
      const int stages = stages_for(ks);
      if (stages >= 2) {
        a.nq = 1;
        if (!pdl_enabled()) a.dbg |= 16;
        if (ring) a.dbg |= 32;
        CUtensorMap tW, tX;
        HY_RET_IF(make_tmap_2d_bf16(&tW, W, N, K, (uint64_t)ldw * 2, 128, 64));
        HY_RET_IF(make_tmap_2d_bf16(&tX, A, M, K, (uint64_t)lda * 2, cbn, 64));
        const int rc = cbn == 32   ? launch_csk_epi<32>(epi, tW, tX, a, a.np, ks, stages, st)
                       : cbn == 64 ? launch_csk_epi<64>(epi, tW, tX, a, a.np, ks, stages, st)
                                   : launch_csk_epi<128>(epi, tW, tX, a, a.np, ks, stages, st);
        if (rc < 0) {
          set_last_error("gemm: no cluster split-K kernel for this epilogue");
          return (int)cudaErrorInvalidValue;
        }
        return rc;
      }
    }
  }
  const size_t need = kCounterBytes + (size_t)sms * 2 * 128 * bn * sizeof(float);
  // stream-K when whole-tile waves would leave SMs idle.  Swap orientation (decode: weight
  // streaming, every SM must pull bytes): a mostly idle last wave (fill < 85%) or a single
  // wave under half full; normal orientation only
  // below 50% fill with a long K loop -- measured there, with K = 1024 or a >= 50% full wave
  // the fp32 partial round trip costs more than the idle SMs (tools/kernel_sweep.py)
  const double dp_eff = (double)T / ((double)ceil_div(T, sms) * sms);
  const bool units_fit = (long long)T * a.nkb < (1LL << 31);  // 32-bit segment math
  bool sk = ws != nullptr && ws_bytes >= need && units_fit &&
            (swap ? (a.nkb >= 4 && (T > sms ? dp_eff < 0.85 : dp_eff < 0.5))
                  : (dp_eff < 0.5 && a.nkb >= 32));
  if (tab_sk == 0) sk = false;
  if (tab_sk == 1) sk = ws != nullptr && ws_bytes >= need && units_fit;
  if (getenv("HY_GEMM_NOSK")) sk = false;
  if (getenv("HY_GEMM_SK")) sk = ws != nullptr && ws_bytes >= need && units_fit;
  int grid;
  if (!sk) {
    grid = std::min(T, sms);
    a.t_dp = T;
    a.u_sk = 0;
  } else {
    const long long U = (long long)T * a.nkb;
    // at most 4 contributors per stream-K tile (T < sms: grid <= 3T)
    grid = (int)std::min<long long>(std::min<long long>(sms, U), T >= sms ? sms : 3LL * T);
    a.t_dp = sk_dp_tiles(T, grid);
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
  CUtensorMap tC = tA;  // unused unless a.tma_out
  if (!swap) HY_RET_IF(out_tmap(&tC, e, M, out_cols, a));
  const int rc = swap ? launch_epi<true>(epi, bn, tA, tB, tC, a, grid, st)
                      : launch_epi<false>(epi, bn, tA, tB, tC, a, grid, st);
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
