// K7 paged prefill attention and K3 ViT varlen attention on 5th-generation tensor cores.
//
// One CTA = one (sequence, query head, two 128-row query tiles).  Warp-specialised:
//   warp 0      TMA producer: both Q tiles once, then K/V tiles of 128 keys into a 2-stage
//               ring (paged: eight 16-token cache blocks per tile through the block table;
//               varlen: the image's rows of the packed QKV buffer)
//   warp 1      single-thread tcgen05.mma issuer, per query tile t and key tile j:
//                 S_t = Q_t K_j^T  (M=128 queries, N=128 keys, K=d; fp32 in TMEM)
//                 O_t += P_t V_j   (M=128, N=d, K=128 keys; P_t read from TMEM where the
//                                   softmax wrote it over S_t, V as an MN-major operand
//                                   straight from its TMA tile)
//               ping-pong: the MMAs of one tile run while the other tile's softmax works
//   warps 2..9  softmax, 4 warps per query tile, one query row per thread: tcgen05.ld of
//               the S row, mask, online max/sum in the exp2 domain, P as bf16 pairs
//               tcgen05.st back into TMEM.  O stays in TMEM; it is rescaled (tcgen05.ld/st)
//               only when a row max grows by more than 2^8 -- P stays <= 256, exact in the
//               final O / l.  Finally O / l -> bf16 -> global.
//
// Same math as the mma.sync kernel it replaces, for d in {64, 128}, and d = 80 (Qwen2-VL's
// vision tower) as zero-padded d = 128 tiles (the softmax-bound kernel has tensor-pipe
// headroom for the 1.6x MMA work; attn_prefill.cu's mma.sync kernel is now only the
// HY_ATTN_FA2 A/B reference).
// Reference: epdsim prices prefill attention as 4 S^2 H per chunk (model_cost.py:189) and
// ViT attention as 4 T^2 H_v per image (model_cost.py:160-163).
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <cmath>

namespace hy {

#ifdef HY_ATRACE
// lab-only timeline of CTA 0: [event][j] globaltimer stamps
__device__ unsigned long long g_atrace[8][64];
#define ATR(ev, j)                                                         \
  do {                                                                     \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 64) {                  \
      unsigned long long t_;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));               \
      g_atrace[ev][j] = t_;                                                \
    }                                                                      \
  } while (0)
#else
#define ATR(ev, j)
#endif

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp, far below the bf16 rounding of P)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32x2 FMA / add (FFMA2 / FADD2: two lanes of math per issue slot -- the softmax
// is issue-bound once the S row is in registers)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair on the FMA pipe (FA4's trick for a softmax bound by the 16-per-clock SFU):
// x = n + f with n = round(x) from the 1.5 * 2^23 magic add, f in [-0.5, 0.5], 2^f by a
// degree-3 fit (max relative error 1.4e-4, far below the bf16 rounding of P), and n added
// to the exponent bits.  x is clamped at -127 (the result is then ~0, as P needs).
// HY_ATTN_POLY of every 16 pairs in a 32-key chunk take this path, the rest ex2.approx.
#ifndef HY_ATTN_POLY
#define HY_ATTN_POLY 6
#endif
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& e0, float& e1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  x0 = fmaxf(x0, -127.f);
  x1 = fmaxf(x1, -127.f);
  const uint64_t x2 = pk2(x0, x1);
  const uint64_t t2 = fadd2(x2, pk2(kMagic, kMagic));      // magic + round(x)
  const uint64_t r2 = fadd2(t2, pk2(-kMagic, -kMagic));    // round(x)
  const uint64_t f2 = ffma2(r2, pk2(-1.f, -1.f), x2);      // x - round(x)
  uint64_t p2 = ffma2(f2, pk2(0.05502927f, 0.05502927f), pk2(0.24225698f, 0.24225698f));
  p2 = ffma2(f2, p2, pk2(0.69325305f, 0.69325305f));
  p2 = ffma2(f2, p2, pk2(0.99995134f, 0.99995134f));
  float p0, p1, t0, t1;
  up2(p2, p0, p1);
  up2(t2, t0, t1);
  e0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  e1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

struct TcAttnParams {
  const int* qstart;   // [n_seqs + 1] query rows of each sequence in the Q map
  const int* offset;   // paged: tokens cached before the chunk
  const int* slots;    // paged: block-table row of each sequence
  const int* block_table;
  int bt_stride;
  int q_tiles;         // 256-row query-tile pairs per sequence in the grid
  int n_seqs;
  int group;           // query heads per kv head
  int k_col0, v_col0;  // varlen: column of kv head 0's K / V in the packed QKV map
  long long rows_per_block;  // paged: KV-map rows per cache block (block_stride / d)
  int rows_per_kv;     // paged: rows from a block's K half to its V half (n_kv * 16)
  float scale_log2;
  bf16* out;
  int ld_o;
};

template <int D, int T = 2>
struct TcAttnCfg {
  static constexpr int BQ = 128, BK = 128;
  // T = 2: two query tiles per CTA, 4 softmax warps each, ping-pong between the tiles.
  // T = 1: one query tile, 8 softmax warps (two threads per row, 64 keys each), S double-
  //        buffered over key tiles so Q K^T of tile j+1 runs under the softmax of tile j.
  // T = 3: two query tiles ping-ponging like T = 2, each with 8 softmax warps (two threads per
  //        row like T = 1): half the per-thread softmax chain, 16 softmax warps per CTA.
  static constexpr int TILES = T == 3 ? 2 : T;
  static constexpr int NC = D / 64;               // 64-wide d chunks (one 128B swizzle row)
  static constexpr int CHUNK = 128 * 128;         // bytes of one [128 rows][64 bf16] chunk
  static constexpr int Q_BYTES = NC * CHUNK;      // one query tile
  static constexpr int KV_BYTES = NC * CHUNK;     // K (or V) of one key tile
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int SMEM = TILES * Q_BYTES + 2 * STAGE_BYTES + 1024 + 256;
  // TMEM columns: tile t owns S_t (fp32, 128 cols) at t * 128, overwritten in place by P_t
  // (bf16 pairs, first 64 cols), and O_t at 256 + t * 128
  static constexpr int TMEM_COLS = 512;
  static constexpr int THREADS = T == 3 ? 64 + 512 : 64 + 256;
};

// DV: the real head dim when it is narrower than the D-wide tiles (varlen only): Q/K/V are
// fetched through a 3D map [rows][heads][DV] whose boxes past DV are zero-filled, so the
// padded dims add nothing to S and leave O's extra columns zero; only DV columns are stored.
#ifndef HY_ATTN_MAXNREG
#define HY_ATTN_MAXNREG 200
#endif
template <int D, bool PAGED, int T, int DV = D>
__global__ void __launch_bounds__(T == 3 ? 64 + 512 : 64 + 256, 1) __maxnreg__(T == 3 ? 112 : HY_ATTN_MAXNREG)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const TcAttnParams p) {
  using C = TcAttnCfg<D, T>;
  pdl_wait();  // Q (and for varlen K/V) are written by the previous kernel on the stream
  // grid (heads, q-tile pairs x sequences), heads fastest: the hardware launches CTAs in
  // blockIdx order, so every head's LAST query-tile pair (the most keys under the causal
  // mask) starts before any lighter pair -- longest-first over the whole grid, the light
  // CTAs fill the tail (a 2304-token chunk: 288 CTAs on 148 SMs, SMs were busy 62% of the
  // kernel with heads slowest)
  const int seq = blockIdx.y % p.n_seqs;
  const int qp = p.q_tiles - 1 - blockIdx.y / p.n_seqs;
  const int h = blockIdx.x;
  const int kvh = h / p.group;
  const int q0 = p.qstart[seq];
  const int nq = p.qstart[seq + 1] - q0;
  const int qbase = qp * C::TILES * C::BQ;  // first query row of this CTA within the sequence
  if (qbase >= nq) return;
  const int off = PAGED ? p.offset[seq] : 0;
  const int kv_len = off + nq;
  const int kv_end = PAGED ? min(kv_len, off + qbase + C::TILES * C::BQ) : kv_len;
  const int n_kt = (kv_end + C::BK - 1) / C::BK;
  // the pair's second tile holds no query row (a sequence's last, partial pair): it is
  // skipped -- no Q K^T / P V issued, its softmax warps idle (e.g. a 577-token image: 5 of
  // 6 tiles computed instead of 6)
  const bool t1_live = C::TILES == 2 && qbase + C::BQ < nq;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                               // tile t at t * Q_BYTES
  uint8_t* sKV = smem + C::TILES * C::Q_BYTES;      // stage s: K at s * STAGE, V at + KV_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + 2 * C::STAGE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [2 stages]  K and V of a stage are tracked separately:
  uint64_t* k_empty = bars + 3;   // [2 stages]  K is retired after the Q K^T MMAs, long
  uint64_t* v_full = bars + 5;    // [2 stages]  before V (after P V), so the next-but-one
  uint64_t* v_empty = bars + 7;   // [2 stages]  K tile loads a softmax earlier
  uint64_t* s_full = bars + 9;    // [2 tiles]
  uint64_t* p_full = bars + 11;   // [2 tiles]
  uint64_t* o_done = bars + 13;   // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], T == 2 ? 4 : 8);
      mbar_init(&o_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // only once this CTA holds its TMEM (see gemm_tc_kernel)

  if (warp == 0) {
    // ---------------- TMA producer (lane 0 issues; the warp fetches block-table entries) --
    if (lane == 0) {
      mbar_expect_tx(q_full, C::TILES * C::Q_BYTES);
      for (int t = 0; t < C::TILES; ++t)
        for (int c = 0; c < C::NC; ++c) {
          if (DV != D)
            tma_load_3d(&tmQ, q_full, sQ + t * C::Q_BYTES + c * C::CHUNK, c * 64, h,
                        q0 + qbase + t * C::BQ, kEvictFirst);
          else
            tma_load_2d(&tmQ, q_full, sQ + t * C::Q_BYTES + c * C::CHUNK, h * D + c * 64,
                        q0 + qbase + t * C::BQ, kEvictFirst);
        }
    }
    constexpr int BPT = C::BK / HY_KV_BLOCK_TOKENS;  // cache blocks per key tile (8)
    const int* bt = PAGED ? p.block_table + (size_t)p.slots[seq] * p.bt_stride : nullptr;
    const int last_blk = (kv_end - 1) / HY_KV_BLOCK_TOKENS;
    // lane b < 8 holds the physical id of block b of the current tile; the next tile's ids
    // are fetched before waiting for the stage (one load latency per tile, overlapped).
    // Blocks past the end reload the last valid one (finite data under masked keys).
    int ids = 0;
    if (PAGED && lane < BPT) ids = bt[min(lane, last_blk)];
    for (int j = 0; j < n_kt; ++j) {
      const int st = j & 1;
      int next = 0;
      if (PAGED && lane < BPT && j + 1 < n_kt) next = bt[min((j + 1) * BPT + lane, last_blk)];
      uint8_t* sK = sKV + st * C::STAGE_BYTES;
      uint8_t* sV = sK + C::KV_BYTES;
      const long long row = PAGED ? (long long)ids * p.rows_per_block + kvh * HY_KV_BLOCK_TOKENS : 0;
      // K_j (lane b: block b of the tile; eight lanes drive the TMA unit in parallel)
      if (lane == 0) {
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        ATR(0, j);
        mbar_expect_tx(&k_full[st], C::KV_BYTES);
      }
      __syncwarp();
      if (PAGED) {
        if (lane < BPT)
#pragma unroll
          for (int c = 0; c < C::NC; ++c)
            tma_load_2d(&tmKV, &k_full[st], sK + c * C::CHUNK + lane * 2048, c * 64, (int)row,
                        kEvictNormal);
      } else if (lane == 0) {
#pragma unroll
        for (int c = 0; c < C::NC; ++c) {
          if (DV != D)  // k_col0 is a head index here
            tma_load_3d(&tmKV, &k_full[st], sK + c * C::CHUNK, c * 64, p.k_col0 + kvh,
                        q0 + j * C::BK, kEvictNormal);
          else
            tma_load_2d(&tmKV, &k_full[st], sK + c * C::CHUNK, p.k_col0 + kvh * D + c * 64,
                        q0 + j * C::BK, kEvictNormal);
        }
      }
      // V_j
      if (lane == 0) {
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], C::KV_BYTES);
      }
      __syncwarp();
      if (PAGED) {
        if (lane < BPT)
#pragma unroll
          for (int c = 0; c < C::NC; ++c)
            tma_load_2d(&tmKV, &v_full[st], sV + c * C::CHUNK + lane * 2048, c * 64,
                        (int)(row + p.rows_per_kv), kEvictNormal);
      } else if (lane == 0) {
#pragma unroll
        for (int c = 0; c < C::NC; ++c) {
          if (DV != D)
            tma_load_3d(&tmKV, &v_full[st], sV + c * C::CHUNK, c * 64, p.v_col0 + kvh,
                        q0 + j * C::BK, kEvictNormal);
          else
            tma_load_2d(&tmKV, &v_full[st], sV + c * C::CHUNK, p.v_col0 + kvh * D + c * 64,
                        q0 + j * C::BK, kEvictNormal);
        }
      }
      // warm L2 with the next tile's blocks: its TMA loads (issued once a stage frees up)
      // then hit L2 instead of HBM -- the 32 small boxes per tile are latency-bound
      if (PAGED && j + 1 < n_kt && lane < BPT) {
        const long long row = (long long)next * p.rows_per_block + kvh * HY_KV_BLOCK_TOKENS;
#pragma unroll
        for (int c = 0; c < C::NC; ++c) {
          tma_prefetch_2d(&tmKV, c * 64, (int)row);
          tma_prefetch_2d(&tmKV, c * 64, (int)(row + p.rows_per_kv));
        }
      }
      ids = next;
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      // per tile t the chain S_t(j) -> softmax_t(j) -> PV_t(j) -> S_t(j+1) is serial (P_t
      // lives in S_t's columns); the two tiles interleave so one tile's MMAs run while the
      // other tile's softmax works.  MMAs from this thread execute in issue order.
      // a head dim narrower than the tile (DV = 80 in D = 128 tiles): Q K^T runs only the
      // ceil(DV / 16) k-steps that hold real dims and P V only N = DV_16 output columns -- the
      // zero-filled padding costs no MMA work (37.5% of both for Qwen2-VL's vision tower)
      constexpr int KSTEPS = (DV + 15) / 16;
      constexpr int DV16 = KSTEPS * 16;
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, DV16) | (1u << 16);  // B (= V) MN-major
      auto issue_s = [&](int t, int j) {
        const uint32_t q_addr = smem_u32(sQ + t * C::Q_BYTES);
        const uint32_t k_addr = smem_u32(sKV + (j & 1) * C::STAGE_BYTES);
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
          const int c = ks >> 2, k = ks & 3;
          umma_bf16(tmem + t * 128, smem_desc_k_sw128(q_addr + c * C::CHUNK + k * 32),
                    smem_desc_k_sw128(k_addr + c * C::CHUNK + k * 32), idesc_qk,
                    ks ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {
        mbar_wait(&p_full[t], j & 1);
        ATR(2 + t, j);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sKV + (j & 1) * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < C::BK / 16; ++kk)
          umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                       smem_desc_sw128(v_addr + kk * 2048, C::CHUNK, 1024), idesc_pv,
                       (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&o_done[t]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      if constexpr (C::TILES == 2) {
      issue_s(0, 0);
      if (t1_live) issue_s(1, 0);
      umma_commit(&k_empty[0]);  // K_0 retired once both Q K^T complete
      for (int j = 0; j < n_kt; ++j) {
        const bool more = j + 1 < n_kt;
        mbar_wait(&v_full[j & 1], (j >> 1) & 1);
        // the tile whose softmax finishes first gets the tensor pipe first (the two tiles'
        // softmaxes drift; a fixed order makes the early one wait for the late one)
        bool done[2] = {false, !t1_live};
        bool k_ready = false;
        while (!(done[0] && done[1])) {
#pragma unroll
          for (int t = 0; t < C::TILES; ++t) {
            if (done[t] || !mbar_test(&p_full[t], j & 1)) continue;
            issue_pv(t, j);
            if (more) {
              if (!k_ready) {  // the next key tile is needed only from here on
                mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
                ATR(1, j + 1);
                tc_fence_after();
                k_ready = true;
              }
              issue_s(t, j + 1);
            }
            done[t] = true;
          }
        }
        if (more) umma_commit(&k_empty[(j + 1) & 1]);
        umma_commit(&v_empty[j & 1]);  // V_j retired once both P V complete
      }
      } else {
        // one query tile: S(j) lives in TMEM buffer j & 1 (P(j) over it), O at column 256.
        // S(j+1) is issued before P V(j), so it runs while the softmax works on S(j); it
        // overwrites P(j-1), whose P V was issued (and executes) before it.
        const uint32_t q_addr = smem_u32(sQ);
        auto issue_s1 = [&](int j) {
          const uint32_t k_addr = smem_u32(sKV + (j & 1) * C::STAGE_BYTES);
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const int c = ks >> 2, k = ks & 3;
            umma_bf16(tmem + (j & 1) * 128, smem_desc_k_sw128(q_addr + c * C::CHUNK + k * 32),
                      smem_desc_k_sw128(k_addr + c * C::CHUNK + k * 32), idesc_qk,
                      ks ? 1u : 0u);
          }
          umma_commit(&s_full[j & 1]);
          umma_commit(&k_empty[j & 1]);
        };
        issue_s1(0);
        for (int j = 0; j < n_kt; ++j) {
          if (j + 1 < n_kt) {
            mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
            tc_fence_after();
            issue_s1(j + 1);
          }
          mbar_wait(&v_full[j & 1], (j >> 1) & 1);
          mbar_wait(&p_full[0], j & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sKV + (j & 1) * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk)
            umma_bf16_ts(tmem + 256, tmem + (j & 1) * 128 + kk * 8,
                         smem_desc_sw128(v_addr + kk * 2048, C::CHUNK, 1024), idesc_pv,
                         (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&o_done[0]);
          umma_commit(&v_empty[j & 1]);
        }
      }
    }
  } else {
    if constexpr (T == 2) {
    // ---------------- softmax: tile t = warps 2..5 / 6..9, one query row per thread -------
    const int t = (warp - 2) >> 2;
    const int sub = warp & 3;
    const int row = sub * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(sub * 32) << 16);  // this warp's TMEM lanes
    const uint32_t tS = tl + t * 128, tO = tl + 256 + t * 128;
    const int qrow = qbase + t * C::BQ + row;  // query row within the sequence
    const int qpos = off + qrow;               // absolute position of this query
    float m_used = -INFINITY, l = 0.f;
    const bool live = t == 0 || t1_live;
    for (int j = 0; j < (live ? n_kt : 0); ++j) {
      mbar_wait(&s_full[t], j & 1);
      if (threadIdx.x == 64) ATR(4, j);
      tc_fence_after();
      // one TMEM round trip for the whole S row (4 loads, one wait); the row stays in
      // registers for the P pass.  Tiles entirely inside every row's key range of the warp
      // skip the per-element mask.
      const int kbase = j * C::BK;
      const int kmax = PAGED ? min(kv_len, qpos + 1) : kv_len;  // keys [0, kmax) are valid
      const bool full = __all_sync(0xffffffffu, kbase + C::BK <= kmax);
      // The S row is read from TMEM twice, 64 columns at a time (max, then exp): holding all
      // 128 fp32 values in registers spilled at the 168 registers a 10-warp CTA can have
      uint32_t r[64];
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      // keys 64-127 first: the registers then still hold keys 0-63 for the exp pass
#pragma unroll
      for (int hh = 1; hh >= 0; --hh) {
        tmem_ld_32x32b_x32(tS + hh * 64, r);
        tmem_ld_32x32b_x32(tS + hh * 64 + 32, r + 32);
        tmem_ld_wait();
        if (full) {
#pragma unroll
          for (int u = 0; u < 64; ++u) mx8[u & 7] = fmaxf(mx8[u & 7], __uint_as_float(r[u]));
        } else {
#pragma unroll
          for (int u = 0; u < 64; ++u)
            if (kbase + hh * 64 + u < kmax) mx8[u & 7] = fmaxf(mx8[u & 7], __uint_as_float(r[u]));
        }
      }
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx = mx == -INFINITY ? mx : mx * p.scale_log2;
      const float m_new = fmaxf(m_used, mx);
      if (j >= 1) {
        mbar_wait(&o_done[t], (j - 1) & 1);  // PV_t(j-1) retired: O_t stable
        if (threadIdx.x == 64) ATR(6, j);
        tc_fence_after();
        // tcgen05.ld/st are warp-collective: the warp rescales together when any of its
        // rows' max grew by more than 2^8 (factor 1 for the others)
        const bool need = m_new > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          const float f = !need ? 1.f : (m_used == -INFINITY ? 0.f : exp2f(m_used - m_new));
          l *= f;
          if (need) m_used = m_new;
#pragma unroll 1
          for (int c = 0; c < (DV + 31) / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * f);
            tmem_st_32x32b_x32(tO + c * 32, o);
          }
        }
      } else {
        m_used = m_new;
      }
      const float ms = m_used == -INFINITY ? 0.f : m_used;
      // P_t = exp2(S * scale - m) as bf16 pairs into S_t's first 64 columns (A of PV), 16
      // columns per store; column c of P holds keys 2c, 2c+1 (already in registers)
      uint64_t rs2[2] = {pk2(0.f, 0.f), pk2(0.f, 0.f)};
      const uint64_t sc2 = pk2(p.scale_log2, p.scale_log2), nms2 = pk2(-ms, -ms);
      // exp pass, in key order: keys 0-63 are still in registers, keys 64-127 are read again
      // (P of chunk c goes to columns [16c, 16c + 16), which belong to S chunks <= c, already
      // consumed; S columns 64-127 are never overwritten)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c == 2) {
          tmem_ld_32x32b_x32(tS + 64, r);
          tmem_ld_32x32b_x32(tS + 96, r + 32);
          tmem_ld_wait();
        }
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int k0 = c * 32 + 2 * u;
          const int kr = (c & 1) * 32 + 2 * u;  // register index of key k0
          float x0, x1;
          up2(ffma2(pk2(__uint_as_float(r[kr]), __uint_as_float(r[kr + 1])), sc2, nms2), x0, x1);
          float e0, e1;
          if (u < HY_ATTN_POLY) {
            exp2_poly2(x0, x1, e0, e1);
          } else {
            e0 = ex2_approx(x0);
            e1 = ex2_approx(x1);
          }
          if (!full) {
            e0 = kbase + k0 < kmax ? e0 : 0.f;
            e1 = kbase + k0 + 1 < kmax ? e1 : 0.f;
          }
          rs2[u & 1] = fadd2(rs2[u & 1], pk2(e0, e1));
          pk[u] = pack_bf16x2(e0, e1);
        }
        tmem_st_32x32b_x16(tS + c * 16, pk);
      }
      float ra, rb, rc, rd;
      up2(rs2[0], ra, rb);
      up2(rs2[1], rc, rd);
      const float rs = (ra + rb) + (rc + rd);
      l += rs;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
      if (threadIdx.x == 64) ATR(5, j);
    }
    // O_t / l -> global
    if (live) mbar_wait(&o_done[t], (n_kt - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < (live ? (DV + 31) / 32 : 0); ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tO + c * 32, o);
      tmem_ld_wait();
      if (qrow < nq) {
        bf16* dst = p.out + (size_t)(q0 + qrow) * p.ld_o + (size_t)h * DV + c * 32;
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          if (c * 32 + u >= DV) break;
          float v[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) v[w] = __uint_as_float(o[u + w]) * inv;
          store_bf16x8(dst + u, v);
        }
      }
    }

    } else {
    // ---------------- softmax, two threads per row ------------------------------------------
    // T = 1: one query tile, warps 2..9.  T = 3: two tiles, warps 2..9 (tile 0) and 10..17
    // (tile 1).  Warps w and w + 4 of a tile own the same 32 TMEM lanes (rows); the first
    // takes keys [0, 64) of each key tile, the second [64, 128).  Row maxima are exchanged
    // through shared memory (double-buffered by key-tile parity) with a 64-thread named
    // barrier per (tile, row group).  T = 1 double-buffers S over key tiles (buffer j & 1);
    // T = 3 keeps S_t in buffer t, ping-ponging with the other tile like T = 2.
    __shared__ float xm[2][2][2][128];  // [tile][key-tile parity][key half][row]
    __shared__ float xl[2][2][128];     // [tile][key half][row]
    const int t = T == 3 ? (warp - 2) >> 3 : 0;
    const int sub = warp & 3;
    const int hc = ((warp - 2) >> 2) & 1;  // key / O-column half
    const int row = sub * 32 + lane;
    const int bar_id = 1 + t * 4 + sub;
    const uint32_t tl = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t tO = tl + 256 + t * 128 + hc * (D / 2);
    const int qrow = qbase + t * C::BQ + row;
    const int qpos = off + qrow;
    const int kmax = PAGED ? min(kv_len, qpos + 1) : kv_len;  // keys [0, kmax) are valid
    const bool live = t == 0 || t1_live;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < (live ? n_kt : 0); ++j) {
      const int b = j & 1;
      const int sb = T == 3 ? t : b;  // S / P buffer
      mbar_wait(&s_full[sb], T == 3 ? (j & 1) : ((j >> 1) & 1));
      tc_fence_after();
      const int kbase = j * C::BK + hc * 64;
      const bool full = __all_sync(0xffffffffu, kbase + 64 <= kmax);
      uint32_t r[64];
      tmem_ld_32x32b_x32(tl + sb * 128 + hc * 64, r);
      tmem_ld_32x32b_x32(tl + sb * 128 + hc * 64 + 32, r + 32);
      tmem_ld_wait();
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      if (full) {
#pragma unroll
        for (int u = 0; u < 64; ++u) mx8[u & 7] = fmaxf(mx8[u & 7], __uint_as_float(r[u]));
      } else {
#pragma unroll
        for (int u = 0; u < 64; ++u)
          if (kbase + u < kmax) mx8[u & 7] = fmaxf(mx8[u & 7], __uint_as_float(r[u]));
      }
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      xm[t][b][hc][row] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      mx = fmaxf(mx, xm[t][b][hc ^ 1][row]);
      mx = mx == -INFINITY ? mx : mx * p.scale_log2;
      const float m_new = fmaxf(m_used, mx);
      if (j >= 1) {
        mbar_wait(&o_done[t], (j - 1) & 1);  // P V(j-1) retired: O stable
        tc_fence_after();
        const bool need = m_new > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          const float f = !need ? 1.f : (m_used == -INFINITY ? 0.f : exp2f(m_used - m_new));
          l *= f;
          if (need) m_used = m_new;
#pragma unroll 1
          for (int c = 0; c < D / 64; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * f);
            tmem_st_32x32b_x32(tO + c * 32, o);
          }
        }
      } else {
        m_used = m_new;
      }
      const float ms = m_used == -INFINITY ? 0.f : m_used;
      uint64_t rs2[2] = {pk2(0.f, 0.f), pk2(0.f, 0.f)};
      const uint64_t sc2 = pk2(p.scale_log2, p.scale_log2), nms2 = pk2(-ms, -ms);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int k0 = c * 32 + 2 * u;
          float x0, x1;
          up2(ffma2(pk2(__uint_as_float(r[k0]), __uint_as_float(r[k0 + 1])), sc2, nms2), x0, x1);
          float e0, e1;
          if (u < HY_ATTN_POLY) {
            exp2_poly2(x0, x1, e0, e1);
          } else {
            e0 = ex2_approx(x0);
            e1 = ex2_approx(x1);
          }
          if (!full) {
            e0 = kbase + k0 < kmax ? e0 : 0.f;
            e1 = kbase + k0 + 1 < kmax ? e1 : 0.f;
          }
          rs2[u & 1] = fadd2(rs2[u & 1], pk2(e0, e1));
          pk[u] = pack_bf16x2(e0, e1);
        }
        tmem_st_32x32b_x16(tl + sb * 128 + hc * 32 + c * 16, pk);
      }
      float ra, rb, rc, rd;
      up2(rs2[0], ra, rb);
      up2(rs2[1], rc, rd);
      l += (ra + rb) + (rc + rd);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    // O / (l_lo + l_hi) -> global, each thread its half of the head dims
    if (live) {
    xl[t][hc][row] = l;
    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
    const float lt = l + xl[t][hc ^ 1][row];
    mbar_wait(&o_done[t], (n_kt - 1) & 1);
    tc_fence_after();
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll 1
    for (int c = 0; c < D / 64; ++c) {
      if (hc * (D / 2) + c * 32 >= DV) break;
      uint32_t o[32];
      tmem_ld_32x32b_x32(tO + c * 32, o);
      tmem_ld_wait();
      if (qrow < nq) {
        bf16* dst = p.out + (size_t)(q0 + qrow) * p.ld_o + (size_t)h * DV + hc * (D / 2) + c * 32;
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          if (hc * (D / 2) + c * 32 + u >= DV) break;
          float v[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) v[w] = __uint_as_float(o[u + w]) * inv;
          store_bf16x8(dst + u, v);
        }
      }
    }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int D, bool PAGED, int T, int DV = D>
static int launch_tc_attn(const CUtensorMap& tq, const CUtensorMap& tkv, const TcAttnParams& p,
                          int n_seqs, int n_heads, cudaStream_t st) {
  using C = TcAttnCfg<D, T>;
  HY_CUDA_RET(ensure_smem(attn_tc_kernel<D, PAGED, T, DV>, C::SMEM));
  TcAttnParams pp = p;
  pp.n_seqs = n_seqs;
  HY_CUDA_RET(launch_pdl(attn_tc_kernel<D, PAGED, T, DV>, dim3(n_heads, n_seqs * p.q_tiles),
                         dim3(C::THREADS), C::SMEM, st, tq, tkv, pp));
  HY_LAUNCH_CHECK();
  return 0;
}

// Query tiles per CTA: two (ping-pong between the tiles) or one (two softmax threads per
// row, twice the CTAs), whichever the wave count favours.  HY_ATTN_T=1/2 forces.
static int attn_tiles(int n_seqs, int max_q, int n_heads) {
  const char* e = getenv("HY_ATTN_T");
  const int forced = e ? atoi(e) : 0;
  if (forced >= 1 && forced <= 3) return forced;
  // waves of CTAs x the CTA's time: a two-tile CTA takes ~1.6x a one-tile CTA (its
  // ping-pong makes each tile ~20% cheaper).  Matches every measured case (ViT 1-32 images
  // of 577 / 576-11664 tokens, prefill chunks 616-2304): e.g. one 2916-token Qwen2-VL image
  // 192 two-tile CTAs (2 waves) 117 us vs 368 one-tile CTAs (3 waves) 91 us
  const long long sms = num_sms();
  const long long c2 = (long long)n_seqs * ceil_div(max_q, 256) * n_heads;
  const long long c1 = (long long)n_seqs * ceil_div(max_q, 128) * n_heads;
  const double t2 = 1.6 * (double)((c2 + sms - 1) / sms);
  const double t1 = (double)((c1 + sms - 1) / sms);
  return t1 < t2 ? 1 : 2;
}

// Paged prefill: Q rows of the chunk batch [n_rows, ld_q]; K/V from the paged cache of one
// layer ([block][K,V][kv_head][16][d] inside a block of block_stride elements).
int attn_tc_prefill(const void* q, int ld_q, int n_rows, int n_seqs, const int* qstart,
                    const int* offset, const int* slots, int max_q, int n_heads, int n_kv_heads,
                    int head_dim, const int* block_table, int bt_stride, const void* kv_layer,
                    long long block_stride, float scale, void* out, int ld_o, cudaStream_t st) {
  HY_CHECK_ARG(head_dim == 128 || head_dim == 64, "tcgen05 attention: head_dim 64 or 128");
  HY_CHECK_ARG(block_stride % head_dim == 0, "block stride");
  TcAttnParams p{};
  p.qstart = qstart;
  p.offset = offset;
  p.slots = slots;
  p.block_table = block_table;
  p.bt_stride = bt_stride;
  const int T = attn_tiles(n_seqs, max_q, n_heads);
  p.q_tiles = ceil_div(max_q, 128 * (T == 3 ? 2 : T));
  p.group = n_heads / n_kv_heads;
  p.rows_per_block = block_stride / head_dim;
  p.rows_per_kv = n_kv_heads * HY_KV_BLOCK_TOKENS;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = reinterpret_cast<bf16*>(out);
  p.ld_o = ld_o;
  CUtensorMap tq, tkv;
  HY_RET_IF(make_tmap_2d_bf16(&tq, q, n_rows, (uint64_t)n_heads * head_dim, (uint64_t)ld_q * 2,
                              128, 64));
  // the whole pool as rows of head_dim elements; rows addressed through the block table
  HY_RET_IF(make_tmap_2d_bf16(&tkv, kv_layer, (1ull << 31) - 1, head_dim, (uint64_t)head_dim * 2,
                              HY_KV_BLOCK_TOKENS, 64));
  if (T == 2)
    return head_dim == 128 ? launch_tc_attn<128, true, 2>(tq, tkv, p, n_seqs, n_heads, st)
                           : launch_tc_attn<64, true, 2>(tq, tkv, p, n_seqs, n_heads, st);
  if (T == 3)
    return head_dim == 128 ? launch_tc_attn<128, true, 3>(tq, tkv, p, n_seqs, n_heads, st)
                           : launch_tc_attn<64, true, 3>(tq, tkv, p, n_seqs, n_heads, st);
  return head_dim == 128 ? launch_tc_attn<128, true, 1>(tq, tkv, p, n_seqs, n_heads, st)
                         : launch_tc_attn<64, true, 1>(tq, tkv, p, n_seqs, n_heads, st);
}

// Varlen (ViT): packed QKV rows [n_rows, ld_qkv] = [Q heads | K heads | V heads].
int attn_tc_varlen(const void* qkv, int ld_qkv, int n_rows, int n_segs, const int* seg,
                   int max_len, int n_heads, int head_dim, float scale, void* out, int ld_o,
                   cudaStream_t st) {
  HY_CHECK_ARG(head_dim == 128 || head_dim == 64 || head_dim == 80,
               "tcgen05 attention: head_dim 64, 80 or 128");
  TcAttnParams p{};
  p.qstart = seg;
  const int T = attn_tiles(n_segs, max_len, n_heads);
  p.q_tiles = ceil_div(max_len, 128 * (T == 3 ? 2 : T));
  p.group = 1;
  p.k_col0 = n_heads * head_dim;
  p.v_col0 = 2 * n_heads * head_dim;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = reinterpret_cast<bf16*>(out);
  p.ld_o = ld_o;
  CUtensorMap tm;
  if (head_dim == 80) {
    // Qwen2-VL's vision tower: each head's 80 dims padded to 128 by the TMA's out-of-bounds
    // zero fill (3D map [rows][3 * heads][80]); the tile math is the d = 128 kernel's
    HY_CHECK_ARG((ld_qkv * 2) % 16 == 0, "ld_qkv");
    p.k_col0 = n_heads;  // head indices in the 3D map
    p.v_col0 = 2 * n_heads;
    HY_RET_IF(make_tmap_3d_bf16(&tm, qkv, 80, (uint64_t)3 * n_heads, n_rows, 80 * 2,
                                (uint64_t)ld_qkv * 2, 64, 128));
    return T == 2   ? launch_tc_attn<128, false, 2, 80>(tm, tm, p, n_segs, n_heads, st)
           : T == 3 ? launch_tc_attn<128, false, 3, 80>(tm, tm, p, n_segs, n_heads, st)
                    : launch_tc_attn<128, false, 1, 80>(tm, tm, p, n_segs, n_heads, st);
  }
  HY_RET_IF(make_tmap_2d_bf16(&tm, qkv, n_rows, (uint64_t)3 * n_heads * head_dim,
                              (uint64_t)ld_qkv * 2, 128, 64));
  if (T == 2)
    return head_dim == 128 ? launch_tc_attn<128, false, 2>(tm, tm, p, n_segs, n_heads, st)
                           : launch_tc_attn<64, false, 2>(tm, tm, p, n_segs, n_heads, st);
  if (T == 3)
    return head_dim == 128 ? launch_tc_attn<128, false, 3>(tm, tm, p, n_segs, n_heads, st)
                           : launch_tc_attn<64, false, 3>(tm, tm, p, n_segs, n_heads, st);
  return head_dim == 128 ? launch_tc_attn<128, false, 1>(tm, tm, p, n_segs, n_heads, st)
                         : launch_tc_attn<64, false, 1>(tm, tm, p, n_segs, n_heads, st);
}

}  // namespace hy
