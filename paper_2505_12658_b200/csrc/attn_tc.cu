// K7 paged prefill attention and K3 ViT varlen attention on 5th-generation tensor cores.
//
// One CTA = one (sequence, query head, 128-row query tile).  Warp-specialised:
//   warp 0      TMA producer: the Q tile once, then K/V tiles of 128 keys into a 2-stage ring
//               (paged: eight 16-token cache blocks per tile through the block table;
//               varlen: the image's rows of the packed QKV buffer)
//   warp 1      single-thread tcgen05.mma issuer:
//                 S_j = Q K_j^T   (M=128 queries, N=128 keys, K=d; fp32 in TMEM, double-buffered)
//                 O  += P_j V_j   (M=128, N=d, K=128 keys; P from shared memory, V as an
//                                  MN-major operand straight from its TMA tile)
//               issued as S_0, S_1, PV_0, S_2, PV_1, ... so Q K^T of the next tile runs
//               while the softmax warps work on the current one
//   warps 2..5  softmax: each thread owns one query row -- tcgen05.ld of its S row, mask,
//               online max/sum in the exp2 domain, P as bf16 into shared memory with the
//               128-byte swizzle the MMA descriptor expects.  The O accumulator stays in
//               TMEM; it is rescaled (tcgen05.ld/st of the row) only when the running max
//               grows by more than 2^8 -- P values stay <= 256, exact in the final O / l.
//               Finally O / l -> bf16 -> global.
//
// Same math as the mma.sync kernel it replaces for d in {64, 128} (attn_prefill.cu keeps
// that kernel for other head sizes, e.g. Qwen2-VL's d = 80 vision tower).
// Reference: epdsim prices prefill attention as 4 S^2 H per chunk (model_cost.py:189) and
// ViT attention as 4 T^2 H_v per image (model_cost.py:160-163).
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <cmath>

namespace hy {

struct TcAttnParams {
  const int* qstart;   // [n_seqs + 1] query rows of each sequence in the Q map
  const int* offset;   // paged: tokens cached before the chunk
  const int* slots;    // paged: block-table row of each sequence
  const int* block_table;
  int bt_stride;
  int q_tiles;         // 128-row query tiles per sequence in the grid
  int group;           // query heads per kv head
  int k_col0, v_col0;  // varlen: column of kv head 0's K / V in the packed QKV map
  long long rows_per_block;  // paged: KV-map rows per cache block (block_stride / d)
  int rows_per_kv;     // paged: rows from a block's K half to its V half (n_kv * 16)
  float scale_log2;
  bf16* out;
  int ld_o;
};

template <int D>
struct TcAttnCfg {
  static constexpr int BQ = 128, BK = 128;
  static constexpr int NC = D / 64;               // 64-wide d chunks (one 128B swizzle row)
  static constexpr int CHUNK = 128 * 128;         // bytes of one [128 rows][64 bf16] chunk
  static constexpr int Q_BYTES = NC * CHUNK;
  static constexpr int KV_BYTES = NC * CHUNK;     // K (or V) of one tile
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int P_BYTES = 2 * CHUNK;       // [128 q][128 keys] bf16, 2 key chunks
  static constexpr int SMEM = Q_BYTES + 2 * STAGE_BYTES + P_BYTES + 1024 + 256;
  static constexpr uint32_t TM_S = 0;             // S buffers at columns 0 and 128
  static constexpr uint32_t TM_O = 256;           // O at columns 256 .. 256 + D
  static constexpr int TMEM_COLS = 512;
};

template <int D, bool PAGED>
__global__ void __launch_bounds__(192, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const TcAttnParams p) {
  using C = TcAttnCfg<D>;
  pdl_trigger();
  pdl_wait();  // Q (and for varlen K/V) are written by the previous kernel on the stream
  const int seq = blockIdx.x / p.q_tiles;
  const int qt = blockIdx.x % p.q_tiles;
  const int h = blockIdx.y;
  const int kvh = h / p.group;
  const int q0 = p.qstart[seq];
  const int nq = p.qstart[seq + 1] - q0;
  if (qt * C::BQ >= nq) return;
  const int off = PAGED ? p.offset[seq] : 0;
  const int kv_len = off + nq;
  const int kv_end = PAGED ? min(kv_len, off + qt * C::BQ + C::BQ) : kv_len;
  const int n_kt = (kv_end + C::BK - 1) / C::BK;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + C::Q_BYTES;                 // stage s: K at s * STAGE, V at + KV_BYTES
  uint8_t* sP = sKV + 2 * C::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* p_free = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmKV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(p_free, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int c = 0; c < C::NC; ++c)
        tma_load_2d(&tmQ, q_full, sQ + c * C::CHUNK, h * D + c * 64, q0 + qt * C::BQ, kEvictFirst);
      const int* bt = PAGED ? p.block_table + (size_t)p.slots[seq] * p.bt_stride : nullptr;
      const int last_blk = (kv_end - 1) / HY_KV_BLOCK_TOKENS;
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], C::STAGE_BYTES);
        uint8_t* sK = sKV + st * C::STAGE_BYTES;
        uint8_t* sV = sK + C::KV_BYTES;
        if (PAGED) {
          // 8 cache blocks of 16 tokens; blocks past the end reload the last valid one
          // (finite data under masked keys: P = 0 there, and 0 * finite = 0)
#pragma unroll 1
          for (int b = 0; b < C::BK / HY_KV_BLOCK_TOKENS; ++b) {
            const int blk = min(j * (C::BK / HY_KV_BLOCK_TOKENS) + b, last_blk);
            const long long row = (long long)bt[blk] * p.rows_per_block + kvh * HY_KV_BLOCK_TOKENS;
#pragma unroll
            for (int c = 0; c < C::NC; ++c) {
              tma_load_2d(&tmKV, &kv_full[st], sK + c * C::CHUNK + b * 2048, c * 64, (int)row,
                          kEvictNormal);
              tma_load_2d(&tmKV, &kv_full[st], sV + c * C::CHUNK + b * 2048, c * 64,
                          (int)(row + p.rows_per_kv), kEvictNormal);
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < C::NC; ++c) {
            tma_load_2d(&tmKV, &kv_full[st], sK + c * C::CHUNK, p.k_col0 + kvh * D + c * 64,
                        q0 + j * C::BK, kEvictNormal);
            tma_load_2d(&tmKV, &kv_full[st], sV + c * C::CHUNK, p.v_col0 + kvh * D + c * 64,
                        q0 + j * C::BK, kEvictNormal);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D) | (1u << 16);  // B (= V) MN-major
      auto issue_pv = [&](int i) {
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sKV + (i & 1) * C::STAGE_BYTES + C::KV_BYTES);
        const uint32_t p_addr = smem_u32(sP);
#pragma unroll
        for (int kk = 0; kk < C::BK / 16; ++kk)
          umma_bf16(tmem + C::TM_O, smem_desc_k_sw128(p_addr + (kk >> 2) * C::CHUNK + (kk & 3) * 32),
                    smem_desc_sw128(v_addr + kk * 2048, C::CHUNK, 1024), idesc_pv,
                    (i > 0 || kk > 0) ? 1u : 0u);
        umma_commit(p_free);
        umma_commit(&kv_empty[i & 1]);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sQ);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        mbar_wait(&s_free[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sKV + st * C::STAGE_BYTES);
#pragma unroll
        for (int c = 0; c < C::NC; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + C::TM_S + st * 128, smem_desc_k_sw128(q_addr + c * C::CHUNK + k * 32),
                      smem_desc_k_sw128(k_addr + c * C::CHUNK + k * 32), idesc_qk,
                      (c | k) ? 1u : 0u);
        umma_commit(&s_full[st]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_kt - 1);
    }
  } else {
    // ---------------- softmax warps 2..5: one query row per thread ----------------
    const int sub = warp & 3;
    const int row = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const int qpos = off + qt * C::BQ + row;  // absolute position of this query
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(trow + C::TM_S + b * 128 + c * 32, r + c * 32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[b]);
      const int kbase = j * C::BK;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        const int key = kbase + c;
        const bool ok = key < kv_len && (!PAGED || key <= qpos);
        const float x = ok ? __uint_as_float(r[c]) * p.scale_log2 : -INFINITY;
        r[c] = __float_as_uint(x);
        mx = fmaxf(mx, x);
      }
      const float m_new = fmaxf(m_used, mx);
      if (j >= 1) {
        mbar_wait(p_free, (j - 1) & 1);  // PV_{j-1} retired: O stable, P buffer free
        tc_fence_after();
        // tcgen05.ld/st are warp-collective: the warp rescales together when any of its
        // rows needs it (factor 1 for the others)
        const bool need = m_new > m_used + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          const float f = !need ? 1.f : (m_used == -INFINITY ? 0.f : exp2f(m_used - m_new));
          l *= f;
          if (need) m_used = m_new;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(trow + C::TM_O + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * f);
            tmem_st_32x32b_x32(trow + C::TM_O + c * 32, o);
          }
          tmem_st_wait();
        }
      } else {
        m_used = m_new;
      }
      const float ms = m_used == -INFINITY ? 0.f : m_used;
      // P row -> bf16, 128B-swizzled K-major tile: row `row`, 16-byte chunk c16 of key chunk kc
      const uint32_t prow = smem_u32(sP) + (row >> 3) * 1024 + (row & 7) * 128;
      float rs = 0.f;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc)
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          float e[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            e[t] = exp2f(__uint_as_float(r[kc * 64 + c16 * 8 + t]) - ms);
            rs += e[t];
          }
          const uint32_t a = prow + kc * C::CHUNK + ((c16 ^ (row & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                       "r"(pack_bf16x2(e[0], e[1])), "r"(pack_bf16x2(e[2], e[3])),
                       "r"(pack_bf16x2(e[4], e[5])), "r"(pack_bf16x2(e[6], e[7]))
                       : "memory");
        }
      l += rs;
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // O / l -> global
    mbar_wait(p_free, (n_kt - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int qi = qt * C::BQ + row;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(trow + C::TM_O + c * 32, o);
      tmem_ld_wait();
      if (qi < nq) {
        bf16* dst = p.out + (size_t)(q0 + qi) * p.ld_o + (size_t)h * D + c * 32;
#pragma unroll
        for (int t = 0; t < 32; t += 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __uint_as_float(o[t + u]) * inv;
          store_bf16x8(dst + t, v);
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

template <int D, bool PAGED>
static int launch_tc_attn(const CUtensorMap& tq, const CUtensorMap& tkv, const TcAttnParams& p,
                          int n_seqs, int n_heads, cudaStream_t st) {
  using C = TcAttnCfg<D>;
  static bool attr = false;
  if (!attr) {
    HY_CUDA_RET(cudaFuncSetAttribute(attn_tc_kernel<D, PAGED>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  HY_CUDA_RET(launch_pdl(attn_tc_kernel<D, PAGED>, dim3(n_seqs * p.q_tiles, n_heads), dim3(192),
                         C::SMEM, st, tq, tkv, p));
  HY_LAUNCH_CHECK();
  return 0;
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
  p.q_tiles = ceil_div(max_q, 128);
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
  if (head_dim == 128) return launch_tc_attn<128, true>(tq, tkv, p, n_seqs, n_heads, st);
  return launch_tc_attn<64, true>(tq, tkv, p, n_seqs, n_heads, st);
}

// Varlen (ViT): packed QKV rows [n_rows, ld_qkv] = [Q heads | K heads | V heads].
int attn_tc_varlen(const void* qkv, int ld_qkv, int n_rows, int n_segs, const int* seg,
                   int max_len, int n_heads, int head_dim, float scale, void* out, int ld_o,
                   cudaStream_t st) {
  HY_CHECK_ARG(head_dim == 128 || head_dim == 64, "tcgen05 attention: head_dim 64 or 128");
  TcAttnParams p{};
  p.qstart = seg;
  p.q_tiles = ceil_div(max_len, 128);
  p.group = 1;
  p.k_col0 = n_heads * head_dim;
  p.v_col0 = 2 * n_heads * head_dim;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = reinterpret_cast<bf16*>(out);
  p.ld_o = ld_o;
  CUtensorMap tm;
  HY_RET_IF(make_tmap_2d_bf16(&tm, qkv, n_rows, (uint64_t)3 * n_heads * head_dim,
                              (uint64_t)ld_qkv * 2, 128, 64));
  if (head_dim == 128) return launch_tc_attn<128, false>(tm, tm, p, n_segs, n_heads, st);
  return launch_tc_attn<64, false>(tm, tm, p, n_segs, n_heads, st);
}

}  // namespace hy
