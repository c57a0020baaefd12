// K8: paged-KV decode attention (one query token per running decode entry).
//
// The dominant HBM stream at large decode batches: every step reads the whole cached
// context of every running request, bytes = sum_i (S_i + 1) * kv_bytes_per_token
// (epdsim charges 2*B*H*(S+1)*ratio per layer, model_cost.py:195).
//
// Layout read: KV pool block [layer][K|V][kv_head][16 tok][d], so one (block, head) K
// tile is 16 x d contiguous bf16 (4 KiB at d = 128).
//
// Grid (seq, kv_head, split).  Each of the 4 warps streams whole 16-token blocks:
// a warp-wide 16-byte load covers 2 tokens x 128 dims, 8 loads cover the block's K and
// 8 more its V, all issued before use.  Scores reduce across 16 lanes with xor
// shuffles, softmax is online (exp2 domain), all G = n_heads / n_kv_heads query heads
// of a KV head share each K/V load (GQA).  Warps merge through shared memory; when the
// context is split across CTAs (flash-decoding) a second kernel merges the partials.
#include "common.cuh"
#include "../../include/hydra_sm100.h"
#include "mma_sync.cuh"

#include <algorithm>

namespace hy {

constexpr int DEC_WARPS = 4;

template <int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const bf16* __restrict__ q, int ld_q, int n_kv, const int* __restrict__ slots,
                       const int* __restrict__ ctx_len, const int* __restrict__ block_table,
                       int bt_stride, const bf16* __restrict__ kv, long long block_stride,
                       float scale_log2, int blocks_per_split, bf16* __restrict__ out, int ld_o,
                       float* __restrict__ part, int nsplit) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128;
  const int b = blockIdx.x, kh = blockIdx.y, sp = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, dl = lane & 15;
  const int n_heads = n_kv * G;
  const int ctx = ctx_len[b];
  const int nblk = (ctx + HY_KV_BLOCK_TOKENS - 1) / HY_KV_BLOCK_TOKENS;
  const int blk0 = sp * blocks_per_split;
  const int blk1 = min(nblk, blk0 + blocks_per_split);
  const int* bt = block_table + (size_t)slots[b] * bt_stride;

  float qf[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    load_bf16x8(q + (size_t)b * ld_q + (size_t)(kh * G + g) * D + dl * 8, qf[g]);
#pragma unroll
    for (int j = 0; j < 8; ++j) qf[g][j] *= scale_log2;
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
  }

  const size_t head_off = (size_t)kh * HY_KV_BLOCK_TOKENS * D;
  const size_t v_off = (size_t)n_kv * HY_KV_BLOCK_TOKENS * D;
  for (int jb = blk0 + warp; jb < blk1; jb += DEC_WARPS) {
    const bf16* kb = kv + (size_t)bt[jb] * block_stride + head_off;
    const bf16* vb = kb + v_off;
    uint4 kr[8], vr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) kr[i] = ld_nc_v4(kb + (size_t)(2 * i + half) * D + dl * 8);
#pragma unroll
    for (int i = 0; i < 8; ++i) vr[i] = ld_nc_v4(vb + (size_t)(2 * i + half) * D + dl * 8);
    const int tok_base = jb * HY_KV_BLOCK_TOKENS + half;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float s[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 k0 = unpack_bf16x2(kr[i].x), k1 = unpack_bf16x2(kr[i].y),
               k2 = unpack_bf16x2(kr[i].z), k3 = unpack_bf16x2(kr[i].w);
        float d0 = qf[g][0] * k0.x + qf[g][1] * k0.y + qf[g][2] * k1.x + qf[g][3] * k1.y +
                   qf[g][4] * k2.x + qf[g][5] * k2.y + qf[g][6] * k3.x + qf[g][7] * k3.y;
        d0 += __shfl_xor_sync(0xffffffffu, d0, 8);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 4);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
        s[i] = (tok_base + 2 * i < ctx) ? d0 : -INFINITY;
      }
      float mb = s[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) mb = fmaxf(mb, s[i]);
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
      const float mn = fmaxf(m[g], mb);  // finite: every block holds >= 1 valid token
      const float corr = exp2f(m[g] - mn);
      m[g] = mn;
      float ls = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float p = exp2f(s[i] - mn);
        ls += p;
        float2 v0 = unpack_bf16x2(vr[i].x), v1 = unpack_bf16x2(vr[i].y),
               v2 = unpack_bf16x2(vr[i].z), v3 = unpack_bf16x2(vr[i].w);
        acc[g][0] += p * v0.x; acc[g][1] += p * v0.y;
        acc[g][2] += p * v1.x; acc[g][3] += p * v1.y;
        acc[g][4] += p * v2.x; acc[g][5] += p * v2.y;
        acc[g][6] += p * v3.x; acc[g][7] += p * v3.y;
      }
      l[g] = l[g] * corr + ls;
    }
  }
  // merge the two half-warps (same m, disjoint tokens)
#pragma unroll
  for (int g = 0; g < G; ++g) {
    l[g] += __shfl_xor_sync(0xffffffffu, l[g], 16);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], 16);
  }
  // merge warps through shared memory
  __shared__ float sm_m[DEC_WARPS][G], sm_l[DEC_WARPS][G];
  __shared__ float sm_acc[DEC_WARPS][G][D];
  if (half == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sm_acc[warp][g][dl * 8 + j] = acc[g][j];
      if (dl == 0) {
        sm_m[warp][g] = m[g];
        sm_l[warp][g] = l[g];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DEC_WARPS; ++w) {
        const float f = exp2f(sm_m[w][g] - M);
        L += sm_l[w][g] * f;
        O += sm_acc[w][g][d] * f;
      }
    }
    const int hq = kh * G + g;
    if (nsplit == 1) {
      out[(size_t)b * ld_o + (size_t)hq * D + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    } else {
      float* pp = part + (((size_t)b * n_heads + hq) * nsplit + sp) * (D + 2);
      pp[d] = O;
      if (d == 0) {
        pp[D] = M;
        pp[D + 1] = L;
      }
    }
  }
}

// GQA variant (G >= 4 query heads per KV head): the four warps split the G heads (GW =
// ceil(G / 4) each) and every warp streams the whole KV range, so each lane keeps only GW
// heads of q / accumulators in registers (the G = 7 instance of attn_decode_kernel needed
// 255 registers and spilled, running at ~20% of HBM bandwidth).  The four warps read the
// same lines at about the same time: loads allocate in L1 and HBM sees each byte once.
template <int GW>
__global__ void __launch_bounds__(128)
    attn_decode_gqa_kernel(const bf16* __restrict__ q, int ld_q, int n_kv, int G,
                           const int* __restrict__ slots, const int* __restrict__ ctx_len,
                           const int* __restrict__ block_table, int bt_stride,
                           const bf16* __restrict__ kv, long long block_stride, float scale_log2,
                           int blocks_per_split, bf16* __restrict__ out, int ld_o,
                           float* __restrict__ part, int nsplit) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128;
  const int b = blockIdx.x, kh = blockIdx.y, sp = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, dl = lane & 15;
  const int n_heads = n_kv * G;
  const int g0 = warp * GW;  // first head (within the group) of this warp
  const int ng = min(GW, G - g0);
  if (ng <= 0) return;
  const int ctx = ctx_len[b];
  const int nblk = (ctx + HY_KV_BLOCK_TOKENS - 1) / HY_KV_BLOCK_TOKENS;
  const int blk0 = sp * blocks_per_split;
  const int blk1 = min(nblk, blk0 + blocks_per_split);
  const int* bt = block_table + (size_t)slots[b] * bt_stride;
  float qf[GW][8], m[GW], l[GW], acc[GW][8];
#pragma unroll
  for (int g = 0; g < GW; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
    if (g < ng) {
      load_bf16x8(q + (size_t)b * ld_q + (size_t)(kh * G + g0 + g) * D + dl * 8, qf[g]);
#pragma unroll
      for (int j = 0; j < 8; ++j) qf[g][j] *= scale_log2;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) qf[g][j] = 0.f;
    }
  }
  const size_t head_off = (size_t)kh * HY_KV_BLOCK_TOKENS * D;
  const size_t v_off = (size_t)n_kv * HY_KV_BLOCK_TOKENS * D;
  for (int jb = blk0; jb < blk1; ++jb) {
    const bf16* kb = kv + (size_t)bt[jb] * block_stride + head_off;
    const bf16* vb = kb + v_off;
    uint4 kr[8], vr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) kr[i] = *reinterpret_cast<const uint4*>(kb + (size_t)(2 * i + half) * D + dl * 8);
#pragma unroll
    for (int i = 0; i < 8; ++i) vr[i] = *reinterpret_cast<const uint4*>(vb + (size_t)(2 * i + half) * D + dl * 8);
    const int tok_base = jb * HY_KV_BLOCK_TOKENS + half;
#pragma unroll
    for (int g = 0; g < GW; ++g) {
      float s[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float2 k0 = unpack_bf16x2(kr[i].x), k1 = unpack_bf16x2(kr[i].y),
               k2 = unpack_bf16x2(kr[i].z), k3 = unpack_bf16x2(kr[i].w);
        float d0 = qf[g][0] * k0.x + qf[g][1] * k0.y + qf[g][2] * k1.x + qf[g][3] * k1.y +
                   qf[g][4] * k2.x + qf[g][5] * k2.y + qf[g][6] * k3.x + qf[g][7] * k3.y;
        d0 += __shfl_xor_sync(0xffffffffu, d0, 8);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 4);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
        s[i] = (tok_base + 2 * i < ctx) ? d0 : -INFINITY;
      }
      float mb = s[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) mb = fmaxf(mb, s[i]);
      mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
      const float mn = fmaxf(m[g], mb);  // finite: every block holds >= 1 valid token
      const float corr = exp2f(m[g] - mn);
      m[g] = mn;
      float ls = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float p = exp2f(s[i] - mn);
        ls += p;
        float2 v0 = unpack_bf16x2(vr[i].x), v1 = unpack_bf16x2(vr[i].y),
               v2 = unpack_bf16x2(vr[i].z), v3 = unpack_bf16x2(vr[i].w);
        acc[g][0] += p * v0.x; acc[g][1] += p * v0.y;
        acc[g][2] += p * v1.x; acc[g][3] += p * v1.y;
        acc[g][4] += p * v2.x; acc[g][5] += p * v2.y;
        acc[g][6] += p * v3.x; acc[g][7] += p * v3.y;
      }
      l[g] = l[g] * corr + ls;
    }
  }
  // merge the two half-warps (same m, disjoint tokens) and write this warp's heads
#pragma unroll
  for (int g = 0; g < GW; ++g) {
    l[g] += __shfl_xor_sync(0xffffffffu, l[g], 16);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], 16);
    if (g >= ng || half != 0) continue;
    const int hq = kh * G + g0 + g;
    if (nsplit == 1) {
      float o[8];
      const float inv = l[g] > 0.f ? 1.f / l[g] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = acc[g][j] * inv;
      store_bf16x8(out + (size_t)b * ld_o + (size_t)hq * D + dl * 8, o);
    } else {
      float* pp = part + (((size_t)b * n_heads + hq) * nsplit + sp) * (D + 2);
#pragma unroll
      for (int j = 0; j < 8; ++j) pp[dl * 8 + j] = acc[g][j];
      if (dl == 0) {
        pp[D] = m[g];
        pp[D + 1] = l[g];
      }
    }
  }
}

// GQA on tensor cores (G >= 4 query heads per KV head): the G heads of one KV head are the
// (zero-padded) 16 rows of an mma.sync m16n8k16 tile, so each 16-token cache block costs
// 16 + 16 MMAs instead of G x 16 x 128 CUDA-core FMAs plus shuffles -- the CUDA-core
// kernels above are compute/shuffle-bound at G = 7 (~1.7 TB/s).  Warps split the blocks
// (like the MHA kernel); each warp double-buffers its K/V blocks in shared memory with
// cp.async, S = Q K^T and O += P V run on the tensor pipe with the FA2 register reuse of
// the S accumulators as the P operand, online softmax in the exp2 domain; warps merge
// through shared memory, split-KV partials go through the combine kernel.
constexpr int GQ_LDS = 128 + 8;  // padded bf16 row: conflict-free ldmatrix
constexpr int GQ_SMEM = (16 + DEC_WARPS * 4 * 16) * GQ_LDS * 2;  // Q + per warp 2x(K, V)
__global__ void __launch_bounds__(128)
    attn_decode_gqa_mma_kernel(const bf16* __restrict__ q, int ld_q, int n_kv, int G,
                               const int* __restrict__ slots, const int* __restrict__ ctx_len,
                               const int* __restrict__ block_table, int bt_stride,
                               const bf16* __restrict__ kv, long long block_stride,
                               float scale_log2, int blocks_per_split, bf16* __restrict__ out,
                               int ld_o, float* __restrict__ part, int nsplit) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128, LDS = GQ_LDS, CPR = D / 8;
  extern __shared__ __align__(128) uint8_t gq_smem[];
  bf16* sQ = reinterpret_cast<bf16*>(gq_smem);
  const int b = blockIdx.x, kh = blockIdx.y, sp = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_heads = n_kv * G;
  const int ctx = ctx_len[b];
  const int nblk = (ctx + HY_KV_BLOCK_TOKENS - 1) / HY_KV_BLOCK_TOKENS;
  const int blk0 = sp * blocks_per_split;
  const int blk1 = min(nblk, blk0 + blocks_per_split);
  const int* bt = block_table + (size_t)slots[b] * bt_stride;
  bf16* sK = sQ + 16 * LDS + warp * 4 * 16 * LDS;  // [2 bufs][16][LDS]
  bf16* sV = sK + 2 * 16 * LDS;
  // Q rows: the G heads of this KV head (rows >= G zero)
  for (int c = tid; c < 16 * CPR; c += 128) {
    const int r = c / CPR, col = (c % CPR) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < G) v = *reinterpret_cast<const uint4*>(q + (size_t)b * ld_q + (size_t)(kh * G + r) * D + col);
    *reinterpret_cast<uint4*>(sQ + r * LDS + col) = v;
  }
  const size_t head_off = (size_t)kh * HY_KV_BLOCK_TOKENS * D;
  const size_t v_off = (size_t)n_kv * HY_KV_BLOCK_TOKENS * D;
  auto load_block = [&](int jb, int buf) {
    const bf16* kb = kv + (size_t)bt[jb] * block_stride + head_off;
    const bf16* vb = kb + v_off;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = lane + i * 32;  // 256 16-byte pieces per 16 x 128 block
      const int r = c / CPR, col = (c % CPR) * 8;
      cp_async16(sK + buf * 16 * LDS + r * LDS + col, kb + (size_t)r * D + col, true);
      cp_async16(sV + buf * 16 * LDS + r * LDS + col, vb + (size_t)r * D + col, true);
    }
  };
  __syncthreads();
  uint32_t qf[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int row = (lane & 7) + ((lane >> 3) & 1) * 8;
    const int col = kk * 16 + (lane >> 4) * 8;
    ldsm_x4(smem_u32(sQ + row * LDS + col), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows lane/4 and lane/4 + 8
  int jb = blk0 + warp;
  if (jb < blk1) load_block(jb, 0);
  cp_async_commit();
  for (int it = 0; jb < blk1; jb += DEC_WARPS, ++it) {
    const int buf = it & 1;
    if (jb + DEC_WARPS < blk1) load_block(jb + DEC_WARPS, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const bf16* cK = sK + buf * 16 * LDS;
    const bf16* cV = sV + buf * 16 * LDS;
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int key = (lane & 7) + (lane >> 4) * 8;
      const int col = kk * 16 + ((lane >> 3) & 1) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4(smem_u32(cK + key * LDS + col), b0, b1, b2, b3);
      mma_bf16_16816(s[0], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
      mma_bf16_16816(s[1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
    }
    // scale, mask, online softmax (row lo: s[.][0..1], row hi: s[.][2..3])
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = jb * HY_KV_BLOCK_TOKENS + nt * 8 + (lane & 3) * 2 + e;
        const bool ok = tok < ctx;
        s[nt][e] = ok ? s[nt][e] * scale_log2 : -INFINITY;
        s[nt][2 + e] = ok ? s[nt][2 + e] * scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][e]);
        mx1 = fmaxf(mx1, s[nt][2 + e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: block has a valid token
    const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mn0);
      s[nt][1] = exp2f(s[nt][1] - mn0);
      s[nt][2] = exp2f(s[nt][2] - mn1);
      s[nt][3] = exp2f(s[nt][3] - mn1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= c0;
      o[i][1] *= c0;
      o[i][2] *= c1;
      o[i][3] *= c1;
    }
    const uint32_t a0 = pack_bf16x2(s[0][0], s[0][1]), a1 = pack_bf16x2(s[0][2], s[0][3]);
    const uint32_t a2 = pack_bf16x2(s[1][0], s[1][1]), a3 = pack_bf16x2(s[1][2], s[1][3]);
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      const int key = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int col = dp * 16 + (lane >> 4) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(smem_u32(cV + key * LDS + col), b0, b1, b2, b3);
      mma_bf16_16816(o[2 * dp], a0, a1, a2, a3, b0, b1);
      mma_bf16_16816(o[2 * dp + 1], a0, a1, a2, a3, b2, b3);
    }
    __syncwarp();  // this buffer is refilled two iterations later
  }
  cp_async_wait<0>();
  // row sums over the 4 lanes sharing a row
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  // merge warps through shared memory (reuses the K/V buffers)
  __syncthreads();
  float* sO = reinterpret_cast<float*>(gq_smem);            // [4][16][128]
  float* sM = sO + DEC_WARPS * 16 * D;                       // [4][16]
  float* sL = sM + DEC_WARPS * 16;                           // [4][16]
  const int r0 = lane >> 2, r1 = r0 + 8;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int col = i * 8 + (lane & 3) * 2;
    sO[(warp * 16 + r0) * D + col] = o[i][0];
    sO[(warp * 16 + r0) * D + col + 1] = o[i][1];
    sO[(warp * 16 + r1) * D + col] = o[i][2];
    sO[(warp * 16 + r1) * D + col + 1] = o[i][3];
  }
  if ((lane & 3) == 0) {
    sM[warp * 16 + r0] = m0;
    sM[warp * 16 + r1] = m1;
    sL[warp * 16 + r0] = l0;
    sL[warp * 16 + r1] = l1;
  }
  __syncthreads();
  for (int e = tid; e < G * D; e += blockDim.x) {
    const int g = e / D, d = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, sM[w * 16 + g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DEC_WARPS; ++w) {
        const float f = exp2f(sM[w * 16 + g] - M);
        L += sL[w * 16 + g] * f;
        O += sO[(w * 16 + g) * D + d] * f;
      }
    }
    const int hq = kh * G + g;
    if (nsplit == 1) {
      out[(size_t)b * ld_o + (size_t)hq * D + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    } else {
      float* pp = part + (((size_t)b * n_heads + hq) * nsplit + sp) * (D + 2);
      pp[d] = O;
      if (d == 0) {
        pp[D] = M;
        pp[D + 1] = L;
      }
    }
  }
}

__global__ void attn_decode_combine_kernel(const float* __restrict__ part, int n_heads, int nsplit,
                                           bf16* __restrict__ out, int ld_o) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128;
  const int b = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const float* pp = part + ((size_t)b * n_heads + h) * nsplit * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, pp[s * (D + 2) + D]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < nsplit; ++s) {
      const float f = exp2f(pp[s * (D + 2) + D] - M);
      L += pp[s * (D + 2) + D + 1] * f;
      O += pp[s * (D + 2) + d] * f;
    }
  }
  out[(size_t)b * ld_o + (size_t)h * D + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
}

// KV splits per (sequence, KV head): enough CTAs for ~per_sm per SM.  GQA CTAs (G >= 4
// query heads per KV head, tensor-core kernel) aim for 4 per SM -- each already does G
// heads of work per byte, and fewer splits save the combine pass (Qwen2-VL 28/4, 256 x 660
// context: 70 us at 4 vs 83 us at 8, 5.7 vs 5.4 TB/s at 64 x 4000); MHA keeps 8
// (tools/kernel_sweep.py --what decode; HY_DECODE_CTAS_PER_SM overrides for A/B).
static int decode_splits(int n, int n_kv, int max_ctx, int G = 1) {
  const int max_blocks = std::max(1, ceil_div(max_ctx, HY_KV_BLOCK_TOKENS));
  static const int env_per_sm = [] {
    const char* e = getenv("HY_DECODE_CTAS_PER_SM");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const int per_sm = env_per_sm ? env_per_sm : (G >= 4 ? 4 : 8);
  const int target = num_sms() * per_sm;
  int ns = ceil_div(target, std::max(1, n * n_kv));
  ns = std::min(ns, std::max(1, max_blocks / 4));  // >= 4 blocks per split: one per warp
  return std::max(1, std::min(ns, 64));
}

}  // namespace hy

using namespace hy;

extern "C" size_t hy_attn_decode_workspace_bytes(int n, int n_heads, int head_dim, int max_ctx) {
  const int ns = decode_splits(n, n_heads, max_ctx);  // n_kv <= n_heads: upper bound
  return (size_t)n * n_heads * std::max(ns, 64) * (head_dim + 2) * sizeof(float);
}

extern "C" int hy_attn_decode_paged(const void* q, int ld_q, int n, int n_heads, int n_kv_heads,
                                    int head_dim, const int* slots, const int* ctx, int max_ctx,
                                    const int* block_table, int bt_stride, const void* kv_layer,
                                    long long block_stride, float scale, void* out, int ld_o,
                                    void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  HY_CHECK_ARG(head_dim == 128, "decode attention supports head_dim 128");
  HY_CHECK_ARG(n_kv_heads > 0 && n_heads % n_kv_heads == 0, "heads");
  if (n <= 0) return 0;
  const int G = n_heads / n_kv_heads;
  int ns = decode_splits(n, n_kv_heads, max_ctx, G);
  const size_t need = (size_t)n * n_heads * ns * (head_dim + 2) * sizeof(float);
  if (ns > 1 && (workspace == nullptr || need > workspace_bytes)) ns = 1;
  const int max_blocks = std::max(1, ceil_div(max_ctx, HY_KV_BLOCK_TOKENS));
  const int bps = ceil_div(max_blocks, ns);
  ns = ceil_div(max_blocks, bps);
  dim3 grid(n, n_kv_heads, ns);
  const float sl2 = scale * 1.4426950408889634f;
  const bf16* qp = reinterpret_cast<const bf16*>(q);
  const bf16* kvp = reinterpret_cast<const bf16*>(kv_layer);
  bf16* op = reinterpret_cast<bf16*>(out);
  float* part = reinterpret_cast<float*>(workspace);
#define HY_DEC_CASE(GG)                                                                        \
  case GG:                                                                                     \
    HY_CUDA_RET(launch_pdl(attn_decode_kernel<GG>, dim3(grid), dim3(128), 0, stream, qp, ld_q, n_kv_heads, slots, ctx,         \
                                                     block_table, bt_stride, kvp, block_stride, \
                                                     sl2, bps, op, ld_o, part, ns));            \
    break;
  if (G >= 4 && G <= 16 && !getenv("HY_DECODE_GQA_CUDA")) {
    HY_CUDA_RET(ensure_smem(attn_decode_gqa_mma_kernel,
                            std::max(GQ_SMEM, (DEC_WARPS * 16 * 130 + 64) * 4)));
    HY_CUDA_RET(launch_pdl(attn_decode_gqa_mma_kernel, dim3(grid), dim3(128),
                           (size_t)std::max(GQ_SMEM, (DEC_WARPS * 16 * 130 + 64) * 4), stream,
                           qp, ld_q, n_kv_heads, G, slots, ctx, block_table, bt_stride, kvp,
                           block_stride, sl2, bps, op, ld_o, part, ns));
  } else if (G >= 4 && G <= 16) {
    // warps split the heads: GW = ceil(G / 4) heads per warp
    auto launch_gqa = [&](auto kern) {
      return launch_pdl(kern, dim3(grid), dim3(128), 0, stream, qp, ld_q, n_kv_heads, G, slots,
                        ctx, block_table, bt_stride, kvp, block_stride, sl2, bps, op, ld_o, part,
                        ns);
    };
    if (G <= 4)
      HY_CUDA_RET(launch_gqa(attn_decode_gqa_kernel<1>));
    else if (G <= 8)
      HY_CUDA_RET(launch_gqa(attn_decode_gqa_kernel<2>));
    else
      HY_CUDA_RET(launch_gqa(attn_decode_gqa_kernel<4>));
  } else switch (G) {
    HY_DEC_CASE(1)
    HY_DEC_CASE(2)
    HY_DEC_CASE(4)
    HY_DEC_CASE(7)
    HY_DEC_CASE(8)
    default:
      set_last_error("decode attention: unsupported GQA group " + std::to_string(G));
      return (int)cudaErrorInvalidValue;
  }
#undef HY_DEC_CASE
  HY_LAUNCH_CHECK();
  if (ns > 1) {
    HY_CUDA_RET(launch_pdl(attn_decode_combine_kernel, dim3(dim3(n, n_heads)), dim3(128), 0, stream, part, n_heads, ns, op, ld_o));
    HY_LAUNCH_CHECK();
  }
  return 0;
}
