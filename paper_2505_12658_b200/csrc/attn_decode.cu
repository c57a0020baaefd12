// K8: paged-KV decode attention (one query token per running decode entry).
//
// The dominant HBM stream at large decode batches: every step reads the whole cached
// context of every running request, bytes = sum_i (S_i + 1) * kv_bytes_per_token
// (epdsim charges 2*B*H*(S+1)*ratio per layer, model_cost.py:195).
//
// Layout read: KV pool block [layer][K|V][kv_head][16 tok][d], so one (block, head) K
// tile is 16 x d contiguous bf16 (4 KiB at d = 128).
//
// Grid (kv_head, seq, split).  Each of the 4 warps streams whole 16-token blocks:
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

// CO = 1: the same kernel as a separate function whose shared-memory carveout is set to the
// maximum, so its CTAs can share SMs with a GEMM (co-resident mode); CO = 0 keeps the
// default carveout (a larger L1: ~13% faster when it runs alone, 7.0 vs 6.1 TB/s).
template <int G, int CO = 0>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const bf16* __restrict__ q, int ld_q, int n_kv, const int* __restrict__ slots,
                       const int* __restrict__ ctx_len, const int* __restrict__ block_table,
                       int bt_stride, const bf16* __restrict__ kv, long long block_stride,
                       float scale_log2, int blocks_per_split, bf16* __restrict__ out, int ld_o,
                       float* __restrict__ part, int nsplit) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128;
  const int b = blockIdx.y, kh = blockIdx.x, sp = blockIdx.z;  // grid (kv head, seq, split)
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
  const int b = blockIdx.y, kh = blockIdx.x, sp = blockIdx.z;  // grid (kv head, seq, split)
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
  const int b = blockIdx.y, kh = blockIdx.x, sp = blockIdx.z;  // grid (kv head, seq, split)
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

// K8b: MHA decode attention with the KV stream landing in shared memory through bulk
// copies (cp.async.bulk + mbarrier) instead of register loads.
//
// Built to run on the SAME SMs as a tensor-bound GEMM of another row group (decode /
// prefill split): a register-load kernel is capped by the L1 space its in-flight lines
// need (28 KB beside a GEMM that takes the maximum shared carveout), while bulk copies land
// in a small explicit ring -- NW warps x SPW stages x 8 KB (K and V tile of one 16-token
// block of one head) -- that fits next to the GEMM's operand ring.  Each warp is an
// independent pipeline: lane 0 issues the copies of the next stages (the item's q rides in
// its first stage), all 32 lanes consume, and items (sequence, head, KV split) come from a
// global ticket counter, so SMs slowed by a co-resident GEMM simply take fewer items.  The
// last warp to finish resets the counter for the next launch.
constexpr int DB_STAGE = 2 * HY_KV_BLOCK_TOKENS * 128 * 2 + 256;  // K | V | q (256 B)

template <int NW, int SPW>
__global__ void __launch_bounds__(32 * NW)
    attn_decode_bulk_kernel(const bf16* __restrict__ q, int ld_q, int n, int n_heads,
                            const int* __restrict__ slots, const int* __restrict__ ctx_len,
                            const int* __restrict__ block_table, int bt_stride,
                            const bf16* __restrict__ kv, long long block_stride, float scale_log2,
                            int bps, int nsplit, bf16* __restrict__ out, int ld_o,
                            float* __restrict__ part, int* __restrict__ ctr) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128;
  extern __shared__ __align__(128) uint8_t db_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, dl = lane & 15;
  uint8_t* ring = db_smem + (size_t)warp * SPW * DB_STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(db_smem + (size_t)NW * SPW * DB_STAGE) + warp * SPW;
  int2* meta = reinterpret_cast<int2*>(db_smem + (size_t)NW * SPW * DB_STAGE + NW * SPW * 8) +
               warp * SPW;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < SPW; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int n_items = n * n_heads * nsplit;
  const size_t head_bytes = (size_t)HY_KV_BLOCK_TOKENS * D;  // ELEMENTS of one head's tile
  const size_t v_off = (size_t)n_heads * head_bytes;

  // ---- load cursor (warp-uniform): current item, its block range, block ids in lanes
  int l_item = -1, l_b = 0, l_h = 0, l_blk = 0, l_end = 0, l_first = 0, l_bid = 0;
  int next_t = 0;
  if (lane == 0) next_t = atomicAdd(ctr, 1);
  next_t = __shfl_sync(0xffffffffu, next_t, 0);
  bool exhausted = false;
  auto advance_item = [&]() {
    while (true) {
      const int t = next_t;
      if (t >= n_items) {
        exhausted = true;
        return;
      }
      int nt = 0;
      if (lane == 0) nt = atomicAdd(ctr, 1);  // one ticket ahead: latency overlaps this item
      next_t = __shfl_sync(0xffffffffu, nt, 0);
      const int sp = t / (n * n_heads);
      const int r = t - sp * n * n_heads;
      const int b = r / n_heads, h = r - b * n_heads;
      const int nblk = (ctx_len[b] + HY_KV_BLOCK_TOKENS - 1) / HY_KV_BLOCK_TOKENS;
      const int b0 = sp * bps, b1 = min(nblk, b0 + bps);
      if (b0 >= b1) {  // empty split of a short sequence: an empty partial for the combine
        float* pp = part + ((size_t)r * nsplit + sp) * (D + 2);
        for (int i = lane; i < D + 2; i += 32) pp[i] = i == D ? -INFINITY : 0.f;
        continue;
      }
      l_item = t;
      l_b = b;
      l_h = h;
      l_blk = l_first = b0;
      l_end = b1;
      const int* bt = block_table + (size_t)slots[b] * bt_stride;
      l_bid = b0 + lane < b1 ? bt[b0 + lane] : 0;  // bps <= 32
      return;
    }
  };
  auto issue = [&](int st) {
    if (!exhausted && l_blk >= l_end) advance_item();
    const uint32_t sb = smem_u32(ring + (size_t)st * DB_STAGE);
    if (exhausted) {
      if (lane == 0) {
        meta[st] = make_int2(-1, 0);
        mbar_arrive(&bar[st]);
      }
      return;
    }
    const int bid = __shfl_sync(0xffffffffu, l_bid, l_blk - l_first);
    if (lane == 0) {
      const bool first = l_blk == l_first;
      meta[st] = make_int2(l_item, l_blk | (first ? (1 << 30) : 0));
      fence_proxy_async_smem();  // the consumer's reads of this stage precede the refill
      mbar_expect_tx(&bar[st], 2 * head_bytes * 2 + (first ? D * 2 : 0));
      const bf16* kb = kv + (size_t)bid * block_stride + (size_t)l_h * head_bytes;
      bulk_load_1d(sb, kb, head_bytes * 2, smem_u32(&bar[st]), kEvictFirst);
      bulk_load_1d(sb + head_bytes * 2, kb + v_off, head_bytes * 2, smem_u32(&bar[st]), kEvictFirst);
      if (first)
        bulk_load_1d(sb + 4 * head_bytes, q + (size_t)l_b * ld_q + (size_t)l_h * D, D * 2,
                     smem_u32(&bar[st]), kEvictFirst);
    }
    ++l_blk;
  };

#pragma unroll
  for (int st = 0; st < SPW; ++st) issue(st);

  // ---- consumer
  int c_item = -1, c_ctx = 0;
  float qf[8], m = -INFINITY, l = 0.f, acc[8];
  auto finish = [&]() {
    if (c_item < 0) return;
    l += __shfl_xor_sync(0xffffffffu, l, 16);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 16);
    const int sp = c_item / (n * n_heads);
    const int r = c_item - sp * n * n_heads;  // = b * n_heads + h
    if (half == 0) {
      if (nsplit == 1) {
        const int b = r / n_heads, h = r - b * n_heads;
        float o[8];
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = acc[j] * inv;
        store_bf16x8(out + (size_t)b * ld_o + (size_t)h * D + dl * 8, o);
      } else {
        float* pp = part + ((size_t)r * nsplit + sp) * (D + 2);
        float2* p2 = reinterpret_cast<float2*>(pp + dl * 8);  // rows of D + 2 floats: 8B aligned
#pragma unroll
        for (int j = 0; j < 4; ++j) p2[j] = make_float2(acc[2 * j], acc[2 * j + 1]);
        if (dl == 0) {
          pp[D] = m;
          pp[D + 1] = l;
        }
      }
    }
  };
  int st = 0;
  uint32_t ph = 0;
  while (true) {
    mbar_wait(&bar[st], ph);
    const int2 md = meta[st];
    if (md.x < 0) break;
    const uint32_t sb = smem_u32(ring + (size_t)st * DB_STAGE);
    if (md.x != c_item) {
      finish();
      c_item = md.x;
      c_ctx = ctx_len[(md.x % (n * n_heads)) / n_heads];
      m = -INFINITY;
      l = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
      const float4 q0 = lds_f32x4(sb + 4 * head_bytes + dl * 16);
      const uint32_t qw[4] = {__float_as_uint(q0.x), __float_as_uint(q0.y), __float_as_uint(q0.z),
                              __float_as_uint(q0.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(qw[j]);
        qf[2 * j] = f.x * scale_log2;
        qf[2 * j + 1] = f.y * scale_log2;
      }
    }
    const int jb = md.y & ((1 << 30) - 1);
    const int ctx = c_ctx;
    const int tok_base = jb * HY_KV_BLOCK_TOKENS + half;
    float s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 kq = lds_f32x4(sb + (2 * i + half) * D * 2 + dl * 16);
      const float2 k0 = unpack_bf16x2(__float_as_uint(kq.x)), k1 = unpack_bf16x2(__float_as_uint(kq.y)),
                   k2 = unpack_bf16x2(__float_as_uint(kq.z)), k3 = unpack_bf16x2(__float_as_uint(kq.w));
      float d0 = qf[0] * k0.x + qf[1] * k0.y + qf[2] * k1.x + qf[3] * k1.y + qf[4] * k2.x +
                 qf[5] * k2.y + qf[6] * k3.x + qf[7] * k3.y;
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
    const float mn = fmaxf(m, mb);  // finite: every block holds >= 1 valid token
    const float corr = exp2f(m - mn);
    m = mn;
    float ls = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] *= corr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float p = exp2f(s[i] - mn);
      ls += p;
      const float4 vq = lds_f32x4(sb + 2 * head_bytes + (2 * i + half) * D * 2 + dl * 16);
      const float2 v0 = unpack_bf16x2(__float_as_uint(vq.x)), v1 = unpack_bf16x2(__float_as_uint(vq.y)),
                   v2 = unpack_bf16x2(__float_as_uint(vq.z)), v3 = unpack_bf16x2(__float_as_uint(vq.w));
      acc[0] += p * v0.x; acc[1] += p * v0.y;
      acc[2] += p * v1.x; acc[3] += p * v1.y;
      acc[4] += p * v2.x; acc[5] += p * v2.y;
      acc[6] += p * v3.x; acc[7] += p * v3.y;
    }
    l = l * corr + ls;
    __syncwarp();  // every lane has read the stage before lane 0 refills it
    issue(st);
    if (++st == SPW) {
      st = 0;
      ph ^= 1;
    }
  }
  finish();
  // the last warp of the grid resets the ticket counter (every warp has taken its last
  // ticket before it counts itself done)
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)(gridDim.x * NW) - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

// K8c: decode attention built to share every SM with a tensor-bound GEMM of another row
// group (co-resident mode, decode / prefill split).  Three things make it fit beside a
// GEMM CTA (181.5 KB of shared memory, 46 K registers) and still pull bytes:
//  * the KV stream lands in a small explicit shared-memory ring through bulk copies
//    (cp.async.bulk, one 256-byte token row per lane, rows padded to 272 bytes so ldmatrix
//    is conflict-free) -- not through L1, which a GEMM's maximum carveout shrinks to 28 KB;
//  * S = Q K^T and O += P V run on mma.sync m16n8k16 with the G query heads of a KV head as
//    the tile rows (G = 1 for MHA: one useful row, but 32 MMAs per 16-token block instead of
//    ~350 CUDA-core instructions), so one warp consumes ~4x more bytes per second;
//  * at most ONE CTA per SM: a CTA that lands on an SM already holding one exits at once
//    (per-SM flags), so two of them can never take the room a GEMM CTA needs.
// Items (sequence, KV head, split) come from a ticket counter; each warp streams whole items
// through its own ring (lane 0 issues, all lanes consume), block ids reloaded 32 at a time.
// PAD = false (lab): the K and V tiles arrive as two 4 KB copies in the pool's own 256-byte
// row layout (ldmatrix then has 8-way bank conflicts) -- to weigh the per-copy cost of the
// TMA engine against the conflicts.
template <int G, bool PAD = true>
struct DcCfg {
  static constexpr int LDS = PAD ? 136 : 128;            // row stride (bf16): 272 / 256 bytes
  static constexpr int TILE = 16 * LDS * 2;              // one 16-token K or V tile
  static constexpr int Q_BYTES = G * LDS * 2;
  static constexpr int STAGE = 2 * TILE + Q_BYTES;       // K | V | q rows of the item
};

template <int G, int NW, int SPW, bool PAD = true>
__global__ void __launch_bounds__(32 * NW)
    attn_decode_co_kernel(const bf16* __restrict__ q, int ld_q, int n, int n_kv,
                          const int* __restrict__ slots, const int* __restrict__ ctx_len,
                          const int* __restrict__ block_table, int bt_stride,
                          const bf16* __restrict__ kv, long long block_stride, float scale_log2,
                          int bps, int nsplit, bf16* __restrict__ out, int ld_o,
                          float* __restrict__ part, int* __restrict__ ctr) {
  pdl_trigger();
  constexpr int D = 128;
  constexpr int STAGE = DcCfg<G, PAD>::STAGE;
  constexpr int DC_LDS = DcCfg<G, PAD>::LDS, DC_TILE = DcCfg<G, PAD>::TILE;
  extern __shared__ __align__(128) uint8_t dc_smem[];
  __shared__ int s_dup;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* sm_flag = ctr + 256;
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s_dup = atomicCAS(sm_flag + (smid & 255), 0, 1) != 0 ? 1 : 0;
  }
  __syncthreads();
  if (s_dup) {  // another CTA of this grid owns this SM: leave the room to the GEMM
    if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
    return;
  }
  pdl_wait();
  uint8_t* ring = dc_smem + (size_t)warp * SPW * STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(dc_smem + (size_t)NW * SPW * STAGE) + warp * SPW;
  int2* meta = reinterpret_cast<int2*>(dc_smem + (size_t)NW * SPW * STAGE + NW * SPW * 8) + warp * SPW;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < SPW; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int n_items = n * n_kv * nsplit;
  const size_t tile_elems = (size_t)HY_KV_BLOCK_TOKENS * D;
  const size_t v_off = (size_t)n_kv * tile_elems;

  // ---- load cursor (warp-uniform)
  int l_item = -1, l_b = 0, l_h = 0, l_blk = 0, l_end = 0, l_first = 0, l_base = 0, l_bid = 0;
  const int* l_bt = nullptr;
  int next_t = 0;
  if (lane == 0) next_t = atomicAdd(ctr, 1);
  next_t = __shfl_sync(0xffffffffu, next_t, 0);
  bool exhausted = false;
  auto advance_item = [&]() {
    while (true) {
      const int t = next_t;
      if (t >= n_items) {
        exhausted = true;
        return;
      }
      int nt = 0;
      if (lane == 0) nt = atomicAdd(ctr, 1);  // one ticket ahead
      next_t = __shfl_sync(0xffffffffu, nt, 0);
      const int sp = t / (n * n_kv);
      const int r = t - sp * n * n_kv;
      const int b = r / n_kv, h = r - b * n_kv;
      const int nblk = (ctx_len[b] + HY_KV_BLOCK_TOKENS - 1) / HY_KV_BLOCK_TOKENS;
      const int b0 = sp * bps, b1 = min(nblk, b0 + bps);
      if (b0 >= b1) {  // empty split: empty partials (M = -inf, L = 0) for the combine
        for (int g = 0; g < G; ++g) {
          float* pp = part + (((size_t)b * n_kv * G + h * G + g) * nsplit + sp) * (D + 2);
          for (int i = lane; i < D + 2; i += 32) pp[i] = i == D ? -INFINITY : 0.f;
        }
        continue;
      }
      l_item = t;
      l_b = b;
      l_h = h;
      l_blk = l_first = l_base = b0;
      l_end = b1;
      l_bt = block_table + (size_t)slots[b] * bt_stride;
      l_bid = b0 + lane < b1 ? l_bt[b0 + lane] : 0;
      return;
    }
  };
  auto issue = [&](int st) {
    if (!exhausted && l_blk >= l_end) advance_item();
    const uint32_t sb = smem_u32(ring + (size_t)st * STAGE);
    if (exhausted) {
      if (lane == 0) {
        meta[st] = make_int2(-1, 0);
        mbar_arrive(&bar[st]);
      }
      return;
    }
    if (l_blk - l_base >= 32) {  // next 32 block ids
      l_base += 32;
      l_bid = l_base + lane < l_end ? l_bt[l_base + lane] : 0;
    }
    const int bid = __shfl_sync(0xffffffffu, l_bid, l_blk - l_base);
    const bool first = l_blk == l_first;
    if (lane == 0) {
      meta[st] = make_int2(l_item, l_blk | (first ? (1 << 30) : 0));
      fence_proxy_async_smem();  // the consumer's reads of this stage precede the refill
      mbar_expect_tx(&bar[st], 2 * tile_elems * 2 + (first ? G * D * 2 : 0));
    }
    __syncwarp();  // expect_tx before any lane's copy can complete
    if (PAD) {
      // lanes 0-15: K rows, 16-31: V rows of this (block, KV head); 256 bytes each
      const bf16* src = kv + (size_t)bid * block_stride + (size_t)l_h * tile_elems +
                        (lane >> 4) * v_off + (size_t)(lane & 15) * D;
      bulk_load_1d(sb + (lane >> 4) * DC_TILE + (lane & 15) * DC_LDS * 2, src, D * 2,
                   smem_u32(&bar[st]), kEvictFirst);
    } else if (lane < 2) {
      const bf16* src = kv + (size_t)bid * block_stride + (size_t)l_h * tile_elems + lane * v_off;
      bulk_load_1d(sb + lane * DC_TILE, src, (uint32_t)tile_elems * 2, smem_u32(&bar[st]),
                   kEvictFirst);
    }
    if (first && lane < G)
      bulk_load_1d(sb + 2 * DC_TILE + lane * DC_LDS * 2,
                   q + (size_t)l_b * ld_q + (size_t)(l_h * G + lane) * D, D * 2,
                   smem_u32(&bar[st]), kEvictFirst);
    ++l_blk;
  };

#pragma unroll
  for (int st = 0; st < SPW; ++st) issue(st);

  // ---- consumer
  const int r0 = lane >> 2;  // accumulator rows r0 (c0, c1) and r0 + 8 (c2, c3)
  int c_item = -1, c_ctx = 0;
  uint32_t qf[8][4];
  float o[16][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  auto finish = [&]() {
    if (c_item < 0) return;
    float L0 = l0 + __shfl_xor_sync(0xffffffffu, l0, 1);
    L0 += __shfl_xor_sync(0xffffffffu, L0, 2);
    const int sp = c_item / (n * n_kv);
    const int r = c_item - sp * n * n_kv;  // = b * n_kv + h
    if (r0 < G) {  // G <= 8: only the c0 / c1 rows carry heads
      const int b = r / n_kv, h = r - b * n_kv;
      const int hq = h * G + r0;
      if (nsplit == 1) {
        const float inv = L0 > 0.f ? 1.f / L0 : 0.f;
        bf16* op = out + (size_t)b * ld_o + (size_t)hq * D + (lane & 3) * 2;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          *reinterpret_cast<uint32_t*>(op + i * 8) = pack_bf16x2(o[i][0] * inv, o[i][1] * inv);
      } else {
        float* pp = part + (((size_t)b * n_kv * G + hq) * nsplit + sp) * (D + 2);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          *reinterpret_cast<float2*>(pp + i * 8 + (lane & 3) * 2) = make_float2(o[i][0], o[i][1]);
        if ((lane & 3) == 0) {
          pp[D] = m0;
          pp[D + 1] = L0;
        }
      }
    }
  };
  int st = 0;
  uint32_t ph = 0;
  while (true) {
    mbar_wait(&bar[st], ph);
    const int2 md = meta[st];
    if (md.x < 0) break;
    const uint32_t sb = smem_u32(ring + (size_t)st * STAGE);
    if (md.x != c_item) {
      finish();
      c_item = md.x;
      c_ctx = ctx_len[(md.x % (n * n_kv)) / n_kv];
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      // q fragments (rows >= G zero): a0 (r0, k), a1 (r0 + 8, k), a2 (r0, k + 8), a3 (r0 + 8, k + 8)
      const uint32_t qa = sb + 2 * DC_TILE + r0 * DC_LDS * 2 + (lane & 3) * 4;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t x0 = 0, x2 = 0;
        if (r0 < G) {
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x0) : "r"(qa + kk * 32));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x2) : "r"(qa + kk * 32 + 16));
        }
        qf[kk][0] = x0;
        qf[kk][1] = 0u;
        qf[kk][2] = x2;
        qf[kk][3] = 0u;
      }
    }
    const int jb = md.y & ((1 << 30) - 1);
    const uint32_t cK = sb, cV = sb + DC_TILE;
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int key = (lane & 7) + (lane >> 4) * 8;
      const int col = kk * 16 + ((lane >> 3) & 1) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4(cK + (key * DC_LDS + col) * 2, b0, b1, b2, b3);
      mma_bf16_16816(s[0], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
      mma_bf16_16816(s[1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
    }
    float mx0 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = jb * HY_KV_BLOCK_TOKENS + nt * 8 + (lane & 3) * 2 + e;
        s[nt][e] = tok < c_ctx ? s[nt][e] * scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    const float mn0 = fmaxf(m0, mx0);  // finite: every block holds a valid token
    const float cr0 = exp2f(m0 - mn0);
    m0 = mn0;
    float rs0 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mn0);
      s[nt][1] = exp2f(s[nt][1] - mn0);
      rs0 += s[nt][0] + s[nt][1];
    }
    l0 = l0 * cr0 + rs0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= cr0;
      o[i][1] *= cr0;
    }
    // P (rows 8-15 zero) as the A operand
    const uint32_t a0 = pack_bf16x2(s[0][0], s[0][1]), a2 = pack_bf16x2(s[1][0], s[1][1]);
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      const int key = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int col = dp * 16 + (lane >> 4) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(cV + (key * DC_LDS + col) * 2, b0, b1, b2, b3);
      mma_bf16_16816(o[2 * dp], a0, 0u, a2, 0u, b0, b1);
      mma_bf16_16816(o[2 * dp + 1], a0, 0u, a2, 0u, b2, b3);
    }
    __syncwarp();  // every lane has read the stage before it is refilled
    issue(st);
    if (++st == SPW) {
      st = 0;
      ph ^= 1;
    }
  }
  finish();
  (void)m1;
  (void)l1;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    sm_flag[smid & 255] = 0;
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
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

// Workspace: [ticket counters: 256 B, zero between launches][split-KV partials]
static constexpr size_t kDecCtrBytes = 2048;  // [0]: tickets, [1]: done; [256..511]: SM flags

extern "C" size_t hy_attn_decode_workspace_bytes(int n, int n_heads, int head_dim, int max_ctx) {
  const int ns = decode_splits(n, n_heads, max_ctx);  // n_kv <= n_heads: upper bound
  return kDecCtrBytes + (size_t)n * n_heads * std::max(ns, 64) * (head_dim + 2) * sizeof(float);
}

namespace hy {
// Per-thread choice of the MHA decode kernel (decode_set_coresident): the bulk-copy kernel
// when the decode attention is meant to share SMs with another stream's GEMM.
static thread_local int t_dec_coresident = 0;
static thread_local int t_dec_nw = 0, t_dec_spw = 0;  // hy_set_decode_kernel
void decode_set_coresident(int on) { t_dec_coresident = on; }

struct BulkCfg {
  int nw, spw;
};
// HY_DECODE_BULK=<nw>,<spw> forces the bulk kernel everywhere (A/B).  Measured beside a GEMM
// it does not pay: one 34 KB CTA per SM keeps too few bytes in flight (2.5-3.5 TB/s alone,
// tools/overlap_lab.py), so co-resident launches use K8 with the maximum carveout instead.
static BulkCfg bulk_cfg() {
  static const BulkCfg env = [] {
    BulkCfg c{0, 0};
    if (const char* e = getenv("HY_DECODE_BULK")) sscanf(e, "%d,%d", &c.nw, &c.spw);
    return c;
  }();
  if (t_dec_nw > 0) return BulkCfg{t_dec_nw, t_dec_spw};
  return env;
}

template <int NW, int SPW>
static int launch_bulk(const bf16* q, int ld_q, int n, int n_heads, const int* slots,
                       const int* ctx, int max_ctx, const int* bt, int bt_stride, const bf16* kv,
                       long long block_stride, float sl2, bf16* out, int ld_o, uint8_t* ws,
                       size_t ws_bytes, cudaStream_t stream) {
  constexpr int SMEM = NW * SPW * (DB_STAGE + 8 + 8);
  auto kern = attn_decode_bulk_kernel<NW, SPW>;
  HY_CUDA_RET(ensure_smem(kern, SMEM));
  HY_CUDA_RET(ensure_max_carveout(kern));
  static thread_local int occ_dev = -1, occ = 0;
  int dev = 0;
  HY_CUDA_RET(cudaGetDevice(&dev));
  if (occ_dev != dev) {
    HY_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * NW, SMEM));
    occ_dev = dev;
  }
  const int max_blocks = std::max(1, ceil_div(max_ctx, HY_KV_BLOCK_TOKENS));
  // items: >= ~8 per warp of one CTA per SM, at most 32 blocks each (block ids in lanes)
  const int want = 8 * num_sms() * NW;
  int ns = std::max(1, std::min(ceil_div(want, std::max(1, n * n_heads)), ceil_div(max_blocks, 4)));
  int bps = std::min(32, ceil_div(max_blocks, ns));
  ns = ceil_div(max_blocks, bps);
  const size_t need = kDecCtrBytes + (size_t)n * n_heads * ns * (128 + 2) * sizeof(float);
  if (ns > 1 && need > ws_bytes) {
    set_last_error("decode attention: workspace too small for the bulk kernel");
    return (int)cudaErrorInvalidValue;
  }
  const long long items = (long long)n * n_heads * ns;
  // CTAs per SM: the occupancy limit alone; ONE beside a GEMM (co-resident mode), so the
  // persistent CTAs never take the shared memory a GEMM CTA needs on any SM
  static const int env_cps = [] {
    const char* e = getenv("HY_DECODE_BULK_CPS");
    return e ? atoi(e) : 0;
  }();
  const int cps = env_cps > 0 ? env_cps : t_dec_coresident ? 1 : std::max(occ, 1);
  static const int env_grid = [] {
    const char* e = getenv("HY_DECODE_BULK_GRID");  // lab: cap the CTA count (SM subsets)
    return e ? atoi(e) : 0;
  }();
  long long g = std::min<long long>((long long)num_sms() * std::min(cps, std::max(occ, 1)),
                                    ceil_div(items, NW));
  if (env_grid > 0) g = std::min<long long>(g, env_grid);
  const int grid = (int)std::max<long long>(1, g);
  int* ctr = reinterpret_cast<int*>(ws);
  float* part = reinterpret_cast<float*>(ws + kDecCtrBytes);
  // the counters start at zero on every call: a caller's workspace may move between calls
  // (hy_lang_forward carves it per batch), so a reset left by the previous launch is not enough
  HY_CUDA_RET(cudaMemsetAsync(ws, 0, kDecCtrBytes, stream));
  HY_CUDA_RET(launch_pdl(kern, dim3(grid), dim3(32 * NW), (size_t)SMEM, stream, q, ld_q, n,
                         n_heads, slots, ctx, bt, bt_stride, kv, block_stride, sl2, bps, ns, out,
                         ld_o, part, ctr));
  HY_LAUNCH_CHECK();
  if (ns > 1) {
    HY_CUDA_RET(launch_pdl(attn_decode_combine_kernel, dim3(n, n_heads), dim3(128), 0, stream,
                           (const float*)part, n_heads, ns, out, ld_o));
    HY_LAUNCH_CHECK();
  }
  return 0;
}

// Co-resident K8c launch: one CTA per SM at most (the kernel enforces it), whole sequences
// per item unless that leaves fewer than ~4 items per warp.
template <int G, int NW, int SPW, bool PAD = true>
static int launch_co(const bf16* q, int ld_q, int n, int n_kv, const int* slots, const int* ctx,
                     int max_ctx, const int* bt, int bt_stride, const bf16* kv,
                     long long block_stride, float sl2, bf16* out, int ld_o, uint8_t* ws,
                     size_t ws_bytes, cudaStream_t stream) {
  constexpr int SMEM = NW * SPW * (DcCfg<G, PAD>::STAGE + 16);
  auto kern = attn_decode_co_kernel<G, NW, SPW, PAD>;
  HY_CUDA_RET(ensure_smem(kern, SMEM));
  HY_CUDA_RET(ensure_max_carveout(kern));
  const int max_blocks = std::max(1, ceil_div(max_ctx, HY_KV_BLOCK_TOKENS));
  const int want = 4 * num_sms() * NW;
  const int ns0 = std::max(
      1, std::min(std::min(ceil_div(want, std::max(1, n * n_kv)), ceil_div(max_blocks, 4)), 64));
  const int bps = ceil_div(max_blocks, ns0);
  const int ns = ceil_div(max_blocks, bps);
  const size_t need = kDecCtrBytes + (size_t)n * n_kv * G * ns * (128 + 2) * sizeof(float);
  if (ns > 1 && need > ws_bytes) {
    set_last_error("decode attention: workspace too small for the co-resident kernel");
    return (int)cudaErrorInvalidValue;
  }
  const long long items = (long long)n * n_kv * ns;
  const int grid = (int)std::max<long long>(1, std::min<long long>(2LL * num_sms(), ceil_div(items, NW)));
  int* ctr = reinterpret_cast<int*>(ws);
  float* part = reinterpret_cast<float*>(ws + kDecCtrBytes);
  HY_CUDA_RET(cudaMemsetAsync(ws, 0, kDecCtrBytes, stream));  // see launch_bulk
  HY_CUDA_RET(launch_pdl(kern, dim3(grid), dim3(32 * NW), (size_t)SMEM, stream, q, ld_q, n, n_kv,
                         slots, ctx, bt, bt_stride, kv, block_stride, sl2, bps, ns, out, ld_o,
                         part, ctr));
  HY_LAUNCH_CHECK();
  if (ns > 1) {
    HY_CUDA_RET(launch_pdl(attn_decode_combine_kernel, dim3(n, n_kv * G), dim3(128), 0, stream,
                           (const float*)part, n_kv * G, ns, out, ld_o));
    HY_LAUNCH_CHECK();
  }
  return 0;
}

// co-resident kernel choice: HY_DECODE_CO=<nw>,<spw> (A/B), default 2 warps x 2 stages
static int co_dispatch(int G, const bf16* q, int ld_q, int n, int n_kv, const int* slots,
                       const int* ctx, int max_ctx, const int* bt, int bt_stride, const bf16* kv,
                       long long block_stride, float sl2, bf16* out, int ld_o, uint8_t* ws,
                       size_t ws_bytes, cudaStream_t stream) {
  BulkCfg env{2, 2};
  int pad = 1;
  if (const char* e = getenv("HY_DECODE_CO")) sscanf(e, "%d,%d,%d", &env.nw, &env.spw, &pad);
  if (!pad && G == 1 && env.nw == 4 && env.spw == 1)
    return launch_co<1, 4, 1, false>(q, ld_q, n, n_kv, slots, ctx, max_ctx, bt, bt_stride, kv,
                                     block_stride, sl2, out, ld_o, ws, ws_bytes, stream);
  if (!pad && G == 1 && env.nw == 2 && env.spw == 2)
    return launch_co<1, 2, 2, false>(q, ld_q, n, n_kv, slots, ctx, max_ctx, bt, bt_stride, kv,
                                     block_stride, sl2, out, ld_o, ws, ws_bytes, stream);
#define HY_CO(GG, NW, SPW)                                                                   \
  if (G == GG && env.nw == NW && env.spw == SPW)                                             \
    return launch_co<GG, NW, SPW>(q, ld_q, n, n_kv, slots, ctx, max_ctx, bt, bt_stride, kv,  \
                                  block_stride, sl2, out, ld_o, ws, ws_bytes, stream);
  HY_CO(1, 2, 2)
  HY_CO(1, 4, 1)
  HY_CO(1, 1, 4)
  HY_CO(7, 2, 2)
  HY_CO(7, 1, 4)
#undef HY_CO
  return -1;  // no co-resident instance: the caller uses the default kernel
}
}  // namespace hy

extern "C" int hy_set_decode_coresident(int on) {
  hy::decode_set_coresident(on ? 1 : 0);
  return 0;
}

extern "C" int hy_set_decode_kernel(int nw, int spw) {
  const bool ok = nw == 0 || (nw == 1 && spw == 4) || (nw == 2 && spw >= 2 && spw <= 4) ||
                  (nw == 4 && (spw == 1 || spw == 2 || spw == 6)) || (nw == 8 && spw == 3) ||
                  (nw == 1 && spw == 5) || (nw == 5 && spw == 1);
  if (!ok) {
    set_last_error("hy_set_decode_kernel: unsupported warps / stages");
    return (int)cudaErrorInvalidValue;
  }
  hy::t_dec_nw = nw;
  hy::t_dec_spw = spw;
  return 0;
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
  if (t_dec_coresident && t_dec_nw == 0 && !getenv("HY_DECODE_NOCO")) {
    uint8_t* wsb = reinterpret_cast<uint8_t*>(workspace);
    HY_CHECK_ARG(wsb != nullptr && workspace_bytes >= kDecCtrBytes, "decode workspace");
    const int rc = co_dispatch(G, reinterpret_cast<const bf16*>(q), ld_q, n, n_kv_heads, slots,
                               ctx, max_ctx, block_table, bt_stride,
                               reinterpret_cast<const bf16*>(kv_layer), block_stride,
                               scale * 1.4426950408889634f, reinterpret_cast<bf16*>(out), ld_o,
                               wsb, workspace_bytes, stream);
    if (rc >= 0) return rc;
  }
  if (G == 1) {
    const BulkCfg bc = bulk_cfg();
    if (bc.nw > 0) {
      uint8_t* wsb = reinterpret_cast<uint8_t*>(workspace);
      HY_CHECK_ARG(wsb != nullptr && workspace_bytes >= kDecCtrBytes, "decode workspace");
      const bf16* qp = reinterpret_cast<const bf16*>(q);
      const bf16* kvp = reinterpret_cast<const bf16*>(kv_layer);
      bf16* op = reinterpret_cast<bf16*>(out);
      const float sl2 = scale * 1.4426950408889634f;
#define HY_BULK(NW, SPW)                                                                    \
  if (bc.nw == NW && bc.spw == SPW)                                                         \
    return launch_bulk<NW, SPW>(qp, ld_q, n, n_heads, slots, ctx, max_ctx, block_table,     \
                                bt_stride, kvp, block_stride, sl2, op, ld_o, wsb,           \
                                workspace_bytes, stream);
      HY_BULK(1, 4)
      HY_BULK(2, 2)
      HY_BULK(2, 3)
      HY_BULK(2, 4)
      HY_BULK(4, 1)
      HY_BULK(4, 2)
      HY_BULK(4, 6)
      HY_BULK(8, 3)
      HY_BULK(1, 5)
      HY_BULK(5, 1)
#undef HY_BULK
      set_last_error("decode attention: no bulk kernel for this warp / stage count");
      return (int)cudaErrorInvalidValue;
    }
  }
  // split-KV partials follow the ticket counters (the bulk kernel's layout)
  workspace = workspace ? reinterpret_cast<uint8_t*>(workspace) + kDecCtrBytes : nullptr;
  workspace_bytes = workspace_bytes > kDecCtrBytes ? workspace_bytes - kDecCtrBytes : 0;
  int ns = decode_splits(n, n_kv_heads, max_ctx, G);
  const size_t need = (size_t)n * n_heads * ns * (head_dim + 2) * sizeof(float);
  if (ns > 1 && (workspace == nullptr || need > workspace_bytes)) ns = 1;
  const int max_blocks = std::max(1, ceil_div(max_ctx, HY_KV_BLOCK_TOKENS));
  const int bps = ceil_div(max_blocks, ns);
  ns = ceil_div(max_blocks, bps);
  // head-major grid: the KV heads of one sequence run on consecutive CTAs and read adjacent
  // 4 KiB tiles of each block (measured 2-3% more bandwidth than sequence-major, 6.82 -> 7.02
  // TB/s at 150 sequences x 600-750 shuffled blocks)
  dim3 grid(n_kv_heads, n, ns);
  const float sl2 = scale * 1.4426950408889634f;
  const bf16* qp = reinterpret_cast<const bf16*>(q);
  const bf16* kvp = reinterpret_cast<const bf16*>(kv_layer);
  bf16* op = reinterpret_cast<bf16*>(out);
  float* part = reinterpret_cast<float*>(workspace);
  static const bool carve_env = getenv("HY_DECODE_CARVEOUT") != nullptr;
  const bool co = carve_env || t_dec_coresident;
#define HY_DEC_CASE(GG)                                                                        \
  case GG:                                                                                     \
    if (co) {                                                                                  \
      HY_CUDA_RET(ensure_max_carveout(attn_decode_kernel<GG, 1>));                             \
      HY_CUDA_RET(launch_pdl(attn_decode_kernel<GG, 1>, dim3(grid), dim3(128), 0, stream, qp,  \
                             ld_q, n_kv_heads, slots, ctx, block_table, bt_stride, kvp,        \
                             block_stride, sl2, bps, op, ld_o, part, ns));                     \
    } else {                                                                                   \
      HY_CUDA_RET(launch_pdl(attn_decode_kernel<GG>, dim3(grid), dim3(128), 0, stream, qp,     \
                             ld_q, n_kv_heads, slots, ctx, block_table, bt_stride, kvp,        \
                             block_stride, sl2, bps, op, ld_o, part, ns));                     \
    }                                                                                          \
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
