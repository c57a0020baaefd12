// K7 paged prefill attention (causal with a chunk offset) and K3 ViT varlen attention
// (block-diagonal, non-causal), one flash-attention kernel templated on the KV source.
//
// This file: the FA2-style kernel on the warp-level tensor-core path (mma.sync m16n8k16
// bf16 -> fp32, cp.async double-buffered K/V) for head sizes the tcgen05 kernel does not
// take (Qwen2-VL vision d = 80), and the C-ABI entry points, which dispatch d = 64 / 128 to
// the tcgen05 + TMEM kernel in attn_tc.cu.
//
// Work per CTA: 64 query rows of one (sequence, head); 4 warps x 16 rows.  K/V tiles of
// 64 keys; paged tiles are 4 consecutive 16-token blocks read through the block table.
// Reference: epdsim charges prefill attention as 4*S^2*H over the chunk only
// (model_cost.py:189); this kernel attends to the full cached prefix [0, offset + i].
#include "common.cuh"
#include "../../include/hydra_sm100.h"
#include "mma_sync.cuh"

namespace hy {

struct FaParams {
  const bf16* q;
  int ld_q;
  // contiguous K/V (varlen ViT): K row j of segment s at k + (qstart[s] + j) * ld_kv
  const bf16* k;
  const bf16* v;
  int ld_kv;
  // paged K/V
  const bf16* kv;
  long long block_stride;
  const int* block_table;
  int bt_stride;
  int n_kv;
  const int* qstart;
  const int* offset;  // paged: tokens cached before the chunk
  const int* slots;
  int group;          // n_heads / n_kv
  int q_tiles;        // q tiles per sequence in the grid
  float scale_log2;
  bf16* out;
  int ld_o;
};

template <int D, bool PAGED>
__global__ void __launch_bounds__(128) attn_fa2_kernel(const FaParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int BQ = 64, BKV = 64, LDS = D + 8;  // padded smem rows: conflict-free ldmatrix
  constexpr int CPR = D / 8;                     // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t fa_smem[];
  bf16* sQ = reinterpret_cast<bf16*>(fa_smem);
  bf16* sK = sQ + BQ * LDS;
  bf16* sV = sK + 2 * BKV * LDS;

  const int seq = blockIdx.x / p.q_tiles;
  const int qt = blockIdx.x % p.q_tiles;
  const int h = blockIdx.y;
  const int kvh = h / p.group;
  const int q0 = p.qstart[seq];
  const int nq = p.qstart[seq + 1] - q0;
  if (qt * BQ >= nq) return;
  const int off = PAGED ? p.offset[seq] : 0;
  const int kv_len = PAGED ? off + nq : nq;
  const int kv_end = PAGED ? min(kv_len, off + qt * BQ + BQ) : kv_len;
  const int n_kt = (kv_end + BKV - 1) / BKV;
  const int* bt = PAGED ? p.block_table + (size_t)p.slots[seq] * p.bt_stride : nullptr;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- async loads ----
  for (int c = tid; c < BQ * CPR; c += 128) {
    int r = c / CPR, col = (c % CPR) * 8;
    int qi = qt * BQ + r;
    bool ok = qi < nq;
    const bf16* src = p.q + (size_t)(q0 + (ok ? qi : 0)) * p.ld_q + (size_t)h * D + col;
    cp_async16(sQ + r * LDS + col, src, ok);
  }
  auto load_kv = [&](int kt, int buf) {
    bf16* dK = sK + buf * BKV * LDS;
    bf16* dV = sV + buf * BKV * LDS;
    for (int c = tid; c < BKV * CPR; c += 128) {
      int r = c / CPR, col = (c % CPR) * 8;
      int key = kt * BKV + r;
      bool ok = key < kv_len;
      int kk = ok ? key : 0;
      const bf16 *ks, *vs;
      if (PAGED) {
        const bf16* blk = p.kv + (size_t)bt[kk / HY_KV_BLOCK_TOKENS] * p.block_stride;
        ks = blk + ((size_t)kvh * HY_KV_BLOCK_TOKENS + kk % HY_KV_BLOCK_TOKENS) * D + col;
        vs = ks + (size_t)p.n_kv * HY_KV_BLOCK_TOKENS * D;
      } else {
        ks = p.k + (size_t)(q0 + kk) * p.ld_kv + (size_t)kvh * D + col;
        vs = p.v + (size_t)(q0 + kk) * p.ld_kv + (size_t)kvh * D + col;
      }
      cp_async16(dK + r * LDS + col, ks, ok);
      cp_async16(dV + r * LDS + col, vs, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[D / 16][4];
  const int r_lo = lane >> 2;  // rows r_lo and r_lo + 8 of this warp's 16
  const int qpos0 = off + qt * BQ + warp * 16 + r_lo;
  const int qpos1 = qpos0 + 8;

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) load_kv(kt + 1, (kt + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        int row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int col = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(smem_u32(sQ + row * LDS + col), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const bf16* cK = sK + (kt & 1) * BKV * LDS;
    const bf16* cV = sV + (kt & 1) * BKV * LDS;
    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 4; ++np) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        int key = np * 16 + (lane & 7) + (lane >> 4) * 8;
        int col = kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(cK + key * LDS + col), b0, b1, b2, b3);
        mma_bf16_16816(s[2 * np], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
        mma_bf16_16816(s[2 * np + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
      }
    }
    // mask + online softmax (exp2 domain)
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int key = kt * BKV + nt * 8 + (lane & 3) * 2 + e;
        bool ok0 = key < kv_len && (!PAGED || key <= qpos0);
        bool ok1 = key < kv_len && (!PAGED || key <= qpos1);
        s[nt][e] = ok0 ? s[nt][e] * p.scale_log2 : -INFINITY;
        s[nt][2 + e] = ok1 ? s[nt][2 + e] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][e]);
        mx1 = fmaxf(mx1, s[nt][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float ms0 = mn0 == -INFINITY ? 0.f : mn0, ms1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = exp2f(m0 - ms0), c1 = exp2f(m1 - ms1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - ms0);
      s[nt][1] = exp2f(s[nt][1] - ms0);
      s[nt][2] = exp2f(s[nt][2] - ms1);
      s[nt][3] = exp2f(s[nt][3] - ms1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= c0;
      o[i][1] *= c0;
      o[i][2] *= c1;
      o[i][3] *= c1;
    }
    // O += P V
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t a0 = pack_bf16x2(s[2 * j][0], s[2 * j][1]);
      uint32_t a1 = pack_bf16x2(s[2 * j][2], s[2 * j][3]);
      uint32_t a2 = pack_bf16x2(s[2 * j + 1][0], s[2 * j + 1][1]);
      uint32_t a3 = pack_bf16x2(s[2 * j + 1][2], s[2 * j + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        int key = j * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int col = dp * 16 + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(cV + key * LDS + col), b0, b1, b2, b3);
        mma_bf16_16816(o[2 * dp], a0, a1, a2, a3, b0, b1);
        mma_bf16_16816(o[2 * dp + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int qi0 = qt * BQ + warp * 16 + r_lo, qi1 = qi0 + 8;
#pragma unroll
  for (int nt = 0; nt < D / 8; ++nt) {
    int col = h * D + nt * 8 + (lane & 3) * 2;
    if (qi0 < nq)
      *reinterpret_cast<uint32_t*>(p.out + (size_t)(q0 + qi0) * p.ld_o + col) =
          pack_bf16x2(o[nt][0] * inv0, o[nt][1] * inv0);
    if (qi1 < nq)
      *reinterpret_cast<uint32_t*>(p.out + (size_t)(q0 + qi1) * p.ld_o + col) =
          pack_bf16x2(o[nt][2] * inv1, o[nt][3] * inv1);
  }
}

template <int D, bool PAGED>
static int launch_fa(const FaParams& p, int n_seqs, int n_heads, cudaStream_t st) {
  constexpr int LDS = D + 8;
  constexpr int smem = (64 + 4 * 64) * LDS * 2;
  HY_CUDA_RET(ensure_smem(attn_fa2_kernel<D, PAGED>, smem));
  dim3 grid(n_seqs * p.q_tiles, n_heads);
  HY_CUDA_RET(launch_pdl(attn_fa2_kernel<D, PAGED>, dim3(grid), dim3(128), smem, st, p));
  HY_LAUNCH_CHECK();
  return 0;
}

int attn_tc_prefill(const void* q, int ld_q, int n_rows, int n_seqs, const int* qstart,
                    const int* offset, const int* slots, int max_q, int n_heads, int n_kv_heads,
                    int head_dim, const int* block_table, int bt_stride, const void* kv_layer,
                    long long block_stride, float scale, void* out, int ld_o, cudaStream_t st);
int attn_tc_varlen(const void* qkv, int ld_qkv, int n_rows, int n_segs, const int* seg,
                   int max_len, int n_heads, int head_dim, float scale, void* out, int ld_o,
                   cudaStream_t st);

// tcgen05 kernel for head_dim 64/128 (and 80 for the varlen ViT path) unless HY_ATTN_FA2 is
// set (A/B measurement only)
static bool use_tc(int head_dim, bool varlen = false) {
  static const bool fa2 = getenv("HY_ATTN_FA2") != nullptr;
  return !fa2 && (head_dim == 64 || head_dim == 128 || (varlen && head_dim == 80));
}

}  // namespace hy

using namespace hy;

extern "C" int hy_attn_prefill_paged(const void* q, int ld_q, int n_rows, int n_seqs,
                                     const int* qstart, const int* offset, const int* slots,
                                     int max_q, int n_heads, int n_kv_heads, int head_dim,
                                     const int* block_table, int bt_stride, const void* kv_layer,
                                     long long block_stride, float scale, void* out, int ld_o,
                                     cudaStream_t stream) {
  HY_CHECK_ARG(n_kv_heads > 0 && n_heads % n_kv_heads == 0, "heads");
  if (n_seqs <= 0 || max_q <= 0 || n_rows <= 0) return 0;
  if (use_tc(head_dim))
    return attn_tc_prefill(q, ld_q, n_rows, n_seqs, qstart, offset, slots, max_q, n_heads,
                           n_kv_heads, head_dim, block_table, bt_stride, kv_layer, block_stride,
                           scale, out, ld_o, stream);
  FaParams p{};
  p.q = reinterpret_cast<const bf16*>(q);
  p.ld_q = ld_q;
  p.kv = reinterpret_cast<const bf16*>(kv_layer);
  p.block_stride = block_stride;
  p.block_table = block_table;
  p.bt_stride = bt_stride;
  p.n_kv = n_kv_heads;
  p.qstart = qstart;
  p.offset = offset;
  p.slots = slots;
  p.group = n_heads / n_kv_heads;
  p.q_tiles = ceil_div(max_q, 64);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = reinterpret_cast<bf16*>(out);
  p.ld_o = ld_o;
  switch (head_dim) {
    case 128: return launch_fa<128, true>(p, n_seqs, n_heads, stream);
    case 64: return launch_fa<64, true>(p, n_seqs, n_heads, stream);
    default:
      set_last_error("prefill attention: unsupported head_dim " + std::to_string(head_dim));
      return (int)cudaErrorInvalidValue;
  }
}

extern "C" int hy_attn_varlen(const void* qkv, int ld_qkv, int n_rows, int n_segs, const int* seg,
                              int max_len, int n_heads, int head_dim, float scale, void* out,
                              int ld_o, cudaStream_t stream) {
  if (n_segs <= 0 || max_len <= 0 || n_rows <= 0) return 0;
  if (use_tc(head_dim, true))
    return attn_tc_varlen(qkv, ld_qkv, n_rows, n_segs, seg, max_len, n_heads, head_dim, scale,
                          out, ld_o, stream);
  FaParams p{};
  const bf16* base = reinterpret_cast<const bf16*>(qkv);
  p.q = base;
  p.ld_q = ld_qkv;
  p.k = base + (size_t)n_heads * head_dim;
  p.v = base + (size_t)2 * n_heads * head_dim;
  p.ld_kv = ld_qkv;
  p.n_kv = n_heads;
  p.qstart = seg;
  p.group = 1;
  p.q_tiles = ceil_div(max_len, 64);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = reinterpret_cast<bf16*>(out);
  p.ld_o = ld_o;
  switch (head_dim) {
    case 64: return launch_fa<64, false>(p, n_segs, n_heads, stream);
    case 80: return launch_fa<80, false>(p, n_segs, n_heads, stream);
    case 128: return launch_fa<128, false>(p, n_segs, n_heads, stream);
    default:
      set_last_error("varlen attention: unsupported head_dim " + std::to_string(head_dim));
      return (int)cudaErrorInvalidValue;
  }
}
