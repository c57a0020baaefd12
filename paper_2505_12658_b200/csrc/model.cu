// Native layer loops for the two towers.  One C-ABI call runs a whole batch so the
// per-kernel launch cost is paid in C++, not through ctypes:
//
//   hy_lang_forward : a mixed decode + chunked-prefill batch of the Llama-style decoder
//                     (what epdsim's language_work prices, model_cost.py:171-197)
//   hy_vit_forward  : an encode batch of the ViT + projector, writing projected visual
//                     tokens straight into the request's image-cache blocks
//                     (what vision_work prices, model_cost.py:151-168)
#include "common.cuh"
#include "../../include/hydra_sm100.h"

#include <algorithm>
#include <cmath>

namespace hy {
int gemm_bf16(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K,
              const HyGemmEpilogue* e, void* ws, size_t ws_bytes, cudaStream_t st, int force_mode);
int rmsnorm(const void* x, int ldx, const void* w, void* out, int ldo, int rows, int cols,
            float eps, const int* row_idx, cudaStream_t st);
int layernorm(const void* x, int ldx, const void* w, const void* b, void* out, int ldo, int rows,
              int cols, float eps, const int* row_idx, cudaStream_t st);
int vit_assemble(const HyImageDesc* images, int n_images, int n_tokens, int hidden, int cls,
                 const void* patch_rows, const void* cls_emb, const void* pos_emb, int max_pos,
                 const void* ln_w, const void* ln_b, float eps, void* out, cudaStream_t st);
int vit_gather_visual(const HyImageDesc* images, int n_images, int n_visual, int hidden, int cls,
                      const void* h, void* out, cudaStream_t st);

static constexpr size_t kGemmWs = 64ull << 20;  // split-K partials

// Opt-in (HY_ATTN_FORK=1): measured on B200 (tools/mixed_batch.py, 64-256 decodes at ctx
// 300-700 + 512-2816-token prefill chunks) the overlap is within +-2% of the serial order --
// decode attention already fills every SM, so the prefill CTAs only fill its tail.
static bool attn_fork_enabled() {
  const char* e = getenv("HY_ATTN_FORK");
  return e && e[0] == '1';
}

struct Carve {
  uint8_t* base;
  size_t off = 0;
  explicit Carve(void* b) : base(reinterpret_cast<uint8_t*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct LangWs {
  bf16 *x, *t, *qkv, *attn, *f, *tout;
  float* logits;
  void* gemm_ws;
  void* dec_ws;
  size_t dec_ws_bytes;
};

static size_t lang_carve(const HyLangModel* m, int max_rows, int max_out, int max_decode,
                         int max_ctx, void* base, LangWs* w) {
  Carve c(base);
  const int qkv_cols = (m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  LangWs l{};
  // the GEMM workspace holds stream-K arrival counters that must stay zero between
  // calls: it lives at a fixed offset (the start), independent of the batch shape
  l.gemm_ws = c.take<uint8_t>(kGemmWs);
  l.x = c.take<bf16>((size_t)max_rows * m->hidden);
  l.t = c.take<bf16>((size_t)max_rows * m->hidden);
  l.qkv = c.take<bf16>((size_t)max_rows * qkv_cols);
  l.attn = c.take<bf16>((size_t)max_rows * m->n_heads * m->head_dim);
  l.f = c.take<bf16>((size_t)max_rows * m->ffn);
  l.tout = c.take<bf16>((size_t)std::max(max_out, 1) * m->hidden);
  l.logits = c.take<float>((size_t)std::max(max_out, 1) * m->vocab);
  l.dec_ws_bytes =
      hy_attn_decode_workspace_bytes(std::max(max_decode, 1), m->n_heads, m->head_dim, max_ctx);
  l.dec_ws = c.take<uint8_t>(l.dec_ws_bytes);
  if (w) *w = l;
  return c.off + 256;
}

}  // namespace hy

using namespace hy;

extern "C" size_t hy_lang_workspace_bytes(const HyLangModel* m, int max_rows, int max_out,
                                          int max_decode, int max_ctx) {
  return lang_carve(m, max_rows, max_out, max_decode, max_ctx, nullptr, nullptr);
}

extern "C" int hy_lang_forward(const HyLangModel* m, const HyLangBatch* b, const HyKvCache* kv,
                               const void* image_rows, int* last_tok, void* workspace,
                               size_t workspace_bytes, cudaStream_t st) {
  HY_CHECK_ARG(m && b && kv && workspace, "null argument");
  if (b->n_rows <= 0) return 0;
  HY_CHECK_ARG(m->n_heads * m->head_dim == m->hidden || m->n_heads * m->head_dim > 0, "heads");
  const int H = m->hidden, D = m->head_dim;
  const int QD = m->n_heads * D;
  const int qkv_cols = (m->n_heads + 2 * m->n_kv_heads) * D;
  const int R = b->n_rows;
  LangWs w{};
  size_t need = lang_carve(m, R, b->n_out, b->n_decode, b->max_ctx, workspace, &w);
  if (need > workspace_bytes) {
    set_last_error("hy_lang_forward: workspace too small (" + std::to_string(need) + " > " +
                   std::to_string(workspace_bytes) + ")");
    return (int)cudaErrorInvalidValue;
  }
  auto G = [&](const bf16* A, int lda, const void* W, int M, int N, int K, const void* bias,
               const void* res, int ldr, int act, void* out, int ldc, int f32) {
    HyGemmEpilogue e{};
    e.bias = bias;
    e.residual = res;
    e.ldr = ldr;
    e.act = act;
    e.out = out;
    e.ldc = ldc;
    e.out_f32 = f32;
    timer_mark(HY_KCLASS_GEMM, st, true, 0.0);
    int rc = gemm_bf16(A, lda, reinterpret_cast<const bf16*>(W), K, M, N, K, &e, w.gemm_ws,
                       kGemmWs, st, 0);
    timer_mark(HY_KCLASS_GEMM, st, false, 2.0 * M * N * K,
               ((long long)M << 42) | ((long long)N << 21) | (long long)K);
    return rc;
  };
  const float scale = 1.0f / sqrtf((float)D);
  HY_RET_IF(hy_merge_embed(b->tok, R, m->embed, image_rows, H, last_tok, b->row_slot, w.x, st));
  const int nd = b->n_decode;
  const int np_rows = R - nd;
  for (int li = 0; li < m->n_layers; ++li) {
    const HyLangLayerW& L = m->layers[li];
    bf16* kv_layer = reinterpret_cast<bf16*>(kv->base) + (size_t)li * kv->layer_stride;
    HY_RET_IF(rmsnorm(w.x, H, L.attn_norm, w.t, H, R, H, m->rms_eps, nullptr, st));
    HY_RET_IF(G(w.t, H, L.w_qkv, R, qkv_cols, H, L.b_qkv, nullptr, 0, HY_ACT_NONE, w.qkv,
                qkv_cols, 0));
    HY_RET_IF(hy_rope_kv_append(w.qkv, qkv_cols, R, m->n_heads, m->n_kv_heads, D, b->pos,
                                b->row_slot, kv->block_table, kv->bt_stride, kv_layer,
                                kv->block_stride, m->rope_theta, st));
    // decode attention (HBM-bound) and prefill attention (tensor-bound) read disjoint rows
    // of qkv and write disjoint rows of attn: the prefill part runs on a side stream so the
    // two can overlap
    const bool fork = nd > 0 && b->n_prefill > 0 && np_rows > 0 && attn_fork_enabled();
    cudaStream_t pst = st;
    cudaEvent_t join = nullptr;
    if (fork) HY_RET_IF(side_fork(st, &pst, &join));
    if (nd > 0) {
      timer_mark(HY_KCLASS_DECODE_ATTN, st, true, 0.0);
      HY_RET_IF(hy_attn_decode_paged(w.qkv, qkv_cols, nd, m->n_heads, m->n_kv_heads, D,
                                     b->row_slot, b->dec_ctx, b->max_ctx, kv->block_table,
                                     kv->bt_stride, kv_layer, kv->block_stride, scale, w.attn, QD,
                                     w.dec_ws, w.dec_ws_bytes, st));
      timer_mark(HY_KCLASS_DECODE_ATTN, st, false, 0.0);
    }
    if (b->n_prefill > 0 && np_rows > 0) {
      timer_mark(HY_KCLASS_PREFILL_ATTN, pst, true, 0.0);
      HY_RET_IF(hy_attn_prefill_paged(w.qkv + (size_t)nd * qkv_cols, qkv_cols, np_rows, b->n_prefill,
                                      b->pf_qstart, b->pf_offset, b->pf_slot, b->pf_max_q,
                                      m->n_heads, m->n_kv_heads, D, kv->block_table,
                                      kv->bt_stride, kv_layer, kv->block_stride, scale,
                                      w.attn + (size_t)nd * QD, QD, pst));
      timer_mark(HY_KCLASS_PREFILL_ATTN, pst, false, 0.0);
    }
    if (fork) HY_RET_IF(side_join(st, pst, join));
    HY_RET_IF(G(w.attn, QD, L.w_o, R, H, QD, nullptr, w.x, H, HY_ACT_NONE, w.x, H, 0));
    HY_RET_IF(rmsnorm(w.x, H, L.ffn_norm, w.t, H, R, H, m->rms_eps, nullptr, st));
    HY_RET_IF(G(w.t, H, L.w_gate_up, R, 2 * m->ffn, H, nullptr, nullptr, 0, HY_ACT_SWIGLU, w.f,
                m->ffn, 0));
    HY_RET_IF(G(w.f, m->ffn, L.w_down, R, H, m->ffn, nullptr, w.x, H, HY_ACT_NONE, w.x, H, 0));
  }
  if (b->n_out > 0) {
    HY_RET_IF(rmsnorm(w.x, H, m->final_norm, w.tout, H, b->n_out, H, m->rms_eps, b->out_rows, st));
    float* logits = b->out_logits ? b->out_logits : w.logits;
    HY_RET_IF(G(w.tout, H, m->lm_head, b->n_out, m->vocab, H, nullptr, nullptr, 0, HY_ACT_NONE,
                logits, m->vocab, 1));
    HY_RET_IF(hy_argmax_f32(logits, b->n_out, m->vocab, m->vocab, b->out_tokens, b->out_slot,
                            last_tok, st));
  }
  return 0;
}

// ---------------------------------------------------------------------------
// ViT + projector
// ---------------------------------------------------------------------------
namespace hy {
struct VitWs {
  bf16 *patches, *pe, *h, *t, *qkv, *a, *f, *v, *p;
  void* gemm_ws;
};
static size_t vit_carve(const HyVitModel* m, int max_tokens, void* base, VitWs* w) {
  Carve c(base);
  VitWs v{};
  v.gemm_ws = c.take<uint8_t>(kGemmWs);  // fixed offset: see lang_carve
  const int Hv = m->hidden;
  v.patches = c.take<bf16>((size_t)max_tokens * m->k_pad);
  v.pe = c.take<bf16>((size_t)max_tokens * Hv);
  v.h = c.take<bf16>((size_t)max_tokens * Hv);
  v.t = c.take<bf16>((size_t)max_tokens * Hv);
  v.qkv = c.take<bf16>((size_t)max_tokens * 3 * Hv);
  v.a = c.take<bf16>((size_t)max_tokens * Hv);
  v.f = c.take<bf16>((size_t)max_tokens * std::max(m->mlp, m->proj_hidden));
  v.v = c.take<bf16>((size_t)max_tokens * Hv);
  v.p = c.take<bf16>((size_t)max_tokens * m->proj_hidden);
  if (w) *w = v;
  return c.off + 256;
}
}  // namespace hy

extern "C" size_t hy_vit_workspace_bytes(const HyVitModel* m, int max_tokens, int max_image_tokens) {
  (void)max_image_tokens;
  return vit_carve(m, max_tokens, nullptr, nullptr);
}

extern "C" int hy_vit_forward(const HyVitModel* m, const HyVitBatch* b, void* workspace,
                              size_t workspace_bytes, cudaStream_t st) {
  HY_CHECK_ARG(m && b && workspace, "null argument");
  if (b->n_images <= 0) return 0;
  HY_CHECK_ARG(m->merge == 1 || m->merge == 2, "merge");
  const int Hv = m->hidden, T = b->n_tokens;
  VitWs w{};
  size_t need = vit_carve(m, T, workspace, &w);
  if (need > workspace_bytes) {
    set_last_error("hy_vit_forward: workspace too small (" + std::to_string(need) + " > " +
                   std::to_string(workspace_bytes) + ")");
    return (int)cudaErrorInvalidValue;
  }
  auto G = [&](const bf16* A, int lda, const void* W, int M, int N, int K, const void* bias,
               const void* res, int ldr, int act, void* out, int ldc, const int* row_map) {
    HyGemmEpilogue e{};
    e.bias = bias;
    e.residual = res;
    e.ldr = ldr;
    e.act = act;
    e.row_map = row_map;
    e.out = out;
    e.ldc = ldc;
    timer_mark(HY_KCLASS_GEMM, st, true, 0.0);
    int rc = gemm_bf16(A, lda, reinterpret_cast<const bf16*>(W), K, M, N, K, &e, w.gemm_ws,
                       kGemmWs, st, 0);
    timer_mark(HY_KCLASS_GEMM, st, false, 2.0 * M * N * K,
               ((long long)M << 42) | ((long long)N << 21) | (long long)K);
    return rc;
  };
  // K2: patch embedding
  HY_RET_IF(hy_im2col_patches(b->images, b->n_images, b->n_patches, m->patch, m->merge, m->k_pad,
                              w.patches, st));
  HY_RET_IF(G(w.patches, m->k_pad, m->w_patch, b->n_patches, Hv, m->k_pad, nullptr, nullptr, 0,
              HY_ACT_NONE, w.pe, Hv, nullptr));
  HY_RET_IF(vit_assemble(b->images, b->n_images, T, Hv, m->cls, w.pe, m->cls_emb, m->pos_emb,
                         m->max_pos, m->pre_ln ? m->pre_ln_w : nullptr,
                         m->pre_ln ? m->pre_ln_b : nullptr, m->ln_eps, w.h, st));
  const float scale = 1.0f / sqrtf((float)m->head_dim);
  for (int li = 0; li < m->n_layers; ++li) {
    const HyVitLayerW& L = m->layers[li];
    HY_RET_IF(layernorm(w.h, Hv, L.ln1_w, L.ln1_b, w.t, Hv, T, Hv, m->ln_eps, nullptr, st));
    HY_RET_IF(G(w.t, Hv, L.w_qkv, T, 3 * Hv, Hv, L.b_qkv, nullptr, 0, HY_ACT_NONE, w.qkv, 3 * Hv,
                nullptr));
    timer_mark(HY_KCLASS_VIT_ATTN, st, true, 0.0);
    HY_RET_IF(hy_attn_varlen(w.qkv, 3 * Hv, T, b->n_images, b->seg, b->max_image_tokens, m->n_heads,
                             m->head_dim, scale, w.a, Hv, st));
    timer_mark(HY_KCLASS_VIT_ATTN, st, false, 0.0);
    HY_RET_IF(G(w.a, Hv, L.w_o, T, Hv, Hv, L.b_o, w.h, Hv, HY_ACT_NONE, w.h, Hv, nullptr));
    HY_RET_IF(layernorm(w.h, Hv, L.ln2_w, L.ln2_b, w.t, Hv, T, Hv, m->ln_eps, nullptr, st));
    HY_RET_IF(G(w.t, Hv, L.w_fc1, T, m->mlp, Hv, L.b_fc1, nullptr, 0, HY_ACT_QUICK_GELU, w.f,
                m->mlp, nullptr));
    HY_RET_IF(G(w.f, m->mlp, L.w_fc2, T, Hv, m->mlp, L.b_fc2, w.h, Hv, HY_ACT_NONE, w.h, Hv,
                nullptr));
  }
  // projector -> image-cache rows
  const int NV = b->n_visual;
  const bf16* proj_in;
  int k_in;
  if (m->merge == 1) {
    HY_RET_IF(vit_gather_visual(b->images, b->n_images, NV, Hv, m->cls, w.h, w.v, st));
    proj_in = w.v;
    k_in = Hv;
  } else {
    HY_RET_IF(layernorm(w.h, Hv, m->merge_ln_w, m->merge_ln_b, w.t, Hv, T, Hv, m->ln_eps, nullptr,
                        st));
    proj_in = w.t;  // [T, Hv] viewed as [T/4, 4 Hv]: 2x2 windows are contiguous
    k_in = 4 * Hv;
  }
  HY_RET_IF(G(proj_in, k_in, m->w_proj1, NV, m->proj_hidden, k_in, m->b_proj1, nullptr, 0,
              HY_ACT_GELU, w.p, m->proj_hidden, nullptr));
  HY_RET_IF(G(w.p, m->proj_hidden, m->w_proj2, NV, m->lang_hidden, m->proj_hidden, m->b_proj2,
              nullptr, 0, HY_ACT_NONE, b->image_rows, m->lang_hidden, b->out_row_map));
  return 0;
}
