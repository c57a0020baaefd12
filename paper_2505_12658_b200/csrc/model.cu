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
void gemm_set_sms_cap(int sms);
void decode_set_coresident(int on);
void gemm_set_coresident(int on);
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

// Split mode (two row groups on two streams, see hy_lang_forward): HY_LANG_SPLIT=<n> turns
// it on for batches with >= n decode rows (0 / unset: off); HY_SPLIT_SMS SMs (default 24)
// are kept free of GEMM CTAs for the other group's attention.
static int split_min_decodes() {
  const char* e = getenv("HY_LANG_SPLIT");
  return e ? atoi(e) : 0;
}
static int split_reserve_sms() {
  const char* e = getenv("HY_SPLIT_SMS");
  return e ? atoi(e) : 24;
}
// Decode / prefill split (HY_LANG_SPLIT_PD=<n>: batches with >= n decode rows and prefill
// rows): the decode rows and the prefill rows run their whole layer stacks as two independent
// row groups on two streams -- they share only the weights -- so one group's HBM-bound
// decode attention can run while the other group's tensor-bound GEMMs do.
static int split_pd_min_decodes() {
  const char* e = getenv("HY_LANG_SPLIT_PD");
  return e ? atoi(e) : 0;
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
  void* gemm_ws2;
  void* dec_ws;
  void* dec_ws2;
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
  l.gemm_ws2 = c.take<uint8_t>(kGemmWs);  // second row group's GEMMs (split mode)
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
  l.dec_ws2 = c.take<uint8_t>(l.dec_ws_bytes);
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
               const void* res, int ldr, int act, void* out, int ldc, int f32, cudaStream_t s,
               void* gws) {
    HyGemmEpilogue e{};
    e.bias = bias;
    e.residual = res;
    e.ldr = ldr;
    e.act = act;
    e.out = out;
    e.ldc = ldc;
    e.out_f32 = f32;
    timer_mark(HY_KCLASS_GEMM, s, true, 0.0);
    int rc = gemm_bf16(A, lda, reinterpret_cast<const bf16*>(W), K, M, N, K, &e, gws, kGemmWs, s, 0);
    timer_mark(HY_KCLASS_GEMM, s, false, 2.0 * M * N * K,
               ((long long)M << 42) | ((long long)N << 21) | (long long)K);
    return rc;
  };
  const float scale = 1.0f / sqrtf((float)D);
  HY_RET_IF(hy_merge_embed(b->tok, R, m->embed, image_rows, H, last_tok, b->row_slot, w.x, st));
  const int nd = b->n_decode;
  const int np_rows = R - nd;

  // One layer over the rows [r0, r1): the first n_dec of them decode rows, the prefill rows
  // (all of [nd, R)) included when r1 == R.  Every kernel addresses its rows by offset, so
  // two disjoint row ranges can run on two streams at once.
  // part 0: norm, QKV projection, RoPE + KV append; part 1: attention, O projection, MLP
  auto layer = [&](int li, int part, int r0, int r1, int n_dec, cudaStream_t s, void* gws,
                   void* dws) -> int {
    const HyLangLayerW& L = m->layers[li];
    bf16* kv_layer = reinterpret_cast<bf16*>(kv->base) + (size_t)li * kv->layer_stride;
    const int rows = r1 - r0;
    bf16* x = w.x + (size_t)r0 * H;
    bf16* t = w.t + (size_t)r0 * H;
    bf16* qkv = w.qkv + (size_t)r0 * qkv_cols;
    bf16* attn = w.attn + (size_t)r0 * QD;
    bf16* f = w.f + (size_t)r0 * m->ffn;
    if (part == 0) {
      HY_RET_IF(rmsnorm(x, H, L.attn_norm, t, H, rows, H, m->rms_eps, nullptr, s));
      HY_RET_IF(G(t, H, L.w_qkv, rows, qkv_cols, H, L.b_qkv, nullptr, 0, HY_ACT_NONE, qkv,
                  qkv_cols, 0, s, gws));
      HY_RET_IF(hy_rope_kv_append(qkv, qkv_cols, rows, m->n_heads, m->n_kv_heads, D,
                                  b->pos + r0, b->row_slot + r0, kv->block_table, kv->bt_stride,
                                  kv_layer, kv->block_stride, m->rope_theta, s));
      return 0;
    }
    if (n_dec > 0) {
      timer_mark(HY_KCLASS_DECODE_ATTN, s, true, 0.0);
      HY_RET_IF(hy_attn_decode_paged(qkv, qkv_cols, n_dec, m->n_heads, m->n_kv_heads, D,
                                     b->row_slot + r0, b->dec_ctx + r0, b->max_ctx,
                                     kv->block_table, kv->bt_stride, kv_layer, kv->block_stride,
                                     scale, attn, QD, dws, w.dec_ws_bytes, s));
      timer_mark(HY_KCLASS_DECODE_ATTN, s, false, 0.0);
    }
    if (r1 == R && b->n_prefill > 0 && np_rows > 0) {
      timer_mark(HY_KCLASS_PREFILL_ATTN, s, true, 0.0);
      HY_RET_IF(hy_attn_prefill_paged(w.qkv + (size_t)nd * qkv_cols, qkv_cols, np_rows,
                                      b->n_prefill, b->pf_qstart, b->pf_offset, b->pf_slot,
                                      b->pf_max_q, m->n_heads, m->n_kv_heads, D, kv->block_table,
                                      kv->bt_stride, kv_layer, kv->block_stride, scale,
                                      w.attn + (size_t)nd * QD, QD, s));
      timer_mark(HY_KCLASS_PREFILL_ATTN, s, false, 0.0);
    }
    HY_RET_IF(G(attn, QD, L.w_o, rows, H, QD, nullptr, x, H, HY_ACT_NONE, x, H, 0, s, gws));
    HY_RET_IF(rmsnorm(x, H, L.ffn_norm, t, H, rows, H, m->rms_eps, nullptr, s));
    HY_RET_IF(G(t, H, L.w_gate_up, rows, 2 * m->ffn, H, nullptr, nullptr, 0, HY_ACT_SWIGLU, f,
                m->ffn, 0, s, gws));
    HY_RET_IF(G(f, m->ffn, L.w_down, rows, H, m->ffn, nullptr, x, H, HY_ACT_NONE, x, H, 0, s, gws));
    return 0;
  };

  const int split_min = split_min_decodes();
  const int split_pd = split_pd_min_decodes();
  if (split_pd > 0 && nd >= split_pd && np_rows > 0) {
    cudaStream_t side = nullptr;
    cudaEvent_t join = nullptr;
    HY_RET_IF(side_fork(st, &side, &join));
    int rc = 0;
    // HY_SPLIT_CO=1: decode attention as the co-resident kernel (K8c, one CTA per SM beside
    // the prefill group's SLIM GEMMs).  Opt-in: measured, it pulls too few bytes per SM to
    // pay (tools/lab/coresident.sh)
    const char* ce = getenv("HY_SPLIT_CO");  // bits: 1 decode K8c, 2 SLIM GEMMs
    const int co = ce ? atoi(ce) : 0;
    decode_set_coresident(co & 1);
    gemm_set_coresident((co >> 1) & 1);
    for (int li = 0; li < m->n_layers && rc == 0; ++li) {
      rc = layer(li, 0, 0, nd, nd, side, w.gemm_ws2, w.dec_ws);      // decode rows
      if (rc == 0) rc = layer(li, 1, 0, nd, nd, side, w.gemm_ws2, w.dec_ws);
      if (rc == 0) rc = layer(li, 0, nd, R, 0, st, w.gemm_ws, w.dec_ws2);  // prefill rows
      if (rc == 0) rc = layer(li, 1, nd, R, 0, st, w.gemm_ws, w.dec_ws2);
    }
    decode_set_coresident(0);
    gemm_set_coresident(0);
    HY_RET_IF(rc);
    HY_RET_IF(side_join(st, side, join));
  } else if (split_min > 0 && nd >= split_min) {
    // Two row groups on two streams (first half of the decode rows | the rest + prefill):
    // while one group's decode attention streams KV from HBM, the other group's GEMMs keep
    // the tensor cores busy.  GEMM grids leave split_reserve_sms() SMs to the attention.
    const int na = nd / 2;
    cudaStream_t side = nullptr;
    cudaEvent_t join = nullptr;
    HY_RET_IF(side_fork(st, &side, &join));
    gemm_set_sms_cap(num_sms() - split_reserve_sms());
    // group A (side stream) starts half a layer ahead: group B's first QKV projection waits
    // for A's, so from then on A's attention meets B's GEMMs and vice versa
    int rc = layer(0, 0, 0, na, na, side, w.gemm_ws2, w.dec_ws2);
    if (rc == 0) rc = side_mark_and_wait(side, st);
    for (int li = 0; li < m->n_layers && rc == 0; ++li) {
      rc = layer(li, 1, 0, na, na, side, w.gemm_ws2, w.dec_ws2);
      if (rc == 0 && li + 1 < m->n_layers) rc = layer(li + 1, 0, 0, na, na, side, w.gemm_ws2, w.dec_ws2);
      if (rc == 0) rc = layer(li, 0, na, R, nd - na, st, w.gemm_ws, w.dec_ws);
      if (rc == 0) rc = layer(li, 1, na, R, nd - na, st, w.gemm_ws, w.dec_ws);
    }
    gemm_set_sms_cap(0);
    HY_RET_IF(rc);
    HY_RET_IF(side_join(st, side, join));
  } else {
    for (int li = 0; li < m->n_layers; ++li) {
      HY_RET_IF(layer(li, 0, 0, R, nd, st, w.gemm_ws, w.dec_ws));
      HY_RET_IF(layer(li, 1, 0, R, nd, st, w.gemm_ws, w.dec_ws));
    }
  }
  if (b->n_out > 0) {
    HY_RET_IF(rmsnorm(w.x, H, m->final_norm, w.tout, H, b->n_out, H, m->rms_eps, b->out_rows, st));
    float* logits = b->out_logits ? b->out_logits : w.logits;
    HY_RET_IF(G(w.tout, H, m->lm_head, b->n_out, m->vocab, H, nullptr, nullptr, 0, HY_ACT_NONE,
                logits, m->vocab, 1, st, w.gemm_ws));
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
  // HY_VIT_SMS=<n> (A/B): the ViT's GEMM grids use at most n SMs, so a concurrent language
  // batch keeps the rest (the vision stream is rarely the batch's critical path)
  static const int vit_sms = [] {
    const char* e = getenv("HY_VIT_SMS");
    return e ? atoi(e) : 0;
  }();
  struct CapGuard {
    bool on;
    explicit CapGuard(int n) : on(n > 0) {
      if (on) gemm_set_sms_cap(n);
    }
    ~CapGuard() {
      if (on) gemm_set_sms_cap(0);
    }
  } cap_guard(vit_sms);
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
