/*
 * hydra_sm100.h -- C ABI of libhydra_sm100.so, the B200 (sm_100a) executor that
 * replaces the analytical cost model under epdsim's stage-level scheduler.
 *
 * The reference (/root/reference/pkg/src/epdsim) ships no native code: its hot path
 * is two pure functions, and this library is what sits behind them when the
 * simulator's clock is replaced by a real GPU:
 *
 *   batch_latency(batch, reqs, model, hw) -> float        engine.py:500-509
 *       called per instance iteration at cluster.py:295
 *       -> hy_vit_forward   (encode entries,  vision_work   model_cost.py:151-168)
 *       -> hy_lang_forward  (prefill chunks + decode entries, language_work 171-197)
 *   MigrationJob.transfer_seconds(hw) -> float             migration.py:63-64
 *       called at cluster.py:323 (transfer start) and 437 (accounting)
 *       -> hy_copy_blocks   (EP image-embedding handoff, PD KV-block migration)
 *
 * The per-kernel entry points are exported too so the parity tests can drive each
 * kernel against the CPU oracle.
 *
 * Conventions
 *   - every entry point returns 0 or a cudaError_t code; hy_last_error() gives text;
 *   - every pointer is device memory (or a mapped peer pointer) unless stated;
 *   - int32 metadata arrays are device resident; host arrays are marked "host";
 *   - any host thread may call with its own stream, on any device.  Process-wide state is
 *     limited to: the per-(device, kernel) shared-memory attribute and carveout caches
 *     (mutex guarded), one side stream + events per (host thread, device, priority), tuning
 *     knobs read from the environment (HY_*; defaults are the measured best), the measured
 *     GEMM dispatch table (constant, compiled in), the launch counter (hy_launch_count) and
 *     the optional kernel timer hook (hy_set_kernel_timer, a bench/test instrument that must
 *     not be set while several threads launch).  Per-host-thread settings: hy_set_pdl,
 *     hy_set_decode_kernel, hy_set_decode_coresident;
 *   - nothing falls back to the CPU: a missing device or bad argument is an error.
 *
 * Paged layouts (one instance = one GPU)
 *   KV pool   : [num_blocks][layers][2 (K,V)][kv_heads][16 tokens][head_dim] bf16
 *               one block is one contiguous migration unit (8 MiB for LLaVA-1.5-7B)
 *               block geometry = KV_BLOCK_TOKENS (model_cost.py:15)
 *   image pool: [num_blocks][576][lang_hidden] bf16, 576 = IMAGE_BLOCK_TOKENS (model_cost.py:16)
 */
#ifndef HYDRA_SM100_H
#define HYDRA_SM100_H

#include <stddef.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HY_KV_BLOCK_TOKENS 16
#define HY_IMAGE_BLOCK_TOKENS 576

/* epilogue activations */
#define HY_ACT_NONE 0
#define HY_ACT_QUICK_GELU 1 /* x * sigmoid(1.702 x)  (CLIP MLP) */
#define HY_ACT_GELU 2       /* 0.5 x (1 + erf(x / sqrt 2))  (projector) */
#define HY_ACT_SILU 3
#define HY_ACT_SWIGLU 4     /* physical cols [32g,32g+16)=gate, [32g+16,32g+32)=up -> 16 outputs */

/* token-row sentinel: take the input token from last_tok[row_slot[r]] */
#define HY_TOK_FROM_LAST (-2147483647 - 1)

typedef struct HyGemmEpilogue {
  const void* bias;     /* [N] bf16 or NULL (added before the activation) */
  const void* residual; /* [M, ldr] bf16 or NULL (added after the activation); may alias out */
  int ldr;
  int act;              /* HY_ACT_* */
  const int* row_map;   /* [M] output row index or NULL (identity) */
  void* out;            /* [rows, ldc] bf16, or fp32 when out_f32 */
  int ldc;
  int out_f32;
} HyGemmEpilogue;

/* ---------------- library ---------------- */
const char* hy_last_error(void);
int hy_version(void);
int hy_device_sm_count(void);
/* total kernels launched by this library in this process */
long long hy_launch_count(void);

/* Live per-kernel timing: while a timer is installed, the composite forwards record a
 * (begin, end) cudaEvent pair around every launch of kernel class `klass` on the
 * launching stream, and the launch's algorithmic work (GEMM: 2MNK flops; attention: 0,
 * filled by the caller) into work[i].  events: host array of 2*capacity cudaEvent_t. */
#define HY_KCLASS_DECODE_ATTN 1
#define HY_KCLASS_GEMM 2
#define HY_KCLASS_PREFILL_ATTN 3
#define HY_KCLASS_VIT_ATTN 4
typedef struct HyKernelTimer {
  int klass;
  int capacity;
  int count;
  void* events;  /* cudaEvent_t[2 * capacity] */
  double* work;  /* [capacity] or NULL */
  long long* shape; /* [capacity] or NULL: GEMM (M << 42) | (N << 21) | K */
} HyKernelTimer;
void hy_set_kernel_timer(HyKernelTimer* timer);
/* Programmatic dependent launch for the kernels the CALLING host thread launches next
 * (on != 0): each kernel's prologue -- barrier init, TMEM allocation, the GEMM's weight
 * prefetch -- overlaps the previous kernel's tail.  Off by default; the executor turns it on
 * for decode-only language batches without vision work (measured 9% faster there, 2% slower
 * on mixed batches whose early dependents hold SMs the vision stream needs).  HY_PDL=1 / 0
 * in the environment overrides it for the whole process. */
int hy_set_pdl(int on);

/* ---------------- K1: GEMM (tcgen05 + TMEM + TMA) ---------------- */
/* out = epi(A[M,K] . W[N,K]^T).  K, lda, ldw % 8 == 0, N % 16 == 0.
 * workspace: fp32 split-K partials (may be NULL: no split-K). */
int hy_gemm_bf16(const void* A, int lda, const void* W, int ldw, int M, int N, int K,
                 const HyGemmEpilogue* epi, void* workspace, size_t workspace_bytes,
                 cudaStream_t stream);
/* mode 0 = heuristic, 1 = force swap-AB (decode orientation), 2 = force normal (one CTA per
 * tile), 3 = force the CTA-pair kernel (cta_group::2, 256-row tiles; 256-wide weight tiles, or
 * 128-wide when N % 256 != 0; N % 128 == 0) */
int hy_gemm_bf16_mode(const void* A, int lda, const void* W, int ldw, int M, int N, int K,
                      const HyGemmEpilogue* epi, void* workspace, size_t workspace_bytes,
                      int mode, cudaStream_t stream);

/* ---------------- K4: norms ---------------- */
/* out[i] = norm(x[row_idx ? row_idx[i] : i]) * w (+ b); rows of `cols` bf16 */
int hy_rmsnorm(const void* x, int ldx, const void* w, void* out, int ldo, int rows, int cols,
               float eps, const int* row_idx, cudaStream_t stream);
int hy_layernorm(const void* x, int ldx, const void* w, const void* b, void* out, int ldo,
                 int rows, int cols, float eps, const int* row_idx, cudaStream_t stream);

/* ---------------- K5: image-token merge / embedding gather ---------------- */
/* out[r] = tok[r] >= 0             : embed[tok[r]]
 *          tok[r] == HY_TOK_FROM_LAST: embed[last_tok[row_slot[r]]]
 *          otherwise                : image_rows[-(tok[r]+1)]   (image pool as [blocks*576, H]) */
int hy_merge_embed(const int* tok, int rows, const void* embed, const void* image_rows,
                   int hidden, const int* last_tok, const int* row_slot, void* out,
                   cudaStream_t stream);

/* ---------------- K6: RoPE + paged KV append ---------------- */
/* qkv rows: [q heads | k heads | v heads] x head_dim.  Rotates q in place and writes the
 * rotated k and v of row r into block block_table[row_slot[r]*bt_stride + pos[r]/16],
 * token pos[r]%16, of the layer view kv_layer (= pool base + layer * layer_stride). */
int hy_rope_kv_append(void* qkv, int ld_qkv, int rows, int n_heads, int n_kv_heads, int head_dim,
                      const int* pos, const int* row_slot, const int* block_table, int bt_stride,
                      void* kv_layer, long long block_stride, float rope_theta,
                      cudaStream_t stream);

/* ---------------- K8: paged-KV decode attention ---------------- */
/* q: [n, ld_q] (q heads x d at column 0); ctx[i] keys of slot slots[i]; out [n, ld_o].
 * workspace (hy_attn_decode_workspace_bytes): 2 KB of ticket counters / per-SM flags (the
 * opt-in K8b / K8c kernels reset them on the stream before each launch), then the split-KV
 * partials.  Calls on different streams need different workspaces. */
int hy_attn_decode_paged(const void* q, int ld_q, int n, int n_heads, int n_kv_heads,
                         int head_dim, const int* slots, const int* ctx, int max_ctx,
                         const int* block_table, int bt_stride, const void* kv_layer,
                         long long block_stride, float scale, void* out, int ld_o,
                         void* workspace, size_t workspace_bytes, cudaStream_t stream);
size_t hy_attn_decode_workspace_bytes(int n, int n_heads, int head_dim, int max_ctx);
/* Kernel choice for MHA decode attention on the CALLING host thread: nw > 0 selects the
 * bulk-copy kernel (K8b) with nw warps x spw ring stages per CTA -- built to share SMs with a
 * GEMM on another stream; nw = 0 restores the default (register-load kernel K8).
 * Supported (nw, spw): (1,4) (1,5) (2,2) (2,3) (2,4) (4,1) (4,2) (4,6) (5,1) (8,3).  Returns 0 or cudaErrorInvalidValue. */
int hy_set_decode_kernel(int nw, int spw);
/* Co-resident mode for decode attention on the CALLING host thread (on != 0): the
 * tensor-core kernel K8c that shares every SM with a running GEMM -- at most one CTA per SM,
 * a ~36 KB shared-memory ring -- for GQA groups 1 and 7; other groups use the default kernel.
 * hy_lang_forward's decode / prefill split turns it on for its decode rows. */
int hy_set_decode_coresident(int on);

/* ---------------- K7: paged prefill attention (causal with offset) ---------------- */
/* sequence s owns query rows [qstart[s], qstart[s+1]) at positions offset[s] + i and
 * attends to keys [0, offset[s] + i] of slot slots[s] in the paged cache.  n_rows: rows of
 * the q buffer (qstart[n_seqs]).  head_dim 64/128 runs on tcgen05 (attn_tc.cu). */
int hy_attn_prefill_paged(const void* q, int ld_q, int n_rows, int n_seqs, const int* qstart,
                          const int* offset, const int* slots, int max_q, int n_heads,
                          int n_kv_heads, int head_dim, const int* block_table, int bt_stride,
                          const void* kv_layer, long long block_stride, float scale, void* out,
                          int ld_o, cudaStream_t stream);

/* ---------------- K3: ViT varlen attention (block-diagonal, non-causal) ---------------- */
/* qkv rows [q | k | v] (n_heads x d each); segment s = rows [seg[s], seg[s+1]);
 * n_rows = seg[n_segs].  head_dim 64/128 runs on tcgen05 (attn_tc.cu). */
int hy_attn_varlen(const void* qkv, int ld_qkv, int n_rows, int n_segs, const int* seg, int max_len,
                   int n_heads, int head_dim, float scale, void* out, int ld_o,
                   cudaStream_t stream);

/* ---------------- K9: greedy argmax ---------------- */
/* out_idx[i] = argmax_j logits[i, j] (first maximum); if out_slot, also
 * last_tok[out_slot[i]] = out_idx[i]. */
int hy_argmax_f32(const float* logits, int rows, int vocab, int ld, int* out_idx,
                  const int* out_slot, int* last_tok, cudaStream_t stream);

/* ---------------- K2: ViT patch embedding ---------------- */
typedef struct HyImageDesc {
  const unsigned char* pixels; /* HWC uint8, top-left crop of gh*patch x gw*patch used */
  int row_stride;              /* bytes between pixel rows */
  int gh, gw;                  /* patch grid */
  int tok_start;               /* first ViT token row (includes CLS if present) */
  int patch_start;             /* first patch row */
  int vis_start;               /* first visual (output) token */
  int pad_;
} HyImageDesc;

/* patches[patch_start + i][k] = normalised pixel, k = c*p*p + ky*p + kx, zero for k >= 3p^2;
 * window-major patch order when merge == 2 (2x2 windows contiguous). */
int hy_im2col_patches(const HyImageDesc* images, int n_images, int n_patches, int patch,
                      int merge, int k_pad, void* patches, cudaStream_t stream);

/* ---------------- K10/K11: block migration copy ---------------- */
/* dst_base + dst_ids[i]*block_bytes <- src_base + src_ids[i]*block_bytes, i < n.
 * Pointers may be peer (NVLink) addresses.  ids are device int32 arrays. */
int hy_copy_blocks(const void* src_base, void* dst_base, const int* src_ids, const int* dst_ids,
                   int n, long long block_bytes, cudaStream_t stream);

/* Token-exact variant (SURVEY.md 8b `valid_tail_bytes`): blocks 0..n-2 are copied whole; the
 * last block is viewed as block_bytes / group_bytes groups and only the first
 * tail_group_bytes of each group are copied.  KV block [layers][K|V][kv_heads][16][d]:
 * group = 16*d*2 bytes, tail = valid_tokens*d*2, so the bytes moved equal the reference's
 * MigrationJob.kv_bytes (cluster.py:411, migration.py:63-64).  Image block [576][H]: group =
 * block, tail = valid_rows*H*2.  Records whose size is not a multiple of 16 bytes (e.g. a
 * 4-byte last-token slot) are copied whole with group = tail = block_bytes. */
int hy_copy_blocks_tail(const void* src_base, void* dst_base, const int* src_ids,
                        const int* dst_ids, int n, long long block_bytes, long long group_bytes,
                        long long tail_group_bytes, cudaStream_t stream);

/* peer access for P2P block copies between GPUs driven by one process */
int hy_enable_peer_access(int device, int peer);

/* device metadata maintenance: dst[idx[i]] = val[i] (block-table updates) */
int hy_scatter_i32(int* dst, const int* idx, const int* val, int n, cudaStream_t stream);

/* ---------------- deterministic weight / input synthesis ---------------- */
/* logical element (r, c) of a rows x cols tensor = offset + scale * u(seed, tensor_id, r*cols+c),
 * u uniform in [-1, 1) from a counter hash (restated bit-exactly in oracle/synth.py).
 * perm: 0 = dense [rows][ld]; 1 = SwiGLU interleave: logical rows [0, rows/2) are gate,
 * [rows/2, rows) are up, physical row 32g+j holds gate 16g+j (j<16) / up 16g+j-16. */
int hy_fill_uniform_bf16(void* dst, long long rows, long long cols, long long ld,
                         unsigned long long seed, unsigned long long tensor_id, float scale,
                         float offset, int perm, cudaStream_t stream);

/* ---------------- composite forwards (native layer loop) ---------------- */
typedef struct HyLangLayerW {
  const void* attn_norm; /* [H] */
  const void* w_qkv;     /* [(Hq + 2 Hkv) d, H] */
  const void* b_qkv;     /* [(Hq + 2 Hkv) d] or NULL */
  const void* w_o;       /* [H, Hq d] */
  const void* ffn_norm;  /* [H] */
  const void* w_gate_up; /* [2F, H], SwiGLU-interleaved rows */
  const void* w_down;    /* [H, F] */
} HyLangLayerW;

typedef struct HyLangModel {
  int hidden, n_heads, n_kv_heads, head_dim, n_layers, ffn, vocab;
  float rope_theta, rms_eps;
  const void* embed;          /* [vocab, H] */
  const void* final_norm;     /* [H] */
  const void* lm_head;        /* [vocab, H] */
  const HyLangLayerW* layers; /* host array [n_layers] */
} HyLangModel;

typedef struct HyKvCache {
  void* base;               /* pool base */
  long long block_stride;   /* elements per block (all layers) */
  long long layer_stride;   /* elements per layer inside a block */
  int num_blocks;
  const int* block_table;   /* [slots][bt_stride] */
  int bt_stride;
} HyKvCache;

typedef struct HyLangBatch {
  int n_rows;      /* decode rows first, then the prefill chunks' rows */
  int n_decode;
  int n_prefill;
  const int* tok;      /* [n_rows] see hy_merge_embed */
  const int* pos;      /* [n_rows] */
  const int* row_slot; /* [n_rows] */
  const int* dec_ctx;  /* [n_decode] keys attended (kv_len + 1) */
  const int* pf_qstart;/* [n_prefill + 1] row offsets within the prefill rows */
  const int* pf_offset;/* [n_prefill] tokens already cached (prefill_done) */
  const int* pf_slot;  /* [n_prefill] */
  int pf_max_q;
  int max_ctx;
  int n_out;
  const int* out_rows; /* [n_out] rows whose next token is produced */
  const int* out_slot; /* [n_out] slot whose last_tok is updated */
  int* out_tokens;     /* [n_out] */
  float* out_logits;   /* optional [n_out, vocab] fp32 copy for parity tests, or NULL */
} HyLangBatch;

size_t hy_lang_workspace_bytes(const HyLangModel* m, int max_rows, int max_out, int max_decode,
                               int max_ctx);
int hy_lang_forward(const HyLangModel* m, const HyLangBatch* b, const HyKvCache* kv,
                    const void* image_rows, int* last_tok, void* workspace,
                    size_t workspace_bytes, cudaStream_t stream);

typedef struct HyVitLayerW {
  const void *ln1_w, *ln1_b, *w_qkv, *b_qkv, *w_o, *b_o;
  const void *ln2_w, *ln2_b, *w_fc1, *b_fc1, *w_fc2, *b_fc2;
} HyVitLayerW;

typedef struct HyVitModel {
  int hidden, n_heads, head_dim, n_layers, mlp;
  int patch, k_pad;      /* patch size, padded 3*p*p */
  int cls;               /* 1: prepend a class token (dropped from the output) */
  int pre_ln;            /* 1: LayerNorm after the embeddings (CLIP pre_layrnorm) */
  int merge;             /* 1: one visual token per patch; 2: 2x2 patch merger (Qwen2-VL) */
  int lang_hidden, proj_hidden;
  int max_pos;
  float ln_eps;
  const void* w_patch;   /* [hidden, k_pad] */
  const void* cls_emb;   /* [hidden] */
  const void* pos_emb;   /* [max_pos, hidden] */
  const void *pre_ln_w, *pre_ln_b;
  const HyVitLayerW* layers; /* host array */
  const void *merge_ln_w, *merge_ln_b;      /* merge == 2 */
  const void *w_proj1, *b_proj1;            /* [proj_hidden, hidden * merge^2] */
  const void *w_proj2, *b_proj2;            /* [lang_hidden, proj_hidden] */
} HyVitModel;

typedef struct HyVitBatch {
  int n_images, n_tokens, n_patches, n_visual;
  int max_image_tokens;
  const HyImageDesc* images; /* device [n_images] */
  const int* seg;            /* device [n_images + 1] ViT token offsets */
  const int* out_row_map;    /* device [n_visual] image-pool row of each visual token */
  void* image_rows;          /* image pool as [blocks * 576, lang_hidden] */
} HyVitBatch;

size_t hy_vit_workspace_bytes(const HyVitModel* m, int max_tokens, int max_image_tokens);
int hy_vit_forward(const HyVitModel* m, const HyVitBatch* b, void* workspace,
                   size_t workspace_bytes, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* HYDRA_SM100_H */
