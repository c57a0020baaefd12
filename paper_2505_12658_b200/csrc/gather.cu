// Index-driven data movement kernels on the serving path:
//   K5  hy_merge_embed      image-token merge / embedding gather for prefill windows and decodes
//   K6  hy_rope_kv_append   RoPE on q/k + write of k/v into 16-token paged KV blocks
//   K9  hy_argmax_f32       greedy next token (first maximum, like torch.argmax)
//   K2  hy_im2col_patches   uint8 HWC pixels -> normalised bf16 patch rows for the patch GEMM
//       vit_assemble        [CLS] + patch embeddings + learned positions (+ CLIP pre-LN)
//       vit_gather_visual   drop CLS rows before the projector
//   K10/K11 hy_copy_blocks  block-granular KV / image-cache migration copy (peer pointers OK)
//       hy_fill_uniform_bf16 counter-hash synthetic weights (restated in oracle/synth.py)
// All are HBM/latency-bound byte movers: coalesced 16-byte accesses, no tensor cores.
#include "common.cuh"
#include "../../include/hydra_sm100.h"

namespace hy {

// ---------------------------------------------------------------------------
// K5 merge / embedding gather
// ---------------------------------------------------------------------------
__global__ void merge_embed_kernel(const int* __restrict__ tok, int rows, const bf16* __restrict__ embed,
                                   const bf16* __restrict__ image_rows, int hidden,
                                   const int* __restrict__ last_tok, const int* __restrict__ row_slot,
                                   bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  int r = blockIdx.x;
  if (r >= rows) return;
  int t = tok[r];
  const bf16* src;
  if (t == HY_TOK_FROM_LAST) {
    src = embed + (size_t)last_tok[row_slot[r]] * hidden;
  } else if (t >= 0) {
    src = embed + (size_t)t * hidden;
  } else {
    src = image_rows + (size_t)(-(t + 1)) * hidden;
  }
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(out + (size_t)r * hidden);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) d[i] = s[i];
}

// ---------------------------------------------------------------------------
// K6 RoPE (rotate-half convention) + paged KV append
// ---------------------------------------------------------------------------
__global__ void rope_kv_append_kernel(bf16* __restrict__ qkv, int ld_qkv, int rows, int n_heads,
                                      int n_kv, int d, const int* __restrict__ pos,
                                      const int* __restrict__ row_slot,
                                      const int* __restrict__ block_table, int bt_stride,
                                      bf16* __restrict__ kv, long long block_stride, float theta) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int p = pos[r];
  const int half = d / 2;
  // the rotation angles depend on (position, frequency) only: one sincos per frequency per
  // row, shared by every q and k head (inv_freq_i = theta^(-2i/d) in fp32, HF-style)
  __shared__ float2 cs[128];  // d <= 256
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float inv = 1.0f / powf(theta, (float)(2 * i) / (float)d);
    float sn, cn;
    sincosf((float)p * inv, &sn, &cn);
    cs[i] = make_float2(cn, sn);
  }
  __syncthreads();
  bf16* row = qkv + (size_t)r * ld_qkv;
  const int blk = block_table[(size_t)row_slot[r] * bt_stride + p / HY_KV_BLOCK_TOKENS];
  const int tk = p % HY_KV_BLOCK_TOKENS;
  bf16* kbase = kv + (size_t)blk * block_stride;
  bf16* vbase = kbase + (size_t)n_kv * HY_KV_BLOCK_TOKENS * d;
  if ((half & 7) == 0 && (ld_qkv & 7) == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0) {
    // 16-byte vectors: a work item is 8 dims [i, i+8) of the first half and the matching
    // 8 of the second half of one q/k head, or 8 dims of one v head
    const int vph = half / 8;  // vector pairs per head
    const int n_rot = (n_heads + n_kv) * vph;
    const int total = n_rot + n_kv * (d / 8);
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      if (j < n_rot) {
        const int h = j / vph;
        const int i = (j % vph) * 8;
        bf16* x = row + (size_t)h * d;
        float lo[8], hi[8], olo[8], ohi[8];
        load_bf16x8(x + i, lo);
        load_bf16x8(x + i + half, hi);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float2 a = cs[i + t];
          olo[t] = lo[t] * a.x - hi[t] * a.y;
          ohi[t] = hi[t] * a.x + lo[t] * a.y;
        }
        bf16* dst = h < n_heads ? x : kbase + ((size_t)(h - n_heads) * HY_KV_BLOCK_TOKENS + tk) * d;
        store_bf16x8(dst + i, olo);
        store_bf16x8(dst + i + half, ohi);
      } else {
        const int jj = j - n_rot;
        const int vh = jj / (d / 8);
        const int i = (jj % (d / 8)) * 8;
        const uint4 v = *reinterpret_cast<const uint4*>(row + (size_t)(n_heads + n_kv + vh) * d + i);
        *reinterpret_cast<uint4*>(vbase + ((size_t)vh * HY_KV_BLOCK_TOKENS + tk) * d + i) = v;
      }
    }
    return;
  }
  const int pairs_per_head = half / 2;  // each thread handles dims (i, i+1) and (i+half, i+half+1)
  const int n_rot = (n_heads + n_kv) * pairs_per_head;
  const int total = n_rot + n_kv * (d / 2);
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    if (j < n_rot) {
      int h = j / pairs_per_head;
      int i = (j % pairs_per_head) * 2;
      const float2 a0 = cs[i], a1 = cs[i + 1];
      bf16* x = row + (size_t)h * d;  // q heads then k heads are contiguous
      float2 lo = unpack_bf16x2(*reinterpret_cast<uint32_t*>(x + i));
      float2 hi = unpack_bf16x2(*reinterpret_cast<uint32_t*>(x + i + half));
      float o_lo0 = lo.x * a0.x - hi.x * a0.y;
      float o_lo1 = lo.y * a1.x - hi.y * a1.y;
      float o_hi0 = hi.x * a0.x + lo.x * a0.y;
      float o_hi1 = hi.y * a1.x + lo.y * a1.y;
      uint32_t plo = pack_bf16x2(o_lo0, o_lo1), phi = pack_bf16x2(o_hi0, o_hi1);
      if (h < n_heads) {
        *reinterpret_cast<uint32_t*>(x + i) = plo;
        *reinterpret_cast<uint32_t*>(x + i + half) = phi;
      } else {
        int kh = h - n_heads;
        bf16* dst = kbase + ((size_t)kh * HY_KV_BLOCK_TOKENS + tk) * d;
        *reinterpret_cast<uint32_t*>(dst + i) = plo;
        *reinterpret_cast<uint32_t*>(dst + i + half) = phi;
      }
    } else {
      int jj = j - n_rot;
      int vh = jj / (d / 2);
      int i = (jj % (d / 2)) * 2;
      const bf16* src = row + (size_t)(n_heads + n_kv + vh) * d + i;
      bf16* dst = vbase + ((size_t)vh * HY_KV_BLOCK_TOKENS + tk) * d + i;
      *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
    }
  }
}

// ---------------------------------------------------------------------------
// K9 argmax over fp32 logits (first maximum)
// ---------------------------------------------------------------------------
__global__ void argmax_kernel(const float* __restrict__ logits, int rows, int vocab, int ld,
                              int* __restrict__ out_idx, const int* __restrict__ out_slot,
                              int* __restrict__ last_tok) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float* x = logits + (size_t)r * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const bool vec = (vocab % 4 == 0) && (ld % 4 == 0);
  if (vec) {
    for (int i = threadIdx.x * 4; i < vocab; i += blockDim.x * 4) {
      float4 v = *reinterpret_cast<const float4*>(x + i);
      if (v.x > best) { best = v.x; bi = i; }
      if (v.y > best) { best = v.y; bi = i + 1; }
      if (v.z > best) { best = v.z; bi = i + 2; }
      if (v.w > best) { best = v.w; bi = i + 3; }
    }
  } else {
    for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
      float v = x[i];
      if (v > best) { best = v; bi = i; }
    }
  }
  // reduce: larger value wins, ties -> smaller index
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = l < nw ? sv[l] : -INFINITY;
    bi = l < nw ? si[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (l == 0) {
      if (bi == 0x7fffffff) bi = 0;  // all-NaN row: deterministic token 0
      out_idx[r] = bi;
      if (out_slot && last_tok) last_tok[out_slot[r]] = bi;
    }
  }
}

// ---------------------------------------------------------------------------
// K2 im2col of uint8 HWC images (CLIP normalisation)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_image(const HyImageDesc* im, int n, int key, int which) {
  // largest i with start(i) <= key; which: 0 tok_start, 1 patch_start, 2 vis_start
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    int s = which == 0 ? im[mid].tok_start : which == 1 ? im[mid].patch_start : im[mid].vis_start;
    if (s <= key) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void patch_coords(int i, int gw, int merge, int& py, int& px) {
  if (merge == 2) {
    int w = i >> 2, j = i & 3;
    int wpr = gw >> 1;
    py = 2 * (w / wpr) + (j >> 1);
    px = 2 * (w % wpr) + (j & 1);
  } else {
    py = i / gw;
    px = i % gw;
  }
}

__global__ void im2col_kernel(const HyImageDesc* __restrict__ images, int n_images, int n_patches,
                              int patch, int merge, int k_pad, bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int pr = blockIdx.x;
  if (pr >= n_patches) return;
  const int ii = find_image(images, n_images, pr, 1);
  const HyImageDesc im = images[ii];
  int py, px;
  patch_coords(pr - im.patch_start, im.gw, merge, py, px);
  const float mean[3] = {0.48145466f, 0.4578275f, 0.40821073f};
  const float stdv[3] = {0.26862954f, 0.26130258f, 0.27577711f};
  const int kk = 3 * patch * patch;
  bf16* o = out + (size_t)pr * k_pad;
  for (int k = threadIdx.x; k < k_pad; k += blockDim.x) {
    float v = 0.f;
    if (k < kk) {
      int c = k / (patch * patch);
      int rem = k % (patch * patch);
      int ky = rem / patch, kx = rem % patch;
      int y = py * patch + ky, x = px * patch + kx;
      unsigned char u = im.pixels[(size_t)y * im.row_stride + (size_t)x * 3 + c];
      v = ((float)u * (1.0f / 255.0f) - mean[c]) / stdv[c];
    }
    o[k] = __float2bfloat16_rn(v);
  }
}

// [CLS] + patch rows + learned positions, then optional LayerNorm; one warp per token row.
__global__ void vit_assemble_kernel(const HyImageDesc* __restrict__ images, int n_images,
                                    int n_tokens, int hidden, int cls,
                                    const bf16* __restrict__ patch_rows,
                                    const bf16* __restrict__ cls_emb,
                                    const bf16* __restrict__ pos_emb, int max_pos,
                                    const bf16* __restrict__ ln_w, const bf16* __restrict__ ln_b,
                                    float eps, bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_tokens) return;
  const int ii = find_image(images, n_images, t, 0);
  const HyImageDesc im = images[ii];
  const int j = t - im.tok_start;
  const bf16* src = (cls && j == 0) ? cls_emb
                                    : patch_rows + (size_t)(im.patch_start + j - cls) * hidden;
  const bf16* pe = pos_emb + (size_t)min(j, max_pos - 1) * hidden;
  bf16* o = out + (size_t)t * hidden;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * 8; c < hidden; c += 256) {
    float a[8], b[8];
    load_bf16x8(src + c, a);
    load_bf16x8(pe + c, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // round the embedding sum to bf16 first: the oracle adds in bf16 storage order
      a[k] = __bfloat162float(__float2bfloat16_rn(a[k] + b[k]));
      s1 += a[k];
      s2 += a[k] * a[k];
    }
    store_bf16x8(o + c, a);
  }
  if (!ln_w) return;
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const float mean = s1 / hidden;
  const float rstd = rsqrtf(fmaxf(s2 / hidden - mean * mean, 0.f) + eps);
  __syncwarp();
  for (int c = lane * 8; c < hidden; c += 256) {
    float a[8], g[8], b[8];
    load_bf16x8(o + c, a);
    load_bf16x8(ln_w + c, g);
    load_bf16x8(ln_b + c, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (a[k] - mean) * rstd * g[k] + b[k];
    store_bf16x8(o + c, a);
  }
}

// visual token v -> ViT row (skipping each image's CLS row)
__global__ void vit_gather_visual_kernel(const HyImageDesc* __restrict__ images, int n_images,
                                         int n_visual, int hidden, int cls,
                                         const bf16* __restrict__ h, bf16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int v = blockIdx.x;
  if (v >= n_visual) return;
  const int ii = find_image(images, n_images, v, 2);
  const HyImageDesc im = images[ii];
  const int row = im.tok_start + cls + (v - im.vis_start);
  const uint4* s = reinterpret_cast<const uint4*>(h + (size_t)row * hidden);
  uint4* d = reinterpret_cast<uint4*>(out + (size_t)v * hidden);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) d[i] = s[i];
}

// ---------------------------------------------------------------------------
// K10/K11 block copy
// ---------------------------------------------------------------------------
__global__ void copy_blocks_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   const int* __restrict__ src_ids, const int* __restrict__ dst_ids,
                                   int n, long long block_bytes, int group16, int tail16) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.y;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)src_ids[b] * block_bytes);
  uint4* d = reinterpret_cast<uint4*>(dst + (size_t)dst_ids[b] * block_bytes);
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b == n - 1 && tail16 < group16) {
    // the request's last block: only the first tail16 vectors of every group are valid
    // (KV: tokens [0, valid) of each [layer][K|V][head] slab; image: the valid rows)
    const long long groups = (block_bytes / 16) / group16;
    const long long n16 = groups * tail16;
    for (; i < n16; i += stride) {
      const long long g = i / tail16;
      const long long o = g * group16 + (i - g * tail16);
      d[o] = ld_nc_v4(s + o);
    }
    return;
  }
  const long long n16 = block_bytes / 16;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a0 = ld_nc_v4(s + i), a1 = ld_nc_v4(s + i + stride), a2 = ld_nc_v4(s + i + 2 * stride),
          a3 = ld_nc_v4(s + i + 3 * stride);
    d[i] = a0;
    d[i + stride] = a1;
    d[i + 2 * stride] = a2;
    d[i + 3 * stride] = a3;
  }
  for (; i < n16; i += stride) d[i] = ld_nc_v4(s + i);
}

// element-granular variant for small records whose size is not a multiple of 16 bytes
// (the migrated request's last-token slot: 4 bytes)
__global__ void copy_records_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                    const int* __restrict__ src_ids,
                                    const int* __restrict__ dst_ids, int n, long long bytes) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.y;
  const uint8_t* s = src + (size_t)src_ids[b] * bytes;
  uint8_t* d = dst + (size_t)dst_ids[b] * bytes;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < bytes;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}

// ---------------------------------------------------------------------------
// deterministic synthesis: splitmix64 counter hash -> uniform [-1, 1)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(bf16* __restrict__ dst, long long rows, long long cols,
                                    long long ld, uint64_t key, float scale, float offset,
                                    int perm) {
  pdl_trigger();
  pdl_wait();
  const long long total = rows * ld;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long pr = e / ld, c = e % ld;
    if (c >= cols) {
      dst[e] = __float2bfloat16_rn(0.f);
      continue;
    }
    long long lr = pr;
    if (perm == 1) {
      long long g = pr >> 5, j = pr & 31;
      lr = j < 16 ? 16 * g + j : rows / 2 + 16 * g + (j - 16);
    }
    uint64_t h = splitmix64(key + (uint64_t)(lr * cols + c));
    float u = __fmul_rn((float)(h >> 40), 1.1920928955078125e-07f) - 1.0f;  // 2^-23
    float v = __fadd_rn(__fmul_rn(scale, u), offset);
    dst[e] = __float2bfloat16_rn(v);
  }
}

}  // namespace hy

using namespace hy;

extern "C" int hy_merge_embed(const int* tok, int rows, const void* embed, const void* image_rows,
                              int hidden, const int* last_tok, const int* row_slot, void* out,
                              cudaStream_t stream) {
  HY_CHECK_ARG(hidden % 8 == 0, "hidden % 8");
  if (rows <= 0) return 0;
  HY_CUDA_RET(launch_pdl(merge_embed_kernel, dim3(rows), dim3(128), 0, stream, tok, rows, reinterpret_cast<const bf16*>(embed),
                                               reinterpret_cast<const bf16*>(image_rows), hidden,
                                               last_tok, row_slot, reinterpret_cast<bf16*>(out)));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_rope_kv_append(void* qkv, int ld_qkv, int rows, int n_heads, int n_kv_heads,
                                 int head_dim, const int* pos, const int* row_slot,
                                 const int* block_table, int bt_stride, void* kv_layer,
                                 long long block_stride, float rope_theta, cudaStream_t stream) {
  HY_CHECK_ARG(head_dim % 4 == 0 && head_dim <= 256 && ld_qkv % 2 == 0, "rope: head_dim % 4, <= 256");
  if (rows <= 0) return 0;
  HY_CUDA_RET(launch_pdl(rope_kv_append_kernel, dim3(rows), dim3(256), 0, stream, 
      reinterpret_cast<bf16*>(qkv), ld_qkv, rows, n_heads, n_kv_heads, head_dim, pos, row_slot,
      block_table, bt_stride, reinterpret_cast<bf16*>(kv_layer), block_stride, rope_theta));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_argmax_f32(const float* logits, int rows, int vocab, int ld, int* out_idx,
                             const int* out_slot, int* last_tok, cudaStream_t stream) {
  if (rows <= 0) return 0;
  HY_CUDA_RET(launch_pdl(argmax_kernel, dim3(rows), dim3(256), 0, stream, logits, rows, vocab, ld, out_idx, out_slot, last_tok));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_im2col_patches(const HyImageDesc* images, int n_images, int n_patches, int patch,
                                 int merge, int k_pad, void* patches, cudaStream_t stream) {
  HY_CHECK_ARG(k_pad >= 3 * patch * patch, "k_pad");
  if (n_patches <= 0) return 0;
  HY_CUDA_RET(launch_pdl(im2col_kernel, dim3(n_patches), dim3(128), 0, stream, images, n_images, n_patches, patch, merge, k_pad,
                                               reinterpret_cast<bf16*>(patches)));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_copy_blocks_tail(const void* src_base, void* dst_base, const int* src_ids,
                                   const int* dst_ids, int n, long long block_bytes,
                                   long long group_bytes, long long tail_group_bytes,
                                   cudaStream_t stream) {
  HY_CHECK_ARG(block_bytes > 0 && n >= 0, "copy shape");
  if (n <= 0) return 0;
  if (block_bytes % 16 != 0) {  // small unaligned records: whole records only
    HY_CHECK_ARG(group_bytes == block_bytes && tail_group_bytes == block_bytes,
                 "tail copies need 16-byte aligned blocks");
    long long gx = (block_bytes + 255) / 256;
    dim3 grid((unsigned)(gx < 64 ? gx : 64), n);
    HY_CUDA_RET(launch_pdl(copy_records_kernel, grid, dim3(256), 0, stream,
                           reinterpret_cast<const uint8_t*>(src_base),
                           reinterpret_cast<uint8_t*>(dst_base), src_ids, dst_ids, n,
                           block_bytes));
    HY_LAUNCH_CHECK();
    return 0;
  }
  HY_CHECK_ARG(group_bytes > 0 && group_bytes % 16 == 0 && block_bytes % group_bytes == 0,
               "group_bytes must be a 16-byte multiple dividing block_bytes");
  HY_CHECK_ARG(tail_group_bytes > 0 && tail_group_bytes % 16 == 0 &&
                   tail_group_bytes <= group_bytes, "tail_group_bytes in (0, group_bytes], % 16");
  HY_CHECK_ARG(group_bytes / 16 < (1LL << 31), "group too large");
  long long n16 = block_bytes / 16;
  int threads = 256;
  long long want = (n16 + threads * 4 - 1) / (threads * 4);
  int gx = (int)(want < 256 ? (want < 1 ? 1 : want) : 256);
  dim3 grid(gx, n);
  HY_CUDA_RET(launch_pdl(copy_blocks_kernel, grid, dim3(threads), 0, stream,
                         reinterpret_cast<const uint8_t*>(src_base),
                         reinterpret_cast<uint8_t*>(dst_base), src_ids, dst_ids, n, block_bytes,
                         (int)(group_bytes / 16), (int)(tail_group_bytes / 16)));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_copy_blocks(const void* src_base, void* dst_base, const int* src_ids,
                              const int* dst_ids, int n, long long block_bytes,
                              cudaStream_t stream) {
  HY_CHECK_ARG(block_bytes % 16 == 0, "block_bytes % 16");
  return hy_copy_blocks_tail(src_base, dst_base, src_ids, dst_ids, n, block_bytes, block_bytes,
                             block_bytes, stream);
}

extern "C" int hy_fill_uniform_bf16(void* dst, long long rows, long long cols, long long ld,
                                    unsigned long long seed, unsigned long long tensor_id,
                                    float scale, float offset, int perm, cudaStream_t stream) {
  HY_CHECK_ARG(ld >= cols && rows >= 0, "fill shape");
  if (perm == 1) HY_CHECK_ARG(rows % 32 == 0, "swiglu interleave needs rows % 32 == 0");
  uint64_t key = splitmix64(seed ^ splitmix64(tensor_id));
  long long total = rows * ld;
  if (total == 0) return 0;
  int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  HY_CUDA_RET(launch_pdl(fill_uniform_kernel, dim3((unsigned)blocks), dim3(threads), 0, stream, 
      reinterpret_cast<bf16*>(dst), rows, cols, ld, key, scale, offset, perm));
  HY_LAUNCH_CHECK();
  return 0;
}

// device metadata maintenance: dst[idx[i]] = val[i] (block-table rows)
__global__ void scatter_i32_kernel(int* __restrict__ dst, const int* __restrict__ idx,
                                   const int* __restrict__ val, int n) {
  pdl_trigger();
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = val[i];
}

extern "C" int hy_scatter_i32(int* dst, const int* idx, const int* val, int n,
                              cudaStream_t stream) {
  if (n <= 0) return 0;
  HY_CUDA_RET(launch_pdl(scatter_i32_kernel, dim3((n + 255) / 256), dim3(256), 0, stream, dst, idx, val, n));
  HY_LAUNCH_CHECK();
  return 0;
}

extern "C" int hy_enable_peer_access(int device, int peer) {
  int can = 0;
  HY_CUDA_RET(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) {
    set_last_error("device " + std::to_string(device) + " cannot access peer " +
                   std::to_string(peer));
    return (int)cudaErrorPeerAccessUnsupported;
  }
  int prev = 0;
  HY_CUDA_RET(cudaGetDevice(&prev));
  HY_CUDA_RET(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  HY_CUDA_RET(e);
  return 0;
}

// internal launchers used by the composite ViT forward
namespace hy {
int vit_assemble(const HyImageDesc* images, int n_images, int n_tokens, int hidden, int cls,
                 const void* patch_rows, const void* cls_emb, const void* pos_emb, int max_pos,
                 const void* ln_w, const void* ln_b, float eps, void* out, cudaStream_t st) {
  if (n_tokens <= 0) return 0;
  HY_CHECK_ARG(hidden % 8 == 0, "vit hidden % 8");
  const int threads = 256;
  HY_CUDA_RET(launch_pdl(vit_assemble_kernel, dim3(ceil_div(n_tokens, threads / 32)), dim3(threads), 0, st, 
      images, n_images, n_tokens, hidden, cls, reinterpret_cast<const bf16*>(patch_rows),
      reinterpret_cast<const bf16*>(cls_emb), reinterpret_cast<const bf16*>(pos_emb), max_pos,
      reinterpret_cast<const bf16*>(ln_w), reinterpret_cast<const bf16*>(ln_b), eps,
      reinterpret_cast<bf16*>(out)));
  HY_LAUNCH_CHECK();
  return 0;
}
int vit_gather_visual(const HyImageDesc* images, int n_images, int n_visual, int hidden, int cls,
                      const void* h, void* out, cudaStream_t st) {
  if (n_visual <= 0) return 0;
  HY_CUDA_RET(launch_pdl(vit_gather_visual_kernel, dim3(n_visual), dim3(128), 0, st, images, n_images, n_visual, hidden, cls,
                                                     reinterpret_cast<const bf16*>(h),
                                                     reinterpret_cast<bf16*>(out)));
  HY_LAUNCH_CHECK();
  return 0;
}
}  // namespace hy
