// Verifies the tcgen05 operand layouts the attention kernel needs:
//   D[128 x 128] = P[128 x 64] . V[64 x 128]
// P: K-major SW128, written from registers with the manual 128B swizzle (softmax warps)
// V: [keys][d] row-major in global, TMA boxes of [64 keys][64 d] SW128 -> MN-major B operand
// Tries (LBO, SBO) variants for the MN-major descriptor; prints max error per variant.
#include "../../paper_2505_12658_b200/csrc/common.cuh"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
using namespace hy;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tmV, const bf16* P,
                                            float* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t sraw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sP = s;                  // 128 x 64 bf16 = 16 KB
  uint8_t* sV = s + 16384;          // 2 boxes of 64 keys x 64 d = 2 x 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 16384 + 16384);
  uint64_t* mbar = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) { mbar_init(bar, 1); mbar_init(mbar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(slot, 128);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    mbar_expect_tx(bar, 16384);
    tma_load_2d(&tmV, bar, sV, 0, 0, kEvictNormal);
    tma_load_2d(&tmV, bar, sV + 8192, 64, 0, kEvictNormal);
  }
  // P row tid: 64 bf16 = 8 chunks of 16B, swizzled
  {
    const int r = tid;
    for (int c = 0; c < 8; ++c) {
      uint4 v = *reinterpret_cast<const uint4*>(P + r * 64 + c * 8);
      uint32_t off = (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16);
      *reinterpret_cast<uint4*>(sP + off) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    mbar_wait(bar, 0);
    tc_fence_after();
    // idesc: D f32, A/B bf16, A K-major, B MN-major (bit 16), N=128, M=128
    const uint32_t idesc = idesc_bf16_f32(128, 128) | (1u << 16);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t a = smem_desc_k_sw128(smem_u32(sP) + kk * 32);
      // K step of 16 keys = 2 groups of 8 rows (1024 B each) in the V box
      const uint64_t b = desc_sw128(smem_u32(sV) + kk * 2048, lbo, sbo);
      umma_bf16(tmem, a, b, idesc, kk > 0 ? 1u : 0u);
    }
    umma_commit(mbar);
  }
  mbar_wait(mbar, 0);
  tc_fence_after();
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + c * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[tid * 128 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 128); }
}

__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// P from TMEM: columns 128..159 hold P[row][2j], P[row][2j+1] packed bf16x2
__global__ void __launch_bounds__(128, 1) k_ts(const __grid_constant__ CUtensorMap tmV, const bf16* P,
                                               float* D, int pack_swap) {
  extern __shared__ __align__(1024) uint8_t sraw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sV = s;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 16384);
  uint64_t* mbar = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) { mbar_init(bar, 1); mbar_init(mbar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(slot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    mbar_expect_tx(bar, 16384);
    tma_load_2d(&tmV, bar, sV, 0, 0, kEvictNormal);
    tma_load_2d(&tmV, bar, sV + 8192, 64, 0, kEvictNormal);
  }
  {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) {
      float a = __bfloat162float(P[tid * 64 + 2 * j]), b = __bfloat162float(P[tid * 64 + 2 * j + 1]);
      r[j] = pack_swap ? pack_bf16x2(b, a) : pack_bf16x2(a, b);
    }
    tmem_st_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + 128, r);
    tmem_st_wait();
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid == 0) {
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, 128) | (1u << 16);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t b = smem_desc_sw128(smem_u32(sV) + kk * 2048, 8192, 1024);
      umma_ts(tmem, tmem + 128 + kk * 8, b, idesc, kk > 0 ? 1u : 0u);
    }
    umma_commit(mbar);
  }
  mbar_wait(mbar, 0);
  tc_fence_after();
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + c * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[tid * 128 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

int main() {
  std::vector<uint16_t> hP(128 * 64), hV(64 * 128);
  std::vector<float> fP(128 * 64), fV(64 * 128);
  srand(1);
  auto bf = [](float x, float& back) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x8000) & 0xFFFF0000u; memcpy(&back, &u, 4); return (uint16_t)(u >> 16); };
  for (int i = 0; i < 128 * 64; ++i) hP[i] = bf((rand() % 200 - 100) / 100.f, fP[i]);
  for (int i = 0; i < 64 * 128; ++i) hV[i] = bf((rand() % 200 - 100) / 100.f, fV[i]);
  bf16 *dP, *dV; float* dD;
  cudaMalloc(&dP, hP.size() * 2); cudaMalloc(&dV, hV.size() * 2); cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dP, hP.data(), hP.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, hV.data(), hV.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  // V rows = keys (64), cols = d (128); box [64 rows][64 cols]
  if (make_tmap_2d_bf16(&tm, dV, 64, 128, 256, 64, 64)) { printf("tmap fail\n"); return 1; }
  std::vector<float> ref(128 * 128, 0.f);
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < 128; ++n) {
      double acc = 0;
      for (int kk = 0; kk < 64; ++kk) acc += (double)fP[i * 64 + kk] * fV[kk * 128 + n];
      ref[i * 128 + n] = (float)acc;
    }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  uint32_t variants[][2] = {{8192, 1024}, {1024, 8192}, {16, 1024}, {1024, 16}, {8192, 128}, {128, 8192}};
  for (auto& v : variants) {
    cudaMemset(dD, 0, 128 * 128 * 4);
    k<<<1, 128, 40 * 1024>>>(tm, dP, dD, v[0], v[1]);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(128 * 128);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 128 * 128; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("LBO %5u SBO %5u: max err %.4g %s\n", v[0], v[1], err, e ? cudaGetErrorString(e) : "");
    if (e) return 1;
  }
  cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int sw = 0; sw < 2; ++sw) {
    cudaMemset(dD, 0, 128 * 128 * 4);
    k_ts<<<1, 128, 40 * 1024>>>(tm, dP, dD, sw);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(128 * 128);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 128 * 128; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("A from TMEM, pack_swap %d: max err %.4g %s\n", sw, err, e ? cudaGetErrorString(e) : "");
    if (e) return 1;
  }
  return 0;
}
