// Single-warp-per-SMSP straight-line cost: 32 FADD + 32 STS, timed with clock64.
#include "../../paper_2505_12658_b200/csrc/common.cuh"
#include <cstdio>
using namespace hy;
__device__ long long g_c[8];
__global__ void __launch_bounds__(192, 1) k(float* in, int mode) {
  extern __shared__ __align__(1024) uint8_t s[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* slot = reinterpret_cast<uint32_t*>(s + 65536);
  if (mode & 1) {
    if (warp == 1) tmem_alloc(slot, 256);
    tc_fence_before(); __syncthreads(); tc_fence_after();
  }
  if (warp >= 2) {
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = in[j * 32 + lane];
    __syncwarp();
    long long t0 = clock64();
    float b = in[1000];
    const uint32_t d = smem_u32(s) + (warp - 2) * 4608 + lane * 4;
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_f32(d + j * 144, v[j] + b);
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0) g_c[warp] = t1 - t0;
  }
  if (mode & 1) {
    tc_fence_before(); __syncthreads();
    if (warp == 1) { tc_fence_after(); tmem_dealloc(*slot, 256); }
  }
}
int main() {
  float* in; cudaMalloc(&in, 1 << 20); cudaMemset(in, 0, 1 << 20);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      k<<<1, 192, 200 * 1024>>>(in, mode);
      cudaDeviceSynchronize();
      long long c[8]; cudaMemcpyFromSymbol(c, g_c, sizeof(c));
      printf("mode %d rep %d cycles: %lld %lld %lld %lld\n", mode, rep, c[2], c[3], c[4], c[5]);
    }
  return 0;
}
