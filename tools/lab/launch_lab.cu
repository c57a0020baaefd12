// Launch-overhead lab: what does a 1-CTA tcgen05 kernel pay before doing work?
#include "../../paper_2505_12658_b200/csrc/common.cuh"
#include <cstdio>
using namespace hy;

__global__ void k_empty() {}
__global__ void k_smem(int x) {
  extern __shared__ uint8_t s[];
  if (x == 12345) s[threadIdx.x] = 1;
}
__global__ void k_tmem(int x) {
  extern __shared__ __align__(1024) uint8_t s[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(s);
  if ((threadIdx.x >> 5) == 1) tmem_alloc(slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t base = *slot;
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 1) { tc_fence_after(); tmem_dealloc(base, 256); }
  if (x == 12345) s[threadIdx.x] = 1;
}
__global__ void k_tma(const __grid_constant__ CUtensorMap tm, int x) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 65536);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, 128 * 64 * 2);
    tma_load_2d(&tm, bar, s, 0, 0, kEvictNormal);
  }
  mbar_wait(bar, 0);
  if (x == 12345) s[threadIdx.x] = 1;
}

static cudaStream_t g_st;
template <typename F>
float timeit(F f, int n = 200) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) f();
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(g_st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) f();
  cudaStreamEndCapture(g_st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, g_st);
  cudaStreamSynchronize(g_st);
  cudaEventRecord(a, g_st);
  cudaGraphLaunch(ge, g_st);
  cudaEventRecord(b, g_st);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / n;
}

int main() {
  const int big = 197 * 1024;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaStreamCreate(&g_st);
  void* buf; cudaMalloc(&buf, 1 << 24);
  CUtensorMap tm;
  make_tmap_2d_bf16(&tm, buf, 4096, 64, 128, 128, 64);
  printf("empty 1x192           %.2f us\n", timeit([] { k_empty<<<1, 192, 0, g_st>>>(); }));
  printf("empty 148x192         %.2f us\n", timeit([] { k_empty<<<148, 192, 0, g_st>>>(); }));
  printf("smem 16K 1x192        %.2f us\n", timeit([] { k_smem<<<1, 192, 16384, g_st>>>(0); }));
  printf("smem 197K 1x192       %.2f us\n", timeit([&] { k_smem<<<1, 192, big, g_st>>>(0); }));
  printf("smem 197K 148x192     %.2f us\n", timeit([&] { k_smem<<<148, 192, big, g_st>>>(0); }));
  printf("tmem 197K 1x192       %.2f us\n", timeit([&] { k_tmem<<<1, 192, big, g_st>>>(0); }));
  printf("tmem 16K 1x192        %.2f us\n", timeit([&] { k_tmem<<<1, 192, 16384, g_st>>>(0); }));
  printf("tma 197K 1x192        %.2f us\n", timeit([&] { k_tma<<<1, 192, big, g_st>>>(tm, 0); }));
  printf("tma 80K 1x192         %.2f us\n", timeit([&] { k_tma<<<1, 192, 80 * 1024, g_st>>>(tm, 0); }));
  printf("tma 80K 148x192       %.2f us\n", timeit([&] { k_tma<<<148, 192, 80 * 1024, g_st>>>(tm, 0); }));
  return 0;
}
