// Is a 32 KB tile store from one CTA intrinsically slow?  (graph-timed)
#include "../../paper_2505_12658_b200/csrc/common.cuh"
#include <cstdio>
using namespace hy;
__device__ unsigned long long g_t[8];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}
// thread-per-row 16B stores, 128 rows x 128 bf16
__global__ void k_rows(bf16* out, int ldc, int mode) {
  extern __shared__ __align__(1024) uint8_t s[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(s);
  if (mode & 1) {
    if ((threadIdx.x >> 5) == 0) tmem_alloc(slot, 256);
    tc_fence_before(); __syncthreads(); tc_fence_after();
  }
  unsigned long long t0 = gt();
  const int r = threadIdx.x;
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = r * 0.5f + j;
  if (mode & 2) {
    // coalesced: lane-consecutive 16B, warp covers rows (8 rows x 64B per instr for 128-col tile: 16 lanes/row)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int it = 0; it < 16; ++it) {
      const int row = w * 32 + it * 2 + lane / 16;
      store_bf16x8(out + (size_t)row * ldc + (lane % 16) * 8, v);
    }
  } else {
    for (int c = 0; c < 16; ++c) store_bf16x8(out + (size_t)r * ldc + c * 8, v);
  }
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { g_t[0] = t1 - t0; }
  if (mode & 1) {
    tc_fence_before(); __syncthreads();
    if ((threadIdx.x >> 5) == 0) { tc_fence_after(); tmem_dealloc(*slot, 256); }
  }
}
static cudaStream_t g_st;
template <typename F>
float timeit(F f, int n = 100) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f();
  cudaStreamSynchronize(g_st);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(g_st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) f();
  cudaStreamEndCapture(g_st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, g_st); cudaStreamSynchronize(g_st);
  cudaEventRecord(a, g_st); cudaGraphLaunch(ge, g_st); cudaEventRecord(b, g_st);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  if (cudaGetLastError()) printf("err\n");
  return ms * 1000.f / n;
}
int main() {
  cudaStreamCreate(&g_st);
  bf16* out; cudaMalloc(&out, 64 << 20);
  for (int mode = 0; mode < 4; ++mode)
    for (int ldc : {128, 4096}) {
      float t = timeit([&] { k_rows<<<1, 128, 1024, g_st>>>(out, ldc, mode); });
      unsigned long long tt[8]; cudaMemcpyFromSymbol(tt, g_t, sizeof(tt));
      printf("mode %d ldc %d: %.2f us/launch, in-kernel store loop %llu ns\n", mode, ldc, t, tt[0]);
    }
  return 0;
}
