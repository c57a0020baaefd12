#include "../../paper_2505_12658_b200/csrc/gemm.cu"
#include <cstdio>
#include <cstdlib>
static cudaStream_t g_st;
template <typename F>
float timeit(F f, int n = 50) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f();
  cudaStreamSynchronize(g_st);
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
int main(int argc, char** argv) {
  cudaStreamCreate(&g_st);
  void *A, *W, *C, *ws;
  cudaMalloc(&A, 64 << 20); cudaMalloc(&W, 256 << 20); cudaMalloc(&C, 64 << 20);
  cudaMalloc(&ws, 64 << 20); cudaMemset(ws, 0, 64 << 20);
  cudaMemset(A, 0, 64 << 20); cudaMemset(W, 0, 256 << 20);
  int shapes[][3] = {{128, 128, 64}, {128, 128, 1024}, {256, 4096, 64}, {1024, 2048, 64}, {577, 1024, 1024}, {64, 4096, 4096}, {2304, 4096, 4096}};
  int ns = sizeof(shapes) / sizeof(shapes[0]);
  if (argc > 1) {  // gemm_lab MxNxK ...
    ns = 0;
    for (int i = 1; i < argc && ns < 7; ++i, ++ns)
      sscanf(argv[i], "%dx%dx%d", &shapes[ns][0], &shapes[ns][1], &shapes[ns][2]);
  }
  for (int si = 0; si < ns; ++si) {
    int* s = shapes[si];
    int M = s[0], N = s[1], K = s[2];
    HyGemmEpilogue e{};
    e.out = C; e.ldc = N;
    for (int mode = 0; mode < 4; ++mode) {
      int rc = 0;
      float t = timeit([&] { rc |= hy::gemm_bf16((const hy::bf16*)A, K, (const hy::bf16*)W, K, M, N, K, &e, ws, 64 << 20, g_st, mode); });
      printf("M=%5d N=%5d K=%5d mode=%d  %.2f us %s\n", M, N, K, mode, t, rc ? hy::get_last_error() : "");
#ifdef HY_TRACE
      // one isolated launch, CTA 0 timeline (ns from entry)
      cudaDeviceSynchronize();
      hy::gemm_bf16((const hy::bf16*)A, K, (const hy::bf16*)W, K, M, N, K, &e, ws, 64 << 20, g_st, mode);
      cudaDeviceSynchronize();
      unsigned long long tr[32];
      cudaMemcpyFromSymbol(tr, hy::g_trace, sizeof(tr));
      printf("   trace:");
      for (int i = 1; i < 16; ++i) printf(" %d:%lld", i, (long long)(tr[i] - tr[0]));
      {
        unsigned long long cm[160][10];
        cudaMemcpyFromSymbol(cm, hy::g_ctr, sizeof(cm));
        unsigned long long t0 = ~0ull, tfirst_max = 0, tend_max = 0, tmma_max = 0;
        const int nc = 148;
        for (int c = 0; c < nc; ++c) if (cm[c][0] && cm[c][0] < t0) t0 = cm[c][0];
        printf("\n   per-CTA (ns from first entry): entry/first-full/last-mma/exit\n  ");
        for (int c = 0; c < nc; ++c) {
          if (!cm[c][0] || cm[c][0] < t0) continue;
          if (cm[c][3] - t0 > 1000000000ull) continue;
          if (c < 8 || c % 10 == 0)
            printf(" [%d %lld/%lld/%lld/%lld s%lld e%lld/%lld/%lld]", c, (long long)(cm[c][0] - t0),
                   cm[c][1] ? (long long)(cm[c][1] - t0) : -1LL, cm[c][2] ? (long long)(cm[c][2] - t0) : -1LL,
                   (long long)(cm[c][3] - t0), (long long)cm[c][4],
                   cm[c][6] ? (long long)(cm[c][6] - t0) : -1LL, cm[c][7] ? (long long)(cm[c][7] - t0) : -1LL,
                   cm[c][8] ? (long long)(cm[c][8] - t0) : -1LL);
          if (cm[c][1]) tfirst_max = std::max(tfirst_max, cm[c][1] - t0);
          if (cm[c][2]) tmma_max = std::max(tmma_max, cm[c][2] - t0);
          tend_max = std::max(tend_max, cm[c][3] - t0);
        }
        printf("\n   max first-full %lld  max last-mma %lld  max exit %lld\n", (long long)tfirst_max,
               (long long)tmma_max, (long long)tend_max);
        static unsigned long long zero[160][10];
        cudaMemcpyToSymbol(hy::g_ctr, zero, sizeof(zero));
      }
      printf("   MHz(0->8): %.0f  cycles 10->13: %lld 13->15: %lld\n", (double)(tr[24] - tr[16]) * 1e3 / (double)(tr[8] - tr[0]), (long long)(tr[29]-tr[26]), (long long)(tr[31]-tr[29]));
#endif
    }
  }
  return 0;
}
