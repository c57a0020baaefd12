// Timeline of the tcgen05 attention kernel (CTA 0) on one 2304-token paged prefill chunk.
#include "../../paper_2505_12658_b200/csrc/attn_tc.cu"
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
  const int nh = 32, d = 128, c = argc > 1 ? atoi(argv[1]) : 2304;
  const int nb = (c + 15) / 16;
  const long long be = 2LL * nh * 16 * d;
  void *kv, *q, *o; int *bt, *qs, *offs, *slots;
  cudaMalloc(&kv, (nb + 1) * be * 2); cudaMemset(kv, 0, (nb + 1) * be * 2);
  cudaMalloc(&q, (size_t)c * nh * d * 2); cudaMemset(q, 0, (size_t)c * nh * d * 2);
  cudaMalloc(&o, (size_t)c * nh * d * 2);
  std::vector<int> hbt(nb); for (int i = 0; i < nb; ++i) hbt[i] = i;
  cudaMalloc(&bt, nb * 4); cudaMemcpy(bt, hbt.data(), nb * 4, cudaMemcpyHostToDevice);
  int hqs[2] = {0, c}, z = 0;
  cudaMalloc(&qs, 8); cudaMemcpy(qs, hqs, 8, cudaMemcpyHostToDevice);
  cudaMalloc(&offs, 4); cudaMemcpy(offs, &z, 4, cudaMemcpyHostToDevice);
  cudaMalloc(&slots, 4); cudaMemcpy(slots, &z, 4, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) {
    int rc = hy::attn_tc_prefill(q, nh * d, c, 1, qs, offs, slots, c, nh, nh, d, bt, nb, kv, be,
                                 0.088f, o, nh * d, 0);
    if (rc) { printf("rc %d %s\n", rc, hy::get_last_error()); return 1; }
  }
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it)
    hy::attn_tc_prefill(q, nh * d, c, 1, qs, offs, slots, c, nh, nh, d, bt, nb, kv, be, 0.088f, o, nh * d, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("avg %.1f us  (%.0f TF/s)\n", ms * 1000 / 20, 4.0 * d * nh * (double)c * (c + 1) / 2 / (ms / 20 * 1e-3) / 1e12);
  unsigned long long tr[8][64];
  cudaMemcpyFromSymbol(tr, hy::g_atrace, sizeof(tr));
  unsigned long long t0 = tr[0][0];
  const char* names[] = {"kv_issue", "kv_full(MMA)", "PV0 issue", "PV1 issue", "sm0 S seen", "sm0 P done", "sm0 O seen"};
  for (int e = 0; e < 7; ++e) {
    printf("%-14s", names[e]);
    for (int j = 0; j < 4; ++j) printf(" %8lld", (long long)(tr[e][j] - t0));
    printf("\n");
  }
  return 0;
}
