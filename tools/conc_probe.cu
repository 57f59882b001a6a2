// How many independent single-CTA kernels on separate streams run at once?
// Each kernel spins for `ms` milliseconds on %globaltimer (no inter-kernel waits).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void spin(unsigned long long ns, int* started) {
  unsigned long long t0; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) atomicAdd(started, 1);
  for (;;) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); if (t - t0 > ns) break; }
}
int main(int argc, char** argv) {
  int N = argc > 1 ? atoi(argv[1]) : 32;
  int threads = argc > 2 ? atoi(argv[2]) : 64;
  std::vector<cudaStream_t> s(N);
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  spin<<<1, threads, 0, s[0]>>>(1000, d); cudaDeviceSynchronize();
  cudaEventRecord(a, 0); cudaDeviceSynchronize();
  for (int i = 0; i < N; ++i) spin<<<1, threads, 0, s[i]>>>(20000000ull, d);  // 20 ms each
  for (int i = 0; i < N; ++i) cudaStreamSynchronize(s[i]);
  cudaEventRecord(b, 0); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("N=%d streams, 20 ms kernels: total %.1f ms -> ~%.1f concurrent (%s)\n", N, ms, N * 20.0 / ms,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
