// Effective SM clock under a single-warp dependent FP64 chain (the exact
// backward-substitution regime): clock64 cycles vs %globaltimer ns.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void chain(double* out, double b, long long reps, long long* res) {
  double s = 1.0;
  long long c0 = clock64(); unsigned long long t0 = gt();
  for (long long r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 64; ++i) s = __dsub_rn(s, b);
  }
  long long c1 = clock64(); unsigned long long t1 = gt();
  out[0] = s; res[0] = c1 - c0; res[1] = (long long)(t1 - t0);
}
int main() {
  double* o; long long* r; cudaMalloc(&o, 8); cudaMalloc(&r, 16);
  for (long long reps : {1000LL, 10000LL, 100000LL, 1000000LL, 3000000LL}) {
    chain<<<1, 32>>>(o, 1e-9, reps, r); cudaDeviceSynchronize();
    long long h[2]; cudaMemcpy(h, r, 16, cudaMemcpyDeviceToHost);
    printf("reps %lld: %.2f cycles/op, %.3f ns/op, effective %.0f MHz, %.1f ms\n", reps,
           (double)h[0] / (reps * 64.0), (double)h[1] / (reps * 64.0), h[0] * 1e3 / (double)h[1], h[1] / 1e6);
  }
}
