#include <cstdio>
#include <cuda_runtime.h>
constexpr int G = 8;
__global__ void k(double* out, int n, int reps, long long* cyc, int lanes) {
  extern __shared__ double sh[];
  double* L = sh; double* C = sh + n + 64;
  for (int j = threadIdx.x; j < 4 * n; j += 32) sh[j] = 1e-3 * ((j * 7919) % 1000) / 1000.0;
  __syncwarp();
  long long t0 = clock64();
  double s = 1.0;
  if (threadIdx.x < lanes) {
    const double* cx = C + threadIdx.x * n;
    for (int r = 0; r < reps; ++r) {
      const int cnt = n;
      double la[G], ca[G], lb[G], cb[G];
      auto ld = [&](double* l, double* c, int e) {
#pragma unroll
        for (int u = 0; u < G; ++u) { l[u] = L[e + u]; c[u] = cx[e + u]; }
      };
      auto chain = [&](const double* l, const double* c) {
#pragma unroll
        for (int u = 0; u < G; ++u) s = __dsub_rn(s, __dmul_rn(l[u], c[u]));
      };
      ld(la, ca, 0);
      for (int e = 0; e < cnt; e += 2 * G) {
        ld(lb, cb, e + G);
        chain(la, ca);
        if (e + G >= cnt) break;
        ld(la, ca, e + 2 * G);
        chain(lb, cb);
      }
    }
  }
  cyc[0] = clock64() - t0; out[threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8); long long h;
  int n = 4096, reps = 20;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (4 * n + 256) * 8);
  for (int lanes : {1, 3}) {
    k<<<1, 32, (4 * n + 256) * 8>>>(o, n, reps, c, lanes); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("lanes=%d: %.2f cycles/element (%s)\n", lanes, h / (double)(n * reps), cudaGetErrorString(cudaGetLastError()));
  }
}
