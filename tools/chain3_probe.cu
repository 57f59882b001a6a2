#include <cstdio>
#include <cuda_runtime.h>
// lane a runs chain s -= L[e] * C[a][e] over smem arrays, 8-ahead pipelined
template <int G>
__global__ void k(double* out, int n, int reps, long long* cyc) {
  extern __shared__ double sh[];
  double* L = sh; double* C = sh + n;
  for (int j = threadIdx.x; j < 4 * n; j += 32) sh[j] = 1e-3 * ((j * 7919) % 1000) / 1000.0;
  __syncwarp();
  long long t0 = clock64();
  double s = 1.0;
  if (threadIdx.x < 3) {
    const double* cx = C + threadIdx.x * n;
    for (int r = 0; r < reps; ++r) {
      double la[G], ca[G];
#pragma unroll
      for (int u = 0; u < G; ++u) la[u] = L[u], ca[u] = cx[u];
      for (int e = 0; e < n; e += G) {
        double lnx[G], cnx[G];
#pragma unroll
        for (int u = 0; u < G; ++u) { bool ok = e + G + u < n; lnx[u] = ok ? L[e + G + u] : 0.0; cnx[u] = ok ? cx[e + G + u] : 0.0; }
#pragma unroll
        for (int u = 0; u < G; ++u) s = __dsub_rn(s, __dmul_rn(la[u], ca[u]));
#pragma unroll
        for (int u = 0; u < G; ++u) la[u] = lnx[u], ca[u] = cnx[u];
      }
    }
  }
  cyc[0] = clock64() - t0; out[threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8); long long h;
  int n = 4096, reps = 20;
  cudaFuncSetAttribute(k<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * n * 8);
  cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * n * 8);
  k<8><<<1, 32, 4 * n * 8>>>(o, n, reps, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("G=8: %.2f cycles/element  (%s)\n", h / (double)(n * reps), cudaGetErrorString(cudaGetLastError()));
  k<16><<<1, 32, 4 * n * 8>>>(o, n, reps, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("G=16: %.2f cycles/element\n", h / (double)(n * reps));
}
