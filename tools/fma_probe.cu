#include <cstdio>
#include <cuda_runtime.h>
// (b) s -= l*c with operands in registers (rotating), products independent of s
__global__ void kb(double* out, int reps, long long* cyc, double l0, double c0) {
  double l[8], c[8];
  for (int u = 0; u < 8; ++u) l[u] = l0 * (u + 1), c[u] = c0 / (u + 1);
  double s = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dsub_rn(s, __dmul_rn(l[u], c[u]));
#pragma unroll
    for (int u = 0; u < 8; ++u) l[u] = __dadd_rn(l[u], 1e-30);
  }
  cyc[0] = clock64() - t0; out[0] = s;
}
// (d) s -= p with p precomputed in registers, plus independent DMULs interleaved
__global__ void kd(double* out, int reps, long long* cyc, double p0) {
  double p[8], q[8];
  for (int u = 0; u < 8; ++u) p[u] = p0 * (u + 1), q[u] = p[u];
  double s = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 8; ++u) { s = __dsub_rn(s, p[u]); q[u] = __dmul_rn(q[u], 1.0000001); }
  }
  cyc[0] = clock64() - t0; out[0] = s + q[0] + q[7];
}
// (e) pure chain with 8 different register operands
__global__ void ke(double* out, int reps, long long* cyc, double p0) {
  double p[8];
  for (int u = 0; u < 8; ++u) p[u] = p0 * (u + 1);
  double s = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dsub_rn(s, p[u]);
  }
  cyc[0] = clock64() - t0; out[0] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); long long h; int reps = 20000;
  kb<<<1, 32>>>(o, reps, c, 1e-3, 2e-3); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("(b) s -= l*c regs (+8 DADD bookkeeping per 8): %.2f cycles/element\n", h / (8.0 * reps));
  kd<<<1, 32>>>(o, reps, c, 1e-6); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("(d) s -= p + independent DMUL: %.2f cycles/element\n", h / (8.0 * reps));
  ke<<<1, 32>>>(o, reps, c, 1e-6); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("(e) s -= p: %.2f cycles/element\n", h / (8.0 * reps));
  kd<<<1, 1>>>(o, reps, c, 1e-6); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("(d) 1 thread: %.2f cycles/element\n", h / (8.0 * reps));
}
