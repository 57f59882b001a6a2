// Does F2F (f64<->f32) share the FP64 pipe?  Time a DFMA stream alone, F2F
// alone, and both interleaved.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8]; float f[8];
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-9 + u, f[u] = u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE != 1) x[u] = fma(x[u], a, b);
      if (MODE >= 1) { float g = (float)x[(u + 1) & 7]; f[u] = f[u] * 0.5f + g; x[(u + 3) & 7] += (MODE == 3) ? (double)f[u] : 0.0; }
    }
  }
  double s = 0; for (int u = 0; u < 8; ++u) s += x[u] + f[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"DFMA only", "F2F.F32.F64 + FFMA only", "DFMA + F2F.F32.F64", "DFMA + F2F both ways + DADD"};
  for (int mode = 0; mode < 4; ++mode) {
    auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
    kern<<<148 * 8, 256>>>(o, 10, 0.999999, 1e-7); cudaDeviceSynchronize();
    cudaEventRecord(e0); kern<<<148 * 8, 256>>>(o, 2000, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 8.0 * 2000 * 148 * 8 * 256;
    printf("%-32s %.3f ms  (%.2f Gop/s per op-slot)\n", names[mode], ms, ops / ms / 1e6);
  }
}
