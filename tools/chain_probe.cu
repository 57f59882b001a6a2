// Micro-benchmarks of the exact backward-chain inner loop shape.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain3_reg(double* out, double a, double b, double c, int reps, long long* cyc) {
  double x = 1, y = 2, z = 3;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) { x = __dsub_rn(x, a); y = __dsub_rn(y, b); z = __dsub_rn(z, c); }
  }
  cyc[0] = clock64() - t0; out[0] = x + y + z;
}
__global__ void chain3_smem(double* out, int reps, long long* cyc, int sync) {
  __shared__ double4 ps[32];
  ps[threadIdx.x] = make_double4(1e-9 * threadIdx.x, 2e-9, 3e-9, 0);
  __syncwarp();
  double x = 1, y = 2, z = 3;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) { double4 p = ps[i]; x = __dsub_rn(x, p.x); y = __dsub_rn(y, p.y); z = __dsub_rn(z, p.z); }
    if (sync) { __syncwarp(); ps[threadIdx.x] = make_double4(x * 1e-20, y * 1e-20, z * 1e-20, 0); __syncwarp(); }
  }
  cyc[0] = clock64() - t0; out[0] = x + y + z;
}
__global__ void chain1_smem(double* out, int reps, long long* cyc) {
  __shared__ double ps[32];
  ps[threadIdx.x] = 1e-9 * threadIdx.x;
  __syncwarp();
  double x = 1;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x = __dsub_rn(x, ps[i]);
  }
  cyc[0] = clock64() - t0; out[0] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); long long h;
  int reps = 10000;
  chain3_reg<<<1, 32>>>(o, 1e-9, 2e-9, 3e-9, reps, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("3 chains, reg operands: %.2f cycles/element\n", h / (32.0 * reps));
  chain3_smem<<<1, 32>>>(o, reps, c, 0); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("3 chains, smem double4 operands: %.2f cycles/element\n", h / (32.0 * reps));
  chain3_smem<<<1, 32>>>(o, reps, c, 1); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("3 chains, smem + sync/STS per 32: %.2f cycles/element\n", h / (32.0 * reps));
  chain1_smem<<<1, 32>>>(o, reps, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1 chain, smem operand: %.2f cycles/element\n", h / (32.0 * reps));
  chain3_reg<<<1, 1>>>(o, 1e-9, 2e-9, 3e-9, reps, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("3 chains, reg operands, 1 thread: %.2f cycles/element\n", h / (32.0 * reps));
}
