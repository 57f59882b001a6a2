#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cpa8(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
// mode 0: chain + STS + syncwarp; mode 1: + cp.async issue per iter; mode 2: + cp.async, no syncwarp
__global__ void k(const double* g, double* out, int reps, long long* cyc, int mode) {
  __shared__ double4 ps[2][32];
  __shared__ double ring[8][32];
  const int lane = threadIdx.x;
  ps[0][lane] = make_double4(1e-9 * lane, 2e-9, 3e-9, 0);
  ps[1][lane] = ps[0][lane];
  __syncwarp();
  double x = 1, y = 2, z = 3;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode >= 1) { cpa8(&ring[r & 7][lane], g + ((r * 32 + lane) & 0xfffff)); asm volatile("cp.async.commit_group;"); asm volatile("cp.async.wait_group 6;" ::: "memory"); }
    ps[(r + 1) & 1][lane] = make_double4(1e-9 * lane, 2e-9 * r, 3e-9, 0);
    if (mode != 2) __syncwarp();
    const double4* pc = ps[r & 1];
#pragma unroll
    for (int i = 0; i < 32; ++i) { double4 p = pc[i]; x = __dsub_rn(x, p.x); y = __dsub_rn(y, p.y); z = __dsub_rn(z, p.z); }
    if (mode != 2) __syncwarp();
  }
  cyc[0] = clock64() - t0; out[0] = x + y + z;
}
int main() {
  double *o, *g; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); cudaMalloc(&g, 8 << 20); cudaMemset(g, 0, 8 << 20);
  long long h; int reps = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<1, 32>>>(g, o, reps, c, mode); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %.2f cycles/element\n", mode, h / (32.0 * reps));
  }
}
