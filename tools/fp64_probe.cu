// FP64 microbenchmarks for the roofline denominators of the pair-evaluation
// kernels: DFMA throughput (FP64 vector peak), dependent DADD latency (the
// exact backward-substitution chain), and the accuracy of MUFU.RSQ64H + one
// Newton step used by the fast-mode distance.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dadd_chain(double* out, const double* p, int n, int reps, long long* cyc) {
  double s = p[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 16
    for (int i = 0; i < n; ++i) s = __dsub_rn(s, p[i & 15]);
  }
  long long t1 = clock64();
  out[0] = s;
  cyc[0] = t1 - t0;
}

__global__ void dadd_chain_reg(double* out, double a, double b, int reps, long long* cyc) {
  double s = a;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 64; ++i) s = __dsub_rn(s, b);
  }
  long long t1 = clock64();
  out[0] = s;
  cyc[0] = t1 - t0;
}

__global__ void ddiv_chain(double* out, double a, double b, int reps, long long* cyc) {
  double s = a;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) s = __ddiv_rn(s, b);
  }
  long long t1 = clock64();
  out[0] = s;
  cyc[0] = t1 - t0;
}

__device__ __forceinline__ double rsq64h(double q) {
  double y;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo,hi}, %1;\n\t"
      "rsqrt.approx.ftz.f64 %0, %1;\n\t}" : "=d"(y) : "d"(q));
  return y;
}

__global__ void rsq_acc(const double* q, double* err0, double* err1, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = q[i];
  double y0 = rsq64h(x);
  double t = x * y0;
  double e = fma(-t, y0, 1.0);
  double eta = fma(t, 0.5 * e, t);
  double ex = sqrt(x);
  err0[i] = fabs(t - ex) / ex;
  err1[i] = fabs(eta - ex) / ex;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* d_out; CK(cudaMalloc(&d_out, 1 << 24));
  long long* d_cyc; CK(cudaMalloc(&d_cyc, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 2000;
    dfma_peak<<<blocks, threads>>>(d_out, 10, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_peak<<<blocks, threads>>>(d_out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma_peak blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, flops / ms / 1e9);
  }
  double hp[16]; for (int i = 0; i < 16; ++i) hp[i] = 1e-3 * (i + 1);
  double* d_p; CK(cudaMalloc(&d_p, sizeof hp)); CK(cudaMemcpy(d_p, hp, sizeof hp, cudaMemcpyHostToDevice));
  long long cyc;
  dadd_chain_reg<<<1, 1>>>(d_out, 1.0, 1e-9, 1000, d_cyc); CK(cudaDeviceSynchronize());
  dadd_chain_reg<<<1, 1>>>(d_out, 1.0, 1e-9, 10000, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("dependent DSUB (reg operand): %.2f cycles/op\n", (double)cyc / (10000.0 * 64));
  dadd_chain<<<1, 1>>>(d_out, d_p, 1024, 100, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("dependent DSUB (loaded operand): %.2f cycles/op\n", (double)cyc / (1024.0 * 100));
  ddiv_chain<<<1, 1>>>(d_out, 1.0, 1.0000001, 1000, d_cyc); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("dependent DDIV: %.2f cycles/op\n", (double)cyc / (1000.0 * 16));
  // rsqrt accuracy
  int n = 1 << 20;
  double* hq = (double*)malloc(n * 8);
  srand(1);
  for (int i = 0; i < n; ++i) hq[i] = pow(10.0, -6.0 + 8.0 * rand() / (double)RAND_MAX);
  double *dq, *de0, *de1; CK(cudaMalloc(&dq, n * 8)); CK(cudaMalloc(&de0, n * 8)); CK(cudaMalloc(&de1, n * 8));
  CK(cudaMemcpy(dq, hq, n * 8, cudaMemcpyHostToDevice));
  rsq_acc<<<(n + 255) / 256, 256>>>(dq, de0, de1, n); CK(cudaDeviceSynchronize());
  double* h0 = (double*)malloc(n * 8); double* h1 = (double*)malloc(n * 8);
  CK(cudaMemcpy(h0, de0, n * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(h1, de1, n * 8, cudaMemcpyDeviceToHost));
  double m0 = 0, m1 = 0; for (int i = 0; i < n; ++i) { m0 = fmax(m0, h0[i]); m1 = fmax(m1, h1[i]); }
  printf("rsqrt.approx.f64: max rel err of q*y0 = %.3e, after 1 Newton = %.3e\n", m0, m1);
  return 0;
}
