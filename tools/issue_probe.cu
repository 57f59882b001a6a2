// Marginal cost of non-FP64 instructions on FP64 throughput (sm_100a):
// 16 independent DFMA/DMUL per iteration plus 4 independent instructions of
// one kind; reports FP64 warp-instr/clk/SM.  Drives the K1 pair-loop design
// (which helper ops are "free" next to a saturated FP64 pipe).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/issue_probe tools/issue_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

enum { NONE, IADD, LOP, SHF, LEA, IMADSHL, IMNMX, IMUL, FADD, FMUL, MUFU32, MUFU64, LDS, SEL, NKIND };
static const char* kName[] = {"none", "iadd3", "lop3", "shf.l", "lea", "imad.shl", "imnmx",
                              "imad", "fadd", "fmul", "mufu.rsq f32", "mufu.rsq64h", "lds.64",
                              "sel"};

template <int K>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double a, double b) {
  __shared__ double sh[256];
  sh[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  unsigned v[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  float f[4] = {1.f + threadIdx.x, 2.f, 3.f, 4.f};
  double dv[4] = {1.0 + threadIdx.x, 2.0, 3.0, 4.0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = (k & 1) ? x[k] * a : fma(x[k], a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned s = (unsigned)i + k;
      if (K == IADD) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[k]) : "r"(s));
      if (K == LOP) asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[k]) : "r"(s));
      if (K == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(v[k]) : "r"(s), "r"(k + 1));
      if (K == LEA) v[k] = (v[k] << 3) + s;
      if (K == IMADSHL) asm volatile("shl.b32 %0, %0, 3;" : "+r"(v[k]));
      if (K == IMNMX) asm volatile("min.s32 %0, %0, %1;" : "+r"(v[k]) : "r"(s));
      if (K == IMUL) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(v[k]) : "r"(s));
      if (K == FADD) asm volatile("add.f32 %0, %0, %1;" : "+f"(f[k]) : "f"((float)k));
      if (K == FMUL) asm volatile("mul.f32 %0, %0, %1;" : "+f"(f[k]) : "f"(1.0000001f));
      if (K == MUFU32) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[k]));
      if (K == MUFU64) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(dv[k]));
      if (K == LDS) dv[k] = sh[(threadIdx.x + 32 * k + i) & 255];
      if (K == SEL) v[k] = (s & 1) ? v[k] : s;
    }
  }
  double s = v[0] + v[1] + v[2] + v[3] + f[0] + f[1] + f[2] + f[3] + dv[0] + dv[1] + dv[2] + dv[3];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(int sms, double* d) {
  const int iters = 20000, blocks = sms * 8;
  probe<K><<<blocks, 256>>>(d, 10, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<K><<<blocks, 256>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double instr = blocks * 8.0 * iters * 16;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("16 FP64 + 4 x %-14s %.3f FP64 warp-instr/clk/SM  (%.3f ms)\n", kName[K],
         instr / cycles / sms, ms);
}

template <int K>
void all(int sms, double* d) {
  run<K>(sms, d);
  if constexpr (K + 1 < NKIND) all<K + 1>(sms, d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  CK(cudaMalloc(&d, sizeof(double) * sms * 8 * 256));
  all<0>(sms, d);
  return 0;
}
