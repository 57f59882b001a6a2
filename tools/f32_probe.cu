// FP32 issue/throughput probe (sm_100a) for the FP32 evaluation mode of K1:
// FFMA vs packed FFMA2 (fma.rn.f32x2) vs MUFU (rsqrt / sqrt approx) and a
// mix resembling one FP32 pair.  Reports warp-instructions / clk / SM
// (clock64 per CTA, one wave of resident 256-thread CTAs on every SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f32_probe tools/f32_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

enum { FFMA, FFMA2, RSQ, SQRT, MIX, MIX2, NK };
static const char* kName[] = {"ffma x16", "ffma2 x16", "mufu.rsq x4 (+16 ffma)",
                              "mufu.sqrt x4 (+16 ffma)", "pair-like: 16 ffma + 1 rsq",
                              "pair-like: 8 ffma2 + 1 rsq"};
static const int kInstr[] = {16, 16, 20, 20, 17, 9};

template <int K>
__global__ void __launch_bounds__(256) probe(float* out, u64* cyc, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3f + k;
  u64 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = ((u64)__float_as_uint(1.f + k) << 32) | __float_as_uint(2.f + threadIdx.x);
  const u64 aa = ((u64)__float_as_uint(a) << 32) | __float_as_uint(a);
  const u64 bb = ((u64)__float_as_uint(b) << 32) | __float_as_uint(b);
  float m[4] = {1.f + threadIdx.x, 2.f, 3.f, 4.f};
  __syncthreads();
  const u64 t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (K == FFMA || K == RSQ || K == SQRT || K == MIX) {
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
    }
    if (K == FFMA2 || K == MIX2) {
#pragma unroll
      for (int u = 0; u < (K == FFMA2 ? 2 : 1); ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ffma2(v[k], aa, bb);
    }
    if (K == RSQ)
#pragma unroll
      for (int k = 0; k < 4; ++k) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(m[k]));
    if (K == SQRT)
#pragma unroll
      for (int k = 0; k < 4; ++k) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(m[k]));
    if (K == MIX || K == MIX2) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(m[i & 3]));
  }
  const u64 t1 = clock64();
  float s = m[0] + m[1] + m[2] + m[3];
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += __uint_as_float((unsigned)v[k]) + __uint_as_float((unsigned)(v[k] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(int sms, float* d, u64* c) {
  // exactly the resident CTAs (one wave), so the per-CTA clock span is the
  // SM's shared time
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, probe<K>, 256, 0));
  const int iters = 20000, blocks = sms * per_sm;
  probe<K><<<blocks, 256>>>(d, c, 10, 1.0000001f, 1e-9f);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  probe<K><<<blocks, 256>>>(d, c, iters, 1.0000001f, 1e-9f);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  u64* h = (u64*)malloc(blocks * 8);
  CK(cudaMemcpy(h, c, blocks * 8, cudaMemcpyDeviceToHost));
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += h[i];
  mean /= blocks;
  const double wi = 8.0 * per_sm * iters * kInstr[K];
  // wall-clock rate at the current SM clock (nvidia-smi) for cross-checking clock64
  int khz = 0;
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
  const double wall_cyc = ms * 1e-3 * khz * 1e3;
  printf("%-32s %7.3f warp-instr/clk/SM by clock64, %7.3f by events at %d MHz "
         "(%.1f clock64 cycles/iter/CTA, %d CTAs/SM)\n", kName[K], wi / mean, wi / wall_cyc,
         khz / 1000, mean / iters, per_sm);
  free(h);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* d;
  u64* c;
  CK(cudaMalloc(&d, sms * 8 * 256 * 4));
  CK(cudaMalloc(&c, sms * 8 * 8));
  run<FFMA>(sms, d, c);
  run<FFMA2>(sms, d, c);
  run<RSQ>(sms, d, c);
  run<SQRT>(sms, d, c);
  run<MIX>(sms, d, c);
  run<MIX2>(sms, d, c);
  return 0;
}
