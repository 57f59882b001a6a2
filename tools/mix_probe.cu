// Instruction-mix probe for the K1 pair loop: achievable FP64-pipe rate when
// DFMA/DMUL/DADD are mixed with MUFU.RSQ64H, integer min/max and shared
// loads in the proportions of the fast pair evaluation (16 FP64 : 1 MUFU :
// 2 IMNMX : 2 LDS).  Prints FP64 warp-instructions per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int MODE>
__global__ void __launch_bounds__(256) mix(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  double r = 1.5 + threadIdx.x * 1e-9;
  unsigned sink = 0;
  unsigned iv[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE >= 1 && (k & 1)) x[k] = x[k] * a;  // DMUL share
        else x[k] = fma(x[k], a, b);
      }
    }
    const double q = __hiloint2double(__double2hiint(r) + (i & 0xff), __double2loint(r));
    if (MODE == 2) {  // one MUFU.RSQ64H per 16 FP64
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
      sink ^= __double2hiint(y) ^ __double2loint(y);
    }
    if (MODE == 3) {  // FP32 MUFU.RSQ on the high word (integer re-bias both ways)
      const float f = __int_as_float(__double2hiint(q) * 8 - 0xC0000000);
      float g;
      asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(f));
      const int gi = __float_as_int(g);
      sink ^= ((gi >> 3) + 0x38000000) ^ (gi << 29);
    }
    if (MODE == 5 || MODE == 6) {  // 4 independent IMAD (5) or LOP3 (6) per 16 FP64
#pragma unroll
      for (int k = 0; k < 4; ++k) iv[k] = MODE == 5 ? iv[k] * 3u + (unsigned)i : iv[k] ^ ((unsigned)i + k);
    }
    if (MODE == 7) {  // 4 LDS per 16 FP64
      __shared__ double sh[256];
      sh[threadIdx.x] = q;
      double acc2 = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc2 += sh[(threadIdx.x + 32 * k + i) & 255];
      sink ^= __double2hiint(acc2);
    }
    if (MODE == 4) {  // two MUFU.RSQ64H per 16 FP64
      double y, z;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(q * 1.0));
      sink ^= __double2hiint(y) ^ __double2hiint(z);
    }
  }
  double s = sink + iv[0] + iv[1] + iv[2] + iv[3];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int sms, double* d) {
  const int iters = 20000, blocks = sms * 8;
  mix<MODE><<<blocks, 256>>>(d, 10, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<MODE><<<blocks, 256>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warps = blocks * 8.0;
  const double fp64_per_iter = 16 + (MODE == 4 ? 1 : 0);
  const double instr = warps * iters * fp64_per_iter;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-34s %.3f FP64 warp-instr / clk / SM (%.2f TFLOP/s DFMA-equiv), %.3f ms\n", name,
         instr / cycles / sms, instr * 32 * 2 / (ms * 1e-3) / 1e12, ms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  CK(cudaMalloc(&d, sizeof(double) * sms * 8 * 256));
  run<0>("DFMA only", sms, d);
  run<1>("DFMA + DMUL (1:1)", sms, d);
  run<2>("+ 1 MUFU.RSQ64H per 16", sms, d);
  run<3>("+ 1 f32 MUFU.RSQ (int re-bias)", sms, d);
  run<4>("+ 2 MUFU.RSQ64H per 16", sms, d);
  run<5>("+ 4 independent IMAD per 16", sms, d);
  run<6>("+ 4 independent LOP3 per 16", sms, d);
  return 0;
}
