// greedy_predict.cuh — the speculative pipeline's predictor step as ONE
// thread-block-cluster kernel (included by greedy_spec.cu):
//
//   insert(k)       the exact row append for c_k (rbf.cpp:71-100 /
//                   greedy.cpp:86-112): column, right-looking forward
//                   substitution in the reference's per-row order, the y_k
//                   chain, the pivot test, the row scattered into L;
//   fast_solve(k+1) the predictor's approximate alpha = L^-T y (FMA, any
//                   summation order) on the grown factor.
//
// Why a cluster.  Both passes stream the whole factor (k^2/2 doubles, 64 MB
// at k = 4000); one SM streams it at only ~30-40 GB/s (too few bytes in
// flight), which made the single-CTA insert + solve ~4.5 ms per step, the
// pipeline's bottleneck.  Here C CTAs (one per SM, co-scheduled by the
// cluster launch, so they may wait on one another) share the work:
//
//   * rows / columns are cut into panels of 32; panel q belongs to CTA
//     q % C, warp (q / C) % NW of it;
//   * a panel's owner brings its rows up to date with every published panel
//     (in ascending order -- each row receives the reference's subtractions
//     in ascending m), solves the 32 x 32 diagonal block in one warp (lane t
//     divides, a shuffle broadcasts, the lanes below subtract) and PUBLISHES
//     its 32 values: remote stores into every CTA's copy (DSMEM), then a
//     release increment of every CTA's panel counter;
//   * waiting warps spin on their own CTA's counter (acquire), and prefetch
//     the L block of the panel they wait for into registers meanwhile.
//
// The backward (fast) pass mirrors it from the last panel down with
// x-values.  Exactness of the forward pass: every s_j still sees
// s_j -= L_jm * r_m for m = 0, 1, ..., j-1 in that order and r_j = s_j / L_jj
// through the same correctly rounded reciprocal sequence, so the row, y_k
// and the pivot are bit-identical to insert_row / the reference.
#pragma once

#include "greedy_dev.cuh"

namespace imb {
namespace pred {

constexpr int kC = 8;     // CTAs per cluster (portable)
constexpr int kT = 512;   // threads per CTA
constexpr int kNW = kT / 32;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(out)
               : "r"(gdev::smem_addr(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_remote(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_remote_i(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t addr, uint32_t v) {
  asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(v)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_local(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(gdev::smem_addr(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void fence_cluster() {
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}

// lane 0 spins until the CTA's counter reaches `want`, then the warp proceeds
__device__ __forceinline__ void wait_count(const uint32_t* counter, uint32_t want) {
  if ((threadIdx.x & 31) == 0)
    while (ld_acquire_local(counter) < want) __nanosleep(32);
  __syncwarp();
}

// The cluster's shared state (one per CTA).
struct Smem {
  uint32_t fcount;        // forward panels published
  uint32_t bcount;        // backward panels published
  int node, exact, ok;    // broadcast by rank 0
  double yk[3], dkk[2];   // y_k and (L_kk, 1/L_kk), broadcast by rank 0
  double D[32][33];       // diagonal block of the panel being solved here
};

}  // namespace pred
}  // namespace imb
