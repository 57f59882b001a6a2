// greedy_sweep.cuh — the exact interpolant of the greedy residual sweep
// (greedy.cpp:126-134 -> rbf.cpp:195-203), shared by k_sweep (greedy.cu) and
// k_spec_sweep (greedy_spec.cu).
//
// One CTA = 3 warps x 32 surface points.  The reference fixes only the ORDER
// OF THE SUM f_p = sum_m alpha_m * phi_pm (insertion order m, one rounding
// per product and per add); the phi_pm themselves are independent.  So the
// work is split by stage instead of by point:
//   stage A  (all 3 warps)  phi for a tile of kSwC controls x 32 points: warp
//            q evaluates controls q, q+3, ... of the tile (lane = point, the
//            control's record is a broadcast shared-memory read), four
//            controls per batch through the staged exact pair arithmetic
//            (xt::, common.cuh), and stores phi[c][lane];
//   stage B  (warp q = axis q)  f_q[lane] += alpha_q[c] * phi[c][lane] for
//            c = 0..cnt-1 in order: the three ordered sums of a point run in
//            three different warps.
// Stage B of tile i-1 and stage A of tile i share one barrier interval (phi
// double-buffered, control records triple-buffered), so the latency-bound
// ordered adds overlap the throughput-bound pair evaluation.  Against one
// point per thread (round 1: 2 warps per 64 points, 16 % FP64-pipe activity at
// N_s = 10k) a 10k-point surface now spreads over 313 CTAs / 939 warps.
#pragma once

#include "common.cuh"

namespace imb {
namespace gsw {

constexpr int kT = 96;  // threads per CTA (3 warps)
constexpr int kP = 32;  // surface points per CTA
constexpr int kC = 48;  // controls per tile (16 per warp)

struct Smem {
  double ctl[3][kC][6];  // cx cy cz ax ay az
  double phi[2][kC][kP];
  double f[3][kP];
};

// phi of NCL controls (local indices js into a staged tile) at one point:
// the first four stages of exact_eval (common.cuh), nothing summed.
// KIND < 0: full-range sqrt / division and the runtime basis switch.
template <int KIND, int NCL>
__device__ __forceinline__ void phi_batch(const double* tile, const int (&js)[NCL], double px,
                                          double py, double pz, double (&v)[NCL],
                                          const exact::Recip& rR, int rt_kind) {
  using namespace exact;
#pragma unroll
  for (int k = 0; k < NCL; ++k) {
    const double* c = tile + 6 * js[k];
    const double2 c01 = *reinterpret_cast<const double2*>(c);
    const double cz = c[2];
    const double dx = sub(c01.x, px), dy = sub(c01.y, py), dz = sub(cz, pz);
    v[k] = add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz));
  }
  if (KIND >= 0) {
#pragma unroll
    for (int k = 0; k < NCL; ++k) v[k] = xt::sqrt_rn(v[k]);
#pragma unroll
    for (int k = 0; k < NCL; ++k) v[k] = xt::div_rn(v[k], rR);
#pragma unroll
    for (int k = 0; k < NCL; ++k) v[k] = xt::wendland<KIND < 0 ? C2 : KIND>(v[k]);
  } else {
#pragma unroll
    for (int k = 0; k < NCL; ++k)
      v[k] = wendland_rt(rt_kind, div_rcp(__dsqrt_rn(v[k]), rR));
  }
}

// f = sum_m alpha_m phi(|x - c_m| / R) over controls 0..nc-1 (insertion
// order) for the CTA's 32 points; every thread passes the point of its LANE
// (all three warps the same 32 points).  On return S.f[a][lane] holds the
// three components (a __syncthreads() has made them visible).  `run` false
// (a dead launch) skips the work but keeps the barriers uniform.
template <int KIND>
__device__ __forceinline__ void interpolant(Smem& S, const double* __restrict__ cx,
                                            const double* __restrict__ cy,
                                            const double* __restrict__ cz,
                                            const double* __restrict__ ax,
                                            const double* __restrict__ ay,
                                            const double* __restrict__ az, int nc, double R,
                                            int rt_kind, double px, double py, double pz,
                                            bool run) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const exact::Recip rR = exact::make_recip(R);
  const int ntiles = run ? (nc + kC - 1) / kC : 0;
  auto stage_tile = [&](int t) {  // tile t -> ctl[t % 3]
    const int m0 = t * kC, cnt = min(kC, nc - m0);
    double* dst = &S.ctl[t % 3][0][0];
    for (int e = threadIdx.x; e < cnt; e += kT) {
      double* d = dst + 6 * e;
      d[0] = cx[m0 + e], d[1] = cy[m0 + e], d[2] = cz[m0 + e];
      d[3] = ax[m0 + e], d[4] = ay[m0 + e], d[5] = az[m0 + e];
    }
  };
  double f = 0.0;
  if (ntiles) stage_tile(0);
  __syncthreads();
  for (int t = 0; t <= ntiles; ++t) {
    if (t + 1 < ntiles) stage_tile(t + 1);
    if (t >= 1) {  // stage B: tile t-1, axis q, strictly in control order
      const int cnt = min(kC, nc - (t - 1) * kC);
      const double* al = &S.ctl[(t - 1) % 3][0][3 + q];
      const double* ph = &S.phi[(t - 1) & 1][0][lane];
      if (KIND >= 0) {
        int c = 0;
        for (; c + 8 <= cnt; c += 8) {
          double pr[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pr[u] = exact::mul(al[6 * (c + u)], ph[kP * (c + u)]);
#pragma unroll
          for (int u = 0; u < 8; ++u) f = exact::add(f, pr[u]);
        }
        for (; c < cnt; ++c) f = exact::add(f, exact::mul(al[6 * c], ph[kP * c]));
      } else {
        for (int c = 0; c < cnt; ++c) {  // rbf.cpp:199: zero terms are skipped
          const double phi = ph[kP * c];
          if (phi != 0.0) f = exact::add(f, exact::mul(al[6 * c], phi));
        }
      }
    }
    if (t < ntiles) {  // stage A: tile t, controls q, q+3, ... four per batch
      const int cnt = min(kC, nc - t * kC);
      const double* tile = &S.ctl[t % 3][0][0];
      double* ph = &S.phi[t & 1][0][lane];
#pragma unroll 1
      for (int b = q; b < cnt; b += 12) {
        const int js[4] = {b, min(b + 3, cnt - 1), min(b + 6, cnt - 1), min(b + 9, cnt - 1)};
        double v[4];
        phi_batch<KIND, 4>(tile, js, px, py, pz, v, rR, rt_kind);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (b + 3 * u < cnt) ph[kP * (b + 3 * u)] = v[u];
      }
    }
    __syncthreads();
  }
  S.f[q][lane] = f;
  __syncthreads();
}

}  // namespace gsw
}  // namespace imb
