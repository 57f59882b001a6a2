// greedy_sweep.cuh — the exact interpolant of the greedy residual sweep
// (greedy.cpp:126-134 -> rbf.cpp:195-203), shared by k_sweep (greedy.cu) and
// k_spec_sweep (greedy_spec.cu).
//
// One CTA = 8 warps x 32 surface points.  The reference fixes only the ORDER
// OF THE SUM f_p = sum_m alpha_m * phi_pm (insertion order m, one rounding
// per product and per add); the phi_pm themselves are independent.  So the
// work is split by stage instead of by point:
//   stage A  (all 8 warps)  phi for a tile of kC = 72 controls x 32 points
//            (lane = point, the control's record is a broadcast shared-memory
//            read), four or six controls per batch through the staged exact
//            pair arithmetic (xt::, common.cuh), stored as phi[c][lane]; warps
//            3-7 take 12 controls each (two batches of six), warps 0-2 only 4
//            each, because they also run
//   stage B  (warp q = axis q, q < 3)  f_q[lane] += alpha_q[c] * phi[c][lane]
//            for c = 0..cnt-1 in order: the three ordered sums of a point run
//            in three different warps (on three different SM sub-partitions).
//            12 x 24 = 288 FP64 instructions per A-only warp and tile against
//            4 x 24 + 72 x 2 = 240 (latency-bound adds) per axis warp: the
//            warps reach the tile barrier together.
// Stage B of tile i-1 and stage A of tile i share one barrier interval (phi
// double-buffered, control records triple-buffered), so the latency-bound
// ordered adds overlap the throughput-bound pair evaluation.  Against one
// point per thread (round 1: 2 warps per 64 points, 16 % FP64-pipe activity at
// N_s = 10k) a 10k-point surface now spreads over 313 CTAs / 2504 warps.
#pragma once

#include "common.cuh"

namespace imb {
namespace gsw {

constexpr int kW = 8;        // warps per CTA
constexpr int kT = 32 * kW;  // threads per CTA
constexpr int kP = 32;       // surface points per CTA
constexpr int kAxisC = 4;    // stage-A controls of an axis warp (warps 0-2) per tile
constexpr int kPlainC = 12;  // stage-A controls of the other warps per tile
constexpr int kC = 3 * kAxisC + (kW - 3) * kPlainC;  // controls per tile (72)

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
    if (t >= 1 && q < 3) {  // stage B: tile t-1, axis q, strictly in control order
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
    if (t < ntiles) {  // stage A: tile t, this warp's controls, four per batch
      const int cnt = min(kC, nc - t * kC);
      const double* tile = &S.ctl[t % 3][0][0];
      double* ph = &S.phi[t & 1][0][lane];
      if (q < 3) {  // axis warp: one batch of four
        const int b = kAxisC * q;
        if (b < cnt) {
          const int js[4] = {b, min(b + 1, cnt - 1), min(b + 2, cnt - 1), min(b + 3, cnt - 1)};
          double v[4];
          phi_batch<KIND, 4>(tile, js, px, py, pz, v, rR, rt_kind);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (b + u < cnt) ph[kP * (b + u)] = v[u];
        }
      } else {  // two batches of six (six independent dependency chains per lane)
        const int b0 = 3 * kAxisC + kPlainC * (q - 3);
#pragma unroll 1
        for (int b = b0; b < min(cnt, b0 + kPlainC); b += 6) {
          int js[6];
#pragma unroll
          for (int u = 0; u < 6; ++u) js[u] = min(b + u, cnt - 1);
          double v[6];
          phi_batch<KIND, 6>(tile, js, px, py, pz, v, rR, rt_kind);
#pragma unroll
          for (int u = 0; u < 6; ++u)
            if (b + u < cnt) ph[kP * (b + u)] = v[u];
        }
      }
    }
    __syncthreads();
  }
  if (q < 3) S.f[q][lane] = f;
  __syncthreads();
}

}  // namespace gsw
}  // namespace imb
