// greedy_spec.cu — the exact greedy level as a speculative pipeline
// (north-star b, c; reference greedy_level, greedy.cpp:60-170).
//
// Why.  Step k of the reference re-solves L^T x = y from scratch
// (greedy.cpp:106-111 -> rbf.cpp:114-120): ~k^2/2 dependent subtractions
// whose order fixes alpha's bits, so one step is latency-bound (8-cycle DSUB)
// and a capped 5000-point level is ~2e10 dependent subtractions (~85 s at the
// floor).  The chain of step k+1 needs only L's rows 0..k, i.e. the selection
// c_k -- not alpha_k.  So the selection is PREDICTED from an approximate
// alpha (a blocked FMA triangular solve + an FMA sweep, both cheap and
// parallel) and the next rows / chains start at once, many steps deep, each
// chain on its own SM.  Every step's exact chain and exact sweep still run,
// in the reference's arithmetic; the exact sweep of step k CONFIRMS the
// prediction of c_k.  A wrong prediction (rare except at near-ties) rolls the
// speculative steps back and restarts them from the exact c_k.  Control
// indices, alpha, residual and convergence record are therefore bit-identical
// to the non-speculative engine (greedy.cu) and to the reference.
//
// Step k (k controls c_0..c_{k-1} selected):
//   chain(k)   alpha_k = L_k^-T y_k, exact order           [server CTA k % S]
//   sweep(k)   residual with alpha_k, record[k-1], argmax
//              c_k (or stop), confirm the prediction        [main stream]
//   fsolve(k) + fsweep(k)   predicted c_k                   [predictor stream]
//   insert(k)  L row k, y_k for c_k (exact if sweep(k) already decided,
//              else the prediction)                          [predictor stream]
// insert(k) enables chain(k+1).  Chains run in a persistent kernel of S CTAs
// (one per SM, they spin on per-step flags); alpha_k goes to slot k % S, which
// chain(k+S) reuses once sweep(k) has consumed it.
//
// Protocol words (device): state[k] = EMPTY / predicted node / node|EXACT
// (atomics decide whether insert(k) or sweep(k) came first); ins_ep[k] /
// chain_ep[k] = epoch in which insert(k) / chain(k) completed; ctl.epoch is
// bumped by each rollback and every kernel launched for an older epoch is a
// no-op; ctl.abort stops speculative work between a misprediction and its
// rollback.  Every spin loop has a watchdog (status kStatusWatchdog).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "greedy.hpp"
#include "greedy_dev.cuh"
#include "greedy_predict.cuh"
#include "greedy_sweep.cuh"

namespace imb {

using gdev::better;
using gdev::colstart;
using gdev::globaltimer;
using gdev::ld_volatile;

namespace {

constexpr int kEmpty = -1;
constexpr int kExactBit = 1 << 30;
constexpr int kNodeMask = kExactBit - 1;
constexpr int kSweepT = gsw::kT;  // exact sweep CTA: 8 warps x 32 points (greedy_sweep.cuh)
constexpr int kFastT = 128;      // predictor sweep CTA
constexpr int kFastP = 2;        // points per predictor-sweep thread
constexpr int kFastTile = 256;


__device__ __forceinline__ int4 ld_volatile4(const int* p) {
  int4 w;
  asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(p)
               : "memory");
  return w;
}

// per-step timeline (diagnostics, IMB_SPEC_LOG): tl[e * (cap + 1) + k]
enum : int { kTlInsB, kTlInsE, kTlSolveB, kTlSolveE, kTlFsweepE, kTlSweepB, kTlSweepE,
             kTlChainB, kTlChainE, kTlCount };
__device__ __forceinline__ void tl_mark(const SpecView& v, int e, int k) {
  v.tl[(size_t)e * (v.cap + 1) + k] = globaltimer();
}

__device__ __forceinline__ void st_volatile(int* p, int v) {
  asm volatile("st.volatile.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// uniform "is this launch still current" test, decided by thread 0
__device__ __forceinline__ bool launch_live(const SpecCtl* c, int ep) {
  __shared__ int s_live;
  if (threadIdx.x == 0) {
    const int4 w = ld_volatile4(&c->epoch);
    s_live = w.x == ep && w.y == 0 && w.w == 0;  // epoch, abort, -, done
  }
  __syncthreads();
  return s_live != 0;
}

__device__ void host_publish(const SpecView& v) {
  // mirror of the few words the host loop polls (mapped pinned memory)
  SpecHost* h = v.host;
  h->conf = v.ctl->conf;
  h->abort = v.ctl->abort;
  h->abort_step = v.ctl->abort_step;
  h->status = v.ctl->status;
  __threadfence_system();
  h->done = v.ctl->done;
  __threadfence_system();
}

__device__ void finish(const SpecView& v, int status, int final_step) {
  SpecCtl* c = v.ctl;
  c->status = status;
  c->final_step = final_step;
  __threadfence();
  c->done = 1;
  __threadfence();
  host_publish(v);
}

// ---------------------------------------------------------------------------
// init / rollback
// ---------------------------------------------------------------------------
__global__ void k_spec_init(SpecView v) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int i = t; i < v.n; i += stride) v.selstep[i] = INT_MAX;
  for (int k = t; k <= v.cap; k += stride) {
    v.state[k] = k == 0 ? (0 | kExactBit) : kEmpty;  // c_0 = surface node 0 (greedy.cpp:115)
    v.ins_ep[k] = -1, v.chain_ep[k] = -1, v.ins_node[k] = -1, v.ins_fail[k] = 0;
    v.pred_node[k] = -1, v.pred2_node[k] = -1, v.exact_node[k] = -1;
    v.pred_gap[k] = -1.0, v.exact_gap[k] = -1.0;
    for (int e = 0; e < kTlCount; ++e) v.tl[(size_t)e * (v.cap + 1) + k] = 0;
  }
  if (t == 0) {
    SpecCtl c{};
    c.abort_step = INT_MAX;
    c.rb_step = 0;
    c.status = kStatusRunning;
    *v.ctl = c;
    SpecHost h{};
    *v.host = h;
  }
}

// mispredicted step r: drop every speculative step >= r (c_r is already
// EXACT in state[r]), re-stamp the surviving inserts, bump the epoch.
__global__ void k_spec_rollback(SpecView v) {
  __shared__ int r, ep;
  if (threadIdx.x == 0) r = v.ctl->abort_step, ep = v.ctl->epoch + 1;
  __syncthreads();
  for (int k = threadIdx.x; k <= v.cap; k += blockDim.x) {
    if (k >= r) {
      const int node = v.ins_node[k];
      if (node >= 0 && v.selstep[node] == k) v.selstep[node] = INT_MAX;
      v.ins_node[k] = -1, v.ins_ep[k] = -1, v.ins_fail[k] = 0;
      if (k > r) v.state[k] = kEmpty, v.pred_node[k] = -1;
    } else {
      v.ins_ep[k] = ep;
    }
    if (k > r) v.chain_ep[k] = -1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    SpecCtl* c = v.ctl;
    c->rb_step = r;
    c->rollbacks += 1;
    __threadfence();
    c->epoch = ep;
    __threadfence();
    c->abort_step = INT_MAX;
    c->abort = 0;
    __threadfence();
    host_publish(v);
  }
}

// ---------------------------------------------------------------------------
// insert(k): the row append for c_k (exact if known, else predicted)
// ---------------------------------------------------------------------------
template <int NR, int T>
__global__ void __launch_bounds__(T) k_spec_insert(SpecView v, int k, int ep) {
  extern __shared__ double sh[];
  __shared__ int s_node, s_exact;
  if (threadIdx.x == 0) atomicAdd(&v.ctl->probe[0], 1), v.host->seen[0] = k, tl_mark(v, kTlInsB, k);
  if (!launch_live(v.ctl, ep)) return;
  if (threadIdx.x == 0) {
    int node = -1, exact = 0;
    if (k == 0 || v.ins_ep[k - 1] == ep) {
      int cur = ld_volatile(&v.state[k]);
      if (cur == kEmpty) {
        const int pn = v.pred_node[k];
        if (pn >= 0) {
          const int old = atomicCAS(&v.state[k], kEmpty, pn);
          cur = old == kEmpty ? pn : old;
        }
      }
      if (cur != kEmpty) {
        exact = (cur & kExactBit) != 0;
        node = cur & kNodeMask;
      }
    }
    s_node = node, s_exact = exact;
    if (k == 0) v.ctl->t0 = globaltimer();
  }
  __syncthreads();
  const int node = s_node;
  if (node < 0) return;  // no prediction (no candidate left): sweep(k) decides
  gdev::InsertIO io{v.px, v.py, v.pz, v.tx, v.ty, v.tz, v.cx, v.cy, v.cz, v.Lt, (size_t)v.cap,
                    v.diag, v.yx, v.yy, v.yz, v.kind, v.R, v.rr_global};
  const gdev::AppendOut a = gdev::insert_row<NR, T>(io, k, node, nullptr, 1.0, sh);
  const bool ok = a.ok;
  const double pivot = a.pivot;
  if (threadIdx.x == 0) {
    v.ins_node[k] = node;
    v.pivot[k] = pivot;
    tl_mark(v, kTlInsE, k);
    if (ok) {
      v.cidx[k] = node;
      v.cx[k] = v.px[node], v.cy[k] = v.py[node], v.cz[k] = v.pz[node];
      v.selstep[node] = k;
      __threadfence();
      st_volatile(&v.ins_ep[k], ep);
    } else {
      v.ins_fail[k] = 1;
      if (s_exact) {  // rbf.cpp:92 on the reference's own selection
        v.ctl->fail_node = node;
        v.ctl->fail_row = k;
        v.ctl->fail_pivot = pivot;
        finish(v, kStatusSolveError, k);
      }
      // predicted: sweep(k) tells whether c_k really is this node
    }
  }
}

// ---------------------------------------------------------------------------
// the predictor: approximate alpha_k and the predicted argmax c_k
// ---------------------------------------------------------------------------
// Blocked backward substitution with FMAs (not the reference order): block b
// of 32 rows takes the dot products of its columns' tails with the solved x
// (one warp per column), then one warp solves the 32 x 32 diagonal block.
__global__ void __launch_bounds__(1024) k_fast_solve(SpecView v, int n, int ep) {
  extern __shared__ double xs[];  // [3][cap]
  __shared__ double sb[3][32], rc[32];
  __shared__ double T[32][33];  // T[t][r] = L_{b0+r, b0+t}
  __shared__ int s_ok;
  if (threadIdx.x == 0) atomicAdd(&v.ctl->probe[1], 1), v.host->seen[1] = n, tl_mark(v, kTlSolveB, n);
  if (!launch_live(v.ctl, ep)) return;
  if (threadIdx.x == 0) s_ok = ld_volatile(&v.ins_ep[n - 1]) == ep;
  __syncthreads();
  if (!s_ok) return;
  const size_t cap = v.cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b1 = n; b1 > 0; b1 -= 32) {
    const int b0 = max(0, b1 - 32), nb = b1 - b0;
    if (warp < nb) {
      const int i = b0 + warp;
      const double* col = v.Lt + colstart(i, cap) - i;  // col[j] = L_ji
      double sx = 0.0, sy = 0.0, sz = 0.0;
      int j = b1 + lane;
      // 8 loads in flight per lane (the column walk is latency-bound otherwise)
      for (; j + 7 * 32 < n; j += 8 * 32) {
        double l[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) l[u] = col[j + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int jj = j + 32 * u;
          sx = fma(l[u], xs[jj], sx), sy = fma(l[u], xs[cap + jj], sy);
          sz = fma(l[u], xs[2 * cap + jj], sz);
        }
      }
      for (; j < n; j += 32) {
        const double l = col[j];
        sx = fma(l, xs[j], sx), sy = fma(l, xs[cap + j], sy), sz = fma(l, xs[2 * cap + j], sz);
      }
      for (int o = 16; o; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        sz += __shfl_xor_sync(0xffffffffu, sz, o);
      }
      if (lane > warp && lane < nb) T[warp][lane] = col[b0 + lane];
      if (lane == 0) {
        sb[0][warp] = v.yx[i] - sx, sb[1][warp] = v.yy[i] - sy, sb[2][warp] = v.yz[i] - sz;
        rc[warp] = v.diag[i].y;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double sx = 0.0, sy = 0.0, sz = 0.0, r = 0.0;
      if (lane < nb) sx = sb[0][lane], sy = sb[1][lane], sz = sb[2][lane], r = rc[lane];
      for (int q = nb - 1; q >= 0; --q) {
        const double xx = __shfl_sync(0xffffffffu, sx * r, q);
        const double xy = __shfl_sync(0xffffffffu, sy * r, q);
        const double xz = __shfl_sync(0xffffffffu, sz * r, q);
        if (lane < q) {
          const double l = T[lane][q];
          sx = fma(-l, xx, sx), sy = fma(-l, xy, sy), sz = fma(-l, xz, sz);
        } else if (lane == q) {
          xs[b0 + q] = xx, xs[cap + b0 + q] = xy, xs[2 * cap + b0 + q] = xz;
        }
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    v.fax[i] = xs[i], v.fay[i] = xs[cap + i], v.faz[i] = xs[2 * cap + i];
  if (threadIdx.x == 0) v.host->seen[1] = -n, tl_mark(v, kTlSolveE, n);  // diagnostics
}


// ---------------------------------------------------------------------------
// The predictor step as one cluster kernel: insert(k) + fast_solve(k + 1)
// (greedy_predict.cuh explains the panel / publish scheme).
// Dynamic shared memory: rr[cap] | xb[3][cap].
// ---------------------------------------------------------------------------
__global__ void __cluster_dims__(pred::kC, 1, 1) __launch_bounds__(pred::kT)
    k_predict(SpecView v, int k, int ep) {
  using namespace pred;
  extern __shared__ __align__(16) double dyn[];
  __shared__ Smem S;
  const size_t cap = v.cap;
  double* rr = dyn;       // [cap]: own rows' running values + every published panel
  double* xb = dyn + cap;  // [3][cap]: y staging (rank 0), then published x panels
  const uint32_t rank = ctarank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    S.fcount = 0, S.bcount = 0, S.ok = 0, S.node = -1, S.exact = 0;
  }
  cluster_sync();  // every CTA initialised before any remote write
  // ---- 0. node: exact if sweep(k) already decided, else the prediction ----
  if (rank == 0 && tid == 0) {
    int node = -1, exact = 0;
    const int4 w = ld_volatile4(&v.ctl->epoch);
    if (w.x == ep && w.y == 0 && w.w == 0 && (k == 0 || ld_volatile(&v.ins_ep[k - 1]) == ep)) {
      int cur = ld_volatile(&v.state[k]);
      if (cur == kEmpty) {
        const int pn = v.pred_node[k];
        if (pn >= 0) {
          const int old = atomicCAS(&v.state[k], kEmpty, pn);
          cur = old == kEmpty ? pn : old;
        }
      }
      if (cur != kEmpty) exact = (cur & kExactBit) != 0, node = cur & kNodeMask;
    }
    atomicAdd(&v.ctl->probe[0], 1), v.host->seen[0] = k, tl_mark(v, kTlInsB, k);
    if (k == 0) v.ctl->t0 = globaltimer();
    for (uint32_t c = 0; c < kC; ++c) {
      st_remote_i(mapa(&S.node, c), node);
      st_remote_i(mapa(&S.exact, c), exact);
    }
  }
  cluster_sync();
  const int node = S.node;
  if (node < 0) return;  // uniform: no prediction / stale launch
  // ---- 1. the new column for my rows (greedy.cpp:87-93) ----
  const int P = (k + 31) / 32;
  auto first_own = [&](int np) { return (int)rank + kC * warp < np ? (int)rank + kC * warp : np; };
  auto next_own = [&](int q) { return q + kC * kNW; };
  {
    const double px = v.px[node], py = v.py[node], pz = v.pz[node];
    const exact::Recip rR = exact::make_recip(v.R);
    for (int q = first_own(P); q < P; q = next_own(q)) {
      const int j = 32 * q + lane;
      if (j < k) {
        const double d = exact::dist(v.cx[j], v.cy[j], v.cz[j], px, py, pz);
        rr[j] = exact::wendland_rt(v.kind, exact::div_rcp(d, rR));
      }
    }
  }
  __syncwarp();
  // ---- 2. forward substitution by panels (rbf.cpp:80-87) ----
  // Staging the diagonal block into the CTA's single S.D before the panel's
  // last wait is safe: the previous user of S.D (panel q - kC, same CTA) was
  // solved before panel q - 2 was published, which this warp has waited for.
  auto stage_fwd_D = [&](int q) {
    const int m0 = 32 * q, cnt = min(32, k - m0);
    size_t c = colstart((size_t)m0, cap);
    for (int t = 0; t < cnt; ++t) {
      if (lane > t && lane < cnt) S.D[t][lane] = v.Lt[c + (lane - t)];
      c += cap - (size_t)(m0 + t);
    }
  };
  for (int q = first_own(P); q < P; q = next_own(q)) {
    const int j = 32 * q + lane;
    double s = j < k ? rr[j] : 0.0;
    if (q == 0) stage_fwd_D(q);
    for (int m = 0; m < q; ++m) {
      const int m0 = 32 * m;  // panels below the last are full
      double l[32];
      size_t c = colstart((size_t)m0, cap);
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        l[t] = j < k ? v.Lt[c + (j - m0 - t)] : 0.0;
        c += cap - (size_t)(m0 + t);
      }
      if (m == q - 1) stage_fwd_D(q);
      wait_count(&S.fcount, (uint32_t)m + 1);
#pragma unroll
      for (int t = 0; t < 32; ++t) s = exact::sub(s, exact::mul(l[t], rr[m0 + t]));
    }
    // the 32 x 32 diagonal block, then publish
    const int m0 = 32 * q, cnt = min(32, k - m0);
    const double2 dg = lane < cnt ? v.diag[j] : make_double2(1.0, 1.0);
    __syncwarp();
    for (int t = 0; t < cnt; ++t) {
      if (lane == t) s = exact::div_rcp(s, exact::Recip{dg.x, dg.y});  // r_t = s_t / L_tt
      const double r = __shfl_sync(0xffffffffu, s, t);
      if (lane > t && lane < cnt) s = exact::sub(s, exact::mul(S.D[t][lane], r));
    }
    if (lane < cnt)
      for (uint32_t c = 0; c < kC; ++c) st_remote(mapa(&rr[j], c), s);
    __syncwarp();  // orders the lanes' remote stores before lane 0's release
    if (lane == 0)
      for (uint32_t c = 0; c < kC; ++c) red_release_add(mapa(&S.fcount, c), 1u);
  }
  // ---- 3. y_k, the pivot (rbf.cpp:86-99, 107-112), rank 0 ----
  if (rank == 0) {
    wait_count(&S.fcount, (uint32_t)P);
    __syncthreads();
    for (int j = tid; j < k; j += kT)
      xb[j] = v.yx[j], xb[cap + j] = v.yy[j], xb[2 * cap + j] = v.yz[j];
    __syncthreads();
    if (tid == 0) {
      double sq = 0.0, yx = v.tx[node], yy = v.ty[node], yz = v.tz[node];
#pragma unroll 8
      for (int j = 0; j < k; ++j) {
        const double r = rr[j];
        sq = exact::add(sq, exact::mul(r, r));
        yx = exact::sub(yx, exact::mul(r, xb[j]));
        yy = exact::sub(yy, exact::mul(r, xb[cap + j]));
        yz = exact::sub(yz, exact::mul(r, xb[2 * cap + j]));
      }
      const double pivot_sq = exact::sub(1.0, sq);  // column[k] = 1.0, max_diag = 1
      const double pivot = pivot_sq > 0.0 ? __dsqrt_rn(pivot_sq) : 0.0;
      const int ok = pivot > exact::mul(1e-14, 1.0);
      double dk[2] = {pivot, 0.0}, yk[3] = {0.0, 0.0, 0.0};
      v.ins_node[k] = node;
      v.pivot[k] = pivot;
      if (ok) {
        const exact::Recip pr = exact::make_recip(pivot);
        dk[1] = pr.y;
        yk[0] = exact::div_rcp(yx, pr), yk[1] = exact::div_rcp(yy, pr), yk[2] = exact::div_rcp(yz, pr);
        v.diag[k] = make_double2(pivot, pr.y);
        v.Lt[colstart((size_t)k, cap)] = pivot;
        v.yx[k] = yk[0], v.yy[k] = yk[1], v.yz[k] = yk[2];
      } else {
        v.ins_fail[k] = 1;
        if (S.exact) {  // rbf.cpp:92 on the reference's own selection
          v.ctl->fail_node = node;
          v.ctl->fail_row = k;
          v.ctl->fail_pivot = pivot;
          finish(v, kStatusSolveError, k);
        }
      }
      for (uint32_t c = 0; c < kC; ++c) {
        st_remote_i(mapa(&S.ok, c), ok);
        for (int a = 0; a < 3; ++a) st_remote(mapa(&S.yk[a], c), yk[a]);
        st_remote(mapa(&S.dkk[0], c), dk[0]);
        st_remote(mapa(&S.dkk[1], c), dk[1]);
      }
    }
  }
  cluster_sync();
  if (!S.ok) return;  // uniform
  // ---- 4. scatter the row into the columns, publish insert(k) ----
  for (int q = first_own(P); q < P; q = next_own(q)) {
    const int j = 32 * q + lane;
    if (j < k) v.Lt[colstart((size_t)j, cap) + (k - j)] = rr[j];
  }
  __threadfence();
  cluster_sync();
  if (rank == 0 && tid == 0) {
    v.cidx[k] = node;
    v.cx[k] = v.px[node], v.cy[k] = v.py[node], v.cz[k] = v.pz[node];
    v.selstep[node] = k;
    tl_mark(v, kTlInsE, k);
    __threadfence();
    st_volatile(&v.ins_ep[k], ep);  // chain(k + 1) may start
    if (k + 1 < v.cap) tl_mark(v, kTlSolveB, k + 1);
  }
  if (k + 1 >= v.cap) return;  // no prediction is needed past the cap (uniform)
  // ---- 5. fast backward solve of L^T x = y on n = k + 1 (FMA, any order) ----
  const int n = k + 1, P2 = (n + 31) / 32;
  // own panels in decreasing order: the largest own panel first
  int qtop = first_own(P2);
  if (qtop < P2)
    while (next_own(qtop) < P2) qtop = next_own(qtop);
  for (int q = qtop; q >= 0 && q < P2; q -= kC * kNW) {
    const int i = 32 * q + lane;
    const bool live = i < n;
    // compensated (double-double) accumulation: the prediction's error then
    // comes from the rounding of the x values alone, not from the sums'
    // cancellation (which the ill-conditioned global-support systems amplify)
    double yv[3] = {0.0, 0.0, 0.0}, yl[3] = {0.0, 0.0, 0.0};
    auto sub_dd = [&](int a, double l, double x) {  // (yv, yl)[a] -= l * x
      const double ph = l * x, pl = fma(l, x, -ph);
      const double t = yv[a] - ph, bb = t - yv[a];
      const double e = (yv[a] - (t - bb)) + (-ph - bb);
      yv[a] = t;
      yl[a] += e - pl;
    };
    if (live) {
      if (i == k) yv[0] = S.yk[0], yv[1] = S.yk[1], yv[2] = S.yk[2];
      else yv[0] = v.yx[i], yv[1] = v.yy[i], yv[2] = v.yz[i];
    }
    const size_t ci = live ? colstart((size_t)i, cap) : 0;
    const int i0 = 32 * q, cnt0 = min(32, n - i0);
    auto stage_bwd_D = [&]() {  // (same single-buffer argument as the forward pass)
      for (int t = 0; t < cnt0; ++t)
        if (lane < t) S.D[t][lane] = v.Lt[colstart((size_t)(i0 + lane), cap) + (t - lane)];
    };
    if (q == P2 - 1) stage_bwd_D();
    for (int p = P2 - 1; p > q; --p) {
      const int j0 = 32 * p, cnt = min(32, n - j0);
      double l[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) l[t] = live && t < cnt ? v.Lt[ci + (j0 + t - i)] : 0.0;
      if (p == q + 1) stage_bwd_D();
      wait_count(&S.bcount, (uint32_t)(P2 - p));
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (t < cnt) {
          sub_dd(0, l[t], xb[j0 + t]);
          sub_dd(1, l[t], xb[cap + j0 + t]);
          sub_dd(2, l[t], xb[2 * cap + j0 + t]);
        }
    }
    // diagonal block, from the bottom row up
    const int cnt = cnt0;
    const double rc = !live ? 0.0 : (i == k ? S.dkk[1] : v.diag[i].y);
    __syncwarp();
    for (int t = cnt - 1; t >= 0; --t) {
      const double x0 = __shfl_sync(0xffffffffu, (yv[0] + yl[0]) * rc, t);
      const double x1 = __shfl_sync(0xffffffffu, (yv[1] + yl[1]) * rc, t);
      const double x2 = __shfl_sync(0xffffffffu, (yv[2] + yl[2]) * rc, t);
      if (lane == t) yv[0] = x0, yv[1] = x1, yv[2] = x2;
      if (lane < t) {
        const double l = S.D[t][lane];
        sub_dd(0, l, x0), sub_dd(1, l, x1), sub_dd(2, l, x2);
      }
    }
    if (live) {
      v.fax[i] = yv[0], v.fay[i] = yv[1], v.faz[i] = yv[2];
      for (uint32_t c = 0; c < kC; ++c) {
        st_remote(mapa(&xb[i], c), yv[0]);
        st_remote(mapa(&xb[cap + i], c), yv[1]);
        st_remote(mapa(&xb[2 * cap + i], c), yv[2]);
      }
    }
    __syncwarp();
    if (lane == 0)
      for (uint32_t c = 0; c < kC; ++c) red_release_add(mapa(&S.bcount, c), 1u);
  }
  cluster_sync();  // no CTA leaves while others may still write into it
  if (rank == 0 && tid == 0) {
    atomicAdd(&v.ctl->probe[1], 1), v.host->seen[1] = -n, tl_mark(v, kTlSolveE, n);
  }
}

struct Top2 {
  double v1, v2;
  int i1, i2;
};
// the two best (value, index) pairs, lowest index on ties
__device__ __forceinline__ bool beats(double v, int i, double w, int j) {
  return v > w || (v == w && i < j);
}
__device__ __forceinline__ Top2 merge2(Top2 a, Top2 b) {
  Top2 r;
  if (beats(b.v1, b.i1, a.v1, a.i1)) {
    r.v1 = b.v1, r.i1 = b.i1;
    if (beats(a.v1, a.i1, b.v2, b.i2)) r.v2 = a.v1, r.i2 = a.i1; else r.v2 = b.v2, r.i2 = b.i2;
  } else {
    r.v1 = a.v1, r.i1 = a.i1;
    if (beats(b.v1, b.i1, a.v2, a.i2)) r.v2 = b.v1, r.i2 = b.i1; else r.v2 = a.v2, r.i2 = a.i2;
  }
  return r;
}
__device__ __forceinline__ Top2 warp_top2(Top2 t) {
  for (int o = 16; o; o >>= 1) {
    Top2 u;
    u.v1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
    u.v2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
    u.i1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
    u.i2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
    t = merge2(t, u);
  }
  return t;
}

// Predicted argmax of |E|^2 over the candidates (selstep >= k) with the
// approximate alpha; FMA arithmetic, kFastP points per thread on coordinates
// pre-scaled by 1/R (q = |p - c|^2 / R^2), eta from the rsqrt-based sqrt
// with a second-order correction (fast::sqrt_pos), the support cut as a
// select.
//
// Grid-wide ticket kernels (this one and the exact sweep) never leave a block
// early: the launch-live flags can flip to dead mid-kernel (an abort / done
// raised on the other stream), so a dead block skips its work but still takes
// its ticket, and the last block -- which then also sees the launch dead (the
// flags are monotone within an epoch) -- resets the ticket and returns.
template <int KIND>
__device__ __forceinline__ double fast_phi(double eta) {
  const double u = 1.0 - eta, u2 = u * u;
  if (KIND == C0) return u2;
  if (KIND == C2) return u2 * u2 * fma(4.0, eta, 1.0);
  if (KIND == C4) return u2 * u2 * u2 * fma(fma(35.0 / 3.0, eta, 6.0), eta, 1.0);
  const double u4 = u2 * u2;
  return u4 * u4 * fma(fma(fma(32.0, eta, 25.0), eta, 8.0), eta, 1.0);
}

template <int KIND>
__global__ void __launch_bounds__(kFastT) k_fast_sweep(SpecView v, int k, int ep) {
  __shared__ __align__(16) double ct[kFastTile][6];
  __shared__ Top2 wt[kFastT / 32];
  __shared__ bool last;
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&v.ctl->probe[2], 1), v.host->seen[2] = k;
  const bool live_blk = launch_live(v.ctl, ep);
  const int n = v.n;
  const double ir = 1.0 / v.R;
  double px[kFastP], py[kFastP], pz[kFastP], fx[kFastP], fy[kFastP], fz[kFastP];
#pragma unroll
  for (int s = 0; s < kFastP; ++s) {
    const int i = (blockIdx.x * kFastP + s) * kFastT + threadIdx.x;
    const bool live = i < n;
    px[s] = live ? v.px[i] * ir : 0.0, py[s] = live ? v.py[i] * ir : 0.0;
    pz[s] = live ? v.pz[i] * ir : 0.0;
    fx[s] = fy[s] = fz[s] = 0.0;
  }
  for (int m0 = 0; live_blk && m0 < k; m0 += kFastTile) {
    const int cnt = min(kFastTile, k - m0);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kFastT) {
      ct[t][0] = v.cx[m0 + t] * ir, ct[t][1] = v.cy[m0 + t] * ir, ct[t][2] = v.cz[m0 + t] * ir;
      ct[t][3] = v.fax[m0 + t], ct[t][4] = v.fay[m0 + t], ct[t][5] = v.faz[m0 + t];
    }
    __syncthreads();
#pragma unroll 2
    for (int t = 0; t < cnt; ++t) {
      const double2 c01 = *reinterpret_cast<const double2*>(&ct[t][0]);
      const double2 c23 = *reinterpret_cast<const double2*>(&ct[t][2]);
      const double2 c45 = *reinterpret_cast<const double2*>(&ct[t][4]);
#pragma unroll
      for (int s = 0; s < kFastP; ++s) {
        const double dx = px[s] - c01.x, dy = py[s] - c01.y, dz = pz[s] - c23.x;
        const double q = fma(dx, dx, fma(dy, dy, dz * dz));
        const double eta = fast::sqrt_pos(fmax(q, 1e-300));
        const double phi = q < 1.0 ? fast_phi<KIND>(eta) : 0.0;
        fx[s] = fma(c23.y, phi, fx[s]), fy[s] = fma(c45.x, phi, fy[s]), fz[s] = fma(c45.y, phi, fz[s]);
      }
    }
  }
  Top2 t{-1.0, -1.0, n, n};
#pragma unroll
  for (int s = 0; s < kFastP; ++s) {
    const int i = (blockIdx.x * kFastP + s) * kFastT + threadIdx.x;
    if (i < n && v.selstep[i] >= k) {
      const double ex = v.tx[i] - fx[s], ey = v.ty[i] - fy[s], ez = v.tz[i] - fz[s];
      const double q = fma(ex, ex, fma(ey, ey, ez * ez));
      Top2 u{q >= 0.0 ? q : 0.0, -1.0, i, n};  // NaN -> 0: a candidate always predicts
      t = merge2(t, u);
    }
  }
  t = warp_top2(t);
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kFastT / 32; ++w) t = merge2(t, wt[w]);
    v.fbv[blockIdx.x] = t.v1, v.fbv2[blockIdx.x] = t.v2, v.fbi[blockIdx.x] = t.i1;
    v.fbi[gridDim.x + blockIdx.x] = t.i2;
    __threadfence();
    last = atomicAdd(&v.ctl->fticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // last block: merge the block results with all threads, then across warps
  __threadfence();
  Top2 r{-1.0, -1.0, n, n};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kFastT)
    r = merge2(r, Top2{((volatile double*)v.fbv)[b], ((volatile double*)v.fbv2)[b],
                       ((volatile int*)v.fbi)[b], ((volatile int*)v.fbi)[gridDim.x + b]});
  r = warp_top2(r);
  __syncthreads();  // wt is reused
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < kFastT / 32; ++w) r = merge2(r, wt[w]);
  v.ctl->fticket = 0;
  {
    const int4 w = ld_volatile4(&v.ctl->epoch);
    if (w.x != ep || w.y != 0 || w.w != 0) return;
  }
  v.pred2_node[k] = r.v2 >= 0.0 && r.i2 < n ? r.i2 : -1;
  v.pred_gap[k] = r.v1 > 0.0 ? (r.v1 - fmax(r.v2, 0.0)) / r.v1 : -1.0;
  atomicAdd(&v.ctl->probe[3], 1), v.host->seen[3] = k, tl_mark(v, kTlFsweepE, k);
  __threadfence();
  v.pred_node[k] = (r.v1 >= 0.0 && r.i1 < n) ? r.i1 : -1;
}

// ---------------------------------------------------------------------------
// exact sweep(k): greedy.cpp:122-153 with alpha_k from its slot
// ---------------------------------------------------------------------------
__global__ void k_spec_wait_chain(SpecView v, int k, int ep) {
  atomicAdd(&v.ctl->probe[4], 1), v.host->seen[4] = k;
  const unsigned long long t0 = globaltimer();
  for (;;) {
    const int4 w = ld_volatile4(&v.ctl->epoch);
    if (w.x != ep || w.y != 0 || w.w != 0) return;
    if (ld_volatile(&v.chain_ep[k]) == ep) return;
    if (globaltimer() - t0 > v.watchdog_ns) {
      finish(v, kStatusWatchdog, k);
      return;
    }
    __nanosleep(500);
  }
}

template <int KIND>
__global__ void __launch_bounds__(kSweepT) k_spec_sweep(SpecView v, int k, int ep) {
  __shared__ __align__(16) gsw::Smem S;
  __shared__ double wv[kSweepT / 32], wa[kSweepT / 32], wv2[kSweepT / 32];
  __shared__ int wi[kSweepT / 32], wi2[kSweepT / 32];
  __shared__ bool last;
  if (threadIdx.x == 0 && blockIdx.x == 0)
    atomicAdd(&v.ctl->probe[5], 1), v.host->seen[5] = k, tl_mark(v, kTlSweepB, k);
  const bool live_blk = launch_live(v.ctl, ep);  // see k_fast_sweep on the ticket
  const int n = v.n;
  const int slot = k % v.S;
  const double* ax = v.slots + (size_t)slot * 3 * v.cap;
  const double* ay = ax + v.cap;
  const double* az = ay + v.cap;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * gsw::kP + lane;
  const bool in = i < n;
  const double px = in ? v.px[i] : 0.0, py = in ? v.py[i] : 0.0, pz = in ? v.pz[i] : 0.0;
  // greedy_sweep.cuh: phi by all warps, the ordered sums one axis per warp (warps 0-2)
  gsw::interpolant<KIND>(S, v.cx, v.cy, v.cz, ax, ay, az, k, v.R, v.kind, px, py, pz, live_blk);
  const bool live = in && threadIdx.x < 32;  // warp 0 owns the points from here on
  const double fx = S.f[0][lane], fy = S.f[1][lane], fz = S.f[2][lane];
  double nv = -1.0, all = 0.0, nv2 = -1.0;
  int ni = n, ni2 = n;
  if (live && live_blk) {
    const double ex = exact::sub(v.tx[i], fx), ey = exact::sub(v.ty[i], fy),
                 ez = exact::sub(v.tz[i], fz);
    v.rx[i] = ex, v.ry[i] = ey, v.rz[i] = ez;
    const double nrm = exact::norm(ex, ey, ez);
    if (v.selstep[i] >= k) nv = nrm, ni = i;  // not among c_0..c_{k-1}
    all = nrm;
  }
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, nv, o);
    const double s2 = __shfl_xor_sync(0xffffffffu, nv2, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, ni, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, ni2, o);
    Top2 a{nv, nv2, ni, ni2};
    a = merge2(a, Top2{v2, s2, i2, j2});
    nv = a.v1, nv2 = a.v2, ni = a.i1, ni2 = a.i2;
    const double a2 = __shfl_xor_sync(0xffffffffu, all, o);
    all = (all < a2) ? a2 : all;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) wv[w] = nv, wi[w] = ni, wa[w] = all, wv2[w] = nv2, wi2[w] = ni2;
  __syncthreads();
  if (threadIdx.x == 0) {
    Top2 a{nv, nv2, ni, ni2};
    for (int t = 1; t < kSweepT / 32; ++t) {
      a = merge2(a, Top2{wv[t], wv2[t], wi[t], wi2[t]});
      all = (all < wa[t]) ? wa[t] : all;
    }
    v.bv[blockIdx.x] = a.v1, v.bv2[blockIdx.x] = a.v2, v.bi[blockIdx.x] = a.i1;
    v.bi2[blockIdx.x] = a.i2;
    v.ba[blockIdx.x] = all;
    __threadfence();
    last = atomicAdd(&v.ctl->ticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // final block: grid argmax + decision (greedy.cpp:136-152); the block
  // results are merged by all threads, then across the warps
  __threadfence();
  Top2 r{-1.0, -1.0, n, n};
  double ov = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kSweepT) {
    r = merge2(r, Top2{((volatile double*)v.bv)[b], ((volatile double*)v.bv2)[b],
                       ((volatile int*)v.bi)[b], ((volatile int*)v.bi2)[b]});
    const double a = ((volatile double*)v.ba)[b];
    ov = (ov < a) ? a : ov;
  }
  r = warp_top2(r);
  for (int o = 16; o; o >>= 1) {
    const double a2 = __shfl_xor_sync(0xffffffffu, ov, o);
    ov = (ov < a2) ? a2 : ov;
  }
  __syncthreads();  // the w* arrays are reused
  if ((threadIdx.x & 31) == 0) wv[w] = r.v1, wi[w] = r.i1, wv2[w] = r.v2, wi2[w] = r.i2, wa[w] = ov;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int t = 1; t < kSweepT / 32; ++t) {
    r = merge2(r, Top2{wv[t], wv2[t], wi[t], wi2[t]});
    ov = (ov < wa[t]) ? wa[t] : ov;
  }
  SpecCtl* c = v.ctl;
  c->ticket = 0;
  {
    const int4 w = ld_volatile4(&c->epoch);
    if (w.x != ep || w.y != 0 || w.w != 0) return;
  }
  const double achieved = v.target_max > 0.0 ? exact::div(ov, v.target_max) : 0.0;
  atomicAdd(&c->probe[6], 1), v.host->seen[6] = k, tl_mark(v, kTlSweepE, k);
  v.rec_err[k - 1] = achieved;
  v.rec_sec[k - 1] = (double)(globaltimer() - c->t0) * 1e-9;
  v.exact_gap[k] = r.v1 > 0.0 ? (r.v1 - fmax(r.v2, 0.0)) / r.v1 : -1.0;
  c->achieved = achieved;
  c->overall = ov;
  const int mi = r.i1;
  v.exact_node[k] = mi;
  if (achieved < v.tol) {
    finish(v, kStatusConverged, k);
    return;
  }
  if (k >= v.cap || mi == n) {
    finish(v, kStatusCapHit, k);
    return;
  }
  // c_k = mi.  Publish it; if insert(k) already ran on a prediction, check it.
  const int old = atomicExch(&v.state[k], mi | kExactBit);
  bool mispredict = false;
  if (old != kEmpty && !(old & kExactBit)) {
    if (old == mi) {
      c->hits += 1;
      if (ld_volatile(&v.ins_fail[k])) {  // the reference's own c_k fails rbf.cpp:92
        c->fail_node = mi;
        c->fail_row = k;
        c->fail_pivot = v.pivot[k];
        finish(v, kStatusSolveError, k);
        return;
      }
    } else {
      mispredict = true;
      c->misses += 1;
    }
  } else {
    c->late += 1;  // decided before the predictor got there
  }
  c->conf = k;
  if (mispredict) {
    c->abort_step = k;
    __threadfence();
    c->abort = 1;
  }
  __threadfence();
  host_publish(v);
}

// ---------------------------------------------------------------------------
// chain server: S persistent CTAs, CTA j runs chain(k) for k = j (mod S)
// ---------------------------------------------------------------------------
struct SpecAbort {
  const SpecCtl* c;
  int k, ep;
  __device__ int4 poll_issue() const {
    int4 w;
    asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "l"(&c->epoch));
    return w;
  }
  __device__ bool poll_test(int4 w) const { return w.x != ep || (w.y != 0 && w.z < k) || w.w != 0; }
};

__device__ __forceinline__ int first_step_after(int r, int j, int S) {
  // smallest k > r, k >= 1, with k % S == j
  int k = r + 1;
  k += ((j - k % S) + S) % S;
  if (k < 1) k += S;
  return k;
}

template <bool XS_SMEM>
__global__ void __launch_bounds__(64) k_chain_server(SpecView v) {
  extern __shared__ __align__(16) double sh[];
  __shared__ int s_go, s_k, s_ep;
  const int j = blockIdx.x, S = v.S;
  int k = first_step_after(0, j, S);
  int ep_local = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer();
      int go = 0;
      for (;;) {
        const int4 w = ld_volatile4(&v.ctl->epoch);
        if (w.w != 0) break;  // level done
        if (w.x != ep_local) {
          ep_local = w.x;
          k = first_step_after(ld_volatile(&v.ctl->rb_step), j, S);
        }
        if (w.y == 0 && k <= v.cap && ld_volatile(&v.ins_ep[k - 1]) == w.x &&
            ld_volatile(&v.ctl->conf) >= k - S) {
          go = 1;
          s_ep = w.x;
          break;
        }
        if (globaltimer() - t0 > v.watchdog_ns) {
          finish(v, kStatusWatchdog, k);
          break;
        }
        __nanosleep(200);
      }
      s_go = go, s_k = k;
    }
    __syncthreads();
    if (!s_go) return;
    const int kk = s_k, ep = s_ep;
    if (threadIdx.x == 0) atomicAdd(&v.ctl->probe[7], 1), v.host->seen[7] = kk, tl_mark(v, kTlChainB, kk);
    double* out = v.slots + (size_t)(kk % S) * 3 * v.cap;
    gdev::ChainIO io{v.Lt, (size_t)v.cap, v.diag, v.yx, v.yy, v.yz, out, out + v.cap,
                     out + 2 * v.cap, XS_SMEM ? nullptr : v.xs_global + (size_t)j * 4 * v.cap};
    const bool done = gdev::chain_solve<XS_SMEM, true>(io, kk, sh, SpecAbort{v.ctl, kk, ep});
    if (threadIdx.x == 0 && done) {
      tl_mark(v, kTlChainE, kk);
      __threadfence();
      st_volatile(&v.chain_ep[kk], ep);
      __threadfence();
      const int4 w = ld_volatile4(&v.ctl->epoch);
      if (w.x == ep && !(w.y != 0 && w.z < kk)) k = kk + S;  // else redo after the rollback
    }
    __syncthreads();
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
SpecView GreedyEngine::spec_view() {
  SpecView s{};
  s.n = n_, s.cap = cap_, s.S = spec_S_, s.kind = kind_;
  s.R = R_;
  s.tol = tol_, s.target_max = target_max_;
  s.px = pos_.x.p, s.py = pos_.y.p, s.pz = pos_.z.p;
  s.tx = tgt_.x.p, s.ty = tgt_.y.p, s.tz = tgt_.z.p;
  s.rx = res_.x.p, s.ry = res_.y.p, s.rz = res_.z.p;
  s.cx = cpos_.x.p, s.cy = cpos_.y.p, s.cz = cpos_.z.p;
  s.cidx = cidx_.p;
  s.Lt = lt_.p;
  s.diag = diag_.p;
  s.yx = y_.x.p, s.yy = y_.y.p, s.yz = y_.z.p;
  s.slots = sp_slots_.p;
  s.xs_global = sp_xs_.p;
  s.rr_global = rr_.p;
  s.fax = sp_fa_.p, s.fay = sp_fa_.p + cap_, s.faz = sp_fa_.p + 2 * (size_t)cap_;
  s.selstep = sp_selstep_.p;
  int* w = sp_words_.p;
  const size_t m = (size_t)cap_ + 1;
  s.state = w, s.ins_ep = w + m, s.chain_ep = w + 2 * m, s.ins_node = w + 3 * m,
  s.ins_fail = w + 4 * m, s.pred_node = w + 5 * m, s.pred2_node = w + 6 * m,
  s.exact_node = w + 7 * m;
  s.bi2 = sp_bi2_.p;
  double* d = sp_dwords_.p;
  s.pivot = d, s.pred_gap = d + m, s.exact_gap = d + 2 * m;
  s.bv = bv_.p, s.ba = ba_.p, s.bi = bi_.p;
  s.bv2 = sp_bv2_.p;
  s.fbv = sp_fbv_.p, s.fbv2 = sp_fbv_.p + sp_fnblk_, s.fbi = sp_fbi_.p;
  s.rec_err = rec_err_.p, s.rec_sec = rec_sec_.p;
  s.ctl = sp_ctl_.p;
  s.host = sp_host_dev_;
  s.tl = sp_tl_.p;
  const char* we = std::getenv("IMB_SPEC_WATCHDOG_S");
  s.watchdog_ns = (unsigned long long)((we ? std::atof(we) : 60.0) * 1e9);
  return s;
}

void GreedyEngine::spec_alloc() {
  if (sp_ready_) return;
  const char* e = std::getenv("IMB_SPEC_S");
  spec_S_ = e ? std::max(1, std::atoi(e)) : 32;
  spec_S_ = std::min(spec_S_, std::max(1, ctx_.num_sms - 20));
  const size_t m = (size_t)cap_ + 1;
  sp_slots_.reserve((size_t)spec_S_ * 3 * cap_);
  sp_fa_.reserve(3 * (size_t)cap_);
  sp_selstep_.reserve(n_);
  sp_words_.reserve(8 * m);
  sp_bi2_.reserve(nblk_);
  sp_dwords_.reserve(3 * m);
  sp_bv2_.reserve(nblk_);
  sp_fnblk_ = (n_ + kFastT * kFastP - 1) / (kFastT * kFastP);
  sp_fbv_.reserve(2 * (size_t)sp_fnblk_);
  sp_fbi_.reserve(2 * (size_t)sp_fnblk_);
  sp_ctl_.reserve(1);
  sp_tl_.reserve((size_t)kTlCount * m);
  IMB_CHECK(cudaHostAlloc(&sp_host_, sizeof(SpecHost), cudaHostAllocMapped));
  IMB_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&sp_host_dev_), sp_host_, 0));
  // chain server smem: x / D in shared memory when it fits, else global
  const size_t head = gdev::chain_smem_head();
  sp_xs_smem_ = (size_t)cap_ * 32 + head <= 226 * 1024;
  sp_server_smem_ = sp_xs_smem_ ? (size_t)cap_ * 32 + head : head;
  if (!sp_xs_smem_) sp_xs_.reserve((size_t)spec_S_ * 4 * cap_);
  IMB_CHECK(cudaFuncSetAttribute(k_chain_server<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(sp_server_smem_, 48 * 1024)));
  IMB_CHECK(cudaFuncSetAttribute(k_chain_server<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(sp_server_smem_, 48 * 1024)));
  sp_fsolve_smem_ = 3 * (size_t)cap_ * 8;
  sp_pred_smem_ = 4 * (size_t)cap_ * 8;
  if (sp_pred_smem_ + sizeof(pred::Smem) + 1024 <= 227 * 1024)
    IMB_CHECK(cudaFuncSetAttribute(k_predict, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(sp_pred_smem_, 48 * 1024)));
  IMB_CHECK(cudaFuncSetAttribute(k_fast_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(sp_fsolve_smem_, 48 * 1024)));
  for (auto kern : {k_spec_insert<4, 1024>, k_spec_insert<2, 1024>, k_spec_insert<0, 1024>})
    IMB_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(ins_smem_, 48 * 1024)));
  // Load every kernel of the pipeline now: under lazy module loading (the
  // CUDA 12 default) a kernel's first launch loads its code, which waits for
  // the device -- and the device never idles while the chain server spins.
  {
    cudaFuncAttributes fa;
    const void* fns[] = {
        (const void*)k_spec_init,         (const void*)k_spec_rollback,
        (const void*)k_spec_insert<4, 1024>, (const void*)k_spec_insert<2, 1024>,
        (const void*)k_spec_insert<0, 1024>,
        (const void*)k_fast_solve,        (const void*)k_fast_sweep<C0>,
        (const void*)k_fast_sweep<C2>,    (const void*)k_fast_sweep<C4>,
        (const void*)k_fast_sweep<C6>,
        (const void*)k_predict,
        (const void*)k_spec_wait_chain,   (const void*)k_spec_sweep<-1>,
        (const void*)k_spec_sweep<C0>,    (const void*)k_spec_sweep<C2>,
        (const void*)k_spec_sweep<C4>,    (const void*)k_spec_sweep<C6>,
        (const void*)k_chain_server<true>, (const void*)k_chain_server<false>};
    for (const void* f : fns) IMB_CHECK(cudaFuncGetAttributes(&fa, f));
  }
  int lo, hi;
  IMB_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const char* pe = std::getenv("IMB_SPEC_PRIO");
  if (pe && pe[0] == '0') hi = lo;
  IMB_CHECK(cudaStreamCreateWithPriority(&sp_pred_, cudaStreamNonBlocking, hi));
  IMB_CHECK(cudaStreamCreateWithPriority(&sp_chain_, cudaStreamNonBlocking, lo));
  sp_ready_ = true;
}

void GreedyEngine::spec_free() {
  if (sp_host_) cudaFreeHost(sp_host_);
  if (sp_pred_) cudaStreamDestroy(sp_pred_);
  if (sp_chain_) cudaStreamDestroy(sp_chain_);
  sp_host_ = nullptr, sp_pred_ = nullptr, sp_chain_ = nullptr;
}

const GState& GreedyEngine::run_level_spec() {
  spec_alloc();
  cudaStream_t sm = ctx_.stream, sp = sp_pred_, sc = sp_chain_;
  // the level's state (reset() already cleared GState / sel on the main stream)
  const SpecView v = spec_view();
  k_spec_init<<<std::max(1, std::min(ctx_.num_sms, (n_ + 255) / 256)), 256, 0, sm>>>(v);
  IMB_CHECK(cudaStreamSynchronize(sm));
  // server first, so all S CTAs are resident before anything else runs
  if (sp_xs_smem_)
    k_chain_server<true><<<spec_S_, 64, sp_server_smem_, sc>>>(v);
  else
    k_chain_server<false><<<spec_S_, 64, sp_server_smem_, sc>>>(v);
  IMB_LAUNCH_CHECK();
  volatile SpecHost* h = sp_host_;
  const int S = spec_S_;
  const int fgrid = sp_fnblk_;
  auto launch_insert = [&](int k, int ep) {
    if (ins_ring_ == 4)
      k_spec_insert<4, 1024><<<1, 1024, ins_smem_, sp>>>(v, k, ep);
    else if (ins_ring_ == 2)
      k_spec_insert<2, 1024><<<1, 1024, ins_smem_, sp>>>(v, k, ep);
    else
      k_spec_insert<0, 1024><<<1, 1024, 0, sp>>>(v, k, ep);
  };
  // the cluster predictor (insert(k) + fast_solve(k + 1) in one launch) when
  // its shared memory fits, else the single-CTA insert and fast solve
  const bool cluster_pred = sp_pred_smem_ + sizeof(pred::Smem) + 1024 <= 227 * 1024 &&
                            !std::getenv("IMB_SPEC_NOCLUSTER");
  auto launch_predict = [&](int k, int ep) {
    if (cluster_pred) {
      k_predict<<<pred::kC, pred::kT, sp_pred_smem_, sp>>>(v, k, ep);
    } else {
      launch_insert(k, ep);
      if (k + 1 < cap_) k_fast_solve<<<1, 1024, sp_fsolve_smem_, sp>>>(v, k + 1, ep);
    }
  };
  auto launch_fsweep = [&](int k, int ep) {
    switch (kind_) {
      case C0: k_fast_sweep<C0><<<fgrid, kFastT, 0, sp>>>(v, k, ep); break;
      case C2: k_fast_sweep<C2><<<fgrid, kFastT, 0, sp>>>(v, k, ep); break;
      case C4: k_fast_sweep<C4><<<fgrid, kFastT, 0, sp>>>(v, k, ep); break;
      default: k_fast_sweep<C6><<<fgrid, kFastT, 0, sp>>>(v, k, ep); break;
    }
  };
  auto launch_sweep = [&](int k, int ep) {
    k_spec_wait_chain<<<1, 1, 0, sm>>>(v, k, ep);
    switch (sweep_kind_) {
      case C0: k_spec_sweep<C0><<<nblk_, kSweepT, 0, sm>>>(v, k, ep); break;
      case C2: k_spec_sweep<C2><<<nblk_, kSweepT, 0, sm>>>(v, k, ep); break;
      case C4: k_spec_sweep<C4><<<nblk_, kSweepT, 0, sm>>>(v, k, ep); break;
      case C6: k_spec_sweep<C6><<<nblk_, kSweepT, 0, sm>>>(v, k, ep); break;
      default: k_spec_sweep<-1><<<nblk_, kSweepT, 0, sm>>>(v, k, ep); break;
    }
  };
  int ep = 0, next = 0;  // next step whose predictor / insert work is to be enqueued
  const int la = S + 2;  // lookahead in steps beyond the last confirmed one
  const auto t_start = std::chrono::steady_clock::now();
  for (;;) {
    const int conf = h->conf;
    while (next <= cap_ && next <= conf + la && !h->abort && !h->done) {
      if (next >= 1) {
        // the prediction of c_next (alpha~ from predict(next - 1)) feeds insert(next)
        if (next < cap_) launch_fsweep(next, ep);
        launch_sweep(next, ep);
      }
      if (next < cap_) launch_predict(next, ep);
      IMB_LAUNCH_CHECK();
      ++next;
    }
    if (h->done) break;
    if (h->abort) {
      IMB_CHECK(cudaStreamSynchronize(sp));
      IMB_CHECK(cudaStreamSynchronize(sm));
      if (h->done) break;
      k_spec_rollback<<<1, 1024, 0, sm>>>(v);
      IMB_CHECK(cudaStreamSynchronize(sm));
      ++ep;
      // restart at the mispredicted step r: sweep(r) is done (c_r is EXACT in
      // state[r]), so only insert(r) is re-issued, then steps r+1.. as usual
      const int r = spec_restart_step();
      launch_predict(r, ep);
      IMB_LAUNCH_CHECK();
      next = r + 1;
      continue;
    }
    if (std::getenv("IMB_SPEC_TRACE")) {
      static auto last = std::chrono::steady_clock::now();
      if (std::chrono::steady_clock::now() - last > std::chrono::seconds(3)) {
        last = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[spec] host next=%d conf=%d seen ins %d fsolve %d fsweep %d/%d wait %d sweep %d/%d chain %d\n",
                     next, h->conf, h->seen[0], h->seen[1], h->seen[2], h->seen[3], h->seen[4],
                     h->seen[5], h->seen[6], h->seen[7]);
      }
    }
    if (std::chrono::steady_clock::now() - t_start > std::chrono::seconds(3600))
      throw std::runtime_error("speculative greedy: host watchdog");
    std::this_thread::yield();
  }
  IMB_CHECK(cudaStreamSynchronize(sm));
  IMB_CHECK(cudaStreamSynchronize(sp));
  IMB_CHECK(cudaStreamSynchronize(sc));
  IMB_LAUNCH_CHECK();
  // results -> the engine's buffers / GState
  SpecCtl c;
  IMB_CHECK(cudaMemcpy(&c, sp_ctl_.p, sizeof c, cudaMemcpyDeviceToHost));
  if (c.status == kStatusWatchdog) {
    // diagnostics: the protocol words around the stuck step
    const size_t m = (size_t)cap_ + 1;
    std::vector<int> w(6 * m);
    IMB_CHECK(cudaMemcpy(w.data(), sp_words_.p, w.size() * 4, cudaMemcpyDeviceToHost));
    std::fprintf(stderr,
                 "[spec] watchdog: epoch=%d abort=%d abort_step=%d done=%d rb=%d conf=%d "
                 "final=%d hits=%d misses=%d late=%d rollbacks=%d\n",
                 c.epoch, c.abort, c.abort_step, c.done, c.rb_step, c.conf, c.final_step, c.hits,
                 c.misses, c.late, c.rollbacks);
    std::fprintf(stderr, "[spec] probes: insert %d fsolve %d fsweep %d/%d wait %d sweep %d/%d chains %d\n",
                 c.probe[0], c.probe[1], c.probe[2], c.probe[3], c.probe[4], c.probe[5], c.probe[6],
                 c.probe[7]);
    for (int k = std::max(0, c.conf - 2); k <= std::min(cap_, c.conf + 6); ++k)
      std::fprintf(stderr, "[spec]  k=%d state=%x ins_ep=%d chain_ep=%d ins_node=%d ins_fail=%d pred=%d\n",
                   k, w[k], w[m + k], w[2 * m + k], w[3 * m + k], w[4 * m + k], w[5 * m + k]);
    throw std::runtime_error("speculative greedy: device watchdog");
  }
  const int fs = c.final_step;
  GState& s = *hst_;
  s = GState{};
  s.status = c.status;
  s.achieved = c.achieved;
  s.overall = c.overall;
  s.tol = tol_;
  s.target_max = target_max_;
  if (c.status == kStatusSolveError) {
    s.nc = fs;  // c_0..c_{fs-1} inserted, node fail_node failed at row fs
    s.steps = fs;
    s.fail_node = c.fail_node;
    s.fail_row = c.fail_row;
    s.fail_pivot = c.fail_pivot;
  } else {
    s.nc = fs;
    s.steps = fs;
    const double* a = sp_slots_.p + (size_t)(fs % S) * 3 * cap_;
    IMB_CHECK(cudaMemcpyAsync(alpha_.x.p, a, fs * 8, cudaMemcpyDeviceToDevice, sm));
    IMB_CHECK(cudaMemcpyAsync(alpha_.y.p, a + cap_, fs * 8, cudaMemcpyDeviceToDevice, sm));
    IMB_CHECK(cudaMemcpyAsync(alpha_.z.p, a + 2 * (size_t)cap_, fs * 8, cudaMemcpyDeviceToDevice, sm));
  }
  IMB_CHECK(cudaMemcpyAsync(st_.p, hst_, sizeof(GState), cudaMemcpyHostToDevice, sm));
  IMB_CHECK(cudaStreamSynchronize(sm));
  spec_stats_.hits += c.hits, spec_stats_.misses += c.misses, spec_stats_.late += c.late;
  spec_stats_.rollbacks += c.rollbacks;
  if (std::getenv("IMB_SPEC_LOG")) {
    const size_t m = (size_t)cap_ + 1;
    std::vector<double> pg(m), eg(m);
    std::vector<int> words(8 * m);
    IMB_CHECK(cudaMemcpy(words.data(), sp_words_.p, words.size() * 4, cudaMemcpyDeviceToHost));
    IMB_CHECK(cudaMemcpy(pg.data(), sp_dwords_.p + m, m * 8, cudaMemcpyDeviceToHost));
    IMB_CHECK(cudaMemcpy(eg.data(), sp_dwords_.p + 2 * m, m * 8, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[spec] n=%d cap=%d S=%d steps=%d hits=%d misses=%d late=%d rollbacks=%d\n",
                 n_, cap_, S, fs, c.hits, c.misses, c.late, c.rollbacks);
    if (FILE* f = std::fopen(std::getenv("IMB_SPEC_LOG"), "a")) {
      std::fprintf(f, "# level n=%d cap=%d steps=%d hits=%d misses=%d late=%d rollbacks=%d\n", n_,
                   cap_, fs, c.hits, c.misses, c.late, c.rollbacks);
      // k, predictor gap, exact gap, node inserted at k (last epoch), predicted 1st / 2nd,
      // exact choice
      std::vector<unsigned long long> tl((size_t)kTlCount * m);
      IMB_CHECK(cudaMemcpy(tl.data(), sp_tl_.p, tl.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (auto t : tl)
        if (t) t0 = std::min(t0, t);
      auto us = [&](int e, int k) -> double {
        const unsigned long long t = tl[(size_t)e * m + k];
        return t ? (double)(t - t0) * 1e-3 : -1.0;
      };
      // per step: k, gaps, nodes, then the timeline in microseconds from the
      // level's first event: insert begin/end, fast solve begin/end, fast
      // sweep end, exact sweep begin/end, chain begin/end (last epoch)
      for (int k = 1; k <= fs; ++k) {
        std::fprintf(f, "%d %.3e %.3e %d %d %d %d", k, pg[k], eg[k], words[3 * m + k],
                     words[5 * m + k], words[6 * m + k], words[7 * m + k]);
        for (int e = 0; e < kTlCount; ++e) std::fprintf(f, " %.1f", us(e, k));
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
  }
  return *hst_;
}

int GreedyEngine::spec_restart_step() {
  SpecCtl c;
  IMB_CHECK(cudaMemcpy(&c, sp_ctl_.p, sizeof c, cudaMemcpyDeviceToHost));
  return c.rb_step;
}

}  // namespace imb
