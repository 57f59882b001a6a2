// greedy.cu — K2..K5: multi-level greedy control-point selection with the
// incremental Cholesky factorisation (north-star b, c).
//
// Reference: greedy_level (greedy.cpp:60-170), insert_control (:86-112),
// CholeskyFactor::append / solve (rbf.cpp:71-121), run_multilevel (:172-195),
// solve_weights (rbf.cpp:144-193).
//
// Every greedy step is three kernels on the context stream, with no host
// round trip (the host only polls the device status word every kBatch steps):
//
//   k_insert   (1 CTA)  column phi(c_m, p_new) in control order, the new row
//                       of L by forward substitution in the reference order
//                       (right-looking: s_j -= L_jm r_m for m ascending, which
//                       applies the subtractions to each s_j in exactly the
//                       order of rbf.cpp:84), pivot + the 1e-14 SolveError
//                       test, and the incremental forward solve y_k (the
//                       reference recomputes y_0..y_{k-1} with identical
//                       operations, so caching them is bit-exact).
//   k_backward (1 warp) L^T x = y for the three axes in the reference order
//                       (rbf.cpp:114-120): the dependent-subtraction chain of
//                       ~k^2/2 DSUBs (8 cycles each on B200, tools/fp64_probe)
//                       with the products formed 32-wide by the warp.
//   k_sweep    (grid)   f_i = sum_m alpha_m phi(p_i, c_m) in control order for
//                       every surface node, E_i = t_i - f_i, |E_i|, block then
//                       grid argmax over unselected nodes (ties -> lowest
//                       index, strict > of greedy.cpp:137), overall max, the
//                       stop / cap decision of greedy.cpp:141-152.
//
// All arithmetic is the exact family of common.cuh, so control indices,
// alpha, the residual and the convergence record are bit-identical to the
// reference.  L is stored column-major packed (column i = rows i..cap-1
// contiguous) because both the append and the backward chain walk columns.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <string>

#include "common.cuh"
#include "greedy.hpp"

namespace imb {

namespace {

constexpr int kInsertThreads = 1024;
constexpr int kMaxCap = 8192;  // k_insert: rr + ring[2] in shared memory
constexpr int kSweepThreads = 64;
constexpr int kSweepTile = 128;

__device__ __forceinline__ size_t colstart(size_t i, size_t cap) {
  return i * cap - i * (i - 1) / 2;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// k_insert: greedy.cpp:86-112 / rbf.cpp:71-100
//
// Shared memory: rr[cap] (running s_j, then row[j]) | ring[NR][cap] (columns
// m .. m+NR-1 of L, streamed by cp.async NR-1 steps ahead: every thread
// copies exactly the rows it owns, so cp.async.wait_group alone orders the
// copy before its own use and no barrier guards the ring).  The pivot pair
// (L_mm, 1/L_mm) of row m is held in a register by m's owner thread, loaded
// 1024 steps ahead.  Per step the critical path is the owner's division,
// one barrier and the next owner's mul-sub.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NR, int T = kInsertThreads>
__global__ void __launch_bounds__(T) k_insert(GView g) {
  GState& st = *g.st;
  if (st.status != 0) return;
  extern __shared__ double sh[];
  const size_t cap = g.cap;
  double* rr = sh;          // [cap]
  double* ring = sh + cap;  // [NR][cap]
  const int tid = threadIdx.x;
  const int k = st.nc;
  const int node = st.next;
  if (k == 0 && tid == 0) st.t0 = globaltimer();

  const double px = g.px[node], py = g.py[node], pz = g.pz[node];
  const exact::Recip rR = exact::make_recip(g.R);
  double2 dm = tid < k ? g.diag[tid] : make_double2(1.0, 1.0);  // pivot of my next row
  // column (greedy.cpp:87-93 / rbf.cpp:167-170): phi(distance(c_m, p_new))
  for (int j = tid; j < k; j += T) {
    const double d = exact::dist(g.cx[j], g.cy[j], g.cz[j], px, py, pz);
    rr[j] = exact::wendland_rt(g.kind, exact::div_rcp(d, rR));
  }
  // Right-looking forward substitution (rbf.cpp:80-87): once row[m] is final,
  // every s_j (j > m) does s_j -= L_jm * row[m], so each s_j receives its
  // subtractions in ascending m exactly as in the reference's inner loop.
  // Per step every thread walks only its own rows; the first of them past the
  // issued / updated column and the issued column's start in L are carried
  // incrementally (no per-step division or colstart product: with 1024
  // threads the per-step instruction count, not the L2 latency, bounds this
  // loop).
  int mi = 0, ji = tid > 0 ? tid : T;  // next column to issue, my first row > mi
  const double* ci = g.Lt;             // its start, colstart(mi, cap)
  auto issue_next = [&]() {
    if (mi < k) {
      double* dst = ring + (mi & (NR - 1)) * cap;
      for (int j = ji; j < k; j += T) cp_async8(dst + j, ci + (j - mi));
    }
    cp_async_commit();
    ci += cap - (size_t)mi;  // colstart(mi + 1) = colstart(mi) + cap - mi
    ++mi;
    if (ji == mi) ji += T;
  };
#pragma unroll
  for (int q = 0; q < NR - 1; ++q) issue_next();
  __syncthreads();
  int ju = tid > 0 ? tid : T;  // my first row > m
  for (int m = 0; m < k; ++m) {
    if ((m & (T - 1)) == tid) {
      rr[m] = exact::div_rcp(rr[m], exact::Recip{dm.x, dm.y});  // row[j] = s / lj[j]
      if (m + T < k) dm = g.diag[m + T];
    }
    issue_next();             // column m + NR - 1
    cp_async_wait<NR - 1>();  // my copies of column m have landed
    __syncthreads();
    const double r = rr[m];
    const double* lc = ring + (m & (NR - 1)) * cap;
    for (int j = ju; j < k; j += T) rr[j] = exact::sub(rr[j], exact::mul(lc[j], r));
    if (ju == m + 1) ju += T;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  // stage y_0..y_{k-1} for the forward chain in the ring space when it fits
  const double *yxs = g.yx, *yys = g.yy, *yzs = g.yz;
  if (NR >= 3) {
    double* ys = sh + cap;
    for (int j = tid; j < k; j += T)
      ys[j] = g.yx[j], ys[cap + j] = g.yy[j], ys[2 * cap + j] = g.yz[j];
    yxs = ys, yys = ys + cap, yzs = ys + 2 * cap;
  }
  __syncthreads();
  // sq (rbf.cpp:86) and the forward solve of the new row (rbf.cpp:107-112 for
  // i = k), both sequential chains; 4 independent chains interleaved.
  if (tid == 0) {
    double sq = 0.0;
    double yx = g.tx[node], yy = g.ty[node], yz = g.tz[node];  // rhs_k = target[c_k]
#pragma unroll 8
    for (int j = 0; j < k; ++j) {
      const double r = rr[j];
      sq = exact::add(sq, exact::mul(r, r));
      yx = exact::sub(yx, exact::mul(r, yxs[j]));
      yy = exact::sub(yy, exact::mul(r, yys[j]));
      yz = exact::sub(yz, exact::mul(r, yzs[j]));
    }
    const double diag = 1.0;  // column[k] = 1.0 (greedy.cpp:93)
    st.max_diag = (st.max_diag < diag) ? diag : st.max_diag;
    const double pivot_sq = exact::sub(diag, sq);
    const double pivot = pivot_sq > 0.0 ? __dsqrt_rn(pivot_sq) : 0.0;
    if (!(pivot > exact::mul(1e-14, st.max_diag))) {
      st.status = kStatusSolveError;
      st.fail_node = node;
      st.fail_row = k;
      st.fail_pivot = pivot;
    } else {
      const exact::Recip pr = exact::make_recip(pivot);
      g.diag[k] = make_double2(pivot, pr.y);
      g.Lt[colstart(k, cap)] = pivot;
      g.yx[k] = exact::div_rcp(yx, pr);
      g.yy[k] = exact::div_rcp(yy, pr);
      g.yz[k] = exact::div_rcp(yz, pr);
      if (k == 0 || pivot < st.smallest_pivot) st.smallest_pivot = pivot;
      g.cidx[k] = node;
      g.cx[k] = px, g.cy[k] = py, g.cz[k] = pz;
      g.sel[node] = 1;
      st.nc = k + 1;
    }
  }
  __syncthreads();
  if (st.status != 0) return;
  // scatter the new row into the columns: L_kj at column j, offset k - j
  for (int j = tid; j < k; j += T) g.Lt[colstart(j, cap) + (k - j)] = rr[j];
}

// ---------------------------------------------------------------------------
// k_backward: rbf.cpp:114-120 for x, y, z (greedy.cpp:106-111).
//
// One warp walks the chunks (column i, rows j0..j0+31) of L^T in the
// reference order.  Per chunk the 32 lanes form the products L_ji * x_j for
// the three axes (register prefetch of L two chunks ahead), then EVERY lane
// runs the same 32-long dependent subtraction chain from a shared-memory
// broadcast, fully unrolled so the loads run ahead of the 8-cycle DSUBs.
// Padding rows beyond n contribute +0.0, an exact identity for subtraction.
// ---------------------------------------------------------------------------
struct Chunk {
  int i, j0;
};
__device__ __forceinline__ Chunk next_chunk(Chunk c, int n) {
  if (c.j0 + 32 < n) return {c.i, c.j0 + 32};
  return {c.i - 1, c.i};
}

constexpr int kBwRing = 8;     // blocks of L in flight
constexpr int kBwBlock = 512;  // doubles per block

__device__ __forceinline__ void bw_mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
      static_cast<uint32_t>(__cvta_generic_to_shared(bar))));
}
__device__ __forceinline__ void bw_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void bw_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

// Two warps, producer / consumer, per block of (up to kBwBlock) elements of
// a column of L^T:
//   warp 1 (producer, 32 lanes): P[a][e] = L_ji * x_j[a] for the three axes,
//            from the TMA-streamed L block and x in shared memory, into one
//            of two product buffers;
//   warp 0 (consumer, lanes 0..2): lane a runs the dependent chain
//            s -= P[a][e] of its axis -- a pure LDS + DSUB loop at the 8-cycle
//            DSUB latency -- and closes each column with x_i = s / L_ii.
// The column head (j = i+1) needs x_{i+1}, solved by the consumer at the end
// of the previous block, so the producer leaves it at +0 and passes its L
// value; the consumer applies it first, from registers, keeping the
// reference's ascending-j order (rbf.cpp:116-118).  Every other x_j a block
// needs was solved >= 2 blocks earlier, which the empty-buffer handshake
// orders before the producer reads it.  mbarrier phases: full[b] (producer
// -> consumer), empty[b] (consumer -> producer), ring[r] (TMA -> producer).
struct BwBlock {
  int i, e0;  // column i, elements e0.. of rows j = i+1+e
};

__device__ __forceinline__ void bw_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

constexpr int kBwPad = kBwBlock + 32;

template <bool XS_SMEM, bool TAIL>
__global__ void __launch_bounds__(64) k_backward_t(GView g) {
  const GState& st = *g.st;
  if (st.status != 0) return;
  extern __shared__ __align__(16) double sh[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = st.nc;
  const size_t cap = g.cap;
  uint64_t* ringbar = reinterpret_cast<uint64_t*>(sh);  // [kBwRing]
  uint64_t* full = ringbar + kBwRing;                   // [2]
  uint64_t* empty = full + 2;                           // [2]
  double* headL = sh + kBwRing + 4;                     // [2] (+2 pad)
  double* ring = sh + kBwRing + 8;                      // [kBwRing][kBwBlock+2]
  double* P = ring + kBwRing * (kBwBlock + 2);          // [2][3][kBwPad]
  // comp: X[cap] | Y[cap] | Z[cap] | D[cap]; X/Y/Z start as y and become x
  // once solved (s = x[i] at rbf.cpp:115 reads its own slot)
  double* comp = XS_SMEM ? P + 6 * kBwPad : g.xs_global;
  if (n == 0) return;
  // x_{n-1} = y_{n-1} / L_{n-1,n-1} (rbf.cpp:114-119 with an empty inner
  // loop) is solved here, before the barrier: the producer's second block
  // (column n-3) already reads it, before any empty[] handshake orders the
  // two warps
  for (int j = tid; j < n; j += 64) {
    double vx = g.yx[j], vy = g.yy[j], vz = g.yz[j];
    const double dj = g.diag[j].x;
    if (j == n - 1) {
      const exact::Recip r = exact::make_recip(dj);
      vx = exact::div_rcp(vx, r), vy = exact::div_rcp(vy, r), vz = exact::div_rcp(vz, r);
    }
    comp[j] = vx, comp[cap + j] = vy, comp[2 * cap + j] = vz;
    comp[3 * cap + j] = dj;
  }
  if (tid == 0) {
    for (int r = 0; r < kBwRing + 4; ++r) bw_mbar_init(&ringbar[r]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto next = [&](BwBlock b) -> BwBlock {
    if (b.e0 + kBwBlock < n - 1 - b.i) return {b.i, b.e0 + kBwBlock};
    return {b.i - 1, 0};
  };
  auto src_of = [&](BwBlock b, int& off, int& cnt) -> const double* {
    const double* src = g.Lt + colstart(b.i, cap) + 1 + b.e0;
    const uintptr_t al = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
    off = (int)((reinterpret_cast<uintptr_t>(src) - al) / 8);
    cnt = min(kBwBlock, n - 1 - b.i - b.e0);
    return reinterpret_cast<const double*>(al);
  };
  const double* dd = comp + 3 * cap;
  if (warp == 1) {
    // ---------------- producer ----------------
    auto issue = [&](BwBlock b, int slot) {
      if (lane != 0 || b.i < 0) return;
      int off, cnt;
      const double* al = src_of(b, off, cnt);
      const uint32_t bytes = (uint32_t)(((off + cnt) * 8 + 15) & ~15);
      bw_bulk(ring + slot * (kBwBlock + 2), al, bytes, &ringbar[slot]);
    };
    BwBlock cur{n - 2, 0}, ahead = cur;
    for (int r = 0; r < kBwRing; ++r) {
      issue(ahead, r);
      ahead = next(ahead);
    }
    for (int t = 0; cur.i >= 0; ++t) {
      const int slot = t % kBwRing, pb = t & 1;
      int off, cnt;
      src_of(cur, off, cnt);
      bw_wait(&ringbar[slot], (uint32_t)((t / kBwRing) & 1));
      bw_wait(&empty[pb], (uint32_t)(((t >> 1) & 1) ^ 1));
      const double* lb = ring + slot * (kBwBlock + 2) + off;
      double* pp = P + pb * 3 * kBwPad;
      const int j0 = cur.i + 1 + cur.e0;
      const bool head = cur.e0 == 0;
      for (int e = lane; e < cnt; e += 32) {
        const double l = lb[e];
        if (head && e == 0) {
          headL[pb] = l;
          pp[0] = pp[kBwPad] = pp[2 * kBwPad] = 0.0;  // s - (+0) == s
        } else {
          pp[e] = exact::mul(l, comp[j0 + e]);
          pp[kBwPad + e] = exact::mul(l, comp[cap + j0 + e]);
          pp[2 * kBwPad + e] = exact::mul(l, comp[2 * cap + j0 + e]);
        }
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bw_arrive(&full[pb]);
      }
      issue(ahead, slot);  // refill the slot just consumed
      ahead = next(ahead);
      cur = next(cur);
    }
  } else if (lane < 3) {
    // ---------------- consumer ----------------
    double* cx = comp + (size_t)lane * cap;
    BwBlock cur{n - 2, 0};
    double s = 0.0, rcp_i = 0.0;
    for (int t = 0; cur.i >= 0; ++t) {
      const int pb = t & 1, i = cur.i;
      int off, cnt;
      src_of(cur, off, cnt);
      bw_wait(&full[pb], (uint32_t)((t >> 1) & 1));
      const double* pa = P + pb * 3 * kBwPad + lane * kBwPad;
      if (cur.e0 == 0) {
        s = exact::sub(cx[i], exact::mul(headL[pb], cx[i + 1]));
        if (TAIL) rcp_i = g.diag[i].y;
      }
      // ping-pong register sets: loads of one 16-group run under the chain of
      // the other (no rotation moves); pa is padded so whole groups are safe.
      double ra[16], rb[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) ra[u] = pa[u];
      int e = 0;
      for (; e + 32 <= cnt; e += 32) {
#pragma unroll
        for (int u = 0; u < 16; ++u) rb[u] = pa[e + 16 + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) s = exact::sub(s, ra[u]);
#pragma unroll
        for (int u = 0; u < 16; ++u) ra[u] = pa[e + 32 + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) s = exact::sub(s, rb[u]);
      }
      if (TAIL) {
        // the last 0..31 elements: ra already holds pa[e..e+15] (prefetched by
        // the loop), rb is loaded up front; sub-groups of 4 padded with +0
        // (s - (+0) == s bit for bit, also for s = -0), so no per-element
        // load -> subtract round trips on the chain
        const int rem = cnt - e;
        if (rem > 16) {
#pragma unroll
          for (int u = 0; u < 16; ++u) rb[u] = pa[e + 16 + u];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (4 * q < rem) {
#pragma unroll
            for (int v = 0; v < 4; ++v) s = exact::sub(s, 4 * q + v < rem ? ra[4 * q + v] : 0.0);
          }
        if (rem > 16) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (16 + 4 * q < rem) {
#pragma unroll
              for (int v = 0; v < 4; ++v)
                s = exact::sub(s, 16 + 4 * q + v < rem ? rb[4 * q + v] : 0.0);
            }
        }
      } else {
        for (; e < cnt; ++e) s = exact::sub(s, pa[e]);
      }
      const BwBlock nx = next(cur);
      if (nx.i != i)  // x_i = s / L_ii, reciprocal of L_ii from k_insert (prefetched)
        cx[i] = exact::div_rcp(s, TAIL ? exact::Recip{dd[i], rcp_i} : exact::make_recip(dd[i]));
      __syncwarp(0x7u);
      if (lane == 0) bw_arrive(&empty[pb]);
      cur = nx;
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += 64) g.ax[i] = comp[i], g.ay[i] = comp[cap + i], g.az[i] = comp[2 * cap + i];
}

// ---------------------------------------------------------------------------
// k_sweep: greedy.cpp:122-153
// ---------------------------------------------------------------------------
__device__ __forceinline__ void better(double& v, int& i, double v2, int i2) {
  // max value, lowest index on ties (sequential strict '>' scan)
  if (v2 > v || (v2 == v && i2 < i)) v = v2, i = i2;
}

// KIND >= 0: the staged pair evaluation of the tiled exact kernels
// (xt::/exact_eval, common.cuh: four controls per stage, summed in insertion
// order) -- valid when the host verified |positions| <= 1e100 and R in
// [1e-100, 1e100] (exact_tiled_ok); KIND < 0: one pair at a time with the
// full-range __dsqrt_rn / division and a runtime basis switch.
template <int KIND>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(GView g) {
  GState& st = *g.st;
  if (st.status != 0) return;
  __shared__ __align__(16) double ct[kSweepTile][6];
  __shared__ double wv[kSweepThreads / 32], wa[kSweepThreads / 32];
  __shared__ int wi[kSweepThreads / 32];
  __shared__ bool last;
  const int n = g.n, nc = st.nc;
  const int i = blockIdx.x * kSweepThreads + threadIdx.x;
  const bool live = i < n;
  const double px = live ? g.px[i] : 0.0, py = live ? g.py[i] : 0.0, pz = live ? g.pz[i] : 0.0;
  const exact::Recip rR = exact::make_recip(g.R);
  double fx = 0.0, fy = 0.0, fz = 0.0;
  for (int m0 = 0; m0 < nc; m0 += kSweepTile) {
    const int cnt = min(kSweepTile, nc - m0);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kSweepThreads) {
      ct[t][0] = g.cx[m0 + t], ct[t][1] = g.cy[m0 + t], ct[t][2] = g.cz[m0 + t];
      ct[t][3] = g.ax[m0 + t], ct[t][4] = g.ay[m0 + t], ct[t][5] = g.az[m0 + t];
    }
    __syncthreads();
    if (KIND >= 0) {
      // every thread runs the loop (dead lanes on a zero point: harmless);
      // past cnt the last control is repeated, evaluated but not summed
      const double pxa[1] = {px}, pya[1] = {py}, pza[1] = {pz};
      double fxa[1] = {fx}, fya[1] = {fy}, fza[1] = {fz};
      for (int t = 0; t < cnt; t += 4) {
        const int js[4] = {t, min(t + 1, cnt - 1), min(t + 2, cnt - 1), min(t + 3, cnt - 1)};
        exact_eval<3, KIND < 0 ? C2 : KIND, 1, 4>(&ct[0][0], js, min(4, cnt - t), pxa, pya, pza,
                                                  fxa, fya, fza, rR);
      }
      fx = fxa[0], fy = fya[0], fz = fza[0];
    } else if (live) {
      for (int t = 0; t < cnt; ++t) {
        // distance(surface_positions[i], surface_positions[controls[m]])
        const double d = exact::dist(px, py, pz, ct[t][0], ct[t][1], ct[t][2]);
        const double phi = exact::wendland_rt(g.kind, exact::div_rcp(d, rR));
        if (phi != 0.0) {
          fx = exact::add(fx, exact::mul(ct[t][3], phi));
          fy = exact::add(fy, exact::mul(ct[t][4], phi));
          fz = exact::add(fz, exact::mul(ct[t][5], phi));
        }
      }
    }
  }
  double nv = -1.0, all = 0.0;
  int ni = n;
  if (live) {
    const double ex = exact::sub(g.tx[i], fx), ey = exact::sub(g.ty[i], fy),
                 ez = exact::sub(g.tz[i], fz);
    g.rx[i] = ex, g.ry[i] = ey, g.rz[i] = ez;
    const double nrm = exact::norm(ex, ey, ez);
    if (!g.sel[i]) nv = nrm, ni = i;
    all = nrm;
  }
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, nv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, ni, o);
    better(nv, ni, v2, i2);
    const double a2 = __shfl_xor_sync(0xffffffffu, all, o);
    all = (all < a2) ? a2 : all;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) wv[w] = nv, wi[w] = ni, wa[w] = all;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < kSweepThreads / 32; ++t) {
      better(nv, ni, wv[t], wi[t]);
      all = (all < wa[t]) ? wa[t] : all;
    }
    g.bv[blockIdx.x] = nv, g.bi[blockIdx.x] = ni, g.ba[blockIdx.x] = all;
    __threadfence();
    const unsigned int ticket = atomicAdd(&st.ticket, 1u);
    last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  // final block: grid argmax + decision (greedy.cpp:136-152)
  __threadfence();
  double mv = -1.0, ov = 0.0;
  int mi = n;
  for (int b = 0; b < (int)gridDim.x; ++b) {
    better(mv, mi, ((volatile double*)g.bv)[b], ((volatile int*)g.bi)[b]);
    const double a = ((volatile double*)g.ba)[b];
    ov = (ov < a) ? a : ov;
  }
  st.ticket = 0;
  const double achieved = st.target_max > 0.0 ? exact::div(ov, st.target_max) : 0.0;
  const int step = st.steps;
  g.rec_err[step] = achieved;
  g.rec_sec[step] = (double)(globaltimer() - st.t0) * 1e-9;
  st.steps = step + 1;
  st.achieved = achieved;
  st.overall = ov;
  if (achieved < st.tol) {
    st.status = kStatusConverged;
  } else if (nc >= g.cap || mi == n) {
    st.status = kStatusCapHit;
  } else {
    st.next = mi;
  }
}

// solve_weights driver step: insert node st.next = nc (points in order).
__global__ void k_next_in_order(GView g, int n) {
  GState& st = *g.st;
  if (st.status != 0) return;
  if (st.nc < n) st.next = st.nc;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
GreedyEngine::GreedyEngine(Context& ctx, int n, int cap) : ctx_(ctx), n_(n), cap_(cap) {
  if (cap > kMaxCap)
    throw InvalidArgument("max_points_per_level above " + std::to_string(kMaxCap) +
                          " is not supported by this build");
  pos_.reserve(n);
  tgt_.reserve(n);
  res_.reserve(n);
  sel_.reserve(n);
  cpos_.reserve(cap);
  cidx_.reserve(cap);
  const size_t tri = (size_t)cap * (cap + 1) / 2;
  lt_.reserve(tri + 4);  // +4: 16-byte rounded bulk copies may read past the end
  diag_.reserve(cap);
  y_.reserve(cap);
  alpha_.reserve(cap);
  nblk_ = (n + kSweepThreads - 1) / kSweepThreads;
  bv_.reserve(nblk_);
  ba_.reserve(nblk_);
  bi_.reserve(nblk_);
  rec_err_.reserve(cap + 1);
  rec_sec_.reserve(cap + 1);
  st_.reserve(1);
  IMB_CHECK(cudaMallocHost(&hst_, sizeof(GState)));
  // x workspace of the backward chain: shared memory when it fits
  const size_t head = (8 + 8 + 8 * (512 + 2) + 6 * (512 + 32)) * 8;  // barriers, L ring, products
  const size_t xs_bytes = (size_t)cap * 32 + head;
  if (xs_bytes <= 227 * 1024) {
    bw_smem_ = xs_bytes;
  } else {
    xs_.reserve((size_t)cap * 4);
    bw_smem_ = head;
  }
  for (auto k : {k_backward_t<true, true>, k_backward_t<false, true>, k_backward_t<true, false>,
                 k_backward_t<false, false>})
    IMB_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(bw_smem_, 48 * 1024)));
  // k_insert: rr + ring[2] (+ dg staging, which also makes room for y)
  // k_insert: rr + a ring of 4 columns when it fits (cap <= 5812), else 2
  ins_ring_ = (size_t)cap * 8 * 5 <= 227 * 1024 && !std::getenv("IMB_INSERT_RING2") ? 4 : 2;
  ins_smem_ = (size_t)cap * 8 * (1 + ins_ring_);
  if (const char* e = std::getenv("IMB_INSERT_T")) ins_threads_ = std::atoi(e);
  for (auto kern : {k_insert<4>, k_insert<4, 256>, k_insert<4, 512>, k_insert<2>})
    IMB_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(ins_smem_, 48 * 1024)));
}

GreedyEngine::~GreedyEngine() {
  if (hst_) cudaFreeHost(hst_);
}

GView GreedyEngine::view() {
  GView g{};
  g.st = st_.p;
  g.n = n_;
  g.cap = cap_;
  g.kind = kind_;
  g.R = R_;
  g.px = pos_.x.p, g.py = pos_.y.p, g.pz = pos_.z.p;
  g.tx = tgt_.x.p, g.ty = tgt_.y.p, g.tz = tgt_.z.p;
  g.rx = res_.x.p, g.ry = res_.y.p, g.rz = res_.z.p;
  g.sel = sel_.p;
  g.cidx = cidx_.p;
  g.cx = cpos_.x.p, g.cy = cpos_.y.p, g.cz = cpos_.z.p;
  g.Lt = lt_.p;
  g.diag = diag_.p;
  g.yx = y_.x.p, g.yy = y_.y.p, g.yz = y_.z.p;
  g.ax = alpha_.x.p, g.ay = alpha_.y.p, g.az = alpha_.z.p;
  g.xs_global = xs_.p;
  g.bv = bv_.p, g.ba = ba_.p, g.bi = bi_.p;
  g.rec_err = rec_err_.p;
  g.rec_sec = rec_sec_.p;
  return g;
}

void GreedyEngine::set_positions(const double* host_xyz) {
  upload_points(ctx_, host_xyz, n_, pos_);
  pos_max_abs_ = 0.0;
  for (size_t i = 0; i < (size_t)n_ * 3; ++i) {
    const double v = std::fabs(host_xyz[i]);
    if (!(v <= pos_max_abs_)) pos_max_abs_ = v;  // NaN propagates: no fast sweep
  }
}

void GreedyEngine::set_target(const double* host_xyz) { upload_points(ctx_, host_xyz, n_, tgt_); }

void GreedyEngine::target_from_residual() {
  const size_t b = (size_t)n_ * 8;
  IMB_CHECK(cudaMemcpyAsync(tgt_.x.p, res_.x.p, b, cudaMemcpyDeviceToDevice, ctx_.stream));
  IMB_CHECK(cudaMemcpyAsync(tgt_.y.p, res_.y.p, b, cudaMemcpyDeviceToDevice, ctx_.stream));
  IMB_CHECK(cudaMemcpyAsync(tgt_.z.p, res_.z.p, b, cudaMemcpyDeviceToDevice, ctx_.stream));
}

void GreedyEngine::reset(double tol, double target_max, int kind, double R) {
  kind_ = kind;
  R_ = R;
  const bool staged = !std::getenv("IMB_SWEEP_GENERIC") && kind >= C0 && kind <= C6 &&
                      exact_tiled_ok(R, pos_max_abs_);
  sweep_kind_ = staged ? kind : -1;
  GState s{};
  s.tol = tol;
  s.target_max = target_max;
  s.max_diag = 0.0;
  s.next = 0;
  *hst_ = s;
  IMB_CHECK(cudaMemcpyAsync(st_.p, hst_, sizeof(GState), cudaMemcpyHostToDevice, ctx_.stream));
  IMB_CHECK(cudaMemsetAsync(sel_.p, 0, n_, ctx_.stream));
}

const GState& GreedyEngine::poll() {
  IMB_CHECK(cudaMemcpyAsync(hst_, st_.p, sizeof(GState), cudaMemcpyDeviceToHost, ctx_.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx_.stream));
  return *hst_;
}

void GreedyEngine::launch_backward(const GView& g) {
  const bool tail = !std::getenv("IMB_BW_OLD_TAIL");  // A/B of the row-tail schedule
  if (tail) {
    if (xs_.p)
      k_backward_t<false, true><<<1, 64, bw_smem_, ctx_.stream>>>(g);
    else
      k_backward_t<true, true><<<1, 64, bw_smem_, ctx_.stream>>>(g);
  } else if (xs_.p) {
    k_backward_t<false, false><<<1, 64, bw_smem_, ctx_.stream>>>(g);
  } else {
    k_backward_t<true, false><<<1, 64, bw_smem_, ctx_.stream>>>(g);
  }
}

void GreedyEngine::launch_insert(const GView& g) {
  if (ins_ring_ == 4 && ins_threads_ == 256)
    k_insert<4, 256><<<1, 256, ins_smem_, ctx_.stream>>>(g);
  else if (ins_ring_ == 4 && ins_threads_ == 512)
    k_insert<4, 512><<<1, 512, ins_smem_, ctx_.stream>>>(g);
  else if (ins_ring_ == 4)
    k_insert<4><<<1, kInsertThreads, ins_smem_, ctx_.stream>>>(g);
  else
    k_insert<2><<<1, kInsertThreads, ins_smem_, ctx_.stream>>>(g);
}

void GreedyEngine::enqueue_step(bool sweep) {
  const GView g = view();
  launch_insert(g);
  launch_backward(g);
  if (sweep && sweep_kind_ >= 0) {
    switch (sweep_kind_) {
      case C0: k_sweep<C0><<<nblk_, kSweepThreads, 0, ctx_.stream>>>(g); break;
      case C2: k_sweep<C2><<<nblk_, kSweepThreads, 0, ctx_.stream>>>(g); break;
      case C4: k_sweep<C4><<<nblk_, kSweepThreads, 0, ctx_.stream>>>(g); break;
      default: k_sweep<C6><<<nblk_, kSweepThreads, 0, ctx_.stream>>>(g); break;
    }
  } else if (sweep)
    k_sweep<-1><<<nblk_, kSweepThreads, 0, ctx_.stream>>>(g);
  else
    k_next_in_order<<<1, 1, 0, ctx_.stream>>>(g, n_);
  IMB_LAUNCH_CHECK();
}

const GState& GreedyEngine::run_level(int batch) {
  for (;;) {
    for (int b = 0; b < batch; ++b) enqueue_step(true);
    const GState& s = poll();
    if (s.status != kStatusRunning) return s;
    batch = std::min(batch * 2, 256);
  }
}

const GState& GreedyEngine::factor_all_and_solve() {
  // solve_weights: append every point in order (rbf.cpp:165-178); only the
  // last backward solve matters, but the intermediate ones are cheap next
  // to the O(n^2) append at these sizes and keep one code path.
  const GView g = view();
  for (int k = 0; k < n_; ++k) {
    launch_insert(g);
    k_next_in_order<<<1, 1, 0, ctx_.stream>>>(g, n_);
  }
  launch_backward(g);
  IMB_LAUNCH_CHECK();
  return poll();
}

void GreedyEngine::download(int nc, size_t* idx, double* alpha_aos, double* residual_aos,
                            double* rec_err, double* rec_sec, int steps) {
  std::vector<int> ci(nc);
  std::vector<double> ax(nc), ay(nc), az(nc);
  if (nc) {
    IMB_CHECK(cudaMemcpyAsync(ci.data(), cidx_.p, nc * 4, cudaMemcpyDeviceToHost, ctx_.stream));
    IMB_CHECK(cudaMemcpyAsync(ax.data(), alpha_.x.p, nc * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    IMB_CHECK(cudaMemcpyAsync(ay.data(), alpha_.y.p, nc * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    IMB_CHECK(cudaMemcpyAsync(az.data(), alpha_.z.p, nc * 8, cudaMemcpyDeviceToHost, ctx_.stream));
  }
  std::vector<double> rx, ry, rz;
  if (residual_aos) {
    rx.resize(n_), ry.resize(n_), rz.resize(n_);
    IMB_CHECK(cudaMemcpyAsync(rx.data(), res_.x.p, n_ * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    IMB_CHECK(cudaMemcpyAsync(ry.data(), res_.y.p, n_ * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    IMB_CHECK(cudaMemcpyAsync(rz.data(), res_.z.p, n_ * 8, cudaMemcpyDeviceToHost, ctx_.stream));
  }
  if (rec_err && steps)
    IMB_CHECK(cudaMemcpyAsync(rec_err, rec_err_.p, steps * 8, cudaMemcpyDeviceToHost, ctx_.stream));
  if (rec_sec && steps)
    IMB_CHECK(cudaMemcpyAsync(rec_sec, rec_sec_.p, steps * 8, cudaMemcpyDeviceToHost, ctx_.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx_.stream));
  for (int i = 0; i < nc; ++i) {
    if (idx) idx[i] = (size_t)ci[i];
    if (alpha_aos) alpha_aos[3 * i] = ax[i], alpha_aos[3 * i + 1] = ay[i], alpha_aos[3 * i + 2] = az[i];
  }
  if (residual_aos)
    for (int i = 0; i < n_; ++i)
      residual_aos[3 * i] = rx[i], residual_aos[3 * i + 1] = ry[i], residual_aos[3 * i + 2] = rz[i];
}

}  // namespace imb

// ---------------------------------------------------------------------------
// Diagnostics: time the exact backward chain alone on a synthetic factor
// (unit diagonal, small off-diagonal entries) of size n, to report the
// chain's cycles per element against the 8-cycle dependent-DSUB floor.
// ---------------------------------------------------------------------------
namespace imb {
namespace {
__global__ void k_fill_synthetic(GView g, int n) {
  const size_t cap = g.cap;
  const size_t total = cap * (cap + 1) / 2;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    // column-major packed: find (i, off) lazily via the hash of t
    const unsigned long long h = (t + 1) * 0x9E3779B97F4A7C15ull;
    g.Lt[t] = ((double)(h >> 11) * 0x1.0p-53 - 0.5) * 1e-3;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    g.Lt[colstart(i, cap)] = 1.0;
    const exact::Recip r = exact::make_recip(1.0);
    g.diag[i] = make_double2(1.0, r.y);
    g.yx[i] = 1.0 + i * 1e-6, g.yy[i] = -1.0, g.yz[i] = 0.5;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g.st->status = 0;
    g.st->nc = n;
  }
}
}  // namespace

double GreedyEngine::bench_backward(int n, int reps) {
  const GView g = view();
  k_fill_synthetic<<<256, 256, 0, ctx_.stream>>>(g, n);
  launch_backward(g);  // warm
  cudaEvent_t a, b;
  IMB_CHECK(cudaEventCreate(&a));
  IMB_CHECK(cudaEventCreate(&b));
  IMB_CHECK(cudaEventRecord(a, ctx_.stream));
  for (int r = 0; r < reps; ++r) launch_backward(g);
  IMB_CHECK(cudaEventRecord(b, ctx_.stream));
  IMB_CHECK(cudaEventSynchronize(b));
  float ms = 0;
  IMB_CHECK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  IMB_LAUNCH_CHECK();
  return ms / reps;
}
}  // namespace imb

extern "C" int im_bench_backward_chain(im_context* ctx, int n, int reps, double* ms_per_solve) {
  try {
    imb::GreedyEngine eng(ctx->c, n, n);
    eng.reset(0.5, 1.0, 1, 1.0);
    *ms_per_solve = eng.bench_backward(n, reps);
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(ctx->c.message, sizeof ctx->c.message, "%s", e.what());
    return 3;
  }
}
