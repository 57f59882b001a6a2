// greedy_dev.cuh — device building blocks of the exact greedy (greedy.cu,
// greedy_spec.cu): packed-column addressing, async-copy / mbarrier wrappers,
// the row append of the incremental Cholesky factor (rbf.cpp:71-100) and the
// backward-substitution chain (rbf.cpp:114-120).
//
// L is stored column-major packed: column i = rows i..cap-1 contiguous,
// starting at colstart(i, cap).  Both the append (right-looking forward
// substitution over columns) and the backward chain (column i of L = row i of
// L^T) walk columns.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace imb {
namespace gdev {

__device__ __forceinline__ size_t colstart(size_t i, size_t cap) {
  return i * cap - i * (i - 1) / 2;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_volatile(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// max value, lowest index on ties (the reference's sequential strict '>' scan)
__device__ __forceinline__ void better(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) v = v2, i = i2;
}

// ---- cp.async (k_insert's column ring) ---------------------------------------
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- mbarrier + bulk async copy (the chain's L stream) --------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_addr(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// Forward substitution and row append: rbf.cpp:71-100 / rbf.cpp:107-112
//
// forward_subst solves L s = b for the first k rows, right-looking: once
// s_m is final (s_m / L_mm), every s_j (j > m) does s_j -= L_jm * s_m, so
// each s_j receives its subtractions in ascending m exactly as in the
// reference's inner loops (rbf.cpp:84, rbf.cpp:110).  Shared memory (NR >= 2):
// rr[cap] (running s_j) | ring[NR][cap] (columns m .. m+NR-1 of L, streamed
// by cp.async NR-1 steps ahead: every thread copies exactly the rows it
// owns, so cp.async.wait_group alone orders the copy before its own use and
// no barrier guards the ring).  NR == 0 (factors too large for shared
// memory): rr in global memory, L read directly.  The pivot pair (L_mm,
// 1/L_mm) of row m is held in a register by m's owner thread, loaded T steps
// ahead.  Per step the critical path is the owner's division, one barrier
// and the next owner's mul-sub.
// ---------------------------------------------------------------------------
template <int NR, int T>
__device__ void forward_subst(const double* Lt, const double2* diag, size_t cap, int k, double* rr,
                              double* ring, size_t rs) {  // rs: ring slot stride (>= k)
  const int tid = threadIdx.x;
  double2 dm = tid < k ? diag[tid] : make_double2(1.0, 1.0);  // pivot of my next row
  int mi = 0, ji = tid > 0 ? tid : T;  // next column to issue, my first row > mi
  const double* ci = Lt;               // its start, colstart(mi, cap)
  auto issue_next = [&]() {
    if (NR > 0) {
      if (mi < k) {
        double* dst = ring + (mi & (NR - 1)) * rs;
        for (int j = ji; j < k; j += T) cp_async8(dst + j, ci + (j - mi));
      }
      cp_async_commit();
    }
    ci += cap - (size_t)mi;  // colstart(mi + 1) = colstart(mi) + cap - mi
    ++mi;
    if (ji == mi) ji += T;
  };
  if (NR > 0) {
#pragma unroll
    for (int q = 0; q < NR - 1; ++q) issue_next();
  }
  __syncthreads();
  int ju = tid > 0 ? tid : T;  // my first row > m
  const double* cm = Lt;       // colstart(m, cap) (NR == 0)
  for (int m = 0; m < k; ++m) {
    if ((m & (T - 1)) == tid) {
      rr[m] = exact::div_rcp(rr[m], exact::Recip{dm.x, dm.y});  // s / L_mm
      if (m + T < k) dm = diag[m + T];
    }
    if (NR > 0) {
      issue_next();             // column m + NR - 1
      cp_async_wait<NR - 1>();  // my copies of column m have landed
    }
    __syncthreads();
    const double r = rr[m];
    if (NR > 0) {
      const double* lc = ring + (m & (NR - 1)) * rs;
      for (int j = ju; j < k; j += T) rr[j] = exact::sub(rr[j], exact::mul(lc[j], r));
    } else {
      for (int j = ju; j < k; j += T) rr[j] = exact::sub(rr[j], exact::mul(cm[j - m], r));
      cm += cap - (size_t)m;
    }
    if (ju == m + 1) ju += T;
  }
  if (NR > 0) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}

// forward_subst for a single CTA.  (A single SM streams L at only ~30-40
// GB/s, so the per-column form with its cp.async ring is as fast as a
// 32-column panel form here; the speculative pipeline's predictor spreads
// the substitution over a cluster instead, greedy_predict.cuh.)
template <int NR, int T>
__device__ void forward_subst_any(const double* Lt, const double2* diag, size_t cap, int k,
                                  double* rr, double* ring) {
  forward_subst<NR, T>(Lt, diag, cap, k, rr, ring, cap);
}

struct InsertIO {
  const double *px, *py, *pz;  // surface positions (greedy) -- unused with col_in
  const double *tx, *ty, *tz;  // level target (rhs = target[c_k], greedy.cpp:104); null: no y
  const double *cx, *cy, *cz;  // control positions c_0..c_{k-1} (insertion order)
  double* Lt;
  size_t cap;
  double2* diag;               // (L_kk, refined reciprocal)
  double *yx, *yy, *yz;        // forward solutions y_0..y_{k-1} in, y_k out
  int kind;
  double R;
  double* rr_global;           // [cap] scratch when NR == 0
};

struct AppendOut {
  double pivot, max_diag;
  bool ok;
};

// Appends row k (rbf.cpp:71-100).  The new column is col_in[0..k] when given
// (CholeskyFactor::append), else phi(|c_m - p_node|) with diagonal 1.0
// (greedy.cpp:87-93).  max_diag is the factor's running maximum diagonal,
// updated before the pivot test as in rbf.cpp:89.  On success (pivot >
// 1e-14 * max_diag, rbf.cpp:92) writes diag[k], L_kk, the row L_k0..L_k,k-1
// into the columns and, when the target is given, y_k.  On failure writes
// nothing to L.  Every thread returns the same value.
template <int NR, int T>
__device__ AppendOut insert_row(const InsertIO& g, int k, int node, const double* col_in,
                                double max_diag, double* sh) {
  __shared__ double s_pivot, s_maxd;
  __shared__ int s_ok;
  const size_t cap = g.cap;
  double* rr = NR > 0 ? sh : g.rr_global;  // [cap]
  double* ring = sh + cap;                 // [NR][cap]
  const int tid = threadIdx.x;
  if (col_in) {
    for (int j = tid; j < k; j += T) rr[j] = col_in[j];
  } else {
    // column (greedy.cpp:87-93 / rbf.cpp:167-170): phi(distance(c_m, p_new))
    const double px = g.px[node], py = g.py[node], pz = g.pz[node];
    const exact::Recip rR = exact::make_recip(g.R);
    for (int j = tid; j < k; j += T) {
      const double d = exact::dist(g.cx[j], g.cy[j], g.cz[j], px, py, pz);
      rr[j] = exact::wendland_rt(g.kind, exact::div_rcp(d, rR));
    }
  }
  forward_subst_any<NR, T>(g.Lt, g.diag, cap, k, rr, ring);
  // stage y_0..y_{k-1} for the forward chain in the ring space when it fits
  const bool with_y = g.tx != nullptr;
  const double *yxs = g.yx, *yys = g.yy, *yzs = g.yz;
  if (NR >= 3 && with_y) {
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
    double yx = 0.0, yy = 0.0, yz = 0.0;
    if (with_y) {
      yx = g.tx[node], yy = g.ty[node], yz = g.tz[node];  // rhs_k = target[c_k]
#pragma unroll 8
      for (int j = 0; j < k; ++j) {
        const double r = rr[j];
        sq = exact::add(sq, exact::mul(r, r));
        yx = exact::sub(yx, exact::mul(r, yxs[j]));
        yy = exact::sub(yy, exact::mul(r, yys[j]));
        yz = exact::sub(yz, exact::mul(r, yzs[j]));
      }
    } else {
#pragma unroll 8
      for (int j = 0; j < k; ++j) sq = exact::add(sq, exact::mul(rr[j], rr[j]));
    }
    const double diag = col_in ? col_in[k] : 1.0;  // column[k] (greedy.cpp:93, rbf.cpp:88)
    max_diag = (max_diag < diag) ? diag : max_diag;  // std::max (rbf.cpp:89)
    const double pivot_sq = exact::sub(diag, sq);
    const double pivot = pivot_sq > 0.0 ? __dsqrt_rn(pivot_sq) : 0.0;
    s_pivot = pivot;
    s_maxd = max_diag;
    s_ok = pivot > exact::mul(1e-14, max_diag);
    if (s_ok) {
      const exact::Recip pr = exact::make_recip(pivot);
      g.diag[k] = make_double2(pivot, pr.y);
      g.Lt[colstart(k, cap)] = pivot;
      if (with_y) {
        g.yx[k] = exact::div_rcp(yx, pr);
        g.yy[k] = exact::div_rcp(yy, pr);
        g.yz[k] = exact::div_rcp(yz, pr);
      }
    }
  }
  __syncthreads();
  AppendOut out{s_pivot, s_maxd, s_ok != 0};
  if (out.ok)  // scatter the new row into the columns: L_kj at column j, offset k - j
    for (int j = tid; j < k; j += T) g.Lt[colstart(j, cap) + (k - j)] = rr[j];
  return out;
}

// ---------------------------------------------------------------------------
// Backward chain: rbf.cpp:114-120 for x, y, z (greedy.cpp:106-111).
//
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
// Padding rows beyond n contribute +0.0, an exact identity for subtraction.
//
// Abort (the speculative driver, greedy_spec.cu): the consumer polls
// `abort()` once per block (a load issued at the block's start and tested at
// its end, off the dependent chain); on abort it raises a shared flag before
// releasing its buffer, the producer leaves at its next block and waits for
// its outstanding bulk copies, so the CTA can be reused at once.
// ---------------------------------------------------------------------------
constexpr int kBwRing = 8;     // blocks of L in flight
constexpr int kBwBlock = 512;  // doubles per block
constexpr int kBwPad = kBwBlock + 32;

struct ChainIO {
  const double* Lt;
  size_t cap;
  const double2* diag;
  const double *yx, *yy, *yz;
  double *ox, *oy, *oz;  // x (alpha) out
  double* xs_global;     // 4 * cap workspace when x does not fit in smem
};

struct BwBlock {
  int i, e0;  // column i, elements e0.. of rows j = i+1+e
};

// shared memory bytes of chain_solve: barriers, L ring, products (+ x, D)
__host__ __device__ constexpr size_t chain_smem_head() {
  return (size_t)(8 + 8 + 8 * (kBwBlock + 2) + 6 * kBwPad) * 8;
}

// abort policy of chain_solve: poll_issue() issues the loads (at a block's
// start), poll_test(token) decides (at its end), so the load latency stays
// off the dependent chain
struct NoAbort {
  __device__ int poll_issue() const { return 0; }
  __device__ bool poll_test(int) const { return false; }
};

// Returns true when the solve completed (and x was written to io.o*), false
// when aborted.  Must be called by all 64 threads of the CTA.
template <bool XS_SMEM, bool TAIL, class Abort>
__device__ bool chain_solve(const ChainIO& g, int n, double* sh, const Abort& abort) {
  __shared__ int s_abort;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  if (n <= 0) return true;
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
    for (int r = 0; r < kBwRing + 4; ++r) mbar_init(&ringbar[r]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_abort = 0;
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
      bulk_load(ring + slot * (kBwBlock + 2), al, bytes, &ringbar[slot]);
    };
    BwBlock cur{n - 2, 0}, ahead = cur;
    int issued = 0;
    for (int r = 0; r < kBwRing; ++r) {
      if (ahead.i >= 0) ++issued;
      issue(ahead, r);
      ahead = next(ahead);
    }
    int t = 0;
    for (; cur.i >= 0; ++t) {
      if (*(volatile int*)&s_abort) break;
      const int slot = t % kBwRing, pb = t & 1;
      int off, cnt;
      src_of(cur, off, cnt);
      mbar_wait(&ringbar[slot], (uint32_t)((t / kBwRing) & 1));
      mbar_wait(&empty[pb], (uint32_t)(((t >> 1) & 1) ^ 1));
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
        mbar_arrive(&full[pb]);
      }
      if (ahead.i >= 0) ++issued;
      issue(ahead, slot);  // refill the slot just consumed
      ahead = next(ahead);
      cur = next(cur);
    }
    // drain: every bulk copy issued past block t must land before the CTA
    // reuses its shared memory
    for (int q = t; q < issued; ++q) mbar_wait(&ringbar[q % kBwRing], (uint32_t)((q / kBwRing) & 1));
  } else if (lane < 3) {
    // ---------------- consumer ----------------
    double* cx = comp + (size_t)lane * cap;
    BwBlock cur{n - 2, 0};
    double s = 0.0, rcp_i = 0.0;
    for (int t = 0; cur.i >= 0; ++t) {
      const int pb = t & 1, i = cur.i;
      const auto ab_pending = abort.poll_issue();
      int off, cnt;
      src_of(cur, off, cnt);
      mbar_wait(&full[pb], (uint32_t)((t >> 1) & 1));
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
      if (nx.i != i)  // x_i = s / L_ii, reciprocal of L_ii from the insert (prefetched)
        cx[i] = exact::div_rcp(s, TAIL ? exact::Recip{dd[i], rcp_i} : exact::make_recip(dd[i]));
      const bool ab = __shfl_sync(0x7u, (int)abort.poll_test(ab_pending), 0) != 0;
      __syncwarp(0x7u);
      if (ab && lane == 0) *(volatile int*)&s_abort = 1;  // before the release below
      if (lane == 0) mbar_arrive(&empty[pb]);
      cur = nx;
      if (ab) break;
    }
  }
  __syncthreads();
  const bool aborted = s_abort != 0;
  if (tid == 0)
    for (int r = 0; r < kBwRing + 4; ++r) mbar_inval(&ringbar[r]);
  if (!aborted)
    for (int i = tid; i < n; i += 64)
      g.ox[i] = comp[i], g.oy[i] = comp[cap + i], g.oz[i] = comp[2 * cap + i];
  __syncthreads();
  return !aborted;
}

}  // namespace gdev
}  // namespace imb
