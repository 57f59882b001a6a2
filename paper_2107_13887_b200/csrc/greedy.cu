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
#include "greedy_dev.cuh"
#include "greedy_sweep.cuh"

namespace imb {

namespace {

constexpr int kInsertThreads = 1024;
constexpr int kSweepThreads = gsw::kT;  // greedy_sweep.cuh: 8 warps x 32 points

using gdev::colstart;
using gdev::globaltimer;
using gdev::better;

// ---------------------------------------------------------------------------
// k_insert: greedy.cpp:86-112 / rbf.cpp:71-100 on the engine's step state
// (the row append itself is gdev::insert_row, greedy_dev.cuh)
// ---------------------------------------------------------------------------
template <int NR, int T = kInsertThreads>
__global__ void __launch_bounds__(T) k_insert(GView g) {
  GState& st = *g.st;
  if (st.status != 0) return;
  extern __shared__ double sh[];
  const int k = st.nc;
  const int node = st.next;
  if (k == 0 && threadIdx.x == 0) st.t0 = globaltimer();
  gdev::InsertIO io{g.px, g.py, g.pz, g.tx, g.ty, g.tz, g.cx, g.cy, g.cz, g.Lt, (size_t)g.cap,
                    g.diag, g.yx, g.yy, g.yz, g.kind, g.R, g.rr_global};
  const gdev::AppendOut a = gdev::insert_row<NR, T>(io, k, node, nullptr, st.max_diag, sh);
  const bool ok = a.ok;
  const double pivot = a.pivot;
  if (threadIdx.x == 0) {
    st.max_diag = a.max_diag;
    if (!ok) {
      st.status = kStatusSolveError;
      st.fail_node = node;
      st.fail_row = k;
      st.fail_pivot = pivot;
    } else {
      if (k == 0 || pivot < st.smallest_pivot) st.smallest_pivot = pivot;
      g.cidx[k] = node;
      g.cx[k] = g.px[node], g.cy[k] = g.py[node], g.cz[k] = g.pz[node];
      g.sel[node] = 1;
      st.nc = k + 1;
    }
  }
}

// ---------------------------------------------------------------------------
// k_backward_t: rbf.cpp:114-120 for x, y, z (greedy.cpp:106-111); the chain
// itself is gdev::chain_solve (greedy_dev.cuh)
// ---------------------------------------------------------------------------
template <bool XS_SMEM, bool TAIL>
__global__ void __launch_bounds__(64) k_backward_t(GView g) {
  const GState& st = *g.st;
  if (st.status != 0) return;
  extern __shared__ __align__(16) double sh[];
  gdev::ChainIO io{g.Lt, (size_t)g.cap, g.diag, g.yx, g.yy, g.yz, g.ax, g.ay, g.az, g.xs_global};
  gdev::chain_solve<XS_SMEM, TAIL>(io, st.nc, sh, gdev::NoAbort{});
}

// ---------------------------------------------------------------------------
// k_sweep: greedy.cpp:122-153
// ---------------------------------------------------------------------------

// KIND >= 0: the staged pair evaluation of the tiled exact kernels
// (xt::/exact_eval, common.cuh: four controls per stage, summed in insertion
// order) -- valid when the host verified |positions| <= 1e100 and R in
// [1e-100, 1e100] (exact_tiled_ok); KIND < 0: one pair at a time with the
// full-range __dsqrt_rn / division and a runtime basis switch.
template <int KIND>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(GView g) {
  GState& st = *g.st;
  if (st.status != 0) return;
  __shared__ __align__(16) gsw::Smem S;
  __shared__ double wv[kSweepThreads / 32], wa[kSweepThreads / 32];
  __shared__ int wi[kSweepThreads / 32];
  __shared__ bool last;
  const int n = g.n, nc = st.nc;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * gsw::kP + lane;
  const bool in = i < n;
  const double px = in ? g.px[i] : 0.0, py = in ? g.py[i] : 0.0, pz = in ? g.pz[i] : 0.0;
  // greedy_sweep.cuh: phi by all warps, the ordered sums one axis per warp (warps 0-2)
  gsw::interpolant<KIND>(S, g.cx, g.cy, g.cz, g.ax, g.ay, g.az, nc, g.R, g.kind, px, py, pz, true);
  const bool live = in && threadIdx.x < 32;  // warp 0 owns the points from here on
  const double fx = S.f[0][lane], fy = S.f[1][lane], fz = S.f[2][lane];
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
  if (!last) return;
  // final block: grid argmax + decision (greedy.cpp:136-152); the block
  // results are merged by all threads, then across the warps
  __threadfence();
  double mv = -1.0, ov = 0.0;
  int mi = n;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kSweepThreads) {
    better(mv, mi, ((volatile double*)g.bv)[b], ((volatile int*)g.bi)[b]);
    const double a = ((volatile double*)g.ba)[b];
    ov = (ov < a) ? a : ov;
  }
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, mv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, mi, o);
    better(mv, mi, v2, i2);
    const double a2 = __shfl_xor_sync(0xffffffffu, ov, o);
    ov = (ov < a2) ? a2 : ov;
  }
  __syncthreads();  // wv / wi / wa are reused
  if ((threadIdx.x & 31) == 0) wv[w] = mv, wi[w] = mi, wa[w] = ov;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int t = 1; t < kSweepThreads / 32; ++t) {
    better(mv, mi, wv[t], wi[t]);
    ov = (ov < wa[t]) ? wa[t] : ov;
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
  nblk_ = (n + gsw::kP - 1) / gsw::kP;
  bv_.reserve(nblk_);
  ba_.reserve(nblk_);
  bi_.reserve(nblk_);
  rec_err_.reserve(cap + 1);
  rec_sec_.reserve(cap + 1);
  st_.reserve(1);
  IMB_CHECK(cudaMallocHost(&hst_, sizeof(GState)));
  // x workspace of the backward chain: shared memory when it fits
  const size_t head = gdev::chain_smem_head();  // barriers, L ring, products
  const size_t xs_bytes = (size_t)cap * 32 + head;
  if (xs_bytes <= 226 * 1024) {
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
  // k_insert: rr + 4 columns of staging when it fits (cap <= 5120), else 2
  // (cap <= 8533), else rr in global memory and L read directly
  const size_t smem_max = 200 * 1024;  // + ~25 KB static of the panel substitution
  ins_ring_ = (size_t)cap * 8 * 5 <= smem_max && !std::getenv("IMB_INSERT_RING2") ? 4
              : (size_t)cap * 8 * 3 <= smem_max                                  ? 2
                                                                                  : 0;
  if (const char* e = std::getenv("IMB_INSERT_RING0"))
    if (e[0] == '1') ins_ring_ = 0;  // the global-memory variant, for tests at small sizes
  ins_smem_ = ins_ring_ ? (size_t)cap * 8 * (1 + ins_ring_) : 0;
  if (!ins_ring_) rr_.reserve(cap);
  if (const char* e = std::getenv("IMB_INSERT_T")) ins_threads_ = std::atoi(e);
  for (auto kern : {k_insert<4>, k_insert<4, 256>, k_insert<4, 512>, k_insert<2>, k_insert<0>})
    IMB_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::max<size_t>(ins_smem_, 48 * 1024)));
}

GreedyEngine::~GreedyEngine() {
  if (hst_) cudaFreeHost(hst_);
  spec_free();
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
  g.rr_global = rr_.p;
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
  tol_ = tol;
  target_max_ = target_max;
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
  else if (ins_ring_ == 2)
    k_insert<2><<<1, kInsertThreads, ins_smem_, ctx_.stream>>>(g);
  else
    k_insert<0><<<1, kInsertThreads, 0, ctx_.stream>>>(g);
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
  // the speculative pipeline (greedy_spec.cu) unless IMB_SPEC=0
  const char* e = std::getenv("IMB_SPEC");
  if (!(e && e[0] == '0') && (size_t)cap_ * 24 <= 200 * 1024) return run_level_spec();
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
