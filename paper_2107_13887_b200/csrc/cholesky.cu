// cholesky.cu — the reference's CholeskyFactor (rbf.hpp:41-60, rbf.cpp:71-121)
// and assemble_surface_matrix (rbf.hpp:35-36, rbf.cpp:56-69) on the device,
// behind the C-ABI (include/icemorph_b200.h, im_cholesky_* /
// im_assemble_surface_matrix).
//
// The factor lives in HBM in the greedy engine's layout (column-major packed
// lower triangle with a capacity that doubles as rows are appended) and uses
// the same device routines: append = gdev::insert_row with an explicit column
// (right-looking forward substitution in the reference's per-row order, the
// 1e-14 * max_diag pivot test of rbf.cpp:92), solve = the right-looking
// forward substitution (rbf.cpp:107-112) and the exact backward chain
// (rbf.cpp:114-120).  Results are bit-identical to the reference class; the
// error texts are the reference's.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/icemorph_b200.h"
#include "common.cuh"
#include "greedy_dev.cuh"
#include "runtime.hpp"

using namespace imb;

struct im_cholesky {
  im_context* ctx = nullptr;
  size_t n = 0, cap = 0;
  double max_diag = 0.0, smallest_pivot = 0.0;
  DBuf<double> Lt, col, rr, y, zero, xs, x, dummy;
  DBuf<double2> diag;
  DBuf<gdev::AppendOut> out;
};

namespace {

constexpr int kT = 1024;
constexpr size_t kSmemMax = 226 * 1024;
constexpr size_t kDynMax = 200 * 1024;  // dynamic smem next to the panel kernels' ~25 KB static

// columns of L in flight in shared memory (0: L and the row read from global
// memory; IMB_INSERT_RING0=1 forces it, for tests at small sizes)
int ring_for(size_t cap) {
  if (const char* e = std::getenv("IMB_INSERT_RING0"))
    if (e[0] == '1') return 0;
  return cap * 8 * 5 <= kDynMax ? 4 : cap * 8 * 3 <= kDynMax ? 2 : 0;
}

template <int NR>
__global__ void __launch_bounds__(kT) k_chol_append(gdev::InsertIO io, int k, const double* col,
                                                     double max_diag, gdev::AppendOut* out) {
  extern __shared__ double sh[];
  const gdev::AppendOut a = gdev::insert_row<NR, kT>(io, k, -1, col, max_diag, sh);
  if (threadIdx.x == 0) *out = a;
}

// L y = rhs (rbf.cpp:107-112), right-looking: each y_i receives its
// subtractions in ascending j as in the reference's left-looking loop.
template <int NR>
__global__ void __launch_bounds__(kT) k_chol_forward(const double* Lt, const double2* diag,
                                                      size_t cap, int n, const double* rhs,
                                                      double* rr_global, double* y) {
  extern __shared__ double sh[];
  double* rr = NR > 0 ? sh : rr_global;
  for (int j = threadIdx.x; j < n; j += kT) rr[j] = rhs[j];
  gdev::forward_subst_any<NR, kT>(Lt, diag, cap, n, rr, sh + cap);
  for (int j = threadIdx.x; j < n; j += kT) y[j] = rr[j];
}

// L^T x = y (rbf.cpp:114-120): the exact backward chain on one right-hand
// side (the chain's other two lanes run on zeros).
template <bool XS_SMEM>
__global__ void __launch_bounds__(64) k_chol_backward(gdev::ChainIO io, int n) {
  extern __shared__ __align__(16) double sh[];
  gdev::chain_solve<XS_SMEM, true>(io, n, sh, gdev::NoAbort{});
}

__global__ void k_chol_relayout(const double* from, size_t from_cap, double* to, size_t to_cap,
                                size_t n) {
  // column i, rows i..n-1 (offsets 0..n-1-i)
  for (size_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* s = from + gdev::colstart(i, from_cap);
    double* d = to + gdev::colstart(i, to_cap);
    for (size_t e = threadIdx.x; e < n - i; e += blockDim.x) d[e] = s[e];
  }
}

// rbf.cpp:56-69: entry (i, j) = phi(distance(points[i], points[j])) for the
// upper pair i < j, mirrored; unit diagonal.  Row-major n x n.
__global__ void k_assemble(const double* px, const double* py, const double* pz, size_t n,
                           int kind, double R, double* out) {
  const exact::Recip rR = exact::make_recip(R);
  const size_t total = n * n;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / n, c = t % n;
    if (r == c) {
      out[t] = 1.0;
      continue;
    }
    const size_t i = r < c ? r : c, j = r < c ? c : r;
    const double d = exact::dist(px[i], py[i], pz[i], px[j], py[j], pz[j]);
    out[t] = exact::wendland_rt(kind, exact::div_rcp(d, rR));
  }
}

template <class F>
int chol_guarded(im_cholesky* f, F&& fn) {
  if (!f || !f->ctx) return IM_INVALID_ARGUMENT;
  Context& c = f->ctx->c;
  try {
    IMB_CHECK(cudaSetDevice(c.device));
    fn(c);
    c.status = IM_OK;
    c.message[0] = 0;
  } catch (const InvalidArgument& e) {
    c.status = IM_INVALID_ARGUMENT;
    std::snprintf(c.message, sizeof c.message, "%s", e.what());
  } catch (const SolveFailure& e) {
    c.status = IM_SOLVE_ERROR;
    std::snprintf(c.message, sizeof c.message, "%s", e.what());
  } catch (const std::exception& e) {
    c.status = IM_RUNTIME_ERROR;
    std::snprintf(c.message, sizeof c.message, "%s", e.what());
  }
  return c.status;
}

void grow(im_cholesky& f, Context& c, size_t need) {
  if (need <= f.cap) return;
  size_t cap = std::max<size_t>(64, f.cap);
  while (cap < need) cap *= 2;
  DBuf<double> L;
  L.reserve(cap * (cap + 1) / 2 + 4);  // +4: the chain's 16-byte rounded bulk copies
  IMB_CHECK(cudaMemsetAsync(L.p, 0, (cap * (cap + 1) / 2 + 4) * 8, c.stream));
  if (f.n)
    k_chol_relayout<<<(unsigned)std::min<size_t>(f.n, 4096), 256, 0, c.stream>>>(f.Lt.p, f.cap,
                                                                              L.p, cap, f.n);
  DBuf<double2> d;
  d.reserve(cap);
  if (f.n)
    IMB_CHECK(cudaMemcpyAsync(d.p, f.diag.p, f.n * sizeof(double2), cudaMemcpyDeviceToDevice,
                              c.stream));
  IMB_CHECK(cudaStreamSynchronize(c.stream));
  f.Lt = std::move(L);
  f.diag = std::move(d);
  f.cap = cap;
  f.col.reserve(cap + 1);
  f.y.reserve(cap);
  f.x.reserve(cap);
  f.dummy.reserve(2 * cap);
  f.zero.reserve(cap);
  IMB_CHECK(cudaMemsetAsync(f.zero.p, 0, cap * 8, c.stream));
  if (ring_for(cap) == 0) f.rr.reserve(cap);
}

}  // namespace

extern "C" {

int im_cholesky_create(im_context* ctx, im_cholesky** out) {
  if (!ctx || !out) return IM_INVALID_ARGUMENT;
  *out = nullptr;
  auto* f = new (std::nothrow) im_cholesky();
  if (!f) return IM_RUNTIME_ERROR;
  f->ctx = ctx;
  const int rc = chol_guarded(f, [&](Context&) { f->out.reserve(1); });
  if (rc != IM_OK) {
    delete f;
    return rc;
  }
  *out = f;
  return IM_OK;
}

int im_cholesky_destroy(im_cholesky* f) {
  delete f;
  return IM_OK;
}

size_t im_cholesky_size(const im_cholesky* f) { return f ? f->n : 0; }
double im_cholesky_smallest_pivot(const im_cholesky* f) { return f ? f->smallest_pivot : 0.0; }

// CholeskyFactor::append (rbf.cpp:71-100)
int im_cholesky_append(im_cholesky* f, const double* column, size_t length) {
  return chol_guarded(f, [&](Context& c) {
    if (length != f->n + 1)
      throw InvalidArgument("column length must be current size + 1");
    grow(*f, c, f->n + 1);
    IMB_CHECK(cudaMemcpyAsync(f->col.p, column, length * 8, cudaMemcpyHostToDevice, c.stream));
    gdev::InsertIO io{};
    io.Lt = f->Lt.p, io.cap = f->cap, io.diag = f->diag.p, io.rr_global = f->rr.p;
    const int nr = ring_for(f->cap);
    const size_t smem = nr ? f->cap * 8 * (1 + nr) : 0;
    const int k = (int)f->n;
    switch (nr) {
      case 4:
        IMB_CHECK(cudaFuncSetAttribute(k_chol_append<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        k_chol_append<4><<<1, kT, smem, c.stream>>>(io, k, f->col.p, f->max_diag, f->out.p);
        break;
      case 2:
        IMB_CHECK(cudaFuncSetAttribute(k_chol_append<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        k_chol_append<2><<<1, kT, smem, c.stream>>>(io, k, f->col.p, f->max_diag, f->out.p);
        break;
      default:
        k_chol_append<0><<<1, kT, 0, c.stream>>>(io, k, f->col.p, f->max_diag, f->out.p);
    }
    IMB_LAUNCH_CHECK();
    gdev::AppendOut a;
    sync_copy(c.stream, &a, f->out.p, sizeof a, cudaMemcpyDeviceToHost);
    f->max_diag = a.max_diag;  // updated before the test, kept on failure (rbf.cpp:89-96)
    if (!a.ok)
      throw SolveFailure("matrix not numerically positive definite at row " + std::to_string(k) +
                         " (pivot " + std::to_string(a.pivot) + ")");
    if (f->n == 0 || a.pivot < f->smallest_pivot) f->smallest_pivot = a.pivot;
    ++f->n;
  });
}

// CholeskyFactor::solve (rbf.cpp:102-121)
int im_cholesky_solve(const im_cholesky* fc, const double* rhs, size_t rhs_length, double* x,
                      size_t x_length) {
  im_cholesky* f = const_cast<im_cholesky*>(fc);
  return chol_guarded(f, [&](Context& c) {
    if (rhs_length != f->n || x_length != f->n)
      throw InvalidArgument("rhs size does not match factorization");
    const int n = (int)f->n;
    if (n == 0) return;
    IMB_CHECK(cudaMemcpyAsync(f->col.p, rhs, f->n * 8, cudaMemcpyHostToDevice, c.stream));
    const int nr = ring_for(f->cap);
    const size_t smem = nr ? f->cap * 8 * (1 + nr) : 0;
    switch (nr) {
      case 4:
        IMB_CHECK(cudaFuncSetAttribute(k_chol_forward<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        k_chol_forward<4><<<1, kT, smem, c.stream>>>(f->Lt.p, f->diag.p, f->cap, n, f->col.p,
                                                     f->rr.p, f->y.p);
        break;
      case 2:
        IMB_CHECK(cudaFuncSetAttribute(k_chol_forward<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
        k_chol_forward<2><<<1, kT, smem, c.stream>>>(f->Lt.p, f->diag.p, f->cap, n, f->col.p,
                                                     f->rr.p, f->y.p);
        break;
      default:
        k_chol_forward<0><<<1, kT, 0, c.stream>>>(f->Lt.p, f->diag.p, f->cap, n, f->col.p, f->rr.p,
                                                  f->y.p);
    }
    IMB_LAUNCH_CHECK();
    const size_t head = gdev::chain_smem_head();
    const bool xs_smem = f->cap * 32 + head <= kSmemMax;
    if (!xs_smem) f->xs.reserve(4 * f->cap);
    gdev::ChainIO io{f->Lt.p,  f->cap,         f->diag.p,          f->y.p, f->zero.p,
                     f->zero.p, f->x.p,         f->dummy.p,         f->dummy.p + f->cap,
                     f->xs.p};
    const size_t bsm = xs_smem ? f->cap * 32 + head : head;
    if (xs_smem) {
      IMB_CHECK(cudaFuncSetAttribute(k_chol_backward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(bsm, 48 * 1024)));
      k_chol_backward<true><<<1, 64, bsm, c.stream>>>(io, n);
    } else {
      IMB_CHECK(cudaFuncSetAttribute(k_chol_backward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(bsm, 48 * 1024)));
      k_chol_backward<false><<<1, 64, bsm, c.stream>>>(io, n);
    }
    IMB_LAUNCH_CHECK();
    sync_copy(c.stream, x, f->x.p, f->n * 8, cudaMemcpyDeviceToHost);
  });
}

// assemble_surface_matrix (rbf.cpp:56-69); out: n * n doubles, row-major
int im_assemble_surface_matrix(im_context* ctx, const double* points, size_t n, im_basis basis,
                               double* out) {
  if (!ctx) return IM_INVALID_ARGUMENT;
  im_cholesky tmp;  // only for the guarded error reporting
  tmp.ctx = ctx;
  return chol_guarded(&tmp, [&](Context& c) {
    if (basis.kind < 0 || basis.kind > 3)
      throw InvalidArgument("unknown basis function (expected c0, c2, c4 or c6)");
    if (n == 0) return;
    DPoints p;
    upload_points(c, points, n, p);
    DBuf<double> m;
    m.reserve(n * n);
    const size_t total = n * n;
    const unsigned grid = (unsigned)std::min<size_t>((total + 255) / 256, (size_t)c.num_sms * 16);
    k_assemble<<<grid, 256, 0, c.stream>>>(p.x.p, p.y.p, p.z.p, n, basis.kind,
                                           basis.support_radius, m.p);
    IMB_LAUNCH_CHECK();
    sync_copy(c.stream, out, m.p, total * 8, cudaMemcpyDeviceToHost);
  });
}

}  // extern "C"
