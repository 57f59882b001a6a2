// wall_distance.cu — K6 exact wall distance (north-star d).
//
// Reference: build_distance_index (wall_distance.cpp:13-31) builds a kd-tree
// over the patch nodes (kdtree.cpp:21-57) and queries the exact nearest
// distance of every mesh node (kdtree.cpp:59-87); patch nodes are then forced
// to exactly 0 (:29).  Only the VALUE is contractual, and
// any exact nearest-neighbour search returns the same value because
//   d = sqrt(min_s ((dx*dx + dy*dy) + dz*dz))       (vec.hpp:59, kdtree.cpp:79)
// and a min over exactly computed candidates is order independent.
//
// B200 design: a bounding-volume hierarchy over the patch, built on the
// device each call (as the reference builds its kd-tree each call):
//   * the surface points are sorted by a 63-bit Morton key over their box
//     (CUB radix sort) and cut into buckets of kLeaf consecutive points;
//   * an implicit complete binary tree over the buckets (heap order, leaves
//     padded to a power of two) -- Morton-order halving, so every node is a
//     compact region -- with axis-aligned boxes reduced bottom-up;
//   * one thread per query: a stack walk, nearer child first, pruning every
//     box whose lower bound exceeds min(best, cutoff^2) by a 1e-9 relative
//     margin (the box bound and the point distances are each within a few
//     ulps of exact), scanning bucket points with the exact squared distance
//     of App. A1.
// Queries farther than the cutoff from the whole patch exit after the root
// test: that IS the volume reduction's culling (HBM bound, 24 B in, 8 B out).
// A thin shell like the wing surface made the earlier uniform-grid ring
// search visit ~(2d/h)^3 mostly empty cells per query (9.7 GB/s at cfg4
// scale); the tree visits O(log N_s) boxes.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "runtime.hpp"

namespace imb {

namespace {

constexpr int kLeaf = 8;  // surface points per bucket

struct Tree {
  int L;                       // leaves (power of two)
  int n;                       // surface points
  const double* box;           // [2L][6]: lo xyz, hi xyz (heap order, root 1)
  const double *sx, *sy, *sz;  // Morton-sorted surface points
};

__device__ __forceinline__ unsigned long long spread21(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

__global__ void k_surface_keys(const double* x, const double* y, const double* z, int n, double ox,
                               double oy, double oz, double sx, double sy, double sz,
                               unsigned long long* key, unsigned int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto q = [](double v, double o, double s) {
    const double f = (v - o) * s;
    return (unsigned long long)(f <= 0.0 ? 0.0 : (f >= 2097151.0 ? 2097151.0 : f));
  };
  key[i] = spread21(q(x[i], ox, sx)) | spread21(q(y[i], oy, sy)) << 1 | spread21(q(z[i], oz, sz)) << 2;
  idx[i] = (unsigned)i;
}

__global__ void k_gather_sorted(const double* x, const double* y, const double* z,
                                const unsigned int* idx, int n, double* sx, double* sy,
                                double* sz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned int j = idx[i];
  sx[i] = x[j], sy[i] = y[j], sz[i] = z[j];
}

__global__ void k_leaf_boxes(Tree t, double* box) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= t.L) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int p = b * kLeaf; p < min((b + 1) * kLeaf, t.n); ++p) {
    const double v[3] = {t.sx[p], t.sy[p], t.sz[p]};
    for (int a = 0; a < 3; ++a) lo[a] = fmin(lo[a], v[a]), hi[a] = fmax(hi[a], v[a]);
  }
  double* o = box + (size_t)(t.L + b) * 6;
  for (int a = 0; a < 3; ++a) o[a] = lo[a], o[3 + a] = hi[a];
}

// internal nodes [first, 2 first) from their children (one tree level)
__global__ void k_inner_boxes(double* box, int first) {
  const int i = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * first) return;
  const double *l = box + (size_t)(2 * i) * 6, *r = box + (size_t)(2 * i + 1) * 6;
  double* o = box + (size_t)i * 6;
  for (int a = 0; a < 3; ++a) o[a] = fmin(l[a], r[a]), o[3 + a] = fmax(l[3 + a], r[3 + a]);
}

__device__ __forceinline__ double box_lb(const double* b, double qx, double qy, double qz) {
  const double gx = fmax(0.0, fmax(b[0] - qx, qx - b[3]));
  const double gy = fmax(0.0, fmax(b[1] - qy, qy - b[4]));
  const double gz = fmax(0.0, fmax(b[2] - qz, qz - b[5]));
  return gx * gx + gy * gy + gz * gz;
}

// every node: lower bound of its distance to the patch's root box against the
// cutoff -> +inf (out of range, final) or 0 (in range, to be searched)
__global__ void k_root_test(Tree t, const double* __restrict__ qx, const double* __restrict__ qy,
                            const double* __restrict__ qz, size_t n, double cutoff2, double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = box_lb(t.box + 6, qx[i], qy[i], qz[i]) * (1.0 - 1e-9) > cutoff2 ? INFINITY : 0.0;
}

// ids / order: the in-range nodes in spatial (Morton) order, or null = all n
// nodes in mesh order.  Neighbouring lanes then walk nearly the same boxes.
__global__ void __launch_bounds__(256) k_wall_distance(Tree t, const double* __restrict__ qx_,
                                                       const double* __restrict__ qy_,
                                                       const double* __restrict__ qz_,
                                                       const uint32_t* __restrict__ ids,
                                                       const uint32_t* __restrict__ order, size_t n,
                                                       double cutoff2, double* out) {
  const size_t kk = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kk >= n) return;
  const size_t i = ids ? ids[order[kk]] : kk;
  const double qx = qx_[i], qy = qy_[i], qz = qz_[i];
  const double margin = 1.0 - 1e-9;
  double best = INFINITY;
  // bound = min(best, cutoff^2): boxes whose lower bound exceeds it are skipped
  if (box_lb(t.box + 6, qx, qy, qz) * margin > cutoff2) {
    out[i] = INFINITY;  // farther than the cutoff from the whole patch
    return;
  }
  int stack[48];
  int sp = 0;
  stack[sp++] = 1;
  while (sp) {
    const int v = stack[--sp];
    const double* b = t.box + (size_t)v * 6;
    if (box_lb(b, qx, qy, qz) * margin > fmin(best, cutoff2)) continue;
    if (v >= t.L) {  // bucket: exact squared distances (App. A1 order)
      const int b0 = (v - t.L) * kLeaf, b1 = min(b0 + kLeaf, t.n);
      for (int p = b0; p < b1; ++p) {
        const double s = exact::sqdist(t.sx[p], t.sy[p], t.sz[p], qx, qy, qz);
        if (s < best) best = s;
      }
      continue;
    }
    const double ll = box_lb(t.box + (size_t)(2 * v) * 6, qx, qy, qz);
    const double lr = box_lb(t.box + (size_t)(2 * v + 1) * 6, qx, qy, qz);
    if (ll <= lr) {  // nearer child on top
      stack[sp++] = 2 * v + 1;
      stack[sp++] = 2 * v;
    } else {
      stack[sp++] = 2 * v;
      stack[sp++] = 2 * v + 1;
    }
  }
  out[i] = best < INFINITY ? __dsqrt_rn(best) : INFINITY;
}

}  // namespace

void wall_distance(Context& ctx, const DPoints& nodes, size_t n_nodes, const DPoints& surface,
                   size_t n_surface, int dim, double cutoff, double* d_out) {
  if (n_surface == 0) throw InvalidArgument("cannot build a distance index for an empty patch");
  if (dim != 2 && dim != 3) throw InvalidArgument("kd-tree dim must be 2 or 3");
  if (n_surface > (size_t)1 << 30) throw InvalidArgument("patch too large for the distance index");
  if (n_nodes == 0) return;
  const int ns = (int)n_surface;
  // bounding box of the patch (host: N_s <= ~1e5, one D2H of 3 arrays)
  std::vector<double> hx(n_surface), hy(n_surface), hz(n_surface);
  IMB_CHECK(cudaMemcpyAsync(hx.data(), surface.x.p, n_surface * 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaMemcpyAsync(hy.data(), surface.y.p, n_surface * 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaMemcpyAsync(hz.data(), surface.z.p, n_surface * 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (size_t i = 0; i < n_surface; ++i) {
    const double v[3] = {hx[i], hy[i], hz[i]};
    for (int a = 0; a < 3; ++a) lo[a] = std::min(lo[a], v[a]), hi[a] = std::max(hi[a], v[a]);
  }
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(lo[a]) || !std::isfinite(hi[a]))
      throw InvalidArgument("surface coordinates are not finite");
  double scale[3];
  for (int a = 0; a < 3; ++a) scale[a] = hi[a] > lo[a] ? 2097151.0 / (hi[a] - lo[a]) : 0.0;
  // implicit tree: L leaves (power of two >= buckets), boxes in heap order
  int L = 1;
  while ((size_t)L * kLeaf < n_surface) L *= 2;
  // every buffer of the build comes out of one grow-only context slot (no
  // cudaMalloc / cudaFree per call: with tens of GB resident they cost more
  // than the search itself)
  size_t temp = 0;
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, temp, (unsigned long long*)nullptr,
                                            (unsigned long long*)nullptr, (unsigned int*)nullptr,
                                            (unsigned int*)nullptr, ns, 0, 63, ctx.stream));
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_key = up(n_surface * 8), b_idx = up(n_surface * 4), b_pts = up(n_surface * 8),
               b_box = up((size_t)2 * L * 6 * 8), b_tmp = up(temp);
  unsigned char* base = ctx.buf<unsigned char>(Context::kSlotWallTree,
                                               2 * b_key + 2 * b_idx + 3 * b_pts + b_box + b_tmp);
  unsigned char* cur = base;
  auto take = [&](size_t b) {
    unsigned char* r = cur;
    cur += b;
    return r;
  };
  auto* ka = reinterpret_cast<unsigned long long*>(take(b_key));
  auto* kb = reinterpret_cast<unsigned long long*>(take(b_key));
  auto* ia = reinterpret_cast<unsigned int*>(take(b_idx));
  auto* ib = reinterpret_cast<unsigned int*>(take(b_idx));
  auto* sx = reinterpret_cast<double*>(take(b_pts));
  auto* sy = reinterpret_cast<double*>(take(b_pts));
  auto* sz = reinterpret_cast<double*>(take(b_pts));
  auto* box = reinterpret_cast<double*>(take(b_box));
  unsigned char* tbp = take(b_tmp);
  // Morton sort of the surface points
  const int T = 256;
  k_surface_keys<<<(ns + T - 1) / T, T, 0, ctx.stream>>>(surface.x.p, surface.y.p, surface.z.p, ns,
                                                          lo[0], lo[1], lo[2], scale[0], scale[1],
                                                          scale[2], ka, ia);
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(tbp, temp, ka, kb, ia, ib, ns, 0, 63,
                                            ctx.stream));
  k_gather_sorted<<<(ns + T - 1) / T, T, 0, ctx.stream>>>(surface.x.p, surface.y.p, surface.z.p,
                                                           ib, ns, sx, sy, sz);
  Tree t{L, ns, box, sx, sy, sz};
  k_leaf_boxes<<<(L + T - 1) / T, T, 0, ctx.stream>>>(t, box);
  for (int first = L / 2; first >= 1; first /= 2)
    k_inner_boxes<<<(first + T - 1) / T, T, 0, ctx.stream>>>(box, first);
  IMB_LAUNCH_CHECK();
  const double cutoff2 = std::isfinite(cutoff) ? cutoff * cutoff : INFINITY;
  // Queries in mesh order make the lanes of a warp walk different parts of
  // the tree (far layers of a structured mesh: 32 consecutive nodes span a
  // wide arc).  So: root test for every node, stable compaction of the
  // in-range ones, Morton order of those, and the walk in that order.
  // (measured, sorted vs mesh order: cfg4 mesh 46.7 vs 60.3 ms, cfg3 14.9 vs
  // 16.1 ms, cfg3 without a cutoff 92 vs 139 ms; below a few million nodes
  // the extra passes cost more than they save: cfg2 1.13 vs 1.00 ms)
  if (n_nodes < ((size_t)1 << 22) || std::getenv("IMB_WD_UNSORTED")) {
    k_wall_distance<<<(n_nodes + T - 1) / T, T, 0, ctx.stream>>>(
        t, nodes.x.p, nodes.y.p, nodes.z.p, nullptr, nullptr, n_nodes, cutoff2, d_out);
  } else {
    k_root_test<<<(n_nodes + T - 1) / T, T, 0, ctx.stream>>>(t, nodes.x.p, nodes.y.p, nodes.z.p,
                                                              n_nodes, cutoff2, d_out);
    uint32_t* ids = ctx.buf<uint32_t>(Context::kSlotWallIds, n_nodes);
    const size_t na = compact_active(ctx, d_out, n_nodes, INFINITY, ids);
    if (na) {
      uint32_t* order = ctx.buf<uint32_t>(Context::kSlotWallOrder, na);
      spatial_order(ctx, nodes.x.p, nodes.y.p, nodes.z.p, ids, na, 1.0, order);
      k_wall_distance<<<(na + T - 1) / T, T, 0, ctx.stream>>>(t, nodes.x.p, nodes.y.p, nodes.z.p, ids,
                                                               order, na, cutoff2, d_out);
    }
  }
  IMB_LAUNCH_CHECK();
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
}

}  // namespace imb
