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
// B200 design: a uniform grid over the patch (counting sort of the surface
// points into cells, CSR cell_start + SoA sorted coordinates), one thread per
// query doing a ring search around its (clamped) cell with the exact squared
// distance of App. A1.  The ring loop stops once the lower bound
//   LB(r)^2 = dist(q, grid box)^2 + ((r-1) h)^2
// (projection onto the box is non-expansive) exceeds min(best, cutoff^2) with
// a 1e-9 relative safety margin, so the exact nearest point is always visited
// when it lies inside the cutoff.  With cutoff = D (the volume-reduction
// support distance) nodes farther than D from the whole patch exit after one
// box test: that IS the volume reduction's culling pass, and it is HBM bound
// (24 B coordinates in, 8 B distance out per node).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "runtime.hpp"

namespace imb {

namespace {

struct Grid {
  double ox, oy, oz, h, inv_h;
  double bx0, by0, bz0, bx1, by1, bz1;  // box covered by the cells
  int nx, ny, nz;
  const unsigned long long* start;      // n_cells + 1
  const double *sx, *sy, *sz;           // cell-sorted surface points
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ int cell_coord(double v, double o, double inv_h, int n) {
  const double f = floor((v - o) * inv_h);
  if (!(f >= 0.0)) return 0;  // also catches NaN
  if (f >= (double)(n - 1)) return n - 1;
  return (int)f;
}

__global__ void k_cell_count(const double* x, const double* y, const double* z, size_t n, Grid g,
                             unsigned int* cell_of, unsigned int* counts) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cx = cell_coord(x[i], g.ox, g.inv_h, g.nx);
  const int cy = cell_coord(y[i], g.oy, g.inv_h, g.ny);
  const int cz = cell_coord(z[i], g.oz, g.inv_h, g.nz);
  const unsigned int c = ((unsigned)cz * g.ny + cy) * g.nx + cx;
  cell_of[i] = c;
  atomicAdd(&counts[c], 1u);
}

__global__ void k_cell_fill(const double* x, const double* y, const double* z, size_t n,
                            const unsigned int* cell_of, const unsigned long long* start,
                            unsigned int* cursor, double* sx, double* sy, double* sz) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned int c = cell_of[i];
  const unsigned long long p = start[c] + atomicAdd(&cursor[c], 1u);
  sx[p] = x[i];
  sy[p] = y[i];
  sz[p] = z[i];
}

__device__ __forceinline__ void scan_cell(const Grid& g, int cx, int cy, int cz, double qx,
                                          double qy, double qz, double& best) {
  const unsigned int c = ((unsigned)cz * g.ny + cy) * g.nx + cx;
  const unsigned long long b = g.start[c], e = g.start[c + 1];
  for (unsigned long long p = b; p < e; ++p) {
    // squared_distance(points_[n.point], query): (p - q), App. A1 order
    const double s = exact::sqdist(g.sx[p], g.sy[p], g.sz[p], qx, qy, qz);
    if (s < best) best = s;
  }
}

__global__ void __launch_bounds__(256) k_wall_distance(Grid g, const double* __restrict__ qx_,
                                                       const double* __restrict__ qy_,
                                                       const double* __restrict__ qz_, size_t n,
                                                       double cutoff2, double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double qx = qx_[i], qy = qy_[i], qz = qz_[i];
  const double ex = fmax(0.0, fmax(g.bx0 - qx, qx - g.bx1));
  const double ey = fmax(0.0, fmax(g.by0 - qy, qy - g.by1));
  const double ez = fmax(0.0, fmax(g.bz0 - qz, qz - g.bz1));
  const double db2 = ex * ex + ey * ey + ez * ez;
  const double margin = 1.0 - 1e-9;
  double best = INFINITY;
  if (db2 * margin > cutoff2) {
    out[i] = INFINITY;  // farther than the cutoff from the whole patch
    return;
  }
  const int cx = cell_coord(qx, g.ox, g.inv_h, g.nx);
  const int cy = cell_coord(qy, g.oy, g.inv_h, g.ny);
  const int cz = cell_coord(qz, g.oz, g.inv_h, g.nz);
  const int rmax = max(max(max(cx, g.nx - 1 - cx), max(cy, g.ny - 1 - cy)),
                       max(cz, g.nz - 1 - cz));
  for (int r = 0; r <= rmax; ++r) {
    if (r >= 1) {
      const double l = (double)(r - 1) * g.h;
      const double lb2 = db2 + l * l;
      if (lb2 * margin > fmin(best, cutoff2)) break;
    }
    const int z0 = max(cz - r, 0), z1 = min(cz + r, g.nz - 1);
    const int y0 = max(cy - r, 0), y1 = min(cy + r, g.ny - 1);
    for (int zz = z0; zz <= z1; ++zz) {
      const bool zedge = (zz == cz - r) || (zz == cz + r);
      for (int yy = y0; yy <= y1; ++yy) {
        const bool edge = zedge || (yy == cy - r) || (yy == cy + r);
        if (edge) {
          const int x0 = max(cx - r, 0), x1 = min(cx + r, g.nx - 1);
          for (int xx = x0; xx <= x1; ++xx) scan_cell(g, xx, yy, zz, qx, qy, qz, best);
        } else {
          if (cx - r >= 0) scan_cell(g, cx - r, yy, zz, qx, qy, qz, best);
          if (r > 0 && cx + r < g.nx) scan_cell(g, cx + r, yy, zz, qx, qy, qz, best);
        }
      }
    }
  }
  out[i] = best < INFINITY ? __dsqrt_rn(best) : INFINITY;
}

}  // namespace

void wall_distance(Context& ctx, const DPoints& nodes, size_t n_nodes, const DPoints& surface,
                   size_t n_surface, int dim, double cutoff, double* d_out) {
  if (n_surface == 0) throw InvalidArgument("cannot build a distance index for an empty patch");
  if (dim != 2 && dim != 3) throw InvalidArgument("kd-tree dim must be 2 or 3");
  if (n_nodes == 0) return;
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
  // cell size: ~2 cells per surface point over the non-degenerate axes
  double ext[3], vol = 1.0;
  int deff = 0;
  const double diag = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                (hi[2] - lo[2]) * (hi[2] - lo[2]));
  for (int a = 0; a < 3; ++a) {
    ext[a] = hi[a] - lo[a];
    if (ext[a] > 1e-9 * diag) vol *= ext[a], ++deff;
  }
  double h = 1.0;
  if (deff > 0) {
    const double target = std::max<double>(1.0, 2.0 * (double)n_surface);
    h = std::pow(vol / target, 1.0 / deff);
  }
  if (!(h > 0.0) || !std::isfinite(h)) h = diag > 0 ? diag : 1.0;
  int n[3];
  for (int a = 0; a < 3; ++a) {
    const double c = std::ceil(ext[a] / h);
    n[a] = (int)std::max(1.0, std::min(c, 4096.0));
  }
  while ((double)n[0] * n[1] * n[2] > 16.0e6) {
    h *= 1.25;
    for (int a = 0; a < 3; ++a) n[a] = (int)std::max(1.0, std::min(std::ceil(ext[a] / h), 4096.0));
  }
  // make the cells cover the box exactly: h may grow to fit the 4096 clamp
  for (int a = 0; a < 3; ++a) h = std::max(h, ext[a] / n[a]);
  const size_t n_cells = (size_t)n[0] * n[1] * n[2];

  Grid g{};
  g.ox = lo[0], g.oy = lo[1], g.oz = lo[2];
  g.h = h;
  g.inv_h = 1.0 / h;
  g.nx = n[0], g.ny = n[1], g.nz = n[2];
  g.bx0 = lo[0], g.by0 = lo[1], g.bz0 = lo[2];
  g.bx1 = lo[0] + h * n[0], g.by1 = lo[1] + h * n[1], g.bz1 = lo[2] + h * n[2];

  DBuf<unsigned int> cell_of, counts;
  DBuf<unsigned long long> start;
  DBuf<double> sx, sy, sz;
  cell_of.reserve(n_surface);
  counts.reserve(n_cells);
  start.reserve(n_cells + 1);
  sx.reserve(n_surface), sy.reserve(n_surface), sz.reserve(n_surface);
  IMB_CHECK(cudaMemsetAsync(counts.p, 0, n_cells * 4, ctx.stream));
  const int T = 256;
  k_cell_count<<<(n_surface + T - 1) / T, T, 0, ctx.stream>>>(surface.x.p, surface.y.p, surface.z.p,
                                                               n_surface, g, cell_of.p, counts.p);
  IMB_LAUNCH_CHECK();
  scan_u32_to_u64(ctx, counts.p, n_cells, start.p);
  IMB_CHECK(cudaMemsetAsync(counts.p, 0, n_cells * 4, ctx.stream));
  k_cell_fill<<<(n_surface + T - 1) / T, T, 0, ctx.stream>>>(surface.x.p, surface.y.p, surface.z.p,
                                                              n_surface, cell_of.p, start.p,
                                                              counts.p, sx.p, sy.p, sz.p);
  IMB_LAUNCH_CHECK();
  g.start = start.p;
  g.sx = sx.p, g.sy = sy.p, g.sz = sz.p;
  const double cutoff2 = std::isfinite(cutoff) ? cutoff * cutoff : INFINITY;
  k_wall_distance<<<(n_nodes + T - 1) / T, T, 0, ctx.stream>>>(g, nodes.x.p, nodes.y.p, nodes.z.p,
                                                                n_nodes, cutoff2, d_out);
  IMB_LAUNCH_CHECK();
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));  // local buffers die here
}

}  // namespace imb
