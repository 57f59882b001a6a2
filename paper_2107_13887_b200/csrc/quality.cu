// quality.cu — signed element measures and the inverted-element count on the
// device.
//
// Follows proj/src/quality.cpp:91-148: tri_area (quality.cpp:95-97),
// tet_volume = dot(b - a, cross(c - a, d - a)) / 6 (quality.cpp:91-93 with
// vec.hpp:48-54), the per-kind decompositions of signed_measure
// (quality.cpp:101-133: quad = 2 triangles, hex = 6 tets around the 0-6
// diagonal accumulated left to right, prism = 3 tets, pyramid = 2 tets,
// line = 0) and count_inverted's `measure <= 0` (quality.cpp:142-148).
// Every operation is an explicit __d*_rn intrinsic in the reference's order,
// so measures are bit-identical and the count exact.
//
// Layout: nodes as SoA x/y/z doubles (the deformed mesh is already resident
// in this form inside im_deform), elements in CSR — kinds (int32, mesh.hpp:15-23
// order), offsets (n_elem + 1) and node indices (uint64).  One thread per
// element, grid-stride; the kernel is a gather over 24 B per node reference
// and is bound by HBM/L2 gather traffic.  Malformed
// elements (unknown kind, wrong node count, node index out of range —
// validate_mesh, mesh.cpp:162-186) are reported through an atomicMin on the
// first offending element so the host can raise the reference's message.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "runtime.hpp"

namespace imb {
namespace {

using namespace exact;

struct P3 {
  double x, y, z;
};

__device__ __forceinline__ P3 ld(const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, unsigned long long i) {
  return {__ldg(x + i), __ldg(y + i), __ldg(z + i)};
}

// quality.cpp:91-93; vec.hpp:48-54 (dot left to right, cross component-wise)
__device__ __forceinline__ double tet_volume(const P3& a, const P3& b, const P3& c, const P3& d) {
  const double ux = sub(b.x, a.x), uy = sub(b.y, a.y), uz = sub(b.z, a.z);
  const double vx = sub(c.x, a.x), vy = sub(c.y, a.y), vz = sub(c.z, a.z);
  const double wx = sub(d.x, a.x), wy = sub(d.y, a.y), wz = sub(d.z, a.z);
  const double cx = sub(mul(vy, wz), mul(vz, wy));
  const double cy = sub(mul(vz, wx), mul(vx, wz));
  const double cz = sub(mul(vx, wy), mul(vy, wx));
  return div(add(add(mul(ux, cx), mul(uy, cy)), mul(uz, cz)), 6.0);
}

// quality.cpp:95-97
__device__ __forceinline__ double tri_area(const P3& a, const P3& b, const P3& c) {
  return mul(0.5, sub(mul(sub(b.x, a.x), sub(c.y, a.y)), mul(sub(c.x, a.x), sub(b.y, a.y))));
}

__host__ __device__ __forceinline__ int node_count(int kind) {
  // mesh.cpp:38-49
  switch (kind) {
    case 0: return 2;
    case 1: return 3;
    case 2: return 4;
    case 3: return 4;
    case 4: return 8;
    case 5: return 6;
    case 6: return 5;
  }
  return -1;
}

enum : unsigned long long { kBadKind = 1, kBadCount = 2, kBadIndex = 3 };

__global__ void __launch_bounds__(256) k_signed_measures(
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
    unsigned long long n_nodes, const int* __restrict__ kinds,
    const unsigned long long* __restrict__ offsets, const unsigned long long* __restrict__ conn,
    unsigned long long n_elem, double* __restrict__ out, unsigned long long* __restrict__ count,
    unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       e < n_elem; e += stride) {
    const int kind = kinds[e];
    const unsigned long long o = offsets[e], cnt = offsets[e + 1] - o;
    const int need = node_count(kind);
    unsigned long long err = 0;
    if (need < 0) {
      err = kBadKind;
    } else if (cnt != (unsigned long long)need) {
      err = kBadCount;
    } else {
      for (int k = 0; k < need; ++k)
        if (conn[o + k] >= n_nodes) err = kBadIndex;
    }
    if (err) {
      // (element << 2 | code): the smallest element wins
      atomicMin(bad, (e << 2) | err);
      continue;
    }
    const unsigned long long* n = conn + o;
    double m = 0.0;  // Line (quality.cpp:128-129)
    switch (kind) {
      case 1: m = tri_area(ld(x, y, z, n[0]), ld(x, y, z, n[1]), ld(x, y, z, n[2])); break;
      case 2: {
        const P3 a = ld(x, y, z, n[0]), b = ld(x, y, z, n[1]), c = ld(x, y, z, n[2]),
                 d = ld(x, y, z, n[3]);
        m = add(tri_area(a, b, c), tri_area(a, c, d));
        break;
      }
      case 3:
        m = tet_volume(ld(x, y, z, n[0]), ld(x, y, z, n[1]), ld(x, y, z, n[2]), ld(x, y, z, n[3]));
        break;
      case 4: {
        P3 p[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) p[k] = ld(x, y, z, n[k]);
        // six tets around the 0-6 body diagonal, v += ... from 0.0
        m = 0.0;
        m = add(m, tet_volume(p[0], p[1], p[2], p[6]));
        m = add(m, tet_volume(p[0], p[2], p[3], p[6]));
        m = add(m, tet_volume(p[0], p[3], p[7], p[6]));
        m = add(m, tet_volume(p[0], p[7], p[4], p[6]));
        m = add(m, tet_volume(p[0], p[4], p[5], p[6]));
        m = add(m, tet_volume(p[0], p[5], p[1], p[6]));
        break;
      }
      case 5: {
        P3 p[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) p[k] = ld(x, y, z, n[k]);
        m = add(add(tet_volume(p[0], p[1], p[2], p[3]), tet_volume(p[1], p[2], p[3], p[4])),
                tet_volume(p[2], p[3], p[4], p[5]));
        break;
      }
      case 6: {
        P3 p[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) p[k] = ld(x, y, z, n[k]);
        m = add(tet_volume(p[0], p[1], p[2], p[4]), tet_volume(p[0], p[2], p[3], p[4]));
        break;
      }
      default: break;
    }
    if (out) out[e] = m;
    local += m <= 0.0 ? 1 : 0;  // quality.cpp:145
  }
  // warp-aggregated count: one atomic per warp
  const unsigned w = __reduce_add_sync(0xffffffffu, (unsigned)local);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(count, (unsigned long long)w);
}

const char* kind_name(int kind) {
  // mesh.cpp:51-62
  switch (kind) {
    case 0: return "line";
    case 1: return "triangle";
    case 2: return "quadrilateral";
    case 3: return "tetrahedron";
    case 4: return "hexahedron";
    case 5: return "prism";
    case 6: return "pyramid";
  }
  return "unknown";
}

}  // namespace

size_t signed_measures(Context& ctx, const double* x, const double* y, const double* z,
                       size_t n_nodes, const int* kinds, const unsigned long long* offsets,
                       const unsigned long long* conn, size_t n_elem, double* out) {
  unsigned long long* w = ctx.buf<unsigned long long>(Context::kSlotCounts, 2);
  const unsigned long long init[2] = {0ull, ~0ull};
  unsigned long long* hw = reinterpret_cast<unsigned long long*>(ctx.pinned.reserve(16));
  hw[0] = init[0], hw[1] = init[1];
  IMB_CHECK(cudaMemcpyAsync(w, hw, 16, cudaMemcpyHostToDevice, ctx.stream));
  if (n_elem) {
    const int threads = 256;
    const size_t want = (n_elem + threads - 1) / threads;
    const int grid = (int)std::min<size_t>(want, (size_t)ctx.num_sms * 8);
    k_signed_measures<<<grid, threads, 0, ctx.stream>>>(x, y, z, n_nodes, kinds, offsets, conn,
                                                        n_elem, out, w, w + 1);
    IMB_LAUNCH_CHECK();
  }
  IMB_CHECK(cudaMemcpyAsync(hw, w, 16, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
  if (hw[1] != ~0ull) {
    const unsigned long long e = hw[1] >> 2, code = hw[1] & 3;
    int kind = 0;
    sync_copy(ctx.stream, &kind, kinds + e, sizeof(int), cudaMemcpyDeviceToHost);
    // validate_mesh messages (mesh.cpp:168-185)
    if (code == kBadKind) throw InvalidArgument("element list: unknown element kind");
    if (code == kBadCount)
      throw InvalidArgument(std::string("element list: wrong node count for ") + kind_name(kind));
    unsigned long long o[2] = {0, 0};
    sync_copy(ctx.stream, o, offsets + e, 16, cudaMemcpyDeviceToHost);
    std::string idx = "?";
    for (unsigned long long k = o[0]; k < o[1]; ++k) {
      unsigned long long v = 0;
      sync_copy(ctx.stream, &v, conn + k, 8, cudaMemcpyDeviceToHost);
      if (v >= n_nodes) {
        idx = std::to_string(v);
        break;
      }
    }
    throw InvalidArgument("element list: node index " + idx + " out of range (mesh has " +
                          std::to_string(n_nodes) + " nodes)");
  }
  return (size_t)hw[0];
}

size_t signed_measures_from_host(Context& ctx, const double* x, const double* y, const double* z,
                                 size_t n_nodes, const int* kinds, const size_t* offsets,
                                 const size_t* conn, size_t n_elem, double* out) {
  static_assert(sizeof(size_t) == sizeof(unsigned long long), "size_t must be 64-bit");
  if (n_elem && !(kinds && offsets && conn)) throw InvalidArgument("element arrays are null");
  const size_t n_conn = n_elem ? offsets[n_elem] - offsets[0] : 0;
  if (n_elem && offsets[0] != 0) throw InvalidArgument("element offsets must start at 0");
  int* dk = ctx.buf<int>(Context::kSlotElemKind, n_elem);
  auto* doff = ctx.buf<unsigned long long>(Context::kSlotElemOffset, n_elem + 1);
  auto* dconn = ctx.buf<unsigned long long>(Context::kSlotElemNodes, n_conn);
  double* dout = out ? ctx.buf<double>(Context::kSlotVals, n_elem) : nullptr;
  if (n_elem) {
    IMB_CHECK(cudaMemcpyAsync(dk, kinds, n_elem * sizeof(int), cudaMemcpyHostToDevice, ctx.stream));
    IMB_CHECK(cudaMemcpyAsync(doff, offsets, (n_elem + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (n_conn)
      IMB_CHECK(cudaMemcpyAsync(dconn, conn, n_conn * 8, cudaMemcpyHostToDevice, ctx.stream));
  }
  const size_t inverted = signed_measures(ctx, x, y, z, n_nodes, dk, doff, dconn, n_elem, dout);
  if (out && n_elem) sync_copy(ctx.stream, out, dout, n_elem * 8, cudaMemcpyDeviceToHost);
  return inverted;
}

}  // namespace imb

// ---- orthogonality (quality.cpp:150-236) --------------------------------------
// Face matching without the reference's std::map: every element emits its
// faces (element_faces, quality.cpp:19-49) as records keyed by the sorted
// global node ids (two 64-bit words), a stable two-pass radix sort groups
// equal keys with their uses in element-major order (= the map's per-key
// vector order), and one thread per group applies quality.cpp:178-200.
// Per-element folds use integer atomicMin on the (non-negative) score bits.
// All vector arithmetic follows vec.hpp with explicit IEEE ops; atan2 is
// CUDA's (<= 2 ulp), so scores agree with the reference to ~1e-13 degrees,
// not bit for bit.  The mean is summed on the host in element order.
namespace imb {
namespace {

__constant__ int kFaceCnt[7] = {0, 3, 4, 4, 6, 5, 5};
__constant__ unsigned char kFaceTab[7][6][5] = {
    {{0}},
    {{2, 0, 1}, {2, 1, 2}, {2, 2, 0}},
    {{2, 0, 1}, {2, 1, 2}, {2, 2, 3}, {2, 3, 0}},
    {{3, 0, 1, 2}, {3, 0, 1, 3}, {3, 1, 2, 3}, {3, 0, 2, 3}},
    {{4, 0, 1, 2, 3}, {4, 4, 5, 6, 7}, {4, 0, 1, 5, 4}, {4, 1, 2, 6, 5}, {4, 2, 3, 7, 6},
     {4, 3, 0, 4, 7}},
    {{3, 0, 1, 2}, {3, 3, 4, 5}, {4, 0, 1, 4, 3}, {4, 1, 2, 5, 4}, {4, 2, 0, 3, 5}},
    {{4, 0, 1, 2, 3}, {3, 0, 1, 4}, {3, 1, 2, 4}, {3, 2, 3, 4}, {3, 3, 0, 4}},
};

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 dsub3(D3 a, D3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ D3 dadd3(D3 a, D3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ D3 dscale3(D3 a, double s) { return {mul(a.x, s), mul(a.y, s), mul(a.z, s)}; }
__device__ __forceinline__ double dsq3(D3 a) { return add(add(mul(a.x, a.x), mul(a.y, a.y)), mul(a.z, a.z)); }
__device__ __forceinline__ double ddot3(D3 a, D3 b) { return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z)); }
__device__ __forceinline__ D3 dcross3(D3 a, D3 b) {
  return {sub(mul(a.y, b.z), mul(a.z, b.y)), sub(mul(a.z, b.x), mul(a.x, b.z)),
          sub(mul(a.x, b.y), mul(a.y, b.x))};
}
// vec.hpp:64-67
__device__ __forceinline__ D3 dnormalized(D3 v) {
  const double n = __dsqrt_rn(dsq3(v));
  return n > 0.0 ? dscale3(v, __ddiv_rn(1.0, n)) : D3{0.0, 0.0, 0.0};
}

struct Geo {
  const double *x, *y, *z;
  const int* kinds;
  const unsigned long long *offsets, *conn;
  __device__ D3 node(unsigned long long i) const { return {x[i], y[i], z[i]}; }
  // global nodes of local face f of element e, in the face's own order
  __device__ int face(unsigned long long e, int f, unsigned long long (&g)[4]) const {
    const unsigned char* t = kFaceTab[kinds[e]][f];
    for (int k = 0; k < t[0]; ++k) g[k] = conn[offsets[e] + t[1 + k]];
    return t[0];
  }
};

// quality.cpp:51-55 / 74-78: node sum in order, times 1/count
__device__ D3 centroid(const Geo& G, const unsigned long long* g, int cnt) {
  D3 c{0.0, 0.0, 0.0};
  for (int k = 0; k < cnt; ++k) c = dadd3(c, G.node(g[k]));
  return dscale3(c, __ddiv_rn(1.0, (double)cnt));
}

// quality.cpp:57-72
__device__ D3 face_normal(const Geo& G, const unsigned long long (&g)[4], int cnt) {
  if (cnt == 2) {
    const D3 t = dsub3(G.node(g[1]), G.node(g[0]));
    return dnormalized({t.y, -t.x, 0.0});
  }
  const D3 a = G.node(g[0]), b = G.node(g[1]), c = G.node(g[2]);
  D3 n = dcross3(dsub3(b, a), dsub3(c, a));
  if (cnt == 4) n = dadd3(dnormalized(n), dnormalized(dcross3(dsub3(c, a), dsub3(G.node(g[3]), a))));
  return dnormalized(n);
}

// quality.cpp:82-88
__device__ double face_score(D3 normal, D3 line) {
  const D3 c = dnormalized(line);
  if (dsq3(normal) == 0.0 || dsq3(c) == 0.0) return 0.0;
  const double along = fabs(ddot3(normal, c));
  const double transverse = __dsqrt_rn(dsq3(dcross3(normal, c)));
  return sub(90.0, __ddiv_rn(mul(atan2(transverse, along), 180.0), 3.141592653589793));
}

__global__ void k_face_counts(const int* kinds, size_t n, unsigned* cnt) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) cnt[e] = (unsigned)kFaceCnt[kinds[e]];
}

__global__ void k_face_keys(Geo G, size_t n, const unsigned long long* foff,
                            unsigned long long* khi, unsigned long long* klo, unsigned* ef,
                            unsigned* vals) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int nf = kFaceCnt[G.kinds[e]];
  for (int f = 0; f < nf; ++f) {
    unsigned long long g[4];
    const int c = G.face(e, f, g);
    unsigned s[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    for (int k = 0; k < c; ++k) s[k] = (unsigned)g[k];
    for (int a = 1; a < c; ++a)
      for (int b = a; b > 0 && s[b - 1] > s[b]; --b) {
        const unsigned t = s[b];
        s[b] = s[b - 1], s[b - 1] = t;
      }
    const size_t r = foff[e] + f;
    khi[r] = ((unsigned long long)s[0] << 32) | s[1];
    klo[r] = ((unsigned long long)s[2] << 32) | s[3];
    ef[r] = (unsigned)(e * 8 + f);
    vals[r] = (unsigned)r;
  }
}

__global__ void k_gather_u64(const unsigned long long* src, const unsigned* idx, size_t n,
                             unsigned long long* dst) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_centroids(Geo G, size_t n, double* cx, double* cy, double* cz) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  D3 c{0.0, 0.0, 0.0};
  const unsigned long long o = G.offsets[e], cnt = G.offsets[e + 1] - o;
  for (unsigned long long k = 0; k < cnt; ++k) c = dadd3(c, G.node(G.conn[o + k]));
  c = dscale3(c, __ddiv_rn(1.0, (double)cnt));
  cx[e] = c.x, cy[e] = c.y, cz[e] = c.z;
}

__device__ __forceinline__ void fold_min(unsigned long long* slot, double v) {
  atomicMin(slot, (unsigned long long)__double_as_longlong(v));  // v >= 0: bit order == value order
}

// one thread per sorted face position; the first position of each key group
// handles the group (quality.cpp:178-200)
__global__ void k_face_groups(Geo G, size_t nf, const unsigned* order, const unsigned long long* khi,
                              const unsigned long long* klo, const unsigned* ef,
                              const double* cx, const double* cy, const double* cz,
                              unsigned long long* internal, unsigned long long* boundary,
                              unsigned* degenerate) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const unsigned r0 = order[i];
  const unsigned long long h = khi[r0], l = klo[r0];
  if (i > 0 && khi[order[i - 1]] == h && klo[order[i - 1]] == l) return;
  size_t j = i + 1;
  while (j < nf && khi[order[j]] == h && klo[order[j]] == l) ++j;
  unsigned long long g0[4];
  const unsigned u0 = ef[r0];
  const int cnt = G.face(u0 >> 3, u0 & 7, g0);
  const D3 normal = face_normal(G, g0, cnt);  // uses.front().global
  const bool deg = dsq3(normal) == 0.0;
  if (j - i == 2) {
    const unsigned e0 = ef[order[i]] >> 3, e1 = ef[order[i + 1]] >> 3;
    const D3 line = dsub3(D3{cx[e1], cy[e1], cz[e1]}, D3{cx[e0], cy[e0], cz[e0]});
    const double score = deg ? 0.0 : face_score(normal, line);
    for (size_t u = i; u < j; ++u) {
      const unsigned e = ef[order[u]] >> 3;
      fold_min(&internal[e], score);
      if (deg) atomicOr(&degenerate[e], 1u);
    }
  } else {
    for (size_t u = i; u < j; ++u) {
      const unsigned uu = ef[order[u]], e = uu >> 3;
      unsigned long long g[4];
      const int c = G.face(e, uu & 7, g);
      const D3 line = dsub3(centroid(G, g, c), D3{cx[e], cy[e], cz[e]});
      const double score = deg ? 0.0 : face_score(normal, line);
      fold_min(&boundary[e], score);
      if (deg) atomicOr(&degenerate[e], 1u);
    }
  }
}

// quality.cpp:215-224 per element
__global__ void k_element_scores(size_t n, const unsigned long long* internal,
                                 const unsigned long long* boundary, const unsigned* degenerate,
                                 double* scores) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const unsigned long long unset = 0x7ff0000000000000ull;  // +inf: no face of that kind
  double s = internal[e] != unset ? __longlong_as_double((long long)internal[e])
           : boundary[e] != unset ? __longlong_as_double((long long)boundary[e]) : 90.0;
  if (degenerate[e]) s = 0.0;
  scores[e] = s;
}

__global__ void k_fill_u64(unsigned long long* p, size_t n, unsigned long long v) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace

QualityStats orthogonality_device(Context& ctx, const double* x, const double* y, const double* z,
                                  size_t n_nodes, const int* kinds, const unsigned long long* offsets,
                                  const unsigned long long* conn, size_t n_elem, double* scores,
                                  double* measures) {
  QualityStats q;
  // signed measures + validation (also rejects malformed elements)
  q.inverted = signed_measures(ctx, x, y, z, n_nodes, kinds, offsets, conn, n_elem, measures);
  if (n_elem == 0) return q;
  if (n_elem >= (size_t(1) << 29) || n_nodes >= 0xffffffffull)
    throw InvalidArgument("orthogonality: mesh too large (elements < 2^29, nodes < 2^32)");
  const Geo G{x, y, z, kinds, offsets, conn};
  const unsigned nb = (unsigned)((n_elem + 255) / 256);
  DBuf<unsigned> cnt;
  DBuf<unsigned long long> foff;
  cnt.reserve(n_elem);
  foff.reserve(n_elem + 1);
  k_face_counts<<<nb, 256, 0, ctx.stream>>>(kinds, n_elem, cnt.p);
  scan_u32_to_u64_async(ctx, cnt.p, n_elem, foff.p);
  unsigned long long nf_h = 0;
  IMB_CHECK(cudaMemcpyAsync(&nf_h, foff.p + n_elem, 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
  const size_t nf = (size_t)nf_h;
  if (nf >= 0xffffffffull) throw InvalidArgument("orthogonality: too many faces");
  DBuf<unsigned long long> khi, klo, ks, kg;
  DBuf<unsigned> ef, v0, v1, v2;
  for (auto* b : {&khi, &klo, &ks, &kg}) b->reserve(std::max<size_t>(nf, 1));
  for (auto* b : {&ef, &v0, &v1, &v2}) b->reserve(std::max<size_t>(nf, 1));
  k_face_keys<<<nb, 256, 0, ctx.stream>>>(G, n_elem, foff.p, khi.p, klo.p, ef.p, v0.p);
  // stable LSD: by the low key word, then by the high word
  size_t t1 = 0, t2 = 0;
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, t1, klo.p, ks.p, v0.p, v1.p, (int)nf, 0, 64, ctx.stream));
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, t2, kg.p, ks.p, v1.p, v2.p, (int)nf, 0, 64, ctx.stream));
  DBuf<unsigned char> tmp;
  tmp.reserve(std::max(t1, t2));
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, t1, klo.p, ks.p, v0.p, v1.p, (int)nf, 0, 64, ctx.stream));
  const unsigned fb = (unsigned)((nf + 255) / 256);
  k_gather_u64<<<fb, 256, 0, ctx.stream>>>(khi.p, v1.p, nf, kg.p);
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, t2, kg.p, ks.p, v1.p, v2.p, (int)nf, 0, 64, ctx.stream));
  DBuf<double> cx, cy, cz;
  cx.reserve(n_elem), cy.reserve(n_elem), cz.reserve(n_elem);
  k_centroids<<<nb, 256, 0, ctx.stream>>>(G, n_elem, cx.p, cy.p, cz.p);
  DBuf<unsigned long long> in_s, bd_s;
  DBuf<unsigned> deg;
  in_s.reserve(n_elem), bd_s.reserve(n_elem), deg.reserve(n_elem);
  k_fill_u64<<<nb, 256, 0, ctx.stream>>>(in_s.p, n_elem, 0x7ff0000000000000ull);
  k_fill_u64<<<nb, 256, 0, ctx.stream>>>(bd_s.p, n_elem, 0x7ff0000000000000ull);
  IMB_CHECK(cudaMemsetAsync(deg.p, 0, n_elem * 4, ctx.stream));
  k_face_groups<<<fb, 256, 0, ctx.stream>>>(G, nf, v2.p, khi.p, klo.p, ef.p, cx.p, cy.p, cz.p,
                                            in_s.p, bd_s.p, deg.p);
  DBuf<double> sc;
  sc.reserve(n_elem);
  k_element_scores<<<nb, 256, 0, ctx.stream>>>(n_elem, in_s.p, bd_s.p, deg.p, sc.p);
  IMB_LAUNCH_CHECK();
  std::vector<double> h(n_elem);
  std::vector<unsigned> hd(n_elem);
  IMB_CHECK(cudaMemcpyAsync(h.data(), sc.p, n_elem * 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaMemcpyAsync(hd.data(), deg.p, n_elem * 4, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
  // quality.cpp:225-234: in element order on the host (the reference's sum)
  double sum = 0.0, mn = 90.0;
  for (size_t e = 0; e < n_elem; ++e) {
    sum += h[e];
    mn = h[e] < mn ? h[e] : mn;
    q.degenerate += hd[e] ? 1 : 0;
  }
  q.min_deg = mn;
  q.mean_deg = sum / (double)n_elem;
  if (scores) std::memcpy(scores, h.data(), n_elem * 8);
  return q;
}

QualityStats orthogonality_from_host(Context& ctx, const double* x, const double* y, const double* z,
                                     size_t n_nodes, const int* kinds, const size_t* offsets,
                                     const size_t* conn, size_t n_elem, double* scores,
                                     double* measures) {
  if (n_elem && !(kinds && offsets && conn)) throw InvalidArgument("element arrays are null");
  if (n_elem && offsets[0] != 0) throw InvalidArgument("element offsets must start at 0");
  const size_t n_conn = n_elem ? offsets[n_elem] : 0;
  int* dk = ctx.buf<int>(Context::kSlotElemKind, n_elem);
  auto* doff = ctx.buf<unsigned long long>(Context::kSlotElemOffset, n_elem + 1);
  auto* dconn = ctx.buf<unsigned long long>(Context::kSlotElemNodes, n_conn);
  if (n_elem) {
    IMB_CHECK(cudaMemcpyAsync(dk, kinds, n_elem * sizeof(int), cudaMemcpyHostToDevice, ctx.stream));
    IMB_CHECK(cudaMemcpyAsync(doff, offsets, (n_elem + 1) * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (n_conn)
      IMB_CHECK(cudaMemcpyAsync(dconn, conn, n_conn * 8, cudaMemcpyHostToDevice, ctx.stream));
  }
  DBuf<double> dm;
  if (measures) dm.reserve(std::max<size_t>(n_elem, 1));
  const QualityStats q = orthogonality_device(ctx, x, y, z, n_nodes, dk, doff, dconn, n_elem, scores,
                                              measures ? dm.p : nullptr);
  if (measures && n_elem) sync_copy(ctx.stream, measures, dm.p, n_elem * 8, cudaMemcpyDeviceToHost);
  return q;
}

}  // namespace imb
