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
#include <string>

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
    IMB_CHECK(cudaMemcpy(&kind, kinds + e, sizeof(int), cudaMemcpyDeviceToHost));
    // validate_mesh messages (mesh.cpp:168-185)
    if (code == kBadKind) throw InvalidArgument("element list: unknown element kind");
    if (code == kBadCount)
      throw InvalidArgument(std::string("element list: wrong node count for ") + kind_name(kind));
    unsigned long long o[2] = {0, 0};
    IMB_CHECK(cudaMemcpy(o, offsets + e, 16, cudaMemcpyDeviceToHost));
    std::string idx = "?";
    for (unsigned long long k = o[0]; k < o[1]; ++k) {
      unsigned long long v = 0;
      IMB_CHECK(cudaMemcpy(&v, conn + k, 8, cudaMemcpyDeviceToHost));
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
  if (out && n_elem) IMB_CHECK(cudaMemcpy(out, dout, n_elem * 8, cudaMemcpyDeviceToHost));
  return inverted;
}

}  // namespace imb
