// runtime.hpp — host-side runtime of icemorph-b200: error types, per-call
// context (stream + device arena), device buffers and the kernel launchers
// each .cu file exports to the C-ABI layer (capi.cu).
//
// No global mutable state: every call works on an explicit Context, so two
// contexts (e.g. two host threads) never share streams or scratch — the
// reference's "deform is reentrant" guarantee carries over.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace imb {

// Error taxonomy mirrors the reference's exceptions:
//   std::invalid_argument -> InvalidArgument (status 1)
//   icemorph::SolveError  -> SolveFailure    (status 2)
//   CUDA / runtime        -> CudaError / std::runtime_error (status 3)
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct SolveFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  CudaError(cudaError_t e, const char* call, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + call +
                           " (" + file + ":" + std::to_string(line) + ")") {}
};

#define IMB_CHECK(call)                                                          \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) throw ::imb::CudaError(e_, #call, __FILE__, __LINE__); \
  } while (0)

#define IMB_LAUNCH_CHECK() IMB_CHECK(cudaGetLastError())

// A copy ordered on `stream` and complete on return.  The library's streams
// are non-blocking, so a plain cudaMemcpy (legacy default stream) would not
// order against their kernels.
inline void sync_copy(cudaStream_t stream, void* dst, const void* src, size_t bytes,
                      cudaMemcpyKind kind) {
  IMB_CHECK(cudaMemcpyAsync(dst, src, bytes, kind, stream));
  IMB_CHECK(cudaStreamSynchronize(stream));
}

// Owning device buffer (grow-only).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p, n = o.n;
    o.p = nullptr, o.n = 0;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* reserve(size_t count) {
    if (count > n) {
      release();
      size_t bytes = (count ? count : 1) * sizeof(T);
      IMB_CHECK(cudaMalloc(&p, bytes));
      n = count;
    }
    return p;
  }
};

// Pinned host staging buffer (grow-only).
template <class T>
struct HBuf {
  T* p = nullptr;
  size_t n = 0;
  ~HBuf() {
    if (p) cudaFreeHost(p);
  }
  T* reserve(size_t count) {
    if (count > n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      IMB_CHECK(cudaMallocHost(&p, (count ? count : 1) * sizeof(T)));
      n = count;
    }
    return p;
  }
};

// SoA coordinates on the device.
struct DPoints {
  DBuf<double> x, y, z;
  size_t n = 0;
  void reserve(size_t count) {
    x.reserve(count), y.reserve(count), z.reserve(count);
    n = count;
  }
};

struct HostIOState;  // host_io.cu: thread pool + pinned staging

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int status = 0;
  char message[2048] = {0};
  // scratch
  DBuf<unsigned char> scratch;
  HBuf<unsigned char> pinned;
  double last_kernel_ms = 0.0;
  // host<->device bytes the last im_update_volume actually moved (selective upload)
  unsigned long long last_h2d_bytes = 0, last_d2h_bytes = 0;
  // diagnostic (im_count_pairs): the exact kernels count the pairs they evaluate
  bool count_pairs = false;
  unsigned long long pairs_evaluated = 0;
  size_t error_line = 0;  // line of the last IM_PARSE_ERROR
  // Grow-only device scratch slots reused across calls (no cudaMalloc /
  // cudaFree -- which synchronises the device -- on the hot path).
  enum Slot : int {
    kSlotNodesX, kSlotNodesY, kSlotNodesZ, kSlotDist, kSlotActive, kSlotPerm, kSlotVals,
    kSlotTiles, kSlotBoxes, kSlotStage, kSlotCell, kSlotCounts, kSlotStart, kSlotBox,
    kSlotScanA, kSlotScanB, kSlotElemKind, kSlotElemOffset, kSlotElemNodes, kSlotSortKeyA,
    kSlotSortKeyB, kSlotSortTemp, kSlotIndex, kSlotIndexBox, kSlotBlockOrder, kSlotChunkMax,
    kSlotScaledTiles, kSlotWallTree, kSlotWallIds, kSlotWallOrder, kSlotCount
  };
  DBuf<unsigned char> slots[kSlotCount];
  std::shared_ptr<HostIOState> io;  // created on first staged transfer
  // side streams of the pipelined C-ABI calls (0: uploads + per-chunk prep,
  // 1: downloads), created on first use, destroyed with the context
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaStream_t side_stream(int i) {
    if (!side[i]) IMB_CHECK(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
    return side[i];
  }
  template <class T>
  T* buf(Slot s, size_t count) {
    return reinterpret_cast<T*>(slots[s].reserve(count * sizeof(T) + 16));
  }
};

// ---------------------------------------------------------------------------
// Kernel launchers (definitions in the .cu files)
// ---------------------------------------------------------------------------

// AoS (3 doubles per point) host array -> device SoA.
void upload_points(Context& ctx, const double* host_xyz, size_t n, DPoints& out);
// Gather AoS host points by index list into device SoA.
void upload_points_indexed(Context& ctx, const double* host_xyz, const size_t* idx, size_t n,
                           DPoints& out);

// Control tiles: (cx, cy, cz, ax, ay, az) per control, positions scaled by
// 1/R for the fast path (scale = 1/R) or raw for the exact path (scale = 1).
// Padded to a multiple of kCtrlTile with inert controls.
constexpr int kCtrlTile = 256;
size_t ctrl_padded(size_t n);
// doubles of device storage for the packed tiles of n controls
size_t ctrl_tile_doubles(size_t n);
void pack_controls(Context& ctx, const double* d_cx, const double* d_cy, const double* d_cz,
                   const double* d_ax, const double* d_ay, const double* d_az, size_t n,
                   double scale, double* d_tiles);

void pack_controls_aos(Context& ctx, const double* d_ctrl_aos, const double* d_alpha_aos, size_t n,
                       double scale, double* d_tiles);
// Host packing for the fast path (Morton-sorted tiles + per-tile boxes).
void pack_controls_host(Context& ctx, const double* host_ctrl, const double* host_alpha, size_t n,
                        double scale, bool sort, DBuf<double>& tiles, DBuf<double>& boxes);
void pack_controls_host(Context& ctx, const double* host_ctrl, const double* host_alpha, size_t n,
                        double scale, bool sort, double* d_tiles, double* d_boxes);
// device AoS -> SoA (on `stream`, default ctx.stream)
void aos_to_soa(Context& ctx, const double* d_aos, size_t n, double* x, double* y, double* z,
                cudaStream_t stream = nullptr);
// Asynchronous max |coordinate| and max |z| of n device SoA points (or of the
// points active[0..n) when given) on `stream`: d_out[0..1] receive their bit
// patterns (non-negative doubles order as u64)
void max_abs_points_async(const double* x, const double* y, const double* z, size_t n,
                          unsigned long long* d_out, int num_sms, cudaStream_t stream,
                          const uint32_t* active = nullptr);
// For each of the m node ids bounds[i] (host), the position of the first
// active id >= bounds[i] in the ascending device list active[0..na)
// (synchronous; m <= 1024)
void active_lower_bounds(Context& ctx, const uint32_t* active, size_t na, const size_t* bounds,
                         int m, size_t* out);

enum class Precision : int { Exact = 0, Fast64 = 1, Fast32 = 2 };
// C-ABI precision code (IM_EXACT / IM_FP64 / IM_FP32) -> Precision
inline Precision precision_of(int code) {
  if (code < 0 || code > 2)
    throw InvalidArgument("unknown precision (expected IM_EXACT, IM_FP64 or IM_FP32)");
  return static_cast<Precision>(code);
}

struct VolumeArgs {
  // points (SoA); optional gather list of active node ids (nullptr = identity)
  const double *x = nullptr, *y = nullptr, *z = nullptr;
  const uint32_t* active = nullptr;
  const uint32_t* perm = nullptr;  // spatial processing order of the active positions (fast path)
  size_t n_active = 0;
  // wall distances per node (nullptr = psi == 1, i.e. D = inf)
  const double* dist = nullptr;
  double D = 0.0;
  int psi_kind = 0;
  // controls
  const double* tiles = nullptr;  // packed (pack_controls)
  const double* tile_box = nullptr;  // per-tile boxes (fast path culling) or null
  size_t n_ctrl = 0;
  double R = 1.0;
  int kind = 1;
  int dim = 3;
  Precision precision = Precision::Fast64;
  // exact path: use the tiled kernel (spatial order `perm`, culling with the
  // exact-tile boxes `tile_box`); only when exact_tiled_ok() holds
  bool exact_tiled = false;
  // exact tiled: Morton index of the controls (pack_exact_index_host) for the
  // gathered kernel; null = group culling over the insertion order only
  const double* ctrl_index = nullptr;
  const double* index_box = nullptr;
  double ctrl_diag = 0.0;  // diagonal of the controls' bounding box (gather heuristic)
  // exact tiled kernel: CTA i processes block cta_order[i] of kExactBlock
  // positions (heaviest first, block_order()); null = natural order
  const uint32_t* cta_order = nullptr;
  // outputs: either compacted AoS values (out_val[3k+c]) or accumulate into
  // per-node SoA deltas (acc_x/y/z[node] += value), skipping pinned nodes.
  double* out_val = nullptr;
  double *acc_x = nullptr, *acc_y = nullptr, *acc_z = nullptr;
  const unsigned char* pinned = nullptr;
};

void launch_volume(Context& ctx, const VolumeArgs& a);
// max |coordinate| over device SoA points (synchronous, 16-byte readback);
// *max_abs_z (optional) = max |z| (0 <=> planar input)
double max_abs_points(Context& ctx, const double* x, const double* y, const double* z, size_t n,
                      double* max_abs_z = nullptr);
// ranges under which the tiled exact kernel's sqrt/division shortcuts are
// bit-exact: |coordinates| <= 1e100, R in [1e-100, 1e100]; and its culling
// tests (tile / warp boxes in 1/R-scaled coordinates against 1 + 1e-9) are
// safe: |x| / R <= 1e5 bounds the scaled coordinates' rounding error by
// ~2e-11 (in R units), far inside the margin, so no control with eta < 1
// is ever culled.  Outside these ranges the untiled exact kernel runs.
inline bool exact_tiled_ok(double R, double max_abs) {
  return R >= 1e-100 && R <= 1e100 && max_abs <= 1e100 && max_abs <= 1e5 * R;
}
// Morton index of the controls for the gathered exact kernel: tiles of 256
// (cx, cy, cz, insertion index) raw + per-tile boxes scaled by inv_R
// (device buffers of 4*ctrl_padded(n) and 6*ctrl_padded(n)/256 doubles)
void pack_exact_index_host(Context& ctx, const double* ctrl, size_t n, double inv_R, double* d_midx,
                           double* d_mbox);
// positions per CTA of the exact tiled kernel (128 threads x 2 points)
constexpr int kExactBlock = 256;
// longest-first processing order of the exact kernel's blocks: per block of
// bp ordered positions, the count of controls within R of its box, sorted
// descending (writes ceil(n / bp) block ids to `order`)
void block_order(Context& ctx, const double* x, const double* y, const double* z,
                 const uint32_t* active, const uint32_t* perm, size_t n, int bp,
                 const double* tiles, size_t nc, double R, bool fast_tiles, uint32_t* order);
// whether launch_volume(a) runs the exact tiled kernel with a block order
// (callers may cache block_order() results and pass them as a.cta_order)
bool exact_uses_block_order(const VolumeArgs& a);
// diagonal of the bounding box of n AoS points (host)
double bbox_diagonal(const double* xyz, size_t n);
// per-tile boxes (scaled by inv_R) of exact tiles, real controls only
void exact_tile_boxes(Context& ctx, const double* tiles, size_t n, double inv_R, double* boxes);

// Stable compaction of {i : dist[i] < D} (wall_distance.cpp:56-58).  Writes
// ascending node ids to d_out and returns the count (synchronises).
size_t compact_active(Context& ctx, const double* d_dist, size_t n, double D, uint32_t* d_out);

// Device permutation of the n active positions ordered by grid cells of
// edge ~2R (spatially compact CTAs for the tile culling).
void spatial_order(Context& ctx, const double* x, const double* y, const double* z,
                   const uint32_t* active, size_t n, double R, DBuf<uint32_t>& perm);
// Asynchronous variant (no host synchronisation, context scratch).
void spatial_order(Context& ctx, const double* x, const double* y, const double* z,
                   const uint32_t* active, size_t n, double R, uint32_t* perm);
void scan_u32_to_u64_async(Context& ctx, const unsigned int* in, size_t n, unsigned long long* out);
// Grows every scratch slot spatial_order / the exact block order use to the
// size n needs (so later calls with <= n points never reallocate mid-pipeline)
void reserve_spatial_order(Context& ctx, size_t n);

// Number of (active node, control) pairs with |r_v - r_c| < R (fast path
// arithmetic, tiles packed with scale 1/R).
unsigned long long count_support_pairs(Context& ctx, const DPoints& nodes, const uint32_t* active,
                                       size_t n, const double* tiles, size_t nc, double inv_R);

// Exclusive scan of n u32 counts into n+1 u64 offsets (out[n] = total).
void scan_u32_to_u64(Context& ctx, const unsigned int* in, size_t n, unsigned long long* out);

// Exact wall distance (wall_distance.cpp:13-31).  cutoff = +inf for exact
// distances everywhere; a finite cutoff lets the search stop once no surface
// point can lie closer than cutoff (such nodes get +inf, i.e. inactive).
// quality.cpp:135-148 on the device: signed measure of every element (out may
// be null) and the number with measure <= 0.  Element arrays are device CSR.
size_t signed_measures(Context& ctx, const double* x, const double* y, const double* z,
                       size_t n_nodes, const int* kinds, const unsigned long long* offsets,
                       const unsigned long long* conn, size_t n_elem, double* out);
// quality.cpp:150-236 orthogonality on the device (elements device CSR):
// per-element scores (device pointer, may be null), signed measures (device
// pointer, may be null), report scalars.
struct QualityStats {
  double min_deg = 90.0, mean_deg = 90.0;
  size_t inverted = 0, degenerate = 0;
};
QualityStats orthogonality_device(Context& ctx, const double* x, const double* y, const double* z,
                                  size_t n_nodes, const int* kinds, const unsigned long long* offsets,
                                  const unsigned long long* conn, size_t n_elem, double* scores_host,
                                  double* measures_device);
QualityStats orthogonality_from_host(Context& ctx, const double* x, const double* y, const double* z,
                                     size_t n_nodes, const int* kinds, const size_t* offsets,
                                     const size_t* conn, size_t n_elem, double* scores,
                                     double* measures);
// Same with the element CSR (and out) on the host; uploads through context slots.
size_t signed_measures_from_host(Context& ctx, const double* x, const double* y, const double* z,
                                 size_t n_nodes, const int* kinds, const size_t* offsets,
                                 const size_t* conn, size_t n_elem, double* out);

void wall_distance(Context& ctx, const DPoints& nodes, size_t n_nodes, const DPoints& surface,
                   size_t n_surface, int dim, double cutoff, double* d_out);

}  // namespace imb

// The opaque handle of the C-ABI (include/icemorph_b200.h).
struct im_context {
  imb::Context c;
};
