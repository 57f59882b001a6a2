// capi.cu — the extern "C" boundary (include/icemorph_b200.h).
//
// Host orchestration only: validation with the reference's messages, the
// H2D/D2H transfers, and the kernel sequences of volume.cu, wall_distance.cu
// and greedy.cu.  Host arithmetic that must match the reference bit for bit
// (max_magnitude, the SolveError distances, the surface error) is compiled
// with -ffp-contract=off and follows the cited reference lines.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/icemorph_b200.h"
#include "greedy.hpp"
#include "host_io.hpp"
#include "su2_io.hpp"
#include "runtime.hpp"

namespace imb {
namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t) {
  return std::chrono::duration<double>(Clock::now() - t).count();
}

// ---- host reference arithmetic --------------------------------------------
// vec.hpp:35-36
double hnorm(double x, double y, double z) { return std::sqrt(x * x + y * y + z * z); }
double hdist(const double* a, const double* b) {
  return hnorm(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
}
// greedy.cpp:35-39
double max_magnitude(const double* v, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, hnorm(v[3 * i], v[3 * i + 1], v[3 * i + 2]));
  return m;
}
// rbf.cpp:28-50
double h_wendland(int kind, double eta) {
  if (eta >= 1.0) return 0.0;
  const double u = 1.0 - eta;
  switch (kind) {
    case 0: return u * u;
    case 1: {
      const double u2 = u * u;
      return u2 * u2 * (4.0 * eta + 1.0);
    }
    case 2: {
      const double u2 = u * u;
      const double u6 = u2 * u2 * u2;
      return u6 * ((35.0 / 3.0) * eta * eta + 6.0 * eta + 1.0);
    }
    case 3: {
      const double u2 = u * u;
      const double u8 = u2 * u2 * u2 * u2;
      return u8 * (32.0 * eta * eta * eta + 25.0 * eta * eta + 8.0 * eta + 1.0);
    }
  }
  return 0.0;
}

void check_kind(int kind) {
  if (kind < 0 || kind > 3)
    throw InvalidArgument("unknown basis function (expected c0, c2, c4 or c6)");
}

// greedy.cpp:20-33
void check_config(const im_greedy_config& c) {
  if (!(c.tolerance > 0.0 && c.tolerance < 1.0))
    throw InvalidArgument("greedy tolerance must lie in (0,1)");
  if (c.max_levels < 1) throw InvalidArgument("at least one level is required");
  if (c.max_points_per_level < 1) throw InvalidArgument("per-level point cap must be positive");
  if (!(c.basis.support_radius > 0.0))
    throw InvalidArgument("basis support radius must be positive");
  check_kind(c.basis.kind);
}

std::string fmt_f(double v) { return std::to_string(v); }  // std::to_string == "%f"

// greedy.cpp:41-56
[[noreturn]] void throw_conditioning_nodes(const double* pos, const std::vector<int>& controls,
                                           size_t failed) {
  size_t nearest = failed;
  double best = INFINITY;
  for (int c : controls) {
    const double d = hdist(pos + 3 * (size_t)c, pos + 3 * failed);
    if (d < best) best = d, nearest = (size_t)c;
  }
  throw SolveFailure("ill-conditioned control set: surface nodes " + std::to_string(nearest) +
                     " and " + std::to_string(failed) + " are too close (distance " +
                     fmt_f(best) + ")");
}

// rbf.cpp:125-140
[[noreturn]] void throw_conditioning_points(const double* pts, size_t failed) {
  size_t nearest = 0;
  double best = INFINITY;
  for (size_t i = 0; i < failed; ++i) {
    const double d = hdist(pts + 3 * i, pts + 3 * failed);
    if (d < best) best = d, nearest = i;
  }
  throw SolveFailure("ill-conditioned control set: points " + std::to_string(nearest) + " and " +
                     std::to_string(failed) + " are too close (distance " + fmt_f(best) + ")");
}

template <class F>
int guarded(im_context* ctx, F&& f) {
  if (!ctx) return IM_INVALID_ARGUMENT;
  Context& c = ctx->c;
  try {
    IMB_CHECK(cudaSetDevice(c.device));
    f(c);
    c.status = IM_OK;
    c.message[0] = 0;
  } catch (const ParseFailure& e) {
    c.status = IM_PARSE_ERROR;
    c.error_line = e.line;
    std::snprintf(c.message, sizeof c.message, "%s", e.what());
  } catch (const InvalidArgument& e) {
    c.status = IM_INVALID_ARGUMENT;
    std::snprintf(c.message, sizeof c.message, "%s", e.what());
  } catch (const std::invalid_argument& e) {
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

// IMB_TRACE=1: per-phase host wall times of a C-ABI call on stderr (each mark
// synchronises the stream, so only for diagnosis).
struct PhaseTrace {
  cudaStream_t s;
  bool on;
  Clock::time_point t;
  explicit PhaseTrace(cudaStream_t st) : s(st), on(std::getenv("IMB_TRACE") != nullptr), t(Clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = Clock::now();
    std::fprintf(stderr, "[imb] %-28s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

struct EventTimer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t st) : s(st) {
    IMB_CHECK(cudaEventCreate(&a));
    IMB_CHECK(cudaEventCreate(&b));
    IMB_CHECK(cudaEventRecord(a, s));
  }
  double stop() {
    IMB_CHECK(cudaEventRecord(b, s));
    IMB_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    IMB_CHECK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// One greedy level on an engine whose target is already set.
struct LevelOut {
  int nc = 0, steps = 0, status = 0;
  double achieved = 0, target_max = 0, elapsed = 0;
};

LevelOut run_engine_level(GreedyEngine& eng, const double* host_pos, const im_greedy_config& cfg,
                          double target_max) {
  const auto t0 = Clock::now();
  eng.reset(cfg.tolerance, target_max, cfg.basis.kind, cfg.basis.support_radius);
  const GState& s = eng.run_level();
  LevelOut o;
  o.status = s.status;
  o.nc = s.nc;
  o.steps = s.steps;
  o.achieved = s.achieved;
  o.target_max = target_max;
  if (s.status == kStatusSolveError) {
    std::vector<size_t> idx(s.nc);
    eng.download(s.nc, idx.data(), nullptr, nullptr, nullptr, nullptr, 0);
    std::vector<int> ctl(idx.begin(), idx.end());
    throw_conditioning_nodes(host_pos, ctl, (size_t)s.fail_node);
  }
  o.elapsed = seconds_since(t0);
  return o;
}

void validate_target(const double* t, size_t n) {
  for (size_t i = 0; i < 3 * n; ++i)
    if (!std::isfinite(t[i])) throw InvalidArgument("target displacement is not finite");
}

}  // namespace
}  // namespace imb

using namespace imb;

extern "C" {

const char* im_version(void) { return "icemorph-b200 0.1 (sm_100a)"; }

int im_context_create(im_context** out, int device) {
  if (!out) return IM_INVALID_ARGUMENT;
  *out = nullptr;
  auto* ctx = new (std::nothrow) im_context();
  if (!ctx) return IM_RUNTIME_ERROR;
  ctx->c.device = device;
  int rc = guarded(ctx, [&](Context& c) {
    IMB_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    cudaDeviceProp prop;
    IMB_CHECK(cudaGetDeviceProperties(&prop, device));
    c.num_sms = prop.multiProcessorCount;
    if (prop.major != 10)
      throw std::runtime_error("icemorph-b200 requires an sm_100 (Blackwell B200) device");
  });
  *out = ctx;  // returned even on failure so im_last_error can be read
  return rc;
}

int im_context_destroy(im_context* ctx) {
  if (!ctx) return IM_OK;
  if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  for (cudaStream_t st : ctx->c.side)
    if (st) cudaStreamDestroy(st);
  delete ctx;
  return IM_OK;
}

const char* im_last_error(const im_context* ctx) { return ctx ? ctx->c.message : "null context"; }
double im_last_device_ms(const im_context* ctx) { return ctx ? ctx->c.last_kernel_ms : 0.0; }
unsigned long long im_count_pairs(im_context* ctx, int enable) {
  if (!ctx) return 0;
  const unsigned long long n = ctx->c.pairs_evaluated;
  ctx->c.count_pairs = enable != 0;
  ctx->c.pairs_evaluated = 0;
  return n;
}
void im_last_transfer_bytes(const im_context* ctx, unsigned long long* h2d, unsigned long long* d2h) {
  if (h2d) *h2d = ctx ? ctx->c.last_h2d_bytes : 0;
  if (d2h) *d2h = ctx ? ctx->c.last_d2h_bytes : 0;
}

double im_eval_wendland(int kind, double eta) { return h_wendland(kind, eta); }
double im_eval_basis(im_basis b, double distance) {
  return h_wendland(b.kind, distance / b.support_radius);
}

// wall_distance.cpp:33-38
int im_make_wall_function(double k, double level_target_max, im_wall_function* out) {
  if (!(k > 0.0)) return IM_INVALID_ARGUMENT;
  out->reduction_factor = k;
  out->support_distance = k * level_target_max;
  out->psi_kind = IM_PSI_LINEAR;
  return IM_OK;
}

// wall_distance.cpp:40-44 (+ the Wendland-C2 taper)
double im_eval_wall_function(const im_wall_function* wf, double d) {
  if (wf->support_distance <= 0.0) return d == 0.0 ? 1.0 : 0.0;
  const double xi = d / wf->support_distance;
  if (wf->psi_kind == IM_PSI_WENDLAND_C2) return h_wendland(1, xi);
  return xi < 1.0 ? 1.0 - xi : 0.0;
}

int im_solve_weights(im_context* ctx, const double* points, const double* disp, size_t n,
                     im_basis basis, double* alpha_out) {
  return guarded(ctx, [&](Context& c) {
    check_kind(basis.kind);
    std::fill(alpha_out, alpha_out + 3 * n, 0.0);
    if (n == 0) return;
    bool all_zero = true;  // rbf.cpp:156-163
    for (size_t i = 0; i < 3 * n && all_zero; ++i) all_zero = disp[i] == 0.0;
    if (all_zero) return;
    GreedyEngine eng(c, (int)n, (int)n);
    eng.set_positions(points);
    eng.set_target(disp);
    eng.reset(0.5, 0.0, basis.kind, basis.support_radius);
    EventTimer tm(c.stream);
    const GState& s = eng.factor_all_and_solve();
    c.last_kernel_ms = tm.stop();
    if (s.status == kStatusSolveError) throw_conditioning_points(points, (size_t)s.fail_row);
    eng.download((int)n, nullptr, alpha_out, nullptr, nullptr, nullptr, 0);
  });
}

int im_eval_interpolant(im_context* ctx, const double* ctrl, const double* alpha, size_t nc,
                        im_basis basis, const double* queries, size_t nq, int precision,
                        double* out) {
  return guarded(ctx, [&](Context& c) {
    check_kind(basis.kind);
    precision_of(precision);
    if (nq == 0) return;
    DPoints q;
    upload_points(c, queries, nq, q);
    const size_t np = ctrl_padded(nc);
    DBuf<double> staging, tiles, dout;
    staging.reserve(6 * std::max<size_t>(nc, 1));
    tiles.reserve(ctrl_tile_doubles(nc));
    dout.reserve(3 * nq);
    if (nc) {
      IMB_CHECK(cudaMemcpyAsync(staging.p, ctrl, nc * 24, cudaMemcpyHostToDevice, c.stream));
      IMB_CHECK(cudaMemcpyAsync(staging.p + 3 * nc, alpha, nc * 24, cudaMemcpyHostToDevice, c.stream));
    }
    const bool exact = precision == IM_EXACT;
    DBuf<double> boxes;
    if (exact)
      pack_controls_aos(c, staging.p, staging.p + 3 * nc, nc, 1.0, tiles.p);
    else
      pack_controls_host(c, ctrl, alpha, nc, 1.0 / basis.support_radius, true, tiles, boxes);
    VolumeArgs a;
    a.tile_box = exact ? nullptr : boxes.p;
    a.x = q.x.p, a.y = q.y.p, a.z = q.z.p;
    a.n_active = nq;
    a.tiles = tiles.p;
    a.n_ctrl = nc;
    a.R = basis.support_radius;
    a.kind = basis.kind;
    a.dim = 3;
    a.precision = precision_of(precision);
    a.out_val = dout.p;
    EventTimer tm(c.stream);
    launch_volume(c, a);
    c.last_kernel_ms = tm.stop();
    sync_copy(c.stream, out, dout.p, nq * 24, cudaMemcpyDeviceToHost);
  });
}

int im_greedy_level(im_context* ctx, const double* pos, const double* target, size_t n,
                    const im_greedy_config* cfg, size_t level_index, size_t* control_indices,
                    double* alpha, size_t* n_controls, double* achieved_error, int* cap_hit,
                    double* target_max, double* elapsed_seconds, size_t* record_points,
                    double* record_error, double* record_seconds, size_t* n_records,
                    double* residual) {
  (void)level_index;
  return guarded(ctx, [&](Context& c) {
    check_config(*cfg);
    if (n == 0) throw InvalidArgument("surface point set is empty");
    validate_target(target, n);
    const double tmax = max_magnitude(target, n);
    const int cap = (int)std::min<size_t>(cfg->max_points_per_level, n);
    GreedyEngine eng(c, (int)n, cap);
    eng.set_positions(pos);
    eng.set_target(target);
    EventTimer tm(c.stream);
    LevelOut o = run_engine_level(eng, pos, *cfg, tmax);
    c.last_kernel_ms = tm.stop();
    std::vector<double> sec(o.steps);
    eng.download(o.nc, control_indices, alpha, residual, record_error,
                 record_seconds ? record_seconds : sec.data(), o.steps);
    *n_controls = o.nc;
    *achieved_error = o.achieved;
    *cap_hit = o.status == kStatusCapHit ? 1 : 0;
    *target_max = tmax;
    if (elapsed_seconds) *elapsed_seconds = o.elapsed;
    if (record_points)
      for (int s = 0; s < o.steps; ++s) record_points[s] = (size_t)s + 1;
    *n_records = o.steps;
  });
}

int im_run_multilevel(im_context* ctx, const double* pos, const double* target, size_t n,
                      const im_greedy_config* cfg, size_t* n_levels, size_t* n_controls,
                      size_t* control_indices, double* alpha, double* achieved_error,
                      int* cap_hit, double* level_target_max, double* elapsed_seconds,
                      size_t* n_records, double* record_error, double* target_max,
                      double* final_residual) {
  return guarded(ctx, [&](Context& c) {
    check_config(*cfg);
    const double tmax = max_magnitude(target, n);
    *target_max = tmax;
    if (n == 0) throw InvalidArgument("surface point set is empty");
    validate_target(target, n);
    const size_t m = std::min<size_t>(cfg->max_points_per_level, n);
    const double threshold = std::pow(cfg->tolerance, (double)cfg->max_levels) * tmax;
    GreedyEngine eng(c, (int)n, (int)m);
    eng.set_positions(pos);
    eng.set_target(target);
    std::vector<double> current(target, target + 3 * n);
    EventTimer tm(c.stream);
    size_t nl = 0;
    for (size_t l = 0; l < cfg->max_levels; ++l) {
      const double cur_max = max_magnitude(current.data(), n);
      if (l > 0 && (cur_max == 0.0 || cur_max < threshold)) break;  // greedy.cpp:187
      if (l > 0) eng.target_from_residual();
      LevelOut o = run_engine_level(eng, pos, *cfg, cur_max);
      eng.download(o.nc, control_indices + l * m, alpha + 3 * l * m, current.data(),
                   record_error ? record_error + l * m : nullptr, nullptr, o.steps);
      n_controls[l] = o.nc;
      achieved_error[l] = o.achieved;
      cap_hit[l] = o.status == kStatusCapHit ? 1 : 0;
      level_target_max[l] = cur_max;
      if (elapsed_seconds) elapsed_seconds[l] = o.elapsed;
      n_records[l] = o.steps;
      ++nl;
    }
    c.last_kernel_ms = tm.stop();
    *n_levels = nl;
    if (final_residual) std::memcpy(final_residual, current.data(), 24 * n);
  });
}

int im_signed_measures(im_context* ctx, const double* nodes, size_t n_nodes, const int* kinds,
                       const size_t* offsets, const size_t* conn, size_t n_elem, double* measures,
                       size_t* inverted) {
  return guarded(ctx, [&](Context& c) {
    DPoints dn;
    upload_points(c, nodes, n_nodes, dn);
    EventTimer tm(c.stream);
    const size_t k =
        signed_measures_from_host(c, dn.x.p, dn.y.p, dn.z.p, n_nodes, kinds, offsets, conn, n_elem,
                                  measures);
    c.last_kernel_ms = tm.stop();
    if (inverted) *inverted = k;
  });
}

int im_orthogonality(im_context* ctx, const double* nodes, size_t n_nodes, const int* kinds,
                     const size_t* offsets, const size_t* conn, size_t n_elem, double* scores,
                     double* measures, im_quality_report* rep) {
  return guarded(ctx, [&](Context& c) {
    DPoints dn;
    upload_points(c, nodes, n_nodes, dn);
    EventTimer tm(c.stream);
    const QualityStats q = orthogonality_from_host(c, dn.x.p, dn.y.p, dn.z.p, n_nodes, kinds, offsets,
                                                   conn, n_elem, scores, measures);
    c.last_kernel_ms = tm.stop();
    rep->min_orthogonality_deg = q.min_deg;
    rep->mean_orthogonality_deg = q.mean_deg;
    rep->inverted_count = q.inverted;
    rep->degenerate_count = q.degenerate;
  });
}

int im_count_inverted(im_context* ctx, const double* nodes, size_t n_nodes, const int* kinds,
                      const size_t* offsets, const size_t* conn, size_t n_elem, size_t* inverted) {
  return im_signed_measures(ctx, nodes, n_nodes, kinds, offsets, conn, n_elem, nullptr, inverted);
}

// ---- SU2 mesh I/O -------------------------------------------------------------------
}  // extern "C"
struct im_mesh {
  imb::HostMesh m;
};

namespace imb {
namespace {

// Node-chunk granularity of the selective upload in im_update_volume
// (IMB_E2E_CHUNK overrides; 0 selects the single-pass path): meshes below
// 64k nodes take the single pass; larger ones 64k-node chunks, <= 1024.
size_t e2e_chunk_nodes(size_t n) {
  if (const char* e = std::getenv("IMB_E2E_CHUNK")) {
    const long long v = std::atoll(e);
    return v <= 0 ? n : std::max<size_t>(std::min(n, (size_t)v), (n + 1023) / 1024);
  }
  if (n < (size_t(1) << 16)) return n;
  return std::max(size_t(1) << 16, (n + 1023) / 1024);
}

struct EventSet {
  std::vector<cudaEvent_t> e;
  explicit EventSet(size_t n) : e(n, nullptr) {
    for (auto& x : e) IMB_CHECK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
  }
  ~EventSet() {
    for (auto x : e)
      if (x) cudaEventDestroy(x);
  }
  cudaEvent_t operator[](size_t i) const { return e[i]; }
};

// im_update_volume with transfers cut to what the update reads and
// overlapped with the device work.  The reference API hands over the whole
// mesh on every call, but update_volume only reads the coordinates of nodes
// with d < D (wall_distance.cpp:56-62):
//   side stream 0: the distances (the compaction needs only them), then the
//                  node chunks that hold at least one active node, merged into
//                  runs (AoS upload + SoA conversion per run);
//   ctx.stream:    the stable compaction of the whole mesh while the node
//                  upload has not started, then — once the runs landed — the
//                  range / planarity reduction over the active nodes, the
//                  spatial order and ONE volume kernel over all active nodes
//                  (the single-pass kernel, same block balance);
//   side stream 1: the active ids right after the compaction (widened to
//                  size_t on the host while the kernel runs), the values
//                  after the kernel (direct DMA into page-locked output).
// Layer-ordered meshes keep their near-wall (active) nodes in a few
// contiguous runs, so the node upload shrinks to the active fraction
// (cfg3: ~20 %); any ordering stays correct, it only uploads more.
void update_volume_selective(Context& c, const double* nodes, size_t n_nodes, const double* dist,
                             const double* ctrl, const double* alpha, size_t nc,
                             const im_wall_function* wf, im_basis basis, Precision prec,
                             size_t* entry_nodes, double* entry_values, size_t* n_entries,
                             size_t chunk) {
  PhaseTrace tr(c.stream);
  const double D = wf->support_distance, R = basis.support_radius;
  const bool exact = prec == Precision::Exact;
  cudaStream_t up = c.side_stream(0), down = c.side_stream(1);
  double* dx = c.buf<double>(Context::kSlotNodesX, n_nodes);
  double* dy = c.buf<double>(Context::kSlotNodesY, n_nodes);
  double* dz = c.buf<double>(Context::kSlotNodesZ, n_nodes);
  double* dd = c.buf<double>(Context::kSlotDist, n_nodes);
  uint32_t* active = c.buf<uint32_t>(Context::kSlotActive, n_nodes);
  double* stage = c.buf<double>(Context::kSlotStage, 3 * n_nodes + 6 * nc);
  EventSet ev(4);  // 0: distances up, 1: nodes up, 2: ids down, 3: kernel done
  // 1. distances
  const H2DJob jd{dd, dist, n_nodes * 8};
  staged_h2d(c, &jd, 1, 192, {}, up);
  IMB_CHECK(cudaEventRecord(ev[0], up));
  tr.mark("dist up");
  // 2. stable compaction of the whole mesh, active count per node chunk
  IMB_CHECK(cudaStreamWaitEvent(c.stream, ev[0], 0));
  EventTimer tm(c.stream);
  const size_t na = compact_active(c, dd, n_nodes, D, active);
  *n_entries = na;
  if (na == 0) {
    c.last_kernel_ms = tm.stop();
    return;
  }
  const size_t n_chunks = (n_nodes + chunk - 1) / chunk;
  std::vector<size_t> bounds(n_chunks + 1), pos(n_chunks + 1);
  for (size_t i = 0; i <= n_chunks; ++i) bounds[i] = std::min(n_nodes, i * chunk);
  active_lower_bounds(c, active, na, bounds.data(), (int)n_chunks + 1, pos.data());
  // ids down as soon as they exist
  unsigned char* pin = pinned_out(c, 4 * na + 24 * na + 32);
  uint32_t* pin_ids = reinterpret_cast<uint32_t*>(pin);
  double* pin_vals = reinterpret_cast<double*>(pin + ((4 * na + 15) / 16) * 16);
  IMB_CHECK(cudaEventRecord(ev[2], c.stream));
  IMB_CHECK(cudaStreamWaitEvent(down, ev[2], 0));
  IMB_CHECK(cudaMemcpyAsync(pin_ids, active, 4 * na, cudaMemcpyDeviceToHost, down));
  IMB_CHECK(cudaEventRecord(ev[2], down));
  // 3. node runs holding active nodes: upload + SoA (side stream 0)
  size_t uploaded = 0;
  for (size_t i = 0; i < n_chunks;) {
    if (pos[i + 1] == pos[i]) {
      ++i;
      continue;
    }
    size_t j = i + 1;
    while (j < n_chunks && pos[j + 1] > pos[j]) ++j;
    const size_t b = bounds[i], m = bounds[j] - b;
    const H2DJob jn{stage + 3 * b, nodes + 3 * b, m * 24};
    staged_h2d(c, &jn, 1, 192, {}, up);
    aos_to_soa(c, stage + 3 * b, m, dx + b, dy + b, dz + b, up);
    uploaded += m;
    i = j;
  }
  // 4. controls: host packing overlaps the node upload
  double* tiles = c.buf<double>(Context::kSlotTiles, ctrl_tile_doubles(nc));
  double *boxes = nullptr, *midx = nullptr, *mbox = nullptr;
  double ctrl_max = 0.0;
  for (size_t i = 0; i < 3 * nc; ++i) ctrl_max = std::max(ctrl_max, std::fabs(ctrl[i]));
  bool ctrl_planar = true;
  for (size_t i = 0; i < nc && ctrl_planar; ++i)
    ctrl_planar = ctrl[3 * i + 2] == 0.0 && alpha[3 * i + 2] == 0.0;
  const bool ctrl_tiled_ok = exact && exact_tiled_ok(R, ctrl_max);
  if (exact) {
    double* cs = stage + 3 * n_nodes;
    if (nc) {
      IMB_CHECK(cudaMemcpyAsync(cs, ctrl, nc * 24, cudaMemcpyHostToDevice, c.stream));
      IMB_CHECK(cudaMemcpyAsync(cs + 3 * nc, alpha, nc * 24, cudaMemcpyHostToDevice, c.stream));
    }
    pack_controls_aos(c, cs, cs + 3 * nc, nc, 1.0, tiles);
    if (ctrl_tiled_ok) {
      boxes = c.buf<double>(Context::kSlotBoxes, 6 * (ctrl_padded(nc) / kCtrlTile));
      exact_tile_boxes(c, tiles, nc, 1.0 / R, boxes);
      midx = c.buf<double>(Context::kSlotIndex, 4 * ctrl_padded(nc));
      mbox = c.buf<double>(Context::kSlotIndexBox, 6 * (ctrl_padded(nc) / kCtrlTile));
      pack_exact_index_host(c, ctrl, nc, 1.0 / R, midx, mbox);
    }
  } else {
    boxes = c.buf<double>(Context::kSlotBoxes, 6 * (ctrl_padded(nc) / kCtrlTile));
    pack_controls_host(c, ctrl, alpha, nc, 1.0 / R, true, tiles, boxes);
  }
  IMB_CHECK(cudaEventRecord(ev[1], up));
  IMB_CHECK(cudaStreamWaitEvent(c.stream, ev[1], 0));
  // 5. coordinate range / planarity over the active nodes, then one kernel
  unsigned long long* dmax = c.buf<unsigned long long>(Context::kSlotChunkMax, 2);
  max_abs_points_async(dx, dy, dz, na, dmax, c.num_sms, c.stream, active);
  unsigned long long hm[2];
  IMB_CHECK(cudaMemcpyAsync(hm, dmax, 16, cudaMemcpyDeviceToHost, c.stream));
  IMB_CHECK(cudaStreamSynchronize(c.stream));
  double mx, mz;
  std::memcpy(&mx, &hm[0], 8);
  std::memcpy(&mz, &hm[1], 8);
  tr.mark("compact + node runs up");
  const bool tiled = ctrl_tiled_ok && exact_tiled_ok(R, std::max(mx, ctrl_max));
  const bool planar = mz == 0.0 && ctrl_planar;
  uint32_t* perm = nullptr;
  if (!exact || tiled) {
    perm = c.buf<uint32_t>(Context::kSlotPerm, na);
    spatial_order(c, dx, dy, dz, active, na, R, perm);
  }
  double* vals = c.buf<double>(Context::kSlotVals, 3 * na);
  VolumeArgs a;
  a.x = dx, a.y = dy, a.z = dz;
  a.active = active;
  a.n_active = na;
  a.dist = dd;
  a.D = D;
  a.psi_kind = wf->psi_kind;
  a.tiles = tiles;
  a.n_ctrl = nc;
  a.R = R;
  a.kind = basis.kind;
  a.dim = planar && (!exact || tiled) ? 2 : 3;
  a.precision = prec;
  a.exact_tiled = tiled;
  a.ctrl_index = tiled ? midx : nullptr;
  a.index_box = tiled ? mbox : nullptr;
  a.ctrl_diag = bbox_diagonal(ctrl, nc);
  a.out_val = vals;
  a.tile_box = exact && !tiled ? nullptr : boxes;
  a.perm = perm;
  launch_volume(c, a);
  IMB_CHECK(cudaEventRecord(ev[3], c.stream));
  // 6. values down; the ids are widened on the host meanwhile
  const bool vals_direct = host_is_pinned(entry_values);
  IMB_CHECK(cudaStreamWaitEvent(down, ev[3], 0));
  IMB_CHECK(cudaMemcpyAsync(vals_direct ? entry_values : pin_vals, vals, 24 * na,
                            cudaMemcpyDeviceToHost, down));
  IMB_CHECK(cudaEventSynchronize(ev[2]));
  constexpr size_t kPiece = size_t(1) << 16;
  const int pieces = (int)((na + kPiece - 1) / kPiece);
  host_pool(c).run(pieces, [&](int t) {
    const size_t k0 = (size_t)t * kPiece, k1 = std::min(na, k0 + kPiece);
    for (size_t k = k0; k < k1; ++k) entry_nodes[k] = pin_ids[k];
  });
  c.last_kernel_ms = tm.stop();
  tr.mark("order + kernel");
  IMB_CHECK(cudaStreamSynchronize(down));
  if (!vals_direct)
    host_pool(c).run(pieces, [&](int t) {
      const size_t k0 = (size_t)t * kPiece, k1 = std::min(na, k0 + kPiece);
      std::memcpy(entry_values + 3 * k0, pin_vals + 3 * k0, 24 * (k1 - k0));
    });
  tr.mark("values down");
  c.last_h2d_bytes = 8ull * n_nodes + 24ull * uploaded + 48ull * nc;
  c.last_d2h_bytes = 28ull * na;
  if (std::getenv("IMB_TRACE"))
    std::fprintf(stderr, "[imb]   selective upload: %zu of %zu nodes in %zu-node chunks, %zu active\n",
                 uploaded, n_nodes, chunk, na);
}

}  // namespace
}  // namespace imb

extern "C" {

int im_su2_read(im_context* ctx, const char* path, im_mesh** out) {
  if (!out) return IM_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded(ctx, [&](Context& c) {
    auto* mesh = new im_mesh{read_su2_file(c, host_pool(c), path ? path : "")};
    *out = mesh;
  });
}

int im_mesh_destroy(im_mesh* mesh) {
  delete mesh;
  return IM_OK;
}

int im_mesh_sizes(const im_mesh* mesh, int* dim, size_t* n_nodes, size_t* n_elements,
                  size_t* n_element_nodes, size_t* n_markers) {
  if (!mesh) return IM_INVALID_ARGUMENT;
  const HostMesh& m = mesh->m;
  if (dim) *dim = m.dim;
  if (n_nodes) *n_nodes = m.xyz.size() / 3;
  if (n_elements) *n_elements = m.kinds.size();
  if (n_element_nodes) *n_element_nodes = m.conn.size();
  if (n_markers) *n_markers = m.markers.size();
  return IM_OK;
}

int im_mesh_nodes(const im_mesh* mesh, double* xyz) {
  if (!mesh || !xyz) return IM_INVALID_ARGUMENT;
  std::memcpy(xyz, mesh->m.xyz.data(), mesh->m.xyz.size() * 8);
  return IM_OK;
}

int im_mesh_elements(const im_mesh* mesh, int* kinds, size_t* offsets, size_t* nodes) {
  if (!mesh) return IM_INVALID_ARGUMENT;
  const HostMesh& m = mesh->m;
  if (kinds) std::memcpy(kinds, m.kinds.data(), m.kinds.size() * sizeof(int));
  if (offsets) std::memcpy(offsets, m.offsets.data(), m.offsets.size() * 8);
  if (nodes) std::memcpy(nodes, m.conn.data(), m.conn.size() * 8);
  return IM_OK;
}

int im_mesh_marker_sizes(const im_mesh* mesh, size_t marker, size_t* name_length,
                         size_t* n_elements, size_t* n_element_nodes, size_t* n_nodes) {
  if (!mesh || marker >= mesh->m.markers.size()) return IM_INVALID_ARGUMENT;
  const auto& k = mesh->m.markers[marker];
  if (name_length) *name_length = k.name.size();
  if (n_elements) *n_elements = k.kinds.size();
  if (n_element_nodes) *n_element_nodes = k.conn.size();
  if (n_nodes) *n_nodes = k.nodes.size();
  return IM_OK;
}

int im_mesh_marker(const im_mesh* mesh, size_t marker, char* name, int* kinds, size_t* offsets,
                   size_t* element_nodes, size_t* nodes) {
  if (!mesh || marker >= mesh->m.markers.size()) return IM_INVALID_ARGUMENT;
  const auto& k = mesh->m.markers[marker];
  if (name) std::memcpy(name, k.name.data(), k.name.size());
  if (kinds) std::memcpy(kinds, k.kinds.data(), k.kinds.size() * sizeof(int));
  if (offsets) std::memcpy(offsets, k.offsets.data(), k.offsets.size() * 8);
  if (element_nodes) std::memcpy(element_nodes, k.conn.data(), k.conn.size() * 8);
  if (nodes) std::memcpy(nodes, k.nodes.data(), k.nodes.size() * 8);
  return IM_OK;
}

size_t im_last_error_line(const im_context* ctx) { return ctx ? ctx->c.error_line : 0; }

int im_su2_write(im_context* ctx, const char* path, int dim, const double* xyz, size_t n_nodes,
                 const int* kinds, const size_t* offsets, const size_t* nodes, size_t n_elements,
                 size_t n_markers, const char* const* names, const int* const* m_kinds,
                 const size_t* const* m_offsets, const size_t* const* m_nodes,
                 const size_t* m_n_elements) {
  return guarded(ctx, [&](Context& c) {
    HostMesh m;
    m.dim = dim;
    m.xyz.assign(xyz, xyz + 3 * n_nodes);
    m.kinds.assign(kinds, kinds + n_elements);
    m.offsets.assign(offsets, offsets + n_elements + 1);
    m.conn.assign(nodes, nodes + offsets[n_elements]);
    for (size_t k = 0; k < n_markers; ++k) {
      HostMesh::Marker mk;
      mk.name = names[k];
      const size_t ne = m_n_elements[k];
      mk.kinds.assign(m_kinds[k], m_kinds[k] + ne);
      mk.offsets.assign(m_offsets[k], m_offsets[k] + ne + 1);
      mk.conn.assign(m_nodes[k], m_nodes[k] + m_offsets[k][ne]);
      m.markers.push_back(std::move(mk));
    }
    write_su2_file(host_pool(c), path ? path : "", m);
  });
}

int im_build_distance_index(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
                            const size_t* surface, size_t n_surface, double* out) {
  return guarded(ctx, [&](Context& c) {
    if (n_surface == 0) throw InvalidArgument("cannot build a distance index for an empty patch");
    if (dim != 2 && dim != 3) throw InvalidArgument("kd-tree dim must be 2 or 3");
    for (size_t i = 0; i < n_surface; ++i)
      if (surface[i] >= n_nodes) throw InvalidArgument("surface node index out of range");
    DPoints dn, ds;
    upload_points(c, nodes, n_nodes, dn);
    upload_points_indexed(c, nodes, surface, n_surface, ds);
    DBuf<double> d;
    d.reserve(n_nodes);
    EventTimer tm(c.stream);
    wall_distance(c, dn, n_nodes, ds, n_surface, dim, INFINITY, d.p);
    c.last_kernel_ms = tm.stop();
    sync_copy(c.stream, out, d.p, n_nodes * 8, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n_surface; ++i) out[surface[i]] = 0.0;  // wall_distance.cpp:29
  });
}

int im_update_volume(im_context* ctx, const double* nodes, size_t n_nodes, const double* dist,
                     const double* ctrl, const double* alpha, size_t nc,
                     const im_wall_function* wf, im_basis basis, int precision,
                     size_t* entry_nodes, double* entry_values, size_t* n_entries) {
  return guarded(ctx, [&](Context& c) {
    PhaseTrace tr(c.stream);
    check_kind(basis.kind);
    *n_entries = 0;
    c.last_h2d_bytes = c.last_d2h_bytes = 0;
    const double D = wf->support_distance;
    if (D <= 0.0 || n_nodes == 0) {  // wall_distance.cpp:54
      precision_of(precision);
      return;
    }
    const size_t chunk = e2e_chunk_nodes(n_nodes);
    if (chunk < n_nodes)
      return update_volume_selective(c, nodes, n_nodes, dist, ctrl, alpha, nc, wf, basis,
                                     precision_of(precision), entry_nodes, entry_values,
                                     n_entries, chunk);
    // device buffers come from the context's grow-only slots: no cudaMalloc /
    // cudaFree on this path
    double* dx = c.buf<double>(Context::kSlotNodesX, n_nodes);
    double* dy = c.buf<double>(Context::kSlotNodesY, n_nodes);
    double* dz = c.buf<double>(Context::kSlotNodesZ, n_nodes);
    double* dd = c.buf<double>(Context::kSlotDist, n_nodes);
    uint32_t* active = c.buf<uint32_t>(Context::kSlotActive, n_nodes);
    double* stage = c.buf<double>(Context::kSlotStage, 3 * n_nodes + 6 * nc);
    const bool exact = precision == IM_EXACT;
    // nodes + distances through the pinned staging pool (or straight to the
    // copy engine when the caller's arrays are page-locked)
    const H2DJob up[2] = {{stage, nodes, n_nodes * 24}, {dd, dist, n_nodes * 8}};
    staged_h2d(c, up, 2);
    aos_to_soa(c, stage, n_nodes, dx, dy, dz);
    tr.mark("h2d nodes+dist");
    double* tiles = c.buf<double>(Context::kSlotTiles, ctrl_tile_doubles(nc));
    double* boxes = nullptr;
    if (exact) {
      double* cs = stage + 3 * n_nodes;
      if (nc) {
        IMB_CHECK(cudaMemcpyAsync(cs, ctrl, nc * 24, cudaMemcpyHostToDevice, c.stream));
        IMB_CHECK(cudaMemcpyAsync(cs + 3 * nc, alpha, nc * 24, cudaMemcpyHostToDevice, c.stream));
      }
      pack_controls_aos(c, cs, cs + 3 * nc, nc, 1.0, tiles);
    } else {
      boxes = c.buf<double>(Context::kSlotBoxes, 6 * (ctrl_padded(nc) / kCtrlTile));
      pack_controls_host(c, ctrl, alpha, nc, 1.0 / basis.support_radius, true, tiles, boxes);
    }
    // exact: the tiled kernel (spatial order + exact-safe culling) when the
    // coordinate / R ranges allow its branch-free sqrt and division
    // planar input (z == 0 everywhere) runs the 2-D kernels; the range of the
    // coordinates decides the exact path's kernel (one device reduction)
    double max_z = 0.0;
    const double max_abs = max_abs_points(c, dx, dy, dz, n_nodes, &max_z);
    bool tiled_exact = false;
    double *midx = nullptr, *mbox = nullptr;
    if (exact) {
      double m = max_abs;
      for (size_t i = 0; i < 3 * nc; ++i) m = std::max(m, std::fabs(ctrl[i]));
      tiled_exact = exact_tiled_ok(basis.support_radius, m);
      if (tiled_exact) {
        boxes = c.buf<double>(Context::kSlotBoxes, 6 * (ctrl_padded(nc) / kCtrlTile));
        exact_tile_boxes(c, tiles, nc, 1.0 / basis.support_radius, boxes);
        midx = c.buf<double>(Context::kSlotIndex, 4 * ctrl_padded(nc));
        mbox = c.buf<double>(Context::kSlotIndexBox, 6 * (ctrl_padded(nc) / kCtrlTile));
        pack_exact_index_host(c, ctrl, nc, 1.0 / basis.support_radius, midx, mbox);
      }
    }
    bool planar = max_z == 0.0;
    for (size_t i = 0; i < nc && planar; ++i) planar = ctrl[3 * i + 2] == 0.0 && alpha[3 * i + 2] == 0.0;
    tr.mark("controls + planar");
    EventTimer tm(c.stream);
    const size_t na = compact_active(c, dd, n_nodes, D, active);
    uint32_t* perm = nullptr;
    if ((!exact || tiled_exact) && na) {
      perm = c.buf<uint32_t>(Context::kSlotPerm, na);
      spatial_order(c, dx, dy, dz, active, na, basis.support_radius, perm);
    }
    double* vals = c.buf<double>(Context::kSlotVals, 3 * std::max<size_t>(na, 1));
    VolumeArgs a;
    a.x = dx, a.y = dy, a.z = dz;
    a.active = active;
    a.n_active = na;
    a.dist = dd;
    a.D = D;
    a.psi_kind = wf->psi_kind;
    a.tiles = tiles;
    a.n_ctrl = nc;
    a.R = basis.support_radius;
    a.kind = basis.kind;
    a.dim = planar && (!exact || tiled_exact) ? 2 : 3;
    a.precision = precision_of(precision);
    a.exact_tiled = tiled_exact;
    a.ctrl_index = midx, a.index_box = mbox;
    a.ctrl_diag = bbox_diagonal(ctrl, nc);
    a.out_val = vals;
    a.tile_box = boxes;
    a.perm = perm;
    launch_volume(c, a);
    c.last_kernel_ms = tm.stop();
    tr.mark("compact + order + kernel");
    // ascending node ids (widened to size_t) + values, chunked through pinned
    // memory (wall_distance.cpp:55-62 entry order)
    const D2HJob down[2] = {{active, entry_nodes, na, 4, true}, {vals, entry_values, 3 * na, 8, false}};
    staged_d2h(c, down, 2);
    *n_entries = na;
    c.last_h2d_bytes = 32ull * n_nodes + 48ull * nc;
    c.last_d2h_bytes = 28ull * na;
    tr.mark("d2h");
  });
}

}  // extern "C"
