// pipeline.cu — deform() orchestration on the device (pipeline.cpp:19-106)
// and the resident volume plan used by the benchmark.
//
// deform: surface system = patch ++ pinned (pipeline.cpp:35-53) ->
//         run_multilevel on the device engine (greedy.cu) ->
//         wall distances once on the undeformed mesh, culled at the largest
//         support distance (wall_distance.cu) ->
//         per level: stable compaction of d < D_l, then the volume update
//         accumulated into the resident node array in level order, pinned
//         nodes skipped (pipeline.cpp:64-73) ->
//         surface max/mean error (pipeline.cpp:87-99).
// The mesh crosses PCIe once in each direction.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <unordered_set>
#include <vector>

#include "../../include/icemorph_b200.h"
#include "greedy.hpp"
#include "host_io.hpp"
#include "runtime.hpp"

namespace imb {
namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

double hnorm(double x, double y, double z) { return std::sqrt(x * x + y * y + z * z); }
double max_magnitude(const double* v, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, hnorm(v[3 * i], v[3 * i + 1], v[3 * i + 2]));
  return m;
}

[[noreturn]] void throw_conditioning_nodes(const double* pos, const std::vector<size_t>& controls,
                                           size_t failed) {
  size_t nearest = failed;
  double best = INFINITY;
  for (size_t c : controls) {
    const double* a = pos + 3 * c;
    const double* b = pos + 3 * failed;
    const double d = hnorm(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
    if (d < best) best = d, nearest = c;
  }
  throw SolveFailure("ill-conditioned control set: surface nodes " + std::to_string(nearest) +
                     " and " + std::to_string(failed) + " are too close (distance " +
                     std::to_string(best) + ")");
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

bool all_z_zero(const double* xyz, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (xyz[3 * i + 2] != 0.0) return false;
  return true;
}

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double ms() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float m = 0;
    cudaEventElapsedTime(&m, a, b);
    return m;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

__global__ void k_zero_at(double* d, const unsigned long long* idx, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[idx[i]] = 0.0;
}

__global__ void k_set_flags(unsigned char* f, const unsigned long long* idx, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[idx[i]] = 1;
}

__global__ void k_gather(const double* src, const uint32_t* order, size_t n, double* dst) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

__global__ void k_scatter_aos(const double* x, const double* y, const double* z,
                              const uint32_t* order, size_t n, double* aos) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t o = order[i];
  aos[3 * o] = x[i];
  aos[3 * o + 1] = y[i];
  aos[3 * o + 2] = z[i];
}

__global__ void k_scatter1(const double* src, const uint32_t* order, size_t n, double* dst) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[order[i]] = src[i];
}

__global__ void k_soa_to_aos(const double* x, const double* y, const double* z, size_t n,
                             double* aos) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  aos[3 * i] = x[i];
  aos[3 * i + 1] = y[i];
  aos[3 * i + 2] = z[i];
}

}  // namespace
}  // namespace imb

using namespace imb;

struct im_volume_plan {
  im_context* ctx;
  size_t n = 0;
  int dim = 3;
  DPoints nodes, field;
  DPoints surf;  // the wall (for the HBM-pass benchmark)
  size_t n_surface = 0;
  int sdim = 3;
  DBuf<double> dist, tiles, ctrl_stage;
  DBuf<uint32_t> active;
  size_t nc = 0;
  // multi-level step (bench): per-level packed controls and support distance
  struct Level {
    DBuf<double> tiles, boxes, midx, mbox;
    bool culled = false;
    bool exact_tiled = false;
    bool exact_format = false;  // packed for IM_EXACT (insertion-order tiles)
    double diag = 0.0;
    DBuf<uint32_t> order;  // cached longest-first block order (exact kernel)
    size_t order_n = 0;
    std::vector<double> host_ctrl, host_alpha;  // for count_support (fast-format tiles)
    size_t nc = 0;
    double D = 0.0;
    int psi_kind = 0;
    bool planar = false;  // 2-D kernels: planar mesh, controls and z weights
  };
  Level levels[8];
  int n_levels = 0;
  std::vector<double> host_ctrl, host_alpha;  // set_controls (single-level API)
  DBuf<uint32_t> perm;
  // spatial layout: node k' of the resident arrays is original node order[k']
  // (grid-cell order, so compacted active sets are spatially coherent)
  DBuf<uint32_t> order;
  bool reordered = false;
  DBuf<unsigned char> flush;
};

// the 2-D kernels take z == 0 for nodes and controls and write vz = 0:
// only valid when every control's z and z weight are zero as well
bool planar_controls(const double* ctrl, const double* alpha, size_t nc) {
  for (size_t i = 0; i < nc; ++i)
    if (ctrl[3 * i + 2] != 0.0 || alpha[3 * i + 2] != 0.0) return false;
  return true;
}

double max_abs_host(const double* v, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(v[i]));
  return m;
}

extern "C" {

int im_deform(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
              const size_t* patch, size_t n_patch, const double* disp, const size_t* pinned,
              size_t n_pinned, const im_deform_config* cfg, double* deformed,
              im_deform_report* rep, size_t* level_points, double* level_achieved,
              int* level_cap_hit, double* level_support, size_t* level_touched,
              double* level_seconds) {
  return guarded(ctx, [&](Context& c) {
    const auto t_start = Clock::now();
    if (n_patch == 0) throw InvalidArgument("marker has no nodes");  // pipeline.cpp:26-28
    const im_greedy_config& g = cfg->greedy;
    for (size_t i = 0; i < n_patch; ++i)
      if (patch[i] >= n_nodes) throw InvalidArgument("patch node index out of range");
    for (size_t i = 0; i < n_pinned; ++i)
      if (pinned[i] >= n_nodes) throw InvalidArgument("pinned node index out of range");
    // surface system (pipeline.cpp:35-53)
    std::vector<size_t> surf(patch, patch + n_patch);
    std::unordered_set<size_t> used(surf.begin(), surf.end()), pin(pinned, pinned + n_pinned);
    for (size_t i = 0; i < n_pinned; ++i)
      if (used.insert(pinned[i]).second) surf.push_back(pinned[i]);
    const size_t ns = surf.size();
    std::vector<double> pos(3 * ns), tgt(3 * ns, 0.0);
    for (size_t i = 0; i < ns; ++i) {
      std::memcpy(&pos[3 * i], nodes + 3 * surf[i], 24);
      if (i < n_patch && !pin.count(surf[i])) std::memcpy(&tgt[3 * i], disp + 3 * i, 24);
    }
    // run_multilevel (greedy.cpp:172-195) on the device engine
    if (!(g.tolerance > 0.0 && g.tolerance < 1.0))
      throw InvalidArgument("greedy tolerance must lie in (0,1)");
    if (g.max_levels < 1) throw InvalidArgument("at least one level is required");
    if (g.max_points_per_level < 1) throw InvalidArgument("per-level point cap must be positive");
    if (!(g.basis.support_radius > 0.0)) throw InvalidArgument("basis support radius must be positive");
    for (double v : tgt)
      if (!std::isfinite(v)) throw InvalidArgument("target displacement is not finite");
    const double tmax = max_magnitude(tgt.data(), ns);
    const size_t m = std::min<size_t>(g.max_points_per_level, ns);
    const double threshold = std::pow(g.tolerance, (double)g.max_levels) * tmax;
    const auto t_greedy = Clock::now();
    GreedyEngine eng(c, (int)ns, (int)m);
    eng.set_positions(pos.data());
    eng.set_target(tgt.data());
    std::vector<double> current = tgt;
    struct Lvl {
      std::vector<size_t> idx;
      std::vector<double> alpha;
      double achieved, target_max, seconds;
      bool cap_hit;
    };
    std::vector<Lvl> levels;
    for (size_t l = 0; l < g.max_levels; ++l) {
      const double cur_max = max_magnitude(current.data(), ns);
      if (l > 0 && (cur_max == 0.0 || cur_max < threshold)) break;
      if (l > 0) eng.target_from_residual();
      const auto tl = Clock::now();
      eng.reset(g.tolerance, cur_max, g.basis.kind, g.basis.support_radius);
      const GState s = eng.run_level();
      Lvl lv;
      lv.idx.resize(s.nc);
      lv.alpha.resize(3 * (size_t)s.nc);
      if (s.status == kStatusSolveError) {
        eng.download(s.nc, lv.idx.data(), nullptr, nullptr, nullptr, nullptr, 0);
        throw_conditioning_nodes(pos.data(), lv.idx, (size_t)s.fail_node);
      }
      const size_t li = levels.size();
      const bool rec = cfg->record_error && cfg->record_stride >= (size_t)s.steps;
      eng.download(s.nc, lv.idx.data(), lv.alpha.data(), current.data(),
                   rec ? cfg->record_error + li * cfg->record_stride : nullptr,
                   rec && cfg->record_seconds ? cfg->record_seconds + li * cfg->record_stride
                                              : nullptr,
                   rec ? s.steps : 0);
      lv.achieved = s.achieved;
      lv.cap_hit = s.status == kStatusCapHit;
      lv.target_max = cur_max;
      lv.seconds = since(tl);
      levels.push_back(std::move(lv));
    }
    const double greedy_s = since(t_greedy);

    // support distances (pipeline.cpp:66 / the absolute-D extension)
    std::vector<double> Dl(levels.size());
    double cutoff = 0.0;
    for (size_t l = 0; l < levels.size(); ++l) {
      if (cfg->support_distance >= 0.0) {
        Dl[l] = cfg->support_distance;
      } else {
        if (!(cfg->volume_k > 0.0)) throw InvalidArgument("volume reduction factor must be positive");
        Dl[l] = cfg->volume_k * levels[l].target_max;
      }
      cutoff = std::max(cutoff, Dl[l]);
    }

    // mesh upload and wall distances on the undeformed mesh (pipeline.cpp:61)
    const auto t_dist = Clock::now();
    DPoints dn, acc, ds;
    upload_points(c, nodes, n_nodes, dn);
    acc.reserve(n_nodes);
    IMB_CHECK(cudaMemcpyAsync(acc.x.p, dn.x.p, n_nodes * 8, cudaMemcpyDeviceToDevice, c.stream));
    IMB_CHECK(cudaMemcpyAsync(acc.y.p, dn.y.p, n_nodes * 8, cudaMemcpyDeviceToDevice, c.stream));
    IMB_CHECK(cudaMemcpyAsync(acc.z.p, dn.z.p, n_nodes * 8, cudaMemcpyDeviceToDevice, c.stream));
    upload_points_indexed(c, nodes, patch, n_patch, ds);
    DBuf<double> dist;
    DBuf<unsigned long long> pidx, pinidx;  // separate buffers: patch ids / pinned ids
    DBuf<unsigned char> pinflag;
    const std::vector<unsigned long long> patch_ids(patch, patch + n_patch),
        pinned_ids(pinned, pinned + n_pinned);
    dist.reserve(n_nodes);
    pidx.reserve(std::max<size_t>(n_patch, 1));
    pinidx.reserve(std::max<size_t>(n_pinned, 1));
    pinflag.reserve(n_nodes);
    const bool any_volume = cutoff > 0.0;
    if (any_volume) {
      if (std::isinf(cutoff)) {
        // D = inf: every node is active and psi == 1 regardless of d
        // (xi = d / inf = 0), so the distances are not needed.
        IMB_CHECK(cudaMemsetAsync(dist.p, 0, n_nodes * 8, c.stream));
      } else {
        // stream-ordered copies (the context stream is non-blocking, so a
        // plain cudaMemcpy would not order against the kernels on it); the
        // host vectors stay alive until the synchronisation below
        wall_distance(c, dn, n_nodes, ds, n_patch, dim, cutoff, dist.p);
        IMB_CHECK(cudaMemcpyAsync(pidx.p, patch_ids.data(), n_patch * 8, cudaMemcpyHostToDevice,
                                  c.stream));
        k_zero_at<<<(n_patch + 255) / 256, 256, 0, c.stream>>>(dist.p, pidx.p, n_patch);
      }
    }
    IMB_CHECK(cudaMemsetAsync(pinflag.p, 0, n_nodes, c.stream));
    if (n_pinned) {
      IMB_CHECK(cudaMemcpyAsync(pinidx.p, pinned_ids.data(), n_pinned * 8, cudaMemcpyHostToDevice,
                                c.stream));
      k_set_flags<<<(n_pinned + 255) / 256, 256, 0, c.stream>>>(pinflag.p, pinidx.p, n_pinned);
    }
    IMB_CHECK(cudaStreamSynchronize(c.stream));
    const double dist_s = since(t_dist);

    // per-level volume update (pipeline.cpp:64-85)
    const auto t_vol = Clock::now();
    // the 2-D kernels write vz = 0 * psi: only when every node AND every
    // level's z weight is zero (the reference's DisplacementField is a Vec3,
    // so a planar mesh may still carry a z displacement)
    bool planar = dim == 2 && all_z_zero(nodes, n_nodes);
    for (size_t l = 0; planar && l < levels.size(); ++l)
      for (size_t i = 0; planar && i < levels[l].idx.size(); ++i)
        planar = levels[l].alpha[3 * i + 2] == 0.0;
    DBuf<uint32_t> active;
    active.reserve(n_nodes);
    DBuf<double> stage, tiles, boxes, midx, mbox;
    DBuf<uint32_t> perm;
    // exact mode: tiled kernel when the coordinate / R ranges allow it (the
    // controls are mesh nodes, so the node maximum covers them)
    const bool tiled_exact = cfg->precision == IM_EXACT &&
        exact_tiled_ok(g.basis.support_radius, max_abs_points(c, dn.x.p, dn.y.p, dn.z.p, n_nodes));
    Timer tm(c.stream);
    for (size_t l = 0; l < levels.size(); ++l) {
      const Lvl& lv = levels[l];
      size_t touched = 0;
      if (Dl[l] > 0.0) {  // wall_distance.cpp:54
        const size_t nc = lv.idx.size();
        std::vector<double> cp(3 * nc);
        for (size_t i = 0; i < nc; ++i) std::memcpy(&cp[3 * i], &pos[3 * lv.idx[i]], 24);
        stage.reserve(6 * std::max<size_t>(nc, 1));
        tiles.reserve(ctrl_tile_doubles(nc));
        if (nc) {
          IMB_CHECK(cudaMemcpyAsync(stage.p, cp.data(), nc * 24, cudaMemcpyHostToDevice, c.stream));
          IMB_CHECK(cudaMemcpyAsync(stage.p + 3 * nc, lv.alpha.data(), nc * 24,
                                    cudaMemcpyHostToDevice, c.stream));
        }
        const bool exact = cfg->precision == IM_EXACT;
        if (exact) {
          pack_controls_aos(c, stage.p, stage.p + 3 * nc, nc, 1.0, tiles.p);
          if (tiled_exact) {
            boxes.reserve(6 * (ctrl_padded(nc) / kCtrlTile));
            exact_tile_boxes(c, tiles.p, nc, 1.0 / g.basis.support_radius, boxes.p);
            midx.reserve(4 * ctrl_padded(nc));
            mbox.reserve(6 * (ctrl_padded(nc) / kCtrlTile));
            pack_exact_index_host(c, cp.data(), nc, 1.0 / g.basis.support_radius, midx.p, mbox.p);
          }
        } else {
          pack_controls_host(c, cp.data(), lv.alpha.data(), nc, 1.0 / g.basis.support_radius, true,
                             tiles, boxes);
        }
        touched = compact_active(c, dist.p, n_nodes, Dl[l], active.p);
        if (!exact || tiled_exact)
          spatial_order(c, dn.x.p, dn.y.p, dn.z.p, active.p, touched, g.basis.support_radius, perm);
        VolumeArgs a;
        a.x = dn.x.p, a.y = dn.y.p, a.z = dn.z.p;
        a.active = active.p;
        a.n_active = touched;
        a.dist = dist.p;
        a.D = Dl[l];
        a.psi_kind = cfg->psi_kind;
        a.tiles = tiles.p;
        a.tile_box = exact && !tiled_exact ? nullptr : boxes.p;
        a.perm = exact && !tiled_exact ? nullptr : perm.p;
        a.exact_tiled = tiled_exact;
        a.ctrl_index = tiled_exact ? midx.p : nullptr;
        a.index_box = tiled_exact ? mbox.p : nullptr;
        a.ctrl_diag = bbox_diagonal(cp.data(), nc);
        a.n_ctrl = nc;
        a.R = g.basis.support_radius;
        a.kind = g.basis.kind;
        a.dim = planar ? 2 : 3;
        a.precision = precision_of(cfg->precision);
        a.acc_x = acc.x.p, a.acc_y = acc.y.p, a.acc_z = acc.z.p;
        a.pinned = n_pinned ? pinflag.p : nullptr;
        launch_volume(c, a);
      }
      level_points[l] = lv.idx.size();
      level_achieved[l] = lv.achieved;
      level_cap_hit[l] = lv.cap_hit ? 1 : 0;
      level_support[l] = Dl[l];
      level_touched[l] = touched;
      if (level_seconds) level_seconds[l] = lv.seconds;
    }
    c.last_kernel_ms = tm.ms();
    // count_inverted(deformed) (pipeline.cpp:101) on the resident deformed nodes,
    // and the quality reports before / after (pipeline.cpp:55, 102)
    rep->inverted_elements = 0;
    rep->has_quality = 0;
    if (cfg->n_elements) {
      if (cfg->compute_quality) {
        auto to_rep = [](const QualityStats& q) {
          return im_quality_report{q.min_deg, q.mean_deg, q.inverted, q.degenerate};
        };
        rep->quality_before = to_rep(orthogonality_from_host(
            c, dn.x.p, dn.y.p, dn.z.p, n_nodes, cfg->element_kinds, cfg->element_offsets,
            cfg->element_nodes, cfg->n_elements, nullptr, nullptr));
        const QualityStats after = orthogonality_from_host(
            c, acc.x.p, acc.y.p, acc.z.p, n_nodes, cfg->element_kinds, cfg->element_offsets,
            cfg->element_nodes, cfg->n_elements, nullptr, nullptr);
        rep->quality_after = to_rep(after);
        rep->inverted_elements = after.inverted;
        rep->has_quality = 1;
      } else {
        rep->inverted_elements = signed_measures_from_host(
            c, acc.x.p, acc.y.p, acc.z.p, n_nodes, cfg->element_kinds, cfg->element_offsets,
            cfg->element_nodes, cfg->n_elements, nullptr);
      }
    }
    DBuf<double> aos;
    aos.reserve(3 * n_nodes);
    k_soa_to_aos<<<(n_nodes + 255) / 256, 256, 0, c.stream>>>(acc.x.p, acc.y.p, acc.z.p, n_nodes,
                                                               aos.p);
    const D2HJob down{aos.p, deformed, 3 * n_nodes, 8, false};
    staged_d2h(c, &down, 1);
    const double vol_s = since(t_vol);

    // surface accuracy (pipeline.cpp:87-99)
    double max_err = 0.0, sum_err = 0.0;
    for (size_t i = 0; i < n_patch; ++i) {
      const size_t nd = patch[i];
      const double mx = deformed[3 * nd] - nodes[3 * nd], my = deformed[3 * nd + 1] - nodes[3 * nd + 1],
                   mz = deformed[3 * nd + 2] - nodes[3 * nd + 2];
      const double err = hnorm(disp[3 * i] - mx, disp[3 * i + 1] - my, disp[3 * i + 2] - mz);
      max_err = std::max(max_err, err);
      sum_err += err;
    }
    rep->n_levels = levels.size();
    rep->target_max = tmax;
    rep->surface_max_error = 0.0;
    rep->surface_mean_error = 0.0;
    if (tmax > 0.0) {
      rep->surface_max_error = max_err / tmax;
      rep->surface_mean_error = sum_err / (tmax * (double)n_patch);
    }
    rep->greedy_seconds = greedy_s;
    rep->distance_seconds = dist_s;
    rep->volume_seconds = vol_s;
    rep->total_seconds = since(t_start);
  });
}

int im_volume_plan_create(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
                          const size_t* surface, size_t n_surface, double cutoff,
                          im_volume_plan** out) {
  *out = nullptr;
  auto* p = new im_volume_plan();
  p->ctx = ctx;
  const int rc = guarded(ctx, [&](Context& c) {
    p->n = n_nodes;
    p->dim = dim == 2 && all_z_zero(nodes, n_nodes) ? 2 : 3;
    upload_points(c, nodes, n_nodes, p->nodes);
    p->field.reserve(n_nodes);
    p->dist.reserve(n_nodes);
    p->active.reserve(n_nodes);
    DPoints& ds = p->surf;
    upload_points_indexed(c, nodes, surface, n_surface, ds);
    p->n_surface = n_surface;
    p->sdim = dim;
    Timer tm(c.stream);
    if (cutoff < 0.0) {  // D = inf workloads: distances unused (psi == 1)
      IMB_CHECK(cudaMemsetAsync(p->dist.p, 0, n_nodes * 8, c.stream));
    } else {
      wall_distance(c, p->nodes, n_nodes, ds, n_surface, dim, cutoff, p->dist.p);
      DBuf<unsigned long long> pidx;
      pidx.reserve(n_surface);
      std::vector<unsigned long long> pi(surface, surface + n_surface);
      sync_copy(c.stream, pidx.p, pi.data(), n_surface * 8, cudaMemcpyHostToDevice);
      k_zero_at<<<(n_surface + 255) / 256, 256, 0, c.stream>>>(p->dist.p, pidx.p, n_surface);
    }
    c.last_kernel_ms = tm.ms();
    for (double* f : {p->field.x.p, p->field.y.p, p->field.z.p})
      IMB_CHECK(cudaMemsetAsync(f, 0, n_nodes * 8, c.stream));
    IMB_CHECK(cudaStreamSynchronize(c.stream));
  });
  if (rc != IM_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return IM_OK;
}

int im_volume_plan_destroy(im_volume_plan* p) {
  delete p;
  return IM_OK;
}

int im_volume_plan_set_controls(im_volume_plan* p, const double* ctrl, const double* alpha,
                                size_t nc) {
  return guarded(p->ctx, [&](Context& c) {
    p->nc = nc;
    p->ctrl_stage.reserve(6 * std::max<size_t>(nc, 1));
    p->tiles.reserve(ctrl_tile_doubles(nc));
    if (nc) {
      sync_copy(c.stream, p->ctrl_stage.p, ctrl, nc * 24, cudaMemcpyHostToDevice);
      sync_copy(c.stream, p->ctrl_stage.p + 3 * nc, alpha, nc * 24, cudaMemcpyHostToDevice);
    }
    p->host_ctrl.assign(ctrl, ctrl + 3 * nc);
    p->host_alpha.assign(alpha, alpha + 3 * nc);
    (void)c;
  });
}

int im_volume_plan_run(im_volume_plan* p, const im_wall_function* wf, im_basis basis,
                       int precision, size_t* n_active, double* device_ms) {
  return guarded(p->ctx, [&](Context& c) {
    const double D = wf->support_distance;
    *n_active = 0;
    if (D <= 0.0) return;
    const bool exact = precision == IM_EXACT;
    const bool tiled_exact =
        exact && exact_tiled_ok(basis.support_radius,
                                std::max(max_abs_points(c, p->nodes.x.p, p->nodes.y.p,
                                                        p->nodes.z.p, p->n),
                                         max_abs_host(p->host_ctrl.data(), 3 * p->nc)));
    Timer tm(c.stream);
    DBuf<double> boxes, midx, mbox;
    if (exact) {
      pack_controls_aos(c, p->ctrl_stage.p, p->ctrl_stage.p + 3 * p->nc, p->nc, 1.0, p->tiles.p);
      if (tiled_exact) {
        boxes.reserve(6 * (ctrl_padded(p->nc) / kCtrlTile));
        exact_tile_boxes(c, p->tiles.p, p->nc, 1.0 / basis.support_radius, boxes.p);
        midx.reserve(4 * ctrl_padded(p->nc));
        mbox.reserve(6 * (ctrl_padded(p->nc) / kCtrlTile));
        pack_exact_index_host(c, p->host_ctrl.data(), p->nc, 1.0 / basis.support_radius, midx.p,
                              mbox.p);
      }
    } else {
      pack_controls_host(c, p->host_ctrl.data(), p->host_alpha.data(), p->nc,
                         1.0 / basis.support_radius, true, p->tiles, boxes);
    }
    const size_t na = compact_active(c, p->dist.p, p->n, D, p->active.p);
    VolumeArgs a;
    a.x = p->nodes.x.p, a.y = p->nodes.y.p, a.z = p->nodes.z.p;
    a.active = p->active.p;
    a.n_active = na;
    a.dist = p->dist.p;
    a.D = D;
    a.psi_kind = wf->psi_kind;
    a.tiles = p->tiles.p;
    a.n_ctrl = p->nc;
    a.R = basis.support_radius;
    a.kind = basis.kind;
    a.dim = p->dim == 2 && planar_controls(p->host_ctrl.data(), p->host_alpha.data(), p->nc) ? 2 : 3;
    a.precision = precision_of(precision);
    a.exact_tiled = tiled_exact;
    a.ctrl_index = tiled_exact ? midx.p : nullptr;
    a.index_box = tiled_exact ? mbox.p : nullptr;
    a.ctrl_diag = bbox_diagonal(p->host_ctrl.data(), p->nc);
    a.tile_box = exact && !tiled_exact ? nullptr : boxes.p;
    a.acc_x = p->field.x.p, a.acc_y = p->field.y.p, a.acc_z = p->field.z.p;
    launch_volume(c, a);
    const double ms = tm.ms();
    c.last_kernel_ms = ms;
    if (device_ms) *device_ms = ms;
    *n_active = na;
  });
}

int im_volume_plan_reset_field(im_volume_plan* p) {
  return guarded(p->ctx, [&](Context& c) {
    for (double* f : {p->field.x.p, p->field.y.p, p->field.z.p})
      IMB_CHECK(cudaMemsetAsync(f, 0, p->n * 8, c.stream));
    IMB_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int im_volume_plan_download_field(im_volume_plan* p, double* out) {
  return guarded(p->ctx, [&](Context& c) {
    DBuf<double> aos;
    aos.reserve(3 * p->n);
    if (p->reordered)
      k_scatter_aos<<<(p->n + 255) / 256, 256, 0, c.stream>>>(p->field.x.p, p->field.y.p,
                                                              p->field.z.p, p->order.p, p->n, aos.p);
    else
      k_soa_to_aos<<<(p->n + 255) / 256, 256, 0, c.stream>>>(p->field.x.p, p->field.y.p,
                                                              p->field.z.p, p->n, aos.p);
    IMB_CHECK(cudaMemcpyAsync(out, aos.p, p->n * 24, cudaMemcpyDeviceToHost, c.stream));
    IMB_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int im_volume_plan_distances(im_volume_plan* p, double* out) {
  return guarded(p->ctx, [&](Context& c) {
    if (p->reordered) {
      DBuf<double> tmp;
      tmp.reserve(p->n);
      k_scatter1<<<(p->n + 255) / 256, 256, 0, c.stream>>>(p->dist.p, p->order.p, p->n, tmp.p);
      IMB_CHECK(cudaMemcpyAsync(out, tmp.p, p->n * 8, cudaMemcpyDeviceToHost, c.stream));
      IMB_CHECK(cudaStreamSynchronize(c.stream));
      return;
    }
    IMB_CHECK(cudaMemcpyAsync(out, p->dist.p, p->n * 8, cudaMemcpyDeviceToHost, c.stream));
    IMB_CHECK(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"

extern "C" {

int im_volume_plan_set_level(im_volume_plan* p, int level, const double* ctrl, const double* alpha,
                             size_t nc, double D, int psi_kind, im_basis basis, int precision) {
  return guarded(p->ctx, [&](Context& c) {
    if (level < 0 || level >= 8) throw InvalidArgument("level index out of range (0..7)");
    precision_of(precision);
    const bool tiled_exact =
        precision == IM_EXACT &&
        exact_tiled_ok(basis.support_radius,
                       std::max(max_abs_points(c, p->nodes.x.p, p->nodes.y.p, p->nodes.z.p, p->n),
                                max_abs_host(ctrl, 3 * nc)));
    if (!p->reordered && (precision != IM_EXACT || tiled_exact) && p->n) {
      // one-time spatial layout of the resident mesh (grid cells of ~2R)
      spatial_order(c, p->nodes.x.p, p->nodes.y.p, p->nodes.z.p, nullptr, p->n,
                    basis.support_radius, p->order);
      DBuf<double> tmp;
      tmp.reserve(p->n);
      const unsigned nb = (unsigned)((p->n + 255) / 256);
      for (DBuf<double>* a : {&p->nodes.x, &p->nodes.y, &p->nodes.z, &p->dist}) {
        k_gather<<<nb, 256, 0, c.stream>>>(a->p, p->order.p, p->n, tmp.p);
        IMB_CHECK(cudaMemcpyAsync(a->p, tmp.p, p->n * 8, cudaMemcpyDeviceToDevice, c.stream));
      }
      IMB_CHECK(cudaStreamSynchronize(c.stream));
      p->reordered = true;
    }
    auto& L = p->levels[level];
    L.nc = nc;
    L.planar = p->dim == 2 && planar_controls(ctrl, alpha, nc);
    L.D = D;
    L.psi_kind = psi_kind;
    if (precision == IM_EXACT) {
      L.tiles.reserve(ctrl_tile_doubles(nc));
      DBuf<double> stage;
      stage.reserve(6 * std::max<size_t>(nc, 1));
      if (nc) {
        sync_copy(c.stream, stage.p, ctrl, nc * 24, cudaMemcpyHostToDevice);
        sync_copy(c.stream, stage.p + 3 * nc, alpha, nc * 24, cudaMemcpyHostToDevice);
      }
      pack_controls_aos(c, stage.p, stage.p + 3 * nc, nc, 1.0, L.tiles.p);
      L.culled = tiled_exact;
      if (tiled_exact) {
        L.boxes.reserve(6 * (ctrl_padded(nc) / kCtrlTile));
        exact_tile_boxes(c, L.tiles.p, nc, 1.0 / basis.support_radius, L.boxes.p);
        L.midx.reserve(4 * ctrl_padded(nc));
        L.mbox.reserve(6 * (ctrl_padded(nc) / kCtrlTile));
        pack_exact_index_host(c, ctrl, nc, 1.0 / basis.support_radius, L.midx.p, L.mbox.p);
      }
    } else {
      pack_controls_host(c, ctrl, alpha, nc, 1.0 / basis.support_radius, true, L.tiles, L.boxes);
      L.culled = true;
    }
    L.exact_tiled = tiled_exact;
    L.exact_format = precision == IM_EXACT;
    L.diag = bbox_diagonal(ctrl, nc);
    L.order_n = 0;  // block order recomputed at the next run
    L.host_ctrl.assign(ctrl, ctrl + 3 * nc);
    L.host_alpha.assign(alpha, alpha + 3 * nc);
    IMB_CHECK(cudaStreamSynchronize(c.stream));
    p->n_levels = std::max(p->n_levels, level + 1);
  });
}

// Runs `steps` volume-update steps (every level: compaction of d < D_l, then
// the update accumulated into the resident field).  Each step is bracketed
// by CUDA events on the context stream; with flush_l2 a 256 MiB write evicts
// L2 before each step, outside the timed brackets.  stats (10 doubles):
//   [0] sum of step times (ms)   [1] sum of volume-kernel times (ms)
//   [2] volume-kernel launches    [3] kernels launched per step
//   [4..7] active count of levels 0..3 in the last step
int im_volume_plan_run_steps(im_volume_plan* p, im_basis basis, int precision, int steps,
                             int flush_l2, double* stats) {
  return guarded(p->ctx, [&](Context& c) {
    const Precision prec = precision_of(precision);
    for (int l = 0; l < p->n_levels; ++l)
      if (p->levels[l].D > 0.0 && p->levels[l].exact_format != (prec == Precision::Exact))
        throw InvalidArgument("plan level was set for a different precision (set_level)");
    const size_t flush_bytes = size_t(256) << 20;
    if (flush_l2) p->flush.reserve(flush_bytes);
    cudaEvent_t e0, e1, k0, k1;
    IMB_CHECK(cudaEventCreate(&e0));
    IMB_CHECK(cudaEventCreate(&e1));
    IMB_CHECK(cudaEventCreate(&k0));
    IMB_CHECK(cudaEventCreate(&k1));
    double total = 0.0, kern = 0.0, launches = 0.0, per_step = 0.0;
    for (int s = 0; s < steps; ++s) {
      if (flush_l2) IMB_CHECK(cudaMemsetAsync(p->flush.p, s & 0xff, flush_bytes, c.stream));
      IMB_CHECK(cudaEventRecord(e0, c.stream));
      per_step = 0.0;
      double last_D = NAN;
      size_t last_na = 0;
      for (int l = 0; l < p->n_levels; ++l) {
        auto& L = p->levels[l];
        if (L.D <= 0.0) continue;
        // compaction + spatial order, shared by consecutive levels with the same D
        size_t na = last_na;
        if (!(L.D == last_D)) {
          na = compact_active(c, p->dist.p, p->n, L.D, p->active.p);
          per_step += 1;  // k_compact_active
          last_D = L.D, last_na = na;
        }
        if (l < 4) stats[4 + l] = (double)na;
        VolumeArgs a;
        a.x = p->nodes.x.p, a.y = p->nodes.y.p, a.z = p->nodes.z.p;
        a.active = p->active.p;
        a.n_active = na;
        a.dist = p->dist.p;
        a.D = L.D;
        a.psi_kind = L.psi_kind;
        a.tiles = L.tiles.p;
        a.tile_box = L.culled ? L.boxes.p : nullptr;
        a.n_ctrl = L.nc;
        a.R = basis.support_radius;
        a.kind = basis.kind;
        a.dim = L.planar ? 2 : 3;
        a.precision = prec;
        a.exact_tiled = L.exact_tiled;
        a.ctrl_index = L.exact_tiled ? L.midx.p : nullptr;
        a.index_box = L.exact_tiled ? L.mbox.p : nullptr;
        a.ctrl_diag = L.diag;
        if (exact_uses_block_order(a)) {
          // the active set of a level is the same every step (stable compaction)
          if (L.order_n != na) {
            L.order.reserve(na / kExactBlock + 1);
            block_order(c, a.x, a.y, a.z, a.active, nullptr, na, kExactBlock, L.tiles.p, L.nc,
                        basis.support_radius, false, L.order.p);
            L.order_n = na;
          }
          a.cta_order = L.order.p;
        }
        a.acc_x = p->field.x.p, a.acc_y = p->field.y.p, a.acc_z = p->field.z.p;
        IMB_CHECK(cudaEventRecord(k0, c.stream));
        launch_volume(c, a);
        IMB_CHECK(cudaEventRecord(k1, c.stream));
        IMB_CHECK(cudaEventSynchronize(k1));
        float km = 0.f;
        IMB_CHECK(cudaEventElapsedTime(&km, k0, k1));
        kern += km;
        launches += na ? 1 : 0;
        per_step += na ? 1 : 0;
      }
      IMB_CHECK(cudaEventRecord(e1, c.stream));
      IMB_CHECK(cudaEventSynchronize(e1));
      float ms = 0.f;
      IMB_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(k0);
    cudaEventDestroy(k1);
    stats[0] = total;
    stats[1] = kern;
    stats[2] = launches;
    stats[3] = per_step;
  });
}

// The HBM-bound passes on the plan's resident mesh, for the bench's
// roofline: the wall distance (K6, wall_distance.cpp:13-31) of every node
// with the given cutoff (into scratch, the plan's distances are kept), and
// the stable compaction of d < D (K7, wall_distance.cpp:56-58), each timed
// with CUDA events over `reps` passes.  stats: [0] wall-distance ms per pass,
// [1] compaction ms per pass, [2] active count, [3] nodes with d <= cutoff.
int im_volume_plan_bench_passes(im_volume_plan* p, double cutoff, double D, int reps,
                                double* stats) {
  return guarded(p->ctx, [&](Context& c) {
    DBuf<double> d;
    d.reserve(std::max<size_t>(p->n, 1));
    DBuf<uint32_t> act;
    act.reserve(std::max<size_t>(p->n, 1));
    reps = std::max(reps, 1);
    // warm-up (grid scratch, lazy loading)
    wall_distance(c, p->nodes, p->n, p->surf, p->n_surface, p->sdim, cutoff, d.p);
    Timer tw(c.stream);
    for (int r = 0; r < reps; ++r)
      wall_distance(c, p->nodes, p->n, p->surf, p->n_surface, p->sdim, cutoff, d.p);
    stats[0] = tw.ms() / reps;
    size_t na = compact_active(c, p->dist.p, p->n, D, act.p);
    Timer tc(c.stream);
    for (int r = 0; r < reps; ++r) na = compact_active(c, p->dist.p, p->n, D, act.p);
    stats[1] = tc.ms() / reps;
    stats[2] = (double)na;
    stats[3] = (double)compact_active(c, d.p, p->n, std::nextafter(cutoff, INFINITY), act.p);
  });
}

// Exact count of in-support pairs (eta < 1, the reference's phi != 0 test
// up to rounding at eta == 1) of one plan level over its active set, for the
// algorithmic-flop roofline (22 flops in support, 10 out, 3-D; 17 / 7 in 2-D).
int im_volume_plan_count_support(im_volume_plan* p, int level, im_basis basis,
                                 unsigned long long* in_support, unsigned long long* total) {
  return guarded(p->ctx, [&](Context& c) {
    const auto& L = p->levels[level];
    const size_t na = compact_active(c, p->dist.p, p->n, L.D, p->active.p);
    *total = (unsigned long long)na * L.nc;
    // counted on fast-format tiles whatever the level's precision
    DBuf<double> tiles, boxes;
    pack_controls_host(c, L.host_ctrl.data(), L.host_alpha.data(), L.nc,
                       1.0 / basis.support_radius, true, tiles, boxes);
    *in_support = count_support_pairs(c, p->nodes, p->active.p, na, tiles.p, L.nc,
                                      1.0 / basis.support_radius);
  });
}

}  // extern "C"
