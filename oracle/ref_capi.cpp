// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" driver over the UNMODIFIED reference library, compiled
// from the sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libicemorph_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.
//
// Every entry point calls the reference's own public API (proj/include):
//   ref_eval_wendland        -> eval_wendland            (rbf.cpp:28-50)
//   ref_solve_weights        -> solve_weights            (rbf.cpp:144-193)
//   ref_eval_interpolant     -> eval_interpolant         (rbf.cpp:195-203)
//   ref_greedy_level         -> greedy_level             (greedy.cpp:60-170)
//   ref_run_multilevel       -> run_multilevel           (greedy.cpp:172-195)
//   ref_build_distance_index -> build_distance_index     (wall_distance.cpp:13-31)
//   ref_update_volume        -> update_volume            (wall_distance.cpp:46-64)
//   ref_deform               -> deform                   (pipeline.cpp:19-106)
//   ref_deform_elements      -> deform with volume elements (report.inverted_elements)
//   ref_signed_measures      -> signed_measures / count_inverted (quality.cpp:135-148)
//   ref_assemble_surface_matrix -> assemble_surface_matrix (rbf.cpp:56-69)
//   ref_cholesky_*           -> CholeskyFactor            (rbf.cpp:71-121)
//
// The psi = Wendland-C2 taper (BASELINE cfg1 "psi = Wendland C2 of xi") has
// no reference implementation; for psi_kind == 1 ref_update_volume restates
// wall_distance.cpp:54-61 with eval_wendland(C2, xi) (rbf.cpp:34-37) in place
// of the linear eval_wall_function (wall_distance.cpp:40-44), still calling
// the reference eval_interpolant for the kernel sum.
//
// Status codes: 0 ok, 1 std::invalid_argument, 2 SolveError, 3 other.
// No iostreams are used here (ostream << double crashes the
// reference module once numpy is loaded in-process).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "icemorph/greedy.hpp"
#include "icemorph/mesh_io.hpp"
#include "icemorph/pipeline.hpp"
#include "icemorph/quality.hpp"
#include "icemorph/rbf.hpp"
#include "icemorph/wall_distance.hpp"

using namespace icemorph;

namespace {

thread_local char g_err[1024];
thread_local size_t g_err_line = 0;

int fail(int code, const char* what) {
  std::snprintf(g_err, sizeof g_err, "%s", what);
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err[0] = 0;
    return 0;
  } catch (const SolveError& e) {
    return fail(2, e.what());
  } catch (const ParseError& e) {
    g_err_line = e.line();
    return fail(4, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(1, e.what());
  } catch (const std::exception& e) {
    return fail(3, e.what());
  }
}

std::vector<Vec3> to_vecs(const double* xyz, size_t n) {
  std::vector<Vec3> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return v;
}

void put(double* out, const Vec3& v) {
  out[0] = v.x;
  out[1] = v.y;
  out[2] = v.z;
}

WendlandKind kind_of(int k) {
  switch (k) {
    case 0: return WendlandKind::C0;
    case 1: return WendlandKind::C2;
    case 2: return WendlandKind::C4;
    case 3: return WendlandKind::C6;
  }
  throw std::invalid_argument("unknown basis kind");
}

GreedyConfig greedy_config(double tol, size_t max_levels, size_t cap, int kind, double R) {
  GreedyConfig c;
  c.tolerance = tol;
  c.max_levels = max_levels;
  c.max_points_per_level = cap;
  c.basis = {kind_of(kind), R};
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err; }
size_t ref_last_error_line(void) { return g_err_line; }

double ref_eval_wendland(int kind, double eta) { return eval_wendland(kind_of(kind), eta); }

int ref_solve_weights(const double* pts, const double* disp, size_t n, int kind,
                      double R, double* alpha_out) {
  return guarded([&] {
    const auto p = to_vecs(pts, n);
    const auto d = to_vecs(disp, n);
    const WeightSet w = solve_weights(p, d, {kind_of(kind), R});
    for (size_t i = 0; i < n; ++i) put(alpha_out + 3 * i, w.alpha[i]);
  });
}

int ref_eval_interpolant(const double* ctrl, const double* alpha, size_t nc, int kind,
                         double R, const double* q, size_t nq, double* out) {
  return guarded([&] {
    WeightSet w;
    w.control_positions = to_vecs(ctrl, nc);
    w.alpha = to_vecs(alpha, nc);
    const BasisFunction b{kind_of(kind), R};
    for (size_t i = 0; i < nq; ++i) {
      put(out + 3 * i, eval_interpolant(w, b, {q[3 * i], q[3 * i + 1], q[3 * i + 2]}));
    }
  });
}

// Outputs sized by the caller: indices/alpha/record arrays hold min(cap, n).
int ref_greedy_level(const double* pos, const double* target, size_t n, double tol,
                     size_t cap, int kind, double R, size_t level_index,
                     size_t* out_idx, double* out_alpha, size_t* out_nc,
                     double* out_achieved, int* out_cap_hit, double* out_target_max,
                     double* out_elapsed, size_t* out_rec_points, double* out_rec_error,
                     double* out_rec_seconds, size_t* out_nrec, double* out_residual) {
  return guarded([&] {
    const auto p = to_vecs(pos, n);
    const auto t = to_vecs(target, n);
    const LevelResult r = greedy_level(p, t, greedy_config(tol, 1, cap, kind, R), level_index);
    const size_t nc = r.level.control_indices.size();
    *out_nc = nc;
    for (size_t i = 0; i < nc; ++i) {
      out_idx[i] = r.level.control_indices[i];
      put(out_alpha + 3 * i, r.level.weights.alpha[i]);
    }
    *out_achieved = r.level.achieved_error;
    *out_cap_hit = r.level.cap_hit ? 1 : 0;
    *out_target_max = r.level.target_max;
    *out_elapsed = r.level.elapsed_seconds;
    *out_nrec = r.record.samples.size();
    for (size_t i = 0; i < r.record.samples.size(); ++i) {
      out_rec_points[i] = r.record.samples[i].points;
      out_rec_error[i] = r.record.samples[i].error;
      if (out_rec_seconds) out_rec_seconds[i] = r.record.samples[i].seconds;
    }
    if (out_residual)
      for (size_t i = 0; i < n; ++i) put(out_residual + 3 * i, r.residual[i]);
  });
}

// Flattened multilevel result. Per-level arrays have max_levels slots; the
// index/alpha/record arrays have max_levels * min(cap, n) slots, level l at
// offset l * min(cap, n).
int ref_run_multilevel(const double* pos, const double* target, size_t n, double tol,
                       size_t max_levels, size_t cap, int kind, double R,
                       size_t* out_nlevels, size_t* out_nc, size_t* out_idx,
                       double* out_alpha, double* out_achieved, int* out_cap_hit,
                       double* out_level_target_max, double* out_elapsed,
                       size_t* out_nrec, double* out_rec_error, double* out_target_max,
                       double* out_final_residual) {
  return guarded([&] {
    const auto p = to_vecs(pos, n);
    const auto t = to_vecs(target, n);
    const MultilevelResult r = run_multilevel(p, t, greedy_config(tol, max_levels, cap, kind, R));
    const size_t stride = std::min(cap, n);
    *out_nlevels = r.levels.size();
    for (size_t l = 0; l < r.levels.size(); ++l) {
      const RbfLevel& lv = r.levels[l];
      out_nc[l] = lv.control_indices.size();
      for (size_t i = 0; i < lv.control_indices.size(); ++i) {
        out_idx[l * stride + i] = lv.control_indices[i];
        put(out_alpha + 3 * (l * stride + i), lv.weights.alpha[i]);
      }
      out_achieved[l] = lv.achieved_error;
      out_cap_hit[l] = lv.cap_hit ? 1 : 0;
      out_level_target_max[l] = lv.target_max;
      if (out_elapsed) out_elapsed[l] = lv.elapsed_seconds;
      out_nrec[l] = r.records[l].samples.size();
      if (out_rec_error)
        for (size_t i = 0; i < r.records[l].samples.size(); ++i)
          out_rec_error[l * stride + i] = r.records[l].samples[i].error;
    }
    *out_target_max = r.target_max;
    if (out_final_residual)
      for (size_t i = 0; i < n; ++i) put(out_final_residual + 3 * i, r.final_residual[i]);
  });
}

int ref_build_distance_index(const double* nodes, size_t n_nodes, int dim,
                             const size_t* surface, size_t n_surface, double* out_dist) {
  return guarded([&] {
    Mesh mesh;
    mesh.dim = dim;
    mesh.nodes = to_vecs(nodes, n_nodes);
    const std::vector<size_t> s(surface, surface + n_surface);
    const DistanceIndex idx = build_distance_index(mesh, s);
    std::memcpy(out_dist, idx.distances.data(), n_nodes * sizeof(double));
  });
}

// psi_kind 0 = reference linear taper (update_volume itself), 1 = Wendland C2
// taper (restatement, see header).  nthreads > 1 splits the node range into
// contiguous slices, each processed by the reference code on its own thread;
// the entries are concatenated in slice order, so the output is identical to
// the single-threaded call.  out_idx / out_val must hold n_nodes entries.
int ref_update_volume(const double* nodes, size_t n_nodes, const double* dist,
                      const double* ctrl, const double* alpha, size_t nc, double D,
                      int psi_kind, int kind, double R, size_t* out_idx,
                      double* out_val, size_t* out_n, int nthreads) {
  return guarded([&] {
    const BasisFunction basis{kind_of(kind), R};
    RbfLevel level;
    level.weights.control_positions = to_vecs(ctrl, nc);
    level.weights.alpha = to_vecs(alpha, nc);
    const WallFunction wf{1.0, D};
    if (nthreads < 1) nthreads = 1;
    std::vector<std::vector<std::pair<size_t, Vec3>>> parts(nthreads);
    std::vector<std::exception_ptr> errs(nthreads);
    auto work = [&](int t) {
      try {
        const size_t lo = n_nodes * t / nthreads, hi = n_nodes * (t + 1) / nthreads;
        Mesh mesh;
        mesh.nodes = to_vecs(nodes + 3 * lo, hi - lo);
        DistanceIndex idx;
        idx.distances.assign(dist + lo, dist + hi);
        if (psi_kind == 0) {
          VolumeUpdate u = update_volume(mesh, level, idx, wf, basis);
          for (auto& e : u.entries) e.first += lo;
          parts[t] = std::move(u.entries);
        } else {
          if (wf.support_distance <= 0.0) return;
          for (size_t i = 0; i < mesh.nodes.size(); ++i) {
            const double d = idx.distances[i];
            if (d >= wf.support_distance) continue;
            const double psi = eval_wendland(WendlandKind::C2, d / wf.support_distance);
            Vec3 value = eval_interpolant(level.weights, basis, mesh.nodes[i]);
            parts[t].emplace_back(lo + i, value * psi);
          }
        }
      } catch (...) {
        errs[t] = std::current_exception();
      }
    };
    if (nthreads == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < nthreads; ++t) th.emplace_back(work, t);
      for (auto& x : th) x.join();
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    size_t k = 0;
    for (auto& p : parts)
      for (auto& e : p) {
        out_idx[k] = e.first;
        put(out_val + 3 * k, e.second);
        ++k;
      }
    *out_n = k;
  });
}

// deform() on a mesh given as node array + marker node lists (+ optional
// volume elements for report.inverted_elements; compute_quality is false).  marker 0 is the
// deforming patch; markers 1.. are pinned.  disp holds one displacement per
// node of marker 0 (same order).  Outputs: deformed node array, per-level
// (points, touched, support_distance, achieved, cap_hit), surface errors.
static int deform_impl(const double* nodes, size_t n_nodes, int dim, const size_t* patch,
                       size_t n_patch, const double* disp, const size_t* pinned, size_t n_pinned,
                       double tol, size_t max_levels, size_t cap, int kind, double R,
                       double volume_k, double* out_nodes, size_t* out_nlevels, size_t* out_points,
                       size_t* out_touched, double* out_support, double* out_achieved,
                       int* out_cap_hit, double* out_target_max, double* out_surface_max,
                       double* out_surface_mean, double* out_total_seconds, const int* kinds,
                       const size_t* offsets, const size_t* conn, size_t n_elem,
                       size_t* out_inverted) {
  return guarded([&] {
    Mesh mesh;
    mesh.dim = dim;
    mesh.nodes = to_vecs(nodes, n_nodes);
    mesh.elements.resize(n_elem);
    for (size_t e = 0; e < n_elem; ++e) {
      mesh.elements[e].kind = static_cast<ElementKind>(kinds[e]);
      mesh.elements[e].nodes.assign(conn + offsets[e], conn + offsets[e + 1]);
    }
    Marker m;
    m.name = "patch";
    m.nodes.assign(patch, patch + n_patch);
    mesh.markers.push_back(m);
    DeformationConfig cfg;
    cfg.greedy = greedy_config(tol, max_levels, cap, kind, R);
    cfg.volume_k = volume_k;
    cfg.compute_quality = false;
    if (n_pinned) {
      Marker pm;
      pm.name = "pinned";
      pm.nodes.assign(pinned, pinned + n_pinned);
      mesh.markers.push_back(pm);
      cfg.fixed_markers = {"pinned"};
    }
    DisplacementField f;
    f.patch = "patch";
    for (size_t i = 0; i < n_patch; ++i)
      f.entries[patch[i]] = Vec3{disp[3 * i], disp[3 * i + 1], disp[3 * i + 2]};
    auto [out, rep] = deform(mesh, f, cfg);
    for (size_t i = 0; i < n_nodes; ++i) put(out_nodes + 3 * i, out.nodes[i]);
    *out_nlevels = rep.levels.size();
    for (size_t l = 0; l < rep.levels.size(); ++l) {
      out_points[l] = rep.levels[l].points;
      out_touched[l] = rep.levels[l].touched_nodes;
      out_support[l] = rep.levels[l].support_distance;
      out_achieved[l] = rep.levels[l].achieved_error;
      out_cap_hit[l] = rep.levels[l].cap_hit ? 1 : 0;
    }
    *out_target_max = rep.target_max;
    *out_surface_max = rep.surface_max_error;
    *out_surface_mean = rep.surface_mean_error;
    *out_total_seconds = rep.total_seconds;
    if (out_inverted) *out_inverted = rep.inverted_elements;  // pipeline.cpp:101
  });
}

int ref_deform(const double* nodes, size_t n_nodes, int dim, const size_t* patch,
               size_t n_patch, const double* disp, const size_t* pinned, size_t n_pinned,
               double tol, size_t max_levels, size_t cap, int kind, double R, double volume_k,
               double* out_nodes, size_t* out_nlevels, size_t* out_points,
               size_t* out_touched, double* out_support, double* out_achieved,
               int* out_cap_hit, double* out_target_max, double* out_surface_max,
               double* out_surface_mean, double* out_total_seconds) {
  return deform_impl(nodes, n_nodes, dim, patch, n_patch, disp, pinned, n_pinned, tol, max_levels,
                     cap, kind, R, volume_k, out_nodes, out_nlevels, out_points, out_touched,
                     out_support, out_achieved, out_cap_hit, out_target_max, out_surface_max,
                     out_surface_mean, out_total_seconds, nullptr, nullptr, nullptr, 0, nullptr);
}

// deform on a mesh that carries its volume elements; *out_inverted receives
// report.inverted_elements = count_inverted(deformed) (pipeline.cpp:101).
int ref_deform_elements(const double* nodes, size_t n_nodes, int dim, const size_t* patch,
                        size_t n_patch, const double* disp, const size_t* pinned,
                        size_t n_pinned, double tol, size_t max_levels, size_t cap, int kind,
                        double R, double volume_k, double* out_nodes, size_t* out_nlevels,
                        size_t* out_points, size_t* out_touched, double* out_support,
                        double* out_achieved, int* out_cap_hit, double* out_target_max,
                        double* out_surface_max, double* out_surface_mean,
                        double* out_total_seconds, const int* kinds, const size_t* offsets,
                        const size_t* conn, size_t n_elem, size_t* out_inverted) {
  return deform_impl(nodes, n_nodes, dim, patch, n_patch, disp, pinned, n_pinned, tol, max_levels,
                     cap, kind, R, volume_k, out_nodes, out_nlevels, out_points, out_touched,
                     out_support, out_achieved, out_cap_hit, out_target_max, out_surface_max,
                     out_surface_mean, out_total_seconds, kinds, offsets, conn, n_elem,
                     out_inverted);
}

}  // extern "C"

// ---- quality: signed_measures / count_inverted ------
// Element kinds follow mesh.hpp:15-23 (0 Line, 1 Triangle, 2 Quadrilateral,
// 3 Tetrahedron, 4 Hexahedron, 5 Prism, 6 Pyramid); CSR connectivity.
namespace {
Mesh mesh_with_elements(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                        const size_t* offsets, const size_t* conn, size_t n_elem) {
  Mesh m;
  m.dim = dim;
  m.nodes = to_vecs(nodes, n_nodes);
  m.elements.resize(n_elem);
  for (size_t e = 0; e < n_elem; ++e) {
    m.elements[e].kind = static_cast<ElementKind>(kinds[e]);
    m.elements[e].nodes.assign(conn + offsets[e], conn + offsets[e + 1]);
  }
  return m;
}
}  // namespace

extern "C" int ref_signed_measures(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                                   const size_t* offsets, const size_t* conn, size_t n_elem,
                                   double* out, size_t* inverted) {
  return guarded([&] {
    const Mesh m = mesh_with_elements(nodes, n_nodes, dim, kinds, offsets, conn, n_elem);
    const std::vector<double> v = signed_measures(m);  // quality.cpp:135-140
    std::memcpy(out, v.data(), n_elem * sizeof(double));
    *inverted = count_inverted(m);  // quality.cpp:142-148
  });
}

// orthogonality (quality.cpp:150-236): per-element scores and measures, and
// the report scalars {min, mean, inverted_count, degenerate_count}.
extern "C" int ref_orthogonality(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                                 const size_t* offsets, const size_t* conn, size_t n_elem,
                                 double* out_scores, double* out_measures, double* out_min,
                                 double* out_mean, size_t* out_inverted, size_t* out_degenerate) {
  return guarded([&] {
    const Mesh m = mesh_with_elements(nodes, n_nodes, dim, kinds, offsets, conn, n_elem);
    const QualityReport q = orthogonality(m);
    if (n_elem) {
      std::memcpy(out_scores, q.element_orthogonality_deg.data(), n_elem * sizeof(double));
      std::memcpy(out_measures, q.element_signed_measure.data(), n_elem * sizeof(double));
    }
    *out_min = q.min_orthogonality_deg;
    *out_mean = q.mean_orthogonality_deg;
    *out_inverted = q.inverted_count;
    *out_degenerate = q.degenerate_count;
  });
}

// read_su2 (mesh_io.cpp:127-259).  sizes[0..5] = dim, nodes, elements, element
// nodes, markers, marker-name bytes (names joined by '\n'), then per-marker
// arrays: me[m] elements, mc[m] element nodes, mn[m] nodes (caller allocates
// after a call with xyz == nullptr).
extern "C" int ref_read_su2(const char* path, size_t* sizes, double* xyz, int* kinds,
                            size_t* offsets, size_t* conn, char* names, size_t* me, size_t* mc,
                            size_t* mn, int* mkinds, size_t* moffsets, size_t* mconn,
                            size_t* mnodes) {
  return guarded([&] {
    const Mesh m = read_su2(std::string(path));
    size_t nconn = 0, nbytes = 0;
    for (const auto& e : m.elements) nconn += e.nodes.size();
    for (const auto& k : m.markers) nbytes += k.name.size() + 1;
    sizes[0] = (size_t)m.dim, sizes[1] = m.nodes.size(), sizes[2] = m.elements.size();
    sizes[3] = nconn, sizes[4] = m.markers.size(), sizes[5] = nbytes;
    for (size_t i = 0; i < m.markers.size(); ++i) {
      size_t c = 0;
      for (const auto& e : m.markers[i].elements) c += e.nodes.size();
      me[i] = m.markers[i].elements.size(), mc[i] = c, mn[i] = m.markers[i].nodes.size();
    }
    if (!xyz) return;
    for (size_t i = 0; i < m.nodes.size(); ++i) put(xyz + 3 * i, m.nodes[i]);
    offsets[0] = 0;
    for (size_t e = 0; e < m.elements.size(); ++e) {
      kinds[e] = static_cast<int>(m.elements[e].kind);
      for (size_t k = 0; k < m.elements[e].nodes.size(); ++k) conn[offsets[e] + k] = m.elements[e].nodes[k];
      offsets[e + 1] = offsets[e] + m.elements[e].nodes.size();
    }
    size_t pn = 0, pe = 0, pc = 0, pnod = 0;
    for (const auto& k : m.markers) {
      std::memcpy(names + pn, k.name.data(), k.name.size());
      names[pn + k.name.size()] = '\n';
      pn += k.name.size() + 1;
      for (const auto& e : k.elements) {
        mkinds[pe] = static_cast<int>(e.kind);
        moffsets[pe] = e.nodes.size();
        for (size_t v : e.nodes) mconn[pc++] = v;
        ++pe;
      }
      for (size_t v : k.nodes) mnodes[pnod++] = v;
    }
  });
}

// ---- rbf.hpp:35-60: the dense matrix and the incremental factor ------------
extern "C" int ref_assemble_surface_matrix(const double* pts, size_t n, int kind, double R,
                                           double* out) {
  return guarded([&] {
    BasisFunction b{kind_of(kind), R};
    const std::vector<double> m = assemble_surface_matrix(to_vecs(pts, n), b);
    std::copy(m.begin(), m.end(), out);
  });
}

extern "C" void* ref_cholesky_create(void) { return new CholeskyFactor(); }
extern "C" void ref_cholesky_destroy(void* f) { delete static_cast<CholeskyFactor*>(f); }
extern "C" size_t ref_cholesky_size(void* f) { return static_cast<CholeskyFactor*>(f)->size(); }
extern "C" double ref_cholesky_smallest_pivot(void* f) {
  return static_cast<CholeskyFactor*>(f)->smallest_pivot();
}
extern "C" int ref_cholesky_append(void* f, const double* col, size_t len) {
  return guarded([&] { static_cast<CholeskyFactor*>(f)->append(std::span<const double>(col, len)); });
}
extern "C" int ref_cholesky_solve(void* f, const double* rhs, size_t nr, double* x, size_t nx) {
  return guarded([&] {
    static_cast<CholeskyFactor*>(f)->solve(std::span<const double>(rhs, nr), std::span<double>(x, nx));
  });
}

// ---- generators / writers (host-side helpers of the Python module) ----------
// pin paper_2107_13887_b200/host_tools.py: nodes, quads and markers of
// gen_airfoil_mesh (generators.cpp:45-128), the displacement fields of
// gen_sinusoidal_displacement / gen_ice_bump (generators.cpp:130-333) and the
// bytes written by write_vtk / write_displacements (mesh_io.cpp:311-428).
#include "icemorph/generators.hpp"

extern "C" int ref_gen_airfoil_mesh(double chord, size_t n, size_t m, double* nodes,
                                    size_t* quads, size_t* airfoil, size_t* farfield) {
  return guarded([&] {
    const Mesh mesh = gen_airfoil_mesh(chord, n, m);
    for (size_t i = 0; i < mesh.nodes.size(); ++i) put(nodes + 3 * i, mesh.nodes[i]);
    for (size_t e = 0; e < mesh.elements.size(); ++e)
      for (int k = 0; k < 4; ++k) quads[4 * e + k] = mesh.elements[e].nodes[k];
    const auto& a = mesh.marker("airfoil").nodes;
    const auto& f = mesh.marker("farfield").nodes;
    std::copy(a.begin(), a.end(), airfoil);
    std::copy(f.begin(), f.end(), farfield);
  });
}

// which: 0 sinusoidal (airfoil mode: p0 amplitude, p1 wavenumber),
//        1 ice bump (p0 center, p1 height, p2 width, horns)
extern "C" int ref_gen_field(double chord, size_t n, size_t m, int which, double p0, double p1,
                             double p2, size_t horns, size_t* idx, double* disp, size_t* count) {
  return guarded([&] {
    const Mesh mesh = gen_airfoil_mesh(chord, n, m);
    const DisplacementField f =
        which == 0 ? gen_sinusoidal_displacement(mesh, "airfoil", SinusoidalMode::Airfoil, p0, p1)
                   : gen_ice_bump(mesh, "airfoil", IceBumpParams{p0, p1, p2, horns});
    size_t k = 0;
    for (const auto& [node, d] : f.entries) idx[k] = node, put(disp + 3 * k, d), ++k;
    *count = k;
  });
}

extern "C" int ref_write_airfoil_files(double chord, size_t n, size_t m, const char* vtk_path,
                                       const char* disp_path) {
  return guarded([&] {
    const Mesh mesh = gen_airfoil_mesh(chord, n, m);
    write_vtk(mesh, std::string(vtk_path));
    const DisplacementField f = gen_ice_bump(mesh, "airfoil", IceBumpParams{0.0, 0.02, 0.05, 2});
    write_displacements(f, mesh.dim, std::string(disp_path));
  });
}
