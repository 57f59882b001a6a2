// icemorph_shim.cpp — the reference's public C++ API (icemorph/icemorph.hpp)
// over the B200 C-ABI (include/icemorph_b200.h).  Host-side glue only:
// argument marshalling, the reference's exceptions, and the scalar helpers
// (eval_wendland / eval_basis / wall functions) that the reference also
// evaluates on the host.  Every hot-path call goes to the device.
#include <fstream>
#include <iomanip>
#include <memory>
#include <ostream>
#include <unordered_set>

#include "../../../include/icemorph_b200.h"
#include "icemorph/icemorph.hpp"

namespace icemorph {
namespace {

// One context per host thread: calls from different threads never share a
// stream or scratch (the reference's reentrancy).
im_context* ctx() {
  thread_local struct Holder {
    im_context* c = nullptr;
    Holder() { im_context_create(&c, 0); }
    ~Holder() { im_context_destroy(c); }
  } h;
  return h.c;
}

void check(int rc) {
  if (rc == IM_OK) return;
  const std::string msg = im_last_error(ctx());
  if (rc == IM_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == IM_SOLVE_ERROR) throw SolveError(msg);
  if (rc == IM_PARSE_ERROR) throw ParseError(msg, im_last_error_line(ctx()));
  throw std::runtime_error(msg);
}

im_basis to_c(const BasisFunction& b) { return {static_cast<int>(b.kind), b.support_radius}; }

im_greedy_config to_c(const GreedyConfig& g) {
  return {g.tolerance, g.max_levels, g.max_points_per_level, to_c(g.basis)};
}

const double* xyz(std::span<const Vec3> v) { return v.empty() ? nullptr : &v[0].x; }

}  // namespace

// rbf.cpp:10-26
WendlandKind wendland_kind_from_string(const std::string& name) {
  if (name == "c0" || name == "C0") return WendlandKind::C0;
  if (name == "c2" || name == "C2") return WendlandKind::C2;
  if (name == "c4" || name == "C4") return WendlandKind::C4;
  if (name == "c6" || name == "C6") return WendlandKind::C6;
  throw std::invalid_argument("unknown basis function '" + name + "' (expected c0, c2, c4 or c6)");
}

std::string_view wendland_kind_name(WendlandKind kind) {
  static const char* names[] = {"c0", "c2", "c4", "c6"};
  const int k = static_cast<int>(kind);
  return k >= 0 && k < 4 ? names[k] : "?";
}

double eval_wendland(WendlandKind kind, double eta) {
  return im_eval_wendland(static_cast<int>(kind), eta);
}

double eval_basis(const BasisFunction& basis, double d) { return im_eval_basis(to_c(basis), d); }

// rbf.cpp:56-69 on the device
std::vector<double> assemble_surface_matrix(std::span<const Vec3> points,
                                            const BasisFunction& basis) {
  std::vector<double> m(points.size() * points.size());
  check(im_assemble_surface_matrix(ctx(), xyz(points), points.size(), to_c(basis), m.data()));
  return m;
}

// rbf.cpp:71-121: the factor lives on the device of this thread's context
CholeskyFactor::CholeskyFactor() {
  im_cholesky* f = nullptr;
  check(im_cholesky_create(ctx(), &f));
  handle_ = f;
}
CholeskyFactor::~CholeskyFactor() {
  if (handle_) im_cholesky_destroy(static_cast<im_cholesky*>(handle_));
}
CholeskyFactor::CholeskyFactor(CholeskyFactor&& o) noexcept : handle_(o.handle_) {
  o.handle_ = nullptr;
}
CholeskyFactor& CholeskyFactor::operator=(CholeskyFactor&& o) noexcept {
  if (this != &o) {
    if (handle_) im_cholesky_destroy(static_cast<im_cholesky*>(handle_));
    handle_ = o.handle_;
    o.handle_ = nullptr;
  }
  return *this;
}
std::size_t CholeskyFactor::size() const {
  return im_cholesky_size(static_cast<const im_cholesky*>(handle_));
}
double CholeskyFactor::smallest_pivot() const {
  return im_cholesky_smallest_pivot(static_cast<const im_cholesky*>(handle_));
}
void CholeskyFactor::append(std::span<const double> column) {
  check(im_cholesky_append(static_cast<im_cholesky*>(handle_), column.data(), column.size()));
}
void CholeskyFactor::solve(std::span<const double> rhs, std::span<double> x) const {
  check(im_cholesky_solve(static_cast<const im_cholesky*>(handle_), rhs.data(), rhs.size(),
                          x.data(), x.size()));
}

WeightSet solve_weights(std::span<const Vec3> points, std::span<const Vec3> displacements,
                        const BasisFunction& basis) {
  if (points.size() != displacements.size())
    throw std::invalid_argument("point and displacement counts differ");
  WeightSet w;
  w.control_positions.assign(points.begin(), points.end());
  w.alpha.assign(points.size(), Vec3{});
  check(im_solve_weights(ctx(), xyz(points), xyz(displacements), points.size(), to_c(basis),
                         w.alpha.empty() ? nullptr : &w.alpha[0].x));
  return w;
}

std::vector<Vec3> eval_interpolant(const WeightSet& w, const BasisFunction& basis,
                                   std::span<const Vec3> queries) {
  std::vector<Vec3> out(queries.size());
  check(im_eval_interpolant(ctx(), xyz(w.control_positions), xyz(w.alpha), w.size(), to_c(basis),
                            xyz(queries), queries.size(), IM_EXACT,
                            out.empty() ? nullptr : &out[0].x));
  return out;
}

Vec3 eval_interpolant(const WeightSet& w, const BasisFunction& basis, const Vec3& query) {
  return eval_interpolant(w, basis, std::span<const Vec3>(&query, 1))[0];
}

LevelResult greedy_level(std::span<const Vec3> pos, std::span<const Vec3> target,
                         const GreedyConfig& config, std::size_t level_index) {
  if (target.size() != pos.size())
    throw std::invalid_argument("target size does not match surface size");
  const std::size_t m = std::max<std::size_t>(1, std::min(config.max_points_per_level, pos.size()));
  const im_greedy_config cfg = to_c(config);
  std::vector<std::size_t> idx(m), rp(m);
  std::vector<Vec3> alpha(m);
  std::vector<double> re(m), rs(m);
  LevelResult r;
  r.residual.resize(pos.size());
  size_t nc = 0, nrec = 0;
  double achieved = 0, tmax = 0, el = 0;
  int cap_hit = 0;
  check(im_greedy_level(ctx(), xyz(pos), xyz(target), pos.size(), &cfg, level_index, idx.data(),
                        &alpha[0].x, &nc, &achieved, &cap_hit, &tmax, &el, rp.data(), re.data(),
                        rs.data(), &nrec, r.residual.empty() ? nullptr : &r.residual[0].x));
  r.level.level = level_index;
  r.level.control_indices.assign(idx.begin(), idx.begin() + nc);
  for (std::size_t c : r.level.control_indices) r.level.weights.control_positions.push_back(pos[c]);
  r.level.weights.alpha.assign(alpha.begin(), alpha.begin() + nc);
  r.level.achieved_error = achieved;
  r.level.cap_hit = cap_hit != 0;
  r.level.target_max = tmax;
  r.level.elapsed_seconds = el;
  for (std::size_t s = 0; s < nrec; ++s) r.record.samples.push_back({rp[s], re[s], rs[s]});
  return r;
}

MultilevelResult run_multilevel(std::span<const Vec3> pos, std::span<const Vec3> target,
                                const GreedyConfig& config) {
  if (target.size() != pos.size())
    throw std::invalid_argument("target size does not match surface size");
  const std::size_t m = std::max<std::size_t>(1, std::min(config.max_points_per_level, pos.size()));
  const std::size_t L = std::max<std::size_t>(1, config.max_levels);
  const im_greedy_config cfg = to_c(config);
  std::vector<std::size_t> nc(L), idx(L * m), nrec(L);
  std::vector<Vec3> alpha(L * m);
  std::vector<double> ach(L), ltm(L), el(L), rerr(L * m);
  std::vector<int> caph(L);
  size_t nl = 0;
  MultilevelResult r;
  r.final_residual.resize(pos.size());
  check(im_run_multilevel(ctx(), xyz(pos), xyz(target), pos.size(), &cfg, &nl, nc.data(),
                          idx.data(), &alpha[0].x, ach.data(), caph.data(), ltm.data(), el.data(),
                          nrec.data(), rerr.data(), &r.target_max,
                          r.final_residual.empty() ? nullptr : &r.final_residual[0].x));
  for (std::size_t l = 0; l < nl; ++l) {
    RbfLevel lv;
    lv.level = l;
    lv.control_indices.assign(idx.begin() + l * m, idx.begin() + l * m + nc[l]);
    for (std::size_t c : lv.control_indices) lv.weights.control_positions.push_back(pos[c]);
    lv.weights.alpha.assign(alpha.begin() + l * m, alpha.begin() + l * m + nc[l]);
    lv.achieved_error = ach[l];
    lv.cap_hit = caph[l] != 0;
    lv.target_max = ltm[l];
    lv.elapsed_seconds = el[l];
    ConvergenceRecord rec;
    for (std::size_t s = 0; s < nrec[l]; ++s) rec.samples.push_back({s + 1, rerr[l * m + s], 0.0});
    r.levels.push_back(std::move(lv));
    r.records.push_back(std::move(rec));
  }
  return r;
}

void write_convergence_csv_header(std::ostream& out) { out << "level,points,error,seconds\n"; }

void append_convergence_csv(std::ostream& out, std::size_t level, const ConvergenceRecord& rec) {
  for (const auto& s : rec.samples)
    out << level << ',' << s.points << ',' << std::setprecision(17) << s.error << ','
        << std::setprecision(6) << s.seconds << "\n";
}

const Marker* Mesh::find_marker(std::string_view name) const {
  for (const auto& m : markers)
    if (m.name == name) return &m;
  return nullptr;
}

const Marker& Mesh::marker(std::string_view name) const {
  const Marker* m = find_marker(name);
  if (!m) throw std::invalid_argument("mesh has no marker named '" + std::string(name) + "'");
  return *m;
}

double DisplacementField::max_magnitude() const {
  double m = 0.0;
  for (const auto& [n, d] : entries) m = std::max(m, d.norm());
  return m;
}

DistanceIndex build_distance_index(const Mesh& mesh, const std::string& marker) {
  return build_distance_index(mesh, mesh.marker(marker).nodes);
}

DistanceIndex build_distance_index(const Mesh& mesh, const std::vector<std::size_t>& surface) {
  DistanceIndex idx;
  idx.distances.resize(mesh.nodes.size());
  check(im_build_distance_index(ctx(), xyz(mesh.nodes), mesh.nodes.size(), mesh.dim,
                                surface.data(), surface.size(), idx.distances.data()));
  return idx;
}

WallFunction make_wall_function(double k, double level_target_max) {
  im_wall_function wf{};
  if (im_make_wall_function(k, level_target_max, &wf) != IM_OK)
    throw std::invalid_argument("volume reduction factor must be positive");
  return {wf.reduction_factor, wf.support_distance, wf.psi_kind};
}

double eval_wall_function(const WallFunction& wf, double d) {
  const im_wall_function w{wf.reduction_factor, wf.support_distance, wf.psi_kind};
  return im_eval_wall_function(&w, d);
}

VolumeUpdate update_volume(const Mesh& mesh, const RbfLevel& level, const DistanceIndex& index,
                           const WallFunction& wf, const BasisFunction& basis) {
  if (index.distances.size() != mesh.nodes.size())
    throw std::invalid_argument("distance index does not match the mesh");
  const std::size_t n = mesh.nodes.size();
  std::vector<std::size_t> nodes(n);
  std::vector<Vec3> values(n);
  size_t k = 0;
  const im_wall_function w{wf.reduction_factor, wf.support_distance, wf.psi_kind};
  check(im_update_volume(ctx(), xyz(mesh.nodes), n, index.distances.data(),
                         xyz(level.weights.control_positions), xyz(level.weights.alpha),
                         level.weights.size(), &w, to_c(basis), IM_EXACT, nodes.data(),
                         values.empty() ? nullptr : &values[0].x, &k));
  VolumeUpdate u;
  u.entries.reserve(k);
  for (std::size_t i = 0; i < k; ++i) u.entries.emplace_back(nodes[i], values[i]);
  return u;
}

std::size_t DeformationReport::total_control_points() const {
  std::size_t t = 0;
  for (const auto& l : levels) t += l.points;
  return t;
}

namespace {
// Mesh::elements -> the C-ABI's CSR element arrays.
struct ElementCsr {
  std::vector<int> kinds;
  std::vector<std::size_t> offsets{0}, nodes;
  explicit ElementCsr(const std::vector<Element>& elements) {
    kinds.reserve(elements.size());
    offsets.reserve(elements.size() + 1);
    for (const auto& e : elements) {
      kinds.push_back(static_cast<int>(e.kind));
      nodes.insert(nodes.end(), e.nodes.begin(), e.nodes.end());
      offsets.push_back(nodes.size());
    }
  }
  const std::size_t* conn() const { return nodes.empty() ? offsets.data() : nodes.data(); }
};

std::size_t measures(const Mesh& mesh, const std::vector<Element>& elements, double* out) {
  const ElementCsr csr(elements);
  std::size_t inverted = 0;
  check(im_signed_measures(ctx(), xyz(mesh.nodes), mesh.nodes.size(), csr.kinds.data(),
                           csr.offsets.data(), csr.conn(), elements.size(), out, &inverted));
  return inverted;
}
}  // namespace

std::vector<double> signed_measures(const Mesh& mesh) {
  std::vector<double> m(mesh.elements.size());
  measures(mesh, mesh.elements, m.data());
  return m;
}

double signed_measure(const Mesh& mesh, const Element& element) {
  double m = 0.0;
  measures(mesh, {element}, &m);
  return m;
}

std::size_t count_inverted(const Mesh& mesh) { return measures(mesh, mesh.elements, nullptr); }

Mesh read_su2(const std::string& path) {
  im_mesh* h = nullptr;
  check(im_su2_read(ctx(), path.c_str(), &h));
  std::unique_ptr<im_mesh, int (*)(im_mesh*)> guard(h, im_mesh_destroy);
  int dim = 0;
  std::size_t nn = 0, ne = 0, nc = 0, nm = 0;
  im_mesh_sizes(h, &dim, &nn, &ne, &nc, &nm);
  Mesh m;
  m.dim = dim;
  m.nodes.resize(nn);
  if (nn) im_mesh_nodes(h, &m.nodes[0].x);
  std::vector<int> kinds(ne);
  std::vector<std::size_t> offsets(ne + 1), conn(nc);
  im_mesh_elements(h, kinds.data(), offsets.data(), conn.data());
  m.elements.resize(ne);
  for (std::size_t e = 0; e < ne; ++e) {
    m.elements[e].kind = static_cast<ElementKind>(kinds[e]);
    m.elements[e].nodes.assign(conn.begin() + offsets[e], conn.begin() + offsets[e + 1]);
  }
  for (std::size_t k = 0; k < nm; ++k) {
    std::size_t len = 0, me = 0, mc = 0, mn = 0;
    im_mesh_marker_sizes(h, k, &len, &me, &mc, &mn);
    std::string name(len, '\0');
    std::vector<int> mk(me);
    std::vector<std::size_t> mo(me + 1), mconn(mc);
    Marker mark;
    mark.nodes.resize(mn);
    im_mesh_marker(h, k, name.data(), mk.data(), mo.data(), mconn.data(), mark.nodes.data());
    mark.name = name;
    mark.elements.resize(me);
    for (std::size_t e = 0; e < me; ++e) {
      mark.elements[e].kind = static_cast<ElementKind>(mk[e]);
      mark.elements[e].nodes.assign(mconn.begin() + mo[e], mconn.begin() + mo[e + 1]);
    }
    m.markers.push_back(std::move(mark));
  }
  return m;
}

void write_su2(const Mesh& mesh, const std::string& path) {
  const ElementCsr csr(mesh.elements);
  std::vector<ElementCsr> mcsr;
  for (const auto& k : mesh.markers) mcsr.emplace_back(k.elements);
  std::vector<const char*> names;
  std::vector<const int*> mk;
  std::vector<const std::size_t*> mo, mc;
  std::vector<std::size_t> mn;
  for (std::size_t k = 0; k < mesh.markers.size(); ++k) {
    names.push_back(mesh.markers[k].name.c_str());
    mk.push_back(mcsr[k].kinds.data());
    mo.push_back(mcsr[k].offsets.data());
    mc.push_back(mcsr[k].conn());
    mn.push_back(mesh.markers[k].elements.size());
  }
  check(im_su2_write(ctx(), path.c_str(), mesh.dim, xyz(mesh.nodes), mesh.nodes.size(),
                     csr.kinds.data(), csr.offsets.data(), csr.conn(), mesh.elements.size(),
                     mesh.markers.size(), names.data(), mk.data(), mo.data(), mc.data(), mn.data()));
}

QualityReport orthogonality(const Mesh& mesh) {
  const ElementCsr csr(mesh.elements);
  QualityReport q;
  const std::size_t n = mesh.elements.size();
  q.element_orthogonality_deg.resize(n);
  q.element_signed_measure.resize(n);
  im_quality_report r{};
  check(im_orthogonality(ctx(), xyz(mesh.nodes), mesh.nodes.size(), csr.kinds.data(),
                         csr.offsets.data(), csr.conn(), n, q.element_orthogonality_deg.data(),
                         q.element_signed_measure.data(), &r));
  q.min_orthogonality_deg = r.min_orthogonality_deg;
  q.mean_orthogonality_deg = r.mean_orthogonality_deg;
  q.inverted_count = r.inverted_count;
  q.degenerate_count = r.degenerate_count;
  return q;
}

std::pair<Mesh, DeformationReport> deform(const Mesh& mesh, const DisplacementField& disp,
                                          const DeformationConfig& config) {
  const Marker& marker = mesh.marker(disp.patch);
  if (marker.nodes.empty())
    throw std::invalid_argument("marker '" + disp.patch + "' has no nodes");
  std::vector<std::size_t> pinned;
  for (const auto& name : config.fixed_markers)
    for (std::size_t n : mesh.marker(name).nodes) pinned.push_back(n);
  std::vector<Vec3> d(marker.nodes.size());
  for (std::size_t i = 0; i < marker.nodes.size(); ++i) d[i] = disp.at(marker.nodes[i]);
  const ElementCsr csr(mesh.elements);
  const std::size_t L = std::max<std::size_t>(1, config.greedy.max_levels);
  const std::size_t stride = std::max<std::size_t>(
      1, std::min(config.greedy.max_points_per_level, marker.nodes.size() + pinned.size()));
  std::vector<double> rec_e(L * stride), rec_s(L * stride);
  const im_deform_config cfg{to_c(config.greedy),
                             config.volume_k,
                             config.support_distance,
                             config.psi_kind,
                             config.precision,
                             csr.kinds.data(),
                             csr.offsets.data(),
                             csr.conn(),
                             mesh.elements.size(),
                             config.compute_quality && !mesh.elements.empty() ? 1 : 0,
                             rec_e.data(),
                             rec_s.data(),
                             stride};
  Mesh out = mesh;
  im_deform_report rep{};
  std::vector<std::size_t> pts(L), touched(L);
  std::vector<double> ach(L), sup(L), sec(L);
  std::vector<int> caph(L);
  check(im_deform(ctx(), xyz(mesh.nodes), mesh.nodes.size(), mesh.dim, marker.nodes.data(),
                  marker.nodes.size(), &d[0].x, pinned.empty() ? nullptr : pinned.data(),
                  pinned.size(), &cfg, out.nodes.empty() ? nullptr : &out.nodes[0].x, &rep,
                  pts.data(), ach.data(), caph.data(), sup.data(), touched.data(), sec.data()));
  DeformationReport r;
  r.marker = disp.patch;
  for (std::size_t l = 0; l < rep.n_levels; ++l) {
    LevelSummary s;
    s.level = l;
    s.points = pts[l];
    s.achieved_error = ach[l];
    s.cap_hit = caph[l] != 0;
    s.support_distance = sup[l];
    s.touched_nodes = touched[l];
    s.seconds = sec[l];
    for (std::size_t k = 0; k < pts[l]; ++k)  // LevelSummary::record (pipeline.cpp:83)
      s.record.samples.push_back({k + 1, rec_e[l * stride + k], rec_s[l * stride + k]});
    r.levels.push_back(std::move(s));
  }
  r.target_max = rep.target_max;
  r.surface_max_error = rep.surface_max_error;
  r.surface_mean_error = rep.surface_mean_error;
  r.inverted_elements = rep.inverted_elements;
  if (rep.has_quality) {
    auto to_q = [](const im_quality_report& x) {
      QualityReport q;
      q.min_orthogonality_deg = x.min_orthogonality_deg;
      q.mean_orthogonality_deg = x.mean_orthogonality_deg;
      q.inverted_count = x.inverted_count;
      q.degenerate_count = x.degenerate_count;
      return q;
    };
    r.quality_before = to_q(rep.quality_before);
    r.quality_after = to_q(rep.quality_after);
  }
  r.total_seconds = rep.total_seconds;
  return {std::move(out), std::move(r)};
}

void write_summary(const DeformationReport& report, std::ostream& out) {
  out << std::setprecision(17);
  out << "marker: " << report.marker << "\n";
  out << "levels: " << report.levels.size() << "\n";
  out << "total_control_points: " << report.total_control_points() << "\n";
  out << "target_max: " << report.target_max << "\n";
  out << "surface_max_error: " << report.surface_max_error << "\n";
  out << "surface_mean_error: " << report.surface_mean_error << "\n";
  out << "inverted_elements: " << report.inverted_elements << "\n";
  if (report.quality_before) {
    out << "min_orthogonality_before_deg: " << report.quality_before->min_orthogonality_deg << "\n";
    out << "mean_orthogonality_before_deg: " << report.quality_before->mean_orthogonality_deg
        << "\n";
  }
  if (report.quality_after) {
    out << "min_orthogonality_after_deg: " << report.quality_after->min_orthogonality_deg << "\n";
    out << "mean_orthogonality_after_deg: " << report.quality_after->mean_orthogonality_deg << "\n";
  }
  out << "total_seconds: " << std::setprecision(6) << report.total_seconds << std::setprecision(17)
      << "\n";
  for (const auto& l : report.levels) {
    const std::string p = "level_" + std::to_string(l.level) + "_";
    out << p << "points: " << l.points << "\n" << p << "error: " << l.achieved_error << "\n"
        << p << "cap_hit: " << (l.cap_hit ? 1 : 0) << "\n" << p << "support_distance: "
        << l.support_distance << "\n" << p << "touched_nodes: " << l.touched_nodes << "\n" << p
        << "seconds: " << std::setprecision(6) << l.seconds << std::setprecision(17) << "\n";
  }
}

void write_convergence_csv(const DeformationReport& report, std::ostream& out) {
  write_convergence_csv_header(out);
  for (const auto& l : report.levels) append_convergence_csv(out, l.level, l.record);
}

// pipeline.cpp:143-160
void write_summary(const DeformationReport& report, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write summary file '" + path + "'");
  write_summary(report, out);
}

void write_convergence_csv(const DeformationReport& report, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write report file '" + path + "'");
  write_convergence_csv(report, out);
}

}  // namespace icemorph
