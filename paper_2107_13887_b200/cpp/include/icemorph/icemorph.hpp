// icemorph/icemorph.hpp — the reference library's public C++ API for the
// hot path (proj/include/icemorph/{vec,rbf,greedy,wall_distance,mesh,
// mesh_io,pipeline}.hpp), re-declared with the same names, types and
// semantics and implemented over the B200 C-ABI (include/icemorph_b200.h)
// by paper_2107_13887_b200/cpp/src/icemorph_shim.cpp.  A caller of the
// reference recompiles against this header and links libicemorph_core.so
// (+ libicemorph_b200.so); nothing else changes.
//
// Additive fields (defaults reproduce the reference): WallFunction::psi_kind,
// DeformationConfig::{support_distance, psi_kind, precision}.  Out of scope
// (not on the hot path): mesh I/O, generators, the orthogonality report;
// DeformationReport carries inverted_elements and, with compute_quality and
// mesh elements, the quality reports before / after (scalars only).
#pragma once

#include <cmath>
#include <cstddef>
#include <iosfwd>
#include <limits>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace icemorph {

// ---- vec.hpp -----------------------------------------------------------------
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  Vec3() = default;
  Vec3(double x_, double y_, double z_ = 0.0) : x(x_), y(y_), z(z_) {}
  Vec3& operator+=(const Vec3& o) { x += o.x; y += o.y; z += o.z; return *this; }
  Vec3& operator-=(const Vec3& o) { x -= o.x; y -= o.y; z -= o.z; return *this; }
  Vec3& operator*=(double s) { x *= s; y *= s; z *= s; return *this; }
  double squared_norm() const { return x * x + y * y + z * z; }
  double norm() const { return std::sqrt(squared_norm()); }
};
inline Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
inline Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
inline Vec3 operator*(Vec3 a, double s) { return a *= s; }
inline Vec3 operator*(double s, Vec3 a) { return a *= s; }
inline bool operator==(const Vec3& a, const Vec3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
inline bool operator!=(const Vec3& a, const Vec3& b) { return !(a == b); }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double distance(const Vec3& a, const Vec3& b) { return (a - b).norm(); }
inline double squared_distance(const Vec3& a, const Vec3& b) { return (a - b).squared_norm(); }
inline Vec3 normalized(const Vec3& v) {
  const double n = v.norm();
  return n > 0.0 ? v * (1.0 / n) : Vec3{};
}
static_assert(sizeof(Vec3) == 24, "Vec3 must be three packed doubles (AoS C-ABI)");

// ---- rbf.hpp -------------------------------------------------------------------
class SolveError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
enum class WendlandKind { C0, C2, C4, C6 };
WendlandKind wendland_kind_from_string(const std::string& name);
std::string_view wendland_kind_name(WendlandKind kind);
struct BasisFunction {
  WendlandKind kind = WendlandKind::C2;
  double support_radius = 1.0;
};
double eval_wendland(WendlandKind kind, double eta);
double eval_basis(const BasisFunction& basis, double distance);
/// Dense kernel matrix phi(|r_i - r_j|), unit diagonal, row-major n*n
/// (rbf.hpp:35-36), assembled on the device.
std::vector<double> assemble_surface_matrix(std::span<const Vec3> points,
                                            const BasisFunction& basis);
/// Cholesky factor grown one row at a time (rbf.hpp:41-60), resident on the
/// device (im_cholesky_*): append throws SolveError when the pivot falls
/// below 1e-14 of the largest diagonal seen; solve(rhs, x) solves A x = rhs.
class CholeskyFactor {
 public:
  CholeskyFactor();
  ~CholeskyFactor();
  CholeskyFactor(const CholeskyFactor&) = delete;
  CholeskyFactor& operator=(const CholeskyFactor&) = delete;
  CholeskyFactor(CholeskyFactor&& o) noexcept;
  CholeskyFactor& operator=(CholeskyFactor&& o) noexcept;
  std::size_t size() const;
  void append(std::span<const double> column);
  void solve(std::span<const double> rhs, std::span<double> x) const;
  double smallest_pivot() const;

 private:
  void* handle_ = nullptr;  // im_cholesky*
};
struct WeightSet {
  std::vector<Vec3> control_positions;
  std::vector<Vec3> alpha;
  std::size_t size() const { return control_positions.size(); }
};
WeightSet solve_weights(std::span<const Vec3> points, std::span<const Vec3> displacements,
                        const BasisFunction& basis);
Vec3 eval_interpolant(const WeightSet& weights, const BasisFunction& basis, const Vec3& query);
// batched form (one device launch for many queries; additive)
std::vector<Vec3> eval_interpolant(const WeightSet& weights, const BasisFunction& basis,
                                   std::span<const Vec3> queries);

// ---- greedy.hpp -----------------------------------------------------------------
struct GreedyConfig {
  double tolerance = 0.1;
  std::size_t max_levels = 5;
  std::size_t max_points_per_level = 5000;
  BasisFunction basis;
};
struct ConvergenceSample {
  std::size_t points = 0;
  double error = 0.0;
  double seconds = 0.0;
};
struct ConvergenceRecord {
  std::vector<ConvergenceSample> samples;
};
struct RbfLevel {
  std::size_t level = 0;
  std::vector<std::size_t> control_indices;
  WeightSet weights;
  double achieved_error = 0.0;
  bool cap_hit = false;
  double target_max = 0.0;
  double elapsed_seconds = 0.0;
};
struct LevelResult {
  RbfLevel level;
  ConvergenceRecord record;
  std::vector<Vec3> residual;
};
LevelResult greedy_level(std::span<const Vec3> surface_positions, std::span<const Vec3> target,
                         const GreedyConfig& config, std::size_t level_index = 0);
struct MultilevelResult {
  std::vector<RbfLevel> levels;
  std::vector<ConvergenceRecord> records;
  std::vector<Vec3> final_residual;
  double target_max = 0.0;
};
MultilevelResult run_multilevel(std::span<const Vec3> surface_positions,
                                std::span<const Vec3> target, const GreedyConfig& config);
void write_convergence_csv_header(std::ostream& out);
void append_convergence_csv(std::ostream& out, std::size_t level, const ConvergenceRecord& record);

// ---- mesh.hpp / mesh_io.hpp (data model only) -------------------------------------
enum class ElementKind { Line, Triangle, Quadrilateral, Tetrahedron, Hexahedron, Prism, Pyramid };
struct Element {
  ElementKind kind = ElementKind::Triangle;
  std::vector<std::size_t> nodes;
};
struct Marker {
  std::string name;
  std::vector<Element> elements;
  std::vector<std::size_t> nodes;
};
struct Mesh {
  int dim = 2;
  std::vector<Vec3> nodes;
  std::vector<Element> elements;
  std::vector<Marker> markers;
  std::size_t node_count() const { return nodes.size(); }
  const Marker* find_marker(std::string_view name) const;
  const Marker& marker(std::string_view name) const;
};
struct DisplacementField {
  std::string patch;
  std::map<std::size_t, Vec3> entries;
  Vec3 at(std::size_t node) const {
    auto it = entries.find(node);
    return it == entries.end() ? Vec3{} : it->second;
  }
  double max_magnitude() const;
};

// ---- wall_distance.hpp ---------------------------------------------------------------
struct DistanceIndex {
  std::vector<double> distances;
};
DistanceIndex build_distance_index(const Mesh& mesh, const std::string& marker);
DistanceIndex build_distance_index(const Mesh& mesh, const std::vector<std::size_t>& surface_nodes);
struct WallFunction {
  double reduction_factor = 5.0;
  double support_distance = 0.0;
  int psi_kind = 0;  // additive: 0 linear taper (reference), 1 Wendland C2 of xi
};
WallFunction make_wall_function(double reduction_factor, double level_target_max);
double eval_wall_function(const WallFunction& wf, double wall_distance);
struct VolumeUpdate {
  std::vector<std::pair<std::size_t, Vec3>> entries;
};
VolumeUpdate update_volume(const Mesh& mesh, const RbfLevel& level, const DistanceIndex& index,
                           const WallFunction& wf, const BasisFunction& basis);

// ---- pipeline.hpp -------------------------------------------------------------------------
struct DeformationConfig {
  GreedyConfig greedy;
  double volume_k = 5.0;
  std::vector<std::string> fixed_markers;
  bool compute_quality = true;  // orthogonality before / after (device), needs elements
  // additive: absolute support distance (< 0: reference D_l = volume_k * target_max_l),
  // taper kind, arithmetic (0 exact reference order, 1 FP64 fast path)
  double support_distance = -1.0;
  int psi_kind = 0;
  int precision = 0;
};
struct LevelSummary {
  std::size_t level = 0;
  std::size_t points = 0;
  double achieved_error = 0.0;
  bool cap_hit = false;
  double support_distance = 0.0;
  std::size_t touched_nodes = 0;
  double seconds = 0.0;
  ConvergenceRecord record;
};
// ---- mesh_io.hpp (SU2 subset) ---------------------------------------------------------
class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& what, std::size_t line) : std::runtime_error(what), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_ = 0;
};
Mesh read_su2(const std::string& path);
void write_su2(const Mesh& mesh, const std::string& path);

// ---- quality.hpp ------------------------------------------------------------------
struct QualityReport {
  std::vector<double> element_orthogonality_deg;
  std::vector<double> element_signed_measure;
  double min_orthogonality_deg = 90.0;
  double mean_orthogonality_deg = 90.0;
  std::size_t inverted_count = 0;
  std::size_t degenerate_count = 0;
};
QualityReport orthogonality(const Mesh& mesh);

struct DeformationReport {
  std::string marker;
  std::vector<LevelSummary> levels;
  double target_max = 0.0;
  double surface_max_error = 0.0;
  double surface_mean_error = 0.0;
  std::size_t inverted_elements = 0;
  std::optional<QualityReport> quality_before;  // element vectors left empty
  std::optional<QualityReport> quality_after;
  double total_seconds = 0.0;
  std::size_t total_control_points() const;
};
std::pair<Mesh, DeformationReport> deform(const Mesh& mesh, const DisplacementField& displacement,
                                          const DeformationConfig& config);
void write_summary(const DeformationReport& report, std::ostream& out);
void write_summary(const DeformationReport& report, const std::string& path);

// ---- quality.hpp: the measures deform's report reads (device-evaluated) ------------
std::vector<double> signed_measures(const Mesh& mesh);
double signed_measure(const Mesh& mesh, const Element& element);
std::size_t count_inverted(const Mesh& mesh);
void write_convergence_csv(const DeformationReport& report, std::ostream& out);
void write_convergence_csv(const DeformationReport& report, const std::string& path);

}  // namespace icemorph
