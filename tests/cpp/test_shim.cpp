// C++ client of the reference API (icemorph/icemorph.hpp) backed by the B200
// library: the reference tests' known-answer values, checked through the C++
// shim exactly as a reference caller would use it.  Exit code 0 = all passed.
#include <cmath>
#include <cstdio>
#include <string>

#include <fstream>
#include <random>
#include <vector>

// the reference's per-module headers resolve to the shim (forwarding headers)
#include "icemorph/greedy.hpp"
#include "icemorph/mesh.hpp"
#include "icemorph/mesh_io.hpp"
#include "icemorph/pipeline.hpp"
#include "icemorph/quality.hpp"
#include "icemorph/rbf.hpp"
#include "icemorph/vec.hpp"
#include "icemorph/wall_distance.hpp"

using namespace icemorph;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

int main() {
  // rbf KATs (test_rbf.cpp:40-52, 74-80)
  CHECK(eval_wendland(WendlandKind::C2, 0.5) == 0.1875);
  CHECK(eval_wendland(WendlandKind::C0, 0.5) == 0.25);
  CHECK(eval_basis({WendlandKind::C2, 2.0}, 1.0) == 0.1875);
  // two-point solve (test_rbf.cpp:96-119)
  const BasisFunction b2{WendlandKind::C2, 2.0};
  const std::vector<Vec3> two{{0.0, 0.0}, {1.0, 0.0}};
  const WeightSet w = solve_weights(two, std::vector<Vec3>{{1.0, 0.0}, {0.0, 0.0}}, b2);
  const double bb = 0.1875;
  CHECK(std::abs(w.alpha[0].x - 1.0 / (1.0 - bb * bb)) < 1e-12);
  CHECK(std::abs(w.alpha[1].x + bb / (1.0 - bb * bb)) < 1e-12);
  CHECK(std::abs(eval_interpolant(w, b2, Vec3{0.5, 0.0}).x - 0.6328125 / 1.1875) < 1e-12);
  // duplicate points -> SolveError naming the pair (test_rbf.cpp:223-229)
  bool threw = false;
  try {
    solve_weights(std::vector<Vec3>{{0, 0}, {1e-18, 0}}, std::vector<Vec3>{{1, 0}, {2, 0}},
                  {WendlandKind::C2, 1.0});
  } catch (const SolveError& e) {
    threw = std::string(e.what()).find("points 0 and 1") != std::string::npos;
  }
  CHECK(threw);
  // greedy: three collinear points (test_greedy.cpp:38-51)
  GreedyConfig gc;
  gc.tolerance = 0.1;
  gc.max_levels = 1;
  gc.basis = b2;
  const auto g = greedy_level(std::vector<Vec3>{{0, 0}, {0.5, 0}, {1, 0}},
                              std::vector<Vec3>{{0, 0}, {0, 1}, {0, 0}}, gc);
  CHECK(g.level.control_indices.size() >= 2 && g.level.control_indices[0] == 0 &&
        g.level.control_indices[1] == 1);
  CHECK(g.level.achieved_error < 0.1);
  CHECK(g.record.samples.size() == g.level.control_indices.size());
  // wall distance (test_wall_distance.cpp:29-39)
  Mesh mesh;
  mesh.dim = 2;
  mesh.nodes = {{0.0, 0.0}, {1.0, 0.0}, {0.5, 1.0}, {4.0, 0.0}};
  const DistanceIndex idx = build_distance_index(mesh, std::vector<std::size_t>{0, 1});
  CHECK(idx.distances[0] == 0.0 && idx.distances[1] == 0.0);
  CHECK(std::abs(idx.distances[2] - std::sqrt(1.25)) < 1e-15);
  CHECK(idx.distances[3] == 3.0);
  // wall taper (test_wall_distance.cpp:49-60)
  const WallFunction wf = make_wall_function(5.0, 0.02);
  CHECK(std::abs(eval_wall_function(wf, 0.05) - 0.5) < 1e-12);
  CHECK(eval_wall_function(wf, 0.1) == 0.0);
  // update_volume (test_wall_distance.cpp:62-90)
  Mesh m2;
  m2.dim = 2;
  m2.nodes = {{0.0, 0.0}, {0.0, 0.05}, {0.0, 0.2}, {0.0, 5.0}};
  const DistanceIndex i2 = build_distance_index(m2, std::vector<std::size_t>{0});
  RbfLevel lvl;
  lvl.weights.control_positions = {{0.0, 0.0}};
  lvl.weights.alpha = {{0.0, 0.7, 0.0}};
  lvl.target_max = 0.02;
  const VolumeUpdate u = update_volume(m2, lvl, i2, make_wall_function(5.0, 0.02), b2);
  CHECK(u.entries.size() == 2);
  CHECK(u.entries[0].first == 0 && u.entries[0].second == lvl.weights.alpha[0]);
  CHECK(u.entries[1].first == 1 &&
        std::abs(u.entries[1].second.y - 0.5 * 0.7 * eval_basis(b2, 0.05)) < 1e-14);
  // deform on a small ring mesh with a pinned outer ring (test_pipeline.cpp:61-77)
  Mesh ring;
  ring.dim = 2;
  const int n = 64;
  Marker inner{"wall", {}, {}}, outer{"far", {}, {}};
  for (int layer = 0; layer < 6; ++layer)
    for (int j = 0; j < n; ++j) {
      const double t = 2 * M_PI * j / n, r = 1.0 + 0.5 * layer;
      ring.nodes.push_back({r * std::cos(t), r * std::sin(t)});
      if (layer == 0) inner.nodes.push_back(ring.nodes.size() - 1);
      if (layer == 5) outer.nodes.push_back(ring.nodes.size() - 1);
    }
  ring.markers = {inner, outer};
  DisplacementField f;
  f.patch = "wall";
  for (std::size_t k : inner.nodes)
    f.entries[k] = Vec3{0.0, 0.02 * std::sin(3.0 * std::atan2(ring.nodes[k].y, ring.nodes[k].x))};
  DeformationConfig dc;
  dc.greedy.tolerance = 0.1;
  dc.greedy.max_levels = 3;
  dc.greedy.basis = {WendlandKind::C2, 2.0};
  dc.fixed_markers = {"far"};
  const auto [deformed, report] = deform(ring, f, dc);
  for (std::size_t k : outer.nodes) CHECK(deformed.nodes[k] == ring.nodes[k]);
  CHECK(report.surface_max_error < 1e-3);
  CHECK(!report.levels.empty() && report.total_control_points() > 0);
  CHECK(report.inverted_elements == 0);  // ring has no elements

  // quality.cpp:100-148 (test_quality.cpp:68-78, 115-128)
  Mesh tri;
  tri.dim = 2;
  tri.nodes = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}};
  tri.elements = {{ElementKind::Triangle, {0, 1, 2}}, {ElementKind::Triangle, {0, 2, 1}}};
  CHECK(signed_measure(tri, tri.elements[0]) == 0.5);
  CHECK(signed_measures(tri)[1] == -0.5);
  CHECK(count_inverted(tri) == 1);
  Mesh cube;
  cube.dim = 3;
  for (int k = 0; k < 2; ++k)
    for (int j = 0; j < 2; ++j)
      for (int i = 0; i < 2; ++i) cube.nodes.push_back({double(i), double(j), double(k)});
  cube.elements = {{ElementKind::Hexahedron, {0, 1, 3, 2, 4, 5, 7, 6}}};
  CHECK(std::abs(signed_measure(cube, cube.elements[0]) - 1.0) < 1e-14);
  cube.elements[0].nodes = {4, 5, 7, 6, 0, 1, 3, 2};
  CHECK(count_inverted(cube) == 1);
  // test_quality.cpp:22-34: two right triangles score 90 across the hypotenuse
  Mesh tris;
  tris.dim = 2;
  tris.nodes = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}};
  tris.elements = {{ElementKind::Triangle, {0, 1, 2}}, {ElementKind::Triangle, {0, 2, 3}}};
  const QualityReport q = orthogonality(tris);
  CHECK(std::abs(q.element_orthogonality_deg[0] - 90.0) < 1e-10 &&
        std::abs(q.element_orthogonality_deg[1] - 90.0) < 1e-10 && q.inverted_count == 0);
  // mesh_io: write the triangle pair, read it back (test_mesh_io.cpp:103-124)
  {
    Mesh sq = tris;
    Marker wall;
    wall.name = "wall";
    wall.elements = {{ElementKind::Line, {0, 1}}, {ElementKind::Line, {1, 2}}};
    sq.markers = {wall};
    const std::string path = "/tmp/imb_shim_square.su2";
    write_su2(sq, path);
    const Mesh back = read_su2(path);
    CHECK(back.nodes.size() == 4 && back.nodes[2] == sq.nodes[2] && back.elements.size() == 2);
    CHECK(back.markers.size() == 1 && back.markers[0].nodes == std::vector<std::size_t>({0, 1, 2}));
    std::FILE* f = std::fopen(path.c_str(), "a");
    std::fputs("BOGUS= 1\n", f);
    std::fclose(f);
    bool parse_error = false;
    try {
      read_su2(path);
    } catch (const ParseError& e) {
      parse_error = e.line() > 0 && std::string(e.what()).find("unknown section") != std::string::npos;
    }
    CHECK(parse_error);
  }
  // vec.hpp:48-65
  CHECK(dot(Vec3{1, 2, 3}, Vec3{4, 5, 6}) == 32.0);
  CHECK(cross(Vec3{1, 0, 0}, Vec3{0, 1, 0}) == (Vec3{0, 0, 1}));
  CHECK(normalized(Vec3{3, 4, 0}) == (Vec3{0.6000000000000001, 0.8, 0}) ||
        std::abs(normalized(Vec3{3, 4, 0}).x - 0.6) < 1e-15);
  CHECK(normalized(Vec3{}) == Vec3{});
  // surface matrix KATs (test_rbf.cpp:82-94)
  CHECK(assemble_surface_matrix(two, b2) == (std::vector<double>{1.0, 0.1875, 0.1875, 1.0}));
  CHECK(assemble_surface_matrix(std::vector<Vec3>{{3.0, 4.0}}, b2) == std::vector<double>{1.0});
  CHECK(assemble_surface_matrix(std::vector<Vec3>{{0.0, 0.0}, {2.5, 0.0}}, b2) ==
        (std::vector<double>{1.0, 0.0, 0.0, 1.0}));
  // CholeskyFactor: rows appended one at a time equal a dense solve
  // (test_rbf.cpp:183-213), SolveError / invalid_argument semantics
  {
    std::mt19937 rng(31);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::vector<Vec3> pts(25);
    for (auto& p : pts) p = {u(rng), u(rng), 0.0};
    const BasisFunction b{WendlandKind::C2, 0.8};
    CholeskyFactor f;
    std::vector<double> column;
    for (std::size_t k = 0; k < pts.size(); ++k) {
      column.resize(k + 1);
      for (std::size_t j = 0; j < k; ++j) column[j] = eval_basis(b, distance(pts[j], pts[k]));
      column[k] = 1.0;
      f.append(column);
    }
    CHECK(f.size() == 25 && f.smallest_pivot() > 0.0);
    std::vector<double> rhs(25), x(25);
    for (std::size_t i = 0; i < rhs.size(); ++i) rhs[i] = std::sin(1.7 * i);
    f.solve(rhs, x);
    const std::vector<double> A = assemble_surface_matrix(pts, b);
    double worst = 0.0;
    for (std::size_t i = 0; i < 25; ++i) {
      double r = -rhs[i];
      for (std::size_t j = 0; j < 25; ++j) r += A[i * 25 + j] * x[j];
      worst = std::max(worst, std::abs(r));
    }
    CHECK(worst < 1e-10);
    bool inv = false, solve_err = false, size_err = false;
    try { f.append(std::vector<double>(3, 1.0)); } catch (const std::invalid_argument&) { inv = true; }
    CholeskyFactor g;
    g.append(std::vector<double>{1.0});
    try {
      g.append(std::vector<double>{2.0, 4.0});
    } catch (const SolveError& e) {
      solve_err = std::string(e.what()).find("not numerically positive definite at row 1") !=
                  std::string::npos;
    }
    std::vector<double> x2(2);
    try { g.solve(std::vector<double>{1.0, 2.0}, x2); } catch (const std::invalid_argument&) { size_err = true; }
    CHECK(inv && solve_err && size_err && g.size() == 1);
  }
  // the path overloads of the report writers (pipeline.hpp:59, 62)
  {
    DeformationReport rep;
    rep.marker = "airfoil";
    write_convergence_csv(rep, std::string("/tmp/imb_shim_conv.csv"));
    std::ifstream in("/tmp/imb_shim_conv.csv");
    std::string line;
    std::getline(in, line);
    CHECK(line == "level,points,error,seconds");
    bool threw_path = false;
    try {
      write_summary(rep, std::string("/nonexistent_dir/x.txt"));
    } catch (const std::runtime_error& e) {
      threw_path = std::string(e.what()) == "cannot write summary file '/nonexistent_dir/x.txt'";
    }
    CHECK(threw_path);
  }
  std::printf(failures ? "shim: %d FAILED\n" : "shim: all passed\n", failures);
  return failures ? 1 : 0;
}
