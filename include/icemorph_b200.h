/* include/icemorph_b200.h — C-ABI of the B200-native RBF mesh-deformation
 * hot path (arXiv 2107.13887, reference "icemorph").
 *
 * This is the drop-in boundary: plain pointers, sizes and POD structs, no
 * C++ or torch types.  Every entry point replaces one function of the
 * reference's public C++ API (proj/include/icemorph/*.hpp) and states which.
 * Vectors are AoS x,y,z triples of doubles (the reference's Vec3 layout,
 * vec.hpp:8-12); node indices are size_t.
 *
 * Errors: C++ exceptions cannot cross a C ABI, so every call returns a
 * status and leaves the reference's exception text in im_last_error(ctx):
 *   IM_OK                0
 *   IM_INVALID_ARGUMENT  1   std::invalid_argument in the reference
 *   IM_SOLVE_ERROR       2   icemorph::SolveError (rbf.hpp:13-16)
 *   IM_RUNTIME_ERROR     3   CUDA / other runtime failures
 * The C++ shim (paper_2107_13887_b200/cpp) rethrows the same types.
 *
 * Threading: a context owns one CUDA stream and its scratch; calls on
 * different contexts may run concurrently (the reference's reentrancy,
 * SPEC.md:350).  A context must not be used by two threads at once.
 *
 * Precision (additive extension):
 *   IM_EXACT   reference arithmetic order, bit-identical results (the
 *              default of every wrapper: capi.py, the C++ shim, icemorph)
 *   IM_FP64    FMA fast path, <= 1e-10 relative to the reference on
 *              well-conditioned weights
 *   IM_FP32    the pair arithmetic in FP32 (packed FFMA2, two controls per
 *              instruction) with FP64 coordinates, per-tile FP64 sums and
 *              FP64 outputs: <= 1e-5 relative (north star's FP32 mode) on
 *              well-conditioned weights.  Volume update / interpolant only.
 * Any other precision code fails with IM_INVALID_ARGUMENT.
 */
#ifndef ICEMORPH_B200_H
#define ICEMORPH_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IM_OK 0
#define IM_INVALID_ARGUMENT 1
#define IM_SOLVE_ERROR 2
#define IM_RUNTIME_ERROR 3
#define IM_PARSE_ERROR 4 /* icemorph::ParseError (mesh_io.hpp:14-21); line: im_last_error_line */

/* WendlandKind, rbf.hpp:18 */
#define IM_C0 0
#define IM_C2 1
#define IM_C4 2
#define IM_C6 3

/* taper kind (additive): reference linear psi (wall_distance.cpp:40-44) or
 * Wendland C2 of xi (BASELINE cfg1) */
#define IM_PSI_LINEAR 0
#define IM_PSI_WENDLAND_C2 1

#define IM_EXACT 0
#define IM_FP64 1
#define IM_FP32 2

typedef struct im_context im_context;

/* BasisFunction, rbf.hpp:25-28 */
typedef struct {
  int kind;
  double support_radius;
} im_basis;

/* GreedyConfig, greedy.hpp:12-17 */
typedef struct {
  double tolerance;
  size_t max_levels;
  size_t max_points_per_level;
  im_basis basis;
} im_greedy_config;

/* WallFunction, wall_distance.hpp:26-29, plus the taper kind */
typedef struct {
  double reduction_factor;
  double support_distance;
  int psi_kind;
} im_wall_function;

/* ---- context ------------------------------------------------------------ */
int im_context_create(im_context** out, int device);
int im_context_destroy(im_context* ctx);
const char* im_last_error(const im_context* ctx);
/* device time of the last hot-path kernel sequence, milliseconds */
double im_last_device_ms(const im_context* ctx);
/* host->device / device->host bytes the last im_update_volume moved (its
 * selective upload skips node chunks without active nodes); measurement aid */
void im_last_transfer_bytes(const im_context* ctx, unsigned long long* h2d,
                            unsigned long long* d2h);
/* diagnostic: switches the exact volume kernels' pair counter on / off and
 * returns the pairs they evaluated since the previous call (culling leaves
 * more pairs evaluated than are in support; the counter slows the kernels and
 * is never on inside a timed region) */
unsigned long long im_count_pairs(im_context* ctx, int enable);
/* library build tag (sm_100a) */
const char* im_version(void);

/* ---- host scalar helpers (no device work) --------------------------------
 * eval_wendland  rbf.hpp:30 / rbf.cpp:28-50
 * eval_basis     rbf.hpp:31 / rbf.cpp:52-54
 * make_wall_function / eval_wall_function  wall_distance.hpp:31-32 */
double im_eval_wendland(int kind, double eta);
double im_eval_basis(im_basis basis, double distance);
int im_make_wall_function(double reduction_factor, double level_target_max,
                          im_wall_function* out);
double im_eval_wall_function(const im_wall_function* wf, double wall_distance);

/* ---- rbf ------------------------------------------------------------------
 * solve_weights, rbf.hpp:74-76 (rbf.cpp:144-193).  alpha_out: 3n doubles. */
int im_solve_weights(im_context* ctx, const double* points, const double* displacements,
                     size_t n, im_basis basis, double* alpha_out);

/* assemble_surface_matrix, rbf.hpp:35-36 (rbf.cpp:56-69): the dense kernel
 * matrix phi(|r_i - r_j|) with unit diagonal, row-major n*n doubles in out. */
int im_assemble_surface_matrix(im_context* ctx, const double* points, size_t n, im_basis basis,
                               double* out);

/* CholeskyFactor, rbf.hpp:41-60 (rbf.cpp:71-121): a factor that grows one
 * row at a time, resident on the device (column-major packed, capacity
 * doubling).  append: column = the new row's entries against the existing
 * points followed by the diagonal entry, length size()+1; IM_INVALID_ARGUMENT
 * "column length must be current size + 1", IM_SOLVE_ERROR "matrix not
 * numerically positive definite at row k (pivot p)" when the pivot is not
 * above 1e-14 of the largest diagonal seen (the factor is then unchanged, as
 * in the reference).  solve: A x = rhs, rhs and x of length size(),
 * IM_INVALID_ARGUMENT "rhs size does not match factorization" otherwise.
 * Errors are read with im_last_error(ctx) of the creating context. */
typedef struct im_cholesky im_cholesky;
int im_cholesky_create(im_context* ctx, im_cholesky** out);
int im_cholesky_destroy(im_cholesky* factor);
size_t im_cholesky_size(const im_cholesky* factor);
double im_cholesky_smallest_pivot(const im_cholesky* factor);
int im_cholesky_append(im_cholesky* factor, const double* column, size_t length);
int im_cholesky_solve(const im_cholesky* factor, const double* rhs, size_t rhs_length, double* x,
                      size_t x_length);

/* eval_interpolant, rbf.hpp:80-81 (rbf.cpp:195-203), batched over n_query
 * queries.  out: 3 n_query doubles. */
int im_eval_interpolant(im_context* ctx, const double* control_positions, const double* alpha,
                        size_t n_control, im_basis basis, const double* queries,
                        size_t n_query, int precision, double* out);

/* ---- greedy -----------------------------------------------------------------
 * greedy_level, greedy.hpp:51-54 (greedy.cpp:60-170).  Always exact.
 * Let m = min(max_points_per_level, n).  Caller buffers:
 *   control_indices[m], alpha[3m], record_points[m], record_error[m],
 *   record_seconds[m] (may be NULL), residual[3n] (may be NULL). */
int im_greedy_level(im_context* ctx, const double* surface_positions, const double* target,
                    size_t n, const im_greedy_config* config, size_t level_index,
                    size_t* control_indices, double* alpha, size_t* n_controls,
                    double* achieved_error, int* cap_hit, double* target_max,
                    double* elapsed_seconds, size_t* record_points, double* record_error,
                    double* record_seconds, size_t* n_records, double* residual);

/* run_multilevel, greedy.hpp:66-68 (greedy.cpp:172-195).  Level l's arrays
 * start at offset l*m (m as above); per-level scalars have max_levels slots. */
int im_run_multilevel(im_context* ctx, const double* surface_positions, const double* target,
                      size_t n, const im_greedy_config* config, size_t* n_levels,
                      size_t* n_controls, size_t* control_indices, double* alpha,
                      double* achieved_error, int* cap_hit, double* level_target_max,
                      double* elapsed_seconds, size_t* n_records, double* record_error,
                      double* target_max, double* final_residual);

/* ---- wall distance / volume reduction -----------------------------------------
 * build_distance_index, wall_distance.hpp:20-22 (wall_distance.cpp:13-31).
 * nodes: 3 n_nodes doubles; distances_out: n_nodes doubles. */
int im_build_distance_index(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
                            const size_t* surface_nodes, size_t n_surface,
                            double* distances_out);

/* update_volume, wall_distance.hpp:40-42 (wall_distance.cpp:46-64).
 * entry_nodes[n_nodes] / entry_values[3 n_nodes] receive the ascending
 * sparse update; *n_entries its length. */
int im_update_volume(im_context* ctx, const double* nodes, size_t n_nodes,
                     const double* distances, const double* control_positions,
                     const double* alpha, size_t n_control, const im_wall_function* wf,
                     im_basis basis, int precision, size_t* entry_nodes,
                     double* entry_values, size_t* n_entries);

/* ---- element quality (the part deform reads) ----------------------------------
 * signed_measures / count_inverted, quality.hpp (quality.cpp:100-148) on a
 * mesh given as its node array (3 n_nodes doubles) and its volume elements in
 * CSR form: element_kinds[n_elements] in ElementKind order (mesh.hpp:15-23:
 * 0 line, 1 triangle, 2 quadrilateral, 3 tetrahedron, 4 hexahedron, 5 prism,
 * 6 pyramid), element_offsets[n_elements + 1] (starting at 0) and
 * element_nodes[element_offsets[n_elements]].  measures (nullable) receives
 * n_elements doubles, *inverted (nullable) the count of measure <= 0.
 * Malformed elements raise IM_INVALID_ARGUMENT with validate_mesh's message
 * (mesh.cpp:168-185). */
int im_signed_measures(im_context* ctx, const double* nodes, size_t n_nodes,
                       const int* element_kinds, const size_t* element_offsets,
                       const size_t* element_nodes, size_t n_elements, double* measures,
                       size_t* inverted);
/* count_inverted, quality.hpp (quality.cpp:142-148). */
int im_count_inverted(im_context* ctx, const double* nodes, size_t n_nodes,
                      const int* element_kinds, const size_t* element_offsets,
                      const size_t* element_nodes, size_t n_elements, size_t* inverted);

/* orthogonality, quality.hpp (quality.cpp:150-236): per-element scores in
 * degrees (nullable, n_elements doubles) and signed measures (nullable), the
 * report scalars in *report.  Faces are matched on the device (sorted node
 * keys, radix sort) instead of the reference's std::map; scores agree with
 * the reference to ~1e-13 degrees (CUDA atan2), measures and counts exactly. */
typedef struct {
  double min_orthogonality_deg;
  double mean_orthogonality_deg;
  size_t inverted_count;
  size_t degenerate_count;
} im_quality_report;
int im_orthogonality(im_context* ctx, const double* nodes, size_t n_nodes,
                     const int* element_kinds, const size_t* element_offsets,
                     const size_t* element_nodes, size_t n_elements, double* element_scores,
                     double* element_measures, im_quality_report* report);

/* ---- SU2 mesh I/O (mesh_io.hpp:39-43, mesh_io.cpp:127-309) -------------------
 * im_su2_read parses a SU2 ASCII mesh (NDIME / NPOIN / NELEM / NMARK, any
 * order, '%' comments) into an opaque host mesh with the reference's grammar,
 * validation and "path:line: what" errors (IM_PARSE_ERROR; the line via
 * im_last_error_line), including the coincident-node check (on the device).
 * Accessors copy the arrays out; element kinds are ElementKind ids
 * (mesh.hpp:15-23).  im_su2_write writes the reference's layout (NDIME, NELEM,
 * NPOIN with %.17g coordinates, NMARK). */
typedef struct im_mesh im_mesh;
int im_su2_read(im_context* ctx, const char* path, im_mesh** out);
int im_mesh_destroy(im_mesh* mesh);
int im_mesh_sizes(const im_mesh* mesh, int* dim, size_t* n_nodes, size_t* n_elements,
                  size_t* n_element_nodes, size_t* n_markers);
int im_mesh_nodes(const im_mesh* mesh, double* xyz);
int im_mesh_elements(const im_mesh* mesh, int* kinds, size_t* offsets, size_t* nodes);
int im_mesh_marker_sizes(const im_mesh* mesh, size_t marker, size_t* name_length,
                         size_t* n_elements, size_t* n_element_nodes, size_t* n_nodes);
int im_mesh_marker(const im_mesh* mesh, size_t marker, char* name, int* kinds, size_t* offsets,
                   size_t* element_nodes, size_t* nodes);
size_t im_last_error_line(const im_context* ctx);
int im_su2_write(im_context* ctx, const char* path, int dim, const double* xyz, size_t n_nodes,
                 const int* kinds, const size_t* offsets, const size_t* nodes, size_t n_elements,
                 size_t n_markers, const char* const* marker_names, const int* const* marker_kinds,
                 const size_t* const* marker_offsets, const size_t* const* marker_element_nodes,
                 const size_t* marker_n_elements);

/* ---- pipeline -----------------------------------------------------------------
 * deform, pipeline.hpp:54-56 (pipeline.cpp:19-106) on a mesh given as its
 * node array and the node lists of the deforming patch and of the pinned
 * markers (the hot path reads nothing else of Mesh).
 * displacement: 3 n_patch doubles, one per patch node (DisplacementField::at).
 * support_distance < 0 selects the reference D_l = volume_k * target_max_l
 * (pipeline.cpp:66); >= 0 (inf allowed) is an absolute D (additive).
 * deformed_nodes: 3 n_nodes doubles.  Per-level outputs have max_levels
 * slots.  When the config carries the mesh's volume elements (CSR as for
 * im_signed_measures; n_elements = 0 for none) the report's
 * inverted_elements is count_inverted(deformed) (pipeline.cpp:101),
 * evaluated on the device-resident deformed nodes; with compute_quality the
 * orthogonality reports of the mesh before and after (has_quality = 1). */
typedef struct {
  im_greedy_config greedy;
  double volume_k;
  double support_distance;
  int psi_kind;
  int precision;
  const int* element_kinds;
  const size_t* element_offsets;
  const size_t* element_nodes;
  size_t n_elements;
  int compute_quality; /* with elements: quality_before / quality_after (pipeline.cpp:55, 102) */
  /* optional (NULL: not returned): each level's ConvergenceRecord
   * (LevelSummary::record, pipeline.cpp:83), level l's samples at offset
   * l * record_stride (record_stride >= min(max_points_per_level, patch +
   * pinned nodes)); sample count = level_points[l] */
  double* record_error;
  double* record_seconds;
  size_t record_stride;
} im_deform_config;

typedef struct {
  size_t n_levels;
  double target_max;
  double surface_max_error;
  double surface_mean_error;
  double total_seconds;
  double greedy_seconds;
  double distance_seconds;
  double volume_seconds;
  size_t inverted_elements;
  int has_quality;
  im_quality_report quality_before;
  im_quality_report quality_after;
} im_deform_report;

int im_deform(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
              const size_t* patch_nodes, size_t n_patch, const double* displacement,
              const size_t* pinned_nodes, size_t n_pinned, const im_deform_config* config,
              double* deformed_nodes, im_deform_report* report, size_t* level_points,
              double* level_achieved, int* level_cap_hit, double* level_support_distance,
              size_t* level_touched, double* level_seconds);

/* ---- resident plans (inputs kept in HBM between calls) ------------------------
 * A volume plan uploads the mesh nodes once and computes the wall distances
 * on the device; im_volume_plan_run then performs the culling + compaction
 * + volume update for one level entirely on the device and accumulates the
 * update into the plan's resident displacement field.  cutoff: +inf for exact
 * distances at every node, a finite value to cull beyond it (nodes farther
 * get +inf), < 0 to skip the distance pass (D = inf workloads, psi == 1). */
typedef struct im_volume_plan im_volume_plan;
int im_volume_plan_create(im_context* ctx, const double* nodes, size_t n_nodes, int dim,
                          const size_t* surface_nodes, size_t n_surface, double cutoff,
                          im_volume_plan** out);
int im_volume_plan_destroy(im_volume_plan* plan);
int im_volume_plan_set_controls(im_volume_plan* plan, const double* control_positions,
                                const double* alpha, size_t n_control);
/* one level: compaction at D + update over the active set, accumulated into
 * the resident field; returns the active count; device ms in *device_ms */
int im_volume_plan_run(im_volume_plan* plan, const im_wall_function* wf, im_basis basis,
                       int precision, size_t* n_active, double* device_ms);
int im_volume_plan_reset_field(im_volume_plan* plan);
int im_volume_plan_download_field(im_volume_plan* plan, double* out_xyz);
int im_volume_plan_distances(im_volume_plan* plan, double* out);
/* multi-level steps for the benchmark: level l's packed control set, support
 * distance and taper; run_steps executes `steps` passes over every level
 * (compaction + update), each bracketed by CUDA events, optional L2 flush
 * before each pass outside the brackets.  stats: see pipeline.cu. */
int im_volume_plan_set_level(im_volume_plan* plan, int level, const double* control_positions,
                             const double* alpha, size_t n_control, double support_distance,
                             int psi_kind, im_basis basis, int precision);
int im_volume_plan_run_steps(im_volume_plan* plan, im_basis basis, int precision, int steps,
                             int flush_l2, double* stats);
int im_volume_plan_count_support(im_volume_plan* plan, int level, im_basis basis,
                                 unsigned long long* in_support, unsigned long long* total);

/* The HBM-bound passes on the plan's resident mesh (benchmark): the wall
 * distance with `cutoff` (into scratch) and the compaction of d < D, each
 * timed over `reps` passes.  stats (4 doubles): wall-distance ms per pass,
 * compaction ms per pass, active count at D, nodes within the cutoff. */
int im_volume_plan_bench_passes(im_volume_plan* plan, double cutoff, double D, int reps,
                                double* stats);

/* ---- diagnostics ---------------------------------------------------------------
 * Time the exact backward-substitution chain (rbf.cpp:114-120, 3 axes) of
 * size n on a synthetic factor: ms per solve, for the latency roofline. */
int im_bench_backward_chain(im_context* ctx, int n, int reps, double* ms_per_solve);

#ifdef __cplusplus
}
#endif
#endif /* ICEMORPH_B200_H */
