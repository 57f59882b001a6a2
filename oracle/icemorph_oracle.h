/* oracle/icemorph_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (arXiv 2107.13887 "icemorph",
 * proj/src/{rbf,greedy,wall_distance}.cpp), used as the CPU checker for the
 * CUDA product.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  It is pinned against the reference itself
 * (oracle/_ref/libicemorph_ref.so, built from /root/reference by
 * oracle/Makefile) and against the reference tests' golden values
 * (tests/golden/, tests/test_oracle.py).
 *
 * Arithmetic contract: strict IEEE binary64, no contraction (compiled with
 * -ffp-contract=off), same operation order as the reference.
 *
 * Status codes match the product C-ABI: 0 ok, 1 invalid argument,
 * 2 SolveError, 3 other.  Messages go to or_last_error().
 *
 * Vectors are AoS xyz (3 doubles per point), indices are size_t.
 */
#ifndef ICEMORPH_ORACLE_H
#define ICEMORPH_ORACLE_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* rbf.cpp:28-50 / rbf.cpp:52-54.  kind: 0=C0 1=C2 2=C4 3=C6 */
double or_eval_wendland(int kind, double eta);
double or_eval_basis(int kind, double R, double distance);

/* rbf.cpp:144-193 */
int or_solve_weights(const double* pts, const double* disp, size_t n, int kind,
                     double R, double* alpha_out);
/* rbf.cpp:195-203, batched over nq queries */
int or_eval_interpolant(const double* ctrl, const double* alpha, size_t nc, int kind,
                        double R, const double* q, size_t nq, double* out);

/* greedy.cpp:60-170; arrays sized min(cap, n) by the caller. */
/* greedy sweep threads (bit-identical to the sequential scan); default 1 */
void or_set_sweep_threads(int n);
int or_greedy_level(const double* pos, const double* target, size_t n, double tol,
                    size_t cap, int kind, double R, size_t level_index,
                    size_t* out_idx, double* out_alpha, size_t* out_nc,
                    double* out_achieved, int* out_cap_hit, double* out_target_max,
                    size_t* out_rec_points, double* out_rec_error, size_t* out_nrec,
                    double* out_residual);

/* greedy.cpp:172-195; per-level slots: max_levels, per-level arrays stride
 * min(cap, n). */
int or_run_multilevel(const double* pos, const double* target, size_t n, double tol,
                      size_t max_levels, size_t cap, int kind, double R,
                      size_t* out_nlevels, size_t* out_nc, size_t* out_idx,
                      double* out_alpha, double* out_achieved, int* out_cap_hit,
                      double* out_level_target_max, size_t* out_nrec,
                      double* out_rec_error, double* out_target_max,
                      double* out_final_residual);

/* wall_distance.cpp:13-31 — exact nearest distance (brute force; any exact
 * nearest-neighbour search yields the same value, kdtree.cpp:59-79). */
int or_build_distance_index(const double* nodes, size_t n_nodes, int dim,
                            const size_t* surface, size_t n_surface, double* out_dist,
                            int nthreads);

/* wall_distance.cpp:40-44 (psi_kind 0, linear) and the Wendland-C2 taper
 * extension (psi_kind 1). */
double or_eval_wall_function(int psi_kind, double D, double d);

/* wall_distance.cpp:46-64 with an absolute support distance D.
 * out_idx / out_val hold n_nodes entries. */
int or_update_volume(const double* nodes, size_t n_nodes, const double* dist,
                     const double* ctrl, const double* alpha, size_t nc, double D,
                     int psi_kind, int kind, double R, size_t* out_idx, double* out_val,
                     size_t* out_n, int nthreads);

/* quality.cpp:91-148: signed element measures and the inverted count
 * (measure <= 0).  kinds: mesh.hpp:15-23 order (0 Line .. 6 Pyramid), CSR. */
int or_signed_measures(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                       const size_t* offsets, const size_t* conn, size_t n_elem, double* out,
                       size_t* inverted);

/* quality.cpp:150-236 orthogonality: per-element scores (degrees) and
 * signed measures, min / mean score, inverted and degenerate counts. */
int or_orthogonality(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                     const size_t* offsets, const size_t* conn, size_t n_elem, double* out_scores,
                     double* out_measures, double* out_min, double* out_mean,
                     size_t* out_inverted, size_t* out_degenerate);

#ifdef __cplusplus
}
#endif
#endif
