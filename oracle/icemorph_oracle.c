/* oracle/icemorph_oracle.c — TEST INFRASTRUCTURE ONLY (see icemorph_oracle.h).
 *
 * CPU restatement of the reference hot path, each function citing the
 * reference file:line it follows.  Compiled with -ffp-contract=off so every
 * + - * / sqrt rounds exactly as the reference build does.
 */
#define _GNU_SOURCE
#include "icemorph_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[1024];

const char* or_last_error(void) { return g_err; }

static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* vec.hpp:35-36, 56-60: s = (dx*dx + dy*dy) + dz*dz, d = sqrt(s). */
static double norm3(double x, double y, double z) { return sqrt(x * x + y * y + z * z); }

static double dist3(const double* a, const double* b) {
  return norm3(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
}

/* rbf.cpp:28-50 */
double or_eval_wendland(int kind, double eta) {
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

/* rbf.cpp:52-54 */
double or_eval_basis(int kind, double R, double distance) {
  return or_eval_wendland(kind, distance / R);
}

/* ---- incremental Cholesky, rbf.cpp:71-121 (packed row-major lower) ---- */
typedef struct {
  size_t n, cap;
  double* lower;
  double max_diag, smallest_pivot;
} chol_t;

static int chol_init(chol_t* f, size_t cap) {
  f->n = 0;
  f->cap = cap;
  f->max_diag = 0.0;
  f->smallest_pivot = 0.0;
  f->lower = (double*)malloc(sizeof(double) * (cap * (cap + 1) / 2 + 1));
  return f->lower ? 0 : 3;
}

static void chol_free(chol_t* f) { free(f->lower); }

/* rbf.cpp:71-100.  Returns 0, or 2 with the reference message. */
static int chol_append(chol_t* f, const double* column) {
  const size_t k = f->n;
  double* row = f->lower + k * (k + 1) / 2;
  double sq = 0.0;
  for (size_t j = 0; j < k; ++j) {
    const double* lj = f->lower + j * (j + 1) / 2;
    double s = column[j];
    for (size_t m = 0; m < j; ++m) s -= lj[m] * row[m];
    row[j] = s / lj[j];
    sq += row[j] * row[j];
  }
  const double diag = column[k];
  if (diag > f->max_diag) f->max_diag = diag; /* std::max(max_diag_, diag) */
  const double pivot_sq = diag - sq;
  const double pivot = pivot_sq > 0.0 ? sqrt(pivot_sq) : 0.0;
  if (!(pivot > 1e-14 * f->max_diag)) {
    snprintf(g_err, sizeof g_err,
             "matrix not numerically positive definite at row %zu (pivot %f)", k, pivot);
    return 2;
  }
  row[k] = pivot;
  if (f->n == 0 || pivot < f->smallest_pivot) f->smallest_pivot = pivot;
  ++f->n;
  return 0;
}

/* rbf.cpp:102-121 */
static void chol_solve(const chol_t* f, const double* rhs, double* x) {
  const size_t n = f->n;
  for (size_t i = 0; i < n; ++i) {
    const double* li = f->lower + i * (i + 1) / 2;
    double s = rhs[i];
    for (size_t j = 0; j < i; ++j) s -= li[j] * x[j];
    x[i] = s / li[i];
  }
  for (size_t i = n; i-- > 0;) {
    double s = x[i];
    for (size_t j = i + 1; j < n; ++j) s -= f->lower[j * (j + 1) / 2 + i] * x[j];
    x[i] = s / f->lower[i * (i + 1) / 2 + i];
  }
}

/* rbf.cpp:125-140 */
static int rethrow_conditioning(const double* pts, size_t failed) {
  size_t nearest = 0;
  double best = INFINITY;
  for (size_t i = 0; i < failed; ++i) {
    const double d = dist3(pts + 3 * i, pts + 3 * failed);
    if (d < best) {
      best = d;
      nearest = i;
    }
  }
  snprintf(g_err, sizeof g_err,
           "ill-conditioned control set: points %zu and %zu are too close (distance %f)",
           nearest, failed, best);
  return 2;
}

/* rbf.cpp:144-193 */
int or_solve_weights(const double* pts, const double* disp, size_t n, int kind,
                     double R, double* alpha_out) {
  memset(alpha_out, 0, sizeof(double) * 3 * n);
  if (n == 0) return 0;
  int all_zero = 1;
  for (size_t i = 0; i < 3 * n; ++i)
    if (disp[i] != 0.0) {
      all_zero = 0;
      break;
    }
  if (all_zero) return 0;
  chol_t f;
  if (chol_init(&f, n)) return set_err(3, "out of memory");
  double* column = (double*)malloc(sizeof(double) * (n + 1));
  double* rhs = (double*)malloc(sizeof(double) * n);
  double* sol = (double*)malloc(sizeof(double) * n);
  int rc = 0;
  for (size_t k = 0; k < n && rc == 0; ++k) {
    for (size_t j = 0; j < k; ++j)
      column[j] = or_eval_basis(kind, R, dist3(pts + 3 * j, pts + 3 * k));
    column[k] = 1.0;
    if (chol_append(&f, column)) rc = rethrow_conditioning(pts, k);
  }
  if (rc == 0) {
    for (int axis = 0; axis < 3; ++axis) {
      for (size_t i = 0; i < n; ++i) rhs[i] = disp[3 * i + axis];
      chol_solve(&f, rhs, sol);
      for (size_t i = 0; i < n; ++i) alpha_out[3 * i + axis] = sol[i];
    }
  }
  free(column);
  free(rhs);
  free(sol);
  chol_free(&f);
  return rc;
}

/* rbf.cpp:195-203 */
static void interp1(const double* ctrl, const double* alpha, size_t nc, int kind, double R,
                    const double* q, double* out) {
  double rx = 0.0, ry = 0.0, rz = 0.0;
  for (size_t i = 0; i < nc; ++i) {
    const double phi = or_eval_basis(kind, R, dist3(ctrl + 3 * i, q));
    if (phi != 0.0) {
      rx += alpha[3 * i] * phi;
      ry += alpha[3 * i + 1] * phi;
      rz += alpha[3 * i + 2] * phi;
    }
  }
  out[0] = rx;
  out[1] = ry;
  out[2] = rz;
}

int or_eval_interpolant(const double* ctrl, const double* alpha, size_t nc, int kind,
                        double R, const double* q, size_t nq, double* out) {
  for (size_t i = 0; i < nq; ++i) interp1(ctrl, alpha, nc, kind, R, q + 3 * i, out + 3 * i);
  return 0;
}

/* greedy.cpp:20-33 */
static int check_config(double tol, size_t max_levels, size_t cap, double R) {
  if (!(tol > 0.0 && tol < 1.0)) return set_err(1, "greedy tolerance must lie in (0,1)");
  if (max_levels < 1) return set_err(1, "at least one level is required");
  if (cap < 1) return set_err(1, "per-level point cap must be positive");
  if (!(R > 0.0)) return set_err(1, "basis support radius must be positive");
  return 0;
}

/* greedy.cpp:35-39 */
static double max_magnitude(const double* v, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double x = norm3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    m = (m < x) ? x : m; /* std::max(m, x) */
  }
  return m;
}

/* greedy.cpp:41-56 */
static int rethrow_conditioning_nodes(const double* pos, const size_t* controls, size_t nc,
                                      size_t failed) {
  size_t nearest = failed;
  double best = INFINITY;
  for (size_t m = 0; m < nc; ++m) {
    const double d = dist3(pos + 3 * controls[m], pos + 3 * failed);
    if (d < best) {
      best = d;
      nearest = controls[m];
    }
  }
  snprintf(g_err, sizeof g_err,
           "ill-conditioned control set: surface nodes %zu and %zu are too close "
           "(distance %f)",
           nearest, failed, best);
  return 2;
}

/* Threads for the greedy sweep (greedy.cpp:122-143).  The sweep is
 * independent per surface node; each thread scans a contiguous node range
 * with the reference's strict '>' and the ranges merge in ascending order
 * with the same rule, so argmax (lowest index on ties) and the overall max
 * equal the sequential scan bit for bit.  Used to make full-size 3-D
 * fixtures in reasonable time; 1 (default) is the plain sequential loop. */
static int g_sweep_threads = 1;
void or_set_sweep_threads(int n) { g_sweep_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }

typedef struct {
  const double *pos, *target, *alpha;
  const size_t* controls;
  const char* selected;
  size_t nc, lo, hi;
  int kind;
  double R;
  double* residual;
  double max_norm, overall;
  size_t argmax;
} sweep_job;

static void* sweep_work(void* p) {
  sweep_job* j = (sweep_job*)p;
  const double* pos = j->pos;
  double max_norm = -1.0, overall = 0.0;
  size_t argmax = (size_t)-1;
  for (size_t i = j->lo; i < j->hi; ++i) {
    double fx = 0.0, fy = 0.0, fz = 0.0;
    for (size_t m = 0; m < j->nc; ++m) {
      const double phi =
          or_eval_basis(j->kind, j->R, dist3(pos + 3 * i, pos + 3 * j->controls[m]));
      if (phi != 0.0) {
        fx += j->alpha[3 * m] * phi;
        fy += j->alpha[3 * m + 1] * phi;
        fz += j->alpha[3 * m + 2] * phi;
      }
    }
    double* r = j->residual + 3 * i;
    r[0] = j->target[3 * i] - fx;
    r[1] = j->target[3 * i + 1] - fy;
    r[2] = j->target[3 * i + 2] - fz;
    const double nrm = norm3(r[0], r[1], r[2]);
    if (!j->selected[i] && nrm > max_norm) {
      max_norm = nrm;
      argmax = i;
    }
    overall = (overall < nrm) ? nrm : overall;
  }
  j->max_norm = max_norm, j->overall = overall, j->argmax = argmax;
  return NULL;
}

/* greedy.cpp:60-170 */
int or_greedy_level(const double* pos, const double* target, size_t n, double tol,
                    size_t cap_cfg, int kind, double R, size_t level_index,
                    size_t* out_idx, double* out_alpha, size_t* out_nc,
                    double* out_achieved, int* out_cap_hit, double* out_target_max,
                    size_t* out_rec_points, double* out_rec_error, size_t* out_nrec,
                    double* out_residual) {
  (void)level_index;
  int rc = check_config(tol, 1, cap_cfg, R);
  if (rc) return rc;
  if (n == 0) return set_err(1, "surface point set is empty");
  for (size_t i = 0; i < 3 * n; ++i)
    if (!isfinite(target[i])) return set_err(1, "target displacement is not finite");

  const double target_max = max_magnitude(target, n);
  const size_t cap = cap_cfg < n ? cap_cfg : n;
  size_t nc = 0, nrec = 0;
  size_t* controls = out_idx;
  char* selected = (char*)calloc(n, 1);
  double* alpha = out_alpha;
  double* column = (double*)malloc(sizeof(double) * (cap + 1));
  double* rhs = (double*)malloc(sizeof(double) * cap);
  double* sol = (double*)malloc(sizeof(double) * cap);
  double* residual = out_residual ? out_residual : (double*)malloc(sizeof(double) * 3 * n);
  chol_t f;
  if (chol_init(&f, cap)) return set_err(3, "out of memory");

  size_t node = 0; /* greedy.cpp:115 — seed with the first surface node */
  double achieved = 0.0;
  int cap_hit = 0;
  for (;;) {
    /* insert_control(node), greedy.cpp:86-112 */
    for (size_t m = 0; m < nc; ++m)
      column[m] = or_eval_basis(kind, R, dist3(pos + 3 * controls[m], pos + 3 * node));
    column[nc] = 1.0;
    if (chol_append(&f, column)) {
      rc = rethrow_conditioning_nodes(pos, controls, nc, node);
      break;
    }
    controls[nc++] = node;
    selected[node] = 1;
    for (int axis = 0; axis < 3; ++axis) {
      for (size_t m = 0; m < nc; ++m) rhs[m] = target[3 * controls[m] + axis];
      chol_solve(&f, rhs, sol);
      for (size_t m = 0; m < nc; ++m) alpha[3 * m + axis] = sol[m];
    }

    /* sweep, greedy.cpp:122-143 */
    double max_norm = -1.0;
    size_t argmax = n;
    double overall = 0.0;
    if (g_sweep_threads > 1 && n >= 1024) {
      const int nt = g_sweep_threads;
      pthread_t th[256];
      sweep_job jobs[256];
      for (int t = 0; t < nt; ++t) {
        jobs[t] = (sweep_job){pos, target, alpha, controls, selected, nc, n * t / nt,
                              n * (t + 1) / nt, kind, R, residual, 0.0, 0.0, 0};
        pthread_create(&th[t], NULL, sweep_work, &jobs[t]);
      }
      for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
      for (int t = 0; t < nt; ++t) { /* ascending ranges, strict '>' */
        if (jobs[t].argmax != (size_t)-1 && jobs[t].max_norm > max_norm) {
          max_norm = jobs[t].max_norm;
          argmax = jobs[t].argmax;
        }
        overall = (overall < jobs[t].overall) ? jobs[t].overall : overall;
      }
      goto swept;
    }
    for (size_t i = 0; i < n; ++i) {
      double fx = 0.0, fy = 0.0, fz = 0.0;
      for (size_t m = 0; m < nc; ++m) {
        const double phi = or_eval_basis(kind, R, dist3(pos + 3 * i, pos + 3 * controls[m]));
        if (phi != 0.0) {
          fx += alpha[3 * m] * phi;
          fy += alpha[3 * m + 1] * phi;
          fz += alpha[3 * m + 2] * phi;
        }
      }
      residual[3 * i] = target[3 * i] - fx;
      residual[3 * i + 1] = target[3 * i + 1] - fy;
      residual[3 * i + 2] = target[3 * i + 2] - fz;
      const double nrm = norm3(residual[3 * i], residual[3 * i + 1], residual[3 * i + 2]);
      if (!selected[i] && nrm > max_norm) {
        max_norm = nrm;
        argmax = i;
      }
    }
    for (size_t i = 0; i < n; ++i) {
      const double e = norm3(residual[3 * i], residual[3 * i + 1], residual[3 * i + 2]);
      overall = (overall < e) ? e : overall; /* std::max */
    }
  swept:
    achieved = target_max > 0.0 ? overall / target_max : 0.0;
    if (out_rec_points) out_rec_points[nrec] = nc;
    if (out_rec_error) out_rec_error[nrec] = achieved;
    ++nrec;
    /* greedy.cpp:146-152 */
    if (achieved < tol) break;
    if (nc >= cap || argmax == n) {
      cap_hit = 1;
      break;
    }
    node = argmax;
  }
  *out_nc = nc;
  *out_achieved = achieved;
  *out_cap_hit = cap_hit;
  *out_target_max = target_max;
  if (out_nrec) *out_nrec = nrec;
  if (!out_residual) free(residual);
  free(selected);
  free(column);
  free(rhs);
  free(sol);
  chol_free(&f);
  return rc;
}

/* greedy.cpp:172-195 */
int or_run_multilevel(const double* pos, const double* target, size_t n, double tol,
                      size_t max_levels, size_t cap, int kind, double R,
                      size_t* out_nlevels, size_t* out_nc, size_t* out_idx,
                      double* out_alpha, double* out_achieved, int* out_cap_hit,
                      double* out_level_target_max, size_t* out_nrec,
                      double* out_rec_error, double* out_target_max,
                      double* out_final_residual) {
  int rc = check_config(tol, max_levels, cap, R);
  if (rc) return rc;
  const double target_max = max_magnitude(target, n);
  *out_target_max = target_max;
  const size_t stride = cap < n ? cap : n;
  double* current = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
  double* next = (double*)malloc(sizeof(double) * 3 * (n ? n : 1));
  memcpy(current, target, sizeof(double) * 3 * n);
  const double entry_threshold = pow(tol, (double)max_levels) * target_max;
  size_t nl = 0;
  for (size_t l = 0; l < max_levels; ++l) {
    const double current_max = max_magnitude(current, n);
    if (l > 0 && (current_max == 0.0 || current_max < entry_threshold)) break;
    rc = or_greedy_level(pos, current, n, tol, cap, kind, R, l, out_idx + l * stride,
                         out_alpha + 3 * l * stride, out_nc + l, out_achieved + l,
                         out_cap_hit + l, out_level_target_max + l, NULL,
                         out_rec_error ? out_rec_error + l * stride : NULL, out_nrec + l,
                         next);
    if (rc) break;
    double* t = current;
    current = next;
    next = t;
    ++nl;
  }
  *out_nlevels = nl;
  if (rc == 0 && out_final_residual) memcpy(out_final_residual, current, sizeof(double) * 3 * n);
  free(current);
  free(next);
  return rc;
}

/* ---- wall distance, wall_distance.cpp:13-31 ---- */
typedef struct {
  const double* nodes;
  size_t lo, hi;
  const double* surf;
  size_t ns;
  double* out;
} nn_job;

static void* nn_work(void* p) {
  nn_job* j = (nn_job*)p;
  for (size_t i = j->lo; i < j->hi; ++i) {
    const double* q = j->nodes + 3 * i;
    double best = INFINITY;
    for (size_t s = 0; s < j->ns; ++s) {
      const double* a = j->surf + 3 * s;
      const double dx = a[0] - q[0], dy = a[1] - q[1], dz = a[2] - q[2];
      const double d2 = dx * dx + dy * dy + dz * dz; /* squared_distance, vec.hpp:59 */
      if (d2 < best) best = d2;
    }
    j->out[i] = sqrt(best); /* kdtree.cpp:79 */
  }
  return NULL;
}

int or_build_distance_index(const double* nodes, size_t n_nodes, int dim,
                            const size_t* surface, size_t n_surface, double* out_dist,
                            int nthreads) {
  if (n_surface == 0)
    return set_err(1, "cannot build a distance index for an empty patch");
  if (dim != 2 && dim != 3) return set_err(1, "kd-tree dim must be 2 or 3");
  double* surf = (double*)malloc(sizeof(double) * 3 * n_surface);
  for (size_t s = 0; s < n_surface; ++s) memcpy(surf + 3 * s, nodes + 3 * surface[s], 24);
  if (nthreads < 1) nthreads = 1;
  pthread_t th[256];
  nn_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (nn_job){nodes, n_nodes * t / nthreads, n_nodes * (t + 1) / nthreads, surf,
                       n_surface, out_dist};
    if (nthreads > 1)
      pthread_create(&th[t], NULL, nn_work, &jobs[t]);
    else
      nn_work(&jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  for (size_t s = 0; s < n_surface; ++s) out_dist[surface[s]] = 0.0; /* :29 */
  free(surf);
  return 0;
}

/* wall_distance.cpp:40-44; psi_kind 1 swaps in eval_wendland(C2, xi). */
double or_eval_wall_function(int psi_kind, double D, double d) {
  if (D <= 0.0) return d == 0.0 ? 1.0 : 0.0;
  const double xi = d / D;
  if (psi_kind == 1) return or_eval_wendland(1, xi);
  return xi < 1.0 ? 1.0 - xi : 0.0;
}

/* wall_distance.cpp:46-64 */
typedef struct {
  const double *nodes, *dist, *ctrl, *alpha;
  size_t nc, lo, hi;
  double D, R;
  int psi_kind, kind;
  size_t* idx;
  double* val;
  size_t count;
} vu_job;

static void* vu_work(void* p) {
  vu_job* j = (vu_job*)p;
  size_t k = 0;
  for (size_t i = j->lo; i < j->hi; ++i) {
    const double d = j->dist[i];
    if (d >= j->D) continue;
    const double psi = or_eval_wall_function(j->psi_kind, j->D, d);
    double v[3];
    interp1(j->ctrl, j->alpha, j->nc, j->kind, j->R, j->nodes + 3 * i, v);
    j->idx[k] = i;
    j->val[3 * k] = v[0] * psi;
    j->val[3 * k + 1] = v[1] * psi;
    j->val[3 * k + 2] = v[2] * psi;
    ++k;
  }
  j->count = k;
  return NULL;
}

int or_update_volume(const double* nodes, size_t n_nodes, const double* dist,
                     const double* ctrl, const double* alpha, size_t nc, double D,
                     int psi_kind, int kind, double R, size_t* out_idx, double* out_val,
                     size_t* out_n, int nthreads) {
  *out_n = 0;
  if (D <= 0.0) return 0; /* wall_distance.cpp:54 */
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  vu_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    const size_t lo = n_nodes * t / nthreads, hi = n_nodes * (t + 1) / nthreads;
    jobs[t] = (vu_job){nodes, dist, ctrl, alpha, nc, lo, hi, D, R, psi_kind, kind,
                       out_idx + lo, out_val + 3 * lo, 0};
    if (nthreads > 1)
      pthread_create(&th[t], NULL, vu_work, &jobs[t]);
    else
      vu_work(&jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  /* compact the per-slice outputs in slice (= ascending node) order */
  size_t k = 0;
  for (int t = 0; t < nthreads; ++t) {
    memmove(out_idx + k, jobs[t].idx, sizeof(size_t) * jobs[t].count);
    memmove(out_val + 3 * k, jobs[t].val, sizeof(double) * 3 * jobs[t].count);
    k += jobs[t].count;
  }
  *out_n = k;
  return 0;
}

/* ---- quality.cpp:91-148 ---------------------------------------------------- */
/* quality.cpp:91-93: dot(b - a, cross(c - a, d - a)) / 6, vec.hpp:51-55 order */
static double tet_volume(const double* a, const double* b, const double* c, const double* d) {
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double cx = v[1] * w[2] - v[2] * w[1];
  const double cy = v[2] * w[0] - v[0] * w[2];
  const double cz = v[0] * w[1] - v[1] * w[0];
  return (u[0] * cx + u[1] * cy + u[2] * cz) / 6.0;
}

/* quality.cpp:95-97 */
static double tri_area(const double* a, const double* b, const double* c) {
  return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
}

/* quality.cpp:101-133 */
static double signed_measure(const double* nd, int kind, const size_t* n) {
#define P(i) (nd + 3 * n[i])
  switch (kind) {
    case 1: return tri_area(P(0), P(1), P(2));
    case 2: return tri_area(P(0), P(1), P(2)) + tri_area(P(0), P(2), P(3));
    case 3: return tet_volume(P(0), P(1), P(2), P(3));
    case 4: {
      double v = 0.0;
      v += tet_volume(P(0), P(1), P(2), P(6));
      v += tet_volume(P(0), P(2), P(3), P(6));
      v += tet_volume(P(0), P(3), P(7), P(6));
      v += tet_volume(P(0), P(7), P(4), P(6));
      v += tet_volume(P(0), P(4), P(5), P(6));
      v += tet_volume(P(0), P(5), P(1), P(6));
      return v;
    }
    case 5:
      return tet_volume(P(0), P(1), P(2), P(3)) + tet_volume(P(1), P(2), P(3), P(4)) +
             tet_volume(P(2), P(3), P(4), P(5));
    case 6: return tet_volume(P(0), P(1), P(2), P(4)) + tet_volume(P(0), P(2), P(3), P(4));
    default: return 0.0; /* Line */
  }
#undef P
}

int or_signed_measures(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                       const size_t* offsets, const size_t* conn, size_t n_elem, double* out,
                       size_t* inverted) {
  (void)n_nodes;
  (void)dim;
  size_t count = 0;
  for (size_t e = 0; e < n_elem; ++e) {
    out[e] = signed_measure(nodes, kinds[e], conn + offsets[e]);
    if (out[e] <= 0.0) ++count; /* quality.cpp:145 */
  }
  *inverted = count;
  return 0;
}

/* ---- quality.cpp:150-236 (orthogonality) ------------------------------------ */
/* element_faces, quality.cpp:19-49: local node lists per kind */
static const int kFaceCount[7] = {0, 3, 4, 4, 6, 5, 5};
static const int kFaceNodes[7][6][5] = {
    /* count, nodes... */
    {{0}},
    {{2, 0, 1}, {2, 1, 2}, {2, 2, 0}},
    {{2, 0, 1}, {2, 1, 2}, {2, 2, 3}, {2, 3, 0}},
    {{3, 0, 1, 2}, {3, 0, 1, 3}, {3, 1, 2, 3}, {3, 0, 2, 3}},
    {{4, 0, 1, 2, 3}, {4, 4, 5, 6, 7}, {4, 0, 1, 5, 4}, {4, 1, 2, 6, 5}, {4, 2, 3, 7, 6},
     {4, 3, 0, 4, 7}},
    {{3, 0, 1, 2}, {3, 3, 4, 5}, {4, 0, 1, 4, 3}, {4, 1, 2, 5, 4}, {4, 2, 0, 3, 5}},
    {{4, 0, 1, 2, 3}, {3, 0, 1, 4}, {3, 1, 2, 4}, {3, 2, 3, 4}, {3, 3, 0, 4}},
};

typedef struct {
  size_t key[4]; /* sorted global nodes, padded with SIZE_MAX */
  size_t seq;    /* insertion order (element-major, face order) */
  size_t elem;
  int face;
} FaceRec;

static int face_cmp(const void* a, const void* b) {
  const FaceRec* x = (const FaceRec*)a;
  const FaceRec* y = (const FaceRec*)b;
  for (int k = 0; k < 4; ++k)
    if (x->key[k] != y->key[k]) return x->key[k] < y->key[k] ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq ? 1 : 0);
}

typedef struct { double x, y, z; } V3;
static V3 v3(double x, double y, double z) { V3 r = {x, y, z}; return r; }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V3 vscale(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
static double vsq(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
static double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V3 vcross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
/* vec.hpp:64-67 */
static V3 vnormalized(V3 v) {
  const double n = sqrt(vsq(v));
  return n > 0.0 ? vscale(v, 1.0 / n) : v3(0, 0, 0);
}
static V3 node_at(const double* nodes, size_t i) { return v3(nodes[3 * i], nodes[3 * i + 1], nodes[3 * i + 2]); }

/* quality.cpp:51-55 / 74-78: sum in node order, times 1/count */
static V3 centroid_of(const double* nodes, const size_t* g, size_t cnt) {
  V3 c = v3(0, 0, 0);
  for (size_t k = 0; k < cnt; ++k) c = vadd(c, node_at(nodes, g[k]));
  return vscale(c, 1.0 / (double)cnt);
}

/* quality.cpp:57-72 */
static V3 face_normal(const double* nodes, const size_t* g, int count) {
  if (count == 2) {
    const V3 t = vsub(node_at(nodes, g[1]), node_at(nodes, g[0]));
    return vnormalized(v3(t.y, -t.x, 0.0));
  }
  const V3 a = node_at(nodes, g[0]), b = node_at(nodes, g[1]), c = node_at(nodes, g[2]);
  V3 n = vcross(vsub(b, a), vsub(c, a));
  if (count == 4) {
    const V3 d = node_at(nodes, g[3]);
    n = vadd(vnormalized(n), vnormalized(vcross(vsub(c, a), vsub(d, a))));
  }
  return vnormalized(n);
}

/* quality.cpp:82-88 */
static double face_score(V3 normal, V3 line) {
  const V3 c = vnormalized(line);
  if (vsq(normal) == 0.0 || vsq(c) == 0.0) return 0.0;
  const double along = fabs(vdot(normal, c));
  const double transverse = sqrt(vsq(vcross(normal, c)));
  return 90.0 - atan2(transverse, along) * 180.0 / 3.141592653589793;
}

static void face_global(const size_t* conn, const size_t* offsets, const int* kinds, size_t e,
                        int f, size_t* g, int* count) {
  const int* fn = kFaceNodes[kinds[e]][f];
  *count = fn[0];
  for (int k = 0; k < fn[0]; ++k) g[k] = conn[offsets[e] + fn[1 + k]];
}

int or_orthogonality(const double* nodes, size_t n_nodes, int dim, const int* kinds,
                     const size_t* offsets, const size_t* conn, size_t n_elem, double* out_scores,
                     double* out_measures, double* out_min, double* out_mean,
                     size_t* out_inverted, size_t* out_degenerate) {
  size_t inverted = 0;
  or_signed_measures(nodes, n_nodes, dim, kinds, offsets, conn, n_elem, out_measures, &inverted);
  *out_inverted = inverted;
  *out_degenerate = 0;
  *out_min = 90.0;
  *out_mean = 90.0;
  for (size_t e = 0; e < n_elem; ++e) out_scores[e] = 90.0;
  if (n_elem == 0) return 0;
  size_t nf = 0;
  for (size_t e = 0; e < n_elem; ++e) nf += (size_t)kFaceCount[kinds[e]];
  FaceRec* recs = (FaceRec*)malloc((nf ? nf : 1) * sizeof(FaceRec));
  V3* cen = (V3*)malloc(n_elem * sizeof(V3));
  double* internal = (double*)malloc(n_elem * sizeof(double));
  double* boundary = (double*)malloc(n_elem * sizeof(double));
  char* degen = (char*)calloc(n_elem, 1);
  size_t r = 0;
  for (size_t e = 0; e < n_elem; ++e) {
    for (int f = 0; f < kFaceCount[kinds[e]]; ++f) {
      size_t g[4];
      int cnt;
      face_global(conn, offsets, kinds, e, f, g, &cnt);
      FaceRec* fr = &recs[r];
      for (int k = 0; k < 4; ++k) fr->key[k] = k < cnt ? g[k] : (size_t)-1;
      for (int a = 1; a < cnt; ++a) /* insertion sort of the key */
        for (int b = a; b > 0 && fr->key[b - 1] > fr->key[b]; --b) {
          const size_t t = fr->key[b];
          fr->key[b] = fr->key[b - 1];
          fr->key[b - 1] = t;
        }
      fr->seq = r;
      fr->elem = e;
      fr->face = f;
      ++r;
    }
    cen[e] = centroid_of(nodes, conn + offsets[e], offsets[e + 1] - offsets[e]);
    internal[e] = -1.0;
    boundary[e] = -1.0;
  }
  qsort(recs, nf, sizeof(FaceRec), face_cmp);
  for (size_t i = 0; i < nf;) {
    size_t j = i + 1;
    while (j < nf && memcmp(recs[j].key, recs[i].key, sizeof recs[i].key) == 0) ++j;
    size_t g0[4];
    int cnt;
    face_global(conn, offsets, kinds, recs[i].elem, recs[i].face, g0, &cnt);
    const V3 normal = face_normal(nodes, g0, cnt);
    const int is_deg = vsq(normal) == 0.0;
    if (j - i == 2) {
      const V3 line = vsub(cen[recs[i + 1].elem], cen[recs[i].elem]);
      const double score = is_deg ? 0.0 : face_score(normal, line);
      for (size_t u = i; u < j; ++u) {
        double* slot = &internal[recs[u].elem];
        *slot = *slot < 0.0 ? score : (*slot < score ? *slot : score); /* fold_in */
        if (is_deg) degen[recs[u].elem] = 1;
      }
    } else {
      for (size_t u = i; u < j; ++u) {
        size_t gu[4];
        int cu;
        face_global(conn, offsets, kinds, recs[u].elem, recs[u].face, gu, &cu);
        const V3 line = vsub(centroid_of(nodes, gu, (size_t)cu), cen[recs[u].elem]);
        const double score = is_deg ? 0.0 : face_score(normal, line);
        double* slot = &boundary[recs[u].elem];
        *slot = *slot < 0.0 ? score : (*slot < score ? *slot : score);
        if (is_deg) degen[recs[u].elem] = 1;
      }
    }
    i = j;
  }
  double sum = 0.0, mn = 90.0;
  size_t ndeg = 0;
  for (size_t e = 0; e < n_elem; ++e) {
    double score = internal[e] >= 0.0 ? internal[e] : boundary[e];
    if (score < 0.0) score = 90.0;
    if (degen[e]) {
      score = 0.0;
      ++ndeg;
    }
    out_scores[e] = score;
    sum += score;
    mn = mn < score ? mn : score; /* std::min(min_score, score) */
  }
  *out_min = mn;
  *out_mean = sum / (double)n_elem;
  *out_degenerate = ndeg;
  free(recs);
  free(cen);
  free(internal);
  free(boundary);
  free(degen);
  return 0;
}
