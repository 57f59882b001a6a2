// greedy.hpp — device state and host driver of the exact greedy engine
// (greedy.cu).  Internal to the library; the C-ABI is in capi.cu.
#pragma once

#include <cuda_runtime.h>

#include "runtime.hpp"

namespace imb {

enum : int {
  kStatusRunning = 0,
  kStatusConverged = 1,  // achieved < tolerance (greedy.cpp:146)
  kStatusCapHit = 2,     // cap reached or no candidate left (greedy.cpp:147-151)
  kStatusSolveError = 3, // pivot <= 1e-14 * max_diag (rbf.cpp:92)
  kStatusWatchdog = 4,   // speculative pipeline: a spin loop timed out (never expected)
};

// ---- speculative pipeline (greedy_spec.cu) ---------------------------------
struct __align__(16) SpecCtl {
  int epoch, abort, abort_step, done;  // polled together as one int4
  int rb_step, conf, status, final_step;
  int fail_node, fail_row, ticket, fticket;
  int hits, misses, late, rollbacks;
  double achieved, overall, fail_pivot;
  unsigned long long t0;
  int probe[8];  // launch counters (diagnostics): insert, fsolve, fsweep, fsweep-final,
                 // wait, sweep, sweep-final, server-chain
};
// the words the host loop polls, mirrored into mapped pinned memory
struct SpecHost {
  volatile int conf, abort, abort_step, status, done;
  volatile int seen[8];  // diagnostics: last step each kernel kind started (probe order)
};
struct SpecView {
  int n, cap, S, kind;
  double R, tol, target_max;
  const double *px, *py, *pz, *tx, *ty, *tz;
  double *rx, *ry, *rz;
  double *cx, *cy, *cz;
  int* cidx;
  double* Lt;
  double2* diag;
  double *yx, *yy, *yz;
  double* slots;      // [S][3][cap] alpha of step k in slot k % S
  double* xs_global;  // [S][4][cap] chain workspace when smem is too small
  double* rr_global;  // [cap] insert scratch when smem is too small
  double *fax, *fay, *faz;  // predictor alpha
  int* selstep;       // [n] step at which the node was inserted (INT_MAX: not)
  int *state, *ins_ep, *chain_ep, *ins_node, *ins_fail, *pred_node;  // [cap + 1]
  int *pred2_node, *exact_node;                                      // [cap + 1]
  double *pivot, *pred_gap, *exact_gap;                              // [cap + 1]
  double *bv, *bv2, *ba;
  int *bi, *bi2;
  double *fbv, *fbv2;
  int* fbi;
  double *rec_err, *rec_sec;
  SpecCtl* ctl;
  SpecHost* host;
  unsigned long long watchdog_ns;
  unsigned long long* tl;  // per-step timeline (diagnostics)
};
struct SpecStats {
  long long hits = 0, misses = 0, late = 0, rollbacks = 0;
};

// Device-resident step state (one per level run).
struct GState {
  int status;
  int nc;        // controls selected so far
  int next;      // node inserted by the next k_insert
  int steps;     // sweeps done (= convergence samples)
  int fail_node, fail_row;
  unsigned int ticket;
  int pad;
  double tol, target_max, max_diag, smallest_pivot, achieved, overall, fail_pivot;
  unsigned long long t0;
};

struct GView {
  GState* st;
  int n, cap, kind;
  double R;
  const double *px, *py, *pz;  // surface positions
  const double *tx, *ty, *tz;  // level target
  double *rx, *ry, *rz;        // residual
  unsigned char* sel;
  int* cidx;
  double *cx, *cy, *cz;        // control positions (insertion order)
  double* Lt;                  // column-major packed lower factor
  double2* diag;               // (L_kk, refined reciprocal)
  double *yx, *yy, *yz;        // forward solutions
  double *ax, *ay, *az;        // alpha
  double* xs_global;           // backward-chain workspace when smem is too small
  double* rr_global;           // k_insert row scratch when smem is too small
  double *bv, *ba;
  int* bi;
  double *rec_err, *rec_sec;
};

class GreedyEngine {
 public:
  GreedyEngine(Context& ctx, int n, int cap);
  ~GreedyEngine();
  GreedyEngine(const GreedyEngine&) = delete;
  GreedyEngine& operator=(const GreedyEngine&) = delete;

  void set_positions(const double* host_xyz);
  void set_target(const double* host_xyz);
  void target_from_residual();
  void reset(double tol, double target_max, int kind, double R);
  const GState& run_level(int batch = 8);
  const GState& run_level_spec();
  const SpecStats& spec_stats() const { return spec_stats_; }
  const GState& factor_all_and_solve();
  const GState& poll();
  double bench_backward(int n, int reps);
  void download(int nc, size_t* idx, double* alpha_aos, double* residual_aos, double* rec_err,
                double* rec_sec, int steps);

  // device views for the volume pipeline
  const DPoints& positions() const { return pos_; }
  const DPoints& control_positions() const { return cpos_; }
  const DPoints& alpha() const { return alpha_; }
  const DPoints& residual() const { return res_; }
  int n() const { return n_; }
  int cap() const { return cap_; }

 private:
  GView view();
  SpecView spec_view();
  void spec_alloc();
  void spec_free();
  int spec_restart_step();
  void enqueue_step(bool sweep);
  void launch_backward(const GView& g);
  void launch_insert(const GView& g);

  Context& ctx_;
  int n_, cap_;
  int kind_ = 1;
  double R_ = 1.0;
  int sweep_kind_ = -1;       // k_sweep<KIND> staged path, or -1 (generic)
  double pos_max_abs_ = 0.0;  // max |coordinate| of the surface positions
  int nblk_ = 1;
  size_t bw_smem_ = 0, ins_smem_ = 0;
  int ins_ring_ = 2;  // columns of L in flight in k_insert
  int ins_threads_ = 1024;  // k_insert CTA size
  DPoints pos_, tgt_, res_, cpos_, y_, alpha_;
  DBuf<unsigned char> sel_;
  DBuf<int> cidx_;
  DBuf<double> lt_, xs_, rr_, bv_, ba_, rec_err_, rec_sec_;
  DBuf<double2> diag_;
  DBuf<int> bi_;
  DBuf<GState> st_;
  GState* hst_ = nullptr;
  double tol_ = 0.5, target_max_ = 0.0;
  // speculative pipeline
  bool sp_ready_ = false, sp_xs_smem_ = true;
  int spec_S_ = 32, sp_fnblk_ = 1;
  size_t sp_server_smem_ = 0, sp_fsolve_smem_ = 0, sp_pred_smem_ = 0;
  DBuf<double> sp_slots_, sp_fa_, sp_xs_, sp_dwords_, sp_bv2_, sp_fbv_;
  DBuf<int> sp_selstep_, sp_words_, sp_fbi_, sp_bi2_;
  DBuf<SpecCtl> sp_ctl_;
  DBuf<unsigned long long> sp_tl_;
  SpecHost* sp_host_ = nullptr;
  SpecHost* sp_host_dev_ = nullptr;
  cudaStream_t sp_pred_ = nullptr, sp_chain_ = nullptr;
  SpecStats spec_stats_;
};

}  // namespace imb
