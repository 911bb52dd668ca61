// Device-resident plan (flat arrays in HBM) and the launch entry points of kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

#include "plan.h"

namespace dafmm {

// Passes timed by the profiler, in launch order (DAFMM_PASS_* of dafmm.h).
// gather, p2m, m2m, m2l, l2l, near (P2P, side stream), combine (L2P + identity + scatter), and the
// span of the concurrent part (from the fork to the later of P2P and L2L)
constexpr int kNumPasses = 9;
// marks recorded before the pass they name (EV_FAR_END after L2L); see harvest_profile
enum ProfEvent {
  EV_START, EV_FORK, EV_P2M, EV_M2M, EV_M2L, EV_L2L, EV_FAR_END, EV_NEAR0, EV_NEAR1, EV_JOIN, EV_END,
  EV_LEAF0, EV_LEAF1, EV_COUNT
};

struct DevBatch {
  int items = 0;
  bool wide = false;  // translate_kernel (warp per row) vs translate_rows_kernel (lane per row)
  int ipw = 1;        // translate_rows_kernel: items per warp (lane groups of 32 / ipw)
  bool colmajor = false;  // column-major items: translate_cm_kernel (lane per row, no reductions)
  bool grouped = false;   // mean rows <= 16: translate_cm_kernel<true> (lane groups share a row block)
  int64_t* dst_off = nullptr;
  int32_t* dst_rows = nullptr;
  int32_t* term_ptr = nullptr;
  int64_t* item_mat_off = nullptr;
  int32_t* item_cols = nullptr;
  int64_t* src_off = nullptr;
  int32_t* src_cols = nullptr;
};

struct DevPlan {
  int64_t n = 0;
  int kernel_mode = 0;
  cudaStream_t stream = nullptr;   // the caller's stream (dafmm_set_stream)
  cudaStream_t s_far = nullptr;    // internal high-priority stream: far field (P2M ... L2L)
  cudaStream_t s_near = nullptr;   // internal low-priority stream: P2P, concurrent with the far field
  cudaEvent_t ev_fork = nullptr, ev_join_far = nullptr, ev_join_near = nullptr;
  // leaf-level M2L on its own stream: it needs only the leaves' multipoles (P2M), so it runs
  // beside M2M and the coarse-level M2L / L2L, and joins before the L2L into the leaf level
  cudaStream_t s_leaf = nullptr;
  cudaEvent_t ev_p2m = nullptr, ev_leaf = nullptr;
  // per tree point
  double2* pts_t = nullptr;  // kappa-scaled coordinates
  double* w_t = nullptr;
  double* qk2_t = nullptr;
  double2* D_t = nullptr;
  int32_t* perm = nullptr;
  // expansions and pivots
  int64_t n_mult = 0, n_loc = 0;
  double2* so_xy = nullptr;  // kappa-scaled pivot coordinates
  double2* ti_xy = nullptr;
  double2* ops = nullptr;
  int64_t ops_len = 0;
  DevBatch p2m;
  std::vector<DevBatch> m2m, l2l;
  // M2L
  int m2l_targets = 0;
  int m2l_leaf_targets = 0;       // the first m2l_leaf_targets targets are at the deepest level
  int m2l_grid = 1;               // persistent CTAs (SMs x resident CTAs per SM)
  int near_after = 0;             // 2: the P2P starts when M2M has finished (far chain critical), 0: at the fork
  int* m2l_flag = nullptr;        // raised by the M2M stream when the coarser multipoles are complete
  int* m2l_ticket = nullptr;      // work counters (leaf-level part, rest), reset per matvec
  int64_t* m2l_loc_off = nullptr;
  int32_t* m2l_rows = nullptr;
  int64_t* m2l_stream_ptr = nullptr;  // per target: its source stream in m2l_stream_idx
  int32_t* m2l_stream_idx = nullptr;  // multipole slot of every source pivot, target by target
  int32_t* m2l_item_ptr = nullptr;
  int32_t* m2l_item_code = nullptr;
  int32_t* m2l_item_begin = nullptr;
  int32_t* m2l_item_end = nullptr;
  // stored M2L blocks (dafmm_options.m2l_store): per target node, column-major r x L block
  // (entry (t, s) at m2l_mat_off[target] + s * r + t), H0 units
  int64_t* m2l_mat_off = nullptr;
  double2* m2l_mat = nullptr;
  int m2l_store_grid = 0;
  // pair-stored M2L (Packed::m2l_sym, reading R22): own multipole of each target (column sums),
  // the column-sum slots (one per stream position) and the receiving nodes' slot lists
  int m2l_sym = 0;
  int m2l_pair_grid = 0;
  int64_t* m2l_self_moff = nullptr;
  int32_t* m2l_src_ptr = nullptr;   // pair mode: per target, its source runs (one per partner node):
  int64_t* m2l_src_off = nullptr;   //   first multipole slot of the run
  int32_t* m2l_src_cnt = nullptr;   //   and its length (the partner's outgoing rank)
  double2* m2l_slots = nullptr;
  int m2l_in_nodes = 0;
  int64_t* m2l_in_lo = nullptr;
  int32_t* m2l_in_rows = nullptr;
  int32_t* m2l_in_ptr = nullptr;
  int64_t* m2l_in_off = nullptr;
  // leaves
  int nleaves = 0, max_leaf = 0;
  int32_t* leaf_begin = nullptr;
  int32_t* leaf_end = nullptr;
  int32_t* near_ptr = nullptr;
  int32_t* near_begin = nullptr;
  int32_t* near_end = nullptr;
  int64_t* leaf_loc_off = nullptr;
  int32_t* leaf_rank = nullptr;
  int64_t* leaf_U_off = nullptr;
  int32_t* leaf_band = nullptr;
  // symmetric near field (Packed::p2p_sym): slots of the column sums, two halves of slot_total
  int p2p_sym = 0;
  int64_t slot_total = 0;
  int64_t* leaf_slot_base = nullptr;
  int32_t* in_ptr = nullptr;
  int64_t* in_off = nullptr;
  double2* slots = nullptr;
  // scratch
  double2* x_t = nullptr;
  double2* v_t = nullptr;
  double2* phi = nullptr;          // P2P result (H0 units, tree order)
  double2* mult = nullptr;
  double2* loc = nullptr;
  double2* host_stage = nullptr;  // device vectors for dafmm_matvec_host (x, y)
  // GMRES workspace (allocated on first use)
  int gm_restart = 0;
  double2* gm_V = nullptr;     // (restart + 1) x n
  double2* gm_w = nullptr;
  double2* gm_r = nullptr;
  double2* gm_h = nullptr;     // restart + 1 coefficients
  double2* gm_part = nullptr;  // partial sums
  double2* gm_z = nullptr;     // preconditioned vector (right preconditioning)
  double* gm_hostbuf = nullptr;  // pinned
  int gm_part_blocks = 0;
  int64_t gm_reorth = 0;       // reorthogonalisation passes in the last ls_gmres_solve
  size_t device_bytes = 0;
  double t_ops_device = 0;       // upload_plan: operator formation on the device (F2)
  std::vector<void*> allocations;
  // per-pass CUDA-event profiling (dafmm_set_profiling / dafmm_pass_times)
  int64_t launches = 0;          // kernels launched by run_matvec / run_gmres since the last reset
  bool prof = false;
  bool prof_pending = false;     // events of the last profiled matvec not yet harvested
  cudaEvent_t prof_ev[EV_COUNT] = {};
  double prof_ms[kNumPasses] = {};
  bool prof_side_m2m = false;     // the last matvec ran M2M on the side stream (its time is between the LEAF marks)
  int64_t prof_count = 0;        // profiled matvecs harvested
};

// Enable / disable per-pass event timing; resets the accumulators and the launch counter.
int set_profiling(DevPlan& d, bool on, std::string& err);
// Harvest the events of the last profiled matvec into prof_ms (synchronises on them).
int harvest_profile(DevPlan& d, std::string& err);

int upload_plan(const Packed& pk, const Plan& plan, DevPlan& d, std::string& err);
void free_plan(DevPlan& d);
// y = A x (mask bit 0 near, bit 1 far); x, y device pointers in caller order
int run_matvec(DevPlan& d, const double2* x, double2* y, unsigned mask, std::string& err);
// Right preconditioner z = M^{-1} v (device vectors, caller order, on the handle's stream; v may equal z).
using Precond = std::function<int(const double2* v, double2* z, std::string& err)>;
int run_gmres(DevPlan& d, const double2* f, double2* psi, double tol, int maxit, int restart, int* iters,
              double* relres, double* history, std::string& err, const Precond& prec = nullptr);
// out[i] = H0^(1)(sqrt(z2[i])) by band `code` (device pointers, enqueued on s)
int h0_eval(const double* z2, double2* out, int64_t n, int code, cudaStream_t s, std::string& err);

}  // namespace dafmm
