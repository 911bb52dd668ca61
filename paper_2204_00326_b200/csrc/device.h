// Device-resident plan (flat arrays in HBM) and the launch entry points of kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "plan.h"

namespace dafmm {

struct DevBatch {
  int items = 0;
  int64_t* dst_off = nullptr;
  int32_t* dst_rows = nullptr;
  int32_t* term_ptr = nullptr;
  int64_t* mat_off = nullptr;
  int64_t* src_off = nullptr;
  int32_t* src_cols = nullptr;
};

struct DevPlan {
  int64_t n = 0;
  int kernel_mode = 0;
  KernelConsts kc{};
  cudaStream_t stream = nullptr;
  // per tree point
  double2* pts_t = nullptr;
  double* w_t = nullptr;
  double* qk2_t = nullptr;
  double2* D_t = nullptr;
  int32_t* perm = nullptr;
  // expansions and pivots
  int64_t n_mult = 0, n_loc = 0;
  double2* so_xy = nullptr;
  double2* ti_xy = nullptr;
  double2* ops = nullptr;
  int64_t ops_len = 0;
  DevBatch p2m;
  std::vector<DevBatch> m2m, l2l;
  // M2L
  int m2l_targets = 0;
  int64_t* m2l_loc_off = nullptr;
  int32_t* m2l_rows = nullptr;
  int32_t* m2l_src_ptr = nullptr;
  int64_t* m2l_src_off = nullptr;
  int32_t* m2l_src_cnt = nullptr;
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
  // scratch
  double2* x_t = nullptr;
  double2* v_t = nullptr;
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
  double* gm_hostbuf = nullptr;  // pinned
  int gm_part_blocks = 0;
  size_t device_bytes = 0;
  std::vector<void*> allocations;
};

int upload_plan(const Packed& pk, const Plan& plan, DevPlan& d, std::string& err);
void free_plan(DevPlan& d);
// y = A x (mask bit 0 near, bit 1 far); x, y device pointers in caller order
int run_matvec(DevPlan& d, const double2* x, double2* y, unsigned mask, std::string& err);
int run_gmres(DevPlan& d, const double2* f, double2* psi, double tol, int maxit, int restart, int* iters,
              double* relres, double* history, std::string& err);

}  // namespace dafmm
