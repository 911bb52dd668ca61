// Device-side ACA of the NCA setup (setup_device.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "dafmm.h"
#include "hankel.cuh"

namespace dafmm {

// One ACA problem: the block K[rows, cols] with rows = idx[row_off, row_off + m) and
// cols = idx[col_off, col_off + n) (point indices of the uploaded arrays); the pivots go to
// out_off .. out_off + rank of the output arrays (positions within rows / cols).
//   mode 0: the NCA's ACA (reading R10) on K_ij = G(x_i, x_j) w_j: first row 0, tolerance eps,
//           zero residual rows skipped, rank cap min(m, n, 200, cap > 0 ? cap : 200)
//   mode 1: the HODLR preconditioner's fixed-rank ACA (reading HR2) on the rows of A, q_i G w_j:
//           first row first_row, rank cap `cap`, ends at a zero residual row or column
//   mode 1 with u_out / v_out: the ACA factors themselves are written out (the rank-k approximant
//           sum_l u_l v_l^T, balanced so |u_l| = |v_l|): u_out[(row_off + t) ldo + l], v_out[(col_off + j)
//           ldo + l] for l < ldo (zero for l >= rank)
struct AcaProblem {
  int64_t row_off, col_off;
  int32_t m, n;
  int64_t out_off;
  int32_t first_row = 0, cap = 0, mode = 0, pad = 0;
  double2* u_out = nullptr;
  double2* v_out = nullptr;
  int32_t ldo = 0, pad2 = 0;
};

// Translation operators formed on the device (P:427-562 in the G-only form of DESIGN.md §5):
// one group per (node, kind) shares the LU of its cross matrix M[a][c] = H0(kappa |A_a - B_c|).
//   type 0 (V~, P2M / M2M): A = t^{B,o}, B = s^{B,o}; job column j: x = M^{-1} H(A, src_j),
//           element (row a, column col_start + j) = x_a
//   type 1 (U~, L2L / L2P):  A = t^{B,i}, B = s^{B,i}; job row j: x M = H(src_j, B),
//           element (row j, column col_start + c) = x_c
// Element (row, col) of a job's block sits at off + row stride + col (row-major translation
// items, stride = the item's columns) or off + col rows + row (stride 0: column-major L2P U).
struct OpGroup {
  int32_t a_off, b_off, r, type;  // pivot lists at piv[a_off], piv[b_off] (r each)
  int32_t job_begin, job_end;
};
struct OpJob {
  int64_t off;           // item block start in ops
  int32_t rows, col_start, stride, pad0;
  int64_t src_off;       // caller indices at piv[src_off, src_off + src_len)
  int32_t src_len, pad;
};
constexpr int kDeviceOpsMaxRank = 64;
// Forms every group's blocks into the device array ops (caller-order points, kappa-scaled on
// upload).  DAFMM_ESETUP on a singular cross matrix.
int form_ops_device(const double* pts, int64_t n, double kappa, const std::vector<int32_t>& piv,
                    const std::vector<OpGroup>& groups, const std::vector<OpJob>& jobs, double2* ops,
                    std::string& err);

class DeviceAca {
 public:
  DeviceAca() = default;
  DeviceAca(const DeviceAca&) = delete;
  DeviceAca& operator=(const DeviceAca&) = delete;
  ~DeviceAca();
  // uploads the kappa-scaled points and the weights (caller order)
  // (and q, caller order, when a mode-1 problem will run)
  int init(const double* pts, const double* w, int64_t n, double kappa, std::string& err, const double* q = nullptr);
  // runs every problem (R10 ACA at tolerance eps); probs[i].out_off is assigned here; pivot
  // positions of problem i are piv_row/piv_col[out_off, out_off + rank[i])
  int run(const std::vector<int32_t>& idx, std::vector<AcaProblem>& probs, double eps, std::vector<int32_t>& piv_row,
          std::vector<int32_t>& piv_col, std::vector<int32_t>& rank, int64_t& entries, std::string& err);

 private:
  double2* pts_ = nullptr;
  double* w_ = nullptr;
  double* q_ = nullptr;
  double kappa_ = 0.0;
  cudaStream_t stream_ = nullptr;
};

}  // namespace dafmm
