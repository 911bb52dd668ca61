// HODLR preconditioner of the hybrid solver (Eq. hybrid):
// a Hierarchically Off-Diagonal Low-Rank approximation Ã of the Lippmann-Schwinger matrix A
// with the rank of every off-diagonal block fixed a priori, factorised and applied on the
// device (hodlr.cu).  Readings HR1-HR4 of DESIGN.md §2.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "device.h"
#include "plan.h"

namespace dafmm {

struct HodlrPlan {
  int64_t n = 0;
  int r = 0, n0 = 0;
  int64_t max_block = 0;  // HR5: blocks with more rows are dropped (0: none)
  int depths = 0;   // depths with split nodes (0 .. depths - 1); pairs live at depths 1 .. depths
  int ld = 0;       // columns of Ucat / Vcat = depths * r
  cudaStream_t stream = nullptr;  // the owning DAFMM handle's stream at creation / solve
  // host structure (tree positions of the DAFMM tree order, HR1)
  std::vector<std::vector<int64_t>> split_a, split_m, split_b;  // per depth: split nodes [a, m, b)
  std::vector<int64_t> leaf_a, leaf_n;
  // block pivots (HR2), per depth d + 1 pair: block 2i = rows [a, m) x cols [m, b), 2i + 1 the other
  std::vector<std::vector<int32_t>> blk_ptr;   // per depth: 2 * nodes + 1 offsets into blk_I / blk_J
  std::vector<std::vector<int32_t>> blk_I, blk_J;  // tree positions
  // device
  double2* Ucat = nullptr;   // n x ld: per point, per depth: W = (processed) U of its node's block
  double2* Vcat = nullptr;   // n x ld: per point, per depth: A[I_sibling, t]
  double2* leaf_lu = nullptr;  // per leaf: n_l x n_l inverse of A[leaf, leaf] (by LU), column-major
  int32_t* leaf_prow = nullptr;  // per leaf: row permutation (P b)_i = b[prow[i]]
  int64_t* leaf_a_d = nullptr;
  int32_t* leaf_n_d = nullptr;
  int64_t* leaf_lu_off = nullptr;
  std::vector<int64_t*> split_d;   // per depth: device copy of (a, m, b) triplets
  std::vector<int32_t*> part_d;    // per depth: parts (child node ids 2i / 2i+1, t0, t1)
  std::vector<int> nparts;
  std::vector<std::vector<int32_t>> part_ptr;  // per depth: per child (2 * nodes + 1) offsets into parts
  std::vector<int32_t*> part_ptr_d;
  std::vector<double2*> S_lu;      // per depth: per split node (2r)^2 LU, column-major
  std::vector<int32_t*> S_prow;    // per depth: per split node 2r permutation
  std::vector<double2*> S_inv;     // per depth: per split node S^{-1}, column-major (the apply)
  double2* partial = nullptr;      // parts x r x ncol scratch
  int64_t partial_len = 0;
  double2* C = nullptr;            // per split node 2r x ncol solve buffer
  int64_t C_len = 0;
  double2* xt = nullptr;           // tree-order work vector
  int* status = nullptr;           // device flag: singular pivot
  int32_t* perm = nullptr;         // the DAFMM plan's perm (not owned)
  std::vector<void*> allocations;
  size_t device_bytes = 0;
  double t_aca = 0, t_basis = 0, t_factor = 0;
  int64_t aca_entries = 0;
  int max_rank = 0;
  double mean_rank = 0;
};

// Build Ã of the plan's operator (kernel_mode 0 only) on the device: pivots by the fixed-rank
// ACA (HR2, device), bases, leaf LU and the recursive factorisation (HR3).
int hodlr_create(const Plan& plan, const DevPlan& d, int rank, int leaf_size, int64_t max_block, HodlrPlan& h,
                 std::string& err);
// out = Ã^{-1} in (device pointers, caller order), enqueued on `s`; in may equal out.
int hodlr_apply(HodlrPlan& h, const double2* in, double2* out, cudaStream_t s, std::string& err);
void hodlr_free(HodlrPlan& h);
// .npy files for the oracle: hodlr_blocks (nblocks x 5: depth, a, b, c, d), hodlr_piv_ptr,
// hodlr_I, hodlr_J (tree positions), hodlr_perm (tree position -> caller index), hodlr_meta (r, n0)
int hodlr_export(const HodlrPlan& h, const Plan& plan, const std::string& dir, std::string& err);

}  // namespace dafmm
