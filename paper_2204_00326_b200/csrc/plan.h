// Host-side plan: tree, lists, NCA pivots and operators of one dafmm handle, plus the
// packed flat arrays that are uploaded once to HBM.
#pragma once
#include <array>
#include <complex>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "hankel.cuh"

namespace dafmm {

static_assert(kNumBandCodes <= 48, "dafmm_stats_t band arrays hold 48 codes");

using zd = std::complex<double>;

struct Options {
  double T = 16.0;         // regime threshold (reading R3)
  int self_term = 1;       // 0 zero (point kernel, E1), 1 disk (reading D1)
  int kernel_mode = 0;     // 0 Lippmann-Schwinger y = x + k^2 q (K x); 1 potential y = K x
  int max_level = 20;
  int num_threads = 0;     // host setup threads (0: OpenMP default)
  int host_only = 0;       // skip the device upload
  int symmetric_pivots = 0;  // reading R19 (option): one ACA per node, outgoing skeleton = incoming
  int m2l_store = -1;        // M2L blocks: -1 auto, 0 on the fly every matvec, 1 stored in HBM, 2 stored per pair (R22)
  int hfr_parent_search = 0;  // reading R7b (option): HFR search sets also take the parent's far children
  int w_reading = 0;         // reading R4 of w: 0 circumradius b / sqrt(2), 1 box width b
  int setup_device = 1;      // NCA ACAs on the device (F2); 0: on the host (always for host_only plans)
};

struct Box {
  int64_t ix, iy;
  int32_t begin, end;  // tree-order point range (every box of the adaptive tree is contiguous)
  bool leaf;
};

struct Level {
  int level = 0;
  double b = 0, kb = 0;
  bool hfr = false;
  int ncones = 1;
  std::vector<Box> boxes;                      // non-empty boxes in Morton order
  std::unordered_map<uint64_t, int> index;     // packed (ix, iy) -> box
  std::vector<std::vector<int>> N, IL;         // per box, box indices at this level
  // ILdir[box] = sorted list of (cone, src box, src cone)
  std::vector<std::vector<std::array<int, 3>>> ILdir;
  // nodes: LFR -> one per active box (cone = -1); HFR -> one per active (box, cone)
  std::vector<std::pair<int, int>> nodes;
  std::vector<int> node_of;                    // box * ncones + cone (cone = 0 for LFR) -> node or -1
  int node_id(int box, int cone) const { return node_of[(size_t)box * ncones + (hfr ? cone : 0)]; }
};

struct NodePivots {
  std::vector<int32_t> ti, si, to, so;  // original point indices, in ACA selection order
};

struct Plan {
  Options opt;
  int64_t n = 0;
  double kappa = 0, nca_tol = 0;
  double W = 0, x0 = 0, y0 = 0;
  int L = 0;                         // deepest level
  bool multi_level_leaves = false;   // leaves on more than one level (adaptive tree)
  bool level_restricted = true;      // adjacent leaves differ by at most one level
  // input copies (original order)
  std::vector<double> pts, w, q;
  std::vector<zd> D;                 // self terms D_i (original order)
  std::vector<int32_t> perm;         // tree index -> original index
  std::vector<Level> levels;
  std::vector<std::pair<int, int>> leaves;                  // (level, box), coarse levels first
  std::vector<std::vector<std::pair<int, int>>> near;       // per leaf: source boxes (level, box)
  std::vector<std::vector<NodePivots>> piv;  // [level][node]
  // statistics
  double t_tree = 0, t_lists = 0, t_nca = 0, t_ops = 0, t_pack = 0, t_upload = 0;
  double t_nca_device = 0;  // inside t_nca: the device ACA launches (upload, kernel, download)
  int64_t aca_entries = 0;
};

// Packed device-layout arrays (host copies before upload).
struct Packed {
  // per tree point
  std::vector<double> pts_t;        // 2 per point
  std::vector<double> w_t, qk2_t;   // weights, kappa^2 q
  std::vector<cplx> D_t;            // self term
  std::vector<int32_t> perm;
  // expansion buffers
  int64_t n_mult = 0, n_loc = 0;
  std::vector<double> so_xy, ti_xy;  // 2 per multipole / local slot
  std::vector<cplx> ops;             // all operator blocks, column-major
  // generic translation batches: item -> [term_ptr[i], term_ptr[i+1]) terms
  // item i: dst[dst_off + r] (+)= sum_c M[r][c] s_c, M row-major (rows x item_cols) at
  // ops[item_mat_off]; its columns are the terms [term_ptr[i], term_ptr[i+1]) side by side,
  // term t taking src_cols[t] consecutive sources from src_off[t]
  struct Batch {
    std::vector<int64_t> dst_off;       // per item
    std::vector<int32_t> dst_rows;      // per item
    std::vector<int64_t> item_mat_off;  // per item (into ops)
    std::vector<int32_t> item_cols;     // per item
    std::vector<int32_t> term_ptr;      // items + 1
    std::vector<int64_t> src_off;       // per term
    std::vector<int32_t> src_cols;      // per term
  };
  // operators formed on the device (setup_device, every cross matrix of rank <= 64): ops stays
  // empty on the host and upload_plan runs form_ops_device on these descriptors
  int ops_colmajor = 1;  // translation items column-major (translate_cm_kernel); 0: row-major (env DAFMM_OPS_ROWMAJOR)
  int ops_on_device = 0;
  int64_t ops_len = 0;
  std::vector<int32_t> opd_piv;
  std::vector<std::array<int32_t, 6>> opd_groups;  // a_off, b_off, r, type, job_begin, job_end
  struct OpdJob {
    int64_t off;
    int32_t rows, col_start, stride, pad0;
    int64_t src_off;
    int32_t src_len, pad;
  };
  std::vector<OpdJob> opd_jobs;
  Batch p2m;                         // leaf: dst multipole, src tree points (v), 1 term
  std::vector<Batch> m2m;            // per parent level, processed from fine to coarse
  std::vector<Batch> l2l;            // per parent level, processed from coarse to fine
  // M2L: target nodes with source node CSR
  int m2l_leaf_targets = 0;          // targets [0, m2l_leaf_targets) are at the deepest level L
  std::vector<int64_t> m2l_loc_off;  // per target
  std::vector<int32_t> m2l_rows;     // r_i per target
  std::vector<int32_t> m2l_src_ptr;  // targets + 1
  std::vector<int64_t> m2l_src_off;  // per source entry: multipole offset
  std::vector<int32_t> m2l_src_cnt;  // per source entry: r_o
  std::vector<int64_t> m2l_stream_ptr;  // targets + 1: each target's source-pivot stream
  std::vector<int32_t> m2l_stream_idx;  // multipole slot of every pivot of the stream
  // band-uniform segments of each target's source list: items of target
  // t are [m2l_item_ptr[t], m2l_item_ptr[t+1]); item i covers the pivots
  // [m2l_item_begin[i], m2l_item_end[i]) of t's concatenated source stream, whose pairs with
  // t's pivots all lie in band m2l_item_code[i]
  std::vector<int32_t> m2l_item_ptr;   // targets + 1
  std::vector<int32_t> m2l_item_code, m2l_item_begin, m2l_item_end;
  std::vector<int64_t> m2l_band_entries = std::vector<int64_t>(kNumBandCodes, 0);
  // leaves: near field + L2P + combine
  std::vector<int32_t> leaf_begin, leaf_end;  // tree ranges
  std::vector<int32_t> near_ptr;              // leaves + 1
  std::vector<int32_t> near_begin, near_end;  // per near entry: tree range of the source leaf
  std::vector<int64_t> leaf_loc_off;          // -1: no far field
  std::vector<int32_t> leaf_rank;             // r_i
  std::vector<int64_t> leaf_U_off;
  std::vector<int32_t> leaf_band;             // P2P band code: near if every pair has z <= 8
  // symmetric near field (p2p_sym): each leaf streams only its own leaf and the ranges after it
  // in tree order; the column sums of those pairs (the contributions to the later points) go
  // to slots (two halves: one per warp of a 64-target slice), gathered per leaf at combine
  int p2p_sym = 0;
  std::vector<int64_t> leaf_slot_base;        // per leaf: slot of its first streamed non-own source
  int64_t slot_total = 0;
  std::vector<int32_t> in_ptr;                // leaves + 1: slots holding contributions to the leaf
  std::vector<int64_t> in_off;                // slot of the leaf's first point in each
  std::vector<int64_t> p2p_band_entries = std::vector<int64_t>(kNumBandCodes, 0);
  int max_leaf = 0;
  // statistics
  int64_t p2p_pairs = 0, m2l_entries = 0, m2l_pairs = 0;
  // symmetric stored M2L (reading R22, m2l_store = 2): with one skeleton per node (R19) the block
  // of (B <- A) is the transpose of the block of (A <- B), so every unordered pair {A, B} of
  // interaction-list nodes keeps ONE block, in the stream of its owner (the node with the lower
  // id at the level).  The owner's CTA applies it twice: row sums into its own local
  // expansion, column sums (with its own multipole) into per-stream-position slots, which a
  // gather adds to the other node's local expansion.
  int m2l_sym = 0;
  int64_t m2l_stored_entries = 0;    // entries of the stored blocks (m2l_entries / 2 when m2l_sym)
  std::vector<int64_t> m2l_self_moff;  // per target: its own multipole (column sums)
  std::vector<int64_t> m2l_in_lo;      // per receiving node: local-expansion offset
  std::vector<int32_t> m2l_in_rows;    // per receiving node: its rank
  std::vector<int32_t> m2l_in_ptr;     // receiving nodes + 1
  std::vector<int64_t> m2l_in_off;     // slot (stream position) of the node's first pivot in each owner stream
};

// setup.cpp
int build_plan(Plan& plan, const double* points, const double* weights, const double* q, int64_t n,
               double kappa, int leaf_size, double nca_tol, const Options& opt, std::string& err);
// device_free: free device bytes for the auto choice of the symmetric stored M2L (0: unknown)
int pack_plan(const Plan& plan, Packed& pk, std::string& err, size_t device_free = 0);
int export_plan(const Plan& plan, const std::string& dir, std::string& err);

}  // namespace dafmm
