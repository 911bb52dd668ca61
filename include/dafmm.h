/*
 * dafmm.h — C-ABI of the B200-native DAFMM matvec and GMRES for the discretised 2D
 * Lippmann-Schwinger equation of arxiv 2204.00326 ("PAPER.md", cited P:<line>).
 *
 * Operation (the boundary semantics).  For points x_i, quadrature weights w_i > 0 and a
 * real contrast q_i, the library applies the discrete operator of Eq. 12a/13
 * in point (Nystrom) form:
 *
 *     y = A x,   (A x)_i = x_i + kappa^2 q_i [ sum_{j != i} G(x_i, x_j) w_j x_j + D_i x_i ]
 *
 * with the Helmholtz Green's function G(x,y) = (i/4) H0^(1)(kappa |x - y|) and the
 * self term D_i = integral of G over the equal-area disk of area w_i (reading D1).
 * The sum is evaluated by the Directional Algebraic FMM whose low-rank bases
 * come from the nested cross approximation at tolerance nca_tol; the result
 * matches the dense product within about 10 x nca_tol (relative l2 of y - x).
 *
 * Memory and ownership.  Host arrays passed to dafmm_create are copied; the caller keeps
 * them.  Vectors passed to dafmm_matvec / ls_gmres_solve are DEVICE pointers to N complex128
 * values stored interleaved (re, im) in the caller's point order, 16-byte aligned; they must
 * not alias each other.  The handle owns all device memory of the plan (freed by
 * dafmm_destroy).  Device work is enqueued on the handle's CUDA stream (default: the legacy
 * default stream; set with dafmm_set_stream) and is asynchronous to the host unless stated.
 *
 * Threading.  A handle is immutable after creation apart from its scratch workspace, so calls
 * on one handle must be serialised (same stream, one host thread at a time).  Distinct
 * handles are independent.
 *
 * Errors.  Every int-returning call returns DAFMM_OK (0) on success and a negative code on
 * error; dafmm_last_error() returns a thread-local message for the last failure.
 * ls_gmres_solve returns DAFMM_NOT_CONVERGED (> 0) when maxit is reached — a status, not an
 * error; psi then holds the last iterate.
 */
#ifndef DAFMM_H
#define DAFMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dafmm_plan* dafmm_handle;

enum {
  DAFMM_OK = 0,
  DAFMM_NOT_CONVERGED = 1, /* ls_gmres_solve: maxit reached before tol (not an error) */
  DAFMM_EINVAL = -1,       /* bad argument: n <= 0, kappa <= 0 or non-finite, nca_tol not in
                              (0,1), leaf_size < 1, NaN/Inf input, weight <= 0, duplicate
                              points, null pointer, unsupported option */
  DAFMM_ECUDA = -2,        /* a CUDA runtime call failed (message has the CUDA error) */
  DAFMM_ENOMEM = -3,       /* host or device allocation failed */
  DAFMM_ESETUP = -4        /* NCA setup failed (singular cross matrix) */
};

/* Options of dafmm_create_ex; initialise with dafmm_default_options(). */
typedef struct {
  double T;            /* regime threshold: a box of width b is HFR iff (kappa b)^2 > T
                          (reading R3; default 16) */
  int self_term;       /* D_i = integral of G over the point's cell (Eq. 13): 1 over the
                          equal-area disk of area w_i (reading D1, closed form; default); 2 over the
                          square of side sqrt(w_i) centred on the point (polar form, radial integral
                          exact, 40-node Gauss-Legendre in angle; 4.1e-3 from the disk at kappa h =
                          0.3125); 0: D_i = 0 (point kernel of Experiment 1) */
  int kernel_mode;     /* 0: Lippmann-Schwinger y = x + kappa^2 q o (K x) (default);
                          1: potential y = K x (the N-body sum of Experiment 1) */
  int max_level;       /* deepest tree level allowed (default 20, the maximum) */
  int num_threads;     /* host threads for setup; 0 = OpenMP default */
  int host_only;       /* 1: build the host plan only (no device upload; for inspection and
                          dafmm_export_plan on machines without a GPU); matvec / GMRES then
                          return DAFMM_EINVAL.  Default 0. */
  int symmetric_pivots; /* 0 (default): two ACAs per node (incoming and outgoing), as P:597-634
                           write them.  1: one ACA per node; the outgoing skeleton is the incoming
                           one with rows and columns swapped (reading R19, G symmetric): half the
                           ACA setup time, 3% more M2L work at C4. */
  int m2l_store;       /* M2L blocks A_{t s}: 0 evaluate the kernel entries on the fly in
                          every matvec (fp64-ALU bound); 1 evaluate them once at create time on the
                          device and keep them in HBM (16 B per entry; every matvec then streams
                          them: HBM bound), DAFMM_ENOMEM if they do not fit, DAFMM_EINVAL if a
                          node has more than 128 pivots; -1 (default) auto: store when the blocks
                          take at most half of the free device memory and every node has at most
                          128 pivots, else on the fly.  2: one block per unordered node pair
                          {A, B} (reading R22; needs symmetric_pivots = 1: the block of A <- B is
                          then the transpose of B <- A), applied twice per matvec (row and column
                          sums): half the bytes of 1.  With -1 and symmetric_pivots = 1 the auto
                          choice is 2.  dafmm_stats reports the choice. */
  int hfr_parent_search; /* NCA search sets of a directional node (B, l) whose parent is also
                          directional (P:624-631 use IL(B, l) only): 0 (default) as the paper writes
                          them; 1 also take the children, in the matching child cones, of the
                          parent's IL in the two parent cones nesting in l (reading R7b).  Needed on
                          irregular domains where IL(B, l) spans fewer directions than the parent's
                          far field arriving through the directional L2L (L-shaped random points:
                          1.6e-4 vs dense with 0, 7.5e-9 with 1); on the uniform configs it costs
                          2x the ACA setup and 1.5% more M2L work for no accuracy gain. */
  int setup_device;    /* 1 (default): the ACAs of the NCA setup run on the device, one
                          CTA per (node, direction), level by level; the search sets are still built
                          on the host.  0: on the host (OpenMP).  Host-only plans always use the
                          host.  Both give valid pivots; they may differ where rounding breaks a
                          tie of the ACA's argmax. */
  int w_reading;       /* meaning of w in the directional regime (reading R4): 0 (default)
                          the box circumradius b / sqrt(2): HFR neighbours have centre distance <
                          kappa b^2 / 2, cones have half-angle <= sqrt(2) / (kappa b); 1 the box width
                          b: distance < kappa b^2, half-angle <= 1 / (kappa b) (more neighbours and
                          cones, longer interaction lists).  The regime test (kappa b)^2 > T
                          is the same in both. */
} dafmm_options;

/* Statistics of a plan (sizes, ranks, setup times). */
typedef struct {
  int64_t n;
  int32_t levels;            /* leaf level L */
  int32_t n_nodes;           /* nodes with bases (LFR boxes + HFR (box, cone) pairs) */
  int64_t p2p_pairs;         /* near-field point pairs (i, j), j != i */
  int64_t m2l_entries;       /* kernel entries evaluated by M2L per matvec */
  int64_t m2l_pairs;         /* node pairs in interaction lists */
  int64_t operator_bytes;    /* bytes of stored translation operators */
  int64_t device_bytes;      /* total device bytes owned by the handle */
  double mean_rank_leaf_in, mean_rank_leaf_out;
  int32_t max_rank;
  double setup_tree_s, setup_lists_s, setup_nca_s, setup_ops_s, setup_pack_s, setup_upload_s;
  int64_t aca_entries;       /* kernel entries evaluated by ACA during setup */
  int64_t m2l_band_entries[48]; /* M2L entries per H0 band code (0 generic, 1 near z<=8, 2 near z<=12,
                                    3 near z<=7, 4+b data band b; dafmm_h0_bands) */
  int64_t p2p_band_entries[48]; /* P2P point pairs per band code */
  int32_t m2l_stored;           /* 1: M2L blocks stored in HBM per target node, 2: per node pair
                                   (dafmm_options.m2l_store); 0: evaluated on the fly */
  int64_t m2l_store_bytes;      /* their bytes (0 when evaluated on the fly) */
  int64_t m2l_stream_len;       /* source pivots over all M2L target nodes (multipole gathers per matvec) */
  int64_t n_loc;                /* local-expansion coefficients (M2L outputs) */
  int64_t gmres_reorth;         /* second Gram-Schmidt passes (CGS2) in the last ls_gmres_solve */
  int32_t p2p_symmetric;        /* 1: near-field pairs of different leaves evaluated once (every leaf
                                   has 32 or 64 points); 0: each leaf evaluates all its pairs */
  int64_t m2l_stored_entries;   /* kernel entries in the M2L blocks as stored / streamed per matvec
                                   (m2l_entries / 2 with m2l_store = 2, else m2l_entries) */
  double setup_nca_device_s;    /* part of setup_nca_s spent in the device ACA launches (F2) */
  double setup_ops_device_s;    /* part of setup_upload_s spent forming the operators on the device */
  int32_t level_restricted;     /* 1: every two leaves that share a boundary (edge or corner) are at
                                   most one level apart (the paper's level-restricted tree) */
} dafmm_stats_t;

void dafmm_default_options(dafmm_options* opt);

/* Build the plan on the host (tree, lists, cones, NCA pivots, operators) and
 * upload it to the current CUDA device.
 *   points  host, n x 2 row-major (x1, x2), fp64
 *   weights host, n quadrature weights w_j > 0
 *   q       host, n real contrast values q(x_i)
 *   n, kappa > 0, leaf_size >= 1 (max points per leaf), nca_tol in (0, 1)
 *   out     receives the handle.
 * Synchronous.  Errors: DAFMM_EINVAL, DAFMM_ENOMEM, DAFMM_ECUDA, DAFMM_ESETUP. */
int dafmm_create(const double* points, const double* weights, const double* q, int64_t n, double kappa,
                 int leaf_size, double nca_tol, dafmm_handle* out);
int dafmm_create_ex(const double* points, const double* weights, const double* q, int64_t n, double kappa,
                    int leaf_size, double nca_tol, const dafmm_options* opt, dafmm_handle* out);

/* y = A x (see the top of this file).  x, y: DEVICE pointers, n complex128 each, caller order,
 * no aliasing.  Enqueued on the handle's stream; returns immediately. */
int dafmm_matvec(dafmm_handle h, const void* x, void* y);

/* As dafmm_matvec with only some passes: mask bit 0 = near field (P2P, including
 * the identity and self term), bit 1 = far field (upward, transverse and downward passes,
 * P:667-748).  mask 3 equals dafmm_matvec.  For mask 2 the identity term is omitted. */
#define DAFMM_PART_NEAR 1u
#define DAFMM_PART_FAR 2u
int dafmm_matvec_parts(dafmm_handle h, const void* x, void* y, unsigned mask);

/* As dafmm_matvec with HOST buffers: copies x to the device, applies A, copies y back, and
 * synchronises the handle's stream before returning (the end-to-end path of bench.py). */
int dafmm_matvec_host(dafmm_handle h, const void* x_host, void* y_host);

/* Restarted GMRES(m) (reading R14: zero initial guess, m = restart (<= 0: 50,
 * at most 255), classical Gram-Schmidt with re-orthogonalisation on the device) for A psi = f
 * with the DAFMM product.  f, psi: DEVICE pointers (n complex128, caller order; psi is
 * overwritten).  A restart cycle ends when its implicit (Givens) relative residual <= tol or
 * at maxit inner iterations; the true relative residual ||f - A psi|| / ||f|| is recomputed at
 * every restart and decides convergence (a cycle whose implicit residual met tol while the true
 * one did not is followed by another).  *relres_out receives the final true relative residual.
 * history (nullable, host, maxit + 1 doubles) receives the implicit residual per iteration.
 * The first call (and a call with a different restart) allocates the device workspace:
 * (restart + 3) n complex128 plus small buffers; later calls allocate nothing.
 * Synchronous.  Returns DAFMM_OK (true relres <= tol), DAFMM_NOT_CONVERGED (maxit reached),
 * or an error code (DAFMM_EINVAL: tol <= 0, maxit < 1, restart > 255, f == psi). */
int ls_gmres_solve(dafmm_handle h, const void* f, void* psi, double tol, int maxit, int restart, int* iters_out,
                   double* relres_out, double* history);

/* Use stream s (a cudaStream_t) for all later device work of the handle.  Work already enqueued
 * on the previous stream is ordered before any later work on s (the handle's scratch buffers
 * are shared): s waits on an event recorded on the previous stream. */
int dafmm_set_stream(dafmm_handle h, void* stream);

/* Statistics of the plan (sizes, ranks, setup wall times).  Host only; never fails on a
 * valid handle. */
int dafmm_stats(dafmm_handle h, dafmm_stats_t* out);

/* Per-pass profiling (SURVEY §5 "CUDA events per pass").  dafmm_set_profiling(h, 1) creates
 * CUDA events around each pass of every later matvec and resets the accumulators and the
 * kernel-launch counter; 0 switches event recording off (the counter keeps counting).
 * dafmm_pass_times synchronises on the last profiled matvec and writes the accumulated
 * milliseconds per pass into ms_out[DAFMM_NUM_PASSES], in the order
 *   0 gather (caller order -> tree order, w scaling)
 *   1 P2M (plus the memsets of the expansion buffers)
 *   2 M2M, all levels     3 M2L, all levels but the deepest
 *   4 L2L, all levels
 *   5 near field P2P (on the handle's internal side stream, concurrent with 1-4)
 *   6 combine: L2P + identity + self term + scatter
 *   7 span of the concurrent part: from the fork after the gather to the later of 4 and 5
 *   8 M2L of the deepest level when it runs on a third internal stream from the end of P2M
 *     (build option DAFMM_LEAF_SPLIT; 0 otherwise, the deepest level then being part of 3)
 * plus the number of profiled matvecs and the number of kernels launched by the library since
 * the last reset (either pointer may be NULL).  Passes 1-4 and 5 overlap in time, so their sum
 * exceeds the matvec time; 0 + 7 + 6 is the matvec time.  Errors: DAFMM_EINVAL (null handle /
 * host-only plan), DAFMM_ECUDA. */
#define DAFMM_NUM_PASSES 9
int dafmm_set_profiling(dafmm_handle h, int enable);
int dafmm_pass_times(dafmm_handle h, double* ms_out, int64_t* matvecs_out, int64_t* launches_out);

/* The product's H0^(1) evaluator, exposed band by band for the parity tests (DESIGN.md section 6,
 * "H0 evaluator"; the kernel G = (i/4) H0^(1)(kappa |x - y|) is P:70-72, and the paper leaves
 * the evaluation method open).
 * dafmm_h0_bands writes, for every band code c < min(cap, return value), the z = kappa r
 * interval the band is valid on: zlo[c] < z <= zhi[c] for the near bands (1: z <= 8,
 * 2: z <= 12, 3: z <= 7; zlo = 0), zlo[c] <= z <= zhi[c] for the data bands c >= 4, and
 * (0, inf) for code 0 (generic: near-8 or the asymptotic form, chosen per element).  Either
 * pointer may be NULL.  Returns the number of band codes.  Host only, no GPU needed.
 * dafmm_h0_eval: h0[i] = H0^(1)(sqrt(z2[i])) = J0 + i Y0 (complex128 interleaved), z2 =
 * (kappa r)^2 > 0, by band `band`'s evaluator, in the same lane-blocked code as the P2P and M2L
 * kernels.  z2, h0: DEVICE pointers (n doubles / n complex128, caller-owned); enqueued on
 * `stream` (a cudaStream_t; NULL = the legacy default stream), asynchronous.  Arguments
 * outside the band's interval give unspecified (finite) values.  Errors: DAFMM_EINVAL
 * (n < 0, null pointer with n > 0, band code out of range), DAFMM_ECUDA (launch). */
int dafmm_h0_bands(double* zlo, double* zhi, int cap);
int dafmm_h0_eval(const void* z2, void* h0, int64_t n, int band, void* stream);

/* ---- HODLR preconditioner and hybrid solver (Eq. hybrid; readings HR1-HR4) ----
 * Ã is a Hierarchically Off-Diagonal Low-Rank approximation of the handle's matrix A (kernel_mode
 * 0) in the handle's tree order: a binary tree of midpoint splits of the tree positions with
 * leaves of at most leaf_size points (HR1); the leaf diagonal blocks of A are kept dense, and
 * every off-diagonal sibling block A[alpha, beta] is replaced by its cross approximation
 * A[alpha, J] A[I, J]^{-1} A[I, beta] with pivots from partially pivoted ACA capped at rank
 * `rank` ("apriori fixing the rank"; HR2).  Ã is factorised on the device by the recursive
 * Sherman-Morrison-Woodbury form (HR3): O(N r log N) memory, O(N r log N) per solve.
 *
 * dafmm_hodlr_create: rank in [1, 32], leaf_size in [1, 64]; max_block >= 0: sibling blocks with
 *   more than max_block rows are dropped (rank 0; reading HR5, an option: 0 keeps every block, as
 *   the paper's HODLR does).  Synchronous.  The preconditioner
 *   refers to the handle's device plan: destroy it before the handle.  Errors: DAFMM_EINVAL
 *   (arguments, host-only plan, kernel_mode 1), DAFMM_ENOMEM / DAFMM_ECUDA, DAFMM_ESETUP
 *   (singular leaf block, cross matrix or Woodbury factor).
 * dafmm_hodlr_solve: x = Ã^{-1} b (the HODLR direct solver), b and x DEVICE pointers, n
 *   complex128, caller order (b may equal x).  Enqueued on the handle's stream.
 * dafmm_hodlr_export: writes hodlr_blocks.npy (nblocks x 5: depth, a, b, c, d for the block of
 *   rows [a, b) and columns [c, d) of tree positions), hodlr_piv_ptr.npy, hodlr_I.npy,
 *   hodlr_J.npy (pivots, tree positions), hodlr_perm.npy (tree position -> caller index) and
 *   hodlr_meta.npy (rank, leaf_size, n, max_block) into directory `path`, for the oracle.
 * ls_gmres_solve_prec: as ls_gmres_solve on the right-preconditioned system A Ã^{-1} u = f,
 *   psi = Ã^{-1} u (HR4: the paper writes the left form; the right form keeps the GMRES residual
 *   equal to the true residual ||A psi - f|| / ||f||).  p = NULL gives ls_gmres_solve. */
typedef struct dafmm_hodlr_s* dafmm_hodlr;
typedef struct {
  int32_t rank, leaf_size, depths, leaves, max_rank;
  double mean_rank;
  int64_t max_block;
  int64_t device_bytes, aca_entries;
  double setup_aca_s, setup_basis_s, setup_factor_s;
} dafmm_hodlr_stats_t;
int dafmm_hodlr_create(dafmm_handle h, int rank, int leaf_size, int64_t max_block, dafmm_hodlr* out);
int dafmm_hodlr_solve(dafmm_hodlr p, const void* b, void* x);
int dafmm_hodlr_stats(dafmm_hodlr p, dafmm_hodlr_stats_t* out);
int dafmm_hodlr_export(dafmm_hodlr p, const char* path);
void dafmm_hodlr_destroy(dafmm_hodlr p);
int ls_gmres_solve_prec(dafmm_handle h, dafmm_hodlr p, const void* f, void* psi, double tol, int maxit, int restart,
                        int* iters_out, double* relres_out, double* history);

/* Write the tree, lists, cones and pivot index sets as .npy files into directory `path`
 * (created if missing) for the independent CPU oracle.  Synchronous, host only. */
int dafmm_export_plan(dafmm_handle h, const char* path);

void dafmm_destroy(dafmm_handle h);

/* Thread-local message of the last failed call on this thread ("" if none). */
const char* dafmm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DAFMM_H */
