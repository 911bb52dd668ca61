// C-ABI of include/dafmm.h: argument checking, error plumbing, handle lifetime.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "dafmm.h"
#include "device.h"
#include "hankel.cuh"
#include "hodlr.h"
#include "plan.h"

struct dafmm_plan {
  dafmm::Plan plan;
  dafmm::DevPlan dev;
  int64_t operator_bytes = 0;
  int64_t p2p_pairs = 0, m2l_entries = 0, m2l_pairs = 0, m2l_stream_len = 0, n_loc = 0, m2l_stored_entries = 0;
  int m2l_sym = 0;
  int p2p_sym = 0;
  std::vector<int64_t> m2l_band, p2p_band;
};

struct dafmm_hodlr_s {
  dafmm_plan* owner = nullptr;
  dafmm::HodlrPlan hp;
};

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

void dafmm_default_options(dafmm_options* opt) {
  if (!opt) return;
  dafmm::Options o;
  opt->T = o.T;
  opt->self_term = o.self_term;
  opt->kernel_mode = o.kernel_mode;
  opt->max_level = o.max_level;
  opt->num_threads = o.num_threads;
  opt->host_only = o.host_only;
  opt->symmetric_pivots = o.symmetric_pivots;
  opt->m2l_store = o.m2l_store;
  opt->hfr_parent_search = o.hfr_parent_search;
  opt->setup_device = o.setup_device;
  opt->w_reading = o.w_reading;
}

int dafmm_create_ex(const double* points, const double* weights, const double* q, int64_t n, double kappa,
                    int leaf_size, double nca_tol, const dafmm_options* opt, dafmm_handle* out) {
  if (!out) return fail(DAFMM_EINVAL, "out is null");
  *out = nullptr;
  dafmm::Options o;
  if (opt) {
    o.T = opt->T;
    o.self_term = opt->self_term;
    o.kernel_mode = opt->kernel_mode;
    o.max_level = opt->max_level;
    o.num_threads = opt->num_threads;
    o.host_only = opt->host_only;
    o.symmetric_pivots = opt->symmetric_pivots;
    o.m2l_store = opt->m2l_store;
    o.hfr_parent_search = opt->hfr_parent_search;
    o.setup_device = opt->setup_device;
    o.w_reading = opt->w_reading;
    if (o.m2l_store < -1 || o.m2l_store > 2) return fail(DAFMM_EINVAL, "m2l_store must be -1, 0, 1 or 2");
  }
  std::unique_ptr<dafmm_plan> h;
  try {
    h.reset(new dafmm_plan());
  } catch (const std::bad_alloc&) {
    return fail(DAFMM_ENOMEM, "host allocation failed");
  }
  std::string err;
  int rc;
  try {
    rc = dafmm::build_plan(h->plan, points, weights, q, n, kappa, leaf_size, nca_tol, o, err);
    if (rc != DAFMM_OK) return fail(rc, err);
    double t0 = now_s();
    dafmm::Packed pk;
    size_t free_b = 0, total_b = 0;
    if (!o.host_only && cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
    rc = dafmm::pack_plan(h->plan, pk, err, free_b);
    if (rc != DAFMM_OK) return fail(rc, err);
    double t1 = now_s();
    h->plan.t_ops = t1 - t0;
    if (!o.host_only) {
      rc = dafmm::upload_plan(pk, h->plan, h->dev, err);
      if (rc != DAFMM_OK) {
        dafmm::free_plan(h->dev);
        return fail(rc, err);
      }
      h->plan.t_upload = now_s() - t1;
    }
    h->operator_bytes = (int64_t)pk.ops_len * 16;
    h->p2p_pairs = pk.p2p_pairs;
    h->m2l_entries = pk.m2l_entries;
    h->m2l_stored_entries = pk.m2l_stored_entries;
    h->m2l_sym = pk.m2l_sym;
    h->m2l_pairs = pk.m2l_pairs;
    h->m2l_stream_len = (int64_t)pk.m2l_stream_idx.size();
    h->n_loc = pk.n_loc;
    h->p2p_sym = pk.p2p_sym;
    h->m2l_band = pk.m2l_band_entries;
    h->p2p_band = pk.p2p_band_entries;
  } catch (const std::bad_alloc&) {
    dafmm::free_plan(h->dev);
    return fail(DAFMM_ENOMEM, "host allocation failed during setup");
  }
  *out = h.release();
  g_last_error.clear();
  return DAFMM_OK;
}

int dafmm_create(const double* points, const double* weights, const double* q, int64_t n, double kappa, int leaf_size,
                 double nca_tol, dafmm_handle* out) {
  return dafmm_create_ex(points, weights, q, n, kappa, leaf_size, nca_tol, nullptr, out);
}

int dafmm_matvec_parts(dafmm_handle h, const void* x, void* y, unsigned mask) {
  if (!h || !x || !y) return fail(DAFMM_EINVAL, "null handle or vector");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  if (x == y) return fail(DAFMM_EINVAL, "x and y must not alias");
  if ((mask & 3u) == 0 || (mask & ~3u)) return fail(DAFMM_EINVAL, "mask must be a non-empty subset of {1, 2}");
  std::string err;
  int rc = dafmm::run_matvec(h->dev, (const double2*)x, (double2*)y, mask, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

int dafmm_matvec(dafmm_handle h, const void* x, void* y) { return dafmm_matvec_parts(h, x, y, 3u); }

int dafmm_matvec_host(dafmm_handle h, const void* x_host, void* y_host) {
  if (!h || !x_host || !y_host) return fail(DAFMM_EINVAL, "null handle or vector");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  size_t bytes = sizeof(double2) * (size_t)h->dev.n;
  double2* xd = h->dev.host_stage;
  double2* yd = h->dev.host_stage + h->dev.n;
  cudaStream_t s = h->dev.stream;
  cudaError_t e = cudaMemcpyAsync(xd, x_host, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(DAFMM_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
  std::string err;
  int rc = dafmm::run_matvec(h->dev, xd, yd, 3u, err);
  if (rc != DAFMM_OK) return fail(rc, err);
  e = cudaMemcpyAsync(y_host, yd, bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(DAFMM_ECUDA, std::string("D2H: ") + cudaGetErrorString(e));
  return DAFMM_OK;
}

int ls_gmres_solve(dafmm_handle h, const void* f, void* psi, double tol, int maxit, int restart, int* iters_out,
                   double* relres_out, double* history) {
  if (!h || !f || !psi || !iters_out || !relres_out) return fail(DAFMM_EINVAL, "null argument");
  if (f == psi) return fail(DAFMM_EINVAL, "f and psi must not alias");
  if (!(tol > 0.0) || maxit < 1) return fail(DAFMM_EINVAL, "tol must be > 0 and maxit >= 1");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  std::string err;
  int rc = dafmm::run_gmres(h->dev, (const double2*)f, (double2*)psi, tol, maxit, restart, iters_out, relres_out,
                            history, err);
  if (rc < 0) return fail(rc, err);
  return rc;
}

int dafmm_hodlr_create(dafmm_handle h, int rank, int leaf_size, int64_t max_block, dafmm_hodlr* out) {
  if (!out) return fail(DAFMM_EINVAL, "out is null");
  *out = nullptr;
  if (!h) return fail(DAFMM_EINVAL, "null handle");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  std::unique_ptr<dafmm_hodlr_s> p;
  try {
    p.reset(new dafmm_hodlr_s());
    p->owner = h;
    std::string err;
    int rc = dafmm::hodlr_create(h->plan, h->dev, rank, leaf_size, max_block, p->hp, err);
    if (rc != DAFMM_OK) {
      dafmm::hodlr_free(p->hp);
      return fail(rc, err);
    }
  } catch (const std::bad_alloc&) {
    if (p) dafmm::hodlr_free(p->hp);
    return fail(DAFMM_ENOMEM, "host allocation failed (HODLR)");
  }
  *out = p.release();
  g_last_error.clear();
  return DAFMM_OK;
}

int dafmm_hodlr_solve(dafmm_hodlr p, const void* b, void* x) {
  if (!p || !b || !x) return fail(DAFMM_EINVAL, "null argument");
  std::string err;
  int rc = dafmm::hodlr_apply(p->hp, (const double2*)b, (double2*)x, p->owner->dev.stream, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

int dafmm_hodlr_stats(dafmm_hodlr p, dafmm_hodlr_stats_t* out) {
  if (!p || !out) return fail(DAFMM_EINVAL, "null argument");
  const dafmm::HodlrPlan& hp = p->hp;
  std::memset(out, 0, sizeof(*out));
  out->rank = hp.r;
  out->leaf_size = hp.n0;
  out->max_block = hp.max_block;
  out->depths = hp.depths;
  out->leaves = (int32_t)hp.leaf_a.size();
  out->max_rank = hp.max_rank;
  out->mean_rank = hp.mean_rank;
  out->device_bytes = (int64_t)hp.device_bytes;
  out->aca_entries = hp.aca_entries;
  out->setup_aca_s = hp.t_aca;
  out->setup_basis_s = hp.t_basis;
  out->setup_factor_s = hp.t_factor;
  return DAFMM_OK;
}

int dafmm_hodlr_export(dafmm_hodlr p, const char* path) {
  if (!p || !path) return fail(DAFMM_EINVAL, "null argument");
  std::string err;
  int rc = dafmm::hodlr_export(p->hp, p->owner->plan, path, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

void dafmm_hodlr_destroy(dafmm_hodlr p) {
  if (!p) return;
  if (p->owner && p->owner->dev.stream) cudaStreamSynchronize(p->owner->dev.stream);
  else cudaDeviceSynchronize();
  dafmm::hodlr_free(p->hp);
  delete p;
}

int ls_gmres_solve_prec(dafmm_handle h, dafmm_hodlr p, const void* f, void* psi, double tol, int maxit, int restart,
                        int* iters_out, double* relres_out, double* history) {
  if (!h || !f || !psi || !iters_out || !relres_out) return fail(DAFMM_EINVAL, "null argument");
  if (f == psi) return fail(DAFMM_EINVAL, "f and psi must not alias");
  if (!(tol > 0.0) || maxit < 1) return fail(DAFMM_EINVAL, "tol must be > 0 and maxit >= 1");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  if (p && p->owner != h) return fail(DAFMM_EINVAL, "the preconditioner was built for another handle");
  std::string err;
  dafmm::Precond prec;
  if (p)
    prec = [h, p](const double2* v, double2* z, std::string& e) {
      return dafmm::hodlr_apply(p->hp, v, z, h->dev.stream, e);
    };
  int rc = dafmm::run_gmres(h->dev, (const double2*)f, (double2*)psi, tol, maxit, restart, iters_out, relres_out,
                            history, err, prec);
  if (rc < 0) return fail(rc, err);
  return rc;
}

int dafmm_set_stream(dafmm_handle h, void* stream) {
  if (!h) return fail(DAFMM_EINVAL, "null handle");
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->plan.opt.host_only && s != h->dev.stream) {
    // order the new stream after everything pending on the old one: both use the handle's
    // scratch buffers (x_t, mult, loc, phi, slots, GMRES workspace)
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev, h->dev.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
    cudaEventDestroy(ev);
    if (e != cudaSuccess) return fail(DAFMM_ECUDA, std::string("dafmm_set_stream: ") + cudaGetErrorString(e));
  }
  h->dev.stream = s;
  return DAFMM_OK;
}

int dafmm_set_profiling(dafmm_handle h, int enable) {
  if (!h) return fail(DAFMM_EINVAL, "null handle");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  std::string err;
  int rc = dafmm::set_profiling(h->dev, enable != 0, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

int dafmm_pass_times(dafmm_handle h, double* ms_out, int64_t* matvecs_out, int64_t* launches_out) {
  if (!h || !ms_out) return fail(DAFMM_EINVAL, "null argument");
  if (h->plan.opt.host_only) return fail(DAFMM_EINVAL, "host-only plan");
  std::string err;
  int rc = dafmm::harvest_profile(h->dev, err);
  if (rc != DAFMM_OK) return fail(rc, err);
  for (int p = 0; p < dafmm::kNumPasses; ++p) ms_out[p] = h->dev.prof_ms[p];
  if (matvecs_out) *matvecs_out = h->dev.prof_count;
  if (launches_out) *launches_out = h->dev.launches;
  return DAFMM_OK;
}

int dafmm_stats(dafmm_handle h, dafmm_stats_t* out) {
  if (!h || !out) return fail(DAFMM_EINVAL, "null argument");
  std::memset(out, 0, sizeof(*out));
  const dafmm::Plan& P = h->plan;
  out->n = P.n;
  out->levels = P.L;
  int nodes = 0, maxr = 0;
  double rin = 0, rout = 0;
  int leafnodes = 0;
  for (int l = 1; l <= P.L; ++l) {
    nodes += (int)P.levels[l].nodes.size();
    for (auto& np : P.piv[l]) {
      maxr = std::max(maxr, (int)std::max(np.ti.size(), np.so.size()));
      if (l == P.L) {
        rin += (double)np.ti.size();
        rout += (double)np.so.size();
        ++leafnodes;
      }
    }
  }
  out->n_nodes = nodes;
  out->max_rank = maxr;
  out->mean_rank_leaf_in = leafnodes ? rin / leafnodes : 0.0;
  out->mean_rank_leaf_out = leafnodes ? rout / leafnodes : 0.0;
  out->p2p_pairs = h->p2p_pairs;
  out->m2l_entries = h->m2l_entries;
  out->m2l_pairs = h->m2l_pairs;
  out->operator_bytes = h->operator_bytes;
  out->device_bytes = (int64_t)h->dev.device_bytes;
  out->setup_tree_s = P.t_tree;
  out->setup_lists_s = P.t_lists;
  out->setup_nca_s = P.t_nca;
  out->setup_ops_s = P.t_ops;
  out->setup_pack_s = P.t_pack;
  out->setup_nca_device_s = P.t_nca_device;
  out->level_restricted = P.level_restricted ? 1 : 0;
  out->setup_ops_device_s = h->dev.t_ops_device;
  out->setup_upload_s = P.t_upload;
  out->aca_entries = P.aca_entries;
  out->m2l_stored = h->dev.m2l_mat != nullptr ? (h->m2l_sym ? 2 : 1) : 0;
  out->m2l_store_bytes = h->dev.m2l_mat != nullptr ? h->m2l_stored_entries * 16 : 0;
  out->m2l_stored_entries = h->m2l_stored_entries;
  out->m2l_stream_len = h->m2l_stream_len;
  out->n_loc = h->n_loc;
  out->gmres_reorth = h->dev.gm_reorth;
  out->p2p_symmetric = h->p2p_sym;
  for (size_t b = 0; b < h->m2l_band.size() && b < 48; ++b) out->m2l_band_entries[b] = h->m2l_band[b];
  for (size_t b = 0; b < h->p2p_band.size() && b < 48; ++b) out->p2p_band_entries[b] = h->p2p_band[b];
  return DAFMM_OK;
}

int dafmm_export_plan(dafmm_handle h, const char* path) {
  if (!h || !path) return fail(DAFMM_EINVAL, "null argument");
  std::string err;
  int rc = dafmm::export_plan(h->plan, path, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

void dafmm_destroy(dafmm_handle h) {
  if (!h) return;
  if (!h->plan.opt.host_only) {
    if (h->dev.stream) cudaStreamSynchronize(h->dev.stream);
    else cudaDeviceSynchronize();
  }
  dafmm::free_plan(h->dev);
  delete h;
}

const char* dafmm_last_error(void) { return g_last_error.c_str(); }

int dafmm_h0_bands(double* zlo, double* zhi, int cap) {
  const int nb = dafmm::kNumBandCodes;
  for (int c = 0; c < nb && c < cap; ++c) {
    double lo = 0.0, hi = INFINITY;
    if (c == dafmm::kBandNear7) hi = std::sqrt(dafmm_fit::NEAR7_Z2_MAX);
    else if (c == dafmm::kBandNear8) hi = std::sqrt(dafmm_fit::NEAR8_Z2_MAX);
    else if (c == dafmm::kBandNear12) hi = std::sqrt(dafmm_fit::NEAR12_Z2_MAX);
    else if (c >= dafmm::kBandFarData) {
      lo = dafmm_fit::kFarBandsHost[c - dafmm::kBandFarData].zlo;
      hi = dafmm_fit::kFarBandsHost[c - dafmm::kBandFarData].zhi;
    }
    if (zlo) zlo[c] = lo;
    if (zhi) zhi[c] = hi;
  }
  return nb;
}

int dafmm_h0_eval(const void* z2, void* h0, int64_t n, int band, void* stream) {
  if (n < 0) return fail(DAFMM_EINVAL, "n must be >= 0");
  if (n > 0 && (!z2 || !h0)) return fail(DAFMM_EINVAL, "null argument");
  if (band < 0 || band >= dafmm::kNumBandCodes) return fail(DAFMM_EINVAL, "band code out of range");
  std::string err;
  int rc = dafmm::h0_eval((const double*)z2, (double2*)h0, n, band, (cudaStream_t)stream, err);
  return rc == DAFMM_OK ? DAFMM_OK : fail(rc, err);
}

}  // extern "C"
