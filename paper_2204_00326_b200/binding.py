"""ctypes binding of include/dafmm.h (argument marshalling only).

Device vectors are torch CUDA tensors of dtype complex128 (or raw integer device pointers);
host arrays are numpy.  Functions mirror the C names; ``DAFMM`` is a small owning wrapper.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_lib", os.environ.get("DAFMM_LIB_NAME") or "libdafmm.so")
_lib = None

EXPORTED = ["dafmm_default_options", "dafmm_create", "dafmm_create_ex", "dafmm_matvec", "dafmm_matvec_parts",
            "dafmm_matvec_host", "ls_gmres_solve", "dafmm_set_stream", "dafmm_stats", "dafmm_export_plan",
            "dafmm_destroy", "dafmm_last_error", "dafmm_set_profiling", "dafmm_pass_times", "dafmm_h0_bands",
            "dafmm_h0_eval", "dafmm_hodlr_create", "dafmm_hodlr_solve", "dafmm_hodlr_stats", "dafmm_hodlr_export",
            "dafmm_hodlr_destroy", "ls_gmres_solve_prec"]

NUM_PASSES = 9
PASS_NAMES = ["gather", "p2m", "m2m", "m2l", "l2l", "near", "combine", "overlap_span", "m2l_leaf"]

DAFMM_OK, DAFMM_NOT_CONVERGED = 0, 1
ERRORS = {-1: "DAFMM_EINVAL", -2: "DAFMM_ECUDA", -3: "DAFMM_ENOMEM", -4: "DAFMM_ESETUP"}


class DAFMMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s: %s" % (ERRORS.get(code, code), msg))
        self.code = code


class Options(ctypes.Structure):
    _fields_ = [("T", ctypes.c_double), ("self_term", ctypes.c_int), ("kernel_mode", ctypes.c_int),
                ("max_level", ctypes.c_int), ("num_threads", ctypes.c_int), ("host_only", ctypes.c_int),
                ("symmetric_pivots", ctypes.c_int), ("m2l_store", ctypes.c_int),
                ("hfr_parent_search", ctypes.c_int), ("setup_device", ctypes.c_int),
                ("w_reading", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("levels", ctypes.c_int32), ("n_nodes", ctypes.c_int32),
                ("p2p_pairs", ctypes.c_int64), ("m2l_entries", ctypes.c_int64), ("m2l_pairs", ctypes.c_int64),
                ("operator_bytes", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("mean_rank_leaf_in", ctypes.c_double), ("mean_rank_leaf_out", ctypes.c_double),
                ("max_rank", ctypes.c_int32),
                ("setup_tree_s", ctypes.c_double), ("setup_lists_s", ctypes.c_double),
                ("setup_nca_s", ctypes.c_double), ("setup_ops_s", ctypes.c_double),
                ("setup_pack_s", ctypes.c_double), ("setup_upload_s", ctypes.c_double),
                ("aca_entries", ctypes.c_int64), ("m2l_band_entries", ctypes.c_int64 * 48),
                ("p2p_band_entries", ctypes.c_int64 * 48), ("m2l_stored", ctypes.c_int32),
                ("m2l_store_bytes", ctypes.c_int64), ("m2l_stream_len", ctypes.c_int64), ("n_loc", ctypes.c_int64),
                ("gmres_reorth", ctypes.c_int64), ("p2p_symmetric", ctypes.c_int32),
                ("m2l_stored_entries", ctypes.c_int64), ("setup_nca_device_s", ctypes.c_double),
                ("setup_ops_device_s", ctypes.c_double), ("level_restricted", ctypes.c_int32)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        for k in ("m2l_band_entries", "p2p_band_entries"):
            d[k] = list(d[k])
        return d


class HodlrStats(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("leaf_size", ctypes.c_int32), ("depths", ctypes.c_int32),
                ("leaves", ctypes.c_int32), ("max_rank", ctypes.c_int32), ("mean_rank", ctypes.c_double),
                ("max_block", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("aca_entries", ctypes.c_int64), ("setup_aca_s", ctypes.c_double),
                ("setup_basis_s", ctypes.c_double), ("setup_factor_s", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def library_path():
    return _LIB_PATH


def load():
    """Load the C-ABI library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError("libdafmm.so not built: run `python -m paper_2204_00326_b200.build`")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, dbl, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    lib.dafmm_default_options.argtypes = [ctypes.POINTER(Options)]
    lib.dafmm_create.argtypes = [vp, vp, vp, i64, dbl, i32, dbl, ctypes.POINTER(vp)]
    lib.dafmm_create_ex.argtypes = [vp, vp, vp, i64, dbl, i32, dbl, ctypes.POINTER(Options), ctypes.POINTER(vp)]
    lib.dafmm_matvec.argtypes = [vp, vp, vp]
    lib.dafmm_matvec_parts.argtypes = [vp, vp, vp, ctypes.c_uint]
    lib.dafmm_matvec_host.argtypes = [vp, vp, vp]
    lib.ls_gmres_solve.argtypes = [vp, vp, vp, dbl, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(dbl), vp]
    lib.dafmm_set_stream.argtypes = [vp, vp]
    lib.dafmm_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    lib.dafmm_export_plan.argtypes = [vp, ctypes.c_char_p]
    lib.dafmm_set_profiling.argtypes = [vp, i32]
    lib.dafmm_pass_times.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.dafmm_h0_bands.argtypes = [vp, vp, i32]
    lib.dafmm_h0_eval.argtypes = [vp, vp, i64, i32, vp]
    lib.dafmm_hodlr_create.argtypes = [vp, i32, i32, i64, ctypes.POINTER(vp)]
    lib.dafmm_hodlr_solve.argtypes = [vp, vp, vp]
    lib.dafmm_hodlr_stats.argtypes = [vp, ctypes.POINTER(HodlrStats)]
    lib.dafmm_hodlr_export.argtypes = [vp, ctypes.c_char_p]
    lib.dafmm_hodlr_destroy.argtypes = [vp]
    lib.dafmm_hodlr_destroy.restype = None
    lib.ls_gmres_solve_prec.argtypes = [vp, vp, vp, vp, dbl, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(dbl), vp]
    lib.dafmm_destroy.argtypes = [vp]
    lib.dafmm_destroy.restype = None
    lib.dafmm_last_error.restype = ctypes.c_char_p
    lib.dafmm_last_error.argtypes = []
    _lib = lib
    return lib


def dafmm_last_error():
    return load().dafmm_last_error().decode()


def _check(rc):
    if rc < 0:
        raise DAFMMError(rc, dafmm_last_error())
    return rc


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def _dev(t, n=None):
    """Device pointer of a torch CUDA complex128 tensor (or an int pointer, unchecked); with n,
    the tensor must hold exactly n elements (the library reads / writes n of them)."""
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    if not (t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.complex128"):
        raise ValueError("expected a contiguous CUDA complex128 tensor")
    if n is not None and t.numel() != n:
        raise ValueError("expected %d elements, got %d" % (n, t.numel()))
    return ctypes.c_void_p(t.data_ptr())


def _host_vec(a, n, writeable=False):
    """Pointer of a host complex128 vector of exactly n elements, C-contiguous."""
    if not isinstance(a, np.ndarray) or a.dtype != np.complex128:
        raise ValueError("host vectors must be numpy complex128 arrays")
    if not a.flags.c_contiguous or a.size != n or (writeable and not a.flags.writeable):
        raise ValueError("host vector must be C-contiguous%s with %d elements" % (", writeable," if writeable else "", n))
    return a.ctypes.data_as(ctypes.c_void_p)


def default_options():
    o = Options()
    load().dafmm_default_options(ctypes.byref(o))
    return o


def dafmm_create_ex(points, weights, q, kappa, leaf_size, nca_tol, options=None):
    pts, pp = _host(points, np.float64)
    w, wp = _host(weights, np.float64)
    qq, qp = _host(q, np.float64)
    n = w.size
    if pts.size != 2 * n or qq.size != n:
        raise ValueError("points must be (n, 2) and weights, q length n")
    h = ctypes.c_void_p()
    opt = options if options is not None else default_options()
    _check(load().dafmm_create_ex(pp, wp, qp, n, float(kappa), int(leaf_size), float(nca_tol), ctypes.byref(opt),
                                  ctypes.byref(h)))
    _N_CACHE[h.value] = n
    return h


def dafmm_create(points, weights, q, kappa, leaf_size, nca_tol):
    return dafmm_create_ex(points, weights, q, kappa, leaf_size, nca_tol, None)


_N_CACHE = {}  # handle value -> n (dafmm_create_ex fills it; a handle's n never changes)


def _n_of(h):
    key = h.value if isinstance(h, ctypes.c_void_p) else int(h)
    n = _N_CACHE.get(key)
    if n is None:
        s = Stats()
        _check(load().dafmm_stats(h, ctypes.byref(s)))
        n = _N_CACHE[key] = int(s.n)
    return n


def dafmm_matvec(h, x, y):
    n = _n_of(h)
    return _check(load().dafmm_matvec(h, _dev(x, n), _dev(y, n)))


def dafmm_matvec_parts(h, x, y, mask):
    n = _n_of(h)
    return _check(load().dafmm_matvec_parts(h, _dev(x, n), _dev(y, n), int(mask)))


def dafmm_matvec_host(h, x_host, y_host):
    """x_host, y_host: C-contiguous numpy complex128 arrays of n elements (pinned torch tensors
    are accepted via .numpy())."""
    n = _n_of(h)
    return _check(load().dafmm_matvec_host(h, _host_vec(x_host, n), _host_vec(y_host, n, writeable=True)))


def ls_gmres_solve(h, f, psi, tol, maxit, restart=50, history=None):
    """Returns (status, iterations, true relative residual); history: numpy float64 (maxit+1) or None."""
    it = ctypes.c_int()
    rr = ctypes.c_double()
    hp = None
    if history is not None:
        if history.dtype != np.float64 or history.size < maxit + 1:
            raise ValueError("history must be float64 with maxit + 1 entries")
        hp = history.ctypes.data_as(ctypes.c_void_p)
    n = _n_of(h)
    rc = _check(load().ls_gmres_solve(h, _dev(f, n), _dev(psi, n), float(tol), int(maxit), int(restart), ctypes.byref(it),
                                      ctypes.byref(rr), hp))
    return rc, it.value, rr.value


def _history_ptr(history, maxit):
    if history is None:
        return None
    if history.dtype != np.float64 or history.size < maxit + 1:
        raise ValueError("history must be float64 with maxit + 1 entries")
    return history.ctypes.data_as(ctypes.c_void_p)


def dafmm_hodlr_create(h, rank, leaf_size=64, max_block=0):
    p = ctypes.c_void_p()
    _check(load().dafmm_hodlr_create(h, int(rank), int(leaf_size), int(max_block), ctypes.byref(p)))
    return p


def dafmm_hodlr_solve(p, h, b, x):
    """x = Ã^{-1} b on the device (h: the owning DAFMM handle, for the length check)."""
    n = _n_of(h)
    return _check(load().dafmm_hodlr_solve(p, _dev(b, n), _dev(x, n)))


def dafmm_hodlr_stats(p):
    s = HodlrStats()
    _check(load().dafmm_hodlr_stats(p, ctypes.byref(s)))
    return s.as_dict()


def dafmm_hodlr_export(p, path):
    return _check(load().dafmm_hodlr_export(p, str(path).encode()))


def dafmm_hodlr_destroy(p):
    if p:
        load().dafmm_hodlr_destroy(p)


def ls_gmres_solve_prec(h, p, f, psi, tol, maxit, restart=50, history=None):
    """Right-preconditioned GMRES (HR4); returns (status, iterations, true relative residual)."""
    it = ctypes.c_int()
    rr = ctypes.c_double()
    n = _n_of(h)
    rc = _check(load().ls_gmres_solve_prec(h, p, _dev(f, n), _dev(psi, n), float(tol), int(maxit), int(restart),
                                           ctypes.byref(it), ctypes.byref(rr), _history_ptr(history, maxit)))
    return rc, it.value, rr.value


def dafmm_set_stream(h, stream):
    """stream: a torch.cuda.Stream or a raw cudaStream_t integer."""
    ptr = stream if isinstance(stream, int) else stream.cuda_stream
    return _check(load().dafmm_set_stream(h, ctypes.c_void_p(ptr)))


def dafmm_stats(h):
    s = Stats()
    _check(load().dafmm_stats(h, ctypes.byref(s)))
    return s.as_dict()


def dafmm_set_profiling(h, enable):
    return _check(load().dafmm_set_profiling(h, int(bool(enable))))


def dafmm_pass_times(h):
    """Returns ({pass name: accumulated ms}, profiled matvecs, kernel launches since reset)."""
    ms = (ctypes.c_double * NUM_PASSES)()
    cnt, launches = ctypes.c_int64(), ctypes.c_int64()
    _check(load().dafmm_pass_times(h, ms, ctypes.byref(cnt), ctypes.byref(launches)))
    return dict(zip(PASS_NAMES, list(ms))), cnt.value, launches.value


def dafmm_export_plan(h, path):
    return _check(load().dafmm_export_plan(h, str(path).encode()))


def dafmm_h0_bands():
    """[(zlo, zhi)] per band code: the z = kappa r interval each evaluator band is valid on."""
    lib = load()
    nb = _check(lib.dafmm_h0_bands(None, None, 0))
    lo, hi = (ctypes.c_double * nb)(), (ctypes.c_double * nb)()
    lib.dafmm_h0_bands(ctypes.cast(lo, ctypes.c_void_p), ctypes.cast(hi, ctypes.c_void_p), nb)
    return list(zip(list(lo), list(hi)))


def dafmm_h0_eval(z2, out, band, stream=None):
    """out = H0^(1)(sqrt(z2)) by band `band`: z2 a CUDA float64 tensor, out CUDA complex128 (same n)."""
    if not (z2.is_cuda and z2.is_contiguous() and str(z2.dtype) == "torch.float64"):
        raise ValueError("z2 must be a contiguous CUDA float64 tensor")
    if out.numel() != z2.numel():
        raise ValueError("out must have z2's length")
    ptr = 0 if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
    return _check(load().dafmm_h0_eval(ctypes.c_void_p(z2.data_ptr()), _dev(out), z2.numel(), int(band),
                                       ctypes.c_void_p(ptr)))


def dafmm_destroy(h):
    if h:
        _N_CACHE.pop(h.value if isinstance(h, ctypes.c_void_p) else int(h), None)
        load().dafmm_destroy(h)


class DAFMM:
    """Owning wrapper: ``op = DAFMM(points, w, q, kappa, leaf_size, nca_tol); op.matvec(x, y)``."""

    def __init__(self, points, weights, q, kappa, leaf_size=64, nca_tol=1e-8, **opts):
        o = default_options()
        for k, v in opts.items():
            setattr(o, k, v)
        self.h = dafmm_create_ex(points, weights, q, kappa, leaf_size, nca_tol, o)
        self.n = int(np.asarray(weights).size)

    def set_stream(self, stream):
        dafmm_set_stream(self.h, stream)

    def matvec(self, x, y, mask=3):
        if mask == 3:
            dafmm_matvec(self.h, x, y)
        else:
            dafmm_matvec_parts(self.h, x, y, mask)
        return y

    def matvec_host(self, x_host, y_host):
        dafmm_matvec_host(self.h, x_host, y_host)
        return y_host

    def gmres(self, f, psi, tol, maxit, restart=50, history=None, prec=None):
        """prec: a HODLR of this operator (right preconditioning, HR4) or None."""
        if prec is not None:
            return ls_gmres_solve_prec(self.h, prec.p, f, psi, tol, maxit, restart, history)
        return ls_gmres_solve(self.h, f, psi, tol, maxit, restart, history)

    def stats(self):
        return dafmm_stats(self.h)

    def set_profiling(self, enable=True):
        dafmm_set_profiling(self.h, enable)

    def pass_times(self):
        return dafmm_pass_times(self.h)

    def export_plan(self, path):
        dafmm_export_plan(self.h, path)

    def close(self):
        if self.h:
            dafmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HODLR:
    """Owning wrapper of the HODLR preconditioner of a DAFMM operator:
    ``pc = HODLR(op, rank=16, leaf_size=64); pc.solve(b, x); op.gmres(f, psi, tol, maxit, prec=pc)``."""

    def __init__(self, op, rank=16, leaf_size=64, max_block=0):
        self.op = op  # keeps the owning handle alive
        self.p = dafmm_hodlr_create(op.h, rank, leaf_size, max_block)

    def solve(self, b, x):
        dafmm_hodlr_solve(self.p, self.op.h, b, x)
        return x

    def stats(self):
        return dafmm_hodlr_stats(self.p)

    def export(self, path):
        dafmm_hodlr_export(self.p, path)

    def close(self):
        if self.p:
            dafmm_hodlr_destroy(self.p)
            self.p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
