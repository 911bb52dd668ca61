"""B200-native DAFMM matvec and GMRES for the 2D Lippmann-Schwinger equation (arxiv 2204.00326).

The compute path is the C-ABI library ``_lib/libdafmm.so`` (include/dafmm.h): host setup in
C++ and sm_100a CUDA kernels.  This package is a thin ctypes binding with the same names —
argument marshalling only; there is no CPU fallback: importing fails loudly if the library
is missing (run ``python -m paper_2204_00326_b200.build`` or ``__graft_entry__.build()``).
"""
from .binding import (DAFMMError, Options, Stats, dafmm_create, dafmm_create_ex, dafmm_matvec,  # noqa: F401
                      dafmm_matvec_parts, dafmm_matvec_host, ls_gmres_solve, dafmm_set_stream, dafmm_stats,
                      dafmm_export_plan, dafmm_destroy, dafmm_last_error, dafmm_set_profiling,
                      dafmm_pass_times, dafmm_h0_bands, dafmm_h0_eval, library_path, load, DAFMM, EXPORTED, PASS_NAMES, HODLR, HodlrStats,
                      dafmm_hodlr_create, dafmm_hodlr_solve, dafmm_hodlr_stats, dafmm_hodlr_export,
                      dafmm_hodlr_destroy, ls_gmres_solve_prec)
