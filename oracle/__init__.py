"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the product's hot path
computes: the discrete Lippmann-Schwinger operator of arxiv 2204.00326 applied to a
vector, both by its plain definition (dense O(N^2) sum) and by the paper's
Directional Algebraic FMM step by step (tree and lists P:273-384, nested cross
approximation, the DAFMM passes P:643-755), plus restarted GMRES.

Who may import this package: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg.  Nothing under paper_2204_00326_b200/ imports it,
and it imports nothing from there.  The two implementations share no code; the only shared
module is synth/ (seeded input generators, none of the method's arithmetic).

Precision: complex fp64 throughout.  Every function cites the PAPER.md line ("P:<n>") it
follows; readings of silent/ambiguous passages are the R-numbers of DESIGN.md.

Parity pins (tests/test_oracle_*.py, ``-m "not gpu"``): H0 against mpmath and printed
values, Wronskian, symmetry; the self term against mpmath quadrature; the dense product
against closed-form special cases; lists by brute-force pair completeness; ACA on exact
low-rank matrices; the serial DAFMM against the dense product within 10 x nca_tol (this
bound is the north-star contract: the paper prints no matvec-error values, so the DAFMM
itself is "parity unpinned" beyond that bound — see DESIGN.md §Oracle).
"""
from .core import (h0, h1_small, self_terms, A_block, K_block, dense_matvec, dense_matvec_rows,  # noqa: F401
                   load_library, Problem)
