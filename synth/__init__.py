"""Seeded synthetic inputs shared by the tests, the oracle and the product harness.

This module holds NONE of the method's arithmetic: it only lays out the cell-centred
grids, contrasts q(x), input vectors x and right-hand sides f of BASELINE.json's configs
(recipe in DESIGN.md §Inputs; seeds = reading R13).  Both the oracle and the product are
fed from here; neither is imported by it.
"""
from .configs import CONFIGS, make_problem, grid_points, gaussian_q, disk_q, bumps_q  # noqa: F401
