"""A/B probe of plan options on one config: per option set, setup time, median / min matvec time
(CUDA events, L2 flushed between steps), per-pass times (a separate profiled run), M2L sizes and
the sampled error against the oracle's dense rows.

    python tools/mode_probe.py c4 '{"m2l_store": 1}' '{"symmetric_pivots": 1, "m2l_store": 2}'
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2204_00326_b200 as prod  # noqa: E402
from oracle.core import Problem  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1]
sets = [json.loads(a) for a in sys.argv[2:]] or [{}]
rows = int(os.environ.get("PROBE_ROWS", "64"))
steps = int(os.environ.get("PROBE_STEPS", "20"))
P = make_problem(name)
n = P["points"].shape[0]
prob = Problem(P["points"], P["weights"], P["q"], P["kappa"])
idx = np.sort(np.random.default_rng(5).choice(n, size=min(rows, n), replace=False))
yd = oracle.dense_matvec_rows(prob, P["x"], idx) if rows else None
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = os.environ.get("DAFMM_LIB_NAME", "libdafmm.so")
for opts in sets:
    t0 = time.perf_counter()
    opts = dict(opts)
    tol = opts.pop("nca_tol", P["nca_tol"])  # probe-only key: another ACA tolerance
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, tol, **opts)
    setup = time.perf_counter() - t0
    st = op.stats()
    s = torch.cuda.Stream()
    op.set_stream(s)
    x = torch.from_numpy(P["x"]).cuda()
    y = torch.empty_like(x)

    def run(k):
        ts = []
        for _ in range(k):
            with torch.cuda.stream(s):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            op.matvec(x, y)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return ts

    def run_parts(k, mask):
        ts = []
        for _ in range(k):
            with torch.cuda.stream(s):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            op.matvec(x, y, mask)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    run(3)
    far_only = run_parts(steps, 2)   # isolated: no P2P beside the far field
    near_only = run_parts(steps, 1)
    op.set_profiling(True)
    run_parts(steps, 2)
    far_passes, fcnt, _ = op.pass_times()
    op.set_profiling(False)
    ts = run(steps)
    op.set_profiling(True)
    run(steps)
    passes, cnt, launches = op.pass_times()
    op.set_profiling(False)
    err = None
    if rows:
        yg = y.cpu().numpy()[idx]
        xs = P["x"][idx]
        err = float(np.linalg.norm((yg - xs) - (yd - xs)) / np.linalg.norm(yd - xs))
    print(json.dumps(dict(config=name, lib=lib, opts=opts, setup_s=round(setup, 2), setup_nca_s=round(st["setup_nca_s"], 2),
                          setup_detail={k: round(st[k], 3) for k in ("setup_tree_s", "setup_lists_s", "setup_nca_s",
                                                                     "setup_nca_device_s", "setup_ops_s",
                                                                     "setup_upload_s", "setup_ops_device_s")},
                          ms_median=statistics.median(ts), ms_min=min(ts), far_only_ms=far_only,
                          near_only_ms=near_only,
                          far_only_passes={k: round(v / max(fcnt, 1), 4) for k, v in far_passes.items()
                                           if k in ("p2m", "m2m", "m2l", "l2l")},
                          passes={k: round(v / max(cnt, 1), 4) for k, v in passes.items()},
                          launches_per_mv=launches / max(cnt, 1), m2l_stored=st["m2l_stored"],
                          m2l_entries=st["m2l_entries"], m2l_stored_entries=st["m2l_stored_entries"],
                          m2l_stream_len=st["m2l_stream_len"], n_loc=st["n_loc"], device_gb=st["device_bytes"] / 1e9,
                          rank_leaf_in=st["mean_rank_leaf_in"], max_rank=st["max_rank"], sampled_err=err)), flush=True)
    op.close()
