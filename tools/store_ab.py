"""A/B of the two M2L modes (dafmm_options.m2l_store = 1 stored blocks, 0 on the fly) on one
config: median matvec ms (CUDA events on the handle's stream), per-pass ms, and agreement."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_00326_b200 as prod  # noqa: E402
from synth.configs import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
modes = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 0]
P = make_problem(name)
x = torch.from_numpy(P["x"]).cuda()
ys = {}
for mode in modes:
    t = time.time()
    op = prod.DAFMM(P["points"], P["weights"], P["q"], P["kappa"], 64, P["nca_tol"], m2l_store=mode)
    setup = time.time() - t
    s = torch.cuda.Stream()
    op.set_stream(s)
    y = torch.empty_like(x)
    with torch.cuda.stream(s):
        for _ in range(3):
            op.matvec(x, y)
        s.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            op.matvec(x, y)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        tf, tn = [], []
        for _ in range(reps):  # far field alone, near field alone (no concurrency)
            for mask, acc in ((2, tf), (1, tn)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                op.matvec(x, y, mask)
                e1.record(s)
                e1.synchronize()
                acc.append(e0.elapsed_time(e1))
        op.set_profiling(True)
        for _ in range(5):
            op.matvec(x, y)
        op.matvec(x, y)
        passes, cnt, _ = op.pass_times()
        op.set_profiling(False)
    s.synchronize()
    ys[mode] = y.cpu().numpy()
    st = op.stats()
    print(json.dumps(dict(config=name, m2l_store=mode, stored=st["m2l_stored"], store_gb=st["m2l_store_bytes"] / 1e9,
                          device_gb=st["device_bytes"] / 1e9, setup_s=setup, upload_s=st["setup_upload_s"],
                          ms_median=float(np.median(ts)), ms_min=float(min(ts)),
                          far_only_ms=float(np.median(tf)), near_only_ms=float(np.median(tn)),
                          pass_ms={k: v / max(cnt, 1) for k, v in passes.items()})), flush=True)
    del op
    torch.cuda.empty_cache()
if len(ys) == 2:
    a, b = ys[modes[0]] - P["x"], ys[modes[1]] - P["x"]
    print(json.dumps(dict(rel_diff=float(np.linalg.norm(a - b) / np.linalg.norm(b)))))
