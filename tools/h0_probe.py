"""Accuracy of the product's device H0^(1) evaluator per band against mpmath (40 digits):
max relative error over each band's interval (dafmm_h0_bands), printed as one line per band."""
import json
import os
import sys

import mpmath as mp
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_00326_b200 import binding  # noqa: E402

rng = np.random.default_rng(5)
mp.mp.dps = 40
for code, (lo, hi) in enumerate(binding.dafmm_h0_bands()):
    lo, hi = max(lo, 1e-3), min(hi, 1e3)
    z = np.unique(np.concatenate([np.geomspace(lo, hi, 150), rng.uniform(lo, hi, 150), [lo, hi]]))
    zd = torch.from_numpy(z * z).cuda()
    out = torch.empty(z.size, dtype=torch.complex128, device="cuda")
    binding.dafmm_h0_eval(zd, out, code, torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = np.array([complex(mp.hankel1(0, mp.sqrt(mp.mpf(float(v))))) for v in z * z])
    rel = np.abs(got - ref) / np.abs(ref)
    i = int(np.argmax(rel))
    print(json.dumps(dict(band=code, zlo=lo, zhi=hi, n=int(z.size), max_rel=float(rel.max()), at_z=float(z[i]))))
