"""Launch one fused op a few times on 2^24 elements with chosen parameters (profiling aid for ncu).

    python tools/run_op.py drelu ell=64 lx=7 f=24 mode=literal rounds=20
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2309_04909_b200 import api  # noqa: E402

op = sys.argv[1]
kw = dict(ell=64, lx=7, f=24, mode="guard", rounds=20)
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = v if k == "mode" else int(v)
n = 1 << 24
x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D2")
t0 = torch.from_numpy(x0.view(np.int64)).cuda()
t1 = torch.from_numpy(x1.view(np.int64)).cuda()
prm = api.Params(**kw)
for _ in range(3):
    getattr(api, op)(t0, t1, prm, synth.seeds(0))
torch.cuda.synchronize()
