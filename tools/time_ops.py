"""Quick CUDA-event timing of fused ops on 2^24 elements (tuning aid; bench.py is the measurement).

    python tools/time_ops.py drelu:mode=literal relu:mode=guard,rounds=8 ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2309_04909_b200 import api  # noqa: E402

n = 1 << 24
res = {}
cache = {}
for spec in sys.argv[1:]:
    op, _, rest = spec.partition(":")
    kw = dict(ell=64, lx=7, f=24, mode="guard", rounds=20)
    for a in filter(None, rest.split(",")):
        k, v = a.split("=")
        kw[k] = v if k == "mode" else int(v)
    key = (kw["ell"], kw["lx"], kw["f"])
    if key not in cache:
        x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D2")
        cache[key] = (torch.from_numpy(x0.view(np.int64)).cuda(), torch.from_numpy(x1.view(np.int64)).cuda())
    t0, t1 = cache[key]
    y0, y1 = torch.empty_like(t0), torch.empty_like(t1)
    prm = api.Params(**kw)
    fn = getattr(api, op)
    for _ in range(5):
        fn(t0, t1, prm, synth.seeds(0), 0, y0, y1)
    torch.cuda.synchronize()
    reps = 100 if kw["lx"] <= 7 else 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(t0, t1, prm, synth.seeds(0), 0, y0, y1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[spec] = {"ms": ms, "Gelem_s": n / ms / 1e6}
    print(spec, res[spec], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/time_ops.json", "w"), indent=1)
