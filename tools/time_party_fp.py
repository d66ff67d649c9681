"""Time the full-precision (lx = 31) party-phase kernels alone, 2^24 elements:
P0/P1 send and P2's helper, DReLU and ReLU (tuning aid; BICOPTOR_LIB selects a
variant build).  Prints one JSON line of ms per launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2309_04909_b200 import api  # noqa: E402

n = 1 << 24
dev = torch.device("cuda:0")
LX = int(os.environ.get("TIME_LX", "31"))  # 7: the compact tape (f = 24)
F = 24 if LX == 7 else 0
prm = api.Params(ell=64, lx=LX, f=F, mode=os.environ.get("TIME_MODE", "guard"), rounds=20)  # TIME_MODE=literal: p = 2^31 + 11
sd = synth.seeds(0)
x, x0, x1 = synth.shares(n, 64, LX, F, "D2")
t0 = torch.from_numpy(x0.view(np.int64)).to(dev)
t1 = torch.from_numpy(x1.view(np.int64)).to(dev)
lo0, hi0, tb0 = api.drelu_send(0, t0, prm, sd.s01)
lo1, hi1, tb1 = api.drelu_send(1, t1, prm, sd.s01)
r1, e, c1 = (torch.empty(n, dtype=torch.int64, device=dev) for _ in range(3))


def ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ya, d0 = torch.empty_like(t0), torch.empty_like(t0)
out = {"send_p0": ms(lambda: api.drelu_send(0, t0, prm, sd.s01, out=(lo0, hi0, tb0)), 3),
       "send_p1": ms(lambda: api.drelu_send(1, t1, prm, sd.s01, out=(lo1, hi1, tb1)), 3),
       "send_p0_y": ms(lambda: api.drelu_send(0, t0, prm, sd.s01, out=(lo0, hi0, None), y=ya, seed02=sd.s02), 3),
       "relu_send_p0": ms(lambda: api.relu_send(0, t0, prm, sd.s01, sd.s02, out=(lo0, hi0, tb0, d0)), 3),
       "helper_drelu": ms(lambda: api.drelu_helper(lo0, hi0, lo1, hi1, prm, sd.s02, out=(None, r1))),
       "helper_relu": ms(lambda: api.relu_helper(lo0, hi0, lo1, hi1, prm, sd.s02, sd.s12, out=(e, c1)))}
print(json.dumps(out))
