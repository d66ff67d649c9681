"""Diagnose kernel timing: back-to-back events vs synchronized launches, CPU call overhead."""
import os, sys, time, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_04909_b200 import api

n = 1 << 24
dev = torch.device("cuda:0")
x, x0h, x1h = synth.shares(n, 64, 7, 24, "D2")
x0 = torch.from_numpy(x0h.view(np.int64)).to(dev); x1 = torch.from_numpy(x1h.view(np.int64)).to(dev)
y0 = torch.empty_like(x0); y1 = torch.empty_like(x1)
sd = synth.seeds(0)
out = {}
for R in (20, 8):
    prm = api.Params(rounds=R)
    st = torch.cuda.current_stream()
    for _ in range(10): api.drelu(x0, x1, prm, sd, 0, y0, y1)
    torch.cuda.synchronize()
    # CPU overhead per call
    t0 = time.perf_counter()
    for _ in range(200): api.drelu(x0, x1, prm, sd, 0, y0, y1)
    cpu = (time.perf_counter() - t0) / 200
    torch.cuda.synchronize()
    # back to back events
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(301)]
    ev[0].record()
    for i in range(300):
        api.drelu(x0, x1, prm, sd, 0, y0, y1); ev[i + 1].record()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(300)]
    # synchronized single launches
    single = []
    for i in range(30):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); api.drelu(x0, x1, prm, sd, 0, y0, y1); b.record(); torch.cuda.synchronize()
        single.append(a.elapsed_time(b)); time.sleep(0.01)
    out[R] = {"cpu_ms_per_call": cpu * 1e3, "b2b_first10": per[:10], "b2b_median": float(np.median(per)),
              "b2b_last10": per[-10:], "single_median": float(np.median(single)), "single": single[:10]}
print(json.dumps(out, indent=1))
