"""Sweep the native host-buffer pipeline (chunk sizes) and raw PCIe copy rates."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_04909_b200 import api, host as H
n = 1 << 24
dev = torch.device("cuda:0")
x, x0h, x1h = synth.shares(n, 64, 7, 24, "D2")
hx0 = torch.from_numpy(x0h.view(np.int64)).pin_memory(); hx1 = torch.from_numpy(x1h.view(np.int64)).pin_memory()
hy0 = torch.empty(n, dtype=torch.int64).pin_memory(); hy1 = torch.empty(n, dtype=torch.int64).pin_memory()
d = torch.empty(n, dtype=torch.int64, device=dev)
out = {}
def bw(fn, nbytes, reps=10):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return nbytes * reps / (time.perf_counter() - t) / 1e9
out["h2d_GBs"] = bw(lambda: d.copy_(hx0, non_blocking=True), 8 * n)
out["d2h_GBs"] = bw(lambda: hy0.copy_(d, non_blocking=True), 8 * n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
def both():
    with torch.cuda.stream(s1): d.copy_(hx0, non_blocking=True)
    with torch.cuda.stream(s2): hy0.copy_(d2, non_blocking=True)
out["bidir_GBs_each"] = bw(both, 8 * n)
prm, sd = api.Params(), synth.seeds(0)
for chunk in (1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
    ex = H.HostPipeline(dev, chunk=chunk)
    for _ in range(2): ex.drelu(hx0, hx1, hy0, hy1, prm, sd)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): ex.drelu(hx0, hx1, hy0, hy1, prm, sd)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    out[f"chunk{chunk}"] = n / dt / 1e9
for rep in range(2):
    for chunk in (1 << 20, 1 << 21, 1 << 22, 1 << 23):  # the async entry, back to back (bench e2e)
        ex = H.HostPipeline(dev, chunk=chunk)
        for _ in range(2): ex.drelu(hx0, hx1, hy0, hy1, prm, sd, sync=False)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(40): ex.drelu(hx0, hx1, hy0, hy1, prm, sd, sync=False)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 40
        out[f"async_chunk{chunk}_rep{rep}"] = n / dt / 1e9
print(json.dumps(out))

# the same chunked schedule with copies only (no kernel): the PCIe-side bound of the pipeline
def copy_only(chunk, ns=3):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    bufs = [[torch.empty(chunk, dtype=torch.int64, device=dev) for _ in range(4)] for _ in range(ns)]
    def run():
        for c, a in enumerate(range(0, n, chunk)):
            m = min(chunk, n - a)
            s = streams[c % ns]
            b = bufs[c % ns]
            with torch.cuda.stream(s):
                b[0][:m].copy_(hx0[a:a + m], non_blocking=True)
                b[1][:m].copy_(hx1[a:a + m], non_blocking=True)
                hy0[a:a + m].copy_(b[2][:m], non_blocking=True)
                hy1[a:a + m].copy_(b[3][:m], non_blocking=True)
        torch.cuda.synchronize()
    run()
    t = time.perf_counter()
    for _ in range(10):
        run()
    return n / ((time.perf_counter() - t) / 10) / 1e9
out2 = {f"copy_only_chunk{c}": copy_only(c) for c in (1 << 20, 1 << 21, 1 << 22)}
out2["copy_only_chunk2M_4streams"] = copy_only(1 << 21, 4)
print(json.dumps(out2))
