"""CUDA-event timing of config 2 (bc_ladder_modswitch, one party, ell=64, f=24, guard,
2^28 elements) -- a tuning aid (bench.py's trc_modswitch leg is the measurement).
BICOPTOR_LIB selects a variant build.  Prints ms per call and GB/s (16 B per element)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_04909_b200 import api  # noqa: E402

n = 1 << 28
prm = api.Params(ell=64, lx=7, f=24, mode="guard", rounds=20)
x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device="cuda")
out = torch.empty((n, 8), dtype=torch.uint8, device="cuda")
for _ in range(3):
    api.ladder_modswitch(0, x, prm, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
e0.record()
for _ in range(reps):
    api.ladder_modswitch(0, x, prm, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"lib": os.path.basename(os.environ.get("BICOPTOR_LIB", "default")), "ms": ms, "GBps": 16 * n / ms / 1e6}))
