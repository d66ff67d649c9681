"""Debug aid: run one fused transcript case on the GPU and print the rows whose
message planes differ from the oracle, with the oracle's tape values."""
import sys
import numpy as np
import torch

sys.path[:0] = [".", "tests"]
import synth  # noqa: E402
from oracle import bicoptor as B  # noqa: E402
from paper_2309_04909_b200 import api  # noqa: E402

kw = dict(ell=64, lx=7, f=24, mode=sys.argv[1] if len(sys.argv) > 1 else "guard", rounds=int(sys.argv[2]) if len(sys.argv) > 2 else 8)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4099
SEEDS = synth.seeds(0)
for fn in ("drelu", "relu"):
    for base in (0, 8, 1 << 40):
        x, x0, x1 = synth.shares(n, 64, 7, kw["f"], "D1", run=n)
        j = np.arange(n, dtype=np.uint64) + np.uint64(base)
        ref = getattr(B, fn)(B.Params(**kw), x0, x1, j, SEEDS)
        tr = api.transcript_buffers(n, "cuda:0")
        d = lambda a: torch.from_numpy(a.view(np.int64)).cuda()  # noqa: E731
        y0, y1 = getattr(api, fn)(d(x0), d(x1), api.Params(**kw), SEEDS, elem_base=base, transcript=tr)
        lo0, hi0 = B.encode_msg(ref["W0"])
        lo1, hi1 = B.encode_msg(ref["W1"])
        g = {k: v.cpu().numpy() for k, v in tr.items()}
        bad = np.nonzero((g["w0_lo"] != lo0).any(1) | (g["w1_lo"] != lo1).any(1) | (g["w0_hi"] != hi0) | (g["w1_hi"] != hi1)
                         | (y0.cpu().numpy().view(np.uint64) != ref["y0"]) | (y1.cpu().numpy().view(np.uint64) != ref["y1"]))[0]
        print(fn, base, "bad rows", len(bad), bad[:10])
        tp = B.tape(B.Params(**kw), SEEDS.s01, j)
        for r in bad[:4]:
            print("  row", r, "j", int(j[r]))
            print("   W0 ref", ref["W0"][r].tolist(), "gpu lo", g["w0_lo"][r].tolist(), "hi", int(g["w0_hi"][r]))
            print("   W1 ref", ref["W1"][r].tolist(), "gpu lo", g["w1_lo"][r].tolist(), "hi", int(g["w1_hi"][r]))
            print("   rho", tp["rho"][r].tolist(), "r", tp["r"][r].tolist() if "r" in tp else None)
