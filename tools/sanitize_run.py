"""Exercise every C-ABI entry point once on small ragged inputs (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2309_04909_b200 import api

dev = "cuda:0"
sd = synth.seeds(0)
def t(a): return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
for kw in (dict(), dict(ell=16, lx=7, f=0, mode="literal"), dict(ell=32, lx=5, f=3), dict(mode="literal")):
    prm = api.Params(**kw, rounds=8)
    for n in (1, 13, 1003):
        x, x0, x1 = synth.shares(n, prm.ell, prm.lx, prm.f, "D1")
        a0, a1 = t(x0), t(x1)
        tr = api.transcript_buffers(n, dev)
        api.drelu(a0, a1, prm, sd, 8, transcript=tr)
        api.relu(a0, a1, prm, sd, 8, transcript=tr)
        api.drelu(a0, a1, prm, sd, 16)
        api.relu(a0, a1, prm, sd, 16)
        api.ladder_modswitch(0, a0, prm); api.ladder_modswitch(1, a1, prm)
        api.ladder_modswitch64(0, a0, prm); api.ladder_modswitch64(1, a1, prm)
        api.modswitch64(0, a0, 32, (1 << 32) + 15); api.modswitch64(1, a1, 63, (1 << 64) - 59)
        if prm.ell == 64 and prm.mode == "guard":  # the materialize2 instantiation (bench knob)
            os.environ["BICOPTOR_MATERIALIZE"] = "2"
            api.drelu(a0, a1, prm, sd, 24)
            del os.environ["BICOPTOR_MATERIALIZE"]
        api.trc(0, a0, prm.ell, 3, 1); api.trc(1, a1, prm.ell, 3, 1)
        api.trc_prob(0, a0, prm.ell, 3); api.modswitch(1, a1, 7, 131)
        lo0, hi0, tb0 = api.drelu_send(0, a0, prm, sd.s01, 8)
        lo1, hi1, tb1 = api.drelu_send(1, a1, prm, sd.s01, 8)
        r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, sd.s02, 8, paper_literal=True)
        api.drelu_finish(0, tb0, None, prm, n, sd.s02, 8); api.drelu_finish(1, tb1, r1, prm, n, None, 8)
        api.drelu_send(0, a0, prm, sd.s01, 8, out=(lo0, hi0, None), y=torch.empty_like(a0), seed02=sd.s02)
        L0, H0, T0, d0 = api.relu_send(0, a0, prm, sd.s01, sd.s02, 8)
        L1, H1, T1, d1 = api.relu_send(1, a1, prm, sd.s01, sd.s12, 8)
        e, c1 = api.relu_helper(L0, H0, L1, H1, prm, sd.s02, sd.s12, 8)
        api.relu_finish(0, a0, T0, d0, d1, e, None, prm, sd.s02, 8)
        api.relu_finish(1, a1, T1, d1, d0, e, c1, prm, sd.s12, 8)
# RSS variant (Alg 9), large tape (lx = 31), truncation study, host-buffer entry
prm = api.Params(rounds=8)
for n in (1, 13, 1003):
    x = synth.plaintext(n, 64, 7, 24, "D1")
    xs = [t(v) for v in synth.rss_share(x, 64)]
    api.drelu_rss(*xs, prm, sd, 8)
    api.relu_rss(*xs, prm, sd, 8)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1")
    a0, a1 = t(x0), t(x1)
    big = api.Params(ell=64, lx=31, f=0, rounds=8)
    tr = api.transcript_buffers(n, dev, big)
    api.drelu(a0, a1, big, sd, 8, transcript=tr)
    api.relu(a0, a1, big, sd, 8)
    api.ladder_modswitch64(0, a0, big); api.ladder_modswitch64(1, a1, big)
    for pk in (big, api.Params(ell=64, lx=31, f=0, mode="literal", rounds=8), api.Params(ell=24, lx=10, f=0, rounds=8)):
        x, x0, x1 = synth.shares(n, pk.ell, pk.lx, pk.f, "D1")   # party phases on the uint32 wire planes
        b0, b1 = t(x0), t(x1)
        lo0, hi0, tb0 = api.drelu_send(0, b0, pk, sd.s01, 8)
        lo1, hi1, tb1 = api.drelu_send(1, b1, pk, sd.s01, 8)
        r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, pk, sd.s02, 8, paper_literal=True)
        api.drelu_finish(1, tb1, r1, pk, n, None, 8)
        api.drelu_send(0, b0, pk, sd.s01, 8, out=(lo0, hi0, None), y=torch.empty_like(b0), seed02=sd.s02)
        dp = torch.empty_like(b0)
        L0, H0, T0, d0 = api.relu_send(0, b0, pk, sd.s01, sd.s02, 8, d_peer=dp)
        L1, H1, T1, d1 = api.relu_send(1, b1, pk, sd.s01, sd.s12, 8)
        e, c1 = api.relu_helper(L0, H0, L1, H1, pk, sd.s02, sd.s12, 8, e_dup=torch.empty_like(b0))
        api.relu_finish(1, b1, T1, d1, dp, e, c1, pk, sd.s12, 8)
    api.trc_aby3(a0, a1, 64, 26, sd, 8, q=1, rounds=8)
    api.mul_trc("trc_then_mul", "aby3", a0, a1, a0, a1, 64, 26, sd, 8, rounds=8)
    api.mul_trc("mul_then_trc", "secureml", a0, a1, a0, a1, 64, 26, sd, 8, rounds=8)
    api.trc_count("det", a0, 64, 26, 0, 1000)
    hx0, hx1 = torch.from_numpy(x0.view(np.int64)).pin_memory(), torch.from_numpy(x1.view(np.int64)).pin_memory()
    hy0, hy1 = torch.empty(n, dtype=torch.int64).pin_memory(), torch.empty(n, dtype=torch.int64).pin_memory()
    api.drelu_host(hx0, hx1, hy0, hy1, prm, sd, api.host_workspace(512, dev), 512, 8)
    wsa = api.host_workspace(64, dev)
    api.relu_host(hx0, hx1, hy0, hy1, prm, sd, wsa, 64, 8, sync=False)   # two async requests pipelined
    api.drelu_host(hx0, hx1, hy0, hy1, prm, sd, wsa, 64, 8, sync=False)
    torch.cuda.synchronize()
torch.cuda.synchronize()
print("sanitize_run ok")
