"""Fault injection: one byte of P0's message to P2 is changed between
bc_drelu_send and bc_drelu_helper (the message P2 tests, Alg 7 steps 8-9).
Exactly that element's outputs must stop matching the oracle's fault-free run, and the
faulted run must equal the oracle's helper/finish applied to the faulted message."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import bicoptor as B  # noqa: E402

SEEDS = synth.seeds(0)
DEV = "cuda:0"


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_04909_b200 import api as a
    a.lib()
    return a


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("direction", ["remove_zero", "create_zero"])
def test_flipped_message_byte_breaks_exactly_that_element(api, direction):
    kw = dict(ell=64, lx=7, f=24, mode="guard", rounds=20)
    oprm, prm = B.Params(**kw), api.Params(**kw)
    n, base = 4096, 1 << 16
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    t0 = torch.from_numpy(x0.view(np.int64)).to(DEV)
    t1 = torch.from_numpy(x1.view(np.int64)).to(DEV)
    lo0, hi0, tb0 = api.drelu_send(0, t0, prm, SEEDS.s01, base)
    lo1, hi1, tb1 = api.drelu_send(1, t1, prm, SEEDS.s01, base)
    ref = B.drelu(oprm, x0, x1, j, SEEDS)
    W0 = lo0.cpu().numpy().astype(np.int64) | (((hi0.cpu().numpy()[:, None] >> np.arange(8)) & 1).astype(np.int64) << 8)
    W1 = lo1.cpu().numpy().astype(np.int64) | (((hi1.cpu().numpy()[:, None] >> np.arange(8)) & 1).astype(np.int64) << 8)
    assert np.array_equal(W0, ref["W0"].astype(np.int64)) and np.array_equal(W1, ref["W1"].astype(np.int64))
    zero = (W0 + W1) % 257 == 0
    if direction == "remove_zero":   # the element's only zero slot, W0_m <= 254: lo byte + 1 (no carry into hi)
        cand = [(e, int(np.argmax(zero[e]))) for e in np.nonzero(zero.sum(axis=1) == 1)[0]]
        e, m = next((e, m) for e, m in cand if W0[e, m] <= 254)
        new = W0[e, m] + 1
    else:                            # no zero slot; a slot whose -W1_m mod 257 < 256 keeps hi: set lo so w_m = 0
        cand = [(e, m) for e in np.nonzero(zero.sum(axis=1) == 0)[0] for m in range(8)]
        e, m = next((e, m) for e, m in cand
                    if (257 - W1[e, m]) % 257 < 256 and W0[e, m] < 256 and (257 - W1[e, m]) % 257 != W0[e, m])
        new = (257 - W1[e, m]) % 257
    lo0[e, m] = int(new) & 0xFF    # one byte of the lo0 plane, on the device
    _, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base)
    y0 = api.drelu_finish(0, tb0, None, prm, n, SEEDS.s02, base)
    y1 = api.drelu_finish(1, tb1, r1, prm, n, None, base)
    g0, g1 = _u64(y0), _u64(y1)
    bad = np.nonzero((g0 != ref["y0"]) | (g1 != ref["y1"]))[0]
    assert bad.tolist() == [e]
    # and the faulted outputs are what the oracle's P2 / finish make of the faulted message
    Wf = ref["W0"].copy()
    Wf[e, m] = np.uint64(new)
    h = B.drelu_helper(oprm, Wf, ref["W1"], j, SEEDS.s02)
    assert int(h["z"][e]) == 1 - int(ref["z"][e])
    assert np.array_equal(g0, B.drelu_finish(oprm, 0, ref["t"], h["D0"]))
    assert np.array_equal(g1, B.drelu_finish(oprm, 1, ref["t"], h["D1"]))
