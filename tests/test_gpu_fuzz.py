"""Seeded random sweep of the parameter space on the GPU: (ell, lx, f, mode,
rounds, n, elem_base, input distribution) drawn at random, every fused kernel
and the party phases compared element by element with the oracle, messages
included.  Complements the hand-picked cases of test_gpu_parity.py with
combinations nobody chose (odd ell, windows touching the top bit, ragged n,
large bases)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import bicoptor as B  # noqa: E402

DEV = "cuda:0"
SEEDS = synth.seeds(3)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(DEV)


def host(t):
    return t.cpu().numpy().view(np.uint64)


def _draw(rng):
    """A random valid parameter set (rejection over the fit condition)."""
    while True:
        mode = ["guard", "literal"][rng.integers(2)]
        lx = int(rng.choice([2, 3, 4, 5, 6, 7, 7, 7, 8, 9, 12, 15, 20, 31]))
        w = lx + 1 if mode == "guard" else lx
        ell = int(rng.integers(lx + w + 1, 65)) if lx + w + 1 <= 64 else 64
        if ell < lx + w:
            continue
        f = int(rng.integers(0, ell - lx - w + 1))
        rounds = int(rng.choice([8, 12, 20]))
        try:
            return B.Params(ell=ell, lx=lx, f=f, mode=mode, rounds=rounds)
        except ValueError:
            continue


CASES = list(range(120))


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_04909_b200 import api as a
    a.lib()
    return a


@pytest.mark.parametrize("case", CASES)
def test_random_parameters(api, case):
    rng = np.random.default_rng(1000 + case)
    o = _draw(rng)
    prm = api.Params(ell=o.ell, lx=o.lx, f=o.f, mode=o.mode, rounds=o.rounds)
    n = int(rng.integers(1, 300 if o.layout == "large" else 3000))
    base = int(rng.integers(0, 1 << 40)) // 8 * 8
    x, x0, x1 = synth.shares(n, o.ell, o.lx, o.f, ["D1", "D2"][rng.integers(2)], run=case)
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    for fn in ("drelu", "relu"):
        tr = api.transcript_buffers(n, DEV, prm)
        y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base, transcript=tr)
        ref = getattr(B, fn)(o, x0, x1, j, SEEDS)
        assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"]), (fn, o, n, base)
        if o.layout == "large":  # u64 message planes
            assert np.array_equal(host(tr["w0_lo"]), ref["W0"].astype(np.uint64))
            assert np.array_equal(host(tr["w1_lo"]), ref["W1"].astype(np.uint64))
        else:                    # the byte wire format
            for k in ("0", "1"):
                lo, hi = B.encode_msg(ref["W" + k])
                assert np.array_equal(tr[f"w{k}_lo"].cpu().numpy(), lo)
                assert np.array_equal(tr[f"w{k}_hi"].cpu().numpy(), hi)
    # the party phases on the same inputs (the message wire format of the tape)
    lo0, hi0, tb0 = api.drelu_send(0, dev(x0), prm, SEEDS.s01, base)
    lo1, hi1, tb1 = api.drelu_send(1, dev(x1), prm, SEEDS.s01, base)
    r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base, paper_literal=True)
    ref = B.drelu(o, x0, x1, j, SEEDS)
    assert np.array_equal(host(api.drelu_finish(0, tb0, r0, prm, n, None, base)), ref["y0"])
    assert np.array_equal(host(api.drelu_finish(1, tb1, r1, prm, n, None, base)), ref["y1"])
