"""Seeded random sweep of the parameter space on the GPU: (ell, lx, f, mode,
rounds, n, elem_base, input distribution) drawn at random, every fused kernel
and the party phases compared element by element with the oracle, messages
included.  Complements the hand-picked cases of test_gpu_parity.py with
combinations nobody chose (odd ell, windows touching the top bit, ragged n,
large bases)."""
import os

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


CASES = list(range(int(os.environ.get("BC_FUZZ_CASES", "120"))))  # BC_FUZZ_CASES: longer sweeps


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
        # the same call without a transcript: the instantiation the bench times (other slot
        # arithmetic where it differs, e.g. the p = 2^32 + 15 kernel), here at a random base
        z0, z1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base)
        assert np.array_equal(host(z0), ref["y0"]) and np.array_equal(host(z1), ref["y1"]), (fn, o, n, base, "no tr")
    # the party phases on the same inputs (the message wire format of the tape)
    lo0, hi0, tb0 = api.drelu_send(0, dev(x0), prm, SEEDS.s01, base)
    lo1, hi1, tb1 = api.drelu_send(1, dev(x1), prm, SEEDS.s01, base)
    r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base, paper_literal=True)
    ref = B.drelu(o, x0, x1, j, SEEDS)
    assert np.array_equal(host(api.drelu_finish(0, tb0, r0, prm, n, None, base)), ref["y0"])
    assert np.array_equal(host(api.drelu_finish(1, tb1, r1, prm, n, None, base)), ref["y1"])


@pytest.mark.parametrize("case", list(range(int(os.environ.get("BC_FUZZ_CASES", "120")) // 3)))
def test_random_widened_rows(api, case):
    """The widened rows under random parameters: RSS DReLU / ReLU (compact tape:
    lx = 7 guard, random ell and f), the Bicoptor-1 comparison (slots <= 8), the
    ABY3 truncation and the two fixed-point product orders."""
    from oracle import bicoptor1 as B1, rss, trunc
    rng = np.random.default_rng(5000 + case)
    n = int(rng.integers(1, 2000))
    base = int(rng.integers(0, 1 << 40)) // 8 * 8
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    rounds = int(rng.choice([8, 12, 20]))
    ell = int(rng.integers(16, 65))
    f = int(rng.integers(0, ell - 15 + 1))
    o = B.Params(ell=ell, lx=7, f=f, mode="guard", rounds=rounds)
    prm = api.Params(ell=ell, lx=7, f=f, mode="guard", rounds=rounds)
    x = synth.plaintext(n, ell, 7, f, ["D1", "D2"][rng.integers(2)], run=case)
    xs = synth.rss_share(x, ell, run=case)
    fn = ["drelu_rss", "relu_rss"][case % 2]
    ys = getattr(api, fn)(*(dev(v) for v in xs), prm, SEEDS, elem_base=base)
    ref = getattr(rss, fn)(o, *xs, j, SEEDS)
    for k in range(3):
        assert np.array_equal(host(ys[k]), ref["y"][k]), (fn, ell, f, n, base, k)
    # Bicoptor-1 on random small ladders
    lx = int(rng.integers(2, 8))
    f1 = int(rng.integers(0, 64 - 2 * lx))
    o1 = B.Params(ell=64, lx=lx, f=f1, mode="guard", rounds=rounds)
    x, x0, x1 = synth.shares(n, 64, lx, f1, "D1", run=case)
    y0, y1 = api.drelu_b1(dev(x0), dev(x1), api.Params(ell=64, lx=lx, f=f1, mode="guard", rounds=rounds), SEEDS,
                          elem_base=base)
    r1 = B1.drelu1(o1, x0, x1, j, SEEDS)
    assert np.array_equal(host(y0), r1["y0"]) and np.array_equal(host(y1), r1["y1"]), ("b1", lx, f1)
    # truncation: ABY3 (Alg 2) and the product orders (Alg 3 vs mult-then-trc)
    k = int(rng.integers(0, ell - 6))
    q = int(rng.integers(2))
    x, x0, x1 = synth.shares(n, ell, 5, min(k, ell - 7), "D1", run=case + 1)
    t0, t1 = api.trc_aby3(dev(x0), dev(x1), ell, k, SEEDS, elem_base=base, q=q, rounds=rounds)
    e0, e1 = trunc.trc_aby3(x0, x1, trunc.aby3_pre(ell, k, j, SEEDS, rounds, q), k, ell)
    assert np.array_equal(host(t0), e0) and np.array_equal(host(t1), e1), ("aby3", ell, k, q)
    order = ["mul_then_trc", "trc_then_mul"][rng.integers(2)]
    alg = ["secureml", "aby3"][rng.integers(2)]
    ff = int(rng.integers(1, max(2, ell // 3)))
    X = synth.plaintext(n, ell, 5, min(ff, ell - 7), "D1", run=case + 2)
    Y = synth.plaintext(n, ell, 5, min(ff, ell - 7), "D1", run=case + 3)
    a0, a1 = synth.share(X, ell, run=case + 4)
    b0, b1 = synth.share(Y, ell, run=case + 5)
    z0, z1 = api.mul_trc(order, alg, dev(a0), dev(a1), dev(b0), dev(b1), ell, ff, SEEDS, elem_base=base,
                         rounds=rounds)
    ref = getattr(trunc, order)(alg, a0, a1, b0, b1, ff, ell, j, SEEDS, rounds)
    assert np.array_equal(host(z0), ref[0]) and np.array_equal(host(z1), ref[1]), (order, alg, ell, ff)
