"""Pins for oracle.bicoptor1 (the Bicoptor-1 comparison point, NEXT #4):
plaintext sign at ell = 64 and 32, DReLU(0) = t, the message size of Table 1 /
P:990, the recursive sum against its definition written out per element, and
the paper's motivation (sec. 6): at ell = 16 the probabilistic truncation's e1
breaks Bicoptor-1 on some inputs -- exactly on elements with an e1 in some
ladder truncation -- while Bicoptor 2.0 is exact on the same inputs."""
import numpy as np

import synth
from oracle import bicoptor as B
from oracle import bicoptor1 as B1
from oracle import ring, trunc
from plain import band_sign

SEEDS = synth.seeds(0)


def test_sign_ell64_and_32():
    for ell, f in ((64, 24), (32, 0)):
        prm = B.Params(ell=ell, lx=7, f=f)
        for dist in ("D1", "D2"):
            x = synth.plaintext(20000, ell, 7, f, dist)
            x0, x1 = synth.share(x, ell)
            d = B1.drelu1(prm, x0, x1, np.arange(x.size, dtype=np.uint64), SEEDS)
            y = B.reconstruct(d["y0"], d["y1"], ell)
            s, valid = band_sign(x, ell, 7, f)
            assert valid.sum() > 15000
            assert np.array_equal(y[valid], s[valid])
            zero = x == 0
            assert np.array_equal(y[zero], d["t"][zero])


def test_message_size():
    """(lx + 1) slots of ell bits: 8 x 64 = 512 at the 5+2 key bits (2048 -> 512)."""
    prm = B.Params(ell=64, lx=7, f=24)
    x, x0, x1 = synth.shares(10, 64, 7, 24, "D1")
    m = B1.drelu1_send(prm, 0, x0, np.arange(10, dtype=np.uint64), SEEDS.s01)
    assert m["W"].shape == (10, 8) and m["W"].dtype == np.uint64
    assert m["W"].shape[1] * prm.ell == 512


def test_recursive_sums_definition():
    prm = B.Params(ell=64, lx=7, f=24)
    rng = np.random.default_rng(3)
    u = rng.integers(0, 2**64 - 1, (50, 8), dtype=np.uint64, endpoint=True)
    for party in (0, 1):
        v = B1.recursive_sums(prm, party, u)
        for r in range(50):
            for i in range(8):
                want = (sum(int(a) for a in u[r, i:]) - (1 if party == 0 else 0)) % 2**64
                assert int(v[r, i]) == want


def test_e1_breaks_bicoptor1_not_bicoptor2_at_ell16():
    """Every in-band x x 64 sharings at ell = 16, lx = 7, f = 0.  Bicoptor 2.0
    (deterministic truncation) is exact; Bicoptor-1 mis-signs some elements, and
    each of them has an e1 (C30) in one of its SecureML ladder truncations."""
    ell, lx, f = 16, 7, 0
    prm = B.Params(ell=ell, lx=lx, f=f)
    xi = np.arange(1, 1 << lx, dtype=np.uint64)
    x = np.repeat(np.concatenate([xi, np.uint64(1 << ell) - xi]), 64)
    x0, x1 = synth.share(x, ell)
    j = np.arange(x.size, dtype=np.uint64)
    s, _ = band_sign(x, ell, lx, f)
    d2 = B.drelu(prm, x0, x1, j, SEEDS)
    assert np.array_equal(B.reconstruct(d2["y0"], d2["y1"], ell), s)
    d1 = B1.drelu1(prm, x0, x1, j, SEEDS)
    bad = B.reconstruct(d1["y0"], d1["y1"], ell) != s
    assert 0 < bad.sum() < 0.05 * x.size
    # e1 in some truncation of the blinded shares (same t as the protocol used)
    tp = B1.tape1(prm, SEEDS.s01, j)
    sb = np.where(tp["t"] == 1, ring.neg(x, ell), x).astype(np.uint64)
    s0 = np.where(tp["t"] == 1, ring.neg(x0, ell), x0).astype(np.uint64)
    s1 = np.where(tp["t"] == 1, ring.neg(x1, ell), x1).astype(np.uint64)
    any_e1 = np.zeros(x.size, dtype=bool)
    for i in range(lx + 1):
        y = ring.add(ring.trc_secureml(0, s0, f + i, ell), ring.trc_secureml(1, s1, f + i, ell), ell)
        any_e1 |= trunc.classify(sb, y, f + i, ell) == trunc.E1
    assert np.all(any_e1[bad])


def test_golden_fallback_indices_reject():
    """The fixture tests/golden/b1_fallback.txt lists elements whose tape word 0
    rejects; decoding them still yields valid Fisher-Yates digits (fallback)."""
    import os
    from oracle.chacha import chacha_blocks
    path = os.path.join(os.path.dirname(__file__), "golden", "b1_fallback.txt")
    rej = [int(v) for v in open(path).read().split() if v.strip().isdigit()]
    assert len(rej) >= 2
    j = np.array(rej, dtype=np.uint64)
    w0 = chacha_blocks(SEEDS.s01, B1.L_TAPE1, 3 * j, 20)[:, 0] & np.uint32(0x7FFFFFFF)
    assert np.all(w0 >= np.uint32((2**31 // 40320) * 40320))
    tp = B1.tape1(B.Params(), SEEDS.s01, j)
    assert np.all(tp["k"] <= np.arange(8))
