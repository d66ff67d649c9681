"""Pins for oracle.trunc (truncation study): the paper's
8-bit worked examples, the exact per-x e1 law (xi masks of 2^ell, reading C18)
and the e1 condition of Corollary clr:cut2, Theorem newcut2 (Alg 4 has no e1)
with its exact one-bit-error count, the Beaver product against plaintext, and
the mult-then-trc vs trc-then-mult behaviour of sec. 5."""
import numpy as np
import pytest

import synth
from oracle import ring, trunc

SEEDS = synth.seeds(0)


def test_worked_example_e1_and_alg4():
    """x = 0100 1011, R = 1110 0000, ell = 8, k = 4.
    SecureML gives 1111 0100 (an e1); Alg 4 gives 0100 = cut(x, 4)."""
    x, R, ell, k = 0b01001011, 0b11100000, 8, 4
    x0, x1 = (x + R) % 256, (-R) % 256
    assert (x0, x1) == (0b00101011, 0b00100000)
    y0, y1 = trunc.trc_secureml_pair(np.array([x0], np.uint64), np.array([x1], np.uint64), k, ell)
    y = int(ring.add(y0, y1, ell)[0])
    assert y == 0b11110100
    assert trunc.classify(x, y, k, ell)[0] == trunc.E1
    yd = (int(ring.trc_det(0, np.uint64(x0), k, ell)) + int(ring.trc_det(1, np.uint64(x1), k, ell))) % 16
    assert yd == 0b0100 and trunc.classify(x, yd, k, ell, ell - k)[0] == trunc.EXACT


@pytest.mark.parametrize("ell,k", [(8, 4), (8, 1), (10, 3), (10, 7)])
def test_e1_count_is_xi_and_alg4_has_none(ell, k):
    """Over all 2^ell masks: Alg 1 and Alg 2 fail with e1 for exactly xi masks
    (for both signs; C18); Alg 4 never does (Theorem newcut2), and its one-bit
    error occurs for exactly (xi mod 2^k) 2^(ell-k) masks (the carry out of the
    low k bits)."""
    lx = ell - 2
    for xi in list(range(1, 1 << lx, 7)) + [(1 << lx) - 1]:
        for x in (xi, (1 << ell) - xi):
            for alg in ("secureml", "aby3"):
                c = trunc.count_masks(alg, x, k, ell)
                assert c[trunc.E1] == xi, (alg, x)
                assert c.sum() == 1 << ell
            c = trunc.count_masks("det", x, k, ell)
            assert c[trunc.E1] == 0
            assert c[trunc.E0] == (xi % (1 << k)) * (1 << (ell - k))


def test_e1_condition_matches_corollary():
    """Corollary clr:cut2: for positive x, e1 iff LT(x + R, x); for negative x,
    iff LT(x, x + R) -- checked against the class of the reconstructed output."""
    ell, k = 16, 5
    rng = np.random.default_rng(1)
    xi = rng.integers(1, 1 << 13, 20000).astype(np.uint64)
    neg = rng.integers(0, 2, 20000).astype(bool)
    x = np.where(neg, ring.neg(xi, ell), xi).astype(np.uint64)
    R = rng.integers(0, 1 << ell, 20000).astype(np.uint64)
    x0, x1 = ring.add(x, R, ell), ring.neg(R, ell)
    y0, y1 = trunc.trc_secureml_pair(x0, x1, k, ell)
    cls = trunc.classify(x, ring.add(y0, y1, ell), k, ell)
    e1 = np.where(neg, ring.LT(x, x0), ring.LT(x0, x)).astype(bool)
    assert np.array_equal(cls == trunc.E1, e1)
    assert e1.sum() > 100


def test_aby3_preprocessing_and_no_wrap_is_exact_or_e0():
    ell, k = 64, 26
    j = np.arange(5000, dtype=np.uint64)
    pre = trunc.aby3_pre(ell, k, j, SEEDS)
    r = ring.add(pre["r0"], pre["r1"], ell)
    assert np.array_equal(ring.add(pre["rp0"], pre["rp1"], ell), ring.cut(r, k))
    x = synth.plaintext(5000, 64, 5, 26, "D1")
    x0, x1 = synth.share(x, 64)
    y0, y1 = trunc.trc_aby3(x0, x1, pre, k, ell)
    cls = trunc.classify(x, ring.add(y0, y1, ell), k, ell)
    pos = x < np.uint64(1 << 63)
    alpha = ring.add(x, r, ell)
    wrap = np.where(pos, ring.LT(alpha, x), ring.LT(x, alpha)).astype(bool)
    assert np.array_equal(cls == trunc.E1, wrap)


def test_beaver_product():
    ell = 64
    n = 4000
    j = np.arange(n, dtype=np.uint64)
    rng = np.random.default_rng(2)
    x, y = (rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True) for _ in range(2))
    x0, x1 = synth.share(x, ell, run=1)
    y0, y1 = synth.share(y, ell, run=2)
    tr = trunc.triple(ell, j, SEEDS)
    assert np.array_equal(ring.add(tr["c0"], tr["c1"], ell),
                          ring.mul(ring.add(tr["a0"], tr["a1"], ell), ring.add(tr["b0"], tr["b1"], ell), ell))
    z0, z1 = trunc.mul_beaver(x0, x1, y0, y1, tr, ell)
    with np.errstate(over="ignore"):
        assert np.array_equal(ring.add(z0, z1, ell), x * y)


@pytest.mark.parametrize("alg", ["secureml", "aby3"])
def test_mult_then_trc_fails_trc_then_mult_does_not(alg):
    """Sec. 5 at the paper's parameters (ell = 64, 5+26 fixed point):
    the product of two 31-bit values has ~62 bits, so multiply-then-truncate hits
    e1 with probability ~|xy| / 2^64; truncate-then-multiply (Alg 3) keeps every
    error within the precision loss of truncating the operands."""
    ell, f, n = 64, 26, 20000
    X = synth.plaintext(n, 64, 5, 26, "D1", run=3)
    Y = synth.plaintext(n, 64, 5, 26, "D1", run=4)
    x0, x1 = synth.share(X, ell, run=5)
    y0, y1 = synth.share(Y, ell, run=6)
    j = np.arange(n, dtype=np.uint64)
    want = np.array([int(a) * int(b) >> f for a, b in zip(trunc.signed(X, ell), trunc.signed(Y, ell))], dtype=object)
    m0, m1 = trunc.mul_then_trc(alg, x0, x1, y0, y1, f, ell, j, SEEDS)
    err_m = trunc.signed(ring.add(m0, m1, ell), ell) - want
    t0, t1 = trunc.trc_then_mul(alg, x0, x1, y0, y1, f, ell, j, SEEDS)
    err_t = trunc.signed(ring.add(t0, t1, ell), ell) - want
    big = 1 << 30                                                       # e1 = +-cut(2^64, 26) = 2^38
    n_e1 = sum(1 for e in err_m if abs(e) > big)
    # expected number of e1 events: sum over elements of |xy| / 2^64
    expect = float(sum(abs(int(a) * int(b)) for a, b in zip(trunc.signed(X, ell), trunc.signed(Y, ell)))) / 2**64
    assert expect > 100
    assert abs(n_e1 - expect) < 6 * np.sqrt(expect)
    assert all(abs(e) <= 1 for e in err_m if abs(e) <= big)          # otherwise only the one-bit e0
    # Alg 3: |x'y' - xy/2^f| <= |x|/2^13 + |y|/2^13 + 1 (each operand loses < 1 ulp of 2^13)
    bound = [abs(int(a)) / 2**13 + abs(int(b)) / 2**13 + 2 for a, b in zip(trunc.signed(X, ell), trunc.signed(Y, ell))]
    assert all(abs(e) <= b for e, b in zip(err_t, bound))
