"""Pins for oracle.ring: the paper's worked examples, its theorems (exhaustive at
small ell), the e1 law and the modulo-switch closed form."""
import os

import numpy as np
import pytest

from oracle import ring

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.txt")


def _examples():
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        ident, cite, alg, x, R, k1, k2, exp, bits = [s.strip() for s in line.split("|")]
        yield ident, cite, alg, int(x, 2), int(R, 2), int(k1), int(k2), int(exp, 2), int(bits)


@pytest.mark.parametrize("ex", list(_examples()), ids=lambda e: e[0])
def test_worked_examples(ex):
    ident, cite, alg, x, R, k1, k2, exp, bits = ex
    ell = 8
    x0, x1 = (x + R) % 256, (-R) % 256          # P:213 sharing
    if alg == "alg1":
        got = (ring.trc_secureml(0, x0, k1, ell) + ring.trc_secureml(1, x1, k1, ell)) % 256
    elif alg == "alg4":
        got = (ring.trc_det(0, x0, k1, ell) + ring.trc_det(1, x1, k1, ell)) % (1 << (ell - k1))
    else:
        got = (ring.trc_det_mid(0, x0, k1, k2, ell) + ring.trc_det_mid(1, x1, k1, k2, ell)) % (1 << (ell - k1 - k2))
    assert got == exp and bits == (8 if alg == "alg1" else ell - k1 - k2)


def test_share_level_values_printed_in_examples():
    # P:51 (e0): cut([x]_0,4) = 0000 1111, cut(-[x]_1,4) = 0000 1010
    x, R = 0b01001011, 0b10101010
    assert ring.cut((x + R) % 256, 4) == 0b1111 and ring.cut((R) % 256, 4) == 0b1010
    # P:62 (e1): 0000 0010 and 0000 1110
    R = 0b11100000
    assert ring.cut((x + R) % 256, 4) == 0b0010 and ring.cut(R, 4) == 0b1110
    # P:751 (Alg 5): 010 and 110
    assert ring.cut_mid((x + R) % 256, 4, 1, 8) == 0b010 and ring.cut_mid(R, 4, 1, 8) == 0b110


def test_cut_definition_small():
    # cut(2^ell, k) = 2^(ell-k); cut(a, 0) = a; cut_mid(a, k, 0) = cut(a, k)
    assert ring.cut(1 << 8, 3) == 1 << 5
    for a in range(256):
        assert ring.cut(a, 0) == a
        for k in range(9):
            assert ring.cut_mid(a, k, 0, 8) == ring.cut(a, k)
    assert ring.cut_mid(0xFF, 2, 2, 8) == 0b1111


ELL = 8
A = np.repeat(np.arange(256, dtype=np.uint64), 256)
Bv = np.tile(np.arange(256, dtype=np.uint64), 256)


@pytest.mark.parametrize("k", range(0, 9))
def test_thm_cut_exhaustive(k):
    """Theorem thm:cut (reading C17: 'a' is alpha), every alpha, beta in Z_256."""
    s = (A + Bv) % np.uint64(256)
    rhs = ring.cut(A, k) + ring.cut(Bv, k) - ring.LT(s, A) * np.uint64(1 << (ELL - k))
    bit = ring.cut(s, k).astype(np.int64) - rhs.astype(np.int64)
    assert set(np.unique(bit)) <= {0, 1}
    d = (A + np.uint64(256) - Bv) % np.uint64(256)
    rhs2 = ring.cut(A, k).astype(np.int64) - ring.cut(Bv, k).astype(np.int64) + ring.LT(A, d).astype(np.int64) * (1 << (ELL - k))
    bit2 = rhs2 - ring.cut(d, k).astype(np.int64)
    assert set(np.unique(bit2)) <= {0, 1}


@pytest.mark.parametrize("k1,k2", [(k1, k2) for k1 in range(0, 8) for k2 in range(0, 8 - k1)])
def test_thm_newcut2_exhaustive(k1, k2):
    """Theorem thm:newcut2: cut(a+-b, k1, k2) = cut(a) +- cut(b) +- bit mod 2^(ell-k1-k2)."""
    M = 1 << (ELL - k1 - k2)
    s = (A + Bv) % np.uint64(256)
    d = (A + np.uint64(256) - Bv) % np.uint64(256)
    ca, cb = ring.cut_mid(A, k1, k2, ELL).astype(np.int64), ring.cut_mid(Bv, k1, k2, ELL).astype(np.int64)
    bit = (ring.cut_mid(s, k1, k2, ELL).astype(np.int64) - ca - cb) % M
    bit2 = (ca - cb - ring.cut_mid(d, k1, k2, ELL).astype(np.int64)) % M
    assert set(np.unique(bit)) <= {0, 1} and set(np.unique(bit2)) <= {0, 1}


def test_alg4_alg5_exact_e0_law():
    """Theorem thm:newtrc2 with Lemma lmm:pattern2:
    for every in-band x and every R (ell=8, lx=5), the reconstructed Alg 5
    output is cut(xi,k1,k2) + bit (positive) or -cut(xi,k1,k2) - bit
    (negative), and bit is exactly the carry/borrow out of the k1 low bits."""
    ell, lx = 8, 5
    R = np.arange(256, dtype=np.uint64)
    for xi in range(1, 1 << lx):
        for neg in (False, True):
            x = (-xi) % 256 if neg else xi
            x0 = (np.uint64(x) + R) % np.uint64(256)
            x1 = (np.uint64(256) - R) % np.uint64(256)
            for k1 in range(0, 5):
                for k2 in range(0, ell - k1 - 1):
                    M = 1 << (ell - k1 - k2)
                    got = (ring.trc_det_mid(0, x0, k1, k2, ell) + ring.trc_det_mid(1, x1, k1, k2, ell)) % np.uint64(M)
                    low = np.uint64((1 << k1) - 1)
                    plain = (xi >> k1) & (M - 1)
                    if not neg:
                        bit = ((np.uint64(xi) & low) + (R & low)) >> np.uint64(k1)
                        exp = (np.uint64(plain) + bit) % np.uint64(M)
                    else:
                        bit = ((R & low) < (np.uint64(xi) & low)).astype(np.uint64)
                        exp = (np.uint64(2 * M) - np.uint64(plain) - bit) % np.uint64(M)
                    assert np.array_equal(got, exp), (xi, neg, k1, k2)


def test_alg1_e1_count_is_xi():
    """Corollary clr:cut2: Alg 1 fails (e1) exactly when
    LT(x+R, x) (positive) / not LT(x+R, x) (negative; reading C3); count = xi masks of 2^ell
    (reading C18), the paper's 2^-(ell-lx-1) being the band-wide bound."""
    ell, k = 8, 3
    R = np.arange(256, dtype=np.uint64)
    for xi in range(1, 32):
        for neg in (False, True):
            x = (-xi) % 256 if neg else xi
            x0 = (np.uint64(x) + R) % np.uint64(256)
            x1 = (np.uint64(256) - R) % np.uint64(256)
            got = (ring.trc_secureml(0, x0, k, ell) + ring.trc_secureml(1, x1, k, ell)) % np.uint64(256)
            good = {xi >> k, (xi >> k) + 1} if not neg else {(-(xi >> k)) % 256, (-(xi >> k) - 1) % 256}
            fail = ~np.isin(got, np.array(sorted(good), dtype=np.uint64))
            # e1 iff LT(x+R, x) for positive x, iff not LT(x+R, x) for negative x
            # (clr:cut2 with 2^ell - [x]_1 = R; at R = 0 the negative case errs, C3/C18)
            pred = (x0 < np.uint64(x)) if not neg else ~(x0 < np.uint64(x))
            assert np.array_equal(fail, pred) and int(fail.sum()) == xi


@pytest.mark.parametrize("lp", range(1, 11))
def test_modswitch_zero_iff_zero_exhaustive(lp):
    """Alg 6 correctness argument, every share pair in Z_{2^lp}; the
    nonzero image is x or x - 2^lp mod p, and both outputs lie in Z_p^*."""
    p = ring.prime_above(lp)
    M = 1 << lp
    a = np.repeat(np.arange(M, dtype=np.uint64), M)
    b = np.tile(np.arange(M, dtype=np.uint64), M)
    x = (a + b) % np.uint64(M)
    o0, o1 = ring.modswitch(0, a, lp, p), ring.modswitch(1, b, lp, p)
    s = (o0 + o1) % np.uint64(p)
    assert np.array_equal(s == 0, x == 0)
    nz = x != 0
    xs = x[nz].astype(np.int64)
    assert np.all((s[nz].astype(np.int64) == xs % p) | (s[nz].astype(np.int64) == (xs - M) % p))
    assert o0.min() >= 1 and o1.min() >= 1 and o0.max() < p and o1.max() < p


def test_prime_above():
    # smallest prime > 2^w; brute-force primality by trial division over all candidates
    expect = {2: 5, 3: 11, 4: 17, 5: 37, 6: 67, 7: 131, 8: 257, 9: 521, 10: 1031}
    for w, p in expect.items():
        assert ring.prime_above(w) == p
        assert all(any(c % d == 0 for d in range(2, c)) for c in range((1 << w) + 1, p))
