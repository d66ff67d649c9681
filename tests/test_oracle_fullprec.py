"""Pins for the large-tape oracle path (lx >= 8; full precision lx = 31 without
key bits): tape invariants, brute-force sign / ReLU against
plaintext, the literal-mode false-positive set, and the wire size of Table 1's
formula at lx = 31."""
import math

import numpy as np
import pytest

import synth
from oracle import bicoptor as B
from oracle.chacha import element_u32
from plain import band_sign, relu_plain
from test_oracle_drelu import _literal_fp_set

SEEDS = synth.seeds(0)


def _raw_perm_rejects(prm, j):
    """Rows with a rejected Fisher-Yates draw, from the raw keystream."""
    T = element_u32(SEEDS.s01, B.L_TAPEL, prm.rounds, j, 112)
    h = np.ascontiguousarray(T[:, :16]).view("<u2").reshape(-1, 32).astype(np.int64)
    S = prm.slots
    rej = np.zeros(j.size, dtype=bool)
    for m in range(1, S):
        rej |= h[:, S - m] >= (65536 // (m + 1)) * (m + 1)
    return rej, h


def _raw_draws(prm, j):
    """The 48-bit mask and reshare draws of slots 0..31 straight from the keystream
    bytes (tape layout of DESIGN.md sec. 4, written out independently of the oracle)."""
    T = element_u32(SEEDS.s01, B.L_TAPEL, prm.rounds, j, 112)
    D = np.ascontiguousarray(T[:, 16:]).view(np.uint8).reshape(-1, 384).astype(object)
    r = np.array([[sum(int(D[i, 96 * (m // 8) + 6 * (m % 8) + b]) << (8 * b) for b in range(6)) for m in range(32)]
                  for i in range(j.size)], dtype=object)
    rho = np.array([[sum(int(D[i, 96 * (m // 8) + 48 + 6 * (m % 8) + b]) << (8 * b) for b in range(6))
                     for m in range(32)] for i in range(j.size)], dtype=object)
    return r, rho


def _raw_draw_rejects(prm, j):
    """Rows with a rejected 48-bit mask or reshare draw among the first S slots."""
    r, rho = _raw_draws(prm, j)
    p, S = prm.p, prm.slots
    rl, pl = ((1 << 48) // (p - 1)) * (p - 1), ((1 << 48) // p) * p
    return np.array([any(r[i, m] >= rl or rho[i, m] >= pl for m in range(S)) for i in range(j.size)])


def test_params_full_precision():
    g = B.Params(ell=64, lx=31, f=0, mode="guard")
    lit = B.Params(ell=64, lx=31, f=0, mode="literal")
    assert (g.w, g.p, g.slots, g.layout) == (32, 2**32 + 15, 32, "large")
    assert (lit.w, lit.p, lit.slots, lit.layout) == (31, 2**31 + 11, 32, "large")
    with pytest.raises(ValueError):
        B.Params(ell=64, lx=32, f=0)
    with pytest.raises(ValueError):
        B.Params(ell=64, lx=31, f=2)   # 2 + 31 + 32 > 64


def test_wire_bits_full_precision():
    """Step 8's message is (lx+1) slots of ceil(log2 p) bits: 32 x 32 = 1024 in the
    paper's literal domain (31*31 ~ 1,000 bits), 32 x 33 in guard mode."""
    for mode, bits in (("literal", 1024), ("guard", 1056)):
        prm = B.Params(ell=64, lx=31, f=0, mode=mode)
        assert prm.slots * math.ceil(math.log2(prm.p)) == bits


def test_large_tape_invariants_and_fallback():
    prm = B.Params(ell=64, lx=31, f=0)
    n = 6000
    j = np.arange(n, dtype=np.uint64)
    tp = B.tape(prm, SEEDS.s01, j)
    S, p = prm.slots, prm.p
    r = np.array(tp["r"].tolist(), dtype=object)
    rho = np.array(tp["rho"].tolist(), dtype=object)
    assert min(r.ravel()) >= 1 and max(r.ravel()) <= p - 1
    assert min(rho.ravel()) >= 0 and max(rho.ravel()) <= p - 1
    assert max(r.ravel()) > 2**32 - 2**28            # the draws span Z_p, not just 32 bits
    assert abs(int(tp["t"].sum()) - n // 2) < 5 * math.sqrt(n)
    perm = B.shuffle(tp["k"], np.tile(np.arange(S, dtype=np.uint64), (n, 1)))
    assert np.all(np.sort(perm, axis=1) == np.arange(S))
    pos0 = np.argmax(perm == 0, axis=1)
    cnt = np.bincount(pos0, minlength=S)
    assert np.all(np.abs(cnt - n / S) < 6 * math.sqrt(n / S))
    # elements with a rejected raw draw take the fallback stream; the rest decode directly
    rej, h = _raw_perm_rejects(prm, j)
    assert 5 <= rej.sum() <= 60                      # ~0.35 % of elements
    direct = np.nonzero(~rej)[0][:200]
    for m in range(1, S):
        assert np.array_equal(tp["k"][direct, m], h[direct, S - m] % (m + 1))
    assert np.all(tp["k"][rej] <= np.arange(S))
    # the 48-bit draws: r_m (Montgomery form) and rho_m from the raw bytes where nothing rejects
    jd = np.arange(64, dtype=np.uint64)
    ur, uq = _raw_draws(prm, jd)
    tpd = B.tape(prm, SEEDS.s01, jd)
    rinv = pow(2, -64, p)
    for i in np.nonzero(~_raw_draw_rejects(prm, jd))[0][:40]:
        for m in range(S):
            assert tpd["r"][i, m] == (1 + ur[i, m] % (p - 1)) * rinv % p
            assert tpd["rho"][i, m] == uq[i, m] % p


def test_large_tape_48bit_draw_rejections():
    """A 48-bit draw rejects with probability < 2^-15 (p - 1, p ~ 2^32): the rows that
    reject are found from the raw bytes, and the oracle's values there still lie in
    range (they came from the fallback stream)."""
    prm = B.Params(ell=64, lx=31, f=0, rounds=8)
    j = np.arange(3000, dtype=np.uint64)
    rej = _raw_draw_rejects(prm, j)
    assert 1 <= rej.sum() <= 15                      # expected 3000 * 64 * ~2^-16.5 ~ 2.1
    tp = B.tape(prm, SEEDS.s01, j[rej])
    assert all(1 <= int(v) < prm.p for v in np.ravel(tp["r"])) and all(0 <= int(v) < prm.p for v in np.ravel(tp["rho"]))


@pytest.mark.parametrize("ell,lx,f", [(24, 10, 0), (20, 8, 1)])
def test_drelu_large_bruteforce_sign(ell, lx, f):
    """Every in-band nonzero x x 8 sharings: the large-tape DReLU opens to the
    plaintext sign, ReLU to max(x, 0) (guard mode)."""
    prm = B.Params(ell=ell, lx=lx, f=f)
    assert prm.layout == "large"
    xi = np.arange(1 << f, 1 << (f + lx), dtype=np.uint64)
    x = np.repeat(np.concatenate([xi, np.uint64(1 << ell) - xi]), 8)
    x0, x1 = synth.share(x, ell)
    j = np.arange(x.size, dtype=np.uint64)
    d = B.drelu(prm, x0, x1, j, SEEDS)
    r = B.relu(prm, x0, x1, j, SEEDS)
    s, valid = band_sign(x, ell, lx, f)
    assert valid.all()
    assert np.array_equal(B.reconstruct(d["y0"], d["y1"], ell), s)
    assert np.array_equal(B.reconstruct(r["y0"], r["y1"], ell), relu_plain(x, ell, lx, f))


def test_drelu_full_precision_ell64():
    """lx = 31, f = 0, ell = 64 (5+26 fixed point with no key bits): D1 and D2
    batches; sign exact on every nonzero input, ReLU = x * DReLU; x = 0 opens to t."""
    for mode in ("guard", "literal"):
        prm = B.Params(ell=64, lx=31, f=0, mode=mode)
        for dist in ("D1", "D2"):
            x = synth.plaintext(1500, 64, 31, 0, dist)
            x0, x1 = synth.share(x, 64)
            j = np.arange(x.size, dtype=np.uint64)
            d = B.drelu(prm, x0, x1, j, SEEDS)
            y = B.reconstruct(d["y0"], d["y1"], 64)
            s, valid = band_sign(x, 64, 31, 0)
            assert valid.sum() > 1400
            if mode == "guard":
                assert np.array_equal(y[valid], s[valid])
            else:   # literal: a false positive needs one of 31 sums to hit 0 mod 2^31 -- none here
                assert np.mean(y[valid] == s[valid]) > 0.99
            zero = x == 0
            assert np.array_equal(y[zero], d["t"][zero])


def test_literal_large_false_positive_set():
    """Literal mode at lx = 10 mis-signs only inputs of the analytic set (C6)."""
    ell, lx, f = 24, 10, 0
    lit = B.Params(ell=ell, lx=lx, f=f, mode="literal")
    xi = np.arange(1, 1 << lx, dtype=np.uint64)
    x = np.repeat(np.concatenate([xi, np.uint64(1 << ell) - xi]), 4)
    x0, x1 = synth.share(x, ell)
    d = B.drelu(lit, x0, x1, np.arange(x.size, dtype=np.uint64), SEEDS)
    y = B.reconstruct(d["y0"], d["y1"], ell)
    s, _ = band_sign(x, ell, lx, f)
    bad = y != s
    mis = set(np.minimum(x[bad], np.uint64(1 << ell) - x[bad]).tolist())
    fp = _literal_fp_set(ell, lx, f)
    assert mis <= fp and len(mis) > 0
