"""Pins for oracle.rss (Alg 9): RSS sharing algebra, the secret
multiplication, and DReLU / ReLU reconstructed against plaintext by brute force."""
import numpy as np
import pytest

import synth
from oracle import bicoptor as B
from oracle import ring, rss
from plain import band_sign, relu_plain

SEEDS = synth.seeds(0)


def test_zero_share_and_multiplication():
    prm = B.Params(ell=64, lx=7, f=24)
    n = 5000
    j = np.arange(n, dtype=np.uint64)
    g = rss.zero_share(prm, SEEDS, j, rss.L_MUL)
    assert np.all(rss.reconstruct(g, 64) == 0)
    rng = np.random.default_rng(4)
    a = [rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True) for _ in range(3)]
    b = [rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True) for _ in range(3)]
    z = rss.rss_mul(prm, a, b, g)
    with np.errstate(over="ignore"):
        assert np.array_equal(rss.reconstruct(z, 64), rss.reconstruct(a, 64) * rss.reconstruct(b, 64))


def test_preprocessing_reconstructs_t_s_and_xor():
    """Alg 9 preprocessing: [t] opens to the seed01 bit t, [s] to P2's bit s,
    [s xor t] to s xor t; [t]_1 is the only component that depends on t."""
    prm = B.Params(ell=16, lx=7, f=0)
    j = np.arange(4000, dtype=np.uint64)
    pre = rss.preprocess(prm, SEEDS, j)
    assert np.array_equal(rss.reconstruct(pre["tsh"], 16), pre["t"])
    assert np.array_equal(rss.reconstruct(pre["ssh"], 16), pre["s"])
    assert np.array_equal(rss.reconstruct(pre["u"], 16), pre["s"] ^ pre["t"])
    assert 1500 < int(pre["s"].sum()) < 2500


@pytest.mark.parametrize("ell,lx,f", [(12, 5, 0), (16, 7, 0), (16, 6, 1)])
def test_drelu_rss_bruteforce(ell, lx, f):
    """Every in-band nonzero x, 32 sharings each: RSS DReLU opens to the plaintext
    sign, RSS ReLU to max(x, 0)."""
    prm = B.Params(ell=ell, lx=lx, f=f)
    xi = np.arange(1 << f, 1 << (f + lx), dtype=np.uint64)
    x = np.repeat(np.concatenate([xi, np.uint64(1 << ell) - xi]), 32)
    xs = synth.rss_share(x, ell)
    j = np.arange(x.size, dtype=np.uint64)
    d = rss.drelu_rss(prm, *xs, j, SEEDS)
    s, valid = band_sign(x, ell, lx, f)
    assert valid.all() and np.array_equal(rss.reconstruct(d["y"], ell), s)
    r = rss.relu_rss(prm, *xs, j, SEEDS)
    assert np.array_equal(rss.reconstruct(r["y"], ell), relu_plain(x, ell, lx, f))


def test_drelu_rss_ell64_matches_ubl_sign():
    """At ell=64 (5+2 key bits) RSS DReLU opens to the plaintext sign wherever the
    key bits determine it, exactly like UBL DReLU on the same x (D1 and D2)."""
    prm = B.Params(ell=64, lx=7, f=24)
    for dist in ("D1", "D2"):
        x = synth.plaintext(20000, 64, 7, 24, dist)
        j = np.arange(x.size, dtype=np.uint64)
        xs = synth.rss_share(x, 64)
        d = rss.drelu_rss(prm, *xs, j, SEEDS)
        x0, x1 = synth.share(x, 64)
        u = B.drelu(prm, x0, x1, j, SEEDS)
        sgn, valid = band_sign(x, 64, 7, 24)
        yr, yu = rss.reconstruct(d["y"], 64), B.reconstruct(u["y0"], u["y1"], 64)
        assert valid.sum() > 15000
        assert np.array_equal(yr[valid], sgn[valid]) and np.array_equal(yu[valid], sgn[valid])
        assert np.array_equal(yr[x == 0], d["t"][x == 0])   # DReLU(0) = t (reading C13)
