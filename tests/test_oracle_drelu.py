"""Pins for oracle.bicoptor: DReLU / ReLU reconstructed against plaintext sign and
ReLU by brute force; the sign-determination table; tape invariants; the
literal-mode false-positive set derived analytically (reading C6)."""
import math
import os

import numpy as np
import pytest

import synth
from oracle import bicoptor as B
from oracle import ring
from plain import band_sign, relu_plain

GOLD = os.path.join(os.path.dirname(__file__), "golden", "dreluexp.txt")
SEEDS = synth.seeds(0)


def _rows():
    for line in open(GOLD):
        line = line.strip()
        if line and not line.startswith("#"):
            i, pv, pe, nv, ne = [s.strip() for s in line.split("|")]
            yield int(i), int(pv, 2), int(pe), int(nv, 2), int(ne)


def test_table_dreluexp_rows():
    """Table tab:dreluexp: ell=64, lx=7, x=+-22, literal domain Z_{2^7},
    no key-bit offset.  Every printed row value is the reconstructed ladder value
    for some mask R, and every reconstruction is the plaintext cut +- e0 in the
    printed direction (reading C16: no single R reproduces a whole column)."""
    prm = B.Params(ell=64, lx=7, f=0, mode="literal")
    rng = np.random.default_rng(1)
    R = rng.integers(0, 2**64, size=4000, dtype=np.uint64, endpoint=False)
    seen = {}
    for neg in (False, True):
        x = np.uint64(2**64 - 22) if neg else np.uint64(22)
        with np.errstate(over="ignore"):
            x0 = x + R
            x1 = np.uint64(0) - R
        u = (B.ladder(prm, 0, x0) + B.ladder(prm, 1, x1)) % np.uint64(128)
        for i in range(8):
            plain = 22 >> i
            ok = {plain % 128, (plain + 1) % 128} if not neg else {(-plain) % 128, (-plain - 1) % 128}
            assert set(np.unique(u[:, i]).tolist()) <= ok
            seen[(neg, i)] = set(np.unique(u[:, i]).tolist())
    for i, pv, pe, nv, ne in _rows():
        assert pv in seen[(False, i)] and nv in seen[(True, i)]
        assert pv == ((22 >> i) + max(pe, 0)) % 128 and nv == (-(22 >> i) + min(ne, 0)) % 128


def _pattern_ok(useq, pos, M):
    """Theorem thm:pattern0 on an opened ladder: positive -> a nonempty
    run of 1s then only 0s up to the top; negative -> a run of M-1 then 0s."""
    one = 1 if pos else M - 1
    idx = [i for i, v in enumerate(useq) if v == one]
    if not idx:
        return False
    last = idx[-1]
    return all(v == 0 for v in useq[last + 1:]) and all(useq[i] == one for i in range(idx[0], last + 1))


def test_ladder_pattern_theorem_exhaustive_ell12():
    """thm:pattern0 + lmm:pattern3-5: every in-band xi in [1, 2^lx), every mask R in
    Z_{2^12}: the opened ladder (beyond the first lambda-1 windows) is a run of
    +-1 followed by zeros."""
    ell, lx = 12, 5
    prm = B.Params(ell=ell, lx=lx, f=0, mode="guard")
    M = 1 << prm.w
    R = np.arange(1 << ell, dtype=np.uint64)
    mk = np.uint64((1 << ell) - 1)
    for xi in range(1, 1 << lx):
        lam = xi.bit_length()
        for neg in (False, True):
            x = np.uint64(((-xi) if neg else xi) % (1 << ell))
            x0 = (x + R) & mk
            x1 = (np.uint64(0) - R) & mk
            u = (B.ladder(prm, 0, x0) + B.ladder(prm, 1, x1)) % np.uint64(M)
            for row in u[:: 97]:
                assert _pattern_ok(row[lam - 1:].tolist(), not neg, M), (xi, neg, row)


def _run(prm, x, run=0):
    x0, x1 = synth.share(x, prm.ell, run)
    j = np.arange(x.size, dtype=np.uint64)
    return B.drelu(prm, x0, x1, j, SEEDS), B.relu(prm, x0, x1, j, SEEDS)


@pytest.mark.parametrize("ell,lx,f", [(12, 5, 0), (12, 4, 2), (16, 7, 0), (16, 6, 1)])
def test_drelu_bruteforce_sign_guard(ell, lx, f):
    """Brute force: every in-band nonzero x (2^f <= xi < 2^(f+lx)) x 64 masks R
    per x; guard mode must reconstruct the plaintext sign exactly, and ReLU must
    reconstruct max(x, 0)."""
    prm = B.Params(ell=ell, lx=lx, f=f, mode="guard")
    xi = np.arange(1 << f, 1 << (f + lx), dtype=np.uint64)
    xs = np.concatenate([xi, (np.uint64(1 << ell) - xi)])
    x = np.repeat(xs, 64)
    d, r = _run(prm, x)
    s, valid = band_sign(x, ell, lx, f)
    assert valid.all()
    assert np.array_equal(B.reconstruct(d["y0"], d["y1"], ell), s)
    assert np.array_equal(B.reconstruct(r["y0"], r["y1"], ell), relu_plain(x, ell, lx, f))


def test_drelu_ell64_keybits_d1_d2():
    """ell=64, f=24, lx=7 (the paper's 5+2 key bits of 5+26): synthetic
    D1 and D2 batches; sign exact wherever it is determined, ReLU = x*DReLU always."""
    prm = B.Params(ell=64, lx=7, f=24, mode="guard")
    for dist in ("D1", "D2"):
        x = synth.plaintext(30000, 64, 7, 24, dist)
        d, r = _run(prm, x)
        y = B.reconstruct(d["y0"], d["y1"], 64)
        s, valid = band_sign(x, 64, 7, 24)
        assert valid.sum() > 20000
        assert np.array_equal(y[valid], s[valid])
        with np.errstate(over="ignore"):
            assert np.array_equal(B.reconstruct(r["y0"], r["y1"], 64), x * y)


def test_drelu_zero_and_tiny():
    """Readings C13/C14: x=0 opens to the random bit t (so ReLU(0)=0); tiny
    |x| < 2^f is undetermined but ReLU error < 2^f."""
    prm = B.Params(ell=64, lx=7, f=24)
    x = np.zeros(4000, dtype=np.uint64)
    d, r = _run(prm, x)
    assert np.array_equal(B.reconstruct(d["y0"], d["y1"], 64), d["t"])
    assert np.all(B.reconstruct(r["y0"], r["y1"], 64) == 0)
    assert 1500 < int(d["t"].sum()) < 2500


def _literal_fp_set(ell, lx, f):
    """Analytic false-positive set of the paper-literal domain (reading C6): a
    negative s = -xi gives v_i = -(cut(xi, f+i) + b_i + cut(xi, f+i+1) + b_{i+1}) - 1
    mod 2^lx with borrow bits b in {0,1}; it is a (false) zero iff that sum is
    0 mod 2^lx for some i and bits."""
    M = 1 << lx
    bad = set()
    for xi in range(1 << f, 1 << (f + lx)):
        for i in range(lx):
            c = (xi >> (f + i)) + (xi >> (f + i + 1))
            # a borrow out of the low k bits needs xi mod 2^k != 0 (Lemma lmm:pattern2)
            bi = (0, 1) if xi % (1 << (f + i)) else (0,)
            bj = (0, 1) if xi % (1 << (f + i + 1)) else (0,)
            if any((c + a + b + 1) % M == 0 for a in bi for b in bj):
                bad.add(xi)
    return bad


def test_literal_mode_false_positive_set():
    """Literal mode mis-signs exactly inputs in the analytic set (both signs,
    because the blinding bit t flips positives into negatives); guard mode on the
    same inputs and tapes has none (reading C6)."""
    ell, lx, f = 16, 7, 0
    lit = B.Params(ell=ell, lx=lx, f=f, mode="literal")
    xi = np.arange(1, 1 << lx, dtype=np.uint64)
    x = np.repeat(np.concatenate([xi, np.uint64(1 << ell) - xi]), 32)
    d, _ = _run(lit, x)
    y = B.reconstruct(d["y0"], d["y1"], ell)
    s, _ = band_sign(x, ell, lx, f)
    mis = np.unique(np.minimum(x[y != s], (np.uint64(1 << ell) - x[y != s])))
    fp = _literal_fp_set(ell, lx, f)
    assert set(mis.tolist()) <= fp and 85 in set(mis.tolist())
    assert fp == {85}


def test_tape_invariants():
    """Tape decode: t is a fair bit, Pi a permutation (uniform over S!), masks
    in Z_p^*, reshares in Z_p; the rejection fallback is exercised."""
    for prm in (B.Params(), B.Params(ell=16, lx=7, f=0, mode="literal"), B.Params(ell=16, lx=4, f=1)):
        n = 60000
        tp = B.tape(prm, SEEDS.s01, np.arange(n, dtype=np.uint64))
        S, p = prm.slots, prm.p
        assert tp["r"].min() >= 1 and tp["r"].max() <= p - 1
        assert tp["rho"].max() <= p - 1
        assert abs(int(tp["t"].sum()) - n // 2) < 5 * math.sqrt(n)
        perm = B.shuffle(tp["k"], np.tile(np.arange(S, dtype=np.uint64), (n, 1)))
        assert np.all(np.sort(perm, axis=1) == np.arange(S))
        # position of slot 0 after the shuffle is uniform over S positions
        pos0 = np.argmax(perm == 0, axis=1)
        cnt = np.bincount(pos0, minlength=S)
        assert np.all(np.abs(cnt - n / S) < 6 * math.sqrt(n / S))
        if prm.compact:
            rb = tp["r"].ravel()
            assert np.bincount(rb.astype(np.int64), minlength=257)[1:].min() > 0


def _compact_rejects(prm, j):
    """Elements whose compact tape has a rejected draw (perm index >= 53261*8!,
    or a reshare word >= 253*257^3), recomputed from the raw keystream."""
    from oracle.chacha import element_u32
    A = element_u32(SEEDS.s01, B.L_TAPEA, prm.rounds, j, 4)
    Bw = element_u32(SEEDS.s01, B.L_TAPEB, prm.rounds, j, 2)
    bad = ((A[:, 0] & 0x7FFFFFFF) >= B.PERM_LIMIT_COMPACT) | (A[:, 3] >= B.RHO_WORD_LIMIT) | \
        (Bw[:, 0] >= B.RHO_WORD_LIMIT) | (Bw[:, 1] >= B.RHO_WORD_LIMIT)
    return np.nonzero(bad)[0], A, Bw


def test_tape_fallback_path():
    """Find elements whose compact tape rejects and check the fallback decode:
    the first rejected reshare word is replaced by the first fallback word
    below the limit, and its digits are what the decode returns."""
    from oracle.chacha import chacha_blocks
    prm = B.Params()
    j = np.arange(40000, dtype=np.uint64)
    rej, A, Bw = _compact_rejects(prm, j)
    assert len(rej) > 0
    tp = B.tape(prm, SEEDS.s01, j[rej])
    for row, jj in enumerate(rej[:8]):
        words = [int(A[jj, 3]), int(Bw[jj, 0]), int(Bw[jj, 1])]
        if (A[jj, 0] & 0x7FFFFFFF) >= B.PERM_LIMIT_COMPACT:
            continue
        k = next(i for i, w in enumerate(words) if w >= B.RHO_WORD_LIMIT)
        fb = [int(w) for w in chacha_blocks(SEEDS.s01, B.L_FALLBACK, [int(jj) * 256], prm.rounds)[0]]
        v = next(w for w in fb if w < B.RHO_WORD_LIMIT)
        got = [int(tp["rho"][row, 3 * k + i]) for i in range(3) if 3 * k + i < 8]
        assert got == [(v // 257 ** i) % 257 for i in range(3)][: len(got)]


def test_reshare_digits_uniform():
    """The base-257 digits of an accepted word are uniform on Z_257 (chi-square)."""
    tp = B.tape(B.Params(), SEEDS.s01, np.arange(60000, dtype=np.uint64))
    cnt = np.bincount(tp["rho"].ravel().astype(np.int64), minlength=257)
    assert cnt.size == 257
    exp = tp["rho"].size / 257
    chi2 = float(((cnt - exp) ** 2 / exp).sum())
    assert chi2 < 256 + 6 * math.sqrt(2 * 256)


def test_mask_and_shuffle_preserve_zero_existence():
    """Alg 7 steps 6-8: for the opened vectors, (W0+W1) mod p is
    v'_{Pi(m)} * r_m, so a zero exists after masking iff it existed before."""
    prm = B.Params(ell=64, lx=7, f=24)
    x, x0, x1 = synth.shares(5000, 64, 7, 24, "D1")
    j = np.arange(5000, dtype=np.uint64)
    m0, m1 = B.drelu_send(prm, 0, x0, j, SEEDS.s01), B.drelu_send(prm, 1, x1, j, SEEDS.s01)
    tp = B.tape(prm, SEEDS.s01, j)
    s0 = np.where(tp["t"] == 1, ring.neg(x0, 64), x0).astype(np.uint64)
    s1 = np.where(tp["t"] == 1, ring.neg(x1, 64), x1).astype(np.uint64)
    v = (B.ladder_modswitch(prm, 0, s0) + B.ladder_modswitch(prm, 1, s1)) % np.uint64(prm.p)
    pv = B.shuffle(tp["k"], v)
    W = (m0["W"] + m1["W"]) % np.uint64(prm.p)
    assert np.array_equal(W, (pv * tp["r"]) % np.uint64(prm.p))
    assert np.array_equal((v == 0).any(axis=1), (W == 0).any(axis=1))


def test_wire_bits_match_table1():
    """Table 1: one-pass cost (lx+1)*(lx+1) = 64 bits per party in the
    paper-literal domain at lx=7; guard mode sends (lx+1)*ceil(log2 257) = 72."""
    for mode, bits in (("literal", 64), ("guard", 72)):
        prm = B.Params(ell=64, lx=7, f=24, mode=mode)
        assert prm.slots * math.ceil(math.log2(prm.p)) == bits


def test_party_composition_matches_drelu():
    prm = B.Params()
    x, x0, x1 = synth.shares(3000, 64, 7, 24, "D2")
    j = np.arange(3000, dtype=np.uint64) + np.uint64(1 << 40)
    d = B.drelu(prm, x0, x1, j, SEEDS)
    m0 = B.drelu_send(prm, 0, x0, j, SEEDS.s01)
    m1 = B.drelu_send(prm, 1, x1, j, SEEDS.s01)
    h = B.drelu_helper(prm, m0["W"], m1["W"], j, SEEDS.s02)
    assert np.array_equal(B.drelu_finish(prm, 0, m0["t"], h["D0"]), d["y0"])
    assert np.array_equal(B.drelu_finish(prm, 1, m1["t"], h["D1"]), d["y1"])
    lo, hi = B.encode_msg(m0["W"])
    back = lo[:, :8].astype(np.uint64) | ((hi[:, None] >> np.arange(8, dtype=np.uint8)) & 1).astype(np.uint64) << np.uint64(8)
    assert np.array_equal(back, m0["W"])


@pytest.mark.parametrize("kw,layout", [(dict(ell=16, lx=7, f=0, mode="literal"), "compact_lit"),
                                       (dict(ell=32, lx=5, f=3, mode="guard"), "pair"),
                                       (dict(ell=12, lx=3, f=1, mode="literal"), "pair")])
def test_pair_tape_raw_draws(kw, layout):
    """Pair tape (p <= 131, layout spec DESIGN.md §4): re-read the 32 keystream bytes
    of each element from whole ChaCha blocks (element j = bytes [32 j, 32 j + 32) of
    the bc2.tpp1 stream), take the 28-bit draws as bit strings, and check
    r_m = 1 + (u mod d) mod (p-1) and rho_m = (u mod d) div (p-1), d = (p-1) p, on
    unrejected elements; on a rejected element the rejected draw is replaced by the
    first fallback word whose low 28 bits fall below the limit.  Also: the pair
    (r, rho) covers Z_p^* x Z_p uniformly (chi-square)."""
    from oracle.chacha import chacha_blocks
    prm = B.Params(**kw)
    S, p = prm.slots, prm.p
    assert prm.layout == layout and p <= 131
    d = (p - 1) * p
    lim = ((1 << 28) // d) * d
    assert lim <= 1 << 28 < lim + d
    fact = math.factorial(S)
    plim = ((1 << 31) // fact) * fact
    n = 4000
    blocks = chacha_blocks(SEEDS.s01, B.L_TAPEP, list(range(n // 2)), prm.rounds)
    raw = np.asarray(blocks, dtype="<u4").tobytes()
    tp = B.tape(prm, SEEDS.s01, np.arange(n, dtype=np.uint64))
    ok_rows = 0
    for jj in range(n):
        e = raw[32 * jj: 32 * jj + 32]
        w0 = int.from_bytes(e[:4], "little")
        bits = "".join(format(b, "08b")[::-1] for b in e[4:])  # LSB-first bit string of D
        u = [int(bits[28 * i: 28 * i + 28][::-1], 2) for i in range(S)]
        assert int(tp["t"][jj]) == w0 >> 31
        if (w0 & 0x7FFFFFFF) >= plim or any(v >= lim for v in u):
            continue
        ok_rows += 1
        assert [int(v) for v in tp["r"][jj]] == [1 + (v % d) % (p - 1) for v in u]
        assert [int(v) for v in tp["rho"][jj]] == [(v % d) // (p - 1) for v in u]
    assert ok_rows > 3980
    # rejected draws: search a wider range from the raw words
    jr = np.arange(1 << 15, dtype=np.uint64)
    T = np.asarray(chacha_blocks(SEEDS.s01, B.L_TAPEP, list(range(1 << 14)), prm.rounds), dtype="<u4")
    T = T.reshape(-1, 8)
    found = 0
    for jj in range(T.shape[0]):
        if (int(T[jj, 0]) & 0x7FFFFFFF) >= plim:
            continue
        D = sum(int(T[jj, w]) << (32 * (w - 1)) for w in range(1, 8))
        bad = [m for m in range(S) if ((D >> (28 * m)) & 0xFFFFFFF) >= lim]
        if len(bad) != 1:
            continue
        m = bad[0]
        fb = [int(w) & 0xFFFFFFF for w in chacha_blocks(SEEDS.s01, B.L_FALLBACK, [jj * 256], prm.rounds)[0]]
        x = next(w for w in fb if w < lim) % d
        got = B.tape(prm, SEEDS.s01, jr[jj:jj + 1])
        assert (int(got["r"][0, m]), int(got["rho"][0, m])) == (1 + x % (p - 1), x // (p - 1))
        found += 1
        if found >= 3:
            break
    expected = (1 << 15) * S * ((1 << 28) - lim) / (1 << 28)
    assert found >= 1 or expected < 3   # p = 11: 2^28 - lim = 6, no rejection in range
    tp = B.tape(prm, SEEDS.s01, np.arange(60000, dtype=np.uint64))
    cells = ((tp["r"] - 1) * p + tp["rho"]).ravel().astype(np.int64)
    cnt = np.bincount(cells, minlength=d)
    assert cnt.size == d and tp["r"].min() >= 1 and tp["rho"].max() <= p - 1
    exp = cells.size / d
    chi2 = float(((cnt - exp) ** 2 / exp).sum())
    assert chi2 < (d - 1) + 6 * math.sqrt(2 * (d - 1))


def _pair_rejects(prm, nblocks):
    """Elements (of the first 2 * nblocks) whose pair tape takes the fallback stream:
    the perm index >= floor(2^31/S!) S! or a 28-bit draw >= floor(2^28/d) d, found
    from the raw keystream words."""
    from oracle.chacha import chacha_blocks
    S, p = prm.slots, prm.p
    d = (p - 1) * p
    lim = ((1 << 28) // d) * d
    fact = math.factorial(S)
    plim = ((1 << 31) // fact) * fact
    T = np.asarray(chacha_blocks(SEEDS.s01, B.L_TAPEP, list(range(nblocks)), prm.rounds), dtype="<u4").reshape(-1, 8)
    out = []
    for jj in range(T.shape[0]):
        D = sum(int(T[jj, w]) << (32 * (w - 1)) for w in range(1, 8))
        if (int(T[jj, 0]) & 0x7FFFFFFF) >= plim or any(((D >> (28 * m)) & 0xFFFFFFF) >= lim for m in range(S)):
            out.append(jj)
    return out
