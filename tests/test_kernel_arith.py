"""CPU checks of the integer identities the CUDA kernels rely on, against their
plain definitions (no oracle involved): each kernel trick is re-expressed in
Python with 32/64-bit wrap-around and compared over its whole domain (or a
large random sample where the domain is 2^64)."""
import numpy as np

M32 = (1 << 32) - 1
M64 = (1 << 64) - 1


def umulhi32(a, b):
    return (a * b) >> 32


# ---- compact path (csrc/bc_compact.cuh) -------------------------------------------------

def test_div257s_exact_below_2pow24():
    """div257s(x) = umulhi(x, 0xFF0100) == x // 257 for every x < 2^24 (the
    kernel applies it to quotients q1 = w // 257 < 2^24 and q2 < 2^16)."""
    x = np.arange(1 << 24, dtype=np.uint64)
    assert np.array_equal((x * np.uint64(0xFF0100)) >> np.uint64(32), x // np.uint64(257))
    # and not one step further: 2^24 = 257 * 65281 - 1 is the first x whose quotient overshoots
    x = np.uint64(1 << 24)
    assert (x * np.uint64(0xFF0100)) >> np.uint64(32) == x // np.uint64(257) + np.uint64(1)


def test_table_v2_offsets_stay_below_2pow24():
    """decode_t2 / elem_both_t2 (csrc/bc_compact.cuh): the reshare offsets o0 = rho + 257 k and
    o1 = 257 K - rho are congruent to +-rho_m mod 257, positive, and keep the messages
    x = v' r + o below 2^24 (div257s' exact range) for every reshare word below the limit."""
    LIM = 253 * 257 ** 3
    rng = np.random.default_rng(7)
    w = np.concatenate([rng.integers(0, LIM, 1 << 20, dtype=np.uint64),
                        np.array([0, 1, 256, 257, LIM - 1, LIM - 257, 257 ** 3 - 1], dtype=np.uint64)])
    q1 = w // np.uint64(257)
    q2 = q1 // np.uint64(257)
    rho = [w % np.uint64(257), q1 % np.uint64(257), q2 % np.uint64(257)]
    o0 = [w - np.uint64(257) * q1, q1, q2]
    o1 = [np.uint64(257) * q1 + np.uint64(257) - w, np.uint64(16710397) - q1, np.uint64(65792) - q2]
    for i in range(3):
        assert (o1[i].astype(np.int64) > 0).all()
        assert np.array_equal(o0[i] % np.uint64(257), rho[i])
        assert np.array_equal((o1[i] + rho[i]) % np.uint64(257), np.zeros_like(w))
        assert int(o0[i].max()) + 256 * 256 < (1 << 24) and int(o1[i].max()) + 256 * 256 < (1 << 24)


def test_div257_exact_all_u32_sample_and_edges():
    """div257(x) = umulhi(x, 0xFF00FF01) >> 8 == x // 257 for every 32-bit x
    (checked on all multiples-of-257 neighbourhoods and 2^22 random values)."""
    rng = np.random.default_rng(0)
    xs = list(rng.integers(0, 2**32, 1 << 16, dtype=np.uint64))
    xs += [q * 257 + d for q in range(0, (1 << 32) // 257, 4099) for d in (0, 1, 255, 256)]
    xs += [M32, M32 - 1, 0, 1, 256, 257]
    for x in xs:
        x = int(x) & M32
        assert (umulhi32(x, 0xFF00FF01) >> 8) == x // 257


def test_mod257s_exact_below_2_18():
    """mod257s(x) = x - 257 umulhi(x, 0xFF0100) == x % 257 for x < 2^18."""
    x = np.arange(1 << 18, dtype=np.uint64)
    q = (x * np.uint64(0xFF0100)) >> np.uint64(32)
    assert np.array_equal(x - np.uint64(257) * q, x % np.uint64(257))


def test_multiplicative_divisibility_test_below_2_25():
    """257 | s  <=>  s * 257^-1 mod 2^32 <= floor((2^32-1)/257) for every s < 2^32 (s -> s 257^-1 is a
    bijection of Z_{2^32} taking the multiples 257 k, k <= floor((2^32-1)/257), to k); checked
    exhaustively below 2^25, the range of P2's sums W0 + x1 in the table kernels (< 257 + 2^24),
    and the same for 131 (the literal table kernel, sums < 2^17)."""
    s = np.arange(1 << 25, dtype=np.uint64)
    lhs = ((s * np.uint64(0xFF00FF01)) & np.uint64(M32)) <= np.uint64(16711935)
    assert (0xFF00FF01 * 257) & M32 == 1
    assert np.array_equal(lhs, s % np.uint64(257) == 0)
    s = np.arange(1 << 18, dtype=np.uint64)
    assert (0xC9484E2B * 131) & M32 == 1 and (2**32 - 1) // 131 == 32786009
    lhs = ((s * np.uint64(0xC9484E2B)) & np.uint64(M32)) <= np.uint64(32786009)
    assert np.array_equal(lhs, s % np.uint64(131) == 0)


def test_p2_distributive_form():
    """P2's test by distributivity (BC_P2_DIST, elem_both_t2 / elem_both_tl): with q0 = x0 div p,
    (W0 + x1) p^-1 = x0 p^-1 + x1 p^-1 - q0 (mod 2^32) because p p^-1 = 1; random x0 < 2^24, x1 < 2^24."""
    rng = np.random.default_rng(11)
    for p, inv in ((257, 0xFF00FF01), (131, 0xC9484E2B)):
        x0 = rng.integers(0, 1 << 24, 1 << 20, dtype=np.uint64)
        x1 = rng.integers(0, 1 << 24, 1 << 20, dtype=np.uint64)
        q0 = x0 // np.uint64(p)
        w0 = x0 - np.uint64(p) * q0
        lhs = ((w0 + x1) * np.uint64(inv)) & np.uint64(M32)
        rhs = (x0 * np.uint64(inv) + x1 * np.uint64(inv) - q0) & np.uint64(M32)
        assert np.array_equal(lhs, rhs)


def test_ladder_swar_all_windows():
    """ladder_swar: for every 15-bit window, the bytes produced by the 64-bit
    spread multiply equal the direct per-slot values u_i + u_{i+1} - 2 (P0) and
    -(u_i + u_{i+1}) (P1), mod 256, with u_i the 8-bit window at bit i."""
    KL = 1 + (1 << 14) + (1 << 28)
    MM = 0x00FF00FF

    def swar(win, party):
        e, o = win & 0x3FFF, (win >> 1) & 0x3FFF
        Elo, Ehi = (e * KL) & M32 & MM, ((e >> 4) + (e << 10)) & MM
        Olo, Ohi = (o * KL) & M32 & MM, ((o >> 4) + (o << 10)) & MM
        Slo = ((Elo >> 16) | (Ehi << 16)) & M32
        Shi = Ehi >> 16
        if party == 0:
            ce_lo, ce_hi = (Elo + Olo + 0x00FE00FE) & M32, (Ehi + Ohi + 0x00FE00FE) & M32
            co_lo, co_hi = (Olo + Slo + 0x00FE00FE) & M32, (Ohi + Shi + 0x00FE00FE) & M32
        else:
            ce_lo, ce_hi = (0x04000400 - Elo - Olo) & M32, (0x04000400 - Ehi - Ohi) & M32
            co_lo, co_hi = (0x04000400 - Olo - Slo) & M32, (0x04000400 - Ohi - Shi) & M32
        lo = (ce_lo & MM) | ((co_lo << 8) & ~MM & M32)
        hi = (ce_hi & MM) | ((co_hi << 8) & ~MM & M32)
        return [(lo >> (8 * k)) & 255 for k in range(4)] + [(hi >> (8 * k)) & 255 for k in range(4)]

    for win in range(1 << 15):
        u = [(win >> i) & 255 for i in range(8)]
        want0 = [(u[i] + (u[i + 1] if i < 7 else 0) - 2) & 255 for i in range(8)]
        want1 = [(-(u[i] + (u[i + 1] if i < 7 else 0))) & 255 for i in range(8)]
        assert swar(win, 0) == want0, win
        assert swar(win, 1) == want1, win


# ---- large path (csrc/bc_large.cuh) -----------------------------------------------------

def _kpl(p):
    inv = p
    for _ in range(5):
        inv = (inv * (2 - p * inv)) & M64
    assert (inv * p) & M64 == 1
    return {"p": p, "pinv": inv, "mu_p": M64 // p, "mu_q": M64 // (p - 1)}


def mont(a, b, k):
    lo, hi = (a * b) & M64, (a * b) >> 64
    mh = (((lo * k["pinv"]) & M64) * k["p"]) >> 64
    return hi - mh if hi >= mh else (hi - mh + k["p"]) & M64


def barrett(u, q, mu):
    r = (u - ((u * mu) >> 64) * q) & M64
    return r - q if r >= q else r


def test_subtractive_redc_and_barrett():
    rng = np.random.default_rng(1)
    for p in (2**32 + 15, 2**31 + 11, 65537, 521, 2053):
        k = _kpl(p)
        rinv = pow(2, -64, p)
        for _ in range(3000):
            a, b = int(rng.integers(0, p)), int(rng.integers(0, p))
            assert mont(a, b, k) == a * b * rinv % p
            u = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
            assert barrett(u, p, k["mu_p"]) == u % p
            assert barrett(u, p - 1, k["mu_q"]) == u % (p - 1)
        for a, b in ((p - 1, p - 1), (0, p - 1), (1, 1)):
            assert mont(a, b, k) == a * b * rinv % p
        for u in (M64, M64 - 1, 0, p, p - 1):
            assert barrett(u, p, k["mu_p"]) == u % p and barrett(u, p - 1, k["mu_q"]) == u % (p - 1)


def test_funnel_windows_match_shifts():
    """slot_values: bits [i, i+w) of a 64-bit value via a clamped 32-bit funnel
    shift equal (v >> i) & (2^w - 1) for i <= 31, and the successor window at
    i + 1 <= 32 (clamped shift of 32 = the high word)."""
    rng = np.random.default_rng(2)

    def fsr(lo, hi, s, clamp):
        s = min(s, 32) if clamp else s & 31
        return (((hi << 32) | lo) >> s) & M32

    for _ in range(2000):
        v = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        lo, hi = v & M32, v >> 32
        for w in (9, 16, 31, 32):
            wm = (1 << w) - 1
            for i in range(32):
                assert fsr(lo, hi, i, False) & wm == (v >> i) & wm
                assert fsr(lo, hi, i + 1, True) & wm == (v >> (i + 1)) & wm


def test_fisher_yates_magic_division():
    """k = d - umulhi(d, ceil(2^32 / s)) s == d mod s for 16-bit d and s <= 32."""
    d = np.arange(1 << 16, dtype=np.uint64)
    for s in range(2, 33):
        magic = (M32 // s) + 1
        q = (d * np.uint64(magic)) >> np.uint64(32)
        assert np.array_equal(d - q * np.uint64(s), d % np.uint64(s)), s


def _fp_quotient(v, qo):
    """The kernel's fpmod48 quotient, emulated exactly: vd = v - (qo-1)/2 (exact in
    binary64), then RN(vd * RN(1/qo) + 1.5 * 2^52), whose grid at that magnitude is
    the integers: round half to even of the exact rational."""
    from fractions import Fraction
    vd = Fraction(v) - Fraction(qo - 1, 2)
    x = vd * Fraction(1.0 / qo) + Fraction(3 << 51)
    fl = x.numerator // x.denominator
    rem = x - fl
    r = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2) else 0)
    return r - (3 << 51)


def test_fpmod48_quotient_exact():
    """floor(u / q) = floor(v / q'), v = u >> s, q = q' 2^s (q' odd), and the binary64
    quotient the large-tape kernel uses (BC_LARGE_FPMOD) is exactly floor(v / q') for
    every draw u < 2^48: the moduli of every large-tape setting (p and p - 1 for
    w = 9..32), random draws and the draws next to multiples of q and to 2^48."""
    from oracle.ring import prime_above
    rng = np.random.default_rng(7)
    for w in range(9, 33):
        p = prime_above(w)
        for q in (p, p - 1):
            s = (q & -q).bit_length() - 1
            qo = q >> s
            us = [0, 1, q - 1, q, q + 1, (1 << 48) - 1, ((1 << 48) // q) * q - 1, ((1 << 48) // q) * q - 2]
            us += [int(v) for v in rng.integers(0, 1 << 48, size=40, dtype=np.uint64)]
            k = [int(v) for v in rng.integers(1, (1 << 48) // q, size=20, dtype=np.uint64)]
            us += [m * q + d for m in k for d in (-1, 0, 1, q // 2, q - 1) if 0 <= m * q + d < (1 << 48)]
            for u in us:
                assert _fp_quotient(u >> s, qo) == u // q, (w, q, u)


def test_small_domain_magic_divisions():
    """The runtime divisions by host-computed magics of the small domains (KP::mag_p,
    mag_q, mag_f): x / d = umulhi(x, ceil(2^32/d)) for every 16-bit value and every
    d = p, p-1 of an lx <= 7 setting (w = 2..8); x / S! = umulhi(x, ceil(2^(31+l)/S!)) >> (l-1)
    for 31-bit indices (l = ceil(log2 S!)), sampled plus the multiples' edges."""
    import math
    from oracle.ring import prime_above
    x16 = np.arange(1 << 16, dtype=np.uint64)
    for w in range(2, 9):
        p = prime_above(w)
        for d in (p, p - 1):
            mag = np.uint64(((1 << 32) + d - 1) // d)
            assert np.array_equal((x16 * mag) >> np.uint64(32), x16 // np.uint64(d)), (w, d)
    rng = np.random.default_rng(3)
    for S in range(3, 9):
        f = math.factorial(S)
        l = (f - 1).bit_length()
        mag = ((1 << (31 + l)) + f - 1) // f
        assert mag < (1 << 32)
        xs = np.concatenate([rng.integers(0, 1 << 31, 100000, dtype=np.uint64),
                             np.array([0, f - 1, f, (1 << 31) - 1], dtype=np.uint64),
                             np.arange(1, 2000, dtype=np.uint64) * np.uint64(f) - np.uint64(1)])
        xs = xs[xs < (1 << 31)]
        q = ((xs * np.uint64(mag)) >> np.uint64(32)) >> np.uint64(l - 1)
        assert np.array_equal(q, xs // np.uint64(f)), S


def test_compact_literal_pair_division():
    """decode_cl (csrc/bc_device.cuh): u / 17030 = umulhi(u, ceil(2^46/17030)) >> 14 for
    every 28-bit u (exhaustive), and x div 130 by the 16-bit magic for x < 17030."""
    pair = 130 * 131
    mag = ((1 << 46) + pair - 1) // pair
    assert mag <= M32
    for c in range(16):
        u = np.arange(c << 24, (c + 1) << 24, dtype=np.uint64)
        q = ((u * np.uint64(mag)) >> np.uint64(32)) >> np.uint64(14)
        assert np.array_equal(q, u // np.uint64(pair))
    x = np.arange(pair, dtype=np.uint64)
    mq = ((1 << 32) + 129) // 130
    assert np.array_equal((x * np.uint64(mq)) >> np.uint64(32), x // np.uint64(130))


def test_pair_tape_runtime_magic():
    """decode_pair (csrc/bc_device.cuh) with make_kp's runtime magic: for every prime the
    pair tape serves (p = prime above 2^w, w = 2..7), d = (p-1) p is not a power of two,
    M = ceil(2^(32+k)/d) < 2^32 with k = floor(log2 d), the bound u e < 2^(32+k) holds
    for u < 2^28 (so u div d is exact everywhere), and a sample plus the edges agree."""
    from oracle.ring import prime_above
    rng = np.random.default_rng(5)
    for w in range(2, 8):
        p = prime_above(w)
        d = (p - 1) * p
        assert d & (d - 1) and d < 1 << 16
        k = d.bit_length() - 1
        mag = ((1 << (32 + k)) + d - 1) // d
        assert mag <= M32 and ((1 << 28) - 1) * (mag * d - (1 << (32 + k))) < 1 << (32 + k)
        u = np.concatenate([rng.integers(0, 1 << 28, 1 << 20, dtype=np.uint64),
                            np.arange(d * 3, dtype=np.uint64), np.arange((1 << 28) - d * 3, 1 << 28, dtype=np.uint64)])
        q = ((u * np.uint64(mag)) >> np.uint64(32)) >> np.uint64(k)
        assert np.array_equal(q, u // np.uint64(d)), p


def test_literal_table_kernel_divisions():
    """elem_both_tl (csrc/bc_compact.cuh): x div 131 = umulhi(x, ceil(2^32/131)) for every x < 2^16
    (P0's message x0 = v' r + rho < 130 * 130 + 131, P1's x1 < 2^16), and the wire value x - 131 q."""
    x = np.arange(1 << 16, dtype=np.uint64)
    q = (x * np.uint64(32786010)) >> np.uint64(32)
    assert -(-(2**32) // 131) == 32786010
    assert np.array_equal(q, x // np.uint64(131))


# ---- large tape at p = 2^32 + 15 (csrc/bc_large.cuh, BC_LARGE_P15) -----------------------

P15 = (1 << 32) + 15


def _fold_p15(x):
    """fold_p15 with the kernel's 32/64-bit wrap-around: y = x0 - 15 x1 (mod 2^64),
    y1 = signed high word, result y0 + (-15 y1 mod 2^32)."""
    y = ((x & M32) - (x >> 32) * 15) & M64
    y1 = (y >> 32) - (1 << 32) if (y >> 63) else (y >> 32)
    return (y & M32) + ((-15 * y1) & M32)


def _mod_c(u, c, q):
    v = (u & M32) - ((c * (u >> 32)) & M32)      # int64 of a u32 minus a u32 product < 2^20
    return v + q if v < 0 else v


def test_p15_fold_and_draw_reductions():
    """fold_p15(x) = x mod p up to one subtraction (result <= 2^32 + 225) for every 64-bit x
    (edges and 2e5 random); mod_p15 / mod_q15 = u mod p / u mod (p-1) for 48-bit draws;
    K15 = 2^-64 mod p (the mask's Montgomery form, reading C28)."""
    rng = np.random.default_rng(15)
    xs = [0, 1, M32, 1 << 32, P15, P15 - 1, M64, M64 - 1, (M32 * M32), (M32 * M32) + P15, (1 << 63), (15 << 32), (15 << 32) - 1]
    xs += [int(v) for v in rng.integers(0, 1 << 63, size=100000, dtype=np.uint64)]
    xs += [int(v) | (1 << 63) for v in rng.integers(0, 1 << 63, size=100000, dtype=np.uint64)]
    xs += [k * P15 + e for k in (1, 2, 3, (1 << 31), M32 - 1) for e in (0, 1, 14, 15, 16)]
    for x in xs:
        x &= M64
        z = _fold_p15(x)
        assert z % P15 == x % P15 and 0 <= z <= (1 << 32) + 225, x
    us = [0, 1, (1 << 48) - 1, P15, P15 - 1, (1 << 32) - 1, 1 << 32] + \
        [int(v) for v in rng.integers(0, 1 << 48, size=200000, dtype=np.uint64)]
    for u in us:
        assert _mod_c(u, 15, P15) == u % P15
        assert _mod_c(u, 14, P15 - 1) == u % (P15 - 1)
    # draws_p15: the same reductions on 32 bits, with the wrap flag exactly "result >= 2^32"
    edge = [(k << 32) + e for k in (0, 1, 2, 0xFFFF) for e in
            (0, 1, 13, 14, 15, 16, 14 * k, 15 * k, 14 * k - 1, 15 * k - 1, M32, M32 - 14)]
    for u in us[:50000] + [v & ((1 << 48) - 1) for v in edge if v >= 0]:
        for v in (u, (u * 7919) & ((1 << 48) - 1)):
            mr, u0 = (14 * (u >> 32)) & M32, u & M32
            ar = 15 if u0 < mr else 1
            rM = ((u0 - mr) + ar) & M32
            mq, v0 = (15 * (v >> 32)) & M32, v & M32
            aq = 15 if v0 < mq else 0
            rho = ((v0 - mq) + aq) & M32
            want_r, want_q = 1 + u % (P15 - 1), v % P15
            ok = rM >= ar and rho >= aq
            assert ok == (want_r < (1 << 32) and want_q < (1 << 32)), (u, v)
            if ok:
                assert rM == want_r and rho == want_q
    assert pow(2, -64, P15) == 0x9876543B


def test_p15_slot_zero_test():
    """The W32 slot of elem_large: W0 = c r + rho reduced, W1 = d r + (p - rho) folded; P2's
    test s0 == 15 s1 on s = W0 + W1 is exactly (c + d) r = 0 (mod p), i.e. c + d = 0 (r a
    unit); and the 64-bit products plus addends never wrap for operands below 2^32."""
    rng = np.random.default_rng(16)
    cases = []
    for _ in range(50000):
        c = int(rng.integers(1, 1 << 32))
        r = int(rng.integers(1, 1 << 32))
        rho = int(rng.integers(0, P15))
        d = (P15 - c) % P15 if rng.random() < 0.3 else int(rng.integers(15, 1 << 32))
        cases.append((c, d, r, rho))
    cases += [(M32, M32, M32, P15 - 1), (1, M32, M32, 0), (M32, 16, M32, P15 - 1), (1, M32, 1, 0),
              (16, M32, M32, 5)]  # c + d = p: a zero slot at the operand edges
    for c, d, r, rho in cases:
        if d >= (1 << 32):
            continue
        x0 = c * r + rho
        x1 = d * r + (P15 - rho)
        assert x0 <= M64 and x1 <= M64
        w0 = _fold_p15(x0)
        w0 = w0 - P15 if w0 >= P15 else w0
        w1 = _fold_p15(x1)
        s = w0 + w1
        assert s < 3 << 32
        got = (s & M32) == 15 * (s >> 32)
        assert got == (((c + d) * r) % P15 == 0), (c, d, r, rho)


# ---- large tape at p = 2^31 + 11 (csrc/bc_large.cuh, BC_LARGE_P31) -----------------------

P31 = (1 << 31) + 11


def _fold31(x):
    y = ((x & M32) - (x >> 32) * 22) & M64
    y1 = (y >> 32) - (1 << 32) if (y >> 63) else (y >> 32)
    return (y & M32) + ((-22 * y1) & M32)


def _red31(x):
    z = _fold31(x)
    return z - 2 * P31 if z >= 2 * P31 else (z - P31 if z >= P31 else z)


def _mod31(u, M, C):
    m, u0 = (C * (u >> 32)) & M32, u & M32
    v = (u0 - m) & M32
    return (v - (M if v >= M else 0) + (C if u0 < m else 0)) & M32


def test_p31_fold_reduce_and_draws():
    """The paper-literal full-precision domain p = 2^31 + 11: fold31 is x mod p within
    [0, 2^32 + 176] and red31 the exact residue for every x < 2^63 (edges and 2e5 random);
    mod31 = u mod p and u mod (p - 1) for 48-bit draws; K31 = 2^-64 mod p (reading C28)."""
    rng = np.random.default_rng(31)
    xs = [0, 1, M32, 1 << 32, P31, P31 - 1, 2 * P31, 2 * P31 - 1, (1 << 63) - 1, P31 * P31 + P31 - 1,
          (1 << 31) * (P31 - 1) + P31 - 1] + [k * P31 + e for k in (1, 2, 3, 1 << 30, (1 << 31) + 9) for e in (0, 1, 21, 22)]
    xs += [int(v) for v in rng.integers(0, 1 << 63, size=200000, dtype=np.uint64)]
    for x in xs:
        z = _fold31(x)
        assert z % P31 == x % P31 and 0 <= z <= (1 << 32) + 176, x
        assert _red31(x) == x % P31, x
    us = [0, 1, (1 << 48) - 1, P31, P31 - 1, M32, 1 << 32] + [(k << 32) + e for k in (1, 2, 0xFFFF)
                                                              for e in (0, 19, 20, 21, 22, 23, 20 * k - 1, 22 * k - 1)]
    us += [int(v) for v in rng.integers(0, 1 << 48, size=200000, dtype=np.uint64)]
    for u in us:
        assert _mod31(u, P31, 22) == u % P31, u
        assert _mod31(u, P31 - 1, 20) == u % (P31 - 1), u
    assert pow(2, -64, P31) == 0x5E69C906


def test_p31_slot_zero_test():
    """The L31 slot: W0 = red31(c r + rho), W1 = fold31(d r + (p - rho)); P2's test
    t = s0 - 22 s1 in {0, p} on s = W0 + W1 is exactly (c + d) r = 0 (mod p); no operand
    product plus addend reaches 2^63."""
    rng = np.random.default_rng(32)
    cases = [(1 << 31, P31 - (1 << 31), P31 - 1, P31 - 1), (1, P31 - 1, P31 - 1, 0), (1 << 31, 11, 1, 5)]
    for _ in range(50000):
        c = int(rng.integers(1, (1 << 31) + 1))
        r = int(rng.integers(1, P31))
        rho = int(rng.integers(0, P31))
        d = (P31 - c) % P31 if rng.random() < 0.3 else int(rng.integers(11, P31))
        cases.append((c, d, r, rho))
    for c, d, r, rho in cases:
        x0, x1 = c * r + rho, d * r + (P31 - rho)
        assert x0 < 1 << 63 and x1 < 1 << 63
        s = _red31(x0) + _fold31(x1)
        assert s < 1 << 33
        t = (s & M32) - 22 * (s >> 32)
        assert (t in (0, P31)) == (((c + d) * r) % P31 == 0), (c, d, r, rho)
