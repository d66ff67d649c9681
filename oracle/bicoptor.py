"""UBL Bicoptor 2.0 DReLU (Alg 7) and ReLU (Alg 8) -- oracle; test infrastructure only.

Follows Alg 7 and Alg 8 step by step, per party,
vectorised over the element batch with numpy (elements are independent,
P:996).  Every random value is drawn from the pre-shared seeds with
the ChaCha keystream of ``oracle.chacha``; the byte layout of those draws is
the spec's own -- the paper fixes none (readings
C9-C11).  The tapes are pinned by re-reading their draws from an independent
keystream (OpenSSL's ChaCha20 via ``cryptography``) for the compact, pair and
large layouts, the permutation by a literal Fisher-Yates over all S! indices,
and every reconstructed output against plaintext sign / ReLU.

Notation: ell ring bits; lx key-bit width (ell_x); f window
offset of the key bits (sec. 6.1, reading C5); w = lx+1 ("guard", default,
reading C6) or lx ("literal", the paper's Z_{2^lx}); p = smallest prime
> 2^w (reading C7); S = lx+1 ladder slots.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import ring
from .chacha import chacha_blocks, element_u32, element_u64, label_u64

# Stream labels (domain separation of the seeds' keystreams).
L_TAPEA = label_u64(b"bc2.tpa1")  # seed01: 16 B/element (compact tape, part A)
L_TAPEB = label_u64(b"bc2.tpb1")  # seed01:  8 B/element (compact tape, part B)
L_TAPEP = label_u64(b"bc2.tpp1")   # seed01: 32 B/element (pair tape: p <= 131, 28-bit (r, rho) draws)
L_TAPEL = label_u64(b"bc2.tpL2")   # seed01: 448 B/element (large tape, lx >= 8; 48-bit draws)
L_FBL = label_u64(b"bc2.fbL2")     # seed01: large-tape fallback, u64 words, counter j*2^20+k
L_FALLBACK = label_u64(b"bc2.fb01")  # seed01: rejection fallback, counter j*256+k
L_RESP = label_u64(b"bc2.resp")    # seed02: [DReLU']_0, 8 B/element
L_A02 = label_u64(b"bc2.ta02")     # seed02: [a]_0, 8 B/element
L_B02 = label_u64(b"bc2.tb02")     # seed02: [b]_0, 8 B/element
L_C02 = label_u64(b"bc2.tc02")     # seed02: [c]_0, 8 B/element
L_A12 = label_u64(b"bc2.ta12")     # seed12: [a]_1, 8 B/element
L_B12 = label_u64(b"bc2.tb12")     # seed12: [b]_1, 8 B/element

PERM_LIMIT_COMPACT = 53261 * 40320  # largest multiple of 8! below 2^31
RHO_WORD_LIMIT = 253 * 257 ** 3     # largest multiple of 257^3 below 2^32


@dataclass(frozen=True)
class Params:
    ell: int = 64
    lx: int = 7
    f: int = 24
    mode: str = "guard"   # "guard": w = lx+1 (default); "literal": w = lx
    rounds: int = 20

    def __post_init__(self):
        if not (2 <= self.ell <= 64):
            raise ValueError("ell must be in [2, 64]")
        if not (2 <= self.lx <= 31):
            raise ValueError("lx must be in [2, 31] (at most 32 ladder slots, p < 2^33)")
        if self.mode not in ("guard", "literal"):
            raise ValueError("mode must be 'guard' or 'literal'")
        if self.f < 0 or self.f + self.lx + self.w > self.ell:
            raise ValueError("window does not fit: need f + lx + w <= ell")
        if self.rounds not in (8, 12, 20):
            raise ValueError("rounds must be 8, 12 or 20")

    @property
    def w(self) -> int:
        return self.lx + 1 if self.mode == "guard" else self.lx

    @property
    def p(self) -> int:
        return ring.prime_above(self.w)

    @property
    def slots(self) -> int:
        return self.lx + 1

    @property
    def compact(self) -> bool:
        """Compact 24-B tape iff p = 257 and 8 slots (masks are exact bytes)."""
        return self.p == 257 and self.slots == 8

    @property
    def layout(self) -> str:
        """PRG tape layout: "compact" (p = 257, 8 slots), "pair" (other lx <= 7, p <= 131),
        "compact_lit" (the pair tape's p = 131, 8-slot case: the paper-literal domain at
        lx = 7, which the kernels compile with constant parameters),
        "large" (lx >= 8: up to 32 slots, p < 2^33; full precision lx = 31)."""
        if self.compact:
            return "compact"
        if self.p == 131 and self.slots == 8:
            return "compact_lit"
        return "pair" if self.lx <= 7 else "large"


# --- PRG tape: t, Pi, r_m, rho_m for one element (Alg 7 steps 1, 6, 7, 8) -------------

def _fallback_words(seed01: bytes, j: int, rounds: int):
    """Sequential u32 words of ChaCha(seed01, L_FALLBACK, counter = j*256 + k)."""
    k = 0
    while True:
        blk = chacha_blocks(seed01, L_FALLBACK, [j * 256 + k], rounds)[0]
        for wd in blk:
            yield int(wd)
        k += 1


def _perm_swaps(idx, S: int):
    """Mixed-radix digits of idx in [0, S!): k_m = idx mod (m+1), idx //= (m+1),
    for m = S-1 .. 1.  Column m of the result is the Fisher-Yates swap partner
    of slot m (column 0 unused)."""
    idx = np.asarray(idx, dtype=np.uint64) % np.uint64(math.factorial(S))
    k = np.zeros(idx.shape + (S,), dtype=np.int64)
    for m in range(S - 1, 0, -1):
        k[..., m] = (idx % np.uint64(m + 1)).astype(np.int64)
        idx = idx // np.uint64(m + 1)
    return k


def tape(prm: Params, seed01: bytes, j) -> dict:
    """Decode the seed01 randomness of elements j.

    Alg 7 step 1: random bit t.  Step 6: permutation Pi as
    Fisher-Yates swaps (reading C9).  Step 7: masks r_m in Z_p^*.
    Step 8: reshare values rho_m in Z_p (reading C11).  Exact
    rejection sampling with a deterministic fallback stream (reading C10).
    The layout is the spec's; its draws are pinned by re-reads from an
    independent keystream (tests/test_oracle_drelu.py, test_oracle_fullprec.py).
    """
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    if prm.layout == "compact":
        return _tape_compact(prm, seed01, j)
    if prm.layout == "large":
        return _tape_large(prm, seed01, j)
    return _tape_pair(prm, seed01, j)  # "pair" and its p = 131, 8-slot case "compact_lit"


def _tape_compact(prm: Params, seed01: bytes, j) -> dict:
    """p = 257, 8 slots.  24 B per element from two regular streams:
    part A (16 B at 16 j): T0 = t (bit 31) | perm index (bits 0..30, reject >= 53261*8!),
                           T1, T2 = mask bytes, r_m = 1 + byte m (exactly uniform on Z_257^*),
                           T3 = reshare word 0;
    part B (8 B at 8 j):   T4, T5 = reshare words 1, 2.
    Reshare word k (reject >= 253 * 257^3) holds rho_{3k}, rho_{3k+1}, rho_{3k+2}
    as its base-257 digits, least significant first (rho_8 is unused)."""
    n, S = j.size, prm.slots
    A = element_u32(seed01, L_TAPEA, prm.rounds, j, 4)
    Bw = element_u32(seed01, L_TAPEB, prm.rounds, j, 2)
    t = (A[:, 0] >> np.uint32(31)).astype(np.uint64)
    idx = (A[:, 0] & np.uint32(0x7FFFFFFF)).astype(np.uint64)
    idx_ok = idx < np.uint64(PERM_LIMIT_COMPACT)
    r = np.ascontiguousarray(A[:, 1:3]).view(np.uint8).reshape(n, 8).astype(np.uint64) + np.uint64(1)
    words = np.stack([A[:, 3], Bw[:, 0], Bw[:, 1]], axis=1).astype(np.uint64)
    words_ok = words < np.uint64(RHO_WORD_LIMIT)
    for row in np.nonzero(~idx_ok | ~words_ok.all(axis=1))[0]:  # rare: fallback stream, in order
        fb = _fallback_words(seed01, int(j[row]), prm.rounds)
        if not idx_ok[row]:
            v = next(fb) & 0x7FFFFFFF
            while v >= PERM_LIMIT_COMPACT:
                v = next(fb) & 0x7FFFFFFF
            idx[row] = v
        for k in range(3):
            if not words_ok[row, k]:
                v = next(fb)
                while v >= RHO_WORD_LIMIT:
                    v = next(fb)
                words[row, k] = v
    P = np.uint64(257)
    digits = np.stack([(words // P ** np.uint64(i)) % P for i in range(3)], axis=2).reshape(n, 9)
    return {"t": t, "k": _perm_swaps(idx, S), "r": r, "rho": digits[:, :8].copy()}


def _tape_pair(prm: Params, seed01: bytes, j) -> dict:
    """Any p <= 131 with 3..8 slots (every lx <= 7 domain but the compact one; at
    lx = 7 literal, p = 131 and 8 slots).  32 B per element at 32 j (label bc2.tpp1,
    two elements per ChaCha block):
    T0 = t (bit 31) | perm index (bits 0..30, reject >= floor(2^31/S!) S!);
    T1..T7 = 224 bits, read as one little-endian integer D, holding up to eight
    28-bit draws u_m = (D >> 28 m) & (2^28 - 1), one per slot m < S.  A draw is a
    pair in Z_{p-1} x Z_p: with d = (p-1) p, reject u >= floor(2^28/d) d, else
    x = u mod d, the mask r_m = 1 + x mod (p-1) and the reshare rho_m = x div (p-1)
    (the pair (x mod (p-1), x div (p-1)) is uniform on Z_{p-1} x Z_p).  A rejected
    draw takes the next word of the fallback stream (its low 31 bits for the index,
    low 28 bits for a draw), in the order index, slots 0..S-1 (reading C10)."""
    n, S, p = j.size, prm.slots, prm.p
    fact = math.factorial(S)
    perm_lim = ((1 << 31) // fact) * fact
    T = element_u32(seed01, L_TAPEP, prm.rounds, j, 8).astype(np.uint64)
    t = T[:, 0] >> np.uint64(31)
    idx = T[:, 0] & np.uint64(0x7FFFFFFF)
    idx_ok = idx < np.uint64(perm_lim)
    D = [sum(int(T[i, w]) << (32 * (w - 1)) for w in range(1, 8)) for i in range(n)]
    u = np.array([[(d >> (28 * m)) & 0xFFFFFFF for m in range(S)] for d in D], dtype=np.uint64).reshape(n, S)
    pair = (p - 1) * p
    lim = ((1 << 28) // pair) * pair
    ok = u < np.uint64(lim)
    x = u % np.uint64(pair)
    for row in np.nonzero(~idx_ok | ~ok.all(axis=1))[0]:
        fb = _fallback_words(seed01, int(j[row]), prm.rounds)
        if not idx_ok[row]:
            v = next(fb) & 0x7FFFFFFF
            while v >= perm_lim:
                v = next(fb) & 0x7FFFFFFF
            idx[row] = v
        for m in range(S):
            if not ok[row, m]:
                v = next(fb) & 0xFFFFFFF
                while v >= lim:
                    v = next(fb) & 0xFFFFFFF
                x[row, m] = v % pair
    r = np.uint64(1) + x % np.uint64(p - 1)
    rho = x // np.uint64(p - 1)
    return {"t": t, "k": _perm_swaps(idx, S), "r": r, "rho": rho}


def _fallback_u64(seed01: bytes, j: int, rounds: int):
    """Sequential u64 words of ChaCha(seed01, L_FBL, counter = j*2^20 + k)."""
    k = 0
    while True:
        blk = chacha_blocks(seed01, L_FBL, [(j << 20) + k], rounds)[0]
        for i in range(8):
            yield int(blk[2 * i]) | (int(blk[2 * i + 1]) << 32)
        k += 1


def _tape_large(prm: Params, seed01: bytes, j) -> dict:
    """lx >= 8 (up to 32 slots, p < 2^33; the full-precision lx = 31 regime,
    P:195).  448 B = 7 ChaCha blocks per element at 448 j (label bc2.tpL2):
      block 0:    32 u16 h; t = h[0] & 1; the Fisher-Yates draw of slot m
                  (m = S-1 .. 1) is h[S-m]: k_m = h mod (m+1), reject h >= floor(2^16/(m+1))(m+1);
      blocks 1-6: 48-bit little-endian draws in groups of 8 slots, 96 B per group g = m div 8:
                  the mask draw u of slot m at byte 96 g + 6 (m mod 8), its reshare draw at
                  96 g + 48 + 6 (m mod 8) (bytes counted from the start of block 1);
                  r_m = (1 + u mod (p-1)) * 2^-64 mod p, reject u >= floor(2^48/(p-1))(p-1) --
                  multiplying by the unit 2^-64 is a bijection of Z_p^*, so r_m is still uniform
                  on Z_p^* (the draw is the mask's Montgomery form, which is what a Montgomery
                  multiplier consumes); rho_m = u mod p, reject u >= floor(2^48/p) p.
    48 bits carry a 33-bit value with a rejection probability below 2^-15 per draw; the
    tape is 7 blocks instead of the 9 that 64-bit draws take (reading C28).
    Slots m >= S leave their draws unused.  A rejected draw -- in the order
    k_{S-1} .. k_1, then r_0, rho_0, r_1, rho_1, .., r_{S-1}, rho_{S-1} -- is replaced by the next
    u64 of the fallback stream (its low 16 bits for a Fisher-Yates draw, its low 48 bits for a
    mask or reshare draw), repeated until accepted (reading C10).  Returns r, rho as Python-int
    object arrays."""
    n, S, p = j.size, prm.slots, prm.p
    T = element_u32(seed01, L_TAPEL, prm.rounds, j, 112)
    h = np.ascontiguousarray(T[:, :16]).view("<u2").reshape(n, 32).astype(np.int64)
    D = np.ascontiguousarray(T[:, 16:]).view(np.uint8).reshape(n, 384)

    def draw48(off):  # (n,) little-endian 48-bit values at byte offset off
        v = np.zeros(n, dtype=np.uint64)
        for b in range(6):
            v |= D[:, off + b].astype(np.uint64) << np.uint64(8 * b)
        return v

    U = np.stack([draw48(96 * (m // 8) + 6 * (m % 8)) for m in range(32)]
                 + [draw48(96 * (m // 8) + 48 + 6 * (m % 8)) for m in range(32)], axis=1)
    t = (h[:, 0] & 1).astype(np.uint64)
    k = np.zeros((n, S), dtype=np.int64)
    hlim = {m: (65536 // (m + 1)) * (m + 1) for m in range(1, S)}
    rlim, plim = ((1 << 48) // (p - 1)) * (p - 1), ((1 << 48) // p) * p  # 2^48 when q | 2^48: no rejection
    m48 = (1 << 48) - 1
    rinv = pow(2, -64, p)                                                 # 2^-64 mod p
    r = np.empty((n, S), dtype=object)
    rho = np.empty((n, S), dtype=object)
    for row in range(n):
        fb = None
        for m in range(S - 1, 0, -1):
            d = int(h[row, S - m])
            while d >= hlim[m]:
                fb = fb or _fallback_u64(seed01, int(j[row]), prm.rounds)
                d = next(fb) & 0xFFFF
            k[row, m] = d % (m + 1)
        for m in range(S):
            u = int(U[row, m])
            while u >= rlim:
                fb = fb or _fallback_u64(seed01, int(j[row]), prm.rounds)
                u = next(fb) & m48
            r[row, m] = (1 + u % (p - 1)) * rinv % p
            u = int(U[row, 32 + m])
            while u >= plim:
                fb = fb or _fallback_u64(seed01, int(j[row]), prm.rounds)
                u = next(fb) & m48
            rho[row, m] = u % p
    return {"t": t, "k": k, "r": r, "rho": rho}


# --- Alg 7 steps 3-5: ladder, pairwise sums, modulo switch --------------------------

def ladder(prm: Params, party: int, s) -> np.ndarray:
    """Alg 7 step 3 with the key-bit offset f (reading C5):
    u_i := trc(s, f+i, ell-w-f-i) mod 2^w for i in [0, lx]  (Alg 5).  (n, S)."""
    s = np.atleast_1d(np.asarray(s, dtype=np.uint64))
    cols = [ring.trc_det_mid(party, s, prm.f + i, prm.ell - prm.w - prm.f - i, prm.ell)
            for i in range(prm.lx + 1)]
    return np.stack(cols, axis=1).astype(np.uint64)


def pairwise(prm: Params, party: int, u) -> np.ndarray:
    """Alg 7 step 4: v_i := u_i + u_{i+1} - 1 (i < lx), v_lx := u_lx - 1,
    all mod 2^w.  The public constant -1 is added by P0 only (reading C8)."""
    one = np.uint64(1 if party == 0 else 0)
    wm = np.uint64(ring.mask(prm.w))
    v = np.empty_like(u)
    with np.errstate(over="ignore"):
        v[:, :-1] = (u[:, :-1] + u[:, 1:] - one) & wm
        v[:, -1] = (u[:, -1] - one) & wm
    return v


def ladder_modswitch(prm: Params, party: int, s) -> np.ndarray:
    """Alg 7 steps 3-5 on a share as given (no blinding): v'_i in Z_p^*, (n, S)."""
    v = pairwise(prm, party, ladder(prm, party, s))
    return ring.modswitch(party, v, prm.w, prm.p)


def ladder_modswitch_bytes(prm: Params, party: int, s) -> np.ndarray:
    """Output format of bc_ladder_modswitch: byte m = v'_m - 1 (v' is never 0,
    see Alg 6), bytes S..7 zero.  (n, 8) uint8."""
    if prm.slots > 8:
        raise ValueError("the byte format holds at most 8 slots (lx <= 7)")
    vp = ladder_modswitch(prm, party, s)
    out = np.zeros((vp.shape[0], 8), dtype=np.uint8)
    out[:, : prm.slots] = (vp - np.uint64(1)).astype(np.uint8)
    return out


# --- Alg 7 per party ---------------------------------------------------------------

def shuffle(k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Alg 7 step 6: Fisher-Yates, for m = S-1 .. 1 swap(v[m], v[k_m])
    (reading C9; both parties use the same seed01-derived k)."""
    v = v.copy()
    rows = np.arange(v.shape[0])
    for m in range(v.shape[1] - 1, 0, -1):
        km = k[:, m]
        a = v[rows, m].copy()
        v[rows, m] = v[rows, km]
        v[rows, km] = a
    return v


def drelu_send(prm: Params, party: int, xb, j, seed01: bytes) -> dict:
    """Alg 7 steps 1-8 for party P0 (party=0) or P1 (party=1).

    1  t from seed01;                      2  s := (-1)^t [x]_b mod 2^ell
    3  ladder u_i (Alg 5);                 4  pairwise v_i
    5  modulo switch (Alg 6);              6  shuffle with Pi
    7  w_m := v_m * r_m mod p;             8  reshare: P0 sends w + rho, P1 sends w - rho
    Returns {"t", "W"} with W the (n, S) message to P2 in Z_p.
    """
    xb = np.atleast_1d(np.asarray(xb, dtype=np.uint64))
    tp = tape(prm, seed01, j)
    t = tp["t"]
    s = np.where(t == 1, ring.neg(xb, prm.ell), xb).astype(np.uint64)       # steps 1-2
    vp = ladder_modswitch(prm, party, s)                                      # steps 3-5
    vp = shuffle(tp["k"], vp)                                                 # step 6
    if prm.layout == "large":                                                 # p up to 2^33: exact ints
        P = prm.p
        wv = (vp.astype(object) * tp["r"]) % P                                # step 7
        W = (wv + tp["rho"]) % P if party == 0 else (wv + P - tp["rho"]) % P  # step 8
        return {"t": t, "W": W.astype(np.uint64)}
    P = np.uint64(prm.p)
    wv = (vp * tp["r"]) % P                                                   # step 7
    if party == 0:                                                            # step 8
        W = (wv + tp["rho"]) % P
    else:
        W = (wv + P - tp["rho"]) % P
    return {"t": t, "W": W}


def zero_test(prm: Params, W0, W1) -> np.ndarray:
    """Alg 7 step 9: P2 reconstructs w_m = W0_m + W1_m mod p and
    sets DReLU' := 1 iff some w_m = 0."""
    wsum = (np.asarray(W0, dtype=np.uint64) + np.asarray(W1, dtype=np.uint64)) % np.uint64(prm.p)
    return (wsum == 0).any(axis=1).astype(np.uint64)


def drelu_helper(prm: Params, W0, W1, j, seed02: bytes) -> dict:
    """Alg 7 steps 9-10: zero test, then reshare DReLU' in Z_{2^ell}:
    [D']_0 := seed02 stream value q, [D']_1 := DReLU' - q (reading C12)."""
    z = zero_test(prm, W0, W1)
    q = element_u64(seed02, L_RESP, prm.rounds, j, 1)[:, 0] & np.uint64(ring.mask(prm.ell))
    return {"z": z, "D0": q, "D1": ring.sub(z, q, prm.ell)}


def drelu_finish(prm: Params, party: int, t, Db) -> np.ndarray:
    """Alg 7 step 11: [DReLU] = t + (1-2t)[DReLU'] mod 2^ell; the
    public t is added by P0 only (reading C8)."""
    t = np.asarray(t, dtype=np.uint64)
    Db = np.asarray(Db, dtype=np.uint64)
    signed = np.where(t == 1, ring.neg(Db, prm.ell), Db).astype(np.uint64)
    if party == 0:
        return ring.add(signed, t, prm.ell)
    return signed


def drelu(prm: Params, x0, x1, j, seeds) -> dict:
    """Alg 7 end to end with all three parties (two rounds)."""
    m0 = drelu_send(prm, 0, x0, j, seeds.s01)
    m1 = drelu_send(prm, 1, x1, j, seeds.s01)
    h = drelu_helper(prm, m0["W"], m1["W"], j, seeds.s02)
    y0 = drelu_finish(prm, 0, m0["t"], h["D0"])
    y1 = drelu_finish(prm, 1, m1["t"], h["D1"])
    return {"y0": y0, "y1": y1, "t": m0["t"], "W0": m0["W"], "W1": m1["W"], **h}


# --- Alg 8: ReLU -------------------------------------------------------------------

def triple(prm: Params, j, seed02: bytes, seed12: bytes) -> dict:
    """Alg 8 preprocessing: P0,P2 draw [a]_0,[b]_0,[c]_0 from seed02;
    P1,P2 draw [a]_1,[b]_1 from seed12; P2 sets [c]_1 := (a0+a1)(b0+b1) - c0."""
    L = prm.ell
    m = np.uint64(ring.mask(L))
    a0, b0, c0 = (element_u64(seed02, lab, prm.rounds, j, 1)[:, 0] & m for lab in (L_A02, L_B02, L_C02))
    a1, b1 = (element_u64(seed12, lab, prm.rounds, j, 1)[:, 0] & m for lab in (L_A12, L_B12))
    c1 = ring.sub(ring.mul(ring.add(a0, a1, L), ring.add(b0, b1, L), L), c0, L)
    return {"a0": a0, "b0": b0, "c0": c0, "a1": a1, "b1": b1, "c1": c1}


def relu_send(prm: Params, party: int, xb, j, seed01: bytes, seed_tr: bytes) -> dict:
    """Alg 8 steps 1 and 4 for P0 / P1: the Alg 7 message to P2
    and the party's share of d = x - a, [d]_b = [x]_b - [a]_b, sent to the other
    computing party.  seed_tr is seed02 (P0, [a]_0) or seed12 (P1, [a]_1)."""
    m = drelu_send(prm, party, xb, j, seed01)
    lab = L_A02 if party == 0 else L_A12
    a = element_u64(seed_tr, lab, prm.rounds, j, 1)[:, 0] & np.uint64(ring.mask(prm.ell))
    return {"t": m["t"], "W": m["W"], "d": ring.sub(np.asarray(xb, dtype=np.uint64), a, prm.ell)}


def relu_helper(prm: Params, W0, W1, j, seed02: bytes, seed12: bytes) -> dict:
    """Alg 8 steps 2-3 for P2: DReLU' by the zero test, then
    e := DReLU' - b (b = [b]_0 + [b]_1) to P0 and P1, and [c]_1 to P1."""
    z = zero_test(prm, W0, W1)
    tr = triple(prm, j, seed02, seed12)
    e = ring.sub(z, ring.add(tr["b0"], tr["b1"], prm.ell), prm.ell)
    return {"z": z, "e": e, "c1": tr["c1"]}


def relu_finish(prm: Params, party: int, xb, t, d_own, d_peer, e, c1, j, seed_tr: bytes) -> np.ndarray:
    """Alg 8 steps 4-5 for P0 / P1:
    d := [d]_0 + [d]_1 (opened);
    [ReLU]_b = t [x]_b + (1-2t)(de + d[b]_b + e[a]_b + [c]_b), de added by P0 only
    (reading C8).  P0 regenerates [a]_0,[b]_0,[c]_0 from seed02, P1 regenerates
    [a]_1,[b]_1 from seed12 and uses the received [c]_1."""
    L = prm.ell
    m = np.uint64(ring.mask(L))
    xb = np.asarray(xb, dtype=np.uint64)
    t = np.asarray(t, dtype=np.uint64)
    d = ring.add(d_own, d_peer, L)
    if party == 0:
        a, b, c = (element_u64(seed_tr, lab, prm.rounds, j, 1)[:, 0] & m for lab in (L_A02, L_B02, L_C02))
        inner = ring.add(ring.add(ring.mul(d, e, L), ring.mul(d, b, L), L), ring.add(ring.mul(e, a, L), c, L), L)
    else:
        a, b = (element_u64(seed_tr, lab, prm.rounds, j, 1)[:, 0] & m for lab in (L_A12, L_B12))
        inner = ring.add(ring.add(ring.mul(d, b, L), ring.mul(e, a, L), L), np.asarray(c1, dtype=np.uint64), L)
    signed = np.where(t == 1, ring.neg(inner, L), inner).astype(np.uint64)
    return ring.add(ring.mul(t, xb, L), signed, L)


def relu(prm: Params, x0, x1, j, seeds) -> dict:
    """Alg 8, all three parties.

    1  P0, P1 run Alg 7 steps 1-8 and send [w] to P2
    2  P2 reconstructs w, DReLU' := 1 iff some w_m = 0
    3  P2 sends e := DReLU' - b to P0 and P1, and [c]_1 to P1
    4  P0, P1 open d := x - a
    5  [ReLU] = t[x] + (1-2t)(de + d[b] + e[a] + [c]) mod 2^ell
    """
    x0 = np.atleast_1d(np.asarray(x0, dtype=np.uint64))
    x1 = np.atleast_1d(np.asarray(x1, dtype=np.uint64))
    m0 = relu_send(prm, 0, x0, j, seeds.s01, seeds.s02)
    m1 = relu_send(prm, 1, x1, j, seeds.s01, seeds.s12)
    h = relu_helper(prm, m0["W"], m1["W"], j, seeds.s02, seeds.s12)
    y0 = relu_finish(prm, 0, x0, m0["t"], m0["d"], m1["d"], h["e"], None, j, seeds.s02)
    y1 = relu_finish(prm, 1, x1, m1["t"], m1["d"], m0["d"], h["e"], h["c1"], j, seeds.s12)
    return {"y0": y0, "y1": y1, "t": m0["t"], "W0": m0["W"], "W1": m1["W"], "z": h["z"],
            "e": h["e"], "c1": h["c1"], "d0": m0["d"], "d1": m1["d"]}


# --- wire format of the P0/P1 -> P2 message (Alg 7 step 8) ---------------------------

def encode_msg(W: np.ndarray):
    """Slot m of W (values < p <= 257) -> low byte plane (n, 8) and a high-bit
    plane (n,) with bit m = bit 8 of W_m.  (ell_x+1) * ceil(log2 p) bits per
    element on the wire: 72 (guard, p=257) / 64 (literal, p=131)."""
    W = np.asarray(W, dtype=np.uint64)
    n, S = W.shape
    if S > 8:
        raise ValueError("the byte wire format holds at most 8 slots (lx <= 7)")
    lo = np.zeros((n, 8), dtype=np.uint8)
    lo[:, :S] = (W & np.uint64(0xFF)).astype(np.uint8)
    hi = np.zeros(n, dtype=np.uint8)
    for m in range(S):
        hi |= ((W[:, m] >> np.uint64(8)) & np.uint64(1)).astype(np.uint8) << np.uint8(m)
    return lo, hi


def encode_msg_large(W: np.ndarray):
    """Large-tape wire format (lx >= 8, up to 32 slots, p < 2^33):
    slot-major low-word plane (S, n) of uint32, row m = W_m mod 2^32 of every
    element, and a high-bit plane (n,) of uint32 with bit m = bit 32 of W_m.
    33 S bits per element: 1,056 at the paper's full precision lx = 31
    ("31 * 31 ~ 1,000 bits")."""
    W = np.asarray(W, dtype=np.uint64)
    n, S = W.shape
    lo = np.ascontiguousarray((W & np.uint64(0xFFFFFFFF)).astype(np.uint32).T)
    hi = np.zeros(n, dtype=np.uint32)
    for m in range(S):
        hi |= ((W[:, m] >> np.uint64(32)) & np.uint64(1)).astype(np.uint32) << np.uint32(m)
    return lo, hi


def reconstruct(y0, y1, ell: int):
    return ring.add(np.asarray(y0, dtype=np.uint64), np.asarray(y1, dtype=np.uint64), ell)
