"""Truncation study -- oracle; test infrastructure only.

Prior-work probabilistic truncation and the e1 analysis (sec. 3-4):
Alg 1 (SecureML; in ``oracle.ring.trc_secureml``), Alg 2 (ABY3,
P:329-342), the error classes of Theorem thm:smltrc / Corollary clr:cut2
(P:320-328); the deterministic Alg 4 for comparison;
and Alg 3 "truncate-then-multiply" against "multiply-then-truncate"
(sec. 5.2), two-party, with a Beaver multiplication.

Readings:
  C29  Alg 2 step 2 "P_i sets alpha/2^k - [r']": the public alpha/2^k = cut(alpha, k)
       is added by P0 only (as C8); step 1 uses [x]_i + [r]_i (the paper's footnote,
       P:341); r and r' = cut(r, k) are preprocessed by P2 as a dealer: [r]_0 and
       [r']_0 from seed02, [r]_1 from seed12, [r']_1 = cut(r, k) - [r']_0 sent to P1.
       Truncation instance q in {0, 1} (Alg 3 truncates two operands) uses labels
       bc2.t<q>r0, bc2.t<q>r1, bc2.t<q>q0.
  C30  error classes of a reconstructed truncation y of a band input x (xi = |x|):
       positive x: y = cut(xi, k) + bit, negative x: y = -cut(xi, k) - bit (thm:smltrc);
       "exact" bit = 0, "e0" bit = 1, "e1" anything else (the LT(.) cut(2^ell, k) term).
       Alg 4 outputs live in Z_{2^(ell-k)} and are classified there.
  C31  Alg 3 with an odd fractional precision f truncates floor(f/2) bits of x and
       ceil(f/2) of y; the Beaver triple is the one of Alg 8 (C24) under the
       labels bc2.ma02, bc2.mb02, bc2.mc02 (seed02), bc2.ma12, bc2.mb12 (seed12).
"""
from __future__ import annotations

import numpy as np

from . import ring
from .chacha import element_u64, label_u64

EXACT, E0, E1 = 0, 1, 2

L_MA02, L_MB02, L_MC02 = (label_u64(s) for s in (b"bc2.ma02", b"bc2.mb02", b"bc2.mc02"))
L_MA12, L_MB12 = (label_u64(s) for s in (b"bc2.ma12", b"bc2.mb12"))


def _lab(q: int, kind: str) -> int:
    return label_u64(f"bc2.t{q}{kind}".encode())


def _u64(seed, lab, j, rounds, ell):
    return element_u64(seed, lab, rounds, j, 1)[:, 0] & np.uint64(ring.mask(ell))


# --- Alg 2: ABY3 truncation ---------------------------------------------------------

def aby3_pre(ell: int, k: int, j, seeds, rounds: int = 20, q: int = 0) -> dict:
    """Alg 2 preprocessing (reading C29): shares of r and of r' := r / 2^k = cut(r, k)."""
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    r0 = _u64(seeds.s02, _lab(q, "r0"), j, rounds, ell)
    r1 = _u64(seeds.s12, _lab(q, "r1"), j, rounds, ell)
    r = ring.add(r0, r1, ell)
    rp0 = _u64(seeds.s02, _lab(q, "q0"), j, rounds, ell)
    rp1 = ring.sub(ring.cut(r, k), rp0, ell)
    return {"r0": r0, "r1": r1, "rp0": rp0, "rp1": rp1}


def trc_aby3(x0, x1, pre: dict, k: int, ell: int):
    """Alg 2: 1. each party publishes [x]_i + [r]_i, all reconstruct
    alpha = x + r mod 2^ell; 2. [trc(x, k)]_i := alpha / 2^k - [r']_i, the public
    alpha / 2^k = cut(alpha, k) added by P0 only (reading C29)."""
    x0 = np.asarray(x0, dtype=np.uint64)
    x1 = np.asarray(x1, dtype=np.uint64)
    alpha = ring.add(ring.add(x0, pre["r0"], ell), ring.add(x1, pre["r1"], ell), ell)
    y0 = ring.sub(ring.cut(alpha, k), pre["rp0"], ell)
    y1 = ring.neg(pre["rp1"], ell)
    return y0, y1


def trc_secureml_pair(x0, x1, k: int, ell: int):
    """Alg 1 for both parties."""
    return ring.trc_secureml(0, x0, k, ell), ring.trc_secureml(1, x1, k, ell)


# --- error classes (reading C30) ------------------------------------------------------

def classify(x, y, k: int, ell: int, out_bits: int | None = None) -> np.ndarray:
    """Class of the reconstructed truncation y of band input x (thm:smltrc,
    clr:cut2): EXACT, E0 (the one-bit error) or E1 (the cut(2^ell, k) error).
    out_bits = ell for Alg 1 / 2, ell - k for Alg 4."""
    out_bits = ell if out_bits is None else out_bits
    x = np.atleast_1d(np.asarray(x, dtype=np.uint64))
    y = np.atleast_1d(np.asarray(y, dtype=np.uint64))
    pos = x < np.uint64(1 << (ell - 1))
    xi = np.where(pos, x, ring.neg(x, ell)).astype(np.uint64)
    cx = ring.cut(xi, k) & np.uint64(ring.mask(out_bits))
    T = np.where(pos, cx, ring.neg(cx, out_bits)).astype(np.uint64)
    d = ring.sub(y, T, out_bits)
    one = np.where(pos, np.uint64(1), np.uint64(ring.mask(out_bits)))
    return np.where(d == 0, EXACT, np.where(d == one, E0, E1)).astype(np.int64)


def count_masks(alg: str, x: int, k: int, ell: int) -> np.ndarray:
    """Brute force over every mask m in Z_{2^ell} (small ell): counts of
    (EXACT, E0, E1) for one band input x.
      "secureml": Alg 1 on [x]_0 = x + m, [x]_1 = -m;
      "aby3":     Alg 2 with r = m (y = cut(x + m, k) - cut(m, k));
      "det":      Alg 4 on [x]_0 = x + m, [x]_1 = -m, in Z_{2^(ell-k)}."""
    m = np.arange(1 << ell, dtype=np.uint64)
    xv = np.full(m.shape, x, dtype=np.uint64)
    x0, x1 = ring.add(xv, m, ell), ring.neg(m, ell)
    if alg == "secureml":
        y0, y1 = trc_secureml_pair(x0, x1, k, ell)
        y, ob = ring.add(y0, y1, ell), ell
    elif alg == "aby3":
        zero = np.zeros_like(m)
        pre = {"r0": m, "r1": zero, "rp0": ring.cut(m, k), "rp1": zero}
        y0, y1 = trc_aby3(xv, zero, pre, k, ell)
        y, ob = ring.add(y0, y1, ell), ell
    elif alg == "det":
        ob = ell - k
        y = ring.add(ring.trc_det(0, x0, k, ell), ring.trc_det(1, x1, k, ell), ob)
    else:
        raise ValueError(alg)
    return np.bincount(classify(xv, y, k, ell, ob), minlength=3)


# --- Alg 3: truncate-then-multiply vs multiply-then-truncate --------------------------

def triple(ell: int, j, seeds, rounds: int = 20) -> dict:
    """Beaver triple from the seeds (reading C31; the construction of Alg 8, C24)."""
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    a0, b0, c0 = (_u64(seeds.s02, lab, j, rounds, ell) for lab in (L_MA02, L_MB02, L_MC02))
    a1, b1 = (_u64(seeds.s12, lab, j, rounds, ell) for lab in (L_MA12, L_MB12))
    c1 = ring.sub(ring.mul(ring.add(a0, a1, ell), ring.add(b0, b1, ell), ell), c0, ell)
    return {"a0": a0, "b0": b0, "c0": c0, "a1": a1, "b1": b1, "c1": c1}


def mul_beaver(x0, x1, y0, y1, tr: dict, ell: int):
    """Two-party Beaver product: open d = x - a, e = y - b;
    [z]_0 = de + d[b]_0 + e[a]_0 + [c]_0, [z]_1 = d[b]_1 + e[a]_1 + [c]_1."""
    L = ell
    d = ring.add(ring.sub(x0, tr["a0"], L), ring.sub(x1, tr["a1"], L), L)
    e = ring.add(ring.sub(y0, tr["b0"], L), ring.sub(y1, tr["b1"], L), L)
    z0 = ring.add(ring.add(ring.mul(d, e, L), ring.mul(d, tr["b0"], L), L),
                  ring.add(ring.mul(e, tr["a0"], L), tr["c0"], L), L)
    z1 = ring.add(ring.add(ring.mul(d, tr["b1"], L), ring.mul(e, tr["a1"], L), L), tr["c1"], L)
    return z0, z1


def _trc(alg: str, z0, z1, k: int, ell: int, j, seeds, rounds: int, q: int):
    if alg == "secureml":
        return trc_secureml_pair(z0, z1, k, ell)
    if alg == "aby3":
        return trc_aby3(z0, z1, aby3_pre(ell, k, j, seeds, rounds, q), k, ell)
    raise ValueError(alg)


def mul_then_trc(alg: str, x0, x1, y0, y1, f: int, ell: int, j, seeds, rounds: int = 20):
    """The usual linear-layer order: z = x y (Beaver), then trc(z, f)."""
    z0, z1 = mul_beaver(x0, x1, y0, y1, triple(ell, j, seeds, rounds), ell)
    return _trc(alg, z0, z1, f, ell, j, seeds, rounds, 0)


def trc_then_mul(alg: str, x0, x1, y0, y1, f: int, ell: int, j, seeds, rounds: int = 20):
    """Alg 3: trc(x, floor(f/2)) and trc(y, ceil(f/2)) (reading C31),
    then the Beaver product of the truncated values."""
    kx, ky = f // 2, f - f // 2
    tx0, tx1 = _trc(alg, x0, x1, kx, ell, j, seeds, rounds, 0)
    ty0, ty1 = _trc(alg, y0, y1, ky, ell, j, seeds, rounds, 1)
    return mul_beaver(tx0, tx1, ty0, ty1, triple(ell, j, seeds, rounds), ell)


def signed(v, ell: int) -> np.ndarray:
    """Two's-complement value of v in Z_{2^ell} as Python ints (object array)."""
    v = np.atleast_1d(np.asarray(v, dtype=np.uint64)).astype(object)
    return np.where(v >= (1 << (ell - 1)), v - (1 << ell), v)
