"""Ring primitives, truncation and modulo switch (oracle; test infrastructure only).

All functions accept Python ints or numpy uint64 arrays holding elements of
Z_{2^ell} (values < 2^ell, ell <= 64) and return the same kind.

Readings of the paper used here:
  C1  cut(a, k) is the right shift floor(a / 2^k) (P:297 writes the unshifted
      sum, but the worked examples P:50-51 and cut(2^ell, k) = 2^(ell-k), P:707,
      shift).
  C2  cut(a, k1, k2) drops the k1 LOW bits and the k2 HIGH bits: bits
      [k1, ell-k2) (definition P:299-300 and example P:745-751; the Alg 5
      header P:733 swaps the words "first"/"last").
  C3  P1's operand 2^ell - [x]_1 is taken as (-[x]_1) mod 2^ell = R, the
      substitution the paper's own analysis makes (Corollary clr:cut2,
      P:367-375).  For Alg 4/5 this is identical to the integer reading
      because cut(2^ell, k1, k2) = 0 mod 2^(ell-k1-k2); for Alg 1 it fixes the
      R = 0 edge case (e1 then hits negative x, so the exact e1 count is xi
      masks for either sign; reading C18).
  C4  "2^ell - cut(...) mod 2^ell'" is -cut(...) mod 2^ell'.
"""
from __future__ import annotations

import numpy as np


def _is_arr(a) -> bool:
    return isinstance(a, np.ndarray)


def mask(bits: int) -> int:
    """2^bits - 1 as a Python int (bits <= 64)."""
    return (1 << bits) - 1


def _u(v, like):
    """Cast a Python int constant to the operand's kind."""
    return np.uint64(v) if _is_arr(like) else v


def neg(a, ell: int):
    """-a mod 2^ell."""
    if _is_arr(a):
        return (np.uint64(0) - a.astype(np.uint64)) & np.uint64(mask(ell))
    if isinstance(a, np.integer):  # exact in Python ints, back to the operand's kind
        return np.uint64((-int(a)) & mask(ell))
    return (-a) & mask(ell)


def add(a, b, ell: int):
    if _is_arr(a) or _is_arr(b):
        with np.errstate(over="ignore"):
            return (np.asarray(a, dtype=np.uint64) + np.asarray(b, dtype=np.uint64)) & np.uint64(mask(ell))
    return (a + b) & mask(ell)


def sub(a, b, ell: int):
    if _is_arr(a) or _is_arr(b):
        with np.errstate(over="ignore"):
            return (np.asarray(a, dtype=np.uint64) - np.asarray(b, dtype=np.uint64)) & np.uint64(mask(ell))
    return (a - b) & mask(ell)


def mul(a, b, ell: int):
    if _is_arr(a) or _is_arr(b):
        with np.errstate(over="ignore"):
            return (np.asarray(a, dtype=np.uint64) * np.asarray(b, dtype=np.uint64)) & np.uint64(mask(ell))
    return (a * b) & mask(ell)


def cut(a, k: int):
    """cut(alpha, k): cut the last k bits of alpha (reading C1)."""
    return a >> _u(k, a)


def cut_mid(a, k1: int, k2: int, ell: int):
    """cut(alpha, k1, k2): cut the last k1 and the first k2 bits, i.e. bits
    [k1, ell-k2) of alpha as an (ell-k1-k2)-bit value (reading C2)."""
    assert 0 <= k1 and 0 <= k2 and k1 + k2 <= ell
    return (a >> _u(k1, a)) & _u(mask(ell - k1 - k2), a)


def LT(a, b):
    """LT(alpha, beta) := 1 iff alpha < beta."""
    if _is_arr(a) or _is_arr(b):
        return (np.asarray(a) < np.asarray(b)).astype(np.uint64)
    return int(a < b)


# --- Alg 1: SecureML probabilistic truncation ---------------------------

def trc_secureml(party: int, xb, k: int, ell: int):
    """Alg 1: P0: cut([x]_0, k) mod 2^ell;
    P1: 2^ell - cut(2^ell - [x]_1, k) mod 2^ell."""
    if party == 0:
        return cut(xb, k) & _u(mask(ell), xb)
    return neg(cut(neg(xb, ell), k), ell)


# --- Alg 4 / Alg 5: deterministic truncation ---------------------------

def trc_det(party: int, xb, k: int, ell: int):
    """Alg 4: result share in Z_{2^(ell-k)}.
    P0: cut([x]_0, k) mod 2^(ell-k);  P1: 2^ell - cut(2^ell - [x]_1, k) mod 2^(ell-k)."""
    return trc_det_mid(party, xb, k, 0, ell)


def trc_det_mid(party: int, xb, k1: int, k2: int, ell: int):
    """Alg 5: result share in Z_{2^(ell-k1-k2)}.
    P0: cut([x]_0, k1, k2) mod 2^(ell-k1-k2);
    P1: 2^ell - cut(2^ell - [x]_1, k1, k2) mod 2^(ell-k1-k2)   (readings C3, C4)."""
    lp = ell - k1 - k2
    if party == 0:
        return cut_mid(xb, k1, k2, ell)
    return neg(cut_mid(neg(xb, ell), k1, k2, ell), lp)


# --- Alg 6: modulo switch ------------------------------------------------

def modswitch(party: int, xb, lp: int, p: int):
    """Alg 6: shares of x in Z_{2^lp} -> shares of x in Z_p.
    P0: [x]_0 := 2^lp mod p if [x]_0 = 0, else [x]_0 mod p.
    P1: [x]_1 := p + [x]_1 - 2^lp mod p."""
    if party == 0:
        if _is_arr(xb):
            return np.where(xb == 0, np.uint64((1 << lp) % p), xb % np.uint64(p)).astype(np.uint64)
        return (1 << lp) % p if xb == 0 else xb % p
    if _is_arr(xb):
        return (np.uint64(p) + xb.astype(np.uint64) - np.uint64(1 << lp)) % np.uint64(p)
    return (p + xb - (1 << lp)) % p


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    d = 2
    while d * d <= n:
        if n % d == 0:
            return False
        d += 1
    return True


def prime_above(w: int) -> int:
    """Smallest prime > 2^w (reading C7: the paper's "log2 p = ell'+1" names
    no prime; the smallest prime above 2^w is the smallest p for which Alg 6
    maps zero <=> zero)."""
    p = (1 << w) + 1
    while not is_prime(p):
        p += 1
    return p
