"""Seeded synthetic inputs for the Bicoptor 2.0 hot path.

Shared by the oracle tests and the CUDA path; it holds none of the method's
arithmetic (no truncation, ladder, PRG tape, masking or zero test).  It only
produces (a) the pre-shared 256-bit seeds and (b) plaintext activations x in
the paper's fixed-point band together with their 2-out-of-2 input sharing
[x]_0 = x + R, [x]_1 = -R (reading C22), R uniform.

Input recipe:
  D1  sign ~ Bern(1/2), lambda ~ U{max(f,1) .. f+lx}, xi ~ U[2^(lambda-1), 2^lambda)
      -- exercises every ladder position.
  D2  x = round(N(0,1) * 2^(f+lx-5)), clipped to |x| < 2^(f+lx) -- activation-like;
      at ell=64, f=24, lx=7 this is N(0,1)*2^26, the paper's 5+26 fixed point.
  Both replace 1% each with edge cases: 0, +-1, +-(2^f-1), +-2^f,
  +-(2^(f+lx)-1), and (lx=7) the literal-mode risk band cut(xi, f) in {84, 85}.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Seeds:
    """Pre-shared seeds seed01, seed02, seed12, and for the RSS variant
    (Alg 9) seed012 (all three parties) and P2's private seed2."""
    s01: bytes
    s02: bytes
    s12: bytes
    s012: bytes = b""
    s2: bytes = b""


def seeds(run: int = 0) -> Seeds:
    """SHA-256("bicoptor/<seed>/run<k>") for each seed."""
    h = lambda tag: hashlib.sha256(f"bicoptor/{tag}/run{run}".encode()).digest()
    return Seeds(h("seed01"), h("seed02"), h("seed12"), h("seed012"), h("seed2"))


def _mask(ell: int) -> np.uint64:
    return np.uint64((1 << ell) - 1)


def plaintext(n: int, ell: int, lx: int, f: int, dist: str = "D1", run: int = 0,
              edge_frac: float = 0.01) -> np.ndarray:
    """n plaintext values x in Z_{2^ell} (uint64), band |x| < 2^(f+lx)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([0xB1C0, run, n, ell, lx, f, {'D1': 1, 'D2': 2}.get(dist, 0)])))
    top = f + lx
    if dist == "D1":
        lam = rng.integers(max(f, 1), top + 1, size=n, dtype=np.int64)
        lo = np.left_shift(np.int64(1), lam - 1)
        xi = lo + (rng.integers(0, 1 << 62, size=n, dtype=np.int64) % lo)
    elif dist == "D2":
        xi = np.rint(np.abs(rng.standard_normal(n)) * float(2 ** (top - 5))).astype(np.int64)
        xi = np.minimum(xi, (1 << top) - 1)
    else:
        raise ValueError(dist)
    neg = rng.integers(0, 2, size=n, dtype=np.int64).astype(bool)
    if edge_frac > 0 and n > 0:
        edges = [0, 1, (1 << f) - 1, 1 << f, (1 << top) - 1]
        if lx == 7:
            edges += [84 << f, (85 << f) + ((1 << f) - 1 if f else 0)]
        edges = [e for e in edges if 0 <= e < (1 << top)]
        sel = rng.random(n) < edge_frac * len(edges)
        xi = xi.copy()
        xi[sel] = np.array(edges, dtype=np.int64)[rng.integers(0, len(edges), size=int(sel.sum()))]
    xu = xi.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = np.where(neg, np.uint64(0) - xu, xu) & _mask(ell)
    return x.astype(np.uint64)


def share(x: np.ndarray, ell: int, run: int = 0):
    """Input sharing [x]_0 = x + R, [x]_1 = -R mod 2^ell with R uniform."""
    x = np.asarray(x, dtype=np.uint64)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([0x5EED, run, x.size, ell])))
    R = rng.integers(0, np.iinfo(np.uint64).max, size=x.size, dtype=np.uint64, endpoint=True) & _mask(ell)
    with np.errstate(over="ignore"):
        x0 = (x + R) & _mask(ell)
        x1 = (np.uint64(0) - R) & _mask(ell)
    return x0.astype(np.uint64), x1.astype(np.uint64)


def rss_share(x: np.ndarray, ell: int, run: int = 0):
    """Replicated 2-out-of-3 input sharing x = x_0 + x_1 + x_2 mod 2^ell with
    x_0, x_1 uniform; party P_i holds (x_i, x_{i+1})."""
    x = np.asarray(x, dtype=np.uint64)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([0x7355, run, x.size, ell])))
    x0 = rng.integers(0, np.iinfo(np.uint64).max, size=x.size, dtype=np.uint64, endpoint=True) & _mask(ell)
    x1 = rng.integers(0, np.iinfo(np.uint64).max, size=x.size, dtype=np.uint64, endpoint=True) & _mask(ell)
    with np.errstate(over="ignore"):
        x2 = (x - x0 - x1) & _mask(ell)
    return x0.astype(np.uint64), x1.astype(np.uint64), x2.astype(np.uint64)


def shares(n: int, ell: int, lx: int, f: int, dist: str = "D1", run: int = 0):
    """(x, x0, x1) for a synthetic batch."""
    x = plaintext(n, ell, lx, f, dist, run)
    x0, x1 = share(x, ell, run)
    return x, x0, x1
