"""Bicoptor (the paper's predecessor, "Bicoptor-1") DReLU as Bicoptor 2.0
describes it -- an in-repo comparison point; oracle, test
infrastructure only.

The paper defines Bicoptor-1 only by contrast with Alg 7 (readings C32-C34):
  * step 3 truncates with SecureML's probabilistic Alg 1, so u_i lives in
    Z_{2^ell} instead of Z_{2^w} (the e1 analysis of sec. 4 applies);
  * step 4 is the recursive sum v_i = sum_{k=i}^{lx} u_k - 1 instead of the
    adjacent pairwise sum;
  * there is no modulo switch: masking, reshare and the zero test stay in
    Z_{2^ell}, so a message is (lx + 1) * ell bits per party;
  * the u_* term that decided DReLU(0) is dropped (P:911 -- it does not change
    ReLU; its definition is not in this paper).
Readings:
  C32  slots i in [0, lx] at offset f (the key-bit window of P:990's first stage:
       2048 -> 512 bits = (lx+1) * 64); the public -1 is P0's (as C8).
  C33  masks r_m are uniform odd elements of Z_{2^ell} (the units, so the zero
       test is preserved: v r = 0 iff v = 0), drawn as u | 1 from a u64 u;
       reshares rho_m are uniform in Z_{2^ell}.
  C34  tape (seed01, label bc1.tape): 192 B = 3 blocks per element at 192 j;
       word 0 = t (bit 31) | perm index (reject >= floor(2^31/S!) S!), words
       2..17 = u64 mask draws r_0..r_7, words 18..33 = u64 reshares rho_0..rho_7;
       the index fallback is ChaCha(seed01, bc1.fbk1, counter j*256 + k) as u32 words.
"""
from __future__ import annotations

import math

import numpy as np

from . import bicoptor as B
from . import ring
from .chacha import chacha_blocks, element_u32, label_u64

L_TAPE1 = label_u64(b"bc1.tape")
L_FB1 = label_u64(b"bc1.fbk1")


def tape1(prm: B.Params, seed01: bytes, j) -> dict:
    """Reading C34."""
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    n, S = j.size, prm.slots
    assert S <= 8
    T = element_u32(seed01, L_TAPE1, prm.rounds, j, 48)
    t = (T[:, 0] >> np.uint32(31)).astype(np.uint64)
    idx = (T[:, 0] & np.uint32(0x7FFFFFFF)).astype(np.uint64)
    lim = ((1 << 31) // math.factorial(S)) * math.factorial(S)
    for row in np.nonzero(idx >= np.uint64(lim))[0]:
        k, v = 0, lim
        while v >= lim:
            blk = chacha_blocks(seed01, L_FB1, [int(j[row]) * 256 + k // 16], prm.rounds)[0]
            v = int(blk[k % 16]) & 0x7FFFFFFF
            k += 1
        idx[row] = v
    U = np.ascontiguousarray(T[:, 2:34]).view("<u8").reshape(n, 16)
    M = np.uint64(ring.mask(prm.ell))
    r = (U[:, :S] | np.uint64(1)) & M                  # odd: a unit of Z_{2^ell} (ell >= 1)
    rho = U[:, 8:8 + S] & M
    return {"t": t, "k": B._perm_swaps(idx, S), "r": r, "rho": rho}


def ladder1(prm: B.Params, party: int, s) -> np.ndarray:
    """Step 3 with Alg 1: u_i = trc(s, f + i) in Z_{2^ell}, i in [0, lx] (C32)."""
    s = np.atleast_1d(np.asarray(s, dtype=np.uint64))
    return np.stack([ring.trc_secureml(party, s, prm.f + i, prm.ell) for i in range(prm.lx + 1)], axis=1)


def recursive_sums(prm: B.Params, party: int, u) -> np.ndarray:
    """Step 4 of Bicoptor-1: v_i = sum_{k=i}^{lx} u_k - 1 (P0 carries the -1)."""
    L = prm.ell
    v = np.empty_like(u)
    acc = np.zeros(u.shape[0], dtype=np.uint64)
    for i in range(u.shape[1] - 1, -1, -1):
        acc = ring.add(acc, u[:, i], L)
        v[:, i] = ring.sub(acc, np.uint64(1 if party == 0 else 0), L)
    return v


def drelu1_send(prm: B.Params, party: int, xb, j, seed01: bytes) -> dict:
    """Steps 1-8 without the modulo switch; W in Z_{2^ell}, (n, lx+1)."""
    L = prm.ell
    xb = np.atleast_1d(np.asarray(xb, dtype=np.uint64))
    tp = tape1(prm, seed01, j)
    s = np.where(tp["t"] == 1, ring.neg(xb, L), xb).astype(np.uint64)      # steps 1-2
    v = recursive_sums(prm, party, ladder1(prm, party, s))                  # steps 3-4
    v = B.shuffle(tp["k"], v)                                               # step 6
    w = ring.mul(v, tp["r"], L)                                             # step 7
    W = ring.add(w, tp["rho"], L) if party == 0 else ring.sub(w, tp["rho"], L)  # step 8
    return {"t": tp["t"], "W": W}


def zero_test1(prm: B.Params, W0, W1) -> np.ndarray:
    return (ring.add(W0, W1, prm.ell) == 0).any(axis=1).astype(np.uint64)


def drelu1(prm: B.Params, x0, x1, j, seeds) -> dict:
    """Bicoptor-1 DReLU, all three parties; steps 10-11 as Alg 7 (same streams)."""
    m0 = drelu1_send(prm, 0, x0, j, seeds.s01)
    m1 = drelu1_send(prm, 1, x1, j, seeds.s01)
    z = zero_test1(prm, m0["W"], m1["W"])
    q = B.element_u64(seeds.s02, B.L_RESP, prm.rounds, j, 1)[:, 0] & np.uint64(ring.mask(prm.ell))
    y0 = B.drelu_finish(prm, 0, m0["t"], q)
    y1 = B.drelu_finish(prm, 1, m1["t"], ring.sub(z, q, prm.ell))
    return {"y0": y0, "y1": y1, "z": z, "t": m0["t"], "W0": m0["W"], "W1": m1["W"]}
