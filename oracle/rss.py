"""RSS variant: Alg 9 (RSS Bicoptor 2.0 DReLU) and RSS ReLU by
secret multiplication -- oracle; test infrastructure only.

Replicated secret sharing: x = x_0 + x_1 + x_2 mod 2^ell, party
P_i holds components (x_i, x_{i+1}) (indices mod 3).  Alg 9 bridges to the UBL
protocol: P0's DReLU input is x_0 + x_1, P1's is x_2 (online step 1), and the
blinding bit t is re-shared in RSS form from seed012 (preprocessing step 1).

Readings:
  C25  each value "generated from seedXY" is the element's u64 of a ChaCha
       stream (seed, label) like every other draw; the
       random bit s is bit 0 of the element's u64 of (seed2, bc2.rs2b).
  C26  "secret multiplication" is the standard RSS product:
       P_i computes z_i = a_i b_i + a_i b_{i+1} + a_{i+1} b_i + g_i with a zero
       sharing g_i = F(k_i) - F(k_{i+1}) from the pairwise seeds
       (k_0 = seed02, k_1 = seed01, k_2 = seed12), then sends z_i to P_{i-1}
       (one round); the product's components are z_0, z_1, z_2.
  C27  the public bit DReLU'' is added to component 0 (the component P0 and P2 hold).
"""
from __future__ import annotations

import numpy as np

from . import bicoptor as B
from . import ring
from .chacha import element_u64, label_u64

L_ALPHA = [label_u64(f"bc2.ra0{k}".encode()) for k in range(3)]  # seed012: [alpha]_k
L_S1 = label_u64(b"bc2.rs01")                                    # seed012: [s]_1
L_S2 = label_u64(b"bc2.rs12")                                    # seed12:  [s]_2
L_SBIT = label_u64(b"bc2.rs2b")                                  # seed2:   s (bit 0)
L_MUL = {"s02": label_u64(b"bc2.rm02"), "s01": label_u64(b"bc2.rm01"), "s12": label_u64(b"bc2.rm12")}
L_MUL2 = {"s02": label_u64(b"bc2.rn02"), "s01": label_u64(b"bc2.rn01"), "s12": label_u64(b"bc2.rn12")}


def _u64(prm, seed, lab, j):
    return element_u64(seed, lab, prm.rounds, j, 1)[:, 0] & np.uint64(ring.mask(prm.ell))


def zero_share(prm, seeds, j, labels):
    """g_i = F(k_i) - F(k_{i+1}) with k_0 = seed02, k_1 = seed01, k_2 = seed12
    (reading C26): sum_i g_i = 0, and P_i can compute g_i from the two seeds it holds."""
    L = prm.ell
    F = [_u64(prm, getattr(seeds, k), labels[k], j) for k in ("s02", "s01", "s12")]
    return [ring.sub(F[i], F[(i + 1) % 3], L) for i in range(3)]


def rss_mul(prm, a, b, g):
    """Reading C26: z_i = a_i b_i + a_i b_{i+1} + a_{i+1} b_i + g_i (mod 2^ell)."""
    L = prm.ell
    z = []
    for i in range(3):
        k = (i + 1) % 3
        z.append(ring.add(ring.add(ring.mul(a[i], b[i], L), ring.mul(a[i], b[k], L), L),
                          ring.add(ring.mul(a[k], b[i], L), g[i], L), L))
    return z


def preprocess(prm, seeds, j):
    """Alg 9 preprocessing: RSS shares of t, s and s XOR t."""
    L = prm.ell
    t = B.tape(prm, seeds.s01, j)["t"]                                  # step 1: t from seed01
    alpha = [_u64(prm, seeds.s012, L_ALPHA[k], j) for k in range(3)]
    beta = [ring.sub(alpha[0], alpha[2], L), ring.sub(alpha[1], alpha[0], L), ring.sub(alpha[2], alpha[1], L)]
    tsh = [beta[0], ring.add(beta[1], t, L), beta[2]]                    # [t]_1 = [beta]_1 + t
    s1 = _u64(prm, seeds.s012, L_S1, j)                                  # step 2
    s2 = _u64(prm, seeds.s12, L_S2, j)
    s = element_u64(seeds.s2, L_SBIT, prm.rounds, j, 1)[:, 0] & np.uint64(1)
    ssh = [ring.sub(ring.sub(s, s1, L), s2, L), s1, s2]                  # [s]_0 = s - [s]_1 - [s]_2
    st = rss_mul(prm, ssh, tsh, zero_share(prm, seeds, j, L_MUL))       # step 3: [s][t]
    u = [ring.sub(ring.add(ssh[i], tsh[i], L), ring.mul(np.uint64(2), st[i], L), L) for i in range(3)]
    return {"t": t, "s": s, "tsh": tsh, "ssh": ssh, "st": st, "u": u}


def drelu_rss(prm, x0, x1, x2, j, seeds) -> dict:
    """Alg 9 online with its preprocessing; returns the RSS
    components y_0, y_1, y_2 of DReLU(x)."""
    L = prm.ell
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    pre = preprocess(prm, seeds, j)
    a = ring.add(np.asarray(x0, dtype=np.uint64), np.asarray(x1, dtype=np.uint64), L)   # P0's input
    m0 = B.drelu_send(prm, 0, a, j, seeds.s01)                                          # Alg 7 steps 1-8
    m1 = B.drelu_send(prm, 1, np.asarray(x2, dtype=np.uint64), j, seeds.s01)
    z = B.zero_test(prm, m0["W"], m1["W"])                                              # step 2
    D2 = z ^ pre["s"]                                                                   # step 3: s XOR DReLU'
    y = []
    for k in range(3):                                                                  # step 5
        uk = pre["u"][k]
        yk = ring.sub(uk, ring.mul(ring.mul(np.uint64(2), D2, L), uk, L), L)
        if k == 0:
            yk = ring.add(yk, D2, L)
        y.append(yk)
    return {"y": y, "z": z, "D2": D2, "W0": m0["W"], "W1": m1["W"], **pre}


def relu_rss(prm, x0, x1, x2, j, seeds) -> dict:
    """RSS ReLU: the secret multiplication [x][DReLU(x)] (reading C26)."""
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    d = drelu_rss(prm, x0, x1, x2, j, seeds)
    xs = [np.asarray(v, dtype=np.uint64) for v in (x0, x1, x2)]
    y = rss_mul(prm, xs, d["y"], zero_share(prm, seeds, j, L_MUL2))
    return {"y": y, "drelu": d["y"], "z": d["z"], "D2": d["D2"]}


def reconstruct(y, ell):
    return ring.add(ring.add(y[0], y[1], ell), y[2], ell)
