"""Plaintext definitions the tests compare reconstructed shares against.

These are the functions DReLU / ReLU compute on the fixed-point band
(P:212-216), written from their definitions, not
from the protocol.
"""
import numpy as np


def _mask(ell):
    return np.uint64((1 << ell) - 1)


def band_sign(x, ell, lx, f):
    """(drelu, valid): drelu = 1 for positive x (x in [0, 2^(f+lx))), 0 for
    negative; valid marks inputs whose sign the key-bit ladder determines,
    2^f <= xi < 2^(f+lx) (readings C13-C15 in DESIGN.md)."""
    x = np.asarray(x, dtype=np.uint64)
    top = np.uint64(1 << (f + lx))
    with np.errstate(over="ignore"):
        negx = (np.uint64(0) - x) & _mask(ell)
    pos = x < top
    neg = (negx < top) & (x != 0)
    xi = np.where(pos, x, negx)
    valid = (pos | neg) & (xi >= np.uint64(1 << f)) & (x != 0)
    return pos.astype(np.uint64), valid


def relu_plain(x, ell, lx, f):
    """max(x, 0) in two's complement over Z_{2^ell} for band inputs."""
    x = np.asarray(x, dtype=np.uint64)
    pos, _ = band_sign(x, ell, lx, f)
    return np.where(pos == 1, x, np.uint64(0)).astype(np.uint64)
