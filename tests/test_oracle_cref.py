"""Pins for the scalar C oracle (oracle/c/bicoptor_ref.c): the RFC 8439 known answers
for its ChaCha block, and bit-exact agreement with the numpy oracle (itself pinned
against the paper) on 10^5 elements per tape layout -- compact (p = 257), pair (p <= 131)
and large (lx >= 8) -- for DReLU and ReLU, outputs and messages, plus the config-2
ladder / modulo switch."""
import numpy as np
import pytest

import synth
from oracle import bicoptor as B
from oracle import cref
from test_oracle_chacha import _vectors

SEEDS = synth.seeds(0)


@pytest.mark.parametrize("vec", list(_vectors()), ids=lambda v: v[0])
def test_cref_chacha_known_answers(vec):
    src, rounds, key, ctr, lab, blk = vec
    assert cref.chacha_block(key, lab, ctr, rounds) == blk


CASES = [
    (dict(ell=64, lx=7, f=24, mode="guard", rounds=20), 100_000, 0),          # compact: the bench workload
    (dict(ell=64, lx=7, f=24, mode="literal", rounds=20), 100_000, 1 << 30),  # pair tape, p = 131, 8 slots
    (dict(ell=32, lx=5, f=3, mode="guard", rounds=12), 100_000, 8),          # pair tape, p = 67, 6 slots
    (dict(ell=16, lx=7, f=0, mode="guard", rounds=8), 100_000, 0),           # config 1 domain
    (dict(ell=64, lx=31, f=0, mode="guard", rounds=20), 4_000, 1 << 40),     # large tape, p = 2^32 + 15, 32 slots
    (dict(ell=24, lx=10, f=0, mode="literal", rounds=8), 20_000, 0),         # large tape, p = 1031
    (dict(ell=64, lx=31, f=0, mode="literal", rounds=12), 3_000, 0),        # large tape, p = 2^31 + 11 (paper-literal)
]


@pytest.mark.parametrize("kw,n,base", CASES, ids=lambda c: str(c))
def test_cref_matches_numpy_oracle(kw, n, base):
    """Both oracles, same seeded inputs (D1 and D2 halves, with the synth edge cases),
    elements base .. base + n - 1: every output share and every message word equal."""
    prm = B.Params(**kw)
    h = n // 2
    xa = synth.plaintext(h, kw["ell"], kw["lx"], kw["f"], "D1")
    xb = synth.plaintext(n - h, kw["ell"], kw["lx"], kw["f"], "D2")
    x0, x1 = synth.share(np.concatenate([xa, xb]), kw["ell"])
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    for relu, fn in ((False, B.drelu), (True, B.relu)):
        if relu and prm.layout == "large" and n > 4000:
            continue
        ref = fn(prm, x0, x1, j, SEEDS)
        got = cref.fused(prm, x0, x1, base, SEEDS, relu=relu, transcript=True)
        assert np.array_equal(got["y0"], ref["y0"]) and np.array_equal(got["y1"], ref["y1"]), relu
        assert np.array_equal(got["W0"], ref["W0"].astype(np.uint64))
        assert np.array_equal(got["W1"], ref["W1"].astype(np.uint64))


@pytest.mark.parametrize("kw", [CASES[0][0], CASES[1][0], CASES[4][0]], ids=str)
def test_cref_ladder_modswitch_matches(kw):
    prm = B.Params(**kw)
    x, x0, x1 = synth.shares(50_000, kw["ell"], kw["lx"], kw["f"], "D1")
    for party, xb in ((0, x0), (1, x1)):
        assert np.array_equal(cref.ladder_modswitch(prm, party, xb), B.ladder_modswitch(prm, party, xb))


def test_cref_threads_do_not_change_results():
    prm = B.Params()
    x, x0, x1 = synth.shares(30_011, 64, 7, 24, "D2")
    a = cref.fused(prm, x0, x1, 5 << 20, SEEDS, threads=1)
    b = cref.fused(prm, x0, x1, 5 << 20, SEEDS, threads=0)
    assert np.array_equal(a["y0"], b["y0"]) and np.array_equal(a["y1"], b["y1"])


def test_cref_rejects_bad_parameters():
    L = cref.lib()
    # window does not fit (f + lx + w = 5 + 7 + 8 > 16), lx out of range, unknown round count
    for args in ((16, 7, 5, 0, 20), (64, 1, 0, 0, 20), (64, 7, 24, 0, 10)):
        assert L.bcref_fused(*args, SEEDS.s01, SEEDS.s02, SEEDS.s12, None, None, None, None, None, None, 0, 0, 0, 1) == -1
