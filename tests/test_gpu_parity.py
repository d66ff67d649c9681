"""GPU parity: the CUDA path through the C ABI against the oracle, element by
element, bit-exact (all integer share arithmetic)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import bicoptor as B  # noqa: E402
from oracle import ring  # noqa: E402
from plain import band_sign, relu_plain  # noqa: E402

SEEDS = synth.seeds(0)


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_04909_b200 import api as a
    a.lib()
    return a


DEV = "cuda:0"


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(DEV)


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def both(prm_kw):
    return B.Params(**prm_kw), prm_kw


PARAMS = [
    dict(ell=64, lx=7, f=24, mode="guard", rounds=20),    # the paper's 5+2 key bits of 5+26
    dict(ell=64, lx=7, f=26, mode="guard", rounds=12),    # 7+0 key bits
    dict(ell=64, lx=7, f=24, mode="guard", rounds=8),
    dict(ell=16, lx=7, f=0, mode="guard", rounds=20),     # config 1
    dict(ell=16, lx=7, f=0, mode="literal", rounds=20),   # paper-literal Z_{2^7}, p = 131 (compact literal tape)
    dict(ell=32, lx=5, f=3, mode="guard", rounds=20),     # p = 67, 6 slots (pair tape)
    dict(ell=12, lx=3, f=1, mode="literal", rounds=8),    # p = 11, 4 slots
    dict(ell=64, lx=7, f=24, mode="literal", rounds=20),  # the bench's paper-literal variant (p = 131, pair tape)
    dict(ell=64, lx=7, f=40, mode="guard", rounds=20),    # compact tape with the window in the high word (f >= 32)
]
SIZES = [1, 7, 8, 9, 1000, 4099]


def _ids(p):
    return f"l{p['ell']}x{p['lx']}f{p['f']}{p['mode'][0]}R{p['rounds']}"


# ---- elementwise primitives --------------------------------------------------------

@pytest.mark.parametrize("ell,k1,k2", [(64, 24, 0), (64, 24, 32), (64, 0, 63), (16, 4, 1), (8, 4, 1), (33, 7, 9)])
def test_trc_parity(api, ell, k1, k2):
    rng = np.random.default_rng(ell * 100 + k1)
    x = rng.integers(0, 2**63, size=4099, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 4099, dtype=np.uint64)
    x &= np.uint64(ring.mask(ell))
    for party in (0, 1):
        got = host(api.trc(party, dev(x), ell, k1, k2))
        assert np.array_equal(got, ring.trc_det_mid(party, x, k1, k2, ell))


@pytest.mark.parametrize("ell,k", [(64, 24), (8, 4), (32, 31), (64, 0)])
def test_trc_prob_parity(api, ell, k):
    rng = np.random.default_rng(k)
    x = rng.integers(0, 2**64 - 1, size=3001, dtype=np.uint64, endpoint=True) & np.uint64(ring.mask(ell))
    x[:5] = 0
    for party in (0, 1):
        assert np.array_equal(host(api.trc_prob(party, dev(x), ell, k)), ring.trc_secureml(party, x, k, ell))


@pytest.mark.parametrize("lp", [1, 7, 8, 16, 31])
def test_modswitch_parity(api, lp):
    p = ring.prime_above(lp)
    rng = np.random.default_rng(lp)
    x = rng.integers(0, 1 << lp, size=2049, dtype=np.uint64)
    x[:3] = 0
    for party in (0, 1):
        got = api.modswitch(party, dev(x), lp, p).cpu().numpy().view(np.uint32).astype(np.uint64)
        assert np.array_equal(got, ring.modswitch(party, x, lp, p))


@pytest.mark.parametrize("kw", PARAMS, ids=_ids)
def test_ladder_modswitch_parity(api, kw):
    oprm = B.Params(**kw)
    x, x0, x1 = synth.shares(4099, kw["ell"], kw["lx"], kw["f"], "D1")
    for party, xs in ((0, x0), (1, x1)):
        got = api.ladder_modswitch(party, dev(xs), api.Params(**kw)).cpu().numpy()
        assert np.array_equal(got, B.ladder_modswitch_bytes(oprm, party, xs))


@pytest.mark.parametrize("lp,p", [(1, 3), (8, 257), (31, (1 << 31) + 11), (32, (1 << 32) + 15), (33, (1 << 33) + 17),
                                  (48, (1 << 48) + 12345), (63, (1 << 63) + 29), (63, (1 << 64) - 59)])
def test_modswitch64_parity(api, lp, p):
    """Alg 6 beyond 31 bits (bc_modswitch64): the full-precision guard domain lp = 32,
    p = 2^32 + 15, and moduli up to 2^64 - 59, against ring.modswitch (Python ints)."""
    rng = np.random.default_rng(lp)
    x = rng.integers(0, 2**64 - 1, size=2049, dtype=np.uint64, endpoint=True)
    x[:3] = 0
    x[3] = np.uint64((1 << lp) - 1)
    xl = [int(v) & ((1 << lp) - 1) for v in x]
    for party in (0, 1):
        got = host(api.modswitch64(party, dev(x), lp, p))
        want = np.array([ring.modswitch(party, v, lp, p) for v in xl], dtype=np.uint64)
        assert np.array_equal(got, want), party


@pytest.mark.parametrize("kw", PARAMS + [dict(ell=64, lx=31, f=0, mode="guard", rounds=20),
                                         dict(ell=64, lx=31, f=0, mode="literal", rounds=8),
                                         dict(ell=40, lx=12, f=3, mode="guard", rounds=8)], ids=_ids)
def test_ladder_modswitch64_parity(api, kw):
    """Alg 7 steps 3-5 with the v'_m as u64 (bc_ladder_modswitch64), every tape up to
    the full-precision 32 slots, n across several warps with a ragged tail."""
    oprm = B.Params(**kw)
    x, x0, x1 = synth.shares(4099, kw["ell"], kw["lx"], kw["f"], "D1")
    for party, xs in ((0, x0), (1, x1)):
        got = api.ladder_modswitch64(party, dev(xs), api.Params(**kw)).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, B.ladder_modswitch(oprm, party, xs)), party


# ---- fused three-party DReLU / ReLU ------------------------------------------------

@pytest.mark.parametrize("kw", PARAMS, ids=_ids)
@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_fused_parity_with_transcript(api, kw, fn):
    oprm = B.Params(**kw)
    prm = api.Params(**kw)
    for n in SIZES:
        for base in (0, 8, 1 << 40):
            x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1", run=n)
            j = np.arange(n, dtype=np.uint64) + np.uint64(base)
            ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
            tr = api.transcript_buffers(n, DEV)
            y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base, transcript=tr)
            assert np.array_equal(host(y0), ref["y0"]), (n, base)
            assert np.array_equal(host(y1), ref["y1"]), (n, base)
            lo0, hi0 = B.encode_msg(ref["W0"])
            lo1, hi1 = B.encode_msg(ref["W1"])
            assert np.array_equal(tr["w0_lo"].cpu().numpy(), lo0) and np.array_equal(tr["w0_hi"].cpu().numpy(), hi0)
            assert np.array_equal(tr["w1_lo"].cpu().numpy(), lo1) and np.array_equal(tr["w1_hi"].cpu().numpy(), hi1)


def test_fused_rejection_fallback(api):
    """Elements whose compact tape rejects (a reshare word >= 253*257^3 or a
    perm index >= 53261*8!) take the fallback stream; they must match the oracle too."""
    from test_oracle_drelu import _compact_rejects
    kw = PARAMS[0]
    oprm = B.Params(**kw)
    rej, _, _ = _compact_rejects(oprm, np.arange(400000, dtype=np.uint64))
    assert len(rej) >= 10
    for r in rej[:10]:
        base = int(r) - int(r) % 8
        x, x0, x1 = synth.shares(64, 64, 7, 24, "D2", run=int(r))
        j = np.arange(64, dtype=np.uint64) + np.uint64(base)
        for fn in ("drelu", "relu"):
            ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
            y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS, elem_base=base)
            assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"])


@pytest.mark.parametrize("kw", [PARAMS[4], PARAMS[5]], ids=_ids)
def test_pair_tape_rejection_fallback(api, kw):
    """Elements whose pair tape rejects a 28-bit draw (p = 131: 2.6e-4 per element,
    p = 67: 5e-5) take the fallback stream; fused DReLU / ReLU and both parties'
    send kernels must match the oracle on them (found from the raw keystream)."""
    from test_oracle_drelu import _pair_rejects
    oprm, prm = B.Params(**kw), api.Params(**kw)
    rej = _pair_rejects(oprm, 1 << 14 if oprm.p == 131 else 1 << 16)
    assert len(rej) >= 3
    for r in rej[:6]:
        base = r - r % 8
        x, x0, x1 = synth.shares(64, kw["ell"], kw["lx"], kw["f"], "D2", run=r)
        j = np.arange(64, dtype=np.uint64) + np.uint64(base)
        for fn in ("drelu", "relu"):
            ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
            y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base)
            assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"]), (fn, r)
        for party, xs in ((0, x0), (1, x1)):
            lo, hi, _ = api.drelu_send(party, dev(xs), prm, SEEDS.s01, base)
            el, eh = _wire(oprm, B.drelu_send(oprm, party, xs, j, SEEDS.s01)["W"])
            assert np.array_equal(_np_plane(lo), el), (party, r)
            if api.wire_format(prm)["hi"] is not None:
                assert np.array_equal(_np_plane(hi), eh), (party, r)


def test_sharding_is_bit_identical(api):
    """elem_base addresses every PRG draw by global index: four shards equal one call."""
    kw = PARAMS[0]
    n = 40000
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    prm = api.Params(**kw)
    for fn in (api.drelu, api.relu):
        y0, y1 = fn(dev(x0), dev(x1), prm, SEEDS)
        cuts = [0, 8, 16000, 30000, n]
        for a, b in zip(cuts[:-1], cuts[1:]):
            s0, s1 = fn(dev(x0[a:b]), dev(x1[a:b]), prm, SEEDS, elem_base=a)
            assert torch.equal(s0, y0[a:b]) and torch.equal(s1, y1[a:b])


@pytest.mark.parametrize("mode,f", [("guard", 0), ("literal", 0), ("guard", 1)])
def test_config1_exhaustive_ell16(api, mode, f):
    """Config 1: DReLU at ell=16, all key bits (lx=7), every x in Z_{2^16} once
    (masks from the synthetic generator), guard and literal mode and the f=1
    variant.  Seed set 0: bit-exact against the oracle for all
    65536 inputs.  64 seed sets: the reconstructed sign is exact on every in-band
    x (guard), or wrong only on the analytic false-positive set (literal, reading
    C6), and oracle parity holds on a sample of each set."""
    kw = dict(ell=16, lx=7, f=f, mode=mode, rounds=20)
    oprm, prm = B.Params(**kw), api.Params(**kw)
    x = np.arange(1 << 16, dtype=np.uint64)
    j = np.arange(x.size, dtype=np.uint64)
    s, valid = band_sign(x, 16, 7, f)
    assert valid.sum() == 2 * ((1 << (f + 7)) - (1 << f))
    from test_oracle_drelu import _literal_fp_set
    fp = _literal_fp_set(16, 7, f) if mode == "literal" else set()
    xi = np.minimum(x, np.uint64(1 << 16) - x)
    allowed = valid & np.isin(xi, np.array(sorted(fp), dtype=np.uint64))
    wrong = np.zeros(x.size, dtype=np.int64)
    rng = np.random.default_rng(21)
    for run in range(64):
        sd = synth.seeds(run)
        x0, x1 = synth.share(x, 16, run=run)
        y0, y1 = api.drelu(dev(x0), dev(x1), prm, sd)
        g0, g1 = host(y0), host(y1)
        if run == 0:
            ref = B.drelu(oprm, x0, x1, j, sd)
            assert np.array_equal(g0, ref["y0"]) and np.array_equal(g1, ref["y1"])
        else:
            idx = np.sort(rng.choice(x.size, 256, replace=False)).astype(np.uint64)
            ref = B.drelu(oprm, x0[idx], x1[idx], idx, sd)
            assert np.array_equal(g0[idx], ref["y0"]) and np.array_equal(g1[idx], ref["y1"]), run
        y = (g0 + g1) & np.uint64(0xFFFF)
        wrong += (valid & (y != s)).astype(np.int64)
    assert not np.any(wrong[valid & ~allowed]), "misclassified outside the analytic set"
    if mode == "literal":
        assert wrong[allowed].sum() > 0      # the literal domain does err there (C6)


def test_config1_all_masks_sign(api):
    """Config 1, exhaustive over masks: the 254 in-band nonzero x times all 2^16
    masks R (16.6M instances) on the GPU; every reconstruction equals the
    plaintext sign (guard mode), ReLU equals max(x,0); oracle parity on a sample."""
    kw = dict(ell=16, lx=7, f=0, mode="guard", rounds=20)
    xi = np.arange(1, 128, dtype=np.uint64)
    xs = np.concatenate([xi, (np.uint64(1 << 16) - xi)])
    R = np.arange(1 << 16, dtype=np.uint64)
    x = np.repeat(xs, R.size)
    Rr = np.tile(R, xs.size)
    x0 = (x + Rr) & np.uint64(0xFFFF)
    x1 = (np.uint64(1 << 16) - Rr) & np.uint64(0xFFFF)
    prm = api.Params(**kw)
    t0, t1 = dev(x0), dev(x1)
    y0, y1 = api.drelu(t0, t1, prm, SEEDS)
    y = host(y0 + y1) & np.uint64(0xFFFF)
    s, valid = band_sign(x, 16, 7, 0)
    assert valid.all() and np.array_equal(y, s)
    r0, r1 = api.relu(t0, t1, prm, SEEDS)
    assert np.array_equal(host(r0 + r1) & np.uint64(0xFFFF), relu_plain(x, 16, 7, 0))
    idx = np.sort(np.random.default_rng(3).choice(x.size, 4096, replace=False)).astype(np.uint64)
    ref = B.drelu(B.Params(**kw), x0[idx], x1[idx], idx, SEEDS)
    assert np.array_equal(host(y0)[idx], ref["y0"]) and np.array_equal(host(y1)[idx], ref["y1"])


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_config3_full_size_sampled(api, fn):
    """Config 3 (2^24 elements, ell=64, 5+2 key bits) in the launch the bench
    times: oracle parity on a seeded 2^14-element sample; reconstructed
    sign / ReLU on every element whose sign the key bits determine."""
    n = 1 << 24
    kw = PARAMS[0]
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS)
    g0, g1 = host(y0), host(y1)
    idx = np.sort(np.random.default_rng(11).choice(n, 1 << 14, replace=False)).astype(np.uint64)
    ref = getattr(B, fn)(B.Params(**kw), x0[idx], x1[idx], idx, SEEDS)
    assert np.array_equal(g0[idx], ref["y0"]) and np.array_equal(g1[idx], ref["y1"])
    with np.errstate(over="ignore"):
        y = g0 + g1
    s, valid = band_sign(x, 64, 7, 24)
    if fn == "drelu":
        assert np.array_equal(y[valid], s[valid])
    else:
        assert np.array_equal(y[valid], relu_plain(x, 64, 7, 24)[valid])


@pytest.mark.parametrize("fn", ["drelu", "relu"])
@pytest.mark.parametrize("kw", [PARAMS[0], PARAMS[7]], ids=_ids)
def test_config3_full_size_exact(api, fn, kw):
    """Config 3 at its full 2^24 elements, in the exact launch the bench times
    (bc_drelu / bc_relu, no transcript, elem_base 0, D2 inputs, seeds run 0):
    EVERY output share against the scalar C oracle (oracle/c, OpenMP over the
    host cores; itself bit-exact with the numpy oracle, test_oracle_cref.py).
    Alg 7, Alg 8 P:1851-1864.  Guard mode (the headline) and the
    bench's paper-literal variant (p = 131)."""
    from oracle import cref
    n = 1 << 24
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS)
    g0, g1 = host(y0), host(y1)
    del y0, y1
    ref = cref.fused(B.Params(**kw), x0, x1, 0, SEEDS, relu=(fn == "relu"))
    bad = np.flatnonzero((g0 != ref["y0"]) | (g1 != ref["y1"]))
    assert bad.size == 0, f"{bad.size} of {n} elements differ, first at {bad[:8]}"


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_materialize2_knob_same_results(api, fn, monkeypatch):
    """BICOPTOR_MATERIALIZE=2 (bench.py's materialize2 leg: both parties' wire values
    reduced, P2 adds W0 + W1) runs another instantiation of the headline kernel; its
    outputs equal the oracle's (Alg 7 step 9)."""
    kw = PARAMS[0]
    n = 40003
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2", run=3)
    monkeypatch.setenv("BICOPTOR_MATERIALIZE", "2")
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS, elem_base=64)
    ref = getattr(B, fn)(B.Params(**kw), x0, x1, np.arange(n, dtype=np.uint64) + np.uint64(64), SEEDS)
    assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"])


def test_config2_ladder_full_size_exact(api):
    """Config 2 (Alg 7 steps 3-5 alone, ell=64, f=24, guard, 2^28 elements, one
    call as the bench times it): every one of the 2^28 x 8 output bytes of both
    parties against the C oracle's v' (byte = v' - 1), compared chunk by chunk;
    plus a seeded 2^14 sample against the numpy oracle.  Alg 5, Alg 6
    P:806-816."""
    from oracle import cref
    n = 1 << 28
    kw = PARAMS[0]
    rng = np.random.default_rng(6)
    x = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    t = dev(x)
    oprm = B.Params(**kw)
    idx = np.sort(rng.choice(n, 1 << 14, replace=False))
    chunk = 1 << 24
    for party in (0, 1):
        out = api.ladder_modswitch(party, t, api.Params(**kw))
        samp = out[torch.from_numpy(idx).to(DEV)].cpu().numpy()
        assert np.array_equal(samp, B.ladder_modswitch_bytes(oprm, party, x[idx]))
        for c in range(0, n, chunk):
            got = out[c:c + chunk].cpu().numpy()
            want = cref.ladder_modswitch(oprm, party, x[c:c + chunk]) - np.uint64(1)
            assert np.array_equal(got, want.astype(np.uint8)), f"party {party} chunk {c >> 24}"
        del out


def test_config2_ladder_full_size_sampled(api):
    """Config 2 (trc + modswitch alone, ell=64, 2^28 elements): sampled parity."""
    n = 1 << 28
    kw = PARAMS[0]
    rng = np.random.default_rng(5)
    x = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    t = dev(x)
    del x
    idx = np.sort(rng.choice(n, 1 << 14, replace=False))
    xs = t[torch.from_numpy(idx).to(DEV)].cpu().numpy().view(np.uint64)
    for party in (0, 1):
        out = api.ladder_modswitch(party, t, api.Params(**kw))
        got = out[torch.from_numpy(idx).to(DEV)].cpu().numpy()
        assert np.array_equal(got, B.ladder_modswitch_bytes(B.Params(**kw), party, xs))
        del out


# ---- party-separated phases on one device ------------------------------------------

def _wire(oprm, W):
    """The oracle's message in the kernels' wire format (byte or uint32 planes)."""
    if oprm.layout == "large":
        return B.encode_msg_large(W)
    return B.encode_msg(W)


def _np_plane(t):
    a = t.cpu().numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a


PARTY_PARAMS = [PARAMS[0], PARAMS[4], PARAMS[5],
                dict(ell=64, lx=31, f=0, mode="guard", rounds=20),     # full precision: uint32 + bit-32 planes
                dict(ell=64, lx=31, f=0, mode="literal", rounds=8),    # p = 2^31 + 11: no bit-32 plane
                dict(ell=24, lx=10, f=0, mode="guard", rounds=8)]


@pytest.mark.parametrize("kw", PARTY_PARAMS, ids=_ids)
def test_party_phases_match_oracle_and_fused(api, kw):
    oprm, prm = B.Params(**kw), api.Params(**kw)
    n, base = (4099 if oprm.layout != "large" else 523), 1 << 20
    x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1")
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    t0, t1 = dev(x0), dev(x1)
    # DReLU
    lo0, hi0, tb0 = api.drelu_send(0, t0, prm, SEEDS.s01, base)
    lo1, hi1, tb1 = api.drelu_send(1, t1, prm, SEEDS.s01, base)
    m0 = B.drelu_send(oprm, 0, x0, j, SEEDS.s01)
    m1 = B.drelu_send(oprm, 1, x1, j, SEEDS.s01)
    for lo, hi, m in ((lo0, hi0, m0), (lo1, hi1, m1)):
        el, eh = _wire(oprm, m["W"])
        assert np.array_equal(_np_plane(lo), el)
        if api.wire_format(prm)["hi"] is not None:
            assert np.array_equal(_np_plane(hi), eh)
        else:
            assert not eh.any()
    r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base, paper_literal=True)
    ya = api.drelu_finish(0, tb0, None, prm, n, SEEDS.s02, base)
    yb = api.drelu_finish(0, tb0, r0, prm, n, None, base)
    y1 = api.drelu_finish(1, tb1, r1, prm, n, None, base)
    f0, f1 = api.drelu(t0, t1, prm, SEEDS, elem_base=base)
    assert torch.equal(ya, f0) and torch.equal(yb, f0) and torch.equal(y1, f1)
    # P0's send with its output in the same kernel (bc_drelu_send_p0): same message, same share
    yp = torch.empty_like(t0)
    lp, hp, _ = api.drelu_send(0, t0, prm, SEEDS.s01, base, out=(*api.msg_buffers(n, DEV, prm)[:2], None),
                               y=yp, seed02=SEEDS.s02)
    assert torch.equal(yp, f0) and torch.equal(lp, lo0) and (api.wire_format(prm)["hi"] is None or torch.equal(hp, hi0))
    # ReLU
    L0, H0, T0, d0 = api.relu_send(0, t0, prm, SEEDS.s01, SEEDS.s02, base)
    L1, H1, T1, d1 = api.relu_send(1, t1, prm, SEEDS.s01, SEEDS.s12, base)
    e, c1 = api.relu_helper(L0, H0, L1, H1, prm, SEEDS.s02, SEEDS.s12, base)
    ref = B.relu(oprm, x0, x1, j, SEEDS)
    assert np.array_equal(host(d0), ref["d0"]) and np.array_equal(host(e), ref["e"]) and np.array_equal(host(c1), ref["c1"])
    # the peer-transport entry points store d and e a second time, bit for bit
    dp, ed = torch.empty_like(d0), torch.empty_like(e)
    api.relu_send(0, t0, prm, SEEDS.s01, SEEDS.s02, base, d_peer=dp)
    api.relu_helper(L0, H0, L1, H1, prm, SEEDS.s02, SEEDS.s12, base, e_dup=ed)
    assert torch.equal(dp, d0) and torch.equal(ed, e)
    z0 = api.relu_finish(0, t0, T0, d0, d1, e, None, prm, SEEDS.s02, base)
    z1 = api.relu_finish(1, t1, T1, d1, d0, e, c1, prm, SEEDS.s12, base)
    g0, g1 = api.relu(t0, t1, prm, SEEDS, elem_base=base)
    assert torch.equal(z0, g0) and torch.equal(z1, g1)
    assert np.array_equal(host(z0), ref["y0"]) and np.array_equal(host(z1), ref["y1"])


# ---- boundary errors ---------------------------------------------------------------

def test_abi_errors(api):
    prm = api.Params()
    x = torch.zeros(33, dtype=torch.int64, device=DEV)
    with pytest.raises(api.BicoptorError, match="aligned|multiple"):
        api.drelu(x[1:17], x[1:17].clone(), prm, SEEDS)          # misaligned x0
    with pytest.raises(api.BicoptorError, match="multiple"):
        api.drelu(x[:16], x[16:32], prm, SEEDS, elem_base=3)     # elem_base % 8
    with pytest.raises(api.BicoptorError, match="overlaps"):
        api.drelu(x[:16], x[16:32], prm, SEEDS, y0=x[:16])      # aliasing
    with pytest.raises(api.BicoptorError, match="window"):
        api.Params(ell=16, lx=7, f=2).c()                        # f + lx + w > ell
    with pytest.raises(api.BicoptorError, match="CUDA tensor"):
        api.drelu(torch.zeros(8, dtype=torch.int64), torch.zeros(8, dtype=torch.int64), prm, SEEDS)
    y0, y1 = api.drelu(x[:0], x[16:16], prm, SEEDS)                # n = 0 is a no-op
    assert y0.numel() == 0


# ---- config 5: E2E-shaped ReLU layer stream (CUDA graph) ---------------------------

def test_relu_stream_graph_matches_eager_and_oracle(api):
    """The CIFAR10_VGG16 ReLU layer sequence at batch 2: the captured CUDA graph
    equals eager launches bit for bit, and sampled outputs of every layer match
    the oracle at that layer's global index range."""
    from paper_2309_04909_b200 import stream as S
    kw = PARAMS[0]
    prm = api.Params(**kw)
    st = S.ReluStream(S.layer_sizes("CIFAR10_VGG16", batch=2), prm, SEEDS, DEV, base=1 << 32)
    rng = np.random.default_rng(9)
    xs = []
    for i, n in enumerate(st.sizes):
        x, x0, x1 = synth.shares(n, 64, 7, 24, "D2", run=i)
        st.x0[i].copy_(dev(x0))
        st.x1[i].copy_(dev(x1))
        xs.append((x, x0, x1))
    st.run_eager()
    eager = [(y0.clone(), y1.clone()) for y0, y1 in zip(st.y0, st.y1)]
    for y in st.y0 + st.y1:
        y.zero_()
    st.capture()
    st.replay()
    torch.cuda.synchronize()
    oprm = B.Params(**kw)
    for i, n in enumerate(st.sizes):
        assert torch.equal(st.y0[i], eager[i][0]) and torch.equal(st.y1[i], eager[i][1])
        idx = np.sort(rng.choice(n, min(n, 512), replace=False))
        x, x0, x1 = xs[i]
        ref = B.relu(oprm, x0[idx], x1[idx], idx.astype(np.uint64) + np.uint64(st.bases[i]), SEEDS)
        assert np.array_equal(host(st.y0[i])[idx], ref["y0"]) and np.array_equal(host(st.y1[i])[idx], ref["y1"])
    # advance(): the next forward re-captured at the next global index range (fresh draws)
    b0 = st.bases[0]
    st.advance()
    assert st.bases[0] == b0 + S.index_span(st.sizes)
    st.replay()
    torch.cuda.synchronize()
    for i, n in enumerate(st.sizes):
        idx = np.sort(rng.choice(n, min(n, 256), replace=False))
        x, x0, x1 = xs[i]
        ref = B.relu(oprm, x0[idx], x1[idx], idx.astype(np.uint64) + np.uint64(st.bases[i]), SEEDS)
        assert np.array_equal(host(st.y0[i])[idx], ref["y0"]) and np.array_equal(host(st.y1[i])[idx], ref["y1"])


# ---- RSS variant (Alg 9) ---------------------------------------------------------------

RSS_PARAMS = [PARAMS[0], PARAMS[1], PARAMS[2], PARAMS[3]]


@pytest.mark.parametrize("kw", RSS_PARAMS, ids=_ids)
@pytest.mark.parametrize("fn", ["drelu_rss", "relu_rss"])
def test_rss_parity(api, kw, fn):
    """bc_drelu_rss / bc_relu_rss: all three output components bit-exact
    against oracle.rss, ragged sizes and several element bases."""
    from oracle import rss
    oprm = B.Params(**kw)
    prm = api.Params(**kw)
    for n in SIZES:
        for base in (0, 8, 1 << 40):
            x = synth.plaintext(n, kw["ell"], kw["lx"], kw["f"], "D1", run=n)
            xs = synth.rss_share(x, kw["ell"], run=n)
            j = np.arange(n, dtype=np.uint64) + np.uint64(base)
            ref = getattr(rss, fn)(oprm, *xs, j, SEEDS)
            ys = getattr(api, fn)(*(dev(v) for v in xs), prm, SEEDS, elem_base=base)
            for k in range(3):
                assert np.array_equal(host(ys[k]), ref["y"][k]), (n, base, k)


@pytest.mark.parametrize("fn", ["drelu_rss", "relu_rss"])
def test_rss_full_size_sampled(api, fn):
    """2^24 elements in one launch: oracle parity on a 2^13 sample; opened sign /
    ReLU on every element the key bits determine."""
    from oracle import rss
    n = 1 << 24
    kw = PARAMS[0]
    x = synth.plaintext(n, 64, 7, 24, "D2")
    xs = synth.rss_share(x, 64)
    ys = [host(t) for t in getattr(api, fn)(*(dev(v) for v in xs), api.Params(**kw), SEEDS)]
    idx = np.sort(np.random.default_rng(12).choice(n, 1 << 13, replace=False)).astype(np.uint64)
    ref = getattr(rss, fn)(B.Params(**kw), *(v[idx] for v in xs), idx, SEEDS)
    for k in range(3):
        assert np.array_equal(ys[k][idx], ref["y"][k])
    with np.errstate(over="ignore"):
        y = ys[0] + ys[1] + ys[2]
    s, valid = band_sign(x, 64, 7, 24)
    want = s if fn == "drelu_rss" else relu_plain(x, 64, 7, 24)
    assert np.array_equal(y[valid], want[valid])


def test_rss_abi_errors(api):
    import ctypes
    L = api.lib()
    cp, cs = api.Params().c(), api.seeds_struct(SEEDS)
    t = [torch.zeros(16, dtype=torch.int64, device=DEV) for _ in range(6)]
    p = [v.data_ptr() for v in t]
    call = lambda *ptrs, n=16, base=0, prm=cp: L.bc_drelu_rss(*ptrs, n, base, ctypes.byref(prm), ctypes.byref(cs),  # noqa: E731
                                                               SEEDS.s012, SEEDS.s2, None)
    assert call(*p) == 0
    assert call(*p, n=0) == 0
    assert call(p[0], p[1], p[2], p[0], p[4], p[5]) == -5      # output aliases an input
    assert call(p[0], p[1], p[2], p[3], p[3], p[5]) == -5      # outputs alias each other
    assert call(p[0] + 8, *p[1:]) == -3                          # misaligned
    assert call(*p, base=4) == -3
    assert call(None, *p[1:]) == -1
    wide = api.Params(ell=16, lx=7, f=0, mode="literal").c()
    assert call(*p, prm=wide) == -1                              # compact tape only


# ---- large tape: lx >= 8, full precision lx = 31 (NEXT #2) ------------------------------

LARGE_PARAMS = [
    dict(ell=64, lx=31, f=0, mode="guard", rounds=20),     # full 5+26 precision, p = 2^32 + 15
    dict(ell=64, lx=31, f=0, mode="literal", rounds=12),   # the paper's Z_{2^31}, p = 2^31 + 11
    dict(ell=24, lx=10, f=0, mode="guard", rounds=8),
    dict(ell=20, lx=8, f=1, mode="guard", rounds=20),
    dict(ell=40, lx=15, f=3, mode="guard", rounds=8),      # p = 65537: p - 1 = 2^16, no mask rejection
]


@pytest.mark.parametrize("kw", LARGE_PARAMS, ids=_ids)
@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_large_parity_with_transcript(api, kw, fn):
    oprm = B.Params(**kw)
    prm = api.Params(**kw)
    for n in (1, 7, 9, 203):
        for base in (0, 1 << 40):
            x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1", run=n)
            j = np.arange(n, dtype=np.uint64) + np.uint64(base)
            ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
            tr = api.transcript_buffers(n, DEV, prm)
            y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base, transcript=tr)
            assert np.array_equal(host(y0), ref["y0"]), (n, base)
            assert np.array_equal(host(y1), ref["y1"]), (n, base)
            assert np.array_equal(host(tr["w0_lo"]), ref["W0"]) and np.array_equal(host(tr["w1_lo"]), ref["W1"])


def test_large_fallback_elements(api):
    """Elements whose Fisher-Yates draws reject (~0.35 % at 32 slots) or whose
    48-bit mask / reshare draws reject (< 2^-15 per draw) take the fallback
    stream; they must match the oracle, messages included."""
    from test_oracle_fullprec import _raw_draw_rejects, _raw_perm_rejects
    kw = LARGE_PARAMS[0]
    oprm, prm = B.Params(**kw), api.Params(**kw)
    rej, _ = _raw_perm_rejects(oprm, np.arange(8000, dtype=np.uint64))
    rows = list(np.nonzero(rej)[0][:8])
    assert len(rows) >= 5
    drej = np.nonzero(_raw_draw_rejects(oprm, np.arange(3000, dtype=np.uint64)))[0]  # a 48-bit draw rejects
    assert len(drej) >= 1
    rows += list(drej[:3])
    for r in rows:
        base = int(r) - int(r) % 8
        x, x0, x1 = synth.shares(16, 64, 31, 0, "D2", run=int(r))
        j = np.arange(16, dtype=np.uint64) + np.uint64(base)
        for fn in ("drelu", "relu"):
            ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
            tr = api.transcript_buffers(16, DEV, prm)
            y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base, transcript=tr)
            assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"])
            assert np.array_equal(host(tr["w0_lo"]), ref["W0"])


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_full_precision_full_size_sampled(api, fn):
    """lx = 31, f = 0, 2^24 elements in the launch the bench times: oracle parity on
    a 2^10 sample; opened sign / ReLU on every nonzero element."""
    n = 1 << 24
    kw = LARGE_PARAMS[0]
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")          # the bench batch: |x| < 2^31
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS)
    g0, g1 = host(y0), host(y1)
    idx = np.sort(np.random.default_rng(13).choice(n, 1 << 10, replace=False)).astype(np.uint64)
    ref = getattr(B, fn)(B.Params(**kw), x0[idx], x1[idx], idx, SEEDS)
    assert np.array_equal(g0[idx], ref["y0"]) and np.array_equal(g1[idx], ref["y1"])
    with np.errstate(over="ignore"):
        y = g0 + g1
    s, valid = band_sign(x, 64, 31, 0)
    want = s if fn == "drelu" else relu_plain(x, 64, 31, 0)
    assert np.array_equal(y[valid], want[valid])


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_full_precision_full_size_exact(api, fn):
    """lx = 31, f = 0, guard (p = 2^32 + 15): all 2^24 outputs of the launch the bench
    times (no transcript, elem_base 0: the W32 kernel with the pseudo-Mersenne slot
    arithmetic) against the scalar C oracle, element by element (Alg 7 P:875-895,
    Alg 8)."""
    from oracle import cref
    n = 1 << 24
    kw = LARGE_PARAMS[0]
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), api.Params(**kw), SEEDS)
    g0, g1 = host(y0), host(y1)
    del y0, y1
    ref = cref.fused(B.Params(**kw), x0, x1, 0, SEEDS, relu=(fn == "relu"))
    bad = np.flatnonzero((g0 != ref["y0"]) | (g1 != ref["y1"]))
    assert bad.size == 0, f"{bad.size} of {n} elements differ, first at {bad[:8]}"


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_literal_full_precision_exact(api, fn):
    """The paper-literal full precision (lx = 31, w = 31, p = 2^31 + 11: the kernels with the
    p = 2^31 + 11 slot arithmetic): 2^22 outputs without a transcript at elem_base 0 against
    the scalar C oracle element by element, and a ragged batch at a high base against the
    numpy oracle, both fused and through the party phases (Alg 7, Alg 8)."""
    from oracle import cref
    kw = LARGE_PARAMS[1]
    oprm, prm = B.Params(**kw), api.Params(**kw)
    n = 1 << 22
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2")
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS)
    ref = cref.fused(oprm, x0, x1, 0, SEEDS, relu=(fn == "relu"))
    bad = np.flatnonzero((host(y0) != ref["y0"]) | (host(y1) != ref["y1"]))
    assert bad.size == 0, f"{bad.size} of {n} elements differ, first at {bad[:8]}"
    m, base = 1003, (1 << 40) + 8
    x, x0, x1 = synth.shares(m, 64, 31, 0, "D1", run=7)
    j = np.arange(m, dtype=np.uint64) + np.uint64(base)
    ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
    y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base)
    assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"])
    if fn == "drelu":
        lo0, hi0, tb0 = api.drelu_send(0, dev(x0), prm, SEEDS.s01, base)
        lo1, hi1, tb1 = api.drelu_send(1, dev(x1), prm, SEEDS.s01, base)
        r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base, paper_literal=True)
        assert np.array_equal(host(api.drelu_finish(0, tb0, r0, prm, m, None, base)), ref["y0"])
        assert np.array_equal(host(api.drelu_finish(1, tb1, r1, prm, m, None, base)), ref["y1"])


@pytest.mark.parametrize("base", [0, 1 << 40])
def test_p15_wide_operand_slots(api, base):
    """The p = 2^32 + 15 kernels' generic path, forced: shares chosen from each element's t
    (the oracle's tape) so that the blinded s_0 = 1 and -s_1 = 1 + k (k < 15).  Window 0 then
    gives P0 c = 2^32 (Alg 6's image of 0) and P1 d = 2^32 + 14 - k >= 2^32 in the slot Pi
    sends it to -- operands the 32-bit fast path flags.  Fused DReLU / ReLU (both elem_base
    ranges: with and without the first-round precomputation) and the party phases equal the
    oracle (Alg 7 steps 3-9)."""
    kw = LARGE_PARAMS[0]
    oprm, prm = B.Params(**kw), api.Params(**kw)
    n = 203
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    t = B.tape(oprm, SEEDS.s01, j)["t"].astype(np.uint64)
    k = np.arange(n, dtype=np.uint64) % np.uint64(15)
    with np.errstate(over="ignore"):
        s0 = np.ones(n, dtype=np.uint64)
        s1 = np.uint64(0) - (np.uint64(1) + k)                   # -s_1 = 1 + k
        x0 = np.where(t == 1, np.uint64(0) - s0, s0)             # s_b = (-1)^t x_b
        x1 = np.where(t == 1, np.uint64(0) - s1, s1)
    for fn in ("drelu", "relu"):
        ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
        y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=int(base))
        assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"]), fn
    lo0, hi0, tb0 = api.drelu_send(0, dev(x0), prm, SEEDS.s01, int(base))
    lo1, hi1, tb1 = api.drelu_send(1, dev(x1), prm, SEEDS.s01, int(base))
    r0, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, int(base), paper_literal=True)
    ref = B.drelu(oprm, x0, x1, j, SEEDS)
    assert np.array_equal(host(api.drelu_finish(0, tb0, r0, prm, n, None, int(base))), ref["y0"])
    assert np.array_equal(host(api.drelu_finish(1, tb1, r1, prm, n, None, int(base))), ref["y1"])


def test_large_abi_errors(api):
    import ctypes
    L = api.lib()
    cp = api.Params(ell=64, lx=31, f=0).c()
    assert cp.p == 2**32 + 15 and cp.slots == 32 and api.TAPE[cp.tape] == "large"
    t = torch.zeros(16, dtype=torch.int64, device=DEV)
    v = torch.zeros((16, 8), dtype=torch.uint8, device=DEV)
    # byte-plane formats hold at most 8 slots
    assert L.bc_ladder_modswitch(0, t.data_ptr(), v.data_ptr(), 16, ctypes.byref(cp), None) == -1
    # large-tape wire format: uint32 planes; at p = 2^32 + 15 the bit-32 plane is required
    lo32 = torch.zeros((16, 32), dtype=torch.int32, device=DEV)
    assert L.bc_drelu_send(0, t.data_ptr(), lo32.data_ptr(), None, v.data_ptr(), 16, 0, ctypes.byref(cp),
                           SEEDS.s01, None) == -1
    assert L.bc_drelu_helper(lo32.data_ptr(), None, lo32.data_ptr(), None, None, t.data_ptr(), 16, 0,
                             ctypes.byref(cp), SEEDS.s02, None) == -1
    # large transcript: u64 planes, hi planes must be NULL
    w = [torch.zeros((16, 32), dtype=torch.int64, device=DEV) for _ in range(2)]
    ys = [torch.zeros(16, dtype=torch.int64, device=DEV) for _ in range(3)]
    cs = api.seeds_struct(SEEDS)
    bad = api.bc_transcript(w[0].data_ptr(), v.data_ptr(), w[1].data_ptr(), None)
    assert L.bc_drelu(t.data_ptr(), ys[2].data_ptr(), ys[0].data_ptr(), ys[1].data_ptr(), 16, 0, ctypes.byref(cp),
                      ctypes.byref(cs), ctypes.byref(bad), None) == -1
    ok = api.bc_transcript(w[0].data_ptr(), None, w[1].data_ptr(), None)
    assert L.bc_drelu(t.data_ptr(), ys[2].data_ptr(), ys[0].data_ptr(), ys[1].data_ptr(), 16, 0, ctypes.byref(cp),
                      ctypes.byref(cs), ctypes.byref(ok), None) == 0


# ---- truncation study (NEXT #3) ----------------------------------------------------------

@pytest.mark.parametrize("ell,k", [(64, 26), (64, 13), (32, 5), (16, 0)])
@pytest.mark.parametrize("q", [0, 1])
def test_trc_aby3_parity(api, ell, k, q):
    from oracle import trunc
    for n in SIZES:
        for base in (0, 1 << 40):
            x, x0, x1 = synth.shares(n, ell, 5, min(k, ell - 7), "D1", run=n + q)
            j = np.arange(n, dtype=np.uint64) + np.uint64(base)
            r0, r1 = trunc.trc_aby3(x0, x1, trunc.aby3_pre(ell, k, j, SEEDS, 20, q), k, ell)
            y0, y1 = api.trc_aby3(dev(x0), dev(x1), ell, k, SEEDS, elem_base=base, q=q)
            assert np.array_equal(host(y0), r0) and np.array_equal(host(y1), r1), (n, base)


@pytest.mark.parametrize("order", ["mul_then_trc", "trc_then_mul"])
@pytest.mark.parametrize("alg", ["secureml", "aby3"])
@pytest.mark.parametrize("ell,f,rounds", [(64, 26, 20), (32, 13, 8)])
def test_mul_trc_parity(api, order, alg, ell, f, rounds):
    from oracle import trunc
    for n in (1, 9, 1000):
        X = synth.plaintext(n, ell, 5, f, "D1", run=1)
        Y = synth.plaintext(n, ell, 5, f, "D1", run=2)
        x0, x1 = synth.share(X, ell, run=3)
        y0, y1 = synth.share(Y, ell, run=4)
        j = np.arange(n, dtype=np.uint64) + np.uint64(64)
        ref = getattr(trunc, order)(alg, x0, x1, y0, y1, f, ell, j, SEEDS, rounds)
        z0, z1 = api.mul_trc(order, alg, dev(x0), dev(x1), dev(y0), dev(y1), ell, f, SEEDS, elem_base=64,
                             rounds=rounds)
        assert np.array_equal(host(z0), ref[0]) and np.array_equal(host(z1), ref[1])


def test_trc_count_exhaustive_ell12(api):
    """Every band x (|x| < 2^10) against all 2^12 masks, three algorithms: the
    GPU counts equal the oracle's brute force, and the e1 counts are xi (Alg 1,
    Alg 2) and 0 (Alg 4)."""
    from oracle import trunc
    ell, k = 12, 4
    xi = np.arange(1, 1 << 10, dtype=np.uint64)
    xs = np.concatenate([xi, np.uint64(1 << ell) - xi])
    xis = np.concatenate([xi, xi])
    for alg in ("secureml", "aby3", "det"):
        got = api.trc_count(alg, dev(xs), ell, k).cpu().numpy()
        ref = np.stack([trunc.count_masks(alg, int(x), k, ell) for x in xs])
        assert np.array_equal(got, ref), alg
        assert np.array_equal(got[:, 2], xis if alg != "det" else np.zeros_like(xis))


def test_trc_count_ell24_closed_forms_and_ranges(api):
    """ell = 24, all 2^24 masks for a sample of x: e1 = xi (Alg 1), and Alg 4's
    one-bit error count is (xi mod 2^k) 2^(ell-k); two half-range calls add up
    to one full-range call."""
    ell, k = 24, 7
    rng = np.random.default_rng(5)
    xi = rng.integers(1, 1 << 21, 64).astype(np.uint64)
    xs = np.concatenate([xi, np.uint64(1 << ell) - xi])
    xis = np.concatenate([xi, xi])
    c1 = api.trc_count("secureml", dev(xs), ell, k).cpu().numpy()
    assert np.array_equal(c1[:, 2], xis.astype(np.int64)) and np.all(c1.sum(axis=1) == 1 << ell)
    cd = api.trc_count("det", dev(xs), ell, k).cpu().numpy()
    assert np.all(cd[:, 2] == 0)
    assert np.array_equal(cd[:, 1], ((xis % (1 << k)) * (1 << (ell - k))).astype(np.int64))
    half = api.trc_count("aby3", dev(xs), ell, k, 0, 1 << 23)
    api.trc_count("aby3", dev(xs), ell, k, 1 << 23, 1 << 23, counts=half)
    assert np.array_equal(half.cpu().numpy(), api.trc_count("aby3", dev(xs), ell, k).cpu().numpy())


def test_trunc_abi_errors(api):
    L = api.lib()
    t = [torch.zeros(16, dtype=torch.int64, device=DEV) for _ in range(6)]
    p = [v.data_ptr() for v in t]
    import ctypes
    cs = api.seeds_struct(SEEDS)
    assert L.bc_trc_aby3(p[0], p[1], p[2], p[3], 16, 0, 64, 64, 20, 0, ctypes.byref(cs), None) == -1   # k >= ell
    assert L.bc_trc_aby3(p[0], p[1], p[2], p[3], 16, 0, 64, 26, 20, 2, ctypes.byref(cs), None) == -1   # q
    assert L.bc_trc_aby3(p[0], p[1], p[0], p[3], 16, 0, 64, 26, 20, 0, ctypes.byref(cs), None) == -5   # alias
    assert L.bc_mul_trc(1, 4, p[0], p[1], p[2], p[3], p[4], p[5], 16, 0, 64, 26, 20, ctypes.byref(cs), None) == -1
    assert L.bc_mul_trc(2, 1, p[0], p[1], p[2], p[3], p[4], p[5], 16, 0, 64, 26, 20, ctypes.byref(cs), None) == -1
    assert L.bc_mul_trc(0, 1, p[0], p[1], p[2], p[3], p[4], p[5], 16, 4, 64, 26, 20, ctypes.byref(cs), None) == -3
    assert L.bc_trc_count(3, p[0], 16, 64, 4, 0, 10, p[1], None) == -1
    assert L.bc_trc_count(1, p[0], 16, 64, 0, 0, 10, p[1], None) == -1   # k >= 1


# ---- host-buffer entry points (e2e) ----------------------------------------------------

@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_host_entry_matches_oracle(api, fn):
    """bc_drelu_host / bc_relu_host on pinned host buffers: ragged chunks and a
    ragged tail, bit-exact against the oracle (and so against the device path)."""
    kw = PARAMS[0]
    n, base = 5003, 1 << 20
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=9)
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    ref = getattr(B, fn)(B.Params(**kw), x0, x1, j, SEEDS)
    hx0 = torch.from_numpy(x0.view(np.int64)).pin_memory()
    hx1 = torch.from_numpy(x1.view(np.int64)).pin_memory()
    for chunk in (8, 1024, 1 << 20):
        hy0 = torch.zeros(n, dtype=torch.int64).pin_memory()
        hy1 = torch.zeros(n, dtype=torch.int64).pin_memory()
        ws = api.host_workspace(chunk, DEV)
        getattr(api, fn + "_host")(hx0, hx1, hy0, hy1, api.Params(**kw), SEEDS, ws, chunk, base)
        assert np.array_equal(hy0.numpy().view(np.uint64), ref["y0"]), chunk
        assert np.array_equal(hy1.numpy().view(np.uint64), ref["y1"]), chunk


@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_host_entry_async_back_to_back(api, fn):
    """bc_*_host_async: three requests enqueued back to back on one workspace (they
    pipeline through the same stream ring), then one synchronisation; each request's
    outputs bit-exact with the oracle."""
    kw = PARAMS[0]
    n, chunk = 3001, 512
    reqs = []
    for r in range(3):
        base = (r + 1) << 16
        x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=20 + r)
        hx0 = torch.from_numpy(x0.view(np.int64)).pin_memory()
        hx1 = torch.from_numpy(x1.view(np.int64)).pin_memory()
        hy0 = torch.zeros(n, dtype=torch.int64).pin_memory()
        hy1 = torch.zeros(n, dtype=torch.int64).pin_memory()
        reqs.append((base, x0, x1, hx0, hx1, hy0, hy1))
    ws = api.host_workspace(chunk, DEV)
    for base, _, _, hx0, hx1, hy0, hy1 in reqs:
        getattr(api, fn + "_host")(hx0, hx1, hy0, hy1, api.Params(**kw), SEEDS, ws, chunk, base, sync=False)
    torch.cuda.synchronize()
    for base, x0, x1, _, _, hy0, hy1 in reqs:
        ref = getattr(B, fn)(B.Params(**kw), x0, x1, np.arange(n, dtype=np.uint64) + np.uint64(base), SEEDS)
        assert np.array_equal(hy0.numpy().view(np.uint64), ref["y0"])
        assert np.array_equal(hy1.numpy().view(np.uint64), ref["y1"])


def test_host_entry_errors(api):
    import ctypes
    L = api.lib()
    cp, cs = api.Params().c(), api.seeds_struct(SEEDS)
    h = [torch.zeros(64, dtype=torch.int64).pin_memory() for _ in range(4)]
    p = [t.data_ptr() for t in h]
    ws = api.host_workspace(64, DEV)
    nb = ws.numel() * 8
    assert L.bc_host_workspace_bytes(64) == nb == 3 * 4 * 64 * 8
    call = lambda *a, chunk=64, wsb=nb, base=0: L.bc_drelu_host(*a, 64, base, ctypes.byref(cp), ctypes.byref(cs),  # noqa: E731
                                                                 ws.data_ptr(), wsb, chunk, None)
    assert call(*p) == 0
    assert call(*p, chunk=12) == -1          # not a multiple of 8
    assert call(*p, wsb=nb - 8) == -1        # workspace too small
    assert call(*p, base=4) == -3
    assert call(p[0], p[1], p[0], p[3]) == -5


# ---- Bicoptor-1 comparison point (NEXT #4) -------------------------------------------------

B1_PARAMS = [PARAMS[0], dict(ell=32, lx=7, f=0, mode="guard", rounds=12), PARAMS[3],
             dict(ell=16, lx=4, f=1, mode="guard", rounds=8)]


@pytest.mark.parametrize("kw", B1_PARAMS, ids=_ids)
def test_b1_parity_with_transcript(api, kw):
    from oracle import bicoptor1 as B1
    oprm, prm = B.Params(**kw), api.Params(**kw)
    for n in SIZES:
        for base in (0, 1 << 40):
            x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1", run=n)
            j = np.arange(n, dtype=np.uint64) + np.uint64(base)
            ref = B1.drelu1(oprm, x0, x1, j, SEEDS)
            S = kw["lx"] + 1
            tr = {"w0_lo": torch.empty((n, S), dtype=torch.int64, device=DEV),
                  "w1_lo": torch.empty((n, S), dtype=torch.int64, device=DEV)}
            y0, y1 = api.drelu_b1(dev(x0), dev(x1), prm, SEEDS, elem_base=base, transcript=tr)
            assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"]), (n, base)
            assert np.array_equal(host(tr["w0_lo"]), ref["W0"]) and np.array_equal(host(tr["w1_lo"]), ref["W1"])


def test_b1_fallback_elements(api):
    """Elements whose Bicoptor-1 perm index rejects (~6e-8 per element; indices
    from tests/golden/b1_fallback.txt, written from the oracle by
    tools/find_b1_fallback.py) take the fallback stream on both sides."""
    import os
    from oracle import bicoptor1 as B1
    kw = PARAMS[0]
    path = os.path.join(os.path.dirname(__file__), "golden", "b1_fallback.txt")
    rej = [int(v) for v in open(path).read().split() if not v.startswith("#") and v.strip().isdigit()]
    assert len(rej) >= 2
    for r in rej:
        base = int(r) - int(r) % 8
        x, x0, x1 = synth.shares(16, 64, 7, 24, "D2", run=int(r))
        jj = np.arange(16, dtype=np.uint64) + np.uint64(base)
        ref = B1.drelu1(B.Params(**kw), x0, x1, jj, SEEDS)
        y0, y1 = api.drelu_b1(dev(x0), dev(x1), api.Params(**kw), SEEDS, elem_base=base)
        assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"])


# ---- the top of the index domain (BC_MAX_INDEX = 2^44) ------------------------------------

HIGH_PARAMS = [PARAMS[0], PARAMS[4], PARAMS[5], dict(ell=64, lx=31, f=0, mode="guard", rounds=8)]


@pytest.mark.parametrize("kw", HIGH_PARAMS, ids=_ids)
def test_high_global_indices(api, kw):
    """Elements at the top of the index domain: every stream counter carries
    into its high word (compact part A counter j/4 ~ 2^42, large tape 9j ~ 2^47,
    fallback j 2^20 ~ 2^64), fused and party kernels bit-exact with the oracle;
    one element more is BC_ERANGE."""
    oprm, prm = B.Params(**kw), api.Params(**kw)
    n = 203 if oprm.layout == "large" else 2051
    base = ((1 << 44) - n) // 8 * 8
    x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1")
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    for fn in ("drelu", "relu"):
        y0, y1 = getattr(api, fn)(dev(x0), dev(x1), prm, SEEDS, elem_base=base)
        ref = getattr(B, fn)(oprm, x0, x1, j, SEEDS)
        assert np.array_equal(host(y0), ref["y0"]) and np.array_equal(host(y1), ref["y1"]), fn
    lo0, hi0, tb0 = api.drelu_send(0, dev(x0), prm, SEEDS.s01, base)
    lo1, hi1, tb1 = api.drelu_send(1, dev(x1), prm, SEEDS.s01, base)
    _, r1 = api.drelu_helper(lo0, hi0, lo1, hi1, prm, SEEDS.s02, base)
    y1 = api.drelu_finish(1, tb1, r1, prm, n, None, base)
    assert np.array_equal(host(y1), B.drelu(oprm, x0, x1, j, SEEDS)["y1"])
    with pytest.raises(api.BicoptorError, match=r"\[-2\]"):
        api.drelu(dev(x0), dev(x1), prm, SEEDS, elem_base=base + 8 * ((n + 15) // 8))
    with pytest.raises(api.BicoptorError, match=r"\[-2\]"):
        api.drelu_send(0, dev(x0), prm, SEEDS.s01, 1 << 44)


def test_high_global_indices_rss_b1_trunc(api):
    from oracle import bicoptor1 as B1, rss, trunc
    n = 1003
    base = ((1 << 44) - n) // 8 * 8
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    kw = PARAMS[0]
    oprm, prm = B.Params(**kw), api.Params(**kw)
    x = synth.plaintext(n, 64, 7, 24, "D1")
    xs = synth.rss_share(x, 64)
    ys = api.drelu_rss(*(dev(v) for v in xs), prm, SEEDS, base)
    ref = rss.drelu_rss(oprm, *xs, j, SEEDS)
    for k in range(3):
        assert np.array_equal(host(ys[k]), ref["y"][k])
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1")
    y0, y1 = api.drelu_b1(dev(x0), dev(x1), prm, SEEDS, base)
    r1 = B1.drelu1(oprm, x0, x1, j, SEEDS)
    assert np.array_equal(host(y0), r1["y0"]) and np.array_equal(host(y1), r1["y1"])
    z0, z1 = api.trc_aby3(dev(x0), dev(x1), 64, 26, SEEDS, elem_base=base, q=1)
    t0, t1 = trunc.trc_aby3(x0, x1, trunc.aby3_pre(64, 26, j, SEEDS, 20, 1), 26, 64)
    assert np.array_equal(host(z0), t0) and np.array_equal(host(z1), t1)


# ---- the largest batch one call takes in this suite: n > 2^31 -------------------------------

@pytest.mark.parametrize("fn", ["drelu", "relu"])
def test_max_size_over_2pow31_sampled(api, fn):
    """n = 2^31 + 13 elements in one call (64 GiB of shares and outputs): no
    32-bit index or size overflow anywhere on the path.  Oracle parity on a
    seeded sample that includes the first and last groups and the 2^31 and
    2^32-element boundaries of the byte offsets."""
    if torch.cuda.get_device_properties(0).total_memory < (96 << 30):
        pytest.skip("needs > 96 GiB of device memory")
    n = (1 << 31) + 13
    g = torch.Generator(device=DEV).manual_seed(2024)
    x0 = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), dtype=torch.int64, device=DEV, generator=g)
    x1 = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), dtype=torch.int64, device=DEV, generator=g)
    kw = PARAMS[0]
    y0, y1 = getattr(api, fn)(x0, x1, api.Params(**kw), SEEDS)
    rng = np.random.default_rng(17)
    idx = np.unique(np.concatenate([np.arange(16), n - 1 - np.arange(16), (1 << 28) + np.arange(-8, 8),
                                    (1 << 29) + np.arange(-8, 8), (1 << 31) + np.arange(-8, 8),
                                    rng.choice(n, 4096, replace=False)]))
    ti = torch.from_numpy(idx.astype(np.int64)).to(DEV)
    s0, s1 = host(x0[ti]), host(x1[ti])
    g0, g1 = host(y0[ti]), host(y1[ti])
    del x0, x1, y0, y1
    torch.cuda.empty_cache()
    ref = getattr(B, fn)(B.Params(**kw), s0, s1, idx.astype(np.uint64), SEEDS)
    assert np.array_equal(g0, ref["y0"]) and np.array_equal(g1, ref["y1"])
