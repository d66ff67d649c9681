"""Out-of-bounds writes, found without compute-sanitizer (closed on this GPU pool): every
output buffer of the C-ABI calls is a view into a larger allocation whose guard bands
before and after it hold a canary pattern; after each call (ragged n: 1, 7, 9, 1003 —
partial groups, one group plus a tail, several CTAs) the bands must be untouched and
the inputs unchanged.  Outputs are also checked against the oracle where they are
results (the parity tests cover that at larger sizes)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import synth  # noqa: E402

PAD = 256  # bytes of canary on each side (16-B aligned views)
CANARY = 0xA5


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_04909_b200 import api
    return api


class Banded:
    """A tensor of `shape` / `dtype` inside a byte buffer with PAD canary bytes on each side."""

    def __init__(self, shape, dtype, dev="cuda:0"):
        item = torch.empty((), dtype=dtype).element_size()
        self.nbytes = int(np.prod(shape)) * item
        self.raw = torch.full((PAD + self.nbytes + PAD,), CANARY, dtype=torch.uint8, device=dev)
        self.t = self.raw[PAD:PAD + self.nbytes].view(dtype).view(shape)

    def intact(self) -> bool:
        r = self.raw.cpu().numpy()
        return bool((r[:PAD] == CANARY).all() and (r[PAD + self.nbytes:] == CANARY).all())


def _u64(a, dev="cuda:0"):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


PARAMS = [
    dict(ell=64, lx=7, f=24, mode="guard", rounds=8),     # compact tape, table kernel (the bench's)
    dict(ell=64, lx=7, f=24, mode="literal", rounds=8),   # paper-literal table kernel
    dict(ell=32, lx=5, f=3, mode="guard", rounds=8),      # pair tape, generic kernel
    dict(ell=16, lx=7, f=0, mode="guard", rounds=8),      # compact tape, ell < 64
    dict(ell=64, lx=31, f=0, mode="guard", rounds=8),     # large tape (full precision)
]
NS = (1, 7, 9, 1003)


@pytest.mark.parametrize("kw", PARAMS, ids=lambda k: f"l{k['ell']}x{k['lx']}f{k['f']}{k['mode'][0]}")
@pytest.mark.parametrize("n", NS)
def test_fused_outputs_stay_in_bounds(kw, n):
    api = _need_gpu()
    from oracle import bicoptor as B
    prm, oprm = api.Params(**kw), B.Params(**kw)
    sd = synth.seeds(3)
    x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1", run=n)
    a0, a1 = _u64(x0), _u64(x1)
    j = np.arange(n, dtype=np.uint64) + np.uint64(8)
    for fn, ofn in ((api.drelu, B.drelu), (api.relu, B.relu)):
        y0, y1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
        tr_shape = api.transcript_buffers(1, "cuda:0", prm)
        tr = {k: Banded((n,) + tuple(v.shape[1:]), v.dtype) for k, v in tr_shape.items()}
        fn(a0, a1, prm, sd, 8, y0=y0.t, y1=y1.t, transcript={k: b.t for k, b in tr.items()})
        torch.cuda.synchronize()
        for b in [y0, y1] + list(tr.values()):
            assert b.intact(), fn.__name__
        ref = ofn(oprm, x0, x1, j, sd)
        assert np.array_equal(y0.t.cpu().numpy().view(np.uint64), ref["y0"])
        assert np.array_equal(y1.t.cpu().numpy().view(np.uint64), ref["y1"])
        # the same without a transcript (the bench's instantiation)
        z0, z1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
        fn(a0, a1, prm, sd, 8, y0=z0.t, y1=z1.t)
        torch.cuda.synchronize()
        assert z0.intact() and z1.intact(), fn.__name__
        assert torch.equal(z0.t, y0.t) and torch.equal(z1.t, y1.t)
    assert np.array_equal(a0.cpu().numpy().view(np.uint64), x0)  # inputs untouched
    assert np.array_equal(a1.cpu().numpy().view(np.uint64), x1)


@pytest.mark.parametrize("kw", PARAMS[:3] + PARAMS[4:], ids=lambda k: f"l{k['ell']}x{k['lx']}f{k['f']}{k['mode'][0]}")
@pytest.mark.parametrize("n", NS)
def test_party_phase_outputs_stay_in_bounds(kw, n):
    """bc_drelu_send / helper / finish and bc_relu_send / helper / finish into banded buffers;
    the chained result equals the fused kernel's."""
    api = _need_gpu()
    prm = api.Params(**kw)
    sd = synth.seeds(4)
    x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D2", run=n + 1)
    a0, a1 = _u64(x0), _u64(x1)
    base = 16
    lo_s, hi_s, tb_s = api.msg_buffers(1, "cuda:0", prm)
    slot_major = api.wire_format(prm)["slot_major"]

    def msg():
        lo = Banded(((lo_s.shape[0], n) if slot_major else (n,) + tuple(lo_s.shape[1:])), lo_s.dtype)
        hi = Banded((n,), hi_s.dtype)
        tb = Banded(((n + 7) // 8,), torch.uint8)
        return lo, hi, tb

    bands = []
    m0, m1 = msg(), msg()
    bands += list(m0) + list(m1)
    api.drelu_send(0, a0, prm, sd.s01, base, out=tuple(b.t for b in m0))
    api.drelu_send(1, a1, prm, sd.s01, base, out=tuple(b.t for b in m1))
    r0, r1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
    bands += [r0, r1]
    api.drelu_helper(m0[0].t, m0[1].t, m1[0].t, m1[1].t, prm, sd.s02, base, paper_literal=True, out=(r0.t, r1.t))
    y0, y1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
    bands += [y0, y1]
    api.drelu_finish(0, m0[2].t, r0.t, prm, n, None, base, out=y0.t)
    api.drelu_finish(1, m1[2].t, r1.t, prm, n, None, base, out=y1.t)
    torch.cuda.synchronize()
    assert all(b.intact() for b in bands), "drelu phases"
    f0, f1 = api.drelu(a0, a1, prm, sd, base)
    assert torch.equal((y0.t + y1.t), (f0 + f1))

    bands = []
    m0, m1 = msg(), msg()
    d0, d1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
    bands += list(m0) + list(m1) + [d0, d1]
    api.relu_send(0, a0, prm, sd.s01, sd.s02, base, out=tuple(b.t for b in m0) + (d0.t,))
    api.relu_send(1, a1, prm, sd.s01, sd.s12, base, out=tuple(b.t for b in m1) + (d1.t,))
    e, c1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
    bands += [e, c1]
    api.relu_helper(m0[0].t, m0[1].t, m1[0].t, m1[1].t, prm, sd.s02, sd.s12, base, out=(e.t, c1.t))
    y0, y1 = Banded((n,), torch.int64), Banded((n,), torch.int64)
    bands += [y0, y1]
    api.relu_finish(0, a0, m0[2].t, d0.t, d1.t, e.t, None, prm, sd.s02, base, out=y0.t)
    api.relu_finish(1, a1, m1[2].t, d1.t, d0.t, e.t, c1.t, prm, sd.s12, base, out=y1.t)
    torch.cuda.synchronize()
    assert all(b.intact() for b in bands), "relu phases"
    f0, f1 = api.relu(a0, a1, prm, sd, base)
    assert torch.equal(y0.t, f0) and torch.equal(y1.t, f1)


@pytest.mark.parametrize("n", NS)
def test_elementwise_and_rss_outputs_stay_in_bounds(n):
    """Alg 4/5/6 primitives, the ladder, the RSS variant and the truncation-study kernels."""
    api = _need_gpu()
    prm = api.Params(ell=64, lx=7, f=24, mode="guard", rounds=8)
    big = api.Params(ell=64, lx=31, f=0, mode="guard", rounds=8)
    sd = synth.seeds(5)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=n + 2)
    a0, a1 = _u64(x0), _u64(x1)
    bands = []

    def out(shape, dtype=torch.int64):
        b = Banded(shape, dtype)
        bands.append(b)
        return b.t

    api.trc(0, a0, 64, 3, 1, out=out((n,)))
    api.trc_prob(1, a1, 64, 5, out=out((n,)))
    api.modswitch(0, a0, 7, 131, out=out((n,), torch.int32))
    api.modswitch64(1, a1, 32, (1 << 32) + 15, out=out((n,)))
    api.ladder_modswitch(0, a0, prm, out=out((n, 8), torch.uint8))
    api.ladder_modswitch64(1, a1, big, out=out((n, 32)))
    x2 = _u64(np.zeros(n, dtype=np.uint64))
    api.drelu_rss(a0, a1, x2, prm, sd, 8, out=(out((n,)), out((n,)), out((n,))))
    api.relu_rss(a0, a1, x2, prm, sd, 8, out=(out((n,)), out((n,)), out((n,))))
    api.trc_aby3(a0, a1, 64, 24, sd, 8, out=(out((n,)), out((n,))))
    api.drelu_b1(a0, a1, prm, sd, 8, y0=out((n,)), y1=out((n,)))
    torch.cuda.synchronize()
    for i, b in enumerate(bands):
        assert b.intact(), i


@pytest.mark.parametrize("n,chunk", [(1, 8), (9, 8), (1003, 64), (5000, 1024)])
def test_host_entries_stay_in_bounds(n, chunk):
    """bc_drelu_host / bc_relu_host (synchronous and async): pinned host inputs and outputs
    inside canary bands, chunked H2D / kernel / D2H with a ragged last chunk; the bands of the
    host outputs and of the device workspace stay intact and the results equal the fused call."""
    api = _need_gpu()
    prm = api.Params(ell=64, lx=7, f=24, mode="guard", rounds=8)
    sd = synth.seeds(6)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D2", run=n + 3)

    def hband(vals=None):
        raw = torch.full((PAD + 8 * n + PAD,), CANARY, dtype=torch.uint8).pin_memory()
        t = raw[PAD:PAD + 8 * n].view(torch.int64)
        if vals is not None:
            t.copy_(torch.from_numpy(np.ascontiguousarray(vals).view(np.int64)))
        return raw, t

    def intact(raw):
        r = raw.numpy()
        return bool((r[:PAD] == CANARY).all() and (r[PAD + 8 * n:] == CANARY).all())

    wsb = api.lib().bc_host_workspace_bytes(chunk)
    ws = Banded((wsb // 8,), torch.int64)
    for fn, host_fn in ((api.drelu, api.drelu_host), (api.relu, api.relu_host)):
        f0, f1 = fn(_u64(x0), _u64(x1), prm, sd, 8)
        for sync in (True, False):
            (rx0, hx0), (rx1, hx1) = hband(x0), hband(x1)
            (ry0, hy0), (ry1, hy1) = hband(), hband()
            host_fn(hx0, hx1, hy0, hy1, prm, sd, ws.t, chunk, 8, sync=sync)
            torch.cuda.synchronize()
            assert all(intact(r) for r in (rx0, rx1, ry0, ry1)) and ws.intact(), (fn.__name__, sync)
            assert torch.equal(hy0, f0.cpu()) and torch.equal(hy1, f1.cpu()), (fn.__name__, sync)
            assert np.array_equal(hx0.numpy().view(np.uint64), x0)
