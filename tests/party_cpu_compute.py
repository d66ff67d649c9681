"""A CPU implementation of the party-phase interface of
paper_2309_04909_b200.party.CudaCompute, built on the oracle.  TEST ONLY: it
lets the party runtime's transport logic (chunking, message order, roles) run
under the gloo backend on machines without GPUs."""
import numpy as np
import torch

from oracle import bicoptor as B


def _np(t):
    return t.numpy().view(np.uint64) if t.dtype == torch.int64 else t.numpy()


def _t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64))


def _prm(p):
    return B.Params(ell=p.ell, lx=p.lx, f=p.f, mode=p.mode, rounds=p.rounds)


def _j(base, n):
    return np.arange(n, dtype=np.uint64) + np.uint64(base)


def _pack_bits(t):
    n = t.size
    out = np.zeros((n + 7) // 8, dtype=np.uint8)
    for i in range(n):
        out[i // 8] |= np.uint8(int(t[i]) << (i % 8))
    return out


def _unpack_bits(b, n):
    return np.array([(int(b[i // 8]) >> (i % 8)) & 1 for i in range(n)], dtype=np.uint64)


def _decode_msg(lo, hi, S):
    """Inverse of B.encode_msg (byte planes, (n, 8)) / B.encode_msg_large (slot-major
    uint32 planes, (S, n))."""
    lo = np.asarray(lo)
    bit = np.uint64(8 if lo.dtype.itemsize == 1 else 32)
    W = (lo[:, :S] if bit == 8 else lo.view(np.uint32).T).astype(np.uint64)
    if hi is not None:
        h = np.asarray(hi).view(np.uint8 if bit == 8 else np.uint32).astype(np.uint64)
        W |= ((h[:, None] >> np.arange(S, dtype=np.uint64)) & np.uint64(1)) << bit
    return W


def _encode(o, W):
    if o.layout == "large":
        lo, hi = B.encode_msg_large(W)
        return torch.from_numpy(lo.view(np.int32)), torch.from_numpy(hi.view(np.int32))
    lo, hi = B.encode_msg(W)
    return torch.from_numpy(lo), torch.from_numpy(hi)


class OracleCompute:
    def __init__(self):
        self.device = torch.device("cpu")

    def empty(self, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    def drelu_send(self, party, x, prm, seed01, base):
        o = _prm(prm)
        m = B.drelu_send(o, party, _np(x), _j(base, x.numel()), seed01)
        lo, hi = _encode(o, m["W"])
        return lo, hi, torch.from_numpy(_pack_bits(m["t"]))

    def drelu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, base, paper_literal=False):
        o = _prm(prm)
        W0 = _decode_msg(_np(lo0), None if hi0 is None else _np(hi0), o.slots)
        W1 = _decode_msg(_np(lo1), None if hi1 is None else _np(hi1), o.slots)
        n = W0.shape[0]
        h = B.drelu_helper(o, W0, W1, _j(base, n), seed02)
        return (_t64(h["D0"]) if paper_literal else None), _t64(h["D1"])

    def drelu_finish(self, party, tb, resp, prm, n, seed02, base, out):
        o = _prm(prm)
        t = _unpack_bits(_np(tb), n)
        if resp is None:
            from oracle.chacha import element_u64
            D = element_u64(seed02, B.L_RESP, o.rounds, _j(base, n), 1)[:, 0] & np.uint64((1 << o.ell) - 1)
        else:
            D = _np(resp)
        out.copy_(_t64(B.drelu_finish(o, party, t, D)))
        return out

    def relu_send(self, party, x, prm, seed01, seed_tr, base):
        o = _prm(prm)
        m = B.relu_send(o, party, _np(x), _j(base, x.numel()), seed01, seed_tr)
        lo, hi = _encode(o, m["W"])
        return lo, hi, torch.from_numpy(_pack_bits(m["t"])), _t64(m["d"])

    def relu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, seed12, base):
        o = _prm(prm)
        W0 = _decode_msg(_np(lo0), None if hi0 is None else _np(hi0), o.slots)
        W1 = _decode_msg(_np(lo1), None if hi1 is None else _np(hi1), o.slots)
        n = W0.shape[0]
        h = B.relu_helper(o, W0, W1, _j(base, n), seed02, seed12)
        return _t64(h["e"]), _t64(h["c1"])

    def relu_finish(self, party, x, tb, d_own, d_peer, e, c1, prm, seed_tr, base, out):
        o = _prm(prm)
        n = x.numel()
        t = _unpack_bits(_np(tb), n)
        y = B.relu_finish(o, party, _np(x), t, _np(d_own), _np(d_peer), _np(e),
                          None if c1 is None else _np(c1), _j(base, n), seed_tr)
        out.copy_(_t64(y))
        return out
