"""TEST ONLY: a CPU stand-in for peer.CudaIpcBackend and for the api phase
kernels, so the peer-memory transport's host logic (rings, doorbells, credits,
roles, chunking) runs under gloo on machines without GPUs.

FileBackend: every inbox is a file-backed shared mapping (np.memmap, MAP_SHARED)
in a directory all ranks see; "exporting" an inbox is naming its file, and a
producer's writes land in the consumer's pages directly, as the kernels' peer
stores do.  Events are no-ops: the CPU compute below is synchronous.
OracleApiCompute: the api phase signatures (out=, d_peer=, e_dup=) over the
oracle-based OracleCompute."""
import os

import numpy as np
import torch

from party_cpu_compute import OracleCompute

_NP = {torch.uint8: np.uint8, torch.int32: np.int32, torch.int64: np.int64}


class FileBackend:
    def __init__(self, root, rank):
        self.root, self.rank, self.k = root, rank, 0
        self._names = {}

    def alloc(self, shape, dtype):
        path = os.path.join(self.root, f"r{self.rank}_{self.k}.bin")
        self.k += 1
        t = torch.from_numpy(np.memmap(path, mode="w+", dtype=_NP[dtype], shape=tuple(shape)))
        self._names[t.data_ptr()] = (path, tuple(shape), _NP[dtype])
        return t

    alloc_inbox = alloc  # every file is its own mapping already

    def export(self, t):
        return self._names[t.data_ptr()]

    @staticmethod
    def open(blob):
        path, shape, dt = blob
        return torch.from_numpy(np.memmap(path, mode="r+", dtype=dt, shape=shape))

    @staticmethod
    def new_event():
        return None

    @staticmethod
    def export_event(ev):
        return None

    @staticmethod
    def open_event(h):
        return None

    @staticmethod
    def record(ev):
        pass

    @staticmethod
    def wait(ev):
        pass

    def close(self):
        pass


class OracleApiCompute(OracleCompute):
    def drelu_send(self, party, x, prm, seed01, base, out, y=None, seed02=None):
        lo, hi, tb = super().drelu_send(party, x, prm, seed01, base)
        out[0].copy_(lo)
        out[1].copy_(hi)
        if out[2] is not None:
            out[2].copy_(tb)
        if y is not None:  # bc_drelu_send_p0: P0's output share in the same call
            self.drelu_finish(0, tb, None, prm, x.numel(), seed02, base, y)
        return out

    def drelu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, base, paper_literal=False, out=None):
        r0, r1 = super().drelu_helper(lo0, hi0, lo1, hi1, prm, seed02, base, paper_literal=paper_literal)
        if paper_literal:
            out[0].copy_(r0)
        out[1].copy_(r1)
        return out

    def relu_send(self, party, x, prm, seed01, seed_tr, base, out, d_peer=None):
        lo, hi, tb, d = super().relu_send(party, x, prm, seed01, seed_tr, base)
        for dst, src in zip(out, (lo, hi, tb, d)):
            dst.copy_(src)
        if d_peer is not None:
            d_peer.copy_(d)
        return out

    def relu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, seed12, base, out, e_dup=None):
        e, c1 = super().relu_helper(lo0, hi0, lo1, hi1, prm, seed02, seed12, base)
        out[0].copy_(e)
        if out[1] is not None:
            out[1].copy_(c1)
        if e_dup is not None:
            e_dup.copy_(e)
        return out
