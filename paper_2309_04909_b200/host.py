"""Host-buffer execution of the fused path: pinned host shares in, pinned host
shares out, with H2D copy / fused kernel / D2H copy pipelined in chunks over
two CUDA streams so the PCIe transfers overlap each other and the kernels.

This is the public entry point a user with host-resident shares calls; the
compute is the same C-ABI kernel (api.drelu / api.relu) on device chunks.
"""
from __future__ import annotations

import torch

from . import api


class HostPipeline:
    def __init__(self, n: int, device, chunks: int = 8, streams: int = 2):
        self.n = n
        self.dev = torch.device(device)
        self.chunks = max(1, chunks)
        per = -(-n // self.chunks)
        self.csize = max(8, -(-per // 8) * 8)  # chunk offsets stay multiples of 8 (elem_base rule)
        self.streams = [torch.cuda.Stream(device=self.dev) for _ in range(streams)]
        self.bufs = [[torch.empty(self.csize, dtype=torch.int64, device=self.dev) for _ in range(4)]
                     for _ in range(streams)]

    def _run(self, fn, hx0, hx1, hy0, hy1, prm, seeds, base):
        for t in (hx0, hx1, hy0, hy1):
            if t.is_cuda or not t.is_pinned():
                raise api.BicoptorError("HostPipeline expects pinned host tensors")
        cur = torch.cuda.current_stream(self.dev)
        for s in self.streams:
            s.wait_stream(cur)
        c = 0
        for a in range(0, self.n, self.csize):
            b = min(self.n, a + self.csize)
            m = b - a
            s = self.streams[c % len(self.streams)]
            x0, x1, y0, y1 = self.bufs[c % len(self.streams)]
            with torch.cuda.stream(s):
                x0[:m].copy_(hx0[a:b], non_blocking=True)
                x1[:m].copy_(hx1[a:b], non_blocking=True)
                fn(x0[:m], x1[:m], prm, seeds, base + a, y0[:m], y1[:m], stream=s)
                hy0[a:b].copy_(y0[:m], non_blocking=True)
                hy1[a:b].copy_(y1[:m], non_blocking=True)
            c += 1
        for s in self.streams:
            cur.wait_stream(s)
        return hy0, hy1

    def drelu(self, hx0, hx1, hy0, hy1, prm, seeds, base: int = 0):
        return self._run(api.drelu, hx0, hx1, hy0, hy1, prm, seeds, base)

    def relu(self, hx0, hx1, hy0, hy1, prm, seeds, base: int = 0):
        return self._run(api.relu, hx0, hx1, hy0, hy1, prm, seeds, base)
