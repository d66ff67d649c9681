"""Host-buffer execution of the fused path (the end-to-end entry a user with
host-resident shares calls): a thin owner of the device workspace around the
native pipeline bc_drelu_host / bc_relu_host (csrc/bc_hostpipe.cu), which
overlaps the H2D copy, the fused kernel and the D2H copy chunk by chunk.
"""
from __future__ import annotations

import torch

from . import api


class HostPipeline:
    def __init__(self, device, chunk: int = 1 << 20):
        if chunk <= 0 or chunk % 8:
            raise api.BicoptorError("chunk must be a positive multiple of 8")
        self.dev = torch.device(device)
        self.chunk = chunk
        self.ws = api.host_workspace(chunk, self.dev)

    @staticmethod
    def _pinned(*ts):
        for t in ts:
            if t.is_cuda or not t.is_pinned():
                raise api.BicoptorError("HostPipeline expects pinned host tensors")

    def drelu(self, hx0, hx1, hy0, hy1, prm, seeds, base: int = 0, sync: bool = True):
        """sync=False enqueues only (a serving loop: consecutive requests pipeline into
        each other); torch.cuda.synchronize(device) then completes the host outputs."""
        self._pinned(hx0, hx1, hy0, hy1)
        with torch.cuda.device(self.dev):
            return api.drelu_host(hx0, hx1, hy0, hy1, prm, seeds, self.ws, self.chunk, base, sync=sync)

    def relu(self, hx0, hx1, hy0, hy1, prm, seeds, base: int = 0, sync: bool = True):
        self._pinned(hx0, hx1, hy0, hy1)
        with torch.cuda.device(self.dev):
            return api.relu_host(hx0, hx1, hy0, hy1, prm, seeds, self.ws, self.chunk, base, sync=sync)
