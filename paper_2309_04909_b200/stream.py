"""Config 5: an E2E-shaped stream of ReLU layers (BASELINE.json configs[4]).

The ReLU layers of the paper's inference networks (Table 7), one
fused bc_relu launch per layer in sequence, captured once into a CUDA graph
so small layers pay no launch overhead.  Each layer's elements get a distinct
global index range (elem_base = running count), so every PRG draw is fresh.

Per-image ReLU counts (activation sizes; the paper does not print the layer
shapes -- conv shapes are the standard networks at the dataset's input size,
FC widths assumed):
  CIFAR10_VGG16   (32x32)  conv 2x65536, 2x32768, 3x16384, 3x8192, 3x2048; FC 2x256
  Tiny_VGG16      (64x64)  conv 2x262144, 2x131072, 3x65536, 3x32768, 3x8192; FC 2x512
  CIFAR10_AlexNet (32x32)  11616, 2304, 2x384, 3x256
Batches are the paper's (Table 7: 240, 60, 1650).
"""
from __future__ import annotations

import torch

from . import api

NETWORKS = {
    "CIFAR10_VGG16": (240, [65536] * 2 + [32768] * 2 + [16384] * 3 + [8192] * 3 + [2048] * 3 + [256] * 2),
    "Tiny_VGG16": (60, [262144] * 2 + [131072] * 2 + [65536] * 3 + [32768] * 3 + [8192] * 3 + [512] * 2),
    "CIFAR10_AlexNet": (1650, [11616, 2304, 384, 384, 256, 256, 256]),
}


def index_span(sizes) -> int:
    """Global element indices one forward over `sizes` occupies (layers padded to 8)."""
    return sum(-(-n // 8) * 8 for n in sizes)


def layer_sizes(name: str, batch: int | None = None):
    b, per_img = NETWORKS[name]
    b = b if batch is None else batch
    return [b * k for k in per_img]


class ReluStream:
    """Device buffers for every layer plus a captured CUDA graph of the layer sequence."""

    def __init__(self, sizes, prm: api.Params, seeds, device, base: int = 0):
        self.sizes = list(sizes)
        self.prm, self.seeds = prm, seeds
        self.dev = torch.device(device)
        self._set_bases(base)
        self.x0 = [torch.empty(n, dtype=torch.int64, device=self.dev) for n in self.sizes]
        self.x1 = [torch.empty(n, dtype=torch.int64, device=self.dev) for n in self.sizes]
        self.y0 = [torch.empty(n, dtype=torch.int64, device=self.dev) for n in self.sizes]
        self.y1 = [torch.empty(n, dtype=torch.int64, device=self.dev) for n in self.sizes]
        self.graph = None

    def _set_bases(self, base: int):
        self.base = base
        self.bases = []
        b = base
        for n in self.sizes:
            self.bases.append(b)
            b += -(-n // 8) * 8  # layer offsets stay multiples of 8 (elem_base rule)

    def advance(self, base: int | None = None):
        """Move the forward to a fresh global index range (default: the next one) and re-capture.
        replay() re-executes the captured protocol instance -- the same t, Pi, r_m, rho_m and
        triples -- which is only sound on the SAME inputs (a timing loop).  Before running on
        new inputs, call advance(): reusing the draws on new shares would open x - x' to P0/P1
        (d = x - a, Alg 8) and give P2 two messages under one mask (Alg 7 steps 7-8)."""
        self._set_bases(self.base + index_span(self.sizes) if base is None else base)
        if self.graph is not None:
            self.capture()
        return self

    @property
    def total(self) -> int:
        return sum(self.sizes)

    def _launch_all(self, stream):
        for i in range(len(self.sizes)):
            api.relu(self.x0[i], self.x1[i], self.prm, self.seeds, self.bases[i], self.y0[i], self.y1[i],
                     stream=stream)

    def run_eager(self):
        self._launch_all(torch.cuda.current_stream(self.dev))

    def capture(self):
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self._launch_all(s)  # warm-up outside capture (grid sizes cached)
        torch.cuda.current_stream(self.dev).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=s):
            self._launch_all(s)
        return self

    def replay(self):
        self.graph.replay()
