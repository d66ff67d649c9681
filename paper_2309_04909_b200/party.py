"""Party-separated execution of Alg 7 / Alg 8: P0, P1, P2 in separate processes
(one GPU each), messages over torch.distributed point-to-point (NCCL over
NVLink on a GPU box).

Roles: in a world of 3k ranks, rank r plays party r % 3 of triple r // 3; each
triple owns its own element range (global index offset = triple * n), so k
triples shard the batch with no cross-triple traffic.

Messages per element (guard mode), Alg 7 / Alg 8:

    DReLU  P0 -> P2  lo 8 B + hi 1 B          P1 -> P2  lo 8 B + hi 1 B
           P2 -> P1  [D']_1 8 B               (P2 -> P0 [D']_0 8 B only if paper_literal;
                                               otherwise P0 derives it from seed02, reading C12)
    ReLU   P0 -> P2, P1 -> P2 as above        P0 <-> P1  [d]_b 8 B each way
           P2 -> P0, P1  e 8 B                P2 -> P1  [c]_1 8 B (preprocessing, reading C20)

The batch is processed in chunks.  Each protocol round of a chunk is one
batch_isend_irecv group; the round-2 receives of chunk k stay in flight while
chunk k+1's local phase runs (with NCCL the waits are stream-ordered, the host
does not block).

`compute` is the phase implementation: by default the CUDA kernels of
`api` (bc_*_send/helper/finish).  Tests substitute a CPU implementation to
exercise this transport logic with the gloo backend on machines without GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import api


@dataclass
class Role:
    party: int      # 0, 1 (computing parties) or 2 (helper)
    triple: int     # which P0/P1/P2 triple this rank belongs to
    peers: tuple    # global ranks of (P0, P1, P2) of this triple

    @staticmethod
    def of(rank: int) -> "Role":
        t = rank // 3
        return Role(rank % 3, t, (3 * t, 3 * t + 1, 3 * t + 2))


class CudaCompute:
    """The product phase implementation: libbicoptor kernels on this rank's GPU."""

    def __init__(self, device):
        self.device = torch.device(device)
        api.lib()

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    drelu_send = staticmethod(api.drelu_send)
    drelu_helper = staticmethod(api.drelu_helper)
    drelu_finish = staticmethod(api.drelu_finish)
    relu_send = staticmethod(api.relu_send)
    relu_helper = staticmethod(api.relu_helper)
    relu_finish = staticmethod(api.relu_finish)


class StagedCudaCompute:
    """The libbicoptor phase kernels with host-resident messages: every phase
    copies its inputs to this rank's GPU, runs the kernel there and returns host
    tensors, so the messages can travel over a host transport (gloo over TCP:
    parties on separate machines, the paper's LAN / WAN setting).
    With NCCL use CudaCompute: the messages then stay in device memory."""

    def __init__(self, device):
        self.device = torch.device(device)
        api.lib()

    @staticmethod
    def empty(shape, dtype):
        return torch.empty(shape, dtype=dtype)

    def _d(self, t):
        return None if t is None else t.to(self.device, non_blocking=False)

    @staticmethod
    def _h(*ts):
        out = tuple(None if t is None else t.cpu() for t in ts)
        return out if len(out) > 1 else out[0]

    def drelu_send(self, party, x, prm, seed01, base):
        return self._h(*api.drelu_send(party, self._d(x), prm, seed01, base))

    def drelu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, base, paper_literal=False):
        return self._h(*api.drelu_helper(self._d(lo0), self._d(hi0), self._d(lo1), self._d(hi1), prm, seed02, base,
                                         paper_literal=paper_literal))

    def drelu_finish(self, party, tbits, resp, prm, n, seed02, base, out):
        out.copy_(api.drelu_finish(party, self._d(tbits), self._d(resp), prm, n, seed02, base).cpu())
        return out

    def relu_send(self, party, x, prm, seed01, seed_tr, base):
        return self._h(*api.relu_send(party, self._d(x), prm, seed01, seed_tr, base))

    def relu_helper(self, lo0, hi0, lo1, hi1, prm, seed02, seed12, base):
        return self._h(*api.relu_helper(self._d(lo0), self._d(hi0), self._d(lo1), self._d(hi1), prm, seed02, seed12,
                                        base))

    def relu_finish(self, party, x, tbits, d_own, d_peer, e, c1, prm, seed_tr, base, out):
        out.copy_(api.relu_finish(party, self._d(x), self._d(tbits), self._d(d_own), self._d(d_peer), self._d(e),
                                  self._d(c1), prm, seed_tr, base).cpu())
        return out


def _chunks(n: int, chunk: int):
    chunk = max(8, (chunk // 8) * 8)  # chunk offsets stay multiples of 8 (elem_base rule)
    return [(a, min(n, a + chunk)) for a in range(0, n, chunk)]


class PartyRunner:
    """Runs DReLU / ReLU for this rank's role over a batch of n elements."""

    def __init__(self, prm: api.Params, seeds, n: int, chunk: int = 1 << 22, compute=None,
                 group=None, paper_literal: bool = False, base: int | None = None, triples: int = 1):
        self.rank = dist.get_rank()
        self.role = Role.of(self.rank)
        self.prm = prm
        self.n = n
        self.chunks = _chunks(n, chunk)
        self.c = compute
        self.group = group
        self.paper_literal = paper_literal
        # run r draws from [base0 + r * triples * n, + n): fresh randomness per run (as peer.PeerPartyRunner)
        span = -(-n // 8) * 8  # index ranges start at multiples of 8 (the elem_base rule)
        self.base0 = self.role.triple * span if base is None else base
        self.stride = triples * span
        self.runs = 0
        self.base = self.base0
        self.fmt = api.wire_format(prm)  # byte planes (p <= 257) or uint32 planes (large tape)
        self.hi_needed = self.fmt["hi"] is not None
        # seeds this party holds: P0 {01, 02}, P1 {01, 12}, P2 {02, 12}
        held = {0: ("s01", "s02"), 1: ("s01", "s12"), 2: ("s02", "s12")}[self.role.party]
        self.seed = {k: getattr(seeds, k) for k in held}
        self.bytes_sent = 0

    # -- messaging helpers ---------------------------------------------------------
    def _msg_bufs(self, m):
        """P2's receive buffers for one chunk: lo0, hi0, lo1, hi1 (hi None if unused)."""
        (los, lot), hf = self.fmt["lo"], self.fmt["hi"]
        shape = (los[0], m) if self.fmt["slot_major"] else (m,) + los
        lo0, lo1 = self.c.empty(shape, lot), self.c.empty(shape, lot)
        hi0 = self.c.empty(m, hf[1]) if hf else None
        hi1 = self.c.empty(m, hf[1]) if hf else None
        return lo0, hi0, lo1, hi1

    # Each protocol round of a chunk is posted as one batch_isend_irecv group
    # (one NCCL group call on GPUs), so the order in which the three parties
    # post their sends and receives cannot deadlock.
    def _send(self, t, dst):
        self.bytes_sent += t.numel() * t.element_size()
        return dist.P2POp(dist.isend, t, self.role.peers[dst], group=self.group)

    def _recv(self, t, src):
        return dist.P2POp(dist.irecv, t, self.role.peers[src], group=self.group)

    @staticmethod
    def _post(ops):
        return dist.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def _wait(works):
        for w in works:
            w.wait()

    # -- DReLU (Alg 7) -----------------------------------------------------------------
    def _next_run(self, elem_base):
        self.base = self.base0 + self.runs * self.stride if elem_base is None else elem_base
        self.runs += 1

    def drelu(self, x=None, elem_base: int | None = None):
        """P0/P1: x is this party's share vector; returns its DReLU share.  P2: x=None, returns None.
        Run r uses the global indices base0 + r * stride + [0, n) unless elem_base is given."""
        self._next_run(elem_base)
        p, c = self.role.party, self.c
        out = c.empty(self.n, torch.int64) if p < 2 else None
        pending = []  # (chunk, state, works) whose round-2 messages are outstanding
        for (a, b) in self.chunks:
            m, base = b - a, self.base + a
            if p < 2:
                lo, hi, tb = c.drelu_send(p, x[a:b], self.prm, self.seed["s01"], base)   # steps 1-8
                ops = [self._send(lo, 2)] + ([self._send(hi, 2)] if self.hi_needed else [])
                works = self._post(ops)                                                  # round 1
                resp = None
                if p == 1 or self.paper_literal:
                    resp = c.empty(m, torch.int64)
                    works += self._post([self._recv(resp, 2)])                           # round 2
                pending.append(((a, b), (tb, resp), works))
            else:
                lo0, hi0, lo1, hi1 = self._msg_bufs(m)
                ops = [self._recv(lo0, 0), self._recv(lo1, 1)]
                if self.hi_needed:
                    ops += [self._recv(hi0, 0), self._recv(hi1, 1)]
                self._wait(self._post(ops))
                r0, r1 = c.drelu_helper(lo0, hi0, lo1, hi1, self.prm, self.seed["s02"], base,
                                        paper_literal=self.paper_literal)                 # steps 9-10
                ops = [self._send(r1, 1)] + ([self._send(r0, 0)] if self.paper_literal else [])
                pending.append(((a, b), None, self._post(ops)))
            if len(pending) > 1:
                self._drelu_finish(*pending.pop(0), out)
        while pending:
            self._drelu_finish(*pending.pop(0), out)
        return out

    def _drelu_finish(self, rng, state, works, out):
        self._wait(works)
        if state is None:
            return
        (a, b), (tb, resp) = rng, state
        seed02 = self.seed.get("s02") if resp is None else None
        self.c.drelu_finish(self.role.party, tb, resp, self.prm, b - a, seed02, self.base + a, out=out[a:b])  # step 11

    # -- ReLU (Alg 8) ------------------------------------------------------------------
    def relu(self, x=None, with_c1: bool = True, elem_base: int | None = None):
        self._next_run(elem_base)
        p, c = self.role.party, self.c
        out = c.empty(self.n, torch.int64) if p < 2 else None
        pending = []
        for (a, b) in self.chunks:
            m, base = b - a, self.base + a
            if p < 2:
                seed_tr = self.seed["s02"] if p == 0 else self.seed["s12"]
                lo, hi, tb, d_own = c.relu_send(p, x[a:b], self.prm, self.seed["s01"], seed_tr, base)  # steps 1, 4
                d_peer = c.empty(m, torch.int64)
                e = c.empty(m, torch.int64)
                c1 = c.empty(m, torch.int64) if p == 1 else None
                # round 1: the message to P2 and the opening of d between P0 and P1
                ops = [self._send(lo, 2)] + ([self._send(hi, 2)] if self.hi_needed else [])
                ops += [self._send(d_own, 1 - p), self._recv(d_peer, 1 - p)]
                works = self._post(ops)
                # round 2: e (and [c]_1 for P1) from P2
                works += self._post([self._recv(e, 2)] + ([self._recv(c1, 2)] if p == 1 else []))
                pending.append(((a, b), (x[a:b], tb, d_own, d_peer, e, c1, seed_tr), works))
            else:
                lo0, hi0, lo1, hi1 = self._msg_bufs(m)
                ops = [self._recv(lo0, 0), self._recv(lo1, 1)]
                if self.hi_needed:
                    ops += [self._recv(hi0, 0), self._recv(hi1, 1)]
                self._wait(self._post(ops))
                e, c1 = c.relu_helper(lo0, hi0, lo1, hi1, self.prm, self.seed["s02"], self.seed["s12"], base)  # steps 2-3
                pending.append(((a, b), None, self._post([self._send(e, 0), self._send(e, 1), self._send(c1, 1)])))
            if len(pending) > 1:
                self._relu_finish(*pending.pop(0), out)
        while pending:
            self._relu_finish(*pending.pop(0), out)
        return out

    def _relu_finish(self, rng, state, works, out):
        self._wait(works)
        if state is None:
            return
        (a, b) = rng
        x, tb, d_own, d_peer, e, c1, seed_tr = state
        self.c.relu_finish(self.role.party, x, tb, d_own, d_peer, e, c1, self.prm, seed_tr, self.base + a,
                           out=out[a:b])  # steps 4-5
