"""Peer-memory transport for the party-separated protocol (Alg 7 / Alg 8 with
P0, P1, P2 in separate processes, one GPU each on an NVSwitch node).

Instead of staging each message in the sender's HBM and moving it with NCCL
send/recv (party.PartyRunner), the phase kernel that PRODUCES a message stores
it straight into the RECEIVING party's HBM: every receive buffer ("inbox") is
exported with CUDA IPC (bc_ipc_export) and mapped into its producers
(bc_ipc_open; across GPUs a peer mapping, so the kernel's stores travel over
NVLink).  Compute and transfer are one kernel, tile by tile:

    DReLU  bc_drelu_send  (P0, P1) -> P2's inbox       lo 8 B + hi 1 B / element   (Alg 7 step 8)
           bc_drelu_helper (P2)    -> P1's inbox       [D']_1 8 B                  (step 10)
                                      (and P0's [D']_0 only in the paper-literal transport, reading C12)
    ReLU   bc_relu_send_to (P0, P1) -> P2's inbox (message) and the other party's inbox ([d]_b)
           bc_relu_helper_to (P2)   -> P0's inbox (e) and P1's inbox (e, [c]_1)      (Alg 8 step 3)

Synchronisation is stream-ordered, never a spinning kernel: every inbox is a
ring of `slots` chunk buffers; a Link (producer -> consumer) pairs each slot
with two interprocess CUDA events.  The producer records FILLED[s] after its
kernel and rings a host doorbell; the consumer's stream waits on FILLED[s]
before its kernel reads the slot, then records CONSUMED[s] and returns a
credit; the producer's stream waits on CONSUMED[s] before it overwrites the
slot again.  Doorbells and credits are tiny host messages over a gloo group:
they only order the host calls (a cudaStreamWaitEvent must follow the
cudaEventRecord it waits for); no host thread waits for the GPU.

Backends: CudaIpcBackend (the product: IPC memory and events on the rank's
GPU) and, for tests on machines without GPUs, a file-backed shared-memory
backend in tests/peer_cpu_backend.py with the oracle-based phase compute.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import api
from .party import Role, _chunks


class CudaIpcBackend:
    """Inboxes in this rank's HBM, exported / mapped with CUDA IPC (bc_ipc_*);
    slot events are interprocess CUDA events on the current stream."""

    def __init__(self, device):
        self.device = torch.device(device)
        self._maps = {}  # handle -> base address of the mapping in this process
        self._pools = []  # one private pool per inbox (alloc_inbox)
        api.lib()

    def alloc(self, shape, dtype):
        """Local working memory (never exported)."""
        return torch.zeros(shape, dtype=dtype, device=self.device)

    def alloc_inbox(self, shape, dtype):
        """An inbox that one producer maps.  bc_ipc_export exports the whole allocation that
        holds the tensor, so every inbox gets a private memory pool: its segment then holds
        that inbox and nothing else -- not this party's own shares or blinding bits, and not
        the inbox another party writes (P2's inbox from P1 must stay invisible to P0)."""
        pool = torch.cuda.MemPool()
        self._pools.append(pool)  # the pool must outlive its tensor
        with torch.cuda.use_mem_pool(pool, device=self.device):
            return torch.zeros(shape, dtype=dtype, device=self.device)

    def export(self, t):
        h, off = api.ipc_export(t)
        return (h, off, tuple(t.shape), t.dtype)

    def open(self, blob):
        h, off, shape, dtype = blob
        if h not in self._maps:  # one mapping per allocation (a handle can be opened once per process)
            self._maps[h] = api.ipc_open(h)
        return api.tensor_at(self._maps[h] + off, shape, dtype)

    @staticmethod
    def new_event():
        return torch.cuda.Event(interprocess=True)

    @staticmethod
    def export_event(ev):
        return bytes(ev.ipc_handle())

    def open_event(self, h):
        return torch.cuda.Event.from_ipc_handle(self.device, h)

    @staticmethod
    def record(ev):
        ev.record(torch.cuda.current_stream())

    @staticmethod
    def wait(ev):
        torch.cuda.current_stream().wait_event(ev)

    def close(self):
        for base in self._maps.values():
            api.ipc_close(base)
        self._maps.clear()


class Link:
    """One direction producer -> consumer: a ring of `slots` chunk buffers in the
    consumer's memory, FILLED / CONSUMED events per slot, doorbells and credits
    as host messages (tags 2*index and 2*index + 1)."""

    def __init__(self, index, src, dst, fields, slots, chunk):
        self.index, self.src, self.dst = index, src, dst  # global ranks
        self.fields = fields                              # name -> (per-element shape, dtype)
        self.slots, self.chunk = slots, chunk
        self.ring = None          # name -> tensor [slots, chunk, ...] (consumer: local; producer: mapped)
        self.filled = None        # [slots] events (producer creates, consumer opens)
        self.consumed = None      # [slots] events (consumer creates, producer opens)
        self.credits = 0          # producer: credits received so far (sequence numbers < credits + slots free)

    # -- setup ------------------------------------------------------------------
    def offer(self, rank, be):
        """What this rank publishes about the link (all_gather'd)."""
        out = {}
        if rank == self.dst:
            self.ring = {k: be.alloc_inbox((self.slots, self.chunk) + shp, dt) for k, (shp, dt) in self.fields.items()}
            self.consumed = [be.new_event() for _ in range(self.slots)]
            out["ring"] = {k: be.export(t) for k, t in self.ring.items()}
            out["consumed"] = [be.export_event(e) for e in self.consumed]
        if rank == self.src:
            self.filled = [be.new_event() for _ in range(self.slots)]
            out["filled"] = [be.export_event(e) for e in self.filled]
        return out

    def accept(self, rank, be, offers):
        if rank == self.src:
            o = offers[self.dst][self.index]
            self.ring = {k: be.open(b) for k, b in o["ring"].items()}
            self.consumed = [be.open_event(h) for h in o["consumed"]]
        if rank == self.dst:
            self.filled = [be.open_event(h) for h in offers[self.src][self.index]["filled"]]

    # -- producer ---------------------------------------------------------------
    def acquire(self, seq, be, g):
        """Slot views for message `seq` (in the consumer's memory); waits until the
        consumer has released message seq - slots from that slot."""
        s = seq % self.slots
        while self.credits + self.slots <= seq:
            c = torch.zeros(1, dtype=torch.int64)
            dist.recv(c, self.dst, group=g, tag=2 * self.index + 1)
            assert int(c[0]) == self.credits, f"link {self.index}: credit {int(c[0])}, expected {self.credits}"
            self.credits += 1
            be.wait(self.consumed[(self.credits - 1) % self.slots])
        return {k: t[s] for k, t in self.ring.items()}

    def publish(self, seq, be, g, works):
        be.record(self.filled[seq % self.slots])
        works.append(dist.isend(torch.tensor([seq], dtype=torch.int64), self.dst, group=g, tag=2 * self.index))

    def drain(self, seq_end, be, g):
        """Producer at teardown: collect the credits still in flight (every message < seq_end)."""
        while self.credits < seq_end:
            c = torch.zeros(1, dtype=torch.int64)
            dist.recv(c, self.dst, group=g, tag=2 * self.index + 1)
            self.credits += 1

    # -- consumer ---------------------------------------------------------------
    def wait(self, seq, be, g):
        """Local slot views holding message `seq`, ordered after its producer kernel."""
        c = torch.zeros(1, dtype=torch.int64)
        dist.recv(c, self.src, group=g, tag=2 * self.index)
        assert int(c[0]) == seq, f"link {self.index}: doorbell {int(c[0])}, expected {seq}"
        s = seq % self.slots
        be.wait(self.filled[s])
        return {k: t[s] for k, t in self.ring.items()}

    def release(self, seq, be, g, works):
        be.record(self.consumed[seq % self.slots])
        works.append(dist.isend(torch.tensor([seq], dtype=torch.int64), self.src, group=g, tag=2 * self.index + 1))


U8, I64 = torch.uint8, torch.int64


class PeerPartyRunner:
    """DReLU (kind="drelu") or ReLU (kind="relu") for this rank's role, messages
    through peer memory.  Ranks as in party.Role: rank r plays party r % 3 of
    triple r // 3.  `group` is a gloo group over the triple's ranks (doorbells,
    credits and the handle exchange); `compute` provides the phase kernels with
    the api signatures (default: the api module itself, i.e. libbicoptor)."""

    def __init__(self, kind, prm: api.Params, seeds, n: int, chunk: int = 1 << 22, slots: int = 2,
                 backend=None, compute=None, group=None, paper_literal: bool = False, base: int | None = None,
                 triples: int = 1):
        assert kind in ("drelu", "relu")
        assert slots >= 2, "two slots per link at least (with one the d exchange of ReLU deadlocks)"
        self.kind, self.prm, self.n = kind, prm, n
        self.rank = dist.get_rank()
        self.role = Role.of(self.rank)
        self.chunks = _chunks(n, chunk)
        self.cmax = max(b - a for a, b in self.chunks) if self.chunks else 0
        self.be = backend
        self.c = compute if compute is not None else api
        self.g = group
        self.literal = paper_literal and kind == "drelu"
        # PRG index range of run r: [base0 + r * stride, + n).  Every run draws fresh t, Pi, r_m,
        # rho_m and triples: reusing them on new inputs would open
        # x - x' to P0/P1 (d = x - a) and hand P2 several messages under one mask.  stride =
        # triples * n keeps the triples sharing the index space disjoint across runs too.
        span = -(-n // 8) * 8  # index ranges start at multiples of 8 (the elem_base rule)
        self.base0 = self.role.triple * span if base is None else base
        self.stride = triples * span
        self.runs = 0
        self.base = self.base0
        fmt = api.wire_format(prm)  # byte planes (p <= 257) or slot-major uint32 planes (large tape)
        self.fmt = fmt
        self.hi_needed = fmt["hi"] is not None
        held = {0: ("s01", "s02"), 1: ("s01", "s12"), 2: ("s02", "s12")}[self.role.party]
        self.seed = {k: getattr(seeds, k) for k in held}
        self.seq = 0   # messages sent per link so far (persists across runs: the rings keep turning)
        P0, P1, P2 = self.role.peers
        msg = {"lo": fmt["lo"]}
        if self.hi_needed:
            msg["hi"] = fmt["hi"]
        L = {"A": Link(0, P0, P2, msg, slots, self.cmax), "B": Link(1, P1, P2, msg, slots, self.cmax)}
        if kind == "drelu":
            L["C"] = Link(2, P2, P1, {"resp": ((), I64)}, slots, self.cmax)
            if self.literal:
                L["D"] = Link(3, P2, P0, {"resp": ((), I64)}, slots, self.cmax)
        else:
            L["E"] = Link(4, P0, P1, {"d": ((), I64)}, slots, self.cmax)
            L["F"] = Link(5, P1, P0, {"d": ((), I64)}, slots, self.cmax)
            L["G"] = Link(6, P2, P0, {"e": ((), I64)}, slots, self.cmax)
            L["H"] = Link(7, P2, P1, {"e": ((), I64), "c1": ((), I64)}, slots, self.cmax)
        self.L = L
        # local buffers of the computing parties: blinding bits, own [d]_b, a dummy hi plane
        p = self.role.party
        if p < 2:
            self.tb = self.be.alloc(((n + 7) // 8,), U8)
            self.d_own = self.be.alloc((n,), I64) if kind == "relu" else None
            self.hi_scratch = None if self.hi_needed else self.be.alloc((self.cmax,), fmt["lo"][1])
        # exchange handles inside the triple
        offer = {lk.index: lk.offer(self.rank, self.be) for lk in L.values()}
        ranks = list(self.role.peers)
        offers = [None] * dist.get_world_size(group) if group is not None else [None] * dist.get_world_size()
        dist.all_gather_object(offers, (self.rank, offer), group=group)
        by_rank = {r: o for r, o in offers}
        for lk in L.values():
            lk.accept(self.rank, self.be, by_rank)
        self._works = []
        self._ranks = ranks

    # ---- helpers -----------------------------------------------------------------
    def _reap(self, keep: int = 64):
        # wait() retires a host message; a Work dropped without wait() can lose its message (gloo)
        while len(self._works) > keep:
            self._works.pop(0).wait()

    def _send_out(self, d, m):
        lo = api.lo_plane(d["lo"], m, self.fmt)
        hi = d["hi"][:m] if self.hi_needed else self.hi_scratch[:m]
        return lo, hi

    def _lo_in(self, src, m):
        return api.lo_plane(src["lo"], m, self.fmt)

    @staticmethod
    def _hi_in(src, m):
        return src["hi"][:m] if "hi" in src else None

    # ---- DReLU (Alg 7) -----------------------------------------------------------------
    def _drelu(self, x, out):
        p, c, be, g, L, W = self.role.party, self.c, self.be, self.g, self.L, self._works
        lag = []  # P1 (and P0 in the literal transport): chunks whose response is outstanding
        for k, (a, b) in enumerate(self.chunks):
            m, base, seq = b - a, self.base + a, self.seq + k
            tb = None
            if p < 2:
                link = L["A"] if p == 0 else L["B"]
                dst = link.acquire(seq, be, g)
                tb = self.tb[a // 8:(b + 7) // 8]
                if p == 1 or self.literal:
                    c.drelu_send(p, x[a:b], self.prm, self.seed["s01"], base,
                                 out=(*self._send_out(dst, m), tb))                                  # steps 1-8
                    link.publish(seq, be, g, W)
                    lag.append((k, seq, a, b, tb))
                else:  # P0 derives [D']_0 from seed02 (reading C12): steps 1-8 and 10-11 in one kernel
                    c.drelu_send(0, x[a:b], self.prm, self.seed["s01"], base, out=(*self._send_out(dst, m), None),
                                 y=out[a:b], seed02=self.seed["s02"])
                    link.publish(seq, be, g, W)
                if len(lag) > 1:
                    self._drelu_finish(*lag.pop(0), out)
            else:
                s0, s1 = L["A"].wait(seq, be, g), L["B"].wait(seq, be, g)
                r1 = L["C"].acquire(seq, be, g)["resp"][:m]
                r0 = L["D"].acquire(seq, be, g)["resp"][:m] if self.literal else None
                c.drelu_helper(self._lo_in(s0, m), self._hi_in(s0, m), self._lo_in(s1, m), self._hi_in(s1, m), self.prm,
                               self.seed["s02"], base, paper_literal=self.literal, out=(r0, r1))     # steps 9-10
                L["A"].release(seq, be, g, W)
                L["B"].release(seq, be, g, W)
                L["C"].publish(seq, be, g, W)
                if self.literal:
                    L["D"].publish(seq, be, g, W)
            self._reap()
        while lag:
            self._drelu_finish(*lag.pop(0), out)

    def _drelu_finish(self, k, seq, a, b, tb, out):
        link = self.L["C"] if self.role.party == 1 else self.L["D"]
        src = link.wait(seq, self.be, self.g)
        self.c.drelu_finish(self.role.party, tb, src["resp"][:b - a], self.prm, b - a, None, self.base + a,
                            out=out[a:b])                                                             # step 11
        link.release(seq, self.be, self.g, self._works)

    # ---- ReLU (Alg 8) ------------------------------------------------------------------
    def _relu(self, x, out):
        p, c, be, g, L, W = self.role.party, self.c, self.be, self.g, self.L, self._works
        lag = []
        for k, (a, b) in enumerate(self.chunks):
            m, base, seq = b - a, self.base + a, self.seq + k
            if p < 2:
                to2, top = (L["A"], L["E"]) if p == 0 else (L["B"], L["F"])
                dst = to2.acquire(seq, be, g)
                dpeer = top.acquire(seq, be, g)["d"][:m]
                tb = self.tb[a // 8:(b + 7) // 8]
                seed_tr = self.seed["s02"] if p == 0 else self.seed["s12"]
                c.relu_send(p, x[a:b], self.prm, self.seed["s01"], seed_tr, base,
                            out=(*self._send_out(dst, m), tb, self.d_own[a:b]), d_peer=dpeer)     # steps 1, 4
                to2.publish(seq, be, g, W)
                top.publish(seq, be, g, W)
                lag.append((seq, a, b, tb, seed_tr))
                if len(lag) > 1:
                    self._relu_finish(x, *lag.pop(0), out)
            else:
                s0, s1 = L["A"].wait(seq, be, g), L["B"].wait(seq, be, g)
                e0 = L["G"].acquire(seq, be, g)["e"][:m]
                h = L["H"].acquire(seq, be, g)
                c.relu_helper(self._lo_in(s0, m), self._hi_in(s0, m), self._lo_in(s1, m), self._hi_in(s1, m), self.prm,
                              self.seed["s02"], self.seed["s12"], base, out=(e0, h["c1"][:m]),
                              e_dup=h["e"][:m])                                                     # steps 2-3
                L["A"].release(seq, be, g, W)
                L["B"].release(seq, be, g, W)
                L["G"].publish(seq, be, g, W)
                L["H"].publish(seq, be, g, W)
            self._reap()
        while lag:
            self._relu_finish(x, *lag.pop(0), out)

    def _relu_finish(self, x, seq, a, b, tb, seed_tr, out):
        p, be, g, L = self.role.party, self.be, self.g, self.L
        m = b - a
        from_peer, from2 = (L["F"], L["G"]) if p == 0 else (L["E"], L["H"])
        dp = from_peer.wait(seq, be, g)["d"][:m]
        s2 = from2.wait(seq, be, g)
        self.c.relu_finish(p, x[a:b], tb, self.d_own[a:b], dp, s2["e"][:m], s2["c1"][:m] if p == 1 else None,
                           self.prm, seed_tr, self.base + a, out=out[a:b])                          # steps 4-5
        from_peer.release(seq, be, g, self._works)
        from2.release(seq, be, g, self._works)

    # ---- public ------------------------------------------------------------------------
    def egress_bytes_per_elem(self) -> dict:
        """Bytes per element this rank's kernels store into each peer's inbox per run (every
        link it produces: the message planes to P2, [d]_b, e, [c]_1, the response), from the
        link field shapes -- the wire cost the protocol pays (Table 1)."""
        out = {}
        for name, lk in self.L.items():
            if lk.src != self.rank:
                continue
            b = 0
            for shp, dt in lk.fields.values():
                k = 1
                for s_ in shp:
                    k *= s_
                b += k * torch.empty((), dtype=dt).element_size()
            out[f"link{name}->P{Role.of(lk.dst).party}"] = b
        return out

    def run(self, x=None, out=None, elem_base: int | None = None):
        """P0/P1: x is this party's share vector (n,), returns its output share.
        P2: x=None, returns None.  Asynchronous on the current stream like the
        kernels themselves: synchronise before reading the result on the host.
        Run r uses the global element indices base0 + r * stride + [0, n) (stride =
        triples * n rounded up to a multiple of 8) unless
        elem_base is given (all three parties must pass the same value)."""
        p = self.role.party
        self.base = self.base0 + self.runs * self.stride if elem_base is None else elem_base
        self.runs += 1
        if p < 2 and out is None:
            out = self.be.alloc((self.n,), I64)
        if self.kind == "drelu":
            self._drelu(x, out)
        else:
            self._relu(x, out)
        self.seq += len(self.chunks)
        return out if p < 2 else None

    def close(self):
        """Collect the outstanding credits, wait for the host messages, unmap the peers'
        inboxes once every rank of the triple is done with them."""
        for lk in self.L.values():
            if lk.src == self.rank:
                lk.drain(self.seq, self.be, self.g)
        for w in self._works:
            w.wait()
        self._works = []
        if torch.cuda.is_available() and isinstance(self.be, CudaIpcBackend):
            torch.cuda.synchronize(self.be.device)
        dist.barrier(group=self.g)
        self.be.close()
        dist.barrier(group=self.g)
