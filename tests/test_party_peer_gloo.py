"""Peer-memory party transport (paper_2309_04909_b200.peer) on CPU: 3 ranks (one
triple) and 6 ranks (two triples) under gloo, inboxes as shared file mappings
(tests/peer_cpu_backend.py), phase compute from the oracle.  Checks the
transport's host logic -- ring slots, doorbells, credits, roles, ragged
chunks, rings that keep turning across runs -- against the oracle's
three-party functions.  The CUDA IPC backend runs in test_gpu_party_peer.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# "guard": compact tape, byte wire planes; "literal": p = 131 (no high-bit plane);
# "large": lx = 10 large tape, uint32 low-word plane only (p = 2053); "large_full": the paper's
# full precision lx = 31 (p = 2^32 + 15: low words and the bit-32 plane); "large_literal": p = 2^31 + 11
CONFIGS = {"guard": dict(ell=64, lx=7, f=24, mode="guard", rounds=8),
           "literal": dict(ell=16, lx=7, f=0, mode="literal", rounds=8),
           "large": dict(ell=24, lx=10, f=0, mode="guard", rounds=8),
           "large_full": dict(ell=64, lx=31, f=0, mode="guard", rounds=8),
           "large_literal": dict(ell=64, lx=31, f=0, mode="literal", rounds=8)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, chunk, slots, mode, literal, runs, outdir):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2309_04909_b200 import peer
    from paper_2309_04909_b200.api import Params
    from peer_cpu_backend import FileBackend, OracleApiCompute

    class P(Params):  # the runner asks prm.c() for p; answer without the CUDA library
        def c(self):
            from oracle import bicoptor as B
            o = B.Params(ell=self.ell, lx=self.lx, f=self.f, mode=self.mode, rounds=self.rounds)
            return type("C", (), {"p": o.p, "slots": o.slots,
                                  "tape": {"pair": 0, "compact": 1, "large": 2, "compact_lit": 3}[o.layout]})()

    prm = P(**CONFIGS[mode])
    role = peer.Role.of(rank)
    x, x0, x1 = synth.shares(n, prm.ell, prm.lx, prm.f, "D1", run=role.triple)
    xs = torch.from_numpy((x0 if role.party == 0 else x1).view(np.int64))
    # every rank takes part in creating every triple's group, in the same order
    group = [dist.new_group([3 * t, 3 * t + 1, 3 * t + 2]) for t in range(world // 3)][role.triple]
    runner = peer.PeerPartyRunner(kind, prm, synth.seeds(0), n, chunk=chunk, slots=slots,
                                  backend=FileBackend(outdir, rank), compute=OracleApiCompute(), group=group,
                                  paper_literal=literal, triples=world // 3)
    ys = [runner.run(xs if role.party < 2 else None) for _ in range(runs)]
    import json
    with open(os.path.join(outdir, f"egress_{rank}.json"), "w") as fh:
        json.dump(runner.egress_bytes_per_elem(), fh)
    runner.close()
    if role.party < 2:
        for r, y in enumerate(ys):
            np.save(os.path.join(outdir, f"y_{rank}_{r}.npy"), y.numpy().view(np.uint64).copy())
    dist.barrier()
    dist.destroy_process_group()


def test_peer_runtime_gloo_single_chunk_many_slots(tmp_path):
    """One chunk (n < chunk) through 4 ring slots, three runs: the credits that are
    never needed inside a run are still collected at close()."""
    import synth
    from oracle import bicoptor as B
    n, chunk, runs = 37, 64, 3
    mp.start_processes(_worker, args=(3, _free_port(), "relu", n, chunk, 4, "guard", False, runs, str(tmp_path)),
                       nprocs=3, join=True, start_method="spawn")
    o = B.Params(**CONFIGS["guard"])
    x, x0, x1 = synth.shares(n, o.ell, o.lx, o.f, "D1", run=0)
    span = -(-n // 8) * 8
    for r in range(runs):  # run r draws fresh randomness: global indices r span + [0, n)
        ref = B.relu(o, x0, x1, np.arange(n, dtype=np.uint64) + np.uint64(r * span), synth.seeds(0))
        assert np.array_equal(np.load(tmp_path / f"y_0_{r}.npy"), ref["y0"])
        assert np.array_equal(np.load(tmp_path / f"y_1_{r}.npy"), ref["y1"])


@pytest.mark.parametrize("mode,msg", [("guard", 9), ("literal", 8)])
def test_peer_egress_bytes_match_table1(tmp_path, mode, msg):
    """The bytes each party's kernels store into its peers' inboxes per element, from the
    inbox field shapes (PeerPartyRunner.egress_bytes_per_elem): the one-pass message to P2
    is (lx+1) ceil(log2 p) bits = 72 (guard, p = 257) or 64 (the paper's Table 1, P:93-96,
    literal p = 131); ReLU adds [d]_b to the other computing party and e (+ [c]_1) from P2."""
    import json
    mp.start_processes(_worker, args=(3, _free_port(), "relu", 64, 64, 2, mode, False, 1, str(tmp_path)),
                       nprocs=3, join=True, start_method="spawn")
    eg = [json.load(open(tmp_path / f"egress_{r}.json")) for r in range(3)]
    assert eg[0] == {"linkA->P2": msg, "linkE->P1": 8}
    assert eg[1] == {"linkB->P2": msg, "linkF->P0": 8}
    assert eg[2] == {"linkG->P0": 8, "linkH->P1": 16}


@pytest.mark.parametrize("kind,world,slots,mode,literal", [
    ("drelu", 3, 2, "guard", False), ("drelu", 3, 3, "guard", True), ("relu", 3, 2, "guard", False),
    ("relu", 6, 2, "guard", False), ("drelu", 3, 2, "literal", False), ("relu", 3, 3, "literal", False),
    ("relu", 3, 2, "large", False), ("drelu", 3, 2, "large_full", True), ("relu", 3, 2, "large_literal", False)])
def test_peer_runtime_gloo(tmp_path, kind, world, slots, mode, literal):
    import synth
    from oracle import bicoptor as B
    n, chunk, runs = 300, 64, 2  # 5 chunks (the last one ragged) through 2-3 slots, twice
    mp.start_processes(_worker, args=(world, _free_port(), kind, n, chunk, slots, mode, literal, runs,
                                      str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    o = B.Params(**CONFIGS[mode])
    ell, lx, f = o.ell, o.lx, o.f
    k, span = world // 3, -(-n // 8) * 8
    for t in range(k):
        x, x0, x1 = synth.shares(n, ell, lx, f, "D1", run=t)
        for r in range(runs):  # run r of triple t: global indices (r k + t) n + [0, n), disjoint over runs and triples
            j = np.arange(n, dtype=np.uint64) + np.uint64((r * k + t) * span)
            ref = getattr(B, kind)(o, x0, x1, j, synth.seeds(0))
            assert np.array_equal(np.load(tmp_path / f"y_{3 * t}_{r}.npy"), ref["y0"]), (t, r)
            assert np.array_equal(np.load(tmp_path / f"y_{3 * t + 1}_{r}.npy"), ref["y1"]), (t, r)
