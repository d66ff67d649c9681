"""Party-separated runtime (paper_2309_04909_b200.party) over torch.distributed
with the gloo backend on CPU: 3 ranks (one triple) and 6 ranks (two triples),
chunked, compared with the oracle's three-party functions.  The phase compute
is the oracle-backed tests/party_cpu_compute.py; the CUDA phase kernels are
checked separately on a GPU (test_gpu_parity.py)."""
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


def _worker(rank, world, port, kind, n, chunk, mode, literal, outdir):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2309_04909_b200 import party
    from paper_2309_04909_b200.api import Params
    from party_cpu_compute import OracleCompute

    class P(Params):  # the runner asks prm.c() for p; answer without the CUDA library
        def c(self):
            from oracle import bicoptor as B
            o = B.Params(ell=self.ell, lx=self.lx, f=self.f, mode=self.mode, rounds=self.rounds)
            return type("C", (), {"p": o.p, "slots": o.slots,
                                  "tape": {"pair": 0, "compact": 1, "large": 2, "compact_lit": 3}[o.layout]})()

    prm = P(**CONFIGS[mode])
    role = party.Role.of(rank)
    x, x0, x1 = synth.shares(n, prm.ell, prm.lx, prm.f, "D1", run=role.triple)
    xs = torch.from_numpy((x0 if role.party == 0 else x1).view(np.int64))
    runner = party.PartyRunner(prm, synth.seeds(0), n, chunk=chunk, compute=OracleCompute(), paper_literal=literal)
    y = runner.drelu(xs if role.party < 2 else None) if kind == "drelu" else runner.relu(xs if role.party < 2 else None)
    if y is not None:
        np.save(os.path.join(outdir, f"y_{rank}.npy"), y.numpy().view(np.uint64))
    np.save(os.path.join(outdir, f"bytes_{rank}.npy"), np.array([runner.bytes_sent]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,mode,literal", [("drelu", 3, "guard", False), ("drelu", 3, "guard", True),
                                                      ("relu", 3, "guard", False), ("relu", 6, "guard", False),
                                                      ("drelu", 3, "literal", False), ("relu", 3, "large", False),
                                                      ("drelu", 3, "large_full", True),
                                                      ("drelu", 3, "large_literal", False)])
def test_party_runtime_gloo(tmp_path, kind, world, mode, literal):
    import synth
    from oracle import bicoptor as B
    n, chunk = 300, 128  # 3 chunks, the last one ragged
    mp.start_processes(_worker, args=(world, _free_port(), kind, n, chunk, mode, literal, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    o = B.Params(**CONFIGS[mode])
    ell, lx, f = o.ell, o.lx, o.f
    for t in range(world // 3):
        x, x0, x1 = synth.shares(n, ell, lx, f, "D1", run=t)
        j = np.arange(n, dtype=np.uint64) + np.uint64(t * (-(-n // 8) * 8))  # triple t starts at a multiple of 8
        ref = getattr(B, kind)(o, x0, x1, j, synth.seeds(0))
        assert np.array_equal(np.load(tmp_path / f"y_{3 * t}.npy"), ref["y0"])
        assert np.array_equal(np.load(tmp_path / f"y_{3 * t + 1}.npy"), ref["y1"])
    # wire bytes per element: P0 -> P2 (ell_x+1) * ceil(log2 p) bits (Table 1)
    b0 = int(np.load(tmp_path / "bytes_0.npy")[0])
    # wire bytes per element: byte planes 8 + 1 (guard) / 8 (literal); uint32 planes 4 S (+ 4 with the bit-32 plane)
    per = {"guard": 9, "literal": 8, "large": 11 * 4, "large_full": 32 * 4 + 4, "large_literal": 32 * 4}[mode]
    extra = (0 if kind == "drelu" else 8)  # ReLU: P0 also sends [d]_0 to P1
    assert b0 == n * (per + extra)
