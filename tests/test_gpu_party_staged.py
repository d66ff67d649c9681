"""Party-separated DReLU / ReLU with the real CUDA phase kernels: three
processes (P0, P1, P2) share cuda:0, the messages travel over gloo through host
memory (party.StagedCudaCompute); each computing party's output share is
bit-exact with the oracle's three-party run."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, chunk, literal, outdir):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2309_04909_b200 import api, party
    prm = api.Params(ell=64, lx=7, f=24, mode="guard", rounds=20)
    role = party.Role.of(rank)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=role.triple)
    xs = torch.from_numpy((x0 if role.party == 0 else x1).view(np.int64))
    runner = party.PartyRunner(prm, synth.seeds(0), n, chunk=chunk, compute=party.StagedCudaCompute("cuda:0"),
                               paper_literal=literal)
    y = runner.drelu(xs if role.party < 2 else None) if kind == "drelu" else runner.relu(xs if role.party < 2 else None)
    if y is not None:
        np.save(os.path.join(outdir, f"y_{rank}.npy"), y.numpy().view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,literal", [("drelu", False), ("drelu", True), ("relu", False)])
def test_party_staged_three_processes(tmp_path, kind, literal):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import synth
    from oracle import bicoptor as B
    n, chunk = 1003, 256
    mp.start_processes(_worker, args=(3, _free_port(), kind, n, chunk, literal, str(tmp_path)), nprocs=3, join=True,
                       start_method="spawn")
    o = B.Params(ell=64, lx=7, f=24, mode="guard", rounds=20)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=0)
    ref = getattr(B, kind)(o, x0, x1, np.arange(n, dtype=np.uint64), synth.seeds(0))
    assert np.array_equal(np.load(tmp_path / "y_0.npy"), ref["y0"])
    assert np.array_equal(np.load(tmp_path / "y_1.npy"), ref["y1"])
