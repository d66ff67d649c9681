"""Peer-memory party transport with the real CUDA phase kernels and CUDA IPC:
P0, P1, P2 are three processes sharing cuda:0; every message is stored by its
producing kernel straight into the receiving process's inbox (bc_ipc_open
mappings), ordered by interprocess events.  Each computing party's output
share is bit-exact with the oracle (small n) and with the fused one-GPU
kernel (large n, several ring turns)."""
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


def _worker(rank, world, port, kind, n, chunk, slots, literal, runs, outdir, kw=None):
    try:
        _work(rank, world, port, kind, n, chunk, slots, literal, runs, outdir, kw)
    except BaseException:
        import traceback
        with open(os.path.join(outdir, f"err_{rank}.txt"), "w") as f:
            f.write(traceback.format_exc())
        raise


def _work(rank, world, port, kind, n, chunk, slots, literal, runs, outdir, kw=None):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import synth
    from paper_2309_04909_b200 import api, peer
    kw = kw or dict(ell=64, lx=7, f=24, mode="guard", rounds=20)
    prm = api.Params(**kw)
    role = peer.Role.of(rank)
    x, x0, x1 = synth.shares(n, kw["ell"], kw["lx"], kw["f"], "D1", run=role.triple)
    xs = torch.from_numpy((x0 if role.party == 0 else x1).view(np.int64)).cuda()
    runner = peer.PeerPartyRunner(kind, prm, synth.seeds(0), n, chunk=chunk, slots=slots,
                                  backend=peer.CudaIpcBackend("cuda:0"), group=dist.group.WORLD,
                                  paper_literal=literal)
    ys = [runner.run(xs if role.party < 2 else None) for _ in range(runs)]
    torch.cuda.synchronize()
    runner.close()
    if role.party < 2:
        for r, y in enumerate(ys):
            np.save(os.path.join(outdir, f"y_{rank}_{r}.npy"), y.cpu().numpy().view(np.uint64))
        # the fused one-GPU kernel on the same shares (bit-exact with the oracle: test_gpu_parity.py)
        t0 = torch.from_numpy(x0.view(np.int64)).cuda()
        t1 = torch.from_numpy(x1.view(np.int64)).cuda()
        span = -(-n // 8) * 8
        for r in range(runs):  # run r draws from global indices r span + [0, n) (one triple)
            ref = getattr(api, kind)(t0, t1, prm, synth.seeds(0), (role.triple + r) * span)[role.party]
            np.save(os.path.join(outdir, f"fused_{rank}_{r}.npy"), ref.cpu().numpy().view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, kind, n, chunk, slots, literal, runs, kw=None):
    try:
        mp.start_processes(_worker, args=(3, _free_port(), kind, n, chunk, slots, literal, runs, str(tmp_path), kw),
                           nprocs=3, join=True, start_method="spawn")
    except Exception:
        errs = "".join(f"--- rank {r}\n" + open(tmp_path / f"err_{r}.txt").read()
                       for r in range(3) if (tmp_path / f"err_{r}.txt").exists())
        raise AssertionError(errs or "worker failed")
    for rank in (0, 1):  # every run equals the fused kernel's share at that run's indices
        for r in range(runs):
            ref = np.load(tmp_path / f"fused_{rank}_{r}.npy")
            assert np.array_equal(np.load(tmp_path / f"y_{rank}_{r}.npy"), ref), (kind, rank, r)


@pytest.mark.parametrize("kind,slots,literal", [("drelu", 2, False), ("drelu", 3, True), ("relu", 2, False)])
def test_party_peer_three_processes_vs_oracle(tmp_path, kind, slots, literal):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import synth
    from oracle import bicoptor as B
    n, chunk = 2003, 256  # 8 chunks, the last ragged, through 2-3 ring slots
    _run(tmp_path, kind, n, chunk, slots, literal, runs=2)
    o = B.Params(ell=64, lx=7, f=24, mode="guard", rounds=20)
    x, x0, x1 = synth.shares(n, 64, 7, 24, "D1", run=0)
    span = -(-n // 8) * 8
    for r in range(2):
        ref = getattr(B, kind)(o, x0, x1, np.arange(n, dtype=np.uint64) + np.uint64(r * span), synth.seeds(0))
        assert np.array_equal(np.load(tmp_path / f"y_0_{r}.npy"), ref["y0"])
        assert np.array_equal(np.load(tmp_path / f"y_1_{r}.npy"), ref["y1"])


@pytest.mark.parametrize("kind", ["drelu", "relu"])
def test_party_peer_large_vs_fused(tmp_path, kind):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _run(tmp_path, kind, (1 << 22) + 13, 1 << 20, 2, False, runs=3)  # 5 chunks x 3 runs: the rings keep turning


@pytest.mark.parametrize("kind", ["drelu", "relu"])
def test_party_peer_full_precision(tmp_path, kind):
    """The large tape through the peer transport: lx = 31 full precision (p = 2^32 + 15),
    slot-major uint32 planes with the bit-32 plane stored into P2's inbox."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    kw = dict(ell=64, lx=31, f=0, mode="guard", rounds=8)
    _run(tmp_path, kind, 2003, 512, 2, kind == "drelu", 2, kw)


def test_inbox_exports_only_itself():
    """Every inbox sits alone in the allocation bc_ipc_export hands to its producer:
    offset 0 and a handle of its own, distinct from the party's local buffers'."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path[:0] = [ROOT]
    from paper_2309_04909_b200 import api, peer
    be = peer.CudaIpcBackend("cuda:0")
    local = be.alloc((1000,), torch.int64)
    boxes = [be.alloc_inbox((2, 4096, 8), torch.uint8), be.alloc_inbox((2, 4096), torch.uint8),
             be.alloc_inbox((2, 4096), torch.int64)]
    local2 = be.alloc((1000,), torch.int64)
    handles = set()
    for b in boxes:
        h, off = api.ipc_export(b)
        assert off == 0
        handles.add(h)
    assert len(handles) == len(boxes)
    assert api.ipc_export(local)[0] not in handles and api.ipc_export(local2)[0] not in handles
