"""Sharded mode's host logic with world_size 2 on CPU (gloo): each rank's
elem_base shard, run through the oracle, concatenates to the unsharded run
bit for bit (the property that lets shards skip any data exchange), and the
max-over-ranks reduction the bench reports is the maximum."""
import os
import socket
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, outdir):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from oracle import bicoptor as B
    from paper_2309_04909_b200 import shard
    x, x0, x1 = synth.shares(world * n, 64, 7, 24, "D1")
    base = shard.elem_base(rank, n)
    o = B.Params(ell=64, lx=7, f=24, rounds=8)
    j = np.arange(n, dtype=np.uint64) + np.uint64(base)
    ref = B.drelu(o, x0[base:base + n], x1[base:base + n], j, synth.seeds(0))
    np.save(os.path.join(outdir, f"y0_{rank}.npy"), ref["y0"])
    np.save(os.path.join(outdir, f"y1_{rank}.npy"), ref["y1"])
    shard.barrier()
    m = shard.max_over_ranks(float(rank) + 0.5)
    np.save(os.path.join(outdir, f"max_{rank}.npy"), np.array([m]))
    dist.destroy_process_group()


def test_shards_concatenate_to_the_unsharded_run(tmp_path):
    import synth
    from oracle import bicoptor as B
    world, n = 2, 200
    mp.start_processes(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x, x0, x1 = synth.shares(world * n, 64, 7, 24, "D1")
    full = B.drelu(B.Params(ell=64, lx=7, f=24, rounds=8), x0, x1, np.arange(world * n, dtype=np.uint64),
                   synth.seeds(0))
    y0 = np.concatenate([np.load(tmp_path / f"y0_{r}.npy") for r in range(world)])
    y1 = np.concatenate([np.load(tmp_path / f"y1_{r}.npy") for r in range(world)])
    assert np.array_equal(y0, full["y0"]) and np.array_equal(y1, full["y1"])
    for r in range(world):
        assert float(np.load(tmp_path / f"max_{r}.npy")[0]) == world - 0.5


def test_elem_base_alignment():
    import pytest

    from paper_2309_04909_b200 import shard
    assert shard.elem_base(3, 1 << 24) == 3 << 24
    with pytest.raises(ValueError):
        shard.elem_base(1, 12)
