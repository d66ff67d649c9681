"""bench.py's N > 1 code paths under torchrun (one process per rank, as the
driver launches them).  This run's GPU boxes have one GPU, so the sharded and
peer-transport paths run with BENCH_SHARE_GPU=1 (every rank on cuda:0, gloo for
the barriers): the numbers are not measurements, the JSON contract, the rank
bookkeeping and the wire accounting are what is checked.  The NCCL party
transport needs one GPU per party and is skipped below 3 devices."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, args, share=True, timeout=900):
    env = {**os.environ}
    if share:
        env["BENCH_SHARE_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py")] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_sharded_world2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = 1 << 20
    line = _torchrun(2, ["--gpus", "2", "--elems", str(n), "--steps", "5", "--warmup", "3", "--no-extras"])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["steps"] == 5 and line["warmup"] >= 3
    assert line["value"] > 0 and line["unit"] == "elements/s"
    # whole-job throughput: both ranks' elements over the max-over-ranks time
    assert abs(line["value"] - 2 * n / (line["ms_per_step"] * 1e-3)) <= 1e-6 * line["value"]
    assert line["gpu_launches"] == 5


@pytest.mark.parametrize("domain,bits", [("guard", 72), ("literal", 64)])
def test_bench_party_peer_world3_wire_bits(domain, bits):
    """Config 4 through the peer-memory transport, three ranks: the one-pass message
    of each computing party is (lx+1) ceil(log2 p) bits per element -- 72 in guard
    mode, 64 (the paper's Table 1) in the literal domain."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    line = _torchrun(3, ["--gpus", "3", "--mode", "party", "--transport", "peer", "--domain", domain,
                         "--party-n", str(1 << 20), "--chunk", str(1 << 18), "--steps", "2", "--warmup", "2"])
    assert line["mode"] == "party" and line["transport"] == "peer" and line["value"] > 0
    assert line["one_pass_bits_per_party"] == {"P0->P2": bits, "P1->P2": bits}
    msg = bits // 8
    # P0, P1: message to P2 + [d]_b to the other computing party; P2: e to both + [c]_1 to P1
    assert line["wire_bytes_per_elem"] == {"P0": msg + 8, "P1": msg + 8, "P2": 24}
    assert line["paper_one_pass_bits"] == 64


def test_bench_party_nccl_world3():
    """Config 4 over NCCL point-to-point: one GPU per party (skipped on smaller boxes)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 3:
        pytest.skip("needs >= 3 GPUs (one per party)")
    line = _torchrun(3, ["--gpus", "3", "--mode", "party", "--transport", "nccl", "--party-n", str(1 << 22),
                         "--chunk", str(1 << 20), "--steps", "3", "--warmup", "2"], share=False)
    assert line["transport"] == "nccl" and line["value"] > 0
    assert line["one_pass_bits_per_party"] == {"P0->P2": 72, "P1->P2": 72}
