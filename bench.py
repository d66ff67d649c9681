#!/usr/bin/env python
"""Benchmark of the Bicoptor 2.0 DReLU / ReLU hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...     (N > 1)

Workload (BASELINE.json config 3): DReLU, ell = 64, the paper's key-bit window
(lx = 7, f = 24: 5+2 of the 5+26 fixed point), guard mode, ChaCha20
PRG, 2^24 elements per GPU, D2 activation-like inputs.  A step is one fused
three-party pass (Alg 7: both computing parties, the helper's zero test and
reshare, the unblinding) over the batch, inputs resident in HBM.  The same
run times ReLU (Alg 8) on the same batch and the trc+modswitch primitive of
config 2 (HBM roofline check); they are reported as sub-objects.

Multi-GPU: elements are independent.  Each rank owns 2^24 elements
at global offset rank * 2^24 (weak scaling); every PRG draw is addressed by
global index, so there is no data-path collective.  Time = max over ranks of
the CUDA-event time between two barriers.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_PER_GPU = 1 << 24
ELL, LX, F, MODE, ROUNDS = 64, 7, 24, "guard", 20
METRIC = "DReLU & ReLU elements/s at ell=64 on 1/2/4/8 B200; % of HBM roofline"
# ALU-pipe work of the PRG, the part of the path that cannot leave the ALU pipe:
# per ChaCha_R block R/2 double rounds x 8 quarter rounds x (4 xor + 4 rotate).
CHACHA_ALU_OPS_PER_BLOCK = {20: 640, 12: 384, 8: 256}
BLOCKS_PER_ELEM = {"drelu": 0.5, "relu": 1.0,   # 3/8 (tape) + 1/8 (resp) or + 5/8 (triples)
                   "drelu_rss": 1.5, "relu_rss": 1.875,  # RSS: 3/8 (tape) + 9/8 (preprocessing) (+ 3/8 ReLU zero share)
                   "drelu_fp": 7.125, "relu_fp": 7.625}  # lx=31 large tape: 7 blocks + the finish streams
BYTES_PER_ELEM = {"drelu": 32, "relu": 32, "ladder": 16,   # algorithmic HBM bytes per element
                  "drelu_rss": 48, "relu_rss": 48, "drelu_fp": 32, "relu_fp": 32}
SM_COUNT_B200 = 148  # nominal; the roofline uses the device's own count
# Global element-index regions of the legs that run other inputs than the headline batch, so no
# two protocol executions of one run (any rank) share PRG draws: the headline owns [0, W 2^24),
# the batch sweep [2^40, + W 2^27), config 5's layer streams [2^41, ...) (BC_MAX_INDEX = 2^44).
SWEEP_BASE, STREAM_BASE = 1 << 40, 1 << 41


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--elems", "--n", dest="n", type=int, default=N_PER_GPU,
                    help="elements per GPU (--elems under torchrun: its parser takes --n as an abbreviation)")
    ap.add_argument("--rounds", type=int, default=ROUNDS)
    ap.add_argument("--no-extras", action="store_true", help="skip ReLU / ladder / variants / e2e / cpu legs")
    ap.add_argument("--only", choices=["drelu", "relu", "ladder", "drelu_rss", "relu_rss", "drelu_fp", "relu_fp",
                                       "drelu_literal", "party_drelu", "party_relu"],
                    help="profiling aid: launch one op steps+warmup times, print nothing")
    ap.add_argument("--op", default="drelu", choices=["drelu", "relu", "drelu_fp", "relu_fp", "drelu_rss", "relu_rss"],
                    help="tuning aid (tools/variants.py): the op of the headline timing with --no-extras")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "party"],
                    help="party: config 4, P0/P1/P2 on distinct GPUs (needs >= 3 ranks), ReLU over NCCL P2P")
    ap.add_argument("--party-n", type=int, default=1 << 26, help="elements per P0/P1/P2 triple (config 4)")
    ap.add_argument("--chunk", type=int, default=1 << 22, help="party mode: elements per pipelined chunk")
    ap.add_argument("--domain", default=MODE, choices=["guard", "literal"],
                    help="party mode: guard (w = lx+1, p = 257, 72-bit messages) or the paper-literal Z_{2^lx} "
                         "(p = 131, 64-bit messages; reading C6)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="party mode: NCCL P2P (party.PartyRunner) or peer memory (peer.PeerPartyRunner: the "
                         "phase kernels store each message into the receiver's HBM over NVLink, CUDA IPC)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "src": "fallback"}


def load_alu_ops():
    """Executed ALU-pipe thread instructions per element per op (tools/alu_ops_json.py from the
    committed ncu source-level SASS mix), or {}."""
    p = os.path.join(ROOT, "profiles", "ncu_alu_ops.json")
    try:
        return json.load(open(p)) if os.path.exists(p) else {}
    except Exception:
        return {}


def load_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline / --impl reference): the scalar C oracle
# (oracle/c/bicoptor_ref.c, OpenMP) as it stands, on a bounded sample of the
# bench workload; the numpy oracle alongside for reference.
# ---------------------------------------------------------------------------
def _workload_slice(lo: int, hi: int):
    """Elements lo .. hi - 1 of the bench workload (D2 activations, run 0 sharing)."""
    import synth
    x = synth.plaintext(hi - lo, ELL, LX, F, "D2", run=lo)
    return synth.share(x, ELL, run=lo)


def cref_rate(relu: bool, rounds: int, threads: int, budget_s: float):
    """Elements/s of the C oracle on `threads` host threads (0 = all): calibrate on a
    small slice, then time one call on a slice sized to about budget_s seconds."""
    from oracle import bicoptor as B, cref
    import synth
    prm = B.Params(ell=ELL, lx=LX, f=F, mode=MODE, rounds=rounds)
    sd = synth.seeds(0)
    m = 1 << 14
    x0, x1 = _workload_slice(0, m)
    t0 = time.perf_counter()
    cref.fused(prm, x0, x1, 0, sd, relu=relu, threads=threads)
    per_s = m / max(time.perf_counter() - t0, 1e-6)
    m = int(min(1 << 24, max(1 << 14, per_s * budget_s)))
    x0, x1 = _workload_slice(0, m)
    t0 = time.perf_counter()
    cref.fused(prm, x0, x1, 0, sd, relu=relu, threads=threads)
    return m / (time.perf_counter() - t0), m


def _oracle_chunk(args):
    """One numpy-oracle worker: generate its slice of the workload, then time only the oracle call."""
    lo, hi, fn, rounds = args
    import synth
    from oracle import bicoptor as B
    prm = B.Params(ell=ELL, lx=LX, f=F, mode=MODE, rounds=rounds)
    x0, x1 = _workload_slice(lo, hi)
    j = np.arange(lo, hi, dtype=np.uint64)
    t0 = time.perf_counter()
    getattr(B, fn)(prm, x0, x1, j, synth.seeds(0))
    return hi - lo, time.perf_counter() - t0


def cpu_baseline(rounds: int):
    """The oracle timed on the host cores (rank 0 at N=1 only): the C oracle single-threaded
    and on all nproc threads (value), plus the numpy oracle on one core."""
    from oracle import cref
    nproc = os.cpu_count() or 1
    threads = cref.threads()
    r1, m1 = cref_rate(False, rounds, 1, 4.0)
    rn, mn = cref_rate(False, rounds, 0, 4.0)
    rr, mr = cref_rate(True, rounds, 0, 3.0)
    cnt, dt = _oracle_chunk((0, 1 << 13, "drelu", rounds))
    return {"value": rn, "unit": "elements/s", "cores": threads, "kind": "oracle",
            "sample": f"C oracle (oracle/c/bicoptor_ref.c, gcc -O2 -fopenmp), DReLU on the bench workload: "
                      f"{mn} elements on {threads} threads (nproc {nproc}); 1 thread: {m1} elements",
            "nproc": nproc, "single_thread": r1, "relu_all_threads": rr,
            "numpy_oracle_one_core": cnt / dt}


def run_reference(a, budget_s: float | None = None):
    """The reference arm for this tier: the C oracle, as it stands, on all host cores
    (tier framing 4).  Each step is a bounded sample of the bench workload (a fresh
    slice of m elements at its own global offset), sized so warmup + steps fit in
    about budget_s seconds."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import bicoptor as B, cref
    import synth
    if budget_s is None:  # BENCH_REF_BUDGET_S: tests shrink the run (default ~1 minute of CPU work)
        budget_s = float(os.environ.get("BENCH_REF_BUDGET_S", "60"))
    threads = cref.threads()
    prm = B.Params(ell=ELL, lx=LX, f=F, mode=MODE, rounds=a.rounds)
    sd = synth.seeds(0)
    per_s, _ = cref_rate(False, a.rounds, 0, 0.5)
    total = max(a.warmup, 3) + a.steps
    m = int(max(1 << 12, min(1 << 24, per_s * budget_s / total)))
    times, vals = [], []
    for s in range(total):
        x0, x1 = _workload_slice(s * m, (s + 1) * m)
        t0 = time.perf_counter()
        cref.fused(prm, x0, x1, s * m, sd, threads=0)
        dt = time.perf_counter() - t0
        if s >= total - a.steps:
            times.append(dt)
            vals.append(m / dt)
    value = float(np.median(vals))
    sample = (f"C oracle (oracle/c/bicoptor_ref.c, OpenMP) on {threads} threads (nproc {os.cpu_count()}): "
              f"{m} elements of the bench workload (DReLU, D2) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": workload_config(a),
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(a):
    return {"workload": f"config3: DReLU ell={ELL} lx={LX} f={F} {MODE} ChaCha{a.rounds}, 2^{int(math.log2(a.n))} elements/GPU, D2",
            "n_per_gpu": a.n, "ell": ELL, "lx": LX, "f": F, "mode": MODE, "rounds": a.rounds, "dist": "D2",
            "parallelism": f"element-sharded x{a.gpus} (3 parties simulated per GPU)",
            "l2": "no flush: inputs+outputs = 32 B/elem = 512 MiB per GPU > 126 MB L2"}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler; only samples stamped inside [mark_start, mark_end] count."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        import datetime
        rows, all_rows = [], []
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                row = (ts, float(parts[1]), float(parts[2]), parts[3:7])
            except ValueError:
                continue
            all_rows.append(row)
            if self.t0 is not None and self.t0 <= ts <= (self.t1 or ts):
                rows.append(row)
        if not rows:
            rows = all_rows[-3:]  # region shorter than the sampling period: nearest samples
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k, v in enumerate(r[3]) if v.lower().startswith("active")})
        return {"sm_mhz": float(np.median([r[1] for r in rows])), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CUDA leg
# ---------------------------------------------------------------------------
def run_cuda(a):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2309_04909_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_SHARE_GPU=1 (testing the N>1 code path on a 1-GPU box): every rank on cuda:0, gloo
    # for the barriers and the max over ranks.  Its numbers are not measurements.
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    api.lib()

    from paper_2309_04909_b200 import shard

    barrier = shard.barrier

    def max_over_ranks(v: float) -> float:
        return shard.max_over_ranks(v, "cpu" if share else dev)

    n = a.n
    base = shard.elem_base(rank, n)
    seeds = synth.seeds(0)
    prm = api.Params(ell=ELL, lx=LX, f=F, mode=MODE, rounds=a.rounds)
    x = synth.plaintext(n, ELL, LX, F, "D2", run=rank)
    x0h, x1h = synth.share(x, ELL, run=rank)
    x0 = torch.from_numpy(x0h.view(np.int64)).to(dev)
    x1 = torch.from_numpy(x1h.view(np.int64)).to(dev)
    y0 = torch.empty_like(x0)
    y1 = torch.empty_like(x1)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps, warmup, launches_per_step=1, clocks=None):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        if clocks:
            clocks.start()
            for _ in range(warmup):  # keep the GPU busy while the sampler comes up
                fn()
            time.sleep(0.2)
            torch.cuda.synchronize(dev)
            clocks.mark_start()
        # two events around the K steps: an event recorded between two launches would wait for the
        # first to drain before the second may start (no tail/head overlap of back-to-back steps)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        for s in range(steps):
            fn()
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
        if clocks:
            clocks.mark_end()
        barrier()
        torch.cuda.synchronize(dev)
        ck = clocks.stop() if clocks else None
        total_ms = ev[0].elapsed_time(ev[1])
        return max_over_ranks(total_ms), None, ck

    if a.only:  # profiling aid (ncu): just the launches, no timing output
        pfp = api.Params(ell=ELL, lx=31, f=0, mode=MODE, rounds=a.rounds)
        plit = api.Params(ell=ELL, lx=LX, f=F, mode="literal", rounds=a.rounds)
        if a.only == "ladder":  # config 2's size, as the bench leg times it
            x_c2 = x0.repeat(((1 << 28) + n - 1) // n)[:1 << 28]
            v_lad = torch.empty((1 << 28, 8), dtype=torch.uint8, device=dev)
        if a.only.startswith("party_"):  # the five party-phase kernels of one step, chained
            lo0, hi0, tb0 = api.msg_buffers(n, dev)
            lo1, hi1, tb1 = api.msg_buffers(n, dev)
            r1, d0, d1, e, c1 = (torch.empty_like(y0) for _ in range(5))
        if a.only.endswith("_rss"):
            xs = [torch.from_numpy(v.view(np.int64)).to(dev) for v in synth.rss_share(x, ELL, run=rank)]
            ys = tuple(torch.empty_like(xs[0]) for _ in range(3))
            f_rss = getattr(api, a.only)
        def party_drelu():
            api.drelu_send(0, x0, prm, seeds.s01, base, out=(lo0, hi0, tb0), stream=stream)
            api.drelu_send(1, x1, prm, seeds.s01, base, out=(lo1, hi1, tb1), stream=stream)
            api.drelu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, base, out=(None, r1), stream=stream)
            api.drelu_finish(0, tb0, None, prm, n, seeds.s02, base, out=y0, stream=stream)
            api.drelu_finish(1, tb1, r1, prm, n, None, base, out=y1, stream=stream)

        def party_relu():
            api.relu_send(0, x0, prm, seeds.s01, seeds.s02, base, out=(lo0, hi0, tb0, d0), stream=stream)
            api.relu_send(1, x1, prm, seeds.s01, seeds.s12, base, out=(lo1, hi1, tb1, d1), stream=stream)
            api.relu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, seeds.s12, base, out=(e, c1), stream=stream)
            api.relu_finish(0, x0, tb0, d0, d1, e, None, prm, seeds.s02, base, out=y0, stream=stream)
            api.relu_finish(1, x1, tb1, d1, d0, e, c1, prm, seeds.s12, base, out=y1, stream=stream)

        op = {"party_drelu": party_drelu, "party_relu": party_relu,
              "drelu_rss": lambda: f_rss(*xs, prm, seeds, base, out=ys, stream=stream),
              "relu_rss": lambda: f_rss(*xs, prm, seeds, base, out=ys, stream=stream),
              "drelu_fp": lambda: api.drelu(x0, x1, pfp, seeds, base, y0, y1, stream=stream),
              "drelu_literal": lambda: api.drelu(x0, x1, plit, seeds, base, y0, y1, stream=stream),
              "relu_fp": lambda: api.relu(x0, x1, pfp, seeds, base, y0, y1, stream=stream),
              "drelu": lambda: api.drelu(x0, x1, prm, seeds, base, y0, y1, stream=stream),
              "relu": lambda: api.relu(x0, x1, prm, seeds, base, y0, y1, stream=stream),
              "ladder": lambda: api.ladder_modswitch(0, x_c2, prm, out=v_lad, stream=stream)}[a.only]
        for _ in range(a.warmup + a.steps):
            op()
        torch.cuda.synchronize(dev)
        return

    # ---- headline: fused DReLU ------------------------------------------------
    ck = Clocks(local)
    head = api.relu if a.op.startswith("relu") else api.drelu
    hprm = prm if not a.op.endswith("_fp") else api.Params(ell=ELL, lx=31, f=0, mode=MODE, rounds=a.rounds)
    step = lambda: head(x0, x1, hprm, seeds, base, y0, y1, stream=stream)  # noqa: E731
    if a.op.endswith("_rss"):  # tuning aid: the RSS kernels on replicated shares of the same x
        xr = [torch.from_numpy(v.view(np.int64)).to(dev) for v in synth.rss_share(x, ELL, run=rank)]
        yr = tuple(torch.empty_like(xr[0]) for _ in range(3))
        f_rss = getattr(api, a.op)
        step = lambda: f_rss(*xr, prm, seeds, base, out=yr, stream=stream)  # noqa: E731
    t_ms, per, clocks = timed(step, a.steps, max(a.warmup, 3), clocks=ck)
    ms = t_ms / a.steps
    value = world * n / (ms * 1e-3)
    peaks = load_peaks()
    traffic = load_traffic()
    alu_ops = load_alu_ops()
    clk_mhz = peaks["sm_max_mhz"]
    # ALU pipe (LOP3/SHF/PRMT/IADD3): 1 warp instruction per 2 clk per SMSP = 16 lanes/clk/SMSP
    sms = torch.cuda.get_device_properties(dev).multi_processor_count or SM_COUNT_B200
    alu_peak = sms * 4 * 16 * clk_mhz * 1e6 / 1e12  # Tops/s

    def roofline(kind, elems_per_s, launch_ms):
        bytes_ = BYTES_PER_ELEM[kind]
        hbm_gbs = elems_per_s * bytes_ / 1e9 / max(world, 1)
        out = {"hbm": {"achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": hbm_gbs / peaks["hbm_gbs"], "bytes_per_elem": bytes_}}
        if kind in BLOCKS_PER_ELEM:
            ops = BLOCKS_PER_ELEM[kind] * CHACHA_ALU_OPS_PER_BLOCK[a.rounds]
            ach = elems_per_s / max(world, 1) * ops / 1e12
            out.update({"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "Tops/s", "frac": ach / alu_peak,
                        "ops_per_elem": ops,
                        "ops_note": "ChaCha xor+rotate word ops (ALU pipe) per element; protocol ops not counted",
                        "peak_note": f"ALU pipe: {sms} SM x 4 SMSP x 16 lanes/clk x {clk_mhz:.0f} MHz ({peaks['src']} sm_max)"})
        else:
            out.update({"bound": "hbm", "achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_gbs / peaks["hbm_gbs"]})
        tr = traffic.get(kind)
        out["traffic"] = tr
        out["launch_ms"] = launch_ms
        out["hbm_frac"] = out["hbm"]["frac"]
        ex = alu_ops.get(kind)
        if ex and out["bound"] == "alu":  # every ALU-pipe instruction the kernel executes (ncu), not just ChaCha's
            ach_ex = elems_per_s / max(world, 1) * ex / 1e12
            out.update({"alu_ops_per_elem_executed": ex, "alu_achieved_executed": ach_ex,
                        "alu_frac_executed": ach_ex / alu_peak, "alu_ops_source": alu_ops.get("_source")})
        return out

    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": a.steps,
        "warmup": max(a.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded; shares of D2 activations)",
        "config": workload_config(a),
        "roofline": roofline(a.op, value, ms),
        "gpu_launches": a.steps,
        "clocks": clocks,
    }

    if not a.no_extras:
        # ---- the headline kernel with BOTH parties' messages reduced to wire values (P2 adds W0 + W1
        # in [0, 257), as the transcript path and the party kernels do); the headline reduces P0's
        # and tests it against P1's congruent message (BC_MATERIALIZE) ----
        os.environ["BICOPTOR_MATERIALIZE"] = "2"
        try:
            t_m2, _, _ = timed(step, max(a.steps // 2, 5), 3)
        finally:
            del os.environ["BICOPTOR_MATERIALIZE"]
        ms_m2 = t_m2 / max(a.steps // 2, 5)
        line["materialize2"] = {"value": world * n / (ms_m2 * 1e-3), "unit": "elements/s", "ms_per_step": ms_m2,
                                "note": "same kernel, both wire values W0, W1 in [0, 257) formed per slot and added "
                                        "by P2 (env BICOPTOR_MATERIALIZE=2); results identical"}
        # ---- ReLU (Alg 8) on the same batch ------------------------------------
        t_ms_r, _, _ = timed(lambda: api.relu(x0, x1, prm, seeds, base, y0, y1, stream=stream),
                             max(a.steps // 2, 5), 3)
        ms_r = t_ms_r / max(a.steps // 2, 5)
        v_r = world * n / (ms_r * 1e-3)
        line["relu"] = {"value": v_r, "unit": "elements/s", "ms_per_step": ms_r, "roofline": roofline("relu", v_r, ms_r)}
        # ---- DReLU across batch sizes: launch-bound small batches to config 3's 2^27 asymptote ----
        sweep = {}
        for lg in (16, 20, 22, 27):
            m = 1 << lg
            xs0 = x0.repeat((m + n - 1) // n)[:m] if m > n else x0[:m]
            xs1 = x1.repeat((m + n - 1) // n)[:m] if m > n else x1[:m]
            ys0, ys1 = torch.empty_like(xs0), torch.empty_like(xs1)
            reps = max(5, min(200, (1 << 28) // m))
            # its own global index range per rank (disjoint from the headline's and the other ranks')
            sb = SWEEP_BASE + shard.elem_base(rank, 1 << 27)
            tv, _, _ = timed(lambda: api.drelu(xs0, xs1, prm, seeds, sb, ys0, ys1, stream=stream), reps, 3)
            sweep[f"2^{lg}"] = world * m / (tv / reps * 1e-3)
            del xs0, xs1, ys0, ys1
        sweep["2^24"] = value
        line["drelu_batch_sweep"] = {"unit": "elements/s", **dict(sorted(sweep.items(), key=lambda kv: int(kv[0][2:]))),
                                     "note": "2^27: the headline batch's shares tiled; smaller batches are prefixes"}
        # ---- ChaCha round-count variants of DReLU --------------------------------
        var = {}
        for R in (12, 8):
            if R == a.rounds:
                continue
            pr = api.Params(ell=ELL, lx=LX, f=F, mode=MODE, rounds=R)
            tv, _, _ = timed(lambda: api.drelu(x0, x1, pr, seeds, base, y0, y1, stream=stream), 50, 3)
            tr_, _, _ = timed(lambda: api.relu(x0, x1, pr, seeds, base, y0, y1, stream=stream), 50, 3)
            var[f"chacha{R}"] = {"drelu": world * n / (tv / 50 * 1e-3), "relu": world * n / (tr_ / 50 * 1e-3)}
        # the paper-literal domain Z_{2^lx} (p = 131, 64-bit messages; reading C6: it mis-signs a band of
        # negatives, so guard mode is the default): the pair tape, one ChaCha block per two elements
        pl = api.Params(ell=ELL, lx=LX, f=F, mode="literal", rounds=a.rounds)
        tl_, _, _ = timed(lambda: api.drelu(x0, x1, pl, seeds, base, y0, y1, stream=stream), 50, 3)
        var["literal"] = {"drelu": world * n / (tl_ / 50 * 1e-3),
                          "note": "mode=literal (w = lx = 7, p = 131): pair tape (28-bit (r, rho) draws), 32 B of keystream per element"}
        line["variants"] = var
        # ---- config 2: ladder + modswitch (Alg 7 steps 3-5), HBM-bound, at config 2's 2^28 ----
        n2 = 1 << 28
        x_c2 = x0.repeat((n2 + n - 1) // n)[:n2]  # the headline batch's shares tiled to 2^28 (2 GiB)
        v_lad = torch.empty((n2, 8), dtype=torch.uint8, device=dev)
        tl, _, _ = timed(lambda: api.ladder_modswitch(0, x_c2, prm, out=v_lad, stream=stream), 20, 3)
        ms_l = tl / 20
        v_l = world * n2 / (ms_l * 1e-3)
        line["trc_modswitch"] = {"value": v_l, "unit": "elements/s", "ms_per_step": ms_l, "n_per_gpu": n2,
                                 "roofline": roofline("ladder", v_l, ms_l),
                                 "note": "config 2: one party, 8 B in + 8 B out per element, 2^28 elements "
                                         "(the headline batch's shares tiled)"}
        del v_lad, x_c2
        # ---- every party's work unshared: the party-phase kernels chained on 1 GPU ----
        line["party_chain_1gpu"] = party_chain(api, prm, seeds, x0, x1, base, dev, stream, timed, world, n)
        # ---- RSS variant (Alg 9): DReLU / ReLU on replicated shares of the same x ----
        line["rss"] = rss_leg(api, prm, seeds, x, base, dev, stream, timed, world, n, roofline, rank)
        # ---- full precision lx = 31, f = 0 (no key bits; large tape, p = 2^32 + 15) ----
        pfp = api.Params(ell=ELL, lx=31, f=0, mode=MODE, rounds=a.rounds)
        fp = {}
        for name, fn in (("drelu_fp", api.drelu), ("relu_fp", api.relu)):
            t_fp, _, _ = timed(lambda: fn(x0, x1, pfp, seeds, base, y0, y1, stream=stream), 10, 3)
            ms_fp = t_fp / 10
            v_fp = world * n / (ms_fp * 1e-3)
            fp[name] = {"value": v_fp, "unit": "elements/s", "ms_per_step": ms_fp,
                        "roofline": roofline(name, v_fp, ms_fp)}
        fp["party_chain_1gpu"] = party_chain(api, pfp, seeds, x0, x1, base, dev, stream, timed, world, n)
        # the paper-literal domain at full precision (w = 31, p = 2^31 + 11: "31 * 31 ~ 1,000 bits")
        plit = api.Params(ell=ELL, lx=31, f=0, mode="literal", rounds=a.rounds)
        for name, fn in (("drelu", api.drelu), ("relu", api.relu)):
            t_fp, _, _ = timed(lambda: fn(x0, x1, plit, seeds, base, y0, y1, stream=stream), 10, 3)
            fp.setdefault("literal", {})[name] = {"value": world * n / (t_fp / 10 * 1e-3), "unit": "elements/s",
                                                  "ms_per_step": t_fp / 10}
        fp["note"] = ("lx=31, f=0, guard (w=32, p=2^32+15, 32 slots): the paper's full 5+26 precision, same batch; "
                      "literal: w=31, p=2^31+11 (the paper's own domain; C6's false positives apply)")
        line["full_precision"] = fp
        # ---- Bicoptor-1 as the paper describes it (NEXT #4), same batch and seeds ----
        t_b1, _, _ = timed(lambda: api.drelu_b1(x0, x1, prm, seeds, base, y0, y1, stream=stream), 20, 3)
        line["bicoptor1"] = {
            "drelu": {"value": world * n / (t_b1 / 20 * 1e-3), "unit": "elements/s", "ms_per_step": t_b1 / 20},
            "one_pass_bits_per_party": (LX + 1) * ELL, "bicoptor2_one_pass_bits_per_party": (LX + 1) * 9,
            "note": "SecureML truncation, recursive sums, no modulo switch, 64-bit masks (readings C32-C34); "
                    "3 ChaCha blocks per element vs 0.5",
        }
        # ---- truncation study (NEXT #3): exact e1 counting, Alg 3 vs mult-then-trc ----
        line["trunc_study"] = trunc_leg(api, seeds, x0, x1, base, dev, stream, timed, world, n)
        # ---- config 5: E2E-shaped ReLU layer streams (CUDA graph per network) ----
        line["config5"] = relu_streams(api, prm, seeds, dev, stream, timed, world, rank)
        # ---- e2e through the public API with pinned HOST buffers ----------------
        line["e2e"] = e2e(api, prm, seeds, x0h, x1h, base, dev, world, max_over_ranks, barrier, a)
    if rank == 0 and world == 1 and not a.no_extras:  # the CPU baseline: rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline(a.rounds)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def party_chain(api, prm, seeds, x0, x1, base, dev, stream, timed, world, n):
    """The fused kernel expands seed01 once for both simulated computing parties.
    In a deployment each party expands its own seeds; this leg runs the party
    kernels back to back on one GPU (P0 send, P1 send, P2 helper, P0 finish, P1
    finish), i.e. every party's PRG and arithmetic, no sharing."""
    import torch
    lo0, hi0, tb0 = api.msg_buffers(n, dev, prm)
    lo1, hi1, tb1 = api.msg_buffers(n, dev, prm)
    r1 = torch.empty(n, dtype=torch.int64, device=dev)
    ya, yb = torch.empty_like(r1), torch.empty_like(r1)
    d0, d1, e, c1 = (torch.empty_like(r1) for _ in range(4))

    def drelu_chain():
        api.drelu_send(0, x0, prm, seeds.s01, base, out=(lo0, hi0, tb0), stream=stream)
        api.drelu_send(1, x1, prm, seeds.s01, base, out=(lo1, hi1, tb1), stream=stream)
        api.drelu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, base, out=(None, r1), stream=stream)
        api.drelu_finish(0, tb0, None, prm, n, seeds.s02, base, out=ya, stream=stream)
        api.drelu_finish(1, tb1, r1, prm, n, None, base, out=yb, stream=stream)

    def relu_chain():
        api.relu_send(0, x0, prm, seeds.s01, seeds.s02, base, out=(lo0, hi0, tb0, d0), stream=stream)
        api.relu_send(1, x1, prm, seeds.s01, seeds.s12, base, out=(lo1, hi1, tb1, d1), stream=stream)
        api.relu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, seeds.s12, base, out=(e, c1), stream=stream)
        api.relu_finish(0, x0, tb0, d0, d1, e, None, prm, seeds.s02, base, out=ya, stream=stream)
        api.relu_finish(1, x1, tb1, d1, d0, e, c1, prm, seeds.s12, base, out=yb, stream=stream)

    res = {}
    reps = 50 if prm.lx <= 7 else 5
    for name, fn in (("drelu", drelu_chain), ("relu", relu_chain)):
        t_ms, _, _ = timed(fn, reps, 3)
        ms = t_ms / reps
        res[name] = {"value": world * n / (ms * 1e-3), "unit": "elements/s", "ms_per_step": ms, "launches_per_step": 5}
    # each party's kernels alone (inputs left in place by the chains above): what one GPU per party
    # would run per step in config 4.  The rate of a P0/P1/P2 triple on three GPUs is bounded by the
    # slowest party, transfers overlapped -- a projection from measured kernels, not a 3-GPU run.
    per = {}
    for name, calls in (
            ("drelu", {"P0": lambda: api.drelu_send(0, x0, prm, seeds.s01, base, out=(lo0, hi0, None), stream=stream,
                                                    y=ya, seed02=seeds.s02),   # one kernel (bc_drelu_send_p0)
                       "P1": lambda: (api.drelu_send(1, x1, prm, seeds.s01, base, out=(lo1, hi1, tb1), stream=stream),
                                      api.drelu_finish(1, tb1, r1, prm, n, None, base, out=yb, stream=stream)),
                       "P2": lambda: api.drelu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, base, out=(None, r1),
                                                      stream=stream)}),
            ("relu", {"P0": lambda: (api.relu_send(0, x0, prm, seeds.s01, seeds.s02, base, out=(lo0, hi0, tb0, d0),
                                                   stream=stream),
                                     api.relu_finish(0, x0, tb0, d0, d1, e, None, prm, seeds.s02, base, out=ya,
                                                     stream=stream)),
                      "P1": lambda: (api.relu_send(1, x1, prm, seeds.s01, seeds.s12, base, out=(lo1, hi1, tb1, d1),
                                                   stream=stream),
                                     api.relu_finish(1, x1, tb1, d1, d0, e, c1, prm, seeds.s12, base, out=yb,
                                                     stream=stream)),
                      "P2": lambda: api.relu_helper(lo0, hi0, lo1, hi1, prm, seeds.s02, seeds.s12, base,
                                                    out=(e, c1), stream=stream)})):
        ms_p = {}
        for pty, fn in calls.items():
            t_p, _, _ = timed(fn, 3 * reps // 5, 3)
            ms_p[pty] = t_p / (3 * reps // 5)
        per[name] = {"ms_per_party": ms_p,
                     "projected_triple_elements_per_s": n / (max(ms_p.values()) * 1e-3)}
    res["per_party"] = per
    res["note"] = "P0,P1 send + P2 helper + P0,P1 finish back to back on one GPU: all parties' work, nothing shared"
    if prm.lx > 7:  # large tape: uint32 planes, 33 S bits (guard, p > 2^32)
        S = prm.lx + 1
        res["wire_bytes_per_elem"] = {"P0->P2": 4 * S + (4 if prm.mode == "guard" else 0),
                                      "paper_one_pass_bits_per_party": S * S}
        return res
    # the messages these kernels exchange, per element (DESIGN.md sec. 4 wire format) vs Table 1
    slots, pbits = LX + 1, 9 if MODE == "guard" else 8
    res["wire_bytes_per_elem"] = {
        "drelu": {"P0->P2": slots * pbits / 8, "P1->P2": slots * pbits / 8, "P2->P1": 8.0},
        "relu": {"P0->P2": slots * pbits / 8, "P1->P2": slots * pbits / 8, "P0<->P1 (d)": 8.0,
                 "P2->P0,P1 (e)": 8.0, "P2->P1 ([c]_1, preprocessing)": 8.0},
        "one_pass_bits_per_party": slots * pbits,
        "paper_one_pass_bits_per_party": (LX + 1) * (LX + 1),
        "note": "Table 1 counts (lx+1)^2 = 64 bits in the paper's literal domain; guard mode (reading C6) "
                "sends lx+1 slots of ceil(log2 257) = 9 bits = 72",
    }
    return res


def rss_leg(api, prm, seeds, x, base, dev, stream, timed, world, n, roofline, rank):
    """Alg 9 (RSS DReLU) and RSS ReLU, all three parties in one fused kernel, on
    replicated shares of the headline batch."""
    import torch
    import synth
    xs = [torch.from_numpy(v.view(np.int64)).to(dev) for v in synth.rss_share(x, ELL, run=rank)]
    ys = tuple(torch.empty_like(xs[0]) for _ in range(3))
    res = {}
    for name in ("drelu_rss", "relu_rss"):
        fn = getattr(api, name)
        t_ms, _, _ = timed(lambda: fn(*xs, prm, seeds, base, out=ys, stream=stream), 50, 3)
        ms = t_ms / 50
        v = world * n / (ms * 1e-3)
        res[name] = {"value": v, "unit": "elements/s", "ms_per_step": ms, "roofline": roofline(name, v, ms)}
    del xs, ys
    return res


def trunc_leg(api, seeds, x0, x1, base, dev, stream, timed, world, n):
    """Sec. 4-5 kernels: bc_trc_count (every mask of a range against a list of
    x, classified exact / e0 / e1) and the fixed-point product in both orders
    (ABY3 truncation, ell = 64, f = 26: the paper's Piranha setting)."""
    import torch
    res = {}
    xs = torch.arange(1, 4097, dtype=torch.int64, device=dev) << 40       # 4096 band inputs at ell = 64
    counts = torch.zeros((4096, 3), dtype=torch.int64, device=dev)
    m = 1 << 20
    t_ms, _, _ = timed(lambda: api.trc_count("secureml", xs, 64, 26, 0, m, counts=counts, stream=stream), 5, 3)
    res["trc_count"] = {"value": world * 4096 * m / (t_ms / 5 * 1e-3), "unit": "protocol evaluations/s",
                        "ms_per_step": t_ms / 5, "note": "Alg 1 on 4096 inputs x 2^20 masks, classified (C30)"}
    z0, z1 = torch.empty_like(x0), torch.empty_like(x1)
    for order in ("mul_then_trc", "trc_then_mul"):
        t_ms, _, _ = timed(lambda: api.mul_trc(order, "aby3", x0, x1, x0, x1, 64, 26, seeds, base, out=(z0, z1),
                                               stream=stream), 20, 3)
        res[order] = {"value": world * n / (t_ms / 20 * 1e-3), "unit": "products/s", "ms_per_step": t_ms / 20,
                      "note": "x * x on the headline batch (5+26 fixed point)"}
    return res


def relu_streams(api, prm, seeds, dev, stream, timed, world, rank):
    """BASELINE config 5: each network's ReLU layers at the paper's batch
    (Table 7), one fused bc_relu per layer, replayed from a CUDA graph.  Inputs
    are seeded shares generated on the device (torch RNG; input generation is
    outside the timed region and holds none of the method's arithmetic)."""
    import torch
    from paper_2309_04909_b200 import shard
    from paper_2309_04909_b200 import stream as S
    out = {}
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    for name in S.NETWORKS:
        sizes = S.layer_sizes(name)
        # rank r's forward owns its own global index range (fresh randomness on every rank)
        st = S.ReluStream(sizes, prm, seeds, dev, base=STREAM_BASE + shard.elem_base(rank, S.index_span(sizes)))
        for x0, x1 in zip(st.x0, st.x1):
            x = (torch.randn(x0.numel(), device=dev, generator=g) * 2 ** 26).round().to(torch.int64)
            r = torch.randint(-2 ** 63, 2 ** 63 - 1, (x0.numel(),), device=dev, generator=g, dtype=torch.int64)
            x0.copy_(x + r)   # [x]_0 = x + R, [x]_1 = -R  (int64 wraps mod 2^64)
            x1.copy_(-r)
        st.capture()
        steps = 20
        t_ms, _, _ = timed(st.replay, steps, 3)
        ms = t_ms / steps
        out[name] = {"relus": st.total, "layers": len(st.sizes), "ms_per_forward": ms,
                     "relu_per_s": world * st.total / (ms * 1e-3), "launches_per_forward": len(st.sizes)}
        del st
        torch.cuda.empty_cache()
    out["note"] = "per GPU, paper batch (Table 7: 240/60/1650); CUDA graph of one bc_relu per layer"
    return out


def e2e(api, prm, seeds, x0h, x1h, base, dev, world, max_over_ranks, barrier, a):
    """Same metric through the C-ABI host-buffer entry bc_drelu_host (via
    host.HostPipeline): pinned host shares in, pinned host shares out, H2D /
    kernel / D2H pipelined natively in chunks inside the timed region."""
    import torch
    from paper_2309_04909_b200 import host as H
    n = x0h.size
    hx0 = torch.from_numpy(x0h.view(np.int64)).pin_memory()
    hx1 = torch.from_numpy(x1h.view(np.int64)).pin_memory()
    hy0 = torch.empty(n, dtype=torch.int64).pin_memory()
    hy1 = torch.empty(n, dtype=torch.int64).pin_memory()
    chunk = 1 << 23  # tools/diag_e2e.py sweep of the async entry: 2^23 best (2.92 G/s); smaller chunks pay per-copy overhead
    ex = H.HostPipeline(dev, chunk=chunk)
    steps = max(5, a.steps // 20)

    def run(sync):
        for _ in range(2):
            ex.drelu(hx0, hx1, hy0, hy1, prm, seeds, base, sync=sync)
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):  # every step copies its inputs in and its outputs out
            ex.drelu(hx0, hx1, hy0, hy1, prm, seeds, base, sync=sync)
        torch.cuda.synchronize(dev)
        return max_over_ranks(time.perf_counter() - t0)

    dt_sync = run(True)
    dt = run(False)
    return {"value": world * n * steps / dt, "unit": "elements/s", "h2d_bytes_per_step": 16 * n,
            "d2h_bytes_per_step": 16 * n, "chunk": chunk,
            "sync_calls_value": world * n * steps / dt_sync,
            "note": "bc_drelu_host_async (C ABI) per step, back to back as a serving loop: pinned x0,x1 -> HBM -> "
                    "fused DReLU -> pinned y0,y1 over 3 streams; one synchronisation at the end; wall clock, max "
                    "over ranks.  sync_calls_value: bc_drelu_host, which returns with the outputs complete"}


def run_party(a):
    """BASELINE config 4: ReLU with P0, P1, P2 on distinct GPUs, messages as NCCL
    point-to-point over NVLink (paper_2309_04909_b200.party).  World = 3k ranks
    (extra ranks idle); each triple owns party-n elements."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2309_04909_b200 import api, party

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world < 3:
        if rank == 0:
            print(json.dumps({"metric": "config4 party-separated ReLU elements/s", "mode": "party",
                              "unavailable": f"needs >= 3 GPUs (one per party), have {world}"}))
        return
    share = os.environ.get("BENCH_SHARE_GPU") == "1"  # testing aid, see run_cuda: every rank on cuda:0, gloo
    if share:
        local = 0
        if a.transport != "peer":
            raise SystemExit("BENCH_SHARE_GPU=1 needs --transport peer (NCCL cannot put two ranks on one GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    k = world // 3
    group = dist.new_group(list(range(3 * k)))
    # peer transport: doorbells / credits / IPC handles over a gloo group per triple
    gloo_triples = [dist.new_group([3 * t, 3 * t + 1, 3 * t + 2], backend="gloo") for t in range(k)] \
        if a.transport == "peer" else None
    n = a.party_n
    prm = api.Params(ell=ELL, lx=LX, f=F, mode=a.domain, rounds=a.rounds)
    seeds = synth.seeds(0)
    t_ms, bytes_sent, msg_bits = 0.0, 0, 0
    if rank < 3 * k:
        role = party.Role.of(rank)
        xs = None
        if role.party < 2:
            x = synth.plaintext(n, ELL, LX, F, "D2", run=role.triple)
            x0, x1 = synth.share(x, ELL, run=role.triple)
            xs = torch.from_numpy((x0 if role.party == 0 else x1).view(np.int64)).to(dev)
        if a.transport == "peer":
            from paper_2309_04909_b200 import peer
            runner = peer.PeerPartyRunner("relu", prm, seeds, n, chunk=a.chunk, backend=peer.CudaIpcBackend(dev),
                                          group=gloo_triples[role.triple], triples=k)
            step = lambda: runner.run(xs)  # noqa: E731
            # egress per step: every link this rank's kernels store into (P0/P1: message + [d]_b; P2: e to
            # both + [c]_1), from the inbox field shapes
            eg = runner.egress_bytes_per_elem()
            wire = sum(eg.values()) * n
            if role.party < 2:  # the one-pass message to P2 (Alg 7 step 8), in bits per element
                msg_bits = 8 * eg["linkA->P2" if role.party == 0 else "linkB->P2"]
        else:
            runner = party.PartyRunner(prm, seeds, n, chunk=a.chunk, compute=party.CudaCompute(dev), group=group,
                                       triples=k)
            step = lambda: runner.relu(xs)  # noqa: E731
        for _ in range(max(a.warmup, 2)):
            step()
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)
        if a.transport == "nccl":
            runner.bytes_sent = 0
        steps = max(1, min(a.steps, 20))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)
        t_ms = e0.elapsed_time(e1) / steps
        bytes_sent = runner.bytes_sent / steps if a.transport == "nccl" else wire
        if a.transport == "nccl" and role.party < 2:
            fmt = api.wire_format(prm)
            msg_bits = 8 * (8 + (1 if fmt["hi"] is not None else 0))
        if a.transport == "peer":
            runner.close()
    rdev = "cpu" if share else dev
    t = torch.tensor([t_ms, bytes_sent, msg_bits], dtype=torch.float64, device=rdev)
    tm = t.clone()
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    per_rank = [torch.zeros(3, dtype=torch.float64, device=rdev) for _ in range(world)]
    dist.all_gather(per_rank, t)
    if rank == 0:
        ms = float(tm[0])
        egress = {f"P{p}": float(per_rank[p][1]) / n for p in range(3)}
        print(json.dumps({
            "metric": f"config4 party-separated ReLU elements/s (P0,P1,P2 on distinct GPUs, "
                      f"{'NCCL P2P' if a.transport == 'nccl' else 'peer-memory stores from the phase kernels'})",
            "mode": "party", "transport": a.transport, "value": k * n / (ms * 1e-3), "unit": "elements/s", "n_gpus": world, "triples": k,
            "ms_per_step": ms, "steps": steps, "chunk": a.chunk, "higher_is_better": True, "dtype": "u64",
            "config": {"workload": f"config4: ReLU ell={ELL} lx={LX} f={F} {a.domain} ChaCha{a.rounds}, 2^{int(math.log2(n))} elements per triple"},
            "wire_bytes_per_elem": egress,
            "one_pass_bits_per_party": {"P0->P2": float(per_rank[0][2]), "P1->P2": float(per_rank[1][2])},
            "paper_one_pass_bits": (LX + 1) * (LX + 1), "guard_one_pass_bits": (LX + 1) * 9,
            "p2_egress_GBs": float(per_rank[2][1]) / (ms * 1e-3) / 1e9}))
    dist.destroy_process_group()


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "party":
        run_party(args)
    else:
        run_cuda(args)
