"""bench.py's output contract on CPU: the reference arm (the oracle on the host
cores, tier framing 4) prints one JSON line with the keys the driver reads; the
product binding refuses CPU tensors (there is no CPU fallback)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = {**os.environ, "BENCH_REF_BUDGET_S": "4"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "elements/s" and line["value"] > 0
    assert line["warmup"] >= 3 and line["steps"] == 2
    assert line["config"]["workload"].startswith("config3")
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["unit"] == line["unit"]


def test_no_cpu_path():
    """The product path has no CPU fallback: CPU tensors are refused before any launch."""
    import pytest
    import torch

    from paper_2309_04909_b200 import api, build
    build.build()
    import synth
    x = torch.zeros(16, dtype=torch.int64)
    with pytest.raises(api.BicoptorError, match="CUDA tensor"):
        api.drelu(x, x.clone(), api.Params(), synth.seeds(0))
    with pytest.raises(api.BicoptorError, match="CUDA tensor"):
        api.ladder_modswitch(0, x, api.Params())
