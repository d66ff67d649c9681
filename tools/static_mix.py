"""Static SASS mix of one kernel under compile-time knobs (no GPU): differences
between variants of the straight-line protocol code show up directly (loops are
counted once, so absolute totals are not per-element counts).

    python tools/static_mix.py <kernel-substring> [-DKNOB=V ...] [--src bc_fused.cu]
"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sass_mix import pipe_of  # noqa: E402
from paper_2309_04909_b200 import build as B  # noqa: E402


def mix(kernel: str, defines, src="bc_fused.cu"):
    with tempfile.TemporaryDirectory() as d:
        obj = os.path.join(d, "k.o")
        cmd = [B.nvcc()] + B.ARCH + B.FLAGS + list(defines) + ["-c", os.path.join(B.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True, capture_output=True)
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0]
        if kernel in name and "$" not in name:
            ops = Counter()
            for line in f.split("\n"):
                m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
                if m:
                    ops[m.group(2)] += 1
            return name, ops
    raise SystemExit(f"no kernel matching {kernel}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-D") and not a.startswith("--src")]
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    src = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--src=")), "bc_fused.cu")
    name, ops = mix(args[0], defs, src)
    pipes = Counter()
    for op, n in ops.items():
        pipes[pipe_of(op)] += n
    print(name[:110])
    print("total", sum(ops.values()), dict(pipes.most_common()))
    print(", ".join(f"{o} {n}" for o, n in ops.most_common(24)))
