"""profiles/ncu_alu_ops.json from the SASS-mix summaries of one profiling round:
executed ALU-pipe thread instructions per element per op (read by bench.py).

    python tools/alu_ops_json.py r2g    # reads profiles/r2g_<op>_sass_mix.txt
"""
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = {"_source": f"ncu --set full source-level SASS mix ({tag}): ALU-pipe thread instructions executed per element"}
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{tag}_*_sass_mix.txt"))):
    op = os.path.basename(f)[len(tag) + 1:-len("_sass_mix.txt")]
    m = re.search(r"pipe alu\s+([0-9.]+)", open(f).read())
    if m:
        out[op] = float(m.group(1))
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_alu_ops.json"), "w"), indent=1)
print(out)
