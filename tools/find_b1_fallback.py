"""Write tests/golden/b1_fallback.txt: element indices j whose Bicoptor-1 tape
(oracle.bicoptor1, reading C34) rejects the permutation index (word 0 & 0x7fffffff
>= floor(2^31/8!) 8!), so the GPU test can exercise the fallback stream.  Calls
only oracle/ (the stored values are the oracle's)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import bicoptor1 as B1  # noqa: E402
from oracle.chacha import chacha_blocks  # noqa: E402

seed01 = synth.seeds(0).s01
lim = (2**31 // 40320) * 40320
found = []
step = 1 << 21
for lo in range(0, 1 << 27, step):
    j = np.arange(lo, lo + step, dtype=np.uint64)
    w0 = chacha_blocks(seed01, B1.L_TAPE1, 3 * j, 20)[:, 0] & np.uint32(0x7FFFFFFF)
    found += [int(v) for v in j[w0 >= np.uint32(lim)]]
    if len(found) >= 3:
        break
with open(os.path.join(ROOT, "tests", "golden", "b1_fallback.txt"), "w") as f:
    f.write("# element indices whose Bicoptor-1 tape (seed run 0, ChaCha20) rejects the perm index;\n")
    f.write("# written by tools/find_b1_fallback.py from oracle/ only\n")
    for v in found[:3]:
        f.write(f"{v}\n")
print(found[:3])
