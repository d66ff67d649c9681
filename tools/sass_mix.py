"""Dynamic SASS instruction mix of a profiled kernel, per processed element.

    python tools/sass_mix.py gpurun_out/prof_<op>.ncu-rep <elements> [--top N]

Reads `ncu --page source --print-source sass` (per-instruction executed
counts), classifies opcodes by pipe (B300_MICROARCH.md: LOP3/SHF/PRMT/IADD3/
SEL/ISETP/... on the ALU pipe, IMAD* on the FMA pipe, IMAD.HI/WIDE at half
rate), and prints thread-instructions per element by opcode and by pipe.
"""
import csv
import io
import subprocess
import sys
from collections import Counter

ALU = {"LOP3", "SHF", "PRMT", "IADD3", "SEL", "ISETP", "LEA", "VIMNMX3", "VIMNMX", "IMNMX", "FLO", "POPC",
       "LOP", "SHL", "SHR", "BMSK", "PLOP3", "IABS", "ICMP"}
FMA = {"IMAD", "IMUL", "FFMA", "FADD", "FMUL", "VIADD"}  # VIADD measured to co-issue with LOP3 (tools/intpipe_bench.cu)


def pipe_of(op: str) -> str:
    base = op.split(".")[0]
    if base in ("IMAD", "IMUL") and (".HI" in op or ".WIDE" in op):
        return "fma_heavy"
    if base in ALU:
        return "alu"
    if base in FMA:
        return "fma"
    if base in ("LDG", "STG", "LDS", "STS", "LDL", "STL", "LD", "ST", "ATOMS", "ATOMG", "RED", "LDSM"):
        return "lsu"
    if base.startswith("U") or base in ("R2UR", "S2UR"):
        return "uniform"
    if base in ("BRA", "BSSY", "BSYNC", "CALL", "RET", "EXIT", "WARPSYNC", "BAR", "NOP"):
        return "control"
    if base in ("MOV", "S2R", "CS2R", "LDC", "LDCU"):
        return "mov/const"
    return "other"


def main():
    rep, elems = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    si, ti = h.index("Source"), h.index("Thread Instructions Executed")
    by_op, by_pipe = Counter(), Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= ti or not r[ti].strip() or r[0] == "Address":  # reports with several kernels repeat the header
            continue
        text = r[si].strip()
        if text.startswith("@"):
            text = text.split(" ", 1)[1].strip()
        op = text.split(" ")[0].rstrip(";")
        n = float(r[ti])
        by_op[op] += n
        by_pipe[pipe_of(op)] += n
    tot = sum(by_op.values())
    print(f"thread instructions per element: {tot / elems:.1f}")
    for k, v in by_pipe.most_common():
        print(f"  pipe {k:10s} {v / elems:8.1f}")
    for k, v in by_op.most_common(top):
        print(f"  {k:28s} {v / elems:8.1f}   [{pipe_of(k)}]")


if __name__ == "__main__":
    main()
