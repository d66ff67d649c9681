"""Build and time tuning variants of the fused kernel (compile-time knobs).

    python tools/variants.py build           # here (CPU): builds paper_2309_04909_b200/variants/*.so
    python tools/variants.py time            # on the GPU box: times each variant (DReLU, R20 and R8;
                                             # VARIANT_OP=relu|drelu_fp|relu_fp|drelu_rss|relu_rss
                                             # times that op instead)
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2309_04909_b200", "variants")
KNOBS = {"BC_ADD_FMA_SEND": [0, 1]}  # knobs in csrc/: also BC_ADD_FMA, BC_MATERIALIZE, BC_FUSED_MINB, BC_ROT_FMA, BC_CHACHA_UNROLL


def variants():
    if os.environ.get("VARIANT_LIST"):  # explicit list: '[{"BC_X": 1}, {}, ...]' ({} = the product library's knobs)
        yield from json.loads(os.environ["VARIANT_LIST"])
        return
    keys = list(KNOBS)
    for vals in itertools.product(*(KNOBS[k] for k in keys)):
        yield dict(zip(keys, vals))


def name(v):
    return "_".join(f"{k.replace('BC_', '').lower()}{x}" for k, x in v.items()) or "default"


if __name__ == "__main__":
    if sys.argv[1] == "build":
        from paper_2309_04909_b200 import build as b
        os.makedirs(VDIR, exist_ok=True)
        for v in variants():
            out = os.path.join(VDIR, f"lib_{name(v)}.so")
            b.build(defines=[f"{k}={x}" for k, x in v.items()], out=out)
            print(out)
    else:
        res = {}
        for v in variants():
            lib = os.path.join(VDIR, f"lib_{name(v)}.so")
            out = {}
            for R in (20, 8):
                r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-extras", "--steps", "300",
                                    "--rounds", str(R)] + (["--op", os.environ["VARIANT_OP"]] if "VARIANT_OP" in os.environ else []),
                                   capture_output=True, text=True,
                                   env={**os.environ, "BICOPTOR_LIB": lib})
                try:
                    out[f"R{R}_ms"] = json.loads(r.stdout.strip().splitlines()[-1])["ms_per_step"]
                except Exception as e:
                    out[f"R{R}_err"] = (r.stderr or str(e))[-300:]
            res[name(v)] = out
            print(name(v), out, flush=True)
        json.dump(res, open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w"), indent=1)
