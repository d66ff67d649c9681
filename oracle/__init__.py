"""CPU oracle for the Bicoptor 2.0 DReLU/ReLU hot path (arXiv 2309.04909).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2309_04909_b200``)
may import, call, link or execute anything under ``oracle/``.  The only
permitted callers are ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.

The oracle is a plain, slow, obviously-correct numpy implementation written
from the paper (``/root/reference/PAPER.md``; citations are ``P:<line>``) in
the paper's order and notation.  It shares no code, tables or constants with
the CUDA path; the only module both sides use is ``synth/`` (seeded input
generation, which holds none of the method's arithmetic).

Modules
  chacha    -- RFC 8439 ChaCha block function and keystream addressing (the
               PRG the paper leaves unnamed; reading C19 in DESIGN.md).
  ring      -- cut / LT / Alg 1, 4, 5 truncation / Alg 6 modulo switch.
  bicoptor  -- Alg 7 UBL DReLU, Alg 8 UBL ReLU, per party and composed; the
               compact, pair and large (full precision) tapes; wire formats.
  rss       -- Alg 9 RSS DReLU and the RSS ReLU.
  trunc     -- the truncation study: Alg 1 / 2 e0-e1 classes, exact mask counting,
               Alg 3 trc-then-mult against mult-then-trc.
  bicoptor1 -- Bicoptor-1's DReLU as Bicoptor 2.0 describes it.

Pins (what fixes each function independently of itself) are listed in
DESIGN.md section "Oracle and its pins"; functions without one say
"parity unpinned" in their docstring.
"""
