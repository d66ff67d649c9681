"""B200-native hot path of Bicoptor 2.0 (arXiv 2309.04909): UBL DReLU / ReLU.

The compute path is libbicoptor.so (hand-written sm_100a CUDA behind the C ABI
in include/bicoptor.h); this package is its thin Python binding (``api``) plus
the party-separated runtime (``party``).  Import is light: the library is
loaded on first use and there is no CPU fallback.
"""
__all__ = ["api"]
