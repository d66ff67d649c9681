"""Thin Python binding of libbicoptor (include/bicoptor.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  PyTorch provides device memory and streams.
There is no CPU fallback: if the shared library is missing or a tensor is not
on a CUDA device, the call raises.

Share vectors are 1-D CUDA tensors of 8-byte elements (torch.int64 or
torch.uint64) holding Z_{2^ell} values bit for bit.
"""
from __future__ import annotations

import ctypes
import functools
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbicoptor.so")

MODE = {"guard": 0, "literal": 1}

c_u64p = ctypes.c_void_p


class BicoptorError(RuntimeError):
    pass


class bc_params(ctypes.Structure):
    _fields_ = [("ell", ctypes.c_int32), ("lx", ctypes.c_int32), ("f", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("rounds", ctypes.c_int32), ("w", ctypes.c_uint32),
                ("slots", ctypes.c_uint32), ("tape", ctypes.c_int32), ("p", ctypes.c_uint64)]


TAPE = {0: "pair", 1: "compact", 2: "large", 3: "compact_lit"}


class bc_seeds(ctypes.Structure):
    _fields_ = [("s01", ctypes.c_uint8 * 32), ("s02", ctypes.c_uint8 * 32), ("s12", ctypes.c_uint8 * 32)]


class bc_transcript(ctypes.Structure):
    _fields_ = [("w0_lo", ctypes.c_void_p), ("w0_hi", ctypes.c_void_p),
                ("w1_lo", ctypes.c_void_p), ("w1_hi", ctypes.c_void_p)]


# name -> (restype, argtypes); mirrors include/bicoptor.h
_P = ctypes.c_void_p
_SIG = {
    "bc_version": (ctypes.c_int, []),
    "bc_last_cuda_error": (ctypes.c_int, []),
    "bc_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "bc_params_init": (ctypes.c_int, [ctypes.POINTER(bc_params), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int]),
    "bc_trc": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "bc_trc_prob": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, _P]),
    "bc_modswitch": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, _P]),
    "bc_ladder_modswitch": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.POINTER(bc_params), _P]),
    "bc_modswitch64": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64, _P]),
    "bc_ladder_modswitch64": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.POINTER(bc_params), _P]),
    "bc_drelu": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                ctypes.POINTER(bc_seeds), ctypes.POINTER(bc_transcript), _P]),
    "bc_relu": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                               ctypes.POINTER(bc_seeds), ctypes.POINTER(bc_transcript), _P]),
    "bc_drelu_send": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                     ctypes.POINTER(bc_params), ctypes.c_char_p, _P]),
    "bc_drelu_send_p0": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                        ctypes.POINTER(bc_params), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_drelu_helper": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                       ctypes.POINTER(bc_params), ctypes.c_char_p, _P]),
    "bc_drelu_finish": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                       ctypes.POINTER(bc_params), ctypes.c_char_p, _P]),
    "bc_relu_send": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                    ctypes.POINTER(bc_params), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_relu_helper": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                      ctypes.POINTER(bc_params), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_relu_finish": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                      ctypes.POINTER(bc_params), ctypes.c_char_p, _P]),
    "bc_relu_send_to": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                       ctypes.POINTER(bc_params), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_relu_helper_to": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                         ctypes.POINTER(bc_params), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_ipc_export": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]),
    "bc_ipc_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bc_ipc_close": (ctypes.c_int, [_P]),
    "bc_drelu_b1": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                   ctypes.POINTER(bc_seeds), ctypes.POINTER(bc_transcript), _P]),
    "bc_host_workspace_bytes": (ctypes.c_size_t, [ctypes.c_size_t]),
    "bc_drelu_host": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                     ctypes.POINTER(bc_seeds), _P, ctypes.c_size_t, ctypes.c_size_t, _P]),
    "bc_relu_host": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                    ctypes.POINTER(bc_seeds), _P, ctypes.c_size_t, ctypes.c_size_t, _P]),
    "bc_drelu_host_async": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                           ctypes.POINTER(bc_params), ctypes.POINTER(bc_seeds), _P, ctypes.c_size_t,
                                           ctypes.c_size_t, _P]),
    "bc_relu_host_async": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                          ctypes.POINTER(bc_params), ctypes.POINTER(bc_seeds), _P, ctypes.c_size_t,
                                          ctypes.c_size_t, _P]),
    "bc_trc_aby3": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, ctypes.POINTER(bc_seeds), _P]),
    "bc_trc_count": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_uint64, _P, _P]),
    "bc_mul_trc": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(bc_seeds), _P]),
    "bc_drelu_rss": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                    ctypes.POINTER(bc_seeds), ctypes.c_char_p, ctypes.c_char_p, _P]),
    "bc_relu_rss": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_uint64, ctypes.POINTER(bc_params),
                                   ctypes.POINTER(bc_seeds), ctypes.c_char_p, ctypes.c_char_p, _P]),
}
EXPORTS = tuple(_SIG)

_lib = None


def lib() -> ctypes.CDLL:
    """Load libbicoptor.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        path = os.environ.get("BICOPTOR_LIB", LIB_PATH)  # tuning experiments load a variant build
        if not os.path.exists(path):
            raise BicoptorError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIG.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().bc_strerror(rc).decode()
        if rc == -4:
            msg += f" (cudaError {lib().bc_last_cuda_error()})"
        raise BicoptorError(f"{what}: {msg} [{rc}]")


@dataclass(frozen=True)
class Params:
    """Protocol parameters (see bc_params in include/bicoptor.h)."""
    ell: int = 64
    lx: int = 7
    f: int = 24
    mode: str = "guard"
    rounds: int = 20

    def c(self) -> bc_params:
        """The derived bc_params (bc_params_init), cached per parameter set: the C side only reads it."""
        key = (self.ell, self.lx, self.f, self.mode, self.rounds)
        p = _PARAMS_CACHE.get(key)
        if p is None:
            p = bc_params()
            _check(lib().bc_params_init(ctypes.byref(p), self.ell, self.lx, self.f, MODE[self.mode], self.rounds),
                   "bc_params_init")
            _PARAMS_CACHE[key] = p
        return p


_PARAMS_CACHE: dict = {}
_SEEDS_CACHE: dict = {}


def seeds_struct(seeds) -> bc_seeds:
    key = (bytes(seeds.s01), bytes(seeds.s02), bytes(seeds.s12))
    s = _SEEDS_CACHE.get(key)
    if s is not None:
        return s
    if len(_SEEDS_CACHE) > 64:
        _SEEDS_CACHE.clear()
    s = _SEEDS_CACHE[key] = bc_seeds()
    for name in ("s01", "s02", "s12"):
        v = getattr(seeds, name)
        assert len(v) == 32
        ctypes.memmove(getattr(s, name), v, 32)
    return s


def _dev(t: torch.Tensor, name: str, itemsize: int | None = 8) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise BicoptorError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if not t.is_contiguous():
        raise BicoptorError(f"{name} must be contiguous")
    if itemsize is not None and t.element_size() != itemsize:
        raise BicoptorError(f"{name} must have {itemsize}-byte elements")
    return t.data_ptr()


def _opt(t, name, itemsize=8):
    return None if t is None else _dev(t, name, itemsize)


def _need(t, name: str, nbytes: int) -> None:
    """The C ABI takes raw pointers and cannot see buffer sizes: refuse a caller buffer
    smaller than the call will read or write (None = not passed)."""
    if t is not None and t.numel() * t.element_size() < nbytes:
        raise BicoptorError(f"{name} holds {t.numel() * t.element_size()} B, the call needs {nbytes} B")


def _need_msg(lo, hi, n: int, prm: "Params", what: str) -> None:
    """Message planes of n elements in the wire format of prm (wire_format)."""
    fmt = wire_format(prm)
    (los, lot), hf = fmt["lo"], fmt["hi"]
    isz = torch.empty((), dtype=lot).element_size()
    _need(lo, f"{what} lo", n * los[0] * isz)
    if hf is not None:
        _need(hi, f"{what} hi", n * torch.empty((), dtype=hf[1]).element_size())


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _on_input_device(fn):
    """Run the call with the device of its first CUDA tensor argument current, so
    the library launches (and allocates outputs) where the inputs live, whatever
    device the caller has current.  The first tensor argument of every entry is
    local memory (an input share, a local inbox, the workspace); outputs may be
    peer mappings (peer.py)."""
    @functools.wraps(fn)
    def run(*args, **kw):
        for a in list(args) + list(kw.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                with torch.cuda.device(a.device):
                    return fn(*args, **kw)
        return fn(*args, **kw)
    return run


def empty_u64(n: int, device) -> torch.Tensor:
    return torch.empty(n, dtype=torch.int64, device=device)


# ---- elementwise primitives --------------------------------------------------------

@_on_input_device
def trc(party: int, x: torch.Tensor, ell: int, k1: int, k2: int = 0, out=None, stream=None) -> torch.Tensor:
    """Alg 4 / Alg 5 deterministic truncation of one party's share."""
    out = torch.empty_like(x) if out is None else out
    _check(lib().bc_trc(party, _dev(x, "x"), _dev(out, "out"), x.numel(), ell, k1, k2, _stream(stream)), "bc_trc")
    return out


@_on_input_device
def trc_prob(party: int, x: torch.Tensor, ell: int, k: int, out=None, stream=None) -> torch.Tensor:
    """Alg 1 SecureML probabilistic truncation of one party's share."""
    out = torch.empty_like(x) if out is None else out
    _check(lib().bc_trc_prob(party, _dev(x, "x"), _dev(out, "out"), x.numel(), ell, k, _stream(stream)), "bc_trc_prob")
    return out


@_on_input_device
def modswitch(party: int, x: torch.Tensor, lp: int, p: int, out=None, stream=None) -> torch.Tensor:
    """Alg 6 modulo switch Z_{2^lp} -> Z_p of one party's share (uint32 out, in int32 storage)."""
    out = torch.empty(x.numel(), dtype=torch.int32, device=x.device) if out is None else out
    _need(out, "out", 4 * x.numel())
    _check(lib().bc_modswitch(party, _dev(x, "x"), _dev(out, "out", 4), x.numel(), lp, p, _stream(stream)),
           "bc_modswitch")
    return out


@_on_input_device
def ladder_modswitch(party: int, x: torch.Tensor, prm: Params, out=None, stream=None) -> torch.Tensor:
    """Alg 7 steps 3-5 on one party's share: (n, 8) uint8, byte m = v'_m - 1."""
    out = torch.empty((x.numel(), 8), dtype=torch.uint8, device=x.device) if out is None else out
    _need(out, "out", 8 * x.numel())
    _check(lib().bc_ladder_modswitch(party, _dev(x, "x"), _dev(out, "out", 1), x.numel(), ctypes.byref(prm.c()),
                                     _stream(stream)), "bc_ladder_modswitch")
    return out


@_on_input_device
def modswitch64(party: int, x: torch.Tensor, lp: int, p: int, out=None, stream=None) -> torch.Tensor:
    """Alg 6 at any width 1 <= lp <= 63, 2^lp < p < 2^64 (uint64 out, in int64 storage)."""
    out = torch.empty_like(x) if out is None else out
    _need(out, "out", 8 * x.numel())
    _check(lib().bc_modswitch64(party, _dev(x, "x"), _dev(out, "out"), x.numel(), lp, p, _stream(stream)),
           "bc_modswitch64")
    return out


@_on_input_device
def ladder_modswitch64(party: int, x: torch.Tensor, prm: Params, out=None, stream=None) -> torch.Tensor:
    """Alg 7 steps 3-5 on one party's share, any tape: (n, slots) uint64 (int64 storage), the v'_m."""
    S = prm.lx + 1
    out = torch.empty((x.numel(), S), dtype=torch.int64, device=x.device) if out is None else out
    _need(out, "out", 8 * S * x.numel())
    _check(lib().bc_ladder_modswitch64(party, _dev(x, "x"), _dev(out, "out"), x.numel(), ctypes.byref(prm.c()),
                                       _stream(stream)), "bc_ladder_modswitch64")
    return out


# ---- fused three-party (simulated on one GPU) ----------------------------------------

def _fused(fn, what, x0, x1, prm, seeds, elem_base, y0, y1, transcript, stream):
    n = x0.numel()
    if x1.numel() != n:
        raise BicoptorError("x0 and x1 differ in length")
    y0 = torch.empty_like(x0) if y0 is None else y0
    y1 = torch.empty_like(x1) if y1 is None else y1
    _need(y0, "y0", 8 * n)
    _need(y1, "y1", 8 * n)
    tr = None
    if transcript is not None:
        S = prm.lx + 1
        for k in ("w0", "w1"):  # large tape / Bicoptor-1: (n, S) u64 planes; otherwise lo (n, 8) + hi (n,) bytes
            _need(transcript.get(k + "_lo"), k + "_lo", n * (8 * S if prm.lx >= 8 or what == "bc_drelu_b1" else 8))
            _need(transcript.get(k + "_hi"), k + "_hi", n)
        tr = bc_transcript(*(_opt(transcript.get(k), k, None) for k in ("w0_lo", "w0_hi", "w1_lo", "w1_hi")))
    cp, cs = prm.c(), seeds_struct(seeds)
    _check(fn(_dev(x0, "x0"), _dev(x1, "x1"), _dev(y0, "y0"), _dev(y1, "y1"), n, elem_base, ctypes.byref(cp),
              ctypes.byref(cs), ctypes.byref(tr) if tr is not None else None, _stream(stream)), what)
    return y0, y1


@_on_input_device
def drelu_b1(x0, x1, prm: Params, seeds, elem_base: int = 0, y0=None, y1=None, transcript=None, stream=None):
    """Bicoptor-1 DReLU (comparison point): returns (y0, y1); transcript = u64 planes
    {"w0_lo", "w1_lo"} of shape (n, lx+1)."""
    return _fused(lib().bc_drelu_b1, "bc_drelu_b1", x0, x1, prm, seeds, elem_base, y0, y1, transcript, stream)


def transcript_buffers(n: int, device, prm: "Params | None" = None) -> dict:
    """Caller-owned buffers for the P0/P1 -> P2 message transcript (large tape:
    W0, W1 as (n, slots) u64 planes; otherwise the byte wire format)."""
    if prm is not None and prm.lx >= 8:
        S = prm.lx + 1
        return {"w0_lo": torch.empty((n, S), dtype=torch.int64, device=device),
                "w1_lo": torch.empty((n, S), dtype=torch.int64, device=device)}
    return {"w0_lo": torch.empty((n, 8), dtype=torch.uint8, device=device),
            "w0_hi": torch.empty(n, dtype=torch.uint8, device=device),
            "w1_lo": torch.empty((n, 8), dtype=torch.uint8, device=device),
            "w1_hi": torch.empty(n, dtype=torch.uint8, device=device)}


@_on_input_device
def drelu(x0, x1, prm: Params, seeds, elem_base: int = 0, y0=None, y1=None, transcript=None, stream=None):
    """Alg 7 with all three parties in one fused kernel: returns (y0, y1), y0 + y1 = DReLU(x)."""
    return _fused(lib().bc_drelu, "bc_drelu", x0, x1, prm, seeds, elem_base, y0, y1, transcript, stream)


@_on_input_device
def relu(x0, x1, prm: Params, seeds, elem_base: int = 0, y0=None, y1=None, transcript=None, stream=None):
    """Alg 8 with all three parties in one fused kernel: returns (y0, y1), y0 + y1 = ReLU(x)."""
    return _fused(lib().bc_relu, "bc_relu", x0, x1, prm, seeds, elem_base, y0, y1, transcript, stream)


# ---- host-buffer entry points (end to end) -------------------------------------------

def _host(t, name):
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise BicoptorError(f"{name} must be a host tensor")
    if not t.is_contiguous() or t.element_size() != 8:
        raise BicoptorError(f"{name} must be contiguous with 8-byte elements")
    return t.data_ptr()


def host_workspace(chunk: int, device) -> torch.Tensor:
    """Device workspace for drelu_host / relu_host at this chunk size."""
    nbytes = lib().bc_host_workspace_bytes(chunk)
    return torch.empty(nbytes // 8, dtype=torch.int64, device=device)


def _host_call(fn, what, hx0, hx1, hy0, hy1, prm, seeds, elem_base, ws, chunk, stream):
    n = hx0.numel()
    if hx1.numel() != n or hy0.numel() != n or hy1.numel() != n:
        raise BicoptorError("host buffers differ in length")
    cp, cs = prm.c(), seeds_struct(seeds)
    _check(fn(_host(hx0, "x0"), _host(hx1, "x1"), _host(hy0, "y0"), _host(hy1, "y1"), n, elem_base,
              ctypes.byref(cp), ctypes.byref(cs), _dev(ws, "ws", None), ws.numel() * ws.element_size(), chunk,
              _stream(stream)), what)
    return hy0, hy1


@_on_input_device
def drelu_host(hx0, hx1, hy0, hy1, prm: Params, seeds, ws, chunk: int = 1 << 20, elem_base: int = 0, stream=None,
               sync: bool = True):
    """bc_drelu_host: host shares in (pinned recommended), host shares out; synchronous.
    sync=False: bc_drelu_host_async, enqueue only (synchronise the stream before reading)."""
    fn, what = (lib().bc_drelu_host, "bc_drelu_host") if sync else (lib().bc_drelu_host_async, "bc_drelu_host_async")
    return _host_call(fn, what, hx0, hx1, hy0, hy1, prm, seeds, elem_base, ws, chunk, stream)


@_on_input_device
def relu_host(hx0, hx1, hy0, hy1, prm: Params, seeds, ws, chunk: int = 1 << 20, elem_base: int = 0, stream=None,
              sync: bool = True):
    """bc_relu_host: as drelu_host for ReLU."""
    fn, what = (lib().bc_relu_host, "bc_relu_host") if sync else (lib().bc_relu_host_async, "bc_relu_host_async")
    return _host_call(fn, what, hx0, hx1, hy0, hy1, prm, seeds, elem_base, ws, chunk, stream)


# ---- party-separated phases ---------------------------------------------------------

def wire_format(prm: Params) -> dict:
    """Per-element shape and dtype of the message planes to P2 (include/bicoptor.h,
    bc_drelu_send): byte planes lo (8 B) + hi (1 B) for slots <= 8, p <= 257; for
    the large tape lo = S low words (uint32, stored slot-major: an (S, n) plane) +
    hi = one word of bit-32 flags.  "hi" is None when every W_m fits the lo plane."""
    c = prm.c()
    if c.tape == 2:  # large: the lo plane is slot-major, (S, n)
        return {"lo": ((c.slots,), torch.int32), "hi": ((), torch.int32) if c.p > 0xFFFFFFFF else None,
                "slot_major": True}
    return {"lo": ((8,), torch.uint8), "hi": ((), torch.uint8) if c.p > 256 else None, "slot_major": False}


def lo_plane(buf: torch.Tensor, m: int, fmt: dict) -> torch.Tensor:
    """The lo plane of m elements inside a buffer sized for more: the first m rows of
    an element-major plane, or an (S, m) view of the first S m words of a slot-major one."""
    if fmt.get("slot_major"):
        S = fmt["lo"][0][0]
        return buf.reshape(-1)[:S * m].view(S, m)
    return buf[:m]


def msg_buffers(n: int, device, prm: "Params | None" = None):
    fmt = wire_format(prm if prm is not None else Params())
    (los, lot), hi_f = fmt["lo"], fmt["hi"]
    lo = torch.empty((los[0], n) if fmt["slot_major"] else (n,) + los, dtype=lot, device=device)
    hi = torch.empty(n, dtype=(hi_f[1] if hi_f else lot), device=device)
    tb = torch.empty((n + 7) // 8, dtype=torch.uint8, device=device)
    return lo, hi, tb


@_on_input_device
def drelu_send(party, x, prm: Params, seed01: bytes, elem_base=0, out=None, stream=None, y=None, seed02=None):
    """Alg 7 steps 1-8 for P0/P1: returns (lo, hi, tbits).  With y (P0 only, and seed02):
    bc_drelu_send_p0, P0's output share computed in the same kernel (reading C12)."""
    n = x.numel()
    lo, hi, tb = msg_buffers(n, x.device, prm) if out is None else out
    _need_msg(lo, hi, n, prm, "drelu_send")
    _need(tb, "tbits", (n + 7) // 8)
    _need(y, "y", 8 * n)
    if y is None:
        _check(lib().bc_drelu_send(party, _dev(x, "x"), _dev(lo, "lo", None), _opt(hi, "hi", None),
                                   _dev(tb, "tbits", 1), n, elem_base, ctypes.byref(prm.c()), seed01,
                                   _stream(stream)), "bc_drelu_send")
    else:
        if party != 0 or seed02 is None:
            raise BicoptorError("drelu_send with y: P0 only, and seed02 is needed")
        _check(lib().bc_drelu_send_p0(_dev(x, "x"), _dev(lo, "lo", None), _opt(hi, "hi", None), _opt(tb, "tbits", 1),
                                      _dev(y, "y"), n, elem_base, ctypes.byref(prm.c()), seed01, seed02,
                                      _stream(stream)), "bc_drelu_send_p0")
    return lo, hi, tb


@_on_input_device
def drelu_helper(lo0, hi0, lo1, hi1, prm: Params, seed02: bytes, elem_base=0, paper_literal=False, out=None,
                 stream=None):
    """Alg 7 steps 9-10 for P2: returns (resp0 or None, resp1)."""
    n = lo0.shape[1] if wire_format(prm)["slot_major"] else lo0.shape[0]  # (S, n) or (n, 8)
    if out is None:
        r0 = torch.empty(n, dtype=torch.int64, device=lo0.device) if paper_literal else None
        r1 = torch.empty(n, dtype=torch.int64, device=lo0.device)
    else:
        r0, r1 = out
    _need_msg(lo0, hi0, n, prm, "drelu_helper P0")
    _need_msg(lo1, hi1, n, prm, "drelu_helper P1")
    _need(r0, "resp0", 8 * n)
    _need(r1, "resp1", 8 * n)
    _check(lib().bc_drelu_helper(_dev(lo0, "lo0", None), _opt(hi0, "hi0", None), _dev(lo1, "lo1", None),
                                 _opt(hi1, "hi1", None),
                                 _opt(r0, "resp0"), _dev(r1, "resp1"), n, elem_base, ctypes.byref(prm.c()), seed02,
                                 _stream(stream)), "bc_drelu_helper")
    return r0, r1


@_on_input_device
def drelu_finish(party, tbits, resp, prm: Params, n: int, seed02: bytes | None = None, elem_base=0, out=None,
                 stream=None):
    """Alg 7 step 11 for P0/P1 (P0 may pass resp=None and seed02)."""
    y = torch.empty(n, dtype=torch.int64, device=tbits.device) if out is None else out
    _need(tbits, "tbits", (n + 7) // 8)
    _need(resp, "resp", 8 * n)
    _need(y, "y", 8 * n)
    _check(lib().bc_drelu_finish(party, _dev(tbits, "tbits", 1), _opt(resp, "resp"), _dev(y, "y"), n, elem_base,
                                 ctypes.byref(prm.c()), seed02, _stream(stream)), "bc_drelu_finish")
    return y


@_on_input_device
def relu_send(party, x, prm: Params, seed01: bytes, seed_tr: bytes, elem_base=0, out=None, d_peer=None,
              stream=None):
    """Alg 8 steps 1, 4 for P0/P1: returns (lo, hi, tbits, dshare).  d_peer: a second
    destination of dshare (bc_relu_send_to), e.g. the other party's mapped inbox."""
    n = x.numel()
    if out is None:
        lo, hi, tb = msg_buffers(n, x.device, prm)
        d = torch.empty_like(x)
    else:
        lo, hi, tb, d = out
    _need_msg(lo, hi, n, prm, "relu_send")
    _need(tb, "tbits", (n + 7) // 8)
    _need(d, "dshare", 8 * n)
    _need(d_peer, "d_peer", 8 * n)
    if d_peer is None:
        _check(lib().bc_relu_send(party, _dev(x, "x"), _dev(lo, "lo", None), _opt(hi, "hi", None),
                                  _dev(tb, "tbits", 1),
                                  _dev(d, "dshare"), n, elem_base, ctypes.byref(prm.c()), seed01, seed_tr,
                                  _stream(stream)), "bc_relu_send")
    else:
        _check(lib().bc_relu_send_to(party, _dev(x, "x"), _dev(lo, "lo", None), _opt(hi, "hi", None),
                                     _dev(tb, "tbits", 1), _dev(d, "dshare"), _dev(d_peer, "d_peer"), n, elem_base,
                                     ctypes.byref(prm.c()), seed01, seed_tr, _stream(stream)), "bc_relu_send_to")
    return lo, hi, tb, d


@_on_input_device
def relu_helper(lo0, hi0, lo1, hi1, prm: Params, seed02: bytes, seed12: bytes, elem_base=0, with_c1=True, out=None,
                e_dup=None, stream=None):
    """Alg 8 steps 2-3 for P2: returns (e, c1 or None).  e_dup: a second destination of
    e (bc_relu_helper_to), e.g. P1's mapped inbox while e goes to P0's."""
    n = lo0.shape[1] if wire_format(prm)["slot_major"] else lo0.shape[0]  # (S, n) or (n, 8)
    if out is None:
        e = torch.empty(n, dtype=torch.int64, device=lo0.device)
        c1 = torch.empty(n, dtype=torch.int64, device=lo0.device) if with_c1 else None
    else:
        e, c1 = out
    _need_msg(lo0, hi0, n, prm, "relu_helper P0")
    _need_msg(lo1, hi1, n, prm, "relu_helper P1")
    for t, name in ((e, "e"), (c1, "c1"), (e_dup, "e_dup")):
        _need(t, name, 8 * n)
    if e_dup is None:
        _check(lib().bc_relu_helper(_dev(lo0, "lo0", None), _opt(hi0, "hi0", None), _dev(lo1, "lo1", None),
                                    _opt(hi1, "hi1", None), _dev(e, "e"), _opt(c1, "c1"), n, elem_base,
                                    ctypes.byref(prm.c()), seed02, seed12, _stream(stream)), "bc_relu_helper")
    else:
        _check(lib().bc_relu_helper_to(_dev(lo0, "lo0", None), _opt(hi0, "hi0", None), _dev(lo1, "lo1", None),
                                       _opt(hi1, "hi1", None), _dev(e, "e"), _dev(e_dup, "e_dup"), _opt(c1, "c1"), n,
                                       elem_base, ctypes.byref(prm.c()), seed02, seed12, _stream(stream)),
               "bc_relu_helper_to")
    return e, c1


@_on_input_device
def relu_finish(party, x, tbits, d_own, d_peer, e, c1, prm: Params, seed_tr: bytes, elem_base=0, out=None,
                stream=None):
    """Alg 8 steps 4-5 for P0/P1."""
    n = x.numel()
    y = torch.empty_like(x) if out is None else out
    _need(tbits, "tbits", (n + 7) // 8)
    for t, name in ((d_own, "d_own"), (d_peer, "d_peer"), (e, "e"), (c1, "c1"), (y, "y")):
        _need(t, name, 8 * n)
    _check(lib().bc_relu_finish(party, _dev(x, "x"), _dev(tbits, "tbits", 1), _dev(d_own, "d_own"),
                                _dev(d_peer, "d_peer"), _dev(e, "e"), _opt(c1, "c1"), _dev(y, "y"), n, elem_base,
                                ctypes.byref(prm.c()), seed_tr, _stream(stream)), "bc_relu_finish")
    return y


# ---- peer memory (CUDA IPC) ----------------------------------------------------------

def ipc_export(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-B handle of the allocation holding t, byte offset of t in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    _check(lib().bc_ipc_export(_dev(t, "t", None), h, ctypes.byref(off)), "bc_ipc_export")
    return h.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation; returns the base address in this process."""
    base = ctypes.c_void_p()
    _check(lib().bc_ipc_open(handle, ctypes.byref(base)), "bc_ipc_open")
    return base.value


def ipc_close(base: int) -> None:
    _check(lib().bc_ipc_close(base), "bc_ipc_close")


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (a mapped peer buffer)."""

    def __init__(self, ptr: int, shape, dtype: torch.dtype):
        typestr = {torch.int64: "<i8", torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def tensor_at(ptr: int, shape, dtype: torch.dtype) -> torch.Tensor:
    """A tensor aliasing device memory at ptr (no copy, no ownership).  Its device is the
    one that owns the memory (a peer GPU for a peer mapping); only its address is used."""
    return torch.as_tensor(_CudaArray(ptr, shape, dtype))


# ---- RSS variant (Alg 9) -------------------------------------------------------------

def _rss(fn, what, x0, x1, x2, prm: Params, seeds, elem_base, out, stream):
    n = x0.numel()
    if x1.numel() != n or x2.numel() != n:
        raise BicoptorError("x0, x1, x2 differ in length")
    y0, y1, y2 = (torch.empty_like(x0), torch.empty_like(x1), torch.empty_like(x2)) if out is None else out
    for name in ("s012", "s2"):
        if len(getattr(seeds, name)) != 32:
            raise BicoptorError(f"seeds.{name} must be 32 bytes")
    cp, cs = prm.c(), seeds_struct(seeds)
    _check(fn(_dev(x0, "x0"), _dev(x1, "x1"), _dev(x2, "x2"), _dev(y0, "y0"), _dev(y1, "y1"), _dev(y2, "y2"), n,
              elem_base, ctypes.byref(cp), ctypes.byref(cs), seeds.s012, seeds.s2, _stream(stream)), what)
    return y0, y1, y2


@_on_input_device
def drelu_rss(x0, x1, x2, prm: Params, seeds, elem_base: int = 0, out=None, stream=None):
    """Alg 9 (RSS DReLU), three parties in one fused kernel: returns (y0, y1, y2), sum = DReLU(x).
    seeds carries s01, s02, s12, s012 and s2 (synth.Seeds)."""
    return _rss(lib().bc_drelu_rss, "bc_drelu_rss", x0, x1, x2, prm, seeds, elem_base, out, stream)


@_on_input_device
def relu_rss(x0, x1, x2, prm: Params, seeds, elem_base: int = 0, out=None, stream=None):
    """RSS ReLU [x][DReLU(x)]: returns (y0, y1, y2), sum = ReLU(x)."""
    return _rss(lib().bc_relu_rss, "bc_relu_rss", x0, x1, x2, prm, seeds, elem_base, out, stream)


# ---- truncation study (sec. 3-5) ---------------------------------------------------------

TRC_ALG = {"secureml": 1, "aby3": 2, "det": 4}
MUL_ORDER = {"mul_then_trc": 0, "trc_then_mul": 1}


@_on_input_device
def trc_aby3(x0, x1, ell: int, k: int, seeds, elem_base: int = 0, q: int = 0, rounds: int = 20, out=None,
             stream=None):
    """Alg 2 (ABY3) for both parties: returns (y0, y1), y0 + y1 = trc(x, k) (probabilistic)."""
    y0, y1 = (torch.empty_like(x0), torch.empty_like(x1)) if out is None else out
    cs = seeds_struct(seeds)
    _check(lib().bc_trc_aby3(_dev(x0, "x0"), _dev(x1, "x1"), _dev(y0, "y0"), _dev(y1, "y1"), x0.numel(), elem_base,
                             ell, k, rounds, q, ctypes.byref(cs), _stream(stream)), "bc_trc_aby3")
    return y0, y1


@_on_input_device
def trc_count(alg: str, x, ell: int, k: int, m_base: int = 0, m_count: int | None = None, counts=None, stream=None):
    """Exact e1 counting: counts[i] += (#exact, #e0, #e1) over masks [m_base, m_base + m_count)."""
    m_count = (1 << ell) if m_count is None else m_count
    counts = torch.zeros((x.numel(), 3), dtype=torch.int64, device=x.device) if counts is None else counts
    _check(lib().bc_trc_count(TRC_ALG[alg], _dev(x, "x"), x.numel(), ell, k, m_base, m_count, _dev(counts, "counts"),
                              _stream(stream)), "bc_trc_count")
    return counts


@_on_input_device
def mul_trc(order: str, alg: str, x0, x1, y0, y1, ell: int, f: int, seeds, elem_base: int = 0, rounds: int = 20,
            out=None, stream=None):
    """Fixed-point product x y / 2^f in the given order (Alg 3 = "trc_then_mul"): returns (z0, z1)."""
    z0, z1 = (torch.empty_like(x0), torch.empty_like(x1)) if out is None else out
    cs = seeds_struct(seeds)
    _check(lib().bc_mul_trc(MUL_ORDER[order], TRC_ALG[alg], _dev(x0, "x0"), _dev(x1, "x1"), _dev(y0, "y0"),
                            _dev(y1, "y1"), _dev(z0, "z0"), _dev(z1, "z1"), x0.numel(), elem_base, ell, f, rounds,
                            ctypes.byref(cs), _stream(stream)), "bc_mul_trc")
    return z0, z1
