"""The C-ABI library loads and exports every symbol include/bicoptor.h declares;
host-only entry points (parameter derivation, error text) agree with the oracle.
No GPU needed: nothing here launches a kernel."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bicoptor.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2309_04909_b200 import api, build
    build.build()
    return api.lib()


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("bc_params_init", "bc_trc", "bc_modswitch", "bc_ladder_modswitch", "bc_drelu", "bc_relu",
                 "bc_drelu_send", "bc_drelu_helper", "bc_drelu_finish", "bc_relu_send", "bc_relu_helper",
                 "bc_relu_finish", "bc_strerror", "bc_trc_prob", "bc_drelu_rss", "bc_relu_rss",
                 "bc_trc_aby3", "bc_trc_count", "bc_mul_trc", "bc_drelu_host", "bc_relu_host", "bc_drelu_b1"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2309_04909_b200 import api
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(api.EXPORTS)


def test_params_derivation_matches_oracle(lib):
    from oracle import bicoptor as B
    from paper_2309_04909_b200 import api
    for ell in (8, 16, 32, 64):
        for lx in (2, 3, 5, 7, 8, 12, 15, 16, 30, 31, 32):
            for mode in ("guard", "literal"):
                for f in (0, 1, 24):
                    try:
                        o = B.Params(ell=ell, lx=lx, f=f, mode=mode, rounds=12)
                    except ValueError:
                        with pytest.raises(api.BicoptorError):
                            api.Params(ell=ell, lx=lx, f=f, mode=mode, rounds=12).c()
                        continue
                    c = api.Params(ell=ell, lx=lx, f=f, mode=mode, rounds=12).c()
                    assert (c.w, c.p, c.slots, api.TAPE[c.tape]) == (o.w, o.p, o.slots, o.layout)


def test_errors_and_strerror(lib):
    from paper_2309_04909_b200 import api
    p = api.bc_params()
    assert lib.bc_params_init(ctypes.byref(p), 64, 7, 24, 0, 7) == -1       # rounds
    assert lib.bc_params_init(ctypes.byref(p), 16, 7, 2, 0, 20) == -2       # window
    assert lib.bc_params_init(None, 64, 7, 24, 0, 20) == -1
    assert b"window" in lib.bc_strerror(-2)
    # a NULL-pointer call is rejected on the host before any launch
    assert lib.bc_drelu(None, None, None, None, 8, 0, ctypes.byref(api.Params().c()), None, None, None) == -1
    assert lib.bc_version() >= 300
    assert ctypes.sizeof(api.bc_params) == 40


def test_host_only_entry_points_validate_without_a_gpu(lib):
    """The peer-memory plumbing refuses NULL arguments before touching CUDA, and
    parameter derivation rejects windows that do not fit (BC_ERANGE) -- no device needed."""
    import ctypes
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    base = ctypes.c_void_p()
    assert lib.bc_ipc_export(None, h, ctypes.byref(off)) == -1
    assert lib.bc_ipc_export(ctypes.c_void_p(16), None, ctypes.byref(off)) == -1
    assert lib.bc_ipc_open(None, ctypes.byref(base)) == -1
    assert lib.bc_ipc_open(h, None) == -1
    assert lib.bc_ipc_close(None) == -1
    from paper_2309_04909_b200 import api
    p = api.bc_params()
    assert lib.bc_params_init(ctypes.byref(p), 64, 31, 2, 0, 20) == -2     # 2 + 31 + 32 > 64
    assert lib.bc_params_init(ctypes.byref(p), 64, 31, 0, 0, 20) == 0
    assert p.tape == 2 and p.slots == 32 and p.p == 2**32 + 15
