"""ChaCha block function and keystream addressing (oracle; test infrastructure only).

The paper never names its PRG: it only assumes pre-shared seeds seed01, seed02,
seed12 from which parties "generate" randomness (P:209, P:876, P:886,
P:1839-1846).  Reading C19: the PRG is ChaCha with the RFC 8439
sec. 2.3 block function, run in DJB's original state layout

    words 0-3   "expand 32-byte k"
    words 4-11  256-bit key (the seed), little endian
    words 12-13 64-bit block counter (low word first)
    words 14-15 64-bit stream label (domain separation), low word first

which is bit-for-bit the RFC 8439 block when counter = c | nonce0 << 32 and
label = nonce1 | nonce2 << 32 (so the RFC test vector pins it).  The round
count R is a parameter (20 = RFC; 12 and 8 run the same double-round loop).

Pinned by: RFC 8439 sec. 2.3.2 test vector (tests/golden/rfc8439_block.txt)
and the independent OpenSSL implementation in the ``cryptography`` package
(tests/test_oracle_chacha.py).
"""
from __future__ import annotations

import numpy as np

SIGMA = np.array([0x61707865, 0x3320646E, 0x79622D32, 0x6B206574], dtype=np.uint32)


def label_u64(name: bytes) -> int:
    """An 8-byte ASCII stream label read as a little-endian u64."""
    assert len(name) == 8
    return int.from_bytes(name, "little")


def _rotl(v: np.ndarray, n: int) -> np.ndarray:
    return (v << np.uint32(n)) | (v >> np.uint32(32 - n))


def _quarter_round(x: np.ndarray, a: int, b: int, c: int, d: int) -> None:
    # RFC 8439 sec. 2.1
    x[a] += x[b]; x[d] ^= x[a]; x[d] = _rotl(x[d], 16)
    x[c] += x[d]; x[b] ^= x[c]; x[b] = _rotl(x[b], 12)
    x[a] += x[b]; x[d] ^= x[a]; x[d] = _rotl(x[d], 8)
    x[c] += x[d]; x[b] ^= x[c]; x[b] = _rotl(x[b], 7)


def chacha_blocks(key: bytes, label: int, counters, rounds: int = 20) -> np.ndarray:
    """Return the ChaCha_R blocks for each 64-bit counter as a (n, 16) uint32 array.

    RFC 8439 sec. 2.3: 10 (R/2) double rounds of column + diagonal quarter
    rounds, then the input state is added word-wise.
    """
    assert len(key) == 32 and rounds % 2 == 0 and rounds > 0
    ctr = np.atleast_1d(np.asarray(counters, dtype=np.uint64))
    n = ctr.size
    st = np.empty((16, n), dtype=np.uint32)
    st[0:4] = SIGMA[:, None]
    st[4:12] = np.frombuffer(key, dtype="<u4").astype(np.uint32)[:, None]
    st[12] = (ctr & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    st[13] = (ctr >> np.uint64(32)).astype(np.uint32)
    st[14] = np.uint32(label & 0xFFFFFFFF)
    st[15] = np.uint32((label >> 32) & 0xFFFFFFFF)
    x = st.copy()
    with np.errstate(over="ignore"):
        for _ in range(rounds // 2):
            _quarter_round(x, 0, 4, 8, 12)
            _quarter_round(x, 1, 5, 9, 13)
            _quarter_round(x, 2, 6, 10, 14)
            _quarter_round(x, 3, 7, 11, 15)
            _quarter_round(x, 0, 5, 10, 15)
            _quarter_round(x, 1, 6, 11, 12)
            _quarter_round(x, 2, 7, 8, 13)
            _quarter_round(x, 3, 4, 9, 14)
        x += st
    return np.ascontiguousarray(x.T)


def block_bytes(key: bytes, label: int, counter: int, rounds: int = 20) -> bytes:
    """One serialized 64-byte block (little-endian words), RFC 8439 sec. 2.3."""
    return chacha_blocks(key, label, [counter], rounds)[0].astype("<u4").tobytes()


def element_bytes(key: bytes, label: int, rounds: int, elems, stride: int) -> np.ndarray:
    """Per-element slices of the keystream: element j owns keystream bytes
    [stride*j, stride*(j+1)) of the stream (key, label).  Returns (n, stride) uint8.

    The keystream is the concatenation of blocks 0, 1, 2, ... (counter = block
    index).  This addressing rule is the spec's; it is
    what makes results independent of how elements are sharded.
    """
    j = np.atleast_1d(np.asarray(elems, dtype=np.uint64))
    n = j.size
    if n == 0:
        return np.zeros((0, stride), dtype=np.uint8)
    off = j * np.uint64(stride)
    first = off // np.uint64(64)
    last = (off + np.uint64(stride - 1)) // np.uint64(64)
    nblk = int((last - first).max()) + 1
    need = np.unique(np.concatenate([first + np.uint64(k) for k in range(nblk)]))
    ks = chacha_blocks(key, label, need, rounds).astype("<u4").view(np.uint8).reshape(-1, 64)
    pos = np.searchsorted(need, first)
    window = np.concatenate([ks[np.minimum(pos + k, len(need) - 1)] for k in range(nblk)], axis=1)
    start = (off % np.uint64(64)).astype(np.int64)
    cols = start[:, None] + np.arange(stride)[None, :]
    return window[np.arange(n)[:, None], cols]


def element_u64(key: bytes, label: int, rounds: int, elems, count: int) -> np.ndarray:
    """Element j owns ``count`` little-endian u64 words at keystream byte 8*count*j."""
    b = element_bytes(key, label, rounds, elems, 8 * count)
    return np.ascontiguousarray(b).view("<u8").reshape(-1, count).astype(np.uint64)


def element_u32(key: bytes, label: int, rounds: int, elems, count: int) -> np.ndarray:
    """Element j owns ``count`` little-endian u32 words at keystream byte 4*count*j."""
    b = element_bytes(key, label, rounds, elems, 4 * count)
    return np.ascontiguousarray(b).view("<u4").reshape(-1, count).astype(np.uint32)
