"""Pins for oracle.chacha: published known answers and an independent implementation."""
import os

import numpy as np
import pytest

from oracle import chacha

GOLD = os.path.join(os.path.dirname(__file__), "golden", "chacha_vectors.txt")


def _vectors():
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        src, rounds, key, ctr, lab, blk = [s.strip() for s in line.split("|")]
        yield src, int(rounds), bytes.fromhex(key), int(ctr, 16), int(lab, 16), bytes.fromhex(blk)


@pytest.mark.parametrize("vec", list(_vectors()), ids=lambda v: v[0])
def test_known_answer_blocks(vec):
    src, rounds, key, ctr, lab, blk = vec
    assert chacha.block_bytes(key, lab, ctr, rounds) == blk


def test_matches_openssl_chacha20():
    """The `cryptography` package's ChaCha20 (OpenSSL; 16-byte nonce = 32-bit
    counter || 96-bit nonce) is an independent implementation of RFC 8439."""
    algorithms = pytest.importorskip("cryptography.hazmat.primitives.ciphers.algorithms")
    from cryptography.hazmat.primitives.ciphers import Cipher
    rng = np.random.default_rng(7)
    for _ in range(20):
        key = rng.bytes(32)
        nonce12 = rng.bytes(12)
        c32 = int(rng.integers(0, 2**32 - 4))
        enc = Cipher(algorithms.ChaCha20(key, c32.to_bytes(4, "little") + nonce12), mode=None).encryptor()
        ref = enc.update(bytes(64 * 3))
        w = np.frombuffer(nonce12, dtype="<u4")
        lab = int(w[1]) | (int(w[2]) << 32)
        got = b"".join(chacha.block_bytes(key, lab, (c32 + i) | (int(w[0]) << 32)) for i in range(3))
        assert got == ref


def test_element_addressing_is_keystream_slicing():
    """element_bytes(j, stride) must equal bytes [stride*j, stride*(j+1)) of the
    concatenated keystream, for every stride the spec uses (brute force)."""
    key = bytes(range(32))
    lab = chacha.label_u64(b"testlabl")
    ks = b"".join(chacha.block_bytes(key, lab, c, 12) for c in range(40))
    for stride in (8, 16, 24, 32, 64):
        j = np.arange(0, (40 * 64) // stride - 1, dtype=np.uint64)
        got = chacha.element_bytes(key, lab, 12, j, stride)
        for jj in (0, 1, 2, 3, 5, 7, 8, 9, len(j) - 1):
            assert bytes(got[jj]) == ks[stride * jj: stride * (jj + 1)]


def test_rounds_differ_and_labels_separate():
    key = bytes(32)
    a = chacha.block_bytes(key, 1, 0, 20)
    assert a != chacha.block_bytes(key, 2, 0, 20)
    assert a != chacha.block_bytes(key, 1, 1, 20)
    assert chacha.block_bytes(key, 1, 0, 8) != chacha.block_bytes(key, 1, 0, 12)
