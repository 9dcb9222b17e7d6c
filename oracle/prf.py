"""PRF restatement (reference prg.py:25-65) -- test infrastructure only.

AES-128-CTR via the reference's own dependency `cryptography` (OpenSSL; the
reference pins it only as >=41, pyproject.toml:10-14), keyed by
BLAKE2b(domain, key=pair_seed, 16 B), zero IV, 128-bit big-endian block
counter.  Seekable: keystream(key, first_u64, n) starts at any u64 index,
which the reference's sequential Prg can only reach by drawing the prefix.
Pinned by the reference KAT (tests/test_prg_transport.py:14-23) through
tests/golden/prf.npz.
"""

from __future__ import annotations

import hashlib

import numpy as np
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes

PAIRS = ("01", "02", "12")


def pair_seeds(master: bytes) -> dict[str, bytes]:
    """prg.py:25-31."""
    return {p: hashlib.blake2b(b"eta" + p.encode(), key=master, digest_size=16).digest()
            for p in PAIRS}


def salt(master: bytes) -> bytes:
    """prg.py:34-36."""
    return hashlib.blake2b(b"salt", key=master, digest_size=16).digest()


def stream_key(seed: bytes, domain: str) -> bytes:
    """prg.py:45-46."""
    return hashlib.blake2b(domain.encode(), key=seed, digest_size=16).digest()


def keystream(key: bytes, first_u64: int, n: int) -> np.ndarray:
    """u64 words first_u64 .. first_u64+n-1 of the AES-CTR stream (prg.py:47-55)."""
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    block0 = first_u64 >> 1
    skip = first_u64 & 1
    nblocks = (skip + n + 1) // 2
    enc = Cipher(algorithms.AES(key), modes.CTR(block0.to_bytes(16, "big"))).encryptor()
    raw = enc.update(b"\x00" * (16 * nblocks))
    words = np.frombuffer(raw, dtype="<u8")
    return words[skip:skip + n].astype(np.uint64)


class Stream:
    """Sequential view with the reference's byte offset (prg.py:39-65)."""

    def __init__(self, seed: bytes, domain: str):
        self.key = stream_key(seed, domain)
        self.offset = 0

    def u64(self, n: int) -> np.ndarray:
        out = keystream(self.key, self.offset // 8, n)
        self.offset += 8 * n
        return out

    def base(self, n: int, width: int) -> np.ndarray:
        return self.u64(n) & np.uint64((1 << width) - 1) if width < 64 else self.u64(n)

    def bits(self, n: int) -> np.ndarray:
        return self.u64(n) & np.uint64(1)
