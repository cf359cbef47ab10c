"""Stream keys (mirror of the reference rng.py:21-60).

Only key derivation lives on the host: ``derive_key`` turns (seed, path) into
the 64-bit key of a stream family exactly as rng.py:38-47 does.  The per-chain
splitmix64 streams themselves (StreamSet, rng.py:63-83) are evaluated on the
device inside the fused sweep: draw t of chain c is
``u(mix64(mix64(key ^ (c+1)G) + (t+1)G))`` — a closed form of StreamSet — so a
chain's draws depend only on (key, c, t) and shard across GPUs unchanged.
"""
from __future__ import annotations

import hashlib

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
_MASK = 0xFFFFFFFFFFFFFFFF


def mix64(z: int) -> int:
    """splitmix64 finalizer on a Python int (rng.py:21-27)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def _label_hash(label) -> int:
    if isinstance(label, (int, np.integer)):
        return mix64((int(label) + GOLDEN) & _MASK)
    digest = hashlib.blake2b(str(label).encode(), digest_size=8).digest()
    return int.from_bytes(digest, "little")


def derive_key(seed, *path) -> np.uint64:
    """Key of the stream family (seed, path...) (rng.py:38-47)."""
    key = mix64(int(seed) & _MASK)
    for element in path:
        key = mix64(key ^ _label_hash(element))
    return np.uint64(key)


def uniform_from_bits(z):
    """Map uint64 words to doubles strictly inside (0, 1) (rng.py:50-53)."""
    z = np.asarray(z, dtype=np.uint64)
    return (z >> np.uint64(12)).astype(np.float64) * (2.0**-52) + 2.0**-53


def counter_uniform(key, counters):
    """Counter-based uniforms (rng.py:56-60); host-side, used for parameter init."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (c + np.uint64(1)) * np.uint64(GOLDEN) ^ np.uint64(key)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return uniform_from_bits(z)


def gaussian_field(key, codes, sigma):
    """Frozen Gaussian field (rng.py:86-96): sigma * ndtri(counter_uniform)."""
    from scipy.special import ndtri

    return sigma * ndtri(counter_uniform(key, codes))
