"""numpy restatement of the reference RNG (rng.py:21-83) — test infrastructure only."""
from __future__ import annotations

import hashlib

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finalizer (rng.py:21-27)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _label_hash(label):  # rng.py:30-35
    if isinstance(label, (int, np.integer)):
        with np.errstate(over="ignore"):
            return mix64(np.uint64(int(label) & 0xFFFFFFFFFFFFFFFF) + GOLDEN)
    digest = hashlib.blake2b(str(label).encode(), digest_size=8).digest()
    return np.uint64(int.from_bytes(digest, "little"))


def derive_key(seed, *path):  # rng.py:38-47
    key = mix64(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF))
    for element in path:
        key = mix64(key ^ _label_hash(element))
    return np.uint64(key)


def uniform_from_bits(z):  # rng.py:50-53
    z = np.asarray(z, dtype=np.uint64)
    return (z >> np.uint64(12)).astype(np.float64) * (2.0**-52) + 2.0**-53


def stream_uniforms(key, chains, t):
    """Closed form of StreamSet (rng.py:63-77): draw t of stream `chain`
    (broadcasts chains against t)."""
    chains = np.asarray(chains, dtype=np.uint64)
    t = np.asarray(t, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s0 = mix64(np.uint64(key) ^ ((chains + np.uint64(1)) * GOLDEN))
        return uniform_from_bits(mix64(s0 + (t + np.uint64(1)) * GOLDEN))


def counter_uniform(key, counters):  # rng.py:56-60
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return uniform_from_bits(mix64(((c + np.uint64(1)) * GOLDEN) ^ np.uint64(key)))


def gaussian_field(key, codes, sigma):  # rng.py:86-96
    from scipy.special import ndtri

    return sigma * ndtri(counter_uniform(key, codes))
