"""Counter-based, seeded random streams for synthetic probe inputs.

This module holds NONE of the method's arithmetic.  It is the one module the
oracle side (tests, bench ``cpu_baseline``) and the CUDA side (parity tests,
bench) share, and it only produces *inputs*: table columns and predicate
batches.  The hash here is the xxHash64 avalanche (different constants and
shifts from the SplitMix64 / MurmurHash3 finalisers the probe uses for its
sample mask and HLL), so no output of the probe
can be reproduced from it.

Every value is a pure function of ``(seed, stream, index)``.  Any row range
``[r0, r1)`` can therefore be generated on its own (one GPU shard, or a small
CPU slice) and equals the same slice of the whole table.  The ops are plain
torch int64 / float64 element-wise ops, which give identical results on CPU and
CUDA, so a table generated on the GPU can be regenerated bit-for-bit on the
host for the oracle.
"""
from __future__ import annotations

import torch

_M64 = (1 << 64) - 1


def _s64(u: int) -> int:
    """uint64 literal -> the int64 with the same bits (torch has no uint64 math)."""
    u &= _M64
    return u - (1 << 64) if u >= (1 << 63) else u


# xxHash64 primes (public constants of the xxHash64 specification).
_P1 = _s64(0x9E3779B185EBCA87)
_P2 = _s64(0xC2B2AE3D27D4EB4F)
_P3 = _s64(0x165667B19E3779F9)
_P4 = _s64(0x85EBCA77C2B2AE63)
_P5 = _s64(0x27D4EB2F165667C5)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bits (torch's >> is arithmetic)."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _avalanche(h: torch.Tensor) -> torch.Tensor:
    h = h ^ _srl(h, 33)
    h = h * _P2
    h = h ^ _srl(h, 29)
    h = h * _P3
    h = h ^ _srl(h, 32)
    return h


def _avalanche_int(h: int) -> int:
    h &= _M64
    h ^= h >> 33
    h = (h * 0xC2B2AE3D27D4EB4F) & _M64
    h ^= h >> 29
    h = (h * 0x165667B19E3779F9) & _M64
    h ^= h >> 32
    return h


def stream_key(seed: int, stream: str) -> int:
    """Key of one named random stream of one seed (host int, signed 64-bit)."""
    s = 0
    for ch in stream.encode():
        s = _avalanche_int((s ^ ch) * 0x27D4EB2F165667C5 + 0x85EBCA77C2B2AE63)
    return _s64(_avalanche_int((seed & _M64) * 0x9E3779B185EBCA87 ^ s))


def bits(seed: int, stream: str, idx: torch.Tensor) -> torch.Tensor:
    """64 random bits (as int64) for every index in ``idx`` (int64 tensor)."""
    key = stream_key(seed, stream)
    return _avalanche(idx * _P1 + key)


def uniform_int(seed: int, stream: str, idx: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Integers in [lo, hi] (inclusive); modulo bias < 2^-30, irrelevant for inputs."""
    span = hi - lo + 1
    assert 0 < span < (1 << 62)
    return _srl(bits(seed, stream, idx), 1) % span + lo


def uniform_f64(seed: int, stream: str, idx: torch.Tensor) -> torch.Tensor:
    """Doubles in [0, 1) with 53 random bits."""
    return _srl(bits(seed, stream, idx), 11).to(torch.float64) * (2.0 ** -53)
