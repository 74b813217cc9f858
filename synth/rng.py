"""Counter-based RNG for the synthetic scenes (SURVEY.md §8(d) "Common generator rules").

Every random number is a pure function of (seed, config_id, stream_id, counter), where the counter
is usually a packed global voxel coordinate.  Inputs are therefore identical for any sharding, any
device and any chunking.  The mixer is SplitMix64 (Steele, Lea & Flood 2014), evaluated on torch
int64 tensors with two's-complement wrap-around; logical right shifts are emulated with masks.

This module holds no arithmetic of the regulariser; it is shared by the oracle tests and the GPU
path only as an input generator (task rule ③).
"""
from __future__ import annotations

import math

import torch

# stream ids
S_NOISE, S_W, S_W0, S_OUTLIER, S_OUTLIER_VAL, S_CLUMP, S_BOX, S_ROUTE = 1, 2, 3, 4, 5, 6, 7, 8
S_NOISE2 = 9  # second uniform of the Box-Muller pair
S_TEST = 10   # random test instances

_M64 = (1 << 64) - 1


def _i64(v: int) -> int:
    """Python int (mod 2^64) -> signed int64 value."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLDEN = _i64(0x9E3779B97F4A7C15)
_MUL1 = _i64(0xBF58476D1CE4E5B9)
_MUL2 = _i64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """SplitMix64 finaliser of (x + golden gamma), int64 in / int64 out (bit pattern of a uint64)."""
    z = x.to(torch.int64) + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _MUL1
    z = (z ^ _lsr(z, 27)) * _MUL2
    return z ^ _lsr(z, 31)


def splitmix64_py(x: int) -> int:
    """Pure-Python reference of :func:`splitmix64` (uint64 result), used by the generator tests."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, config_id: int, stream: int) -> int:
    """64-bit key of one (seed, config, stream) triple."""
    return _i64(splitmix64_py(((seed & 0xFFFFFFFF) << 32) ^ ((config_id & 0xFFFF) << 16) ^ (stream & 0xFFFF)))


def pack_coords(gx: torch.Tensor, gy: torch.Tensor, gz: torch.Tensor) -> torch.Tensor:
    """Pack three signed global voxel coordinates (|c| < 2^20) into one non-negative int64 counter."""
    m = (1 << 21) - 1
    return (gx.to(torch.int64) & m) | ((gy.to(torch.int64) & m) << 21) | ((gz.to(torch.int64) & m) << 42)


def bits(key: int, counter: torch.Tensor) -> torch.Tensor:
    return splitmix64(splitmix64(counter.to(torch.int64) ^ key))


def uniform(key: int, counter: torch.Tensor) -> torch.Tensor:
    """U[0,1) as float64 from the top 53 bits."""
    return _lsr(bits(key, counter), 11).to(torch.float64) * (1.0 / (1 << 53))


def uniform_int(key: int, counter: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Uniform integer in [lo, hi] (inclusive), via floor(U·(hi−lo+1))."""
    n = hi - lo + 1
    return (uniform(key, counter) * n).floor().clamp_(max=n - 1).to(torch.int64) + lo


def normal(key1: int, key2: int, counter: torch.Tensor) -> torch.Tensor:
    """Standard normal via Box–Muller of two independent uniform streams (float64)."""
    u1 = uniform(key1, counter)
    u2 = uniform(key2, counter)
    return torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2.0 * math.pi * u2)
