"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.

This module holds NONE of the method's arithmetic: it only draws numbers.
It is the one module both sides use (DESIGN.md §4 "input recipe").

Generator (counter-based, so any index can be drawn alone — the oracle can
recompute sampled entries of a 1e8-element GPU input without materialising
the rest):

    key   = seed XOR (stream * 0xD1B54A32D192ED03)          (mod 2^64)
    z     = splitmix64_mix(key + i + 0x9E3779B97F4A7C15)    (mod 2^64)
    u     = (z >> 11) * 2^-53                               in [0, 1)
    value = lo + (hi - lo) * u                              (two RN ops)

The mix is done with torch int64 tensor ops (wrapping multiply, masked
logical shifts) so it runs identically on CPU and CUDA; the float step is
two separate elementwise torch kernels (no contraction), so the CPU and the
GPU draw identical bits.
"""
from __future__ import annotations

import torch

MASTER_SEED = 201112984
GOLDEN = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB

# stream ids per operand
S_X, S_Y, S_W, S_ID, S_CELL = 1, 2, 3, 4, 5
S_YJ, S_XJ = 16, 32


def _s64(v: int) -> int:
    """Python int -> the int64 with the same 64-bit pattern."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(t: torch.Tensor, k: int) -> torch.Tensor:
    """logical right shift of int64 bit patterns"""
    return torch.bitwise_and(torch.bitwise_right_shift(t, k), (1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    z = torch.bitwise_xor(z, _lsr(z, 30)) * _s64(M1)
    z = torch.bitwise_xor(z, _lsr(z, 27)) * _s64(M2)
    return torch.bitwise_xor(z, _lsr(z, 31))


def splitmix64_ref(state: int, count: int):
    """Pure-Python sequential splitmix64 (for pinning the tensor version)."""
    out = []
    for _ in range(count):
        state = (state + GOLDEN) & ((1 << 64) - 1)
        z = state
        z = ((z ^ (z >> 30)) * M1) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * M2) & ((1 << 64) - 1)
        out.append(z ^ (z >> 31))
    return out


def raw_bits(stream: int, idx: torch.Tensor, seed: int = MASTER_SEED) -> torch.Tensor:
    key = _s64(seed ^ ((stream * STREAM_MUL) & ((1 << 64) - 1)))
    z = idx.to(torch.int64) + _s64(key + GOLDEN)
    return mix64(z)


def uniform_at(stream: int, idx: torch.Tensor, lo: float = 0.0, hi: float = 1.0,
               seed: int = MASTER_SEED) -> torch.Tensor:
    """fp64 values at the given int64 indices (any device)."""
    z = raw_bits(stream, idx, seed)
    u = _lsr(z, 11).to(torch.float64) * (2.0 ** -53)
    if lo == 0.0 and hi == 1.0:
        return u
    return (u * (hi - lo)) + lo


def uniform(stream: int, n: int, lo: float = 0.0, hi: float = 1.0, *,
            offset: int = 0, device="cpu", seed: int = MASTER_SEED,
            chunk: int = 1 << 26) -> torch.Tensor:
    """n fp64 values for indices offset..offset+n-1 of the given stream."""
    out = torch.empty(n, dtype=torch.float64, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device)
        out[s:e] = uniform_at(stream, idx, lo, hi, seed)
    return out


def dyadic(stream: int, n: int, bits: int = 10, span: int = 4, *, device="cpu",
           seed: int = MASTER_SEED) -> torch.Tensor:
    """Multiples of 2^-bits in [-span, span): exact closed forms stay exact."""
    u = uniform(stream, n, device=device, seed=seed)
    k = torch.floor(u * (2 * span * (1 << bits))) - span * (1 << bits)
    return k * (2.0 ** -bits)


def small_int_blocks(stream: int, G: int, m: int, lo: int = -4, hi: int = 4,
                     seed: int = MASTER_SEED) -> torch.Tensor:
    """(G, m, m) blocks of small integers in [lo, hi] (exact Cramer checks)."""
    u = uniform(stream, G * m * m, seed=seed)
    v = torch.floor(u * (hi - lo + 1)) + lo
    return v.reshape(G, m, m)
