"""Counter-based RNG (splitmix64) over torch int64 tensors.

Counter-based means every draw is a pure function of (seed, stream, index), so
the generated data is identical whatever the device (CPU or CUDA), thread count
or chunking.  Integer-only arithmetic: CPU and CUDA give the same bits.

torch has no uint64 arithmetic, so values live in int64 with two's-complement
wrap-around and logical right shifts emulated by masking.
"""
import torch

_M63 = (1 << 63) - 1


def _s64(c: int) -> int:
    c &= (1 << 64) - 1
    return c - (1 << 64) if c >= (1 << 63) else c


GOLDEN = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser of (x + golden); x: int64 tensor (any device)."""
    z = x + GOLDEN
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def draw(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Non-negative 63-bit hash of (seed, stream, idx)."""
    key = splitmix64(torch.full_like(idx, _s64(seed * 0x100000001B3 + stream * 0x9E37)))
    return splitmix64(idx ^ key) & _M63


def uniform_int(seed: int, stream: int, idx: torch.Tensor, lo, hi) -> torch.Tensor:
    """Integer uniform in [lo, hi] (inclusive); lo/hi scalars or int64 tensors."""
    span = hi - lo + 1
    return lo + draw(seed, stream, idx) % span
