"""Helpers for the GPU parity tests (no method arithmetic here)."""
import numpy as np
import pytest
import torch

try:
    HAS_CUDA = torch.cuda.is_available()
except Exception:  # pragma: no cover
    HAS_CUDA = False

needs_cuda = pytest.mark.skipif(not HAS_CUDA, reason="no CUDA device")


def bits(a):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bits_equal(got, ref, what=""):
    """Bit-exact comparison (DESIGN R23: +0 and -0 differ; any NaN equals any NaN)."""
    g = got.detach().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    both_nan = np.isnan(g) & np.isnan(r)
    diff = (bits(g) != bits(r)) & ~both_nan
    if diff.any():
        i = int(np.nonzero(diff)[0][0])
        raise AssertionError(f"{what}: {int(diff.sum())} of {g.size} differ; first at {i}: "
                             f"gpu={g.flat[i]!r} ref={r.flat[i]!r}")


def padded(t: torch.Tensor, off: int) -> torch.Tensor:
    """Same values in a view starting `off` elements into a fresh buffer
    (exercises the misaligned head/tail paths)."""
    buf = torch.empty(t.numel() + off + 4, dtype=t.dtype, device=t.device)
    v = buf[off:off + t.numel()]
    v.copy_(t)
    return v
