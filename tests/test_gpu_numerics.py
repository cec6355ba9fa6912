"""The fused kernel's division primitive (DESIGN R25) against IEEE on the
device: the Markstein-corrected quotient on the correctly rounded
reciprocal must equal __ddiv_rn bit for bit for every pair whose operands
lie in the fast-path range [2^-480, 2^480) — random magnitudes over the
whole range, mantissa edge cases (all ones, powers of two, quotients next
to 1) and the magnitudes the Brusselator driver divides by."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda]


@pytest.fixture(scope="module")
def S():
    from paper_2011_12984_b200 import sunbw
    return sunbw


@pytest.fixture(scope="module")
def ctx(S):
    c = S.Context(0)
    yield c
    c.destroy()


def rand_magnitudes(stream, n, emin=-479, emax=479):
    m = synth.uniform(stream, n, 1.0, 2.0)
    e = torch.floor(synth.uniform(stream + 100, n, emin, emax))
    s = torch.where(synth.uniform(stream + 200, n) < 0.5, -1.0, 1.0).double()
    return s * torch.ldexp(m, e.long())


def test_division_primitive_random(S, ctx):
    n = 50_000_000
    a = rand_magnitudes(1, n).cuda()
    b = rand_magnitudes(2, n).cuda()
    mism, checked = S.selftest_division(ctx, a, b)
    assert checked == n
    assert mism == 0


def test_division_primitive_edge_mantissas(S, ctx):
    one_minus = np.nextafter(2.0, 0.0)                  # 1.111...1 × 2^0 (all-ones mantissa)
    specials = np.array([1.0, one_minus, 1.5, np.nextafter(1.0, 2.0), 1.0 + 2 ** -26, 3.0, 5e-6,
                         1.0 / 3.0, 0.1, 7.0, 2.0 ** 470, 2.0 ** -470, 1.0000000000000004])
    rng = np.random.default_rng(0)
    base = np.concatenate([specials, rng.uniform(1, 2, 400_000)])
    scales = 2.0 ** rng.integers(-40, 40, base.size)
    b = np.concatenate([base, base * scales, -base, np.full(base.size, one_minus)])
    a = np.concatenate([np.roll(b[:2 * base.size], 7), b[2 * base.size:] * 3, base])
    a = a[: b.size]
    a2 = b * (1 + 2 ** -52)                             # quotients next to 1
    A = np.concatenate([a, a2, b])
    B = np.concatenate([b, b, b])                       # includes a == b
    mism, checked = S.selftest_division(ctx, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    assert checked >= A.size - 16          # a few scaled values leave [2^-480, 2^480)
    assert mism == 0


def test_division_primitive_signed_zero_dividends(S, ctx):
    """+0 / b inside the fast path (a converged Newton correction divides
    zero by the pivot): the quotient keeps the IEEE sign, sign(b); -0
    dividends leave the fast path (the guard sends the cell to IEEE
    division), so only the +0 half is checked."""
    n = 1_000_000
    b = rand_magnitudes(3, n).cuda()
    neg = synth.uniform(4, n, device="cuda") < 0.5
    a = torch.where(neg, -0.0, 0.0).double()
    mism, checked = S.selftest_division(ctx, a, b)
    assert checked == n - int(neg.sum())
    assert mism == 0
