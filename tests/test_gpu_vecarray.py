"""GPU parity of the vector-array fused ops (N_V*VectorArray) against the
oracle's single-vector definitions applied vector by vector: streaming
results bit-exact, norms within 1e-12 (DESIGN R6)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bits_equal, needs_cuda, padded

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


def vecs(stream0, k, n, lo=-1.0, hi=1.0, off=0):
    return [padded(synth.uniform(stream0 + j, n, lo, hi, device="cuda"), off) for j in range(k)]


@pytest.mark.parametrize("n", [1, 33, 4097, 1_000_003])
@pytest.mark.parametrize("k", [1, 3, 8, 11])
def test_streaming_vector_arrays(S, ctx, n, k):
    X, Y = vecs(40, k, n), vecs(60, k, n, off=1)
    Z = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(k)]
    vX, vY, vZ = ([S.NVector(ctx, t) for t in L] for L in (X, Y, Z))
    assert S.N_VLinearSumVectorArray(0.3, vX, -1.7, vY, vZ) == 0
    for j in range(k):
        assert_bits_equal(Z[j], oracle.linear_sum(0.3, X[j].cpu().numpy(), -1.7, Y[j].cpu().numpy()),
                          f"LSVA j={j}")
    c = [0.25 * j - 0.6 for j in range(k)]
    assert S.N_VScaleVectorArray(c, vX, vZ) == 0
    for j in range(k):
        assert_bits_equal(Z[j], oracle.scale(c[j], X[j].cpu().numpy()), f"SVA j={j}")
    assert S.N_VConstVectorArray(2.5, vZ) == 0
    for j in range(k):
        assert torch.all(Z[j] == 2.5)
    # Z_j = c_j X_j in place (Z = X)
    Xc = [t.clone() for t in X]
    vXc = [S.NVector(ctx, t) for t in Xc]
    assert S.N_VScaleVectorArray(c, vXc, vXc) == 0
    for j in range(k):
        assert_bits_equal(Xc[j], oracle.scale(c[j], X[j].cpu().numpy()), f"SVA in place j={j}")
    ctx.check("vector arrays")


@pytest.mark.parametrize("n", [7, 100_003])
@pytest.mark.parametrize("k", [1, 5, 9])
def test_wrms_vector_arrays(S, ctx, n, k):
    X, W = vecs(70, k, n), vecs(90, k, n, 0.5, 1.5)
    idv = (synth.uniform(4, n, device="cuda") > 0.5).double()
    vX, vW = [S.NVector(ctx, t) for t in X], [S.NVector(ctx, t) for t in W]
    got = S.N_VWrmsNormVectorArray(vX, vW)
    gotm = S.N_VWrmsNormMaskVectorArray(vX, vW, S.NVector(ctx, idv))
    for j in range(k):
        ref = oracle.wrms(X[j].cpu().numpy(), W[j].cpu().numpy())
        assert abs(got[j] - ref) <= 1e-12 * ref
        refm = oracle.wrms_mask(X[j].cpu().numpy(), W[j].cpu().numpy(), idv.cpu().numpy())
        assert abs(gotm[j] - refm) <= 1e-12 * max(refm, 1e-300)


def test_multi_vector_arrays(S, ctx):
    n, nvec, nsum = 10_001, 3, 4
    X = vecs(100, nvec, n)
    Ys = [vecs(200 + 10 * i, nsum, n) for i in range(nvec)]
    Zs = [[torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nsum)] for _ in range(nvec)]
    a = [1.0 - j / 8 for j in range(nsum)]
    vX = [S.NVector(ctx, t) for t in X]
    vY = [[S.NVector(ctx, t) for t in row] for row in Ys]
    vZ = [[S.NVector(ctx, t) for t in row] for row in Zs]
    assert S.N_VScaleAddMultiVectorArray(a, vX, vY, vZ) == 0
    for i in range(nvec):
        ref = oracle.scale_add_multi(a, X[i].cpu().numpy(), [t.cpu().numpy() for t in Ys[i]])
        for j in range(nsum):
            assert_bits_equal(Zs[i][j], ref[j], f"SAMVA {i},{j}")
    out = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nvec)]
    c = [0.5, -0.25, 0.125, 2.0]
    assert S.N_VLinearCombinationVectorArray(c, vY, [S.NVector(ctx, t) for t in out]) == 0
    for i in range(nvec):
        assert_bits_equal(out[i], oracle.linear_combination(c, [t.cpu().numpy() for t in Ys[i]]),
                          f"LCVA {i}")
