"""GPU parity of SPGMR (GMRES with the fused multi-vector kernels and the
batched block-LU preconditioner) and of the global-Newton driver against
the oracle.  GMRES reassociates reductions, so parity is to tolerance: the
same number of Arnoldi steps, solutions within 1e-10 relative, driver states
within the north star's 1e-9."""
import numpy as np
import pytest
import torch

import oracle
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


def rand_blocks(stream, G, m, shift):
    return synth.uniform(stream, G * m * m, -1, 1).reshape(G, m, m) + shift * torch.eye(m, dtype=torch.float64)


@pytest.mark.parametrize("prec", [True, False])
@pytest.mark.parametrize("G,m,maxl", [(1000, 3, 30), (50_001, 3, 10), (777, 5, 40)])
def test_spgmr_vs_oracle(S, ctx, prec, G, m, maxl):
    A = rand_blocks(10 + m, G, m, 2.5)
    b = synth.uniform(20, G * m, -1, 1)
    Ad = A.cuda().contiguous()
    M = S.SUNMatrix(ctx, Ad)
    bd = b.cuda()
    x = torch.empty_like(bd)
    LS = S.SUNLinearSolver(S.NVector(ctx, bd), M, spgmr_maxl=maxl, block_prec=prec)
    assert S.SUNLinSolSetup(LS, M) == 0
    S.SUNLinSolSolve(LS, M, S.NVector(ctx, x), S.NVector(ctx, bd), 1e-11)
    ctx.check("spgmr")
    P = oracle.lu_factor(A.numpy())[:2] if prec else None
    xr, steps, res = oracle.gmres(A.numpy(), b.numpy(), P, maxl=maxl, tol=1e-11)
    assert S.SUNLinSolNumIters(LS) == steps
    xg = x.cpu().numpy()
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    r_true = b.numpy() - np.einsum("gij,gj->gi", A.numpy(), xg.reshape(G, m)).reshape(-1)
    if steps < maxl:
        assert np.linalg.norm(r_true) <= 1e-10 * np.linalg.norm(b.numpy())
    assert abs(S.SUNLinSolResNorm(LS) - res) <= 1e-9 * np.linalg.norm(b.numpy())
    # the operator matrix is left intact (the preconditioner factors a copy)
    assert torch.equal(Ad.cpu(), A)


def test_global_newton_driver_C1(S, ctx):
    nx, steps = 64, 200
    y0 = oracle.bruss_ic(nx)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, kx=0.01 * nx, h=1e-3,
                                              linsol=1, maxl=5, lin_tol=1e-10)
    P = S.Problem(ctx, S.bruss_params(dim=1, nx=nx))
    yd = torch.from_numpy(y0).cuda()
    yout = torch.empty_like(yd)
    st = S.Stepper(P, S.NVector(ctx, yd), S.stepper_options(h=1e-3, K=3, linsol=1, maxl=5, lin_tol=1e-10))
    rc, stats = st.advance(steps, S.NVector(ctx, yout))
    assert rc == 0
    assert stats["lin_iters"] == stref["lin_iters"] == 3 * steps
    y = yout.cpu().numpy()
    assert np.max(np.abs(y - yref) / np.maximum(np.abs(yref), 1)) <= 1e-9
    st.destroy(); P.destroy()


def test_global_newton_driver_3D_multirank(S):
    """Global Newton + GMRES over P = 2 fake-communicator ranks: every GMRES
    inner product is a global (allreduced) reduction."""
    from test_gpu_bruss import run_ranks, kappas
    nx, ny, nz, steps = 12, 10, 8, 6
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz, kx=k[0],
                                          ky=k[1], kz=k[2], h=1e-3, linsol=1, maxl=5, lin_tol=1e-10)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)

    def fn(c, r):
        P = S.Problem(c, params)
        n = 3 * P.local_cells
        off = 3 * P.cell_offset
        y = torch.from_numpy(y0[off:off + n].copy()).cuda()
        yout = torch.empty_like(y)
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=1e-3, K=3, linsol=1, maxl=5,
                                                              lin_tol=1e-10, use_graph=False))
        rc, stats = st.advance(steps, S.NVector(c, yout))
        c.stream.synchronize()
        res = (rc, off, yout.cpu().numpy(), stats["lin_iters"])
        st.destroy(); P.destroy()
        return res

    res = run_ranks(S, 2, fn)
    assert all(r[0] == 0 for r in res)
    assert res[0][3] == res[1][3]                     # identical GMRES decisions on both ranks
    y = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    assert np.max(np.abs(y - yref) / np.maximum(np.abs(yref), 1)) <= 1e-9
