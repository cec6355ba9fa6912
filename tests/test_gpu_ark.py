"""GPU parity of the adaptive IMEX ARK driver (BW_ArkEvolve) against the
oracle: the same accepted / rejected step counts and Newton iterations,
final states within the north star's 1e-9 (adaptive step sizes come from
reduced norms, so they agree to rounding, not bits)."""
import numpy as np
import pytest
import torch

import oracle
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


def run(S, ctx, params, y0, t_end, **kw):
    P = S.Problem(ctx, params)
    yd = torch.from_numpy(y0).cuda()
    yout = torch.empty_like(yd)
    A = S.Ark(P, S.NVector(ctx, yd), **kw)
    rc, st = A.evolve(t_end, S.NVector(ctx, yout))
    A.destroy()
    P.destroy()
    return rc, yout.cpu().numpy(), st


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


def test_ark_C1_brusselator(S, ctx):
    nx = 64
    y0 = oracle.bruss_ic(nx)
    rc2, yref, st2 = oracle.ark_integrate(y0, 1.0, h0=1e-4, nx=nx, kx=0.01 * nx)
    rc, y, st = run(S, ctx, S.bruss_params(dim=1, nx=nx), y0, 1.0, h0=1e-4)
    assert rc == rc2 == 0
    for k in ("accepted", "rejected_err", "rejected_nl", "newton_iters", "setups"):
        assert st[k] == st2[k], k
    assert rel(y, yref) <= 1e-9


def test_ark_fixed_step_linear(S, ctx):
    G = 999
    y0 = np.linspace(0.5, 1.5, 3 * G)
    params = S.bruss_params(dim=1, nx=G, kind=1, lam_E=-1.0, lam_I=-10.0)
    rc2, yref, _ = oracle.ark_integrate(y0, 1.0, h0=1.0 / 80, fixed=True, kind=1, nx=G, lam_E=-1.0,
                                        lam_I=-10.0, maxnl=4, tol_nl=1e-4)
    rc, y, st = run(S, ctx, params, y0, 1.0, h0=1.0 / 80, fixed=True, maxnl=4, tol_nl=1e-4)
    assert rc == rc2 == 0 and st["accepted"] == 80
    assert rel(y, yref) <= 1e-12


def test_ark_3D_and_retries(S, ctx):
    nx, ny, nz = 12, 10, 8
    y0 = oracle.bruss_ic(nx, ny, nz)
    kx = 0.01 * nx
    rc2, yref, st2 = oracle.ark_integrate(y0, 0.05, h0=1e-4, nx=nx, ny=ny, nz=nz, kx=kx, ky=0.01 * ny,
                                          kz=0.01 * nz)
    rc, y, st = run(S, ctx, S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz), y0, 0.05, h0=1e-4)
    assert rc == rc2 == 0 and st["accepted"] == st2["accepted"]
    assert rel(y, yref) <= 1e-9
    # one Newton iteration per stage with an unreachable tolerance: every
    # attempt fails and the step is recomputed with h/4 until max_steps
    rc, _, st = run(S, ctx, S.bruss_params(dim=1, nx=64), oracle.bruss_ic(64), 0.01, h0=1e-3,
                    maxnl=1, tol_nl=1e-300, max_steps=5)
    assert rc == 1 and st["rejected_nl"] == 5 and st["accepted"] == 0
