"""GPU parity of the fused step in tolerance mode (newton_mode = 1, the
convergence-tested Newton of the paper's task-local solver, P:388-394;
DESIGN R31) against the oracle's tolerance-mode integration: the same
number of Newton iterations over the run (the per-step count varies, so the
speculative iteration count is exercised in both directions), the same
failure behaviour, and states within the north star's relative 1e-9 (R22)
every 100 steps.  The fused tolerance mode uses the contracted cell step
(R30)."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import needs_cuda
from test_gpu_bruss import kappas, rel_err, run_ranks

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


def run_fused_tol(S, ctx, params, y0, steps, chunk, **kw):
    P = S.Problem(ctx, params)
    yd = torch.from_numpy(y0).cuda()
    yout = torch.empty_like(yd)
    st = S.Stepper(P, S.NVector(ctx, yd), S.stepper_options(fused=True, numerics=1, newton_mode=1,
                                                             use_graph=False, **kw))
    ys, rc, stats = [], 0, None
    done = 0
    while done < steps and rc == 0:
        n = min(chunk, steps - done)
        rc, stats = st.advance(n, S.NVector(ctx, yout))
        done += n
        ys.append(yout.cpu().numpy().copy())
    st.destroy()
    P.destroy()
    return rc, ys, stats


@pytest.mark.parametrize("tol", [1e-3, 1e-5])
def test_fused_tol_C1(S, ctx, tol):
    nx, steps = 64, 1000
    y0 = oracle.bruss_ic(nx)
    kw = dict(kind=0, newton_mode=1, K=5, nx=nx, kx=0.01 * nx, h=1e-3, tol_nl=tol)
    rc, ys, st = run_fused_tol(S, ctx, S.bruss_params(dim=1, nx=nx), y0, steps, 100, h=1e-3, K=5, tol_nl=tol)
    assert rc == 0
    _, _, stref, ylog = oracle.sbdf_integrate(y0, steps, log_every=100, **kw)
    assert st["newton_iters"] == stref["newton_iters"], (st["newton_iters"], stref["newton_iters"])
    for i, y in enumerate(ys):
        assert rel_err(y, ylog[i]) <= 1e-9, (i, rel_err(y, ylog[i]))


def test_fused_tol_3D_in_kernel_advection(S, ctx):
    nx, ny, nz, steps = 128, 6, 4, 100
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    rc, ys, st = run_fused_tol(S, ctx, S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz), y0, steps, 50,
                               h=1e-3, K=5, tol_nl=1e-5)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, newton_mode=1, K=5, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3, tol_nl=1e-5)
    assert rc == 0 and st["newton_iters"] == stref["newton_iters"]
    assert rel_err(ys[-1], yref) <= 1e-9


@pytest.mark.parametrize("chunk", [1, 7, 30])
def test_fused_tol_device_driven_chunks(S, ctx, chunk):
    """One rank with the in-kernel advection: after the first step the
    decisions run on the device (DESIGN R35).  Advance calls of 1, 7 and 30
    steps (the rotation state, the iteration prediction and the statistics
    carry across calls) give the oracle's iteration count and state."""
    nx, ny, nz, steps = 128, 6, 4, 30
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    rc, ys, st = run_fused_tol(S, ctx, S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz), y0, steps, chunk,
                               h=1e-3, K=5, tol_nl=1e-5)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, newton_mode=1, K=5, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3, tol_nl=1e-5)
    assert rc == 0 and st["steps"] == steps
    assert st["newton_iters"] == stref["newton_iters"], (st["newton_iters"], stref["newton_iters"])
    assert rel_err(ys[-1], yref) <= 1e-9


def test_fused_tol_C3(S, ctx):
    """C3 (128^3 cells), 10 steps: the bench-shaped 3D grid."""
    n, steps = 128, 10
    y0 = oracle.bruss_ic(n, n, n)
    k = kappas(n, n, n)
    rc, ys, st = run_fused_tol(S, ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n), y0, steps, steps,
                               h=1e-3, K=5, tol_nl=1e-5)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, newton_mode=1, K=5, nx=n, ny=n, nz=n,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3, tol_nl=1e-5)
    assert rc == 0 and st["newton_iters"] == stref["newton_iters"]
    assert rel_err(ys[-1], yref) <= 1e-9


def test_fused_tol_nonconvergence(S, ctx):
    """One iteration allowed, unreachable tolerance: the first step fails
    (recoverable), as on the composed path and in the oracle."""
    nx = 64
    y0 = oracle.bruss_ic(nx)
    rc, _, st = run_fused_tol(S, ctx, S.bruss_params(dim=1, nx=nx), y0, 5, 5, h=1e-3, K=1, tol_nl=1e-300)
    rc2, _, st2, _ = oracle.sbdf_integrate(y0, 5, kind=0, newton_mode=1, K=1, nx=nx, kx=0.01 * nx, h=1e-3,
                                           tol_nl=1e-300)
    assert rc == S.SUNBW_RECOV_NONCONV and rc2 != 0
    assert st["steps"] == st2["steps"] == 0 and st["newton_iters"] == st2["newton_iters"] == 1


def test_fused_tol_exact_numerics_unsupported(S, ctx):
    P = S.Problem(ctx, S.bruss_params(dim=1, nx=64))
    y = torch.from_numpy(oracle.bruss_ic(64)).cuda()
    with pytest.raises(S.SunbwError):
        S.Stepper(P, S.NVector(ctx, y), S.stepper_options(fused=True, numerics=0, newton_mode=1))
    P.destroy()


@pytest.mark.parametrize("nranks", [2])
def test_fused_tol_multirank(S, nranks):
    """P = 2 logical ranks (fake communicator): the global nu is allreduced,
    so every rank takes the same iteration count; state and count equal the
    one-rank oracle run."""
    nx, ny, nz, steps = 128, 4, 8, 40
    y0 = oracle.bruss_ic(nx, ny, nz)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
    k = kappas(nx, ny, nz)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, newton_mode=1, K=5, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3, tol_nl=1e-5)

    def fn(c, r):
        P = S.Problem(c, params)
        n, off = 3 * P.local_cells, 3 * P.cell_offset
        y = torch.from_numpy(y0[off:off + n].copy()).cuda()
        yout = torch.empty_like(y)
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=1e-3, K=5, tol_nl=1e-5, newton_mode=1,
                                                              use_graph=False, fused=True, numerics=1))
        rc, stats = st.advance(steps, S.NVector(c, yout))
        c.stream.synchronize()
        res = (rc, off, yout.cpu().numpy(), stats["newton_iters"])
        st.destroy(); P.destroy()
        return res

    res = run_ranks(S, nranks, fn)
    assert all(r[0] == 0 for r in res)
    assert len({r[3] for r in res}) == 1 and res[0][3] == stref["newton_iters"]
    y = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    assert rel_err(y, yref) <= 1e-9
