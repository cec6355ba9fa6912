"""Pins for the oracle's Brusselator pieces (O5, O8-O10) and the SBDF
integrator (O11-O13), CPU only.

Independent checks: printed examples (golden, with citations), central
finite differences of the reaction for the Jacobian, exact constant-state
and telescoping properties of the upwind stencil, separability of the 3D
stencil into 1D lines, Gaussian symmetry of the IC, and — for the
integrator — the closed-form solution of the SBDF recurrence on the linear
test equation (characteristic roots), the exp(λt) order-2 convergence, and
spatial-homogeneity / single-cell reductions of the Brusselator run.
"""
import cmath
import math

import numpy as np
import pytest

import oracle
import synth

PR = dict(c=0.01, A=1.0, B=3.5, eps=5e-6, alpha=0.1)


def test_reaction_golden(golden):
    for ex in golden["reaction"]:
        f = oracle.bruss_reaction(ex["y"], PR["A"], PR["B"], PR["eps"])
        assert np.array_equal(f, ex["f"]), ex["cite"]


def test_reaction_special_cases():
    # u = 0 -> (A, 0, (B-w)/eps)  (P:369-371 with u = 0)
    y = np.array([0.0, 2.0, 1.5, 0.0, -1.0, 3.5])
    f = oracle.bruss_reaction(y)
    assert np.array_equal(f, [1.0, 0.0, (3.5 - 1.5) / 5e-6, 1.0, 0.0, 0.0])
    # equilibrium (A, w*/A, w*), w* = B/(1+eps A): f ~ 0 up to (B/eps)·4u
    ws = 3.5 / (1 + 5e-6)
    f = oracle.bruss_reaction([1.0, ws, ws])
    assert np.max(np.abs(f)) <= 3.5 / 5e-6 * 4 * 2 ** -53


def test_jacobian_vs_central_fd():
    G = 100
    y = np.stack([synth.uniform(1, G, 0.5, 2).numpy(), synth.uniform(2, G, 0.5, 4).numpy(),
                  synth.uniform(3, G, 0.5, 4).numpy()], 1).reshape(-1)
    J = oracle.bruss_jacobian(y)
    for g in range(G):
        y0 = y[3 * g:3 * g + 3]
        for k in range(3):
            hk = 1e-6 * max(1.0, abs(y0[k]))
            yp, ym = y0.copy(), y0.copy()
            yp[k] += hk; ym[k] -= hk
            col = (oracle.bruss_reaction(yp) - oracle.bruss_reaction(ym)) / (yp[k] - ym[k])
            for i in range(3):
                scale = max(1.0, abs(J[g, i, k]))
                assert abs(J[g, i, k] - col[i]) <= 1e-6 * scale * (1 / 5e-6 if i == 2 else 1), (g, i, k)
    assert np.all(J[:, 2, 1] == 0.0)                       # J32 = 0 structurally
    M = oracle.scale_add_identity(-0.0, J)
    assert np.array_equal(M, np.tile(np.eye(3), (G, 1, 1)))   # gamma = 0 -> M = I


def test_advection_golden(golden):
    for ex in golden["advection_1d"]:
        nx = ex["nx"]
        dx = ex["b"] / nx
        kx = ex["c"] / dx
        y = np.zeros(3 * nx)
        y[0::3] = ex["u"]
        f = oracle.advection(y, nx, kx=kx)
        assert np.allclose(f[0::3], ex["f_u"], rtol=0, atol=1e-17), ex["cite"]
        assert np.all(f[1::3] == 0) and np.all(f[2::3] == 0)


@pytest.mark.parametrize("shape", [(64, 1, 1), (8, 6, 5), (5, 4, 7)])
def test_advection_constant_telescoping_separable(shape):
    nx, ny, nz = shape
    n = 3 * nx * ny * nz
    k = (0.64, 0.32, 0.16)
    const = np.tile([1.0, 3.5, 3.0], n // 3)
    assert np.all(oracle.advection(const, nx, ny, nz, *k) == 0.0)
    y = synth.uniform(1, n, 0, 1).numpy()
    f = oracle.advection(y, nx, ny, nz, *k)
    for s in range(3):
        assert abs(f[s::3].sum()) <= 1e-12 * n                 # periodic upwind telescopes
    # separability: a state varying only along x reproduces the 1D stencil per line
    line = synth.uniform(2, 3 * nx, 0, 1).numpy().reshape(nx, 3)
    yx = np.broadcast_to(line, (nz, ny, nx, 3)).reshape(-1).copy()
    fx = oracle.advection(yx, nx, ny, nz, *k).reshape(nz, ny, nx, 3)
    f1 = oracle.advection(line.reshape(-1), nx, 1, 1, k[0]).reshape(nx, 3)
    assert np.array_equal(fx, np.broadcast_to(f1, fx.shape))
    if nz > 1:
        col = synth.uniform(3, 3 * nz, 0, 1).numpy().reshape(nz, 3)
        yz = np.broadcast_to(col[:, None, None, :], (nz, ny, nx, 3)).reshape(-1).copy()
        fz = oracle.advection(yz, nx, ny, nz, *k).reshape(nz, ny, nx, 3)
        # only the z term survives: x-term then +y-term are exact zeros
        fz1 = k[2] * (np.roll(col, 1, axis=0) - col)
        assert np.array_equal(fz, np.broadcast_to(fz1[:, None, None, :], fz.shape))
    # periodic translation invariance
    ys = np.roll(y.reshape(nz, ny, nx, 3), 1, axis=2).reshape(-1)
    fs = oracle.advection(ys, nx, ny, nz, *k)
    assert np.array_equal(fs, np.roll(f.reshape(nz, ny, nx, 3), 1, axis=2).reshape(-1))


def test_ic_golden_and_symmetry(golden):
    nx = 64
    y = oracle.bruss_ic(nx).reshape(nx, 3)
    # x_i = i·dx; i = nx/2 sits on mu = b/2 exactly
    assert np.array_equal(y[nx // 2], golden["ic"][0]["uvw_at_mu"]), golden["ic"][0]["cite"]
    p = y[:, 0] - 1.0
    for d in range(1, nx // 2):
        assert p[nx // 2 + d] == p[nx // 2 - d]
    y0 = oracle.bruss_ic(nx, alpha=0.0).reshape(nx, 3)
    assert np.array_equal(y0, np.tile([1.0, 3.5, 3.0], (nx, 1)))
    # 3D: centre cell gets alpha; the Gaussian factorises over the axes
    y3 = oracle.bruss_ic(8, 8, 8).reshape(8, 8, 8, 3)
    assert np.array_equal(y3[4, 4, 4], golden["ic"][0]["uvw_at_mu"])
    px = oracle.bruss_ic(8)[0::3] - 1
    assert abs((y3[2, 4, 7, 0] - 1) - 0.1 * (px[7] / 0.1) * (px[2] / 0.1)) <= 1e-16


# ----------------------------------------------------------------- SBDF
def sbdf_closed_form(y0, zE, zI, nsteps):
    """Closed-form solution of the SBDF1-start / SBDF2 recurrence on
    y' = λ_E y + λ_I y (z = hλ):  y1 = (1+zE)/(1-zI) y0, then
    (3-2zI) y_{n+1} = (4+4zE) y_n - (1+2zE) y_{n-1}, solved by its
    characteristic roots."""
    a, b, c = 3 - 2 * zI, -(4 + 4 * zE), 1 + 2 * zE
    disc = cmath.sqrt(b * b - 4 * a * c)          # complex roots for stiff z_I
    r1, r2 = (-b + disc) / (2 * a), (-b - disc) / (2 * a)
    y1 = (1 + zE) / (1 - zI) * y0
    c2 = (y1 - r1 * y0) / (r2 - r1)
    c1 = y0 - c2
    return (c1 * r1 ** nsteps + c2 * r2 ** nsteps).real


@pytest.mark.parametrize("lamE,lamI,h", [(-1.0, -10.0, 1e-2), (0.5, -200.0, 1e-3), (0.0, -1e4, 1e-3)])
def test_sbdf_linear_closed_form(lamE, lamI, h):
    G = 4
    y0 = synth.uniform(1, 3 * G, 0.5, 1.5).numpy()
    nsteps = 50
    rc, y, st, _ = oracle.sbdf_integrate(y0, nsteps, kind=1, K=2, nx=G, lam_E=lamE, lam_I=lamI, h=h)
    assert rc == 0 and st["steps"] == nsteps and st["setups"] == nsteps
    ref = np.array([sbdf_closed_form(v, h * lamE, h * lamI, nsteps) for v in y0])
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-300)
    # Newton on a linear f_I converges in one iteration: the 2nd update is ~u
    assert st["last_nu"] <= 1e-9


def test_sbdf_second_order_in_h():
    lamE, lamI, T = -1.0, -10.0, 1.0
    y0 = np.ones(3)
    errs = []
    for k in range(4):
        nsteps = 40 * 2 ** k
        rc, y, _, _ = oracle.sbdf_integrate(y0, nsteps, kind=1, K=2, nx=1, lam_E=lamE,
                                            lam_I=lamI, h=T / nsteps)
        errs.append(abs(y[0] - math.exp((lamE + lamI) * T)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(1.8 < o < 2.2 for o in orders), orders


def test_sbdf_zero_rhs_is_identity():
    y0 = synth.uniform(1, 30, -1, 1).numpy()
    # y' = 0: SBDF1 is exact (d = y0 + h·0); SBDF2's d = RN(4/3 y) + RN(-1/3 y)
    # is y only up to rounding, so the state drifts by a few ulp per step
    rc, y, _, _ = oracle.sbdf_integrate(y0, 1, kind=1, K=3, nx=10, lam_E=0.0, lam_I=0.0)
    assert rc == 0 and np.array_equal(y, y0)
    rc, y, _, _ = oracle.sbdf_integrate(y0, 20, kind=1, K=3, nx=10, lam_E=0.0, lam_I=0.0)
    assert rc == 0 and np.max(np.abs(y - y0) / np.abs(y0)) <= 20 * 4 * 2 ** -53


def test_bruss_homogeneous_equals_single_cell():
    # a spatially uniform state has zero advection exactly; every cell then
    # follows the single-cell reaction ODE bit for bit
    nx = 16
    cell = np.array([1.2, 3.1, 2.9])
    y0 = np.tile(cell, nx)
    common = dict(kind=0, K=3, h=1e-3, **{k: PR[k] for k in ("A", "B", "eps")})
    rc, y, _, _ = oracle.sbdf_integrate(y0, 200, nx=nx, kx=0.01 * nx, **common)
    rc1, y1, _, _ = oracle.sbdf_integrate(cell, 200, nx=1, reaction_only=True, **common)
    assert rc == 0 and rc1 == 0
    assert np.array_equal(y.reshape(nx, 3), np.tile(y1, (nx, 1)))


def test_bruss_equilibrium_stays():
    ws = 3.5 / (1 + 5e-6)
    y0 = np.tile([1.0, ws, ws], 8)
    rc, y, _, _ = oracle.sbdf_integrate(y0, 100, kind=0, K=3, nx=8, kx=0.08, h=1e-3)
    assert rc == 0 and np.max(np.abs(y - y0) / np.abs(y0)) <= 1e-14


def test_bruss_fixed_K_vs_full_convergence_C1():
    # C1: 64 cells, b = 1, h = 1e-3 (DESIGN R18); K = 3 certified against
    # iterating to full convergence
    nx = 64
    y0 = oracle.bruss_ic(nx)
    kw = dict(kind=0, nx=nx, kx=0.01 / (1.0 / nx), h=1e-3)
    rc, yK, stK, _ = oracle.sbdf_integrate(y0, 200, newton_mode=0, K=3, **kw)
    rc2, yF, stF, _ = oracle.sbdf_integrate(y0, 200, newton_mode=2, **kw)
    assert rc == 0 and rc2 == 0
    assert np.max(np.abs(yK - yF) / np.maximum(np.abs(yF), 1)) <= 1e-10
    assert stF["newton_iters"] <= 200 * 6


def test_bruss_self_convergence_order2():
    # 2nd-order self-convergence under h-halving on the 1D Brusselator
    nx = 32
    y0 = oracle.bruss_ic(nx)
    kw = dict(kind=0, nx=nx, kx=0.01 * nx, newton_mode=2)
    T = 0.2
    sols = []
    for k in range(4):
        nsteps = 25 * 2 ** k
        rc, y, _, _ = oracle.sbdf_integrate(y0, nsteps, h=T / nsteps, **kw)
        assert rc == 0
        sols.append(y)
    e1 = np.max(np.abs(sols[1] - sols[0])); e2 = np.max(np.abs(sols[2] - sols[1]))
    e3 = np.max(np.abs(sols[3] - sols[2]))
    assert 1.7 < math.log2(e1 / e2) < 2.3 and 1.7 < math.log2(e2 / e3) < 2.3, (e1, e2, e3)


def test_tolerance_mode_converges_and_fails_recoverably():
    nx = 16
    y0 = oracle.bruss_ic(nx)
    kw = dict(kind=0, nx=nx, kx=0.01 * nx, h=1e-3)
    rc, y, st, _ = oracle.sbdf_integrate(y0, 20, newton_mode=1, K=5, tol_nl=1e-3, **kw)
    assert rc == 0 and st["newton_iters"] < 20 * 5
    rc, y, st, _ = oracle.sbdf_integrate(y0, 20, newton_mode=1, K=1, tol_nl=1e-300, **kw)
    assert rc == 1 and st["fails"] == 1


def test_sbdf_block_inverse_solver_matches_lu():
    """The paper's task-local block solve (symbolic Gauss-Jordan inverse,
    P:389-390; linsol = 2) and the LU solve (O6/O7) are the same Newton
    iteration up to rounding: C1 to t = 1 within 1e-12."""
    nx = 64
    y0 = oracle.bruss_ic(nx)
    common = dict(kind=0, K=3, nx=nx, kx=0.01 * nx, h=1e-3)
    rc0, y_lu, _, _ = oracle.sbdf_integrate(y0, 1000, linsol=0, **common)
    rc2, y_gj, st, _ = oracle.sbdf_integrate(y0, 1000, linsol=2, **common)
    assert rc0 == 0 and rc2 == 0 and st["singular"] == 0
    assert np.max(np.abs(y_gj - y_lu) / np.maximum(np.abs(y_lu), 1.0)) <= 1e-12
    # the two solvers round differently: visible after one large first
    # correction (K = 1), absorbed by z + δ once the corrections are tiny
    one = dict(kind=0, K=1, nx=nx, kx=0.01 * nx, h=1e-2)
    a = oracle.sbdf_integrate(y0, 1, linsol=0, **one)[1]
    b = oracle.sbdf_integrate(y0, 1, linsol=2, **one)[1]
    assert not np.array_equal(a, b) and np.max(np.abs(a - b) / np.abs(a)) <= 1e-15


def test_bruss_trajectory_vs_independent_radau():
    """Pins the nonlinear Brusselator trajectory of the SBDF oracle to an
    independent integrator: the semi-discrete system of P:369-371 (first-order
    upwind, periodic, written out here in numpy from the paper's equations,
    not the oracle's RHS) integrated by scipy's Radau IIA at tight
    tolerances.  The oracle's SBDF2 solution at t = 0.2 must approach it at
    second order under h-halving (error ratio ~ 4), with the error of the
    h = 1e-3 run (C1's step) below 1e-5."""
    from scipy.integrate import solve_ivp

    nx, b = 32, 1.0
    c, A, B, eps, alpha = PR["c"], PR["A"], PR["B"], PR["eps"], PR["alpha"]
    dx = b / nx
    x = np.arange(nx) * dx
    p = alpha * np.exp(-((x - b / 2) ** 2) / (2 * (b / 4) ** 2))
    y0 = np.stack([A + p, B / A + p, 3.0 + p], 1).reshape(-1)
    assert np.max(np.abs(y0 - oracle.bruss_ic(nx))) <= 1e-15

    def rhs(t, yy):
        q = yy.reshape(nx, 3)
        u, v, w = q[:, 0], q[:, 1], q[:, 2]
        adv = -c * (q - np.roll(q, 1, axis=0)) / dx           # upwind, c > 0, periodic
        react = np.stack([A - (w + 1) * u + v * u * u, w * u - v * u * u, (B - w) / eps - w * u], 1)
        return (adv + react).reshape(-1)

    def jac(t, yy):
        q = yy.reshape(nx, 3)
        J = np.zeros((3 * nx, 3 * nx))
        for i in range(nx):
            u, v, w = q[i]
            blk = np.array([[2 * u * v - (w + 1), u * u, -u], [w - 2 * u * v, -u * u, u], [-w, 0.0, -1 / eps - u]])
            J[3 * i:3 * i + 3, 3 * i:3 * i + 3] = blk - c / dx * np.eye(3)
            im = (i - 1) % nx
            J[3 * i:3 * i + 3, 3 * im:3 * im + 3] += c / dx * np.eye(3)
        return J

    T = 0.2
    ref = solve_ivp(rhs, (0.0, T), y0, method="Radau", jac=jac, rtol=1e-12, atol=1e-13).y[:, -1]
    errs = []
    for nsteps in (200, 400, 800):
        rc, y, _, _ = oracle.sbdf_integrate(y0, nsteps, kind=0, nx=nx, kx=c / dx, h=T / nsteps,
                                            newton_mode=2, A=A, B=B, eps=eps)
        assert rc == 0
        errs.append(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)))
    assert errs[0] <= 1e-5, errs
    assert 1.7 < math.log2(errs[0] / errs[1]) < 2.3 and 1.7 < math.log2(errs[1] / errs[2]) < 2.3, errs
    # the fixed K = 3 modified Newton of the parity runs and the bench lands on
    # the same solution
    rc, y3, _, _ = oracle.sbdf_integrate(y0, 200, kind=0, nx=nx, kx=c / dx, h=1e-3, K=3, A=A, B=B, eps=eps)
    assert rc == 0 and np.max(np.abs(y3 - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-5


def test_bruss3d_trajectory_vs_independent_radau():
    """The 3D problem of R19 (upwind along x, y, z, periodic; Gaussian IC with
    per-axis σ = L/4): the oracle's SBDF2 against Radau IIA on the
    semi-discrete system written out here, second-order convergence."""
    from scipy.integrate import solve_ivp

    n = 6
    c, A, B, eps, alpha = PR["c"], PR["A"], PR["B"], PR["eps"], PR["alpha"]
    d = 1.0 / n
    ax = np.arange(n) * d
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")        # cell (i, j, k) = (x, y, z)
    r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2
    p = alpha * np.exp(-r2 / (2 * 0.25 ** 2))
    p = np.transpose(p, (2, 1, 0)).reshape(-1)                # index ((k ny + j) nx + i)
    y0 = np.stack([A + p, B / A + p, 3.0 + p], 1).reshape(-1)
    assert np.max(np.abs(y0 - oracle.bruss_ic(n, n, n))) <= 1e-15

    def rhs(t, yy):
        q = yy.reshape(n, n, n, 3)                            # [k, j, i, s]
        adv = -c / d * ((q - np.roll(q, 1, axis=2)) + (q - np.roll(q, 1, axis=1)) + (q - np.roll(q, 1, axis=0)))
        u, v, w = q[..., 0], q[..., 1], q[..., 2]
        react = np.stack([A - (w + 1) * u + v * u * u, w * u - v * u * u, (B - w) / eps - w * u], -1)
        return (adv + react).reshape(-1)

    T = 0.1
    ref = solve_ivp(rhs, (0.0, T), y0, method="Radau", rtol=1e-12, atol=1e-13).y[:, -1]
    errs = []
    for nsteps in (100, 200, 400):
        rc, y, _, _ = oracle.sbdf_integrate(y0, nsteps, kind=0, nx=n, ny=n, nz=n, kx=c / d, ky=c / d, kz=c / d,
                                            h=T / nsteps, newton_mode=2)
        assert rc == 0
        errs.append(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)))
    assert errs[0] <= 1e-5, errs
    assert 1.7 < math.log2(errs[0] / errs[1]) < 2.3 and 1.7 < math.log2(errs[1] / errs[2]) < 2.3, errs
