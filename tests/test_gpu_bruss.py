"""GPU parity of the advection–reaction problem kernels and the Newton-step
driver against the oracle (through the C ABI).

Per-kernel: reaction, Jacobian, advection bit-exact; IC within 4 ulp
(exp is not correctly rounded on either side, DESIGN R13).  Driver: the
state after fixed-K steps is bit-identical to the oracle's (the only
reassociated quantity, the WRMS ν, does not feed back into the state in
fixed-K mode) — the north star's bar is rel 1e-9, asserted separately.
Multi-rank: P logical ranks on one GPU through the in-process fake
communicator (NCCL forbids two ranks per device), bit-identical to P = 1.
"""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bits_equal, needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda]
C, A, B, EPS = 0.01, 1.0, 3.5, 5e-6


@pytest.fixture(scope="module")
def S():
    from paper_2011_12984_b200 import sunbw
    return sunbw


@pytest.fixture(scope="module")
def ctx(S):
    c = S.Context(0)
    yield c
    c.destroy()


def kappas(nx, ny=1, nz=1, L=(1.0, 1.0, 1.0)):
    return (C / (L[0] / nx), C / (L[1] / ny) if ny > 1 else 0.0, C / (L[2] / nz) if nz > 1 else 0.0)


def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


# ------------------------------------------------------------ kernels
def test_reaction_and_jacobian_bit_exact(S, ctx):
    G = 100_003
    y = torch.stack([synth.uniform(1, G, 0.0, 2), synth.uniform(2, G, 0.5, 4),
                     synth.uniform(3, G, 0.5, 4)], 1).reshape(-1)
    yd = y.cuda()
    P = S.Problem(ctx, S.bruss_params(dim=1, nx=G))
    f = torch.empty_like(yd)
    S.BW_ReactionRHS(P, S.NVector(ctx, yd), S.NVector(ctx, f))
    assert_bits_equal(f, oracle.bruss_reaction(y.numpy()), "reaction")
    J = torch.empty(G, 3, 3, dtype=torch.float64, device="cuda")
    S.BW_ReactionJacobian(P, S.NVector(ctx, yd), S.SUNMatrix(ctx, J))
    assert_bits_equal(J.reshape(-1), oracle.bruss_jacobian(y.numpy()).reshape(-1), "jacobian")
    P.destroy()


@pytest.mark.parametrize("shape", [(64, 1, 1), (1000, 1, 1), (16, 12, 8), (33, 7, 5), (64, 64, 32),
                                   (10, 1, 6), (6, 5, 1), (256, 4, 3)])
def test_advection_and_ic(S, ctx, shape):
    nx, ny, nz = shape
    dim = 1 if ny == nz == 1 else 3
    P = S.Problem(ctx, S.bruss_params(dim=dim, nx=nx, ny=ny, nz=nz))
    n = 3 * nx * ny * nz
    y = synth.uniform(1, n, 0.0, 1.0)
    yd = y.cuda()
    f = torch.empty_like(yd)
    S.BW_AdvectionRHS(P, S.NVector(ctx, yd), S.NVector(ctx, f))
    ref = oracle.advection(y.numpy(), nx, ny, nz, *kappas(nx, ny, nz))
    assert_bits_equal(f, ref, f"advection {shape}")
    S.BW_InitialCondition(P, S.NVector(ctx, yd))
    ic = oracle.bruss_ic(nx, ny, nz)
    got = yd.cpu().numpy()
    assert np.max(np.abs(got - ic) / np.abs(ic)) <= 4 * 2 ** -52
    P.destroy()


# ------------------------------------------------------------ driver
def run_gpu(S, ctx, params, y0_np, nsteps, **opts):
    P = S.Problem(ctx, params)
    y0 = torch.from_numpy(y0_np).cuda()
    yout = torch.empty_like(y0)
    st = S.Stepper(P, S.NVector(ctx, y0), S.stepper_options(**opts))
    rc, stats = st.advance(nsteps, S.NVector(ctx, yout))
    st.destroy()
    P.destroy()
    return rc, yout.cpu().numpy(), stats


@pytest.mark.parametrize("mode", ["eager", "graph", "fused", "fused_graph"])
def test_C1_fixed_K_matches_oracle(S, ctx, mode):
    """C1: 1D Brusselator, 64 cells, b = 1, h = 1e-3, K = 3, to t = 1."""
    nx, steps = 64, 1000
    y0 = oracle.bruss_ic(nx)
    kx = kappas(nx)[0]
    opts = dict(h=1e-3, K=3, use_graph=mode in ("graph", "fused_graph"), fused=mode.startswith("fused"))
    rc, y, stats = run_gpu(S, ctx, S.bruss_params(dim=1, nx=nx), y0, steps, **opts)
    assert rc == 0 and stats["steps"] == steps and stats["newton_iters"] == 3 * steps
    rc2, yref, st2, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, kx=kx, h=1e-3)
    assert rc2 == 0
    assert rel_err(y, yref) <= 1e-9                       # north-star bar (DESIGN R22)
    assert_bits_equal(y, yref, f"C1 {mode}")              # same RN sequence: identical bits
    assert abs(stats["last_nu"] - st2["last_nu"]) <= 1e-12 * max(st2["last_nu"], 1e-30) + 1e-300


def test_C1_every_100_steps(S, ctx):
    nx = 64
    y0 = oracle.bruss_ic(nx)
    kx = kappas(nx)[0]
    _, _, _, ylog = oracle.sbdf_integrate(y0, 1000, kind=0, K=3, nx=nx, kx=kx, h=1e-3, log_every=100)
    P = S.Problem(ctx, S.bruss_params(dim=1, nx=nx))
    yd = torch.from_numpy(y0).cuda()
    yout = torch.empty_like(yd)
    st = S.Stepper(P, S.NVector(ctx, yd), S.stepper_options(h=1e-3, K=3))
    for k in range(10):
        rc, _ = st.advance(100, S.NVector(ctx, yout))
        assert rc == 0
        assert rel_err(yout.cpu().numpy(), ylog[k]) <= 1e-9, k
    st.destroy(); P.destroy()


@pytest.mark.parametrize("fused", [False, True])
def test_linear_test_equation_closed_form(S, ctx, fused):
    lamE, lamI, h, nsteps = -1.0, -10.0, 1e-2, 50
    G = 1001
    y0 = synth.uniform(1, 3 * G, 0.5, 1.5).numpy()
    params = S.bruss_params(dim=1, nx=G, kind=1, lam_E=lamE, lam_I=lamI)
    rc, y, _ = run_gpu(S, ctx, params, y0, nsteps, h=h, K=2, fused=fused)
    rc2, yref, _, _ = oracle.sbdf_integrate(y0, nsteps, kind=1, K=2, nx=G, lam_E=lamE, lam_I=lamI, h=h)
    assert rc == 0 and rc2 == 0
    assert_bits_equal(y, yref, "linear test")


def test_3D_small_matches_oracle(S, ctx):
    nx, ny, nz, steps = 16, 12, 8, 10
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
    rc2, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz,
                                            kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    for fused in (False, True):
        rc, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused)
        assert rc == 0 and rc2 == 0
        assert rel_err(y, yref) <= 1e-9
        assert_bits_equal(y, yref, f"3D fused={fused}")


@pytest.mark.parametrize("shape", [(128, 6, 4), (256, 4, 3), (128, 3, 2)])
@pytest.mark.parametrize("fused_adv", [True, False])
def test_3D_fused_step_kernel(S, ctx, shape, fused_adv):
    """The single-kernel step (advection inside the TMA-staged Newton
    kernel, nx % 128 == 0) against the oracle, SBDF1 + SBDF2 steps."""
    nx, ny, nz = shape
    steps = 6
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
    rc, y, stats = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=True,
                           fused_advection=fused_adv, use_graph=True)
    assert rc == 0
    assert_bits_equal(y, yref, f"fused step {shape} adv={fused_adv}")
    assert abs(stats["last_nu"] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]


def test_tolerance_mode(S, ctx):
    nx, steps = 64, 50
    y0 = oracle.bruss_ic(nx)
    kx = kappas(nx)[0]
    rc, y, stats = run_gpu(S, ctx, S.bruss_params(dim=1, nx=nx), y0, steps, h=1e-3, K=5,
                           newton_mode=1, tol_nl=1e-3)
    rc2, yref, st2, _ = oracle.sbdf_integrate(y0, steps, kind=0, newton_mode=1, K=5, tol_nl=1e-3,
                                              nx=nx, kx=kx, h=1e-3)
    assert rc == 0 and rc2 == 0
    assert stats["newton_iters"] == st2["newton_iters"]
    assert rel_err(y, yref) <= 1e-9
    # a tolerance that cannot be met -> recoverable failure code
    rc, _, stats = run_gpu(S, ctx, S.bruss_params(dim=1, nx=nx), y0, 3, h=1e-3, K=1,
                           newton_mode=1, tol_nl=1e-300)
    assert rc == 2 and stats["fails"] == 1


def test_C4_reaction_only_cells(S, ctx):
    """C4 shape (independent reaction cells, batched block Newton only) at a
    reduced count, composed and fused."""
    G, steps = 200_000, 5
    u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
    y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
    params = S.bruss_params(dim=1, nx=G, reaction_only=True)
    rc2, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=G, reaction_only=True, h=1e-3)
    for fused in (False, True):
        rc, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused)
        assert rc == 0
        assert_bits_equal(y, yref, f"C4 fused={fused}")


def _inject_extremes(y0, stream):
    """Cells whose divisions leave the fused kernel's fast range: tiny
    magnitudes (products below 2^-480), exact zeros and negative zeros."""
    y = y0.copy().reshape(-1, 3)
    G = y.shape[0]
    u = synth.uniform(stream, G).numpy()
    y[u < 0.03] *= 1e-160
    y[(u >= 0.03) & (u < 0.05)] = 0.0
    y[(u >= 0.05) & (u < 0.06), 0] = -0.0
    y[(u >= 0.06) & (u < 0.07), 2] = 1e-300
    return y.reshape(-1)


def test_fused_guarded_divisions_fall_back_exactly(S, ctx):
    """The fused kernel divides by Markstein steps on shared reciprocals and
    recomputes a cell with IEEE divisions when any operand guard fails;
    cells built to fail them (and ragged-tail cells) stay bit-identical to
    the oracle, as do the composed kernels."""
    G, steps = 100_003, 3
    u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
    y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
    y0 = _inject_extremes(y0, 77)
    params = S.bruss_params(dim=1, nx=G, reaction_only=True)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=G, reaction_only=True, h=1e-3)
    for fused in (False, True):
        _, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused)
        assert_bits_equal(y, yref, f"extreme cells fused={fused}")


def test_fused_advection_guarded_divisions(S, ctx):
    nx, ny, nz = 128, 4, 3
    steps = 3
    y0 = _inject_extremes(oracle.bruss_ic(nx, ny, nz), 78)
    k = kappas(nx, ny, nz)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz,
                                          kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
    _, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=True, use_graph=True)
    assert_bits_equal(y, yref, "3D fused step with extreme cells")


# ------------------------------------------------------ multi-rank (fake comm)
def run_ranks(S, nranks, fn):
    comm = S.FakeComm(nranks)
    out, errs = [None] * nranks, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                c = S.Context(0, stream)
                c.set_fake_comm(comm, r)
                out[r] = fn(c, r)
                stream.synchronize()
                c.destroy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    comm.destroy()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("dim,fused,linsol", [(1, False, 0), (3, False, 0), (3, True, 0), ("3big", True, 0),
                                              ("3big", True, 2), (3, False, 2)])
def test_multirank_driver_invariance(S, nranks, dim, fused, linsol):
    if dim == 1:
        shape = (96, 1, 1)
    elif dim == "3big":
        shape, dim = (128, 4, 8), 3          # in-kernel advection, halo plane via TMA
    else:
        shape = (12, 10, 8)
    nx, ny, nz = shape
    steps = 8
    y0 = oracle.bruss_ic(nx, ny, nz)
    params = S.bruss_params(dim=dim, nx=nx, ny=ny, nz=nz)
    k = kappas(nx, ny, nz)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3, linsol=linsol)

    def fn(c, r):
        P = S.Problem(c, params)
        n = 3 * P.local_cells
        off = 3 * P.cell_offset
        y = torch.from_numpy(y0[off:off + n].copy()).cuda()
        yout = torch.empty_like(y)
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=1e-3, K=3, use_graph=False,
                                                              fused=fused, linsol=linsol))
        rc, stats = st.advance(steps, S.NVector(c, yout))
        c.stream.synchronize()
        res = (rc, off, yout.cpu().numpy(), stats)
        st.destroy(); P.destroy()
        return res

    res = run_ranks(S, nranks, fn)
    y = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    assert all(r[0] == 0 for r in res)
    assert_bits_equal(y, yref, f"P={nranks} dim={dim}")
    nus = [r[3]["last_nu"] for r in res]
    assert len(set(nus)) == 1                                 # identical global ν on all ranks
    assert abs(nus[0] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]


@pytest.mark.parametrize("nranks", [2, 3])
def test_multirank_reductions(S, nranks):
    n_loc = 100_003
    N = n_loc * nranks
    x = synth.uniform(1, N, -1, 1).numpy()
    w = synth.uniform(3, N, 0.5, 1.5).numpy()

    def fn(c, r):
        xs = torch.from_numpy(x[r * n_loc:(r + 1) * n_loc].copy()).cuda()
        ws = torch.from_numpy(w[r * n_loc:(r + 1) * n_loc].copy()).cuda()
        vx, vw = S.NVector(c, xs), S.NVector(c, ws)
        assert vx.global_length() == N
        return (S.N_VWrmsNorm(vx, vw), S.N_VDotProd(vx, vw), S.N_VMaxNorm(vx), S.N_VMin(vx),
                S.N_VDotProdMulti(vx, [vw, vx]))

    res = run_ranks(S, nranks, fn)
    assert all(r == res[0] for r in res)                      # same bits on every rank
    wr, dt, mx, mn, dm = res[0]
    assert abs(wr - oracle.wrms(x, w)) <= 1e-12 * oracle.wrms(x, w)
    assert abs(dt - oracle.dot(x, w)) <= 1e-12 * float(np.sum(np.abs(x * w)))
    assert mx == oracle.max_norm(x) and mn == oracle.min_(x)
    assert abs(dm[1] - oracle.dot(x, x)) <= 1e-12 * oracle.dot(x, x)


# ------------------------------------------------ full bench-size parity
@pytest.mark.slow
@pytest.mark.parametrize("fused", [True, False])
def test_C5_slab_full_size_two_steps(S, ctx, fused):
    """The bench's workload and launch configuration (256^3 cells, fused
    single-kernel step or the composed path), SBDF1 + SBDF2 steps, the whole
    state against the oracle run on the host (about 15 s of CPU)."""
    n = 256
    steps = 2
    y0 = oracle.bruss_ic(n, n, n)
    k = kappas(n, n, n)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=n, ny=n, nz=n,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    params = S.bruss_params(dim=3, nx=n, ny=n, nz=n)
    rc, y, stats = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused, use_graph=False)
    assert rc == 0
    assert_bits_equal(y, yref, f"C5 256^3 fused={fused}")
    assert abs(stats["last_nu"] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]


@pytest.mark.slow
def test_C4_full_size_1e7_cells(S, ctx):
    """C4: 1e7 independent reaction cells, batched block Newton only, at full
    size, two steps, fused and composed, against the oracle."""
    G, steps = 10_000_000, 2
    u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
    y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=G, reaction_only=True, h=1e-3)
    params = S.bruss_params(dim=1, nx=G, reaction_only=True)
    for fused in (True, False):
        rc, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused)
        assert rc == 0
        assert_bits_equal(y, yref, f"C4 1e7 fused={fused}")


@pytest.mark.slow
def test_C3_128cubed_ten_steps(S, ctx):
    """C3 (3D, 128^3 cells, single B200): 10 steps of the composed path and
    of the single-kernel fused step against the oracle on the whole state."""
    n = 128
    steps = 10
    y0 = oracle.bruss_ic(n, n, n)
    k = kappas(n, n, n)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=n, ny=n, nz=n,
                                          kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    params = S.bruss_params(dim=3, nx=n, ny=n, nz=n)
    for fused in (False, True):
        rc, y, _ = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=3, fused=fused, use_graph=True)
        assert rc == 0
        assert_bits_equal(y, yref, f"C3 128^3 fused={fused}")


def test_fused_pivoting_cells_fall_back_exactly(S, ctx):
    """The fused kernel's fast path factors without row exchanges and sends a
    cell whose Newton matrix needs partial pivoting (|a_ik| > |a_kk|) to the
    exact path, which pivots (first-maximum rule, O6).  Large steps on
    random states make a sizeable fraction of the blocks pivot; the state
    stays bit-identical to the oracle."""
    G, steps, h = 50_001, 3, 0.1
    u = synth.uniform(synth.S_CELL, G, 0.2, 2.0).numpy()
    v = synth.uniform(synth.S_CELL + 10, G, 0.2, 3.0).numpy()
    w = synth.uniform(synth.S_CELL + 11, G, 0.2, 3.0).numpy()
    y0 = np.stack([u, v, w], 1).reshape(-1)
    M = np.eye(3)[None] - h * oracle.bruss_jacobian(y0)
    _, piv, _ = oracle.lu_factor(M)
    assert np.mean(np.any(piv != np.arange(3)[None], axis=1)) > 0.01   # the test exercises pivoting
    params = S.bruss_params(dim=1, nx=G, reaction_only=True)
    rc2, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=G, reaction_only=True, h=h)
    assert rc2 == 0
    for fused in (False, True):
        rc, y, _ = run_gpu(S, ctx, params, y0, steps, h=h, K=3, fused=fused)
        assert rc == 0
        assert_bits_equal(y, yref, f"pivoting cells fused={fused}")


@pytest.mark.parametrize("K", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(128, 3, 2), (300, 1, 1)])
def test_fused_newton_iteration_counts(S, ctx, K, shape):
    """The fused step for every compile-time K other than the bench's 3 (the
    Newton loop is unrolled per K; K = 1 forms the WRMS partial in its only
    iteration), 3D with in-kernel advection and 1D with the stencil kernel
    and a ragged tail: bit-identical states, ν to 1e-12."""
    nx, ny, nz = shape
    dim = 1 if ny == nz == 1 else 3
    steps = 4
    y0 = oracle.bruss_ic(nx, ny, nz)
    k = kappas(nx, ny, nz)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=K, nx=nx, ny=ny, nz=nz,
                                              kx=k[0], ky=k[1], kz=k[2], h=1e-3)
    params = S.bruss_params(dim=dim, nx=nx, ny=ny, nz=nz)
    rc, y, stats = run_gpu(S, ctx, params, y0, steps, h=1e-3, K=K, fused=True, use_graph=True)
    assert rc == 0 and stats["newton_iters"] == K * steps
    assert_bits_equal(y, yref, f"fused K={K} {shape}")
    assert abs(stats["last_nu"] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]


# ------------------------------------------- block inverse (symbolic GJ, R29)
@pytest.mark.parametrize("case", ["C1", "3D", "C4", "extreme", "K1"])
def test_fused_block_inverse_matches_oracle(S, ctx, case):
    """The paper's task-local block solve — each 3x3 Newton block inverted by
    symbolic Gauss-Jordan and applied as a matrix-vector product (P:389-390,
    linsol = 2) — in the fused step: bit-identical to the oracle's GJ path."""
    K, h = 3, 1e-3
    if case == "C1":
        nx, ny, nz, steps = 64, 1, 1, 1000
        y0 = oracle.bruss_ic(nx)
        params, dim = S.bruss_params(dim=1, nx=nx), 1
        ro = False
    elif case in ("3D", "K1"):
        nx, ny, nz, steps = 128, 6, 4, 6
        y0 = oracle.bruss_ic(nx, ny, nz)
        params, ro = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz), False
        K = 1 if case == "K1" else 3
    else:
        G, steps = 100_003, 3
        nx, ny, nz = G, 1, 1
        u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
        y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
        if case == "extreme":
            y0 = _inject_extremes(y0, 79)
        params, ro = S.bruss_params(dim=1, nx=G, reaction_only=True), True
    k = kappas(nx, ny, nz) if not ro else (0.0, 0.0, 0.0)
    rc2, yref, stref, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=K, nx=nx, ny=ny, nz=nz,
                                                kx=k[0], ky=k[1], kz=k[2], h=h, reaction_only=ro,
                                                linsol=2)
    rc, y, stats = run_gpu(S, ctx, params, y0, steps, h=h, K=K, fused=True, linsol=2)
    if case != "extreme":
        assert rc2 == 0 and rc == 0
        assert abs(stats["last_nu"] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]
    assert_bits_equal(y, yref, f"GJ {case}")


def test_block_inverse_zero_pivot_is_singular(S, ctx):
    """Gauss-Jordan without row exchanges meets a zero pivot on a block that
    partial pivoting would factor: reported as a singular block (the
    method's limitation), like the oracle."""
    G = 300
    u = synth.uniform(synth.S_CELL, G, 0.5, 1.5).numpy()
    y0 = np.stack([u, 2.0 * u, 3.0 + 0 * u], 1).reshape(-1)
    # M_00 = 1 - γ(2uv - (w + 1)) = 0 for cell 17: choose v so that 2uv = w + 1 + 1/γ
    h = 1e-3
    y0[3 * 17 + 1] = (y0[3 * 17 + 2] + 1.0 + 1.0 / h) / (2.0 * y0[3 * 17])
    M = np.eye(3)[None] - h * oracle.bruss_jacobian(y0)
    if M[17, 0, 0] != 0.0:
        pytest.skip("no exact zero pivot from this construction")
    _, flag = oracle.gj_inverse(M)
    assert flag == 18
    params = S.bruss_params(dim=1, nx=G, reaction_only=True)
    rc, _, stats = run_gpu(S, ctx, params, y0, 1, h=h, K=3, fused=True, linsol=2)
    assert rc != 0 and stats["singular"] == 18


# ------------------------------------ small problems: many steps per launch
@pytest.mark.parametrize("case", ["C1", "3D_8cubed", "linear", "reaction_only", "C1_GJ", "K5"])
def test_fused_multistep_small_problems(S, ctx, case):
    """A fused fixed-K Advance on one rank with at most 512 cells runs in one
    launch with the state on chip (launch-bound small problems);
    it is bit-identical to the oracle and to one launch per step."""
    K, linsol, kw, steps = 3, 0, {}, 300
    if case in ("C1", "C1_GJ", "K5"):
        nx, ny, nz, dim = 64, 1, 1, 1
        y0 = oracle.bruss_ic(nx)
        linsol = 2 if case == "C1_GJ" else 0
        K = 5 if case == "K5" else 3
        params = S.bruss_params(dim=1, nx=nx)
        okw = dict(kind=0, nx=nx, kx=kappas(nx)[0])
    elif case == "3D_8cubed":
        nx = ny = nz = 8
        y0 = oracle.bruss_ic(nx, ny, nz)
        params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
        k = kappas(nx, ny, nz)
        okw = dict(kind=0, nx=nx, ny=ny, nz=nz, kx=k[0], ky=k[1], kz=k[2])
    elif case == "linear":
        G = 200
        y0 = synth.uniform(1, 3 * G, 0.5, 1.5).numpy()
        params = S.bruss_params(dim=1, nx=G, kind=1, lam_E=-1.0, lam_I=-10.0)
        okw = dict(kind=1, nx=G, lam_E=-1.0, lam_I=-10.0)
    else:
        G = 500
        u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
        y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
        params = S.bruss_params(dim=1, nx=G, reaction_only=True)
        okw = dict(kind=0, nx=G, reaction_only=True)
    rc2, yref, stref, _ = oracle.sbdf_integrate(y0, steps, K=K, h=1e-3, linsol=linsol, **okw)
    assert rc2 == 0
    outs = []
    for single in (False, True):
        P = S.Problem(ctx, params)
        yd = torch.from_numpy(y0).cuda()
        yout = torch.empty_like(yd)
        st = S.Stepper(P, S.NVector(ctx, yd), S.stepper_options(h=1e-3, K=K, fused=True, linsol=linsol,
                                                                 single_step_launches=single))
        l0 = ctx.launches
        rc, stats = st.advance(100)                    # two calls: the state carries over
        rc2b, stats = st.advance(steps - 100, S.NVector(ctx, yout))
        launches = ctx.launches - l0
        st.destroy(); P.destroy()
        assert rc == 0 and rc2b == 0 and stats["steps"] == steps and stats["newton_iters"] == K * steps
        assert_bits_equal(yout.cpu().numpy(), yref, f"{case} single={single}")
        assert abs(stats["last_nu"] - stref["last_nu"]) <= 1e-12 * stref["last_nu"]
        outs.append(launches)
    assert outs[0] < outs[1]                           # far fewer launches in one-launch mode


@pytest.mark.parametrize("peer", ["1", "0"])
@pytest.mark.parametrize("nranks", [2, 4])
def test_multirank_fused_copy_engine_halo(S, nranks, peer, monkeypatch):
    """The fused step at P > 1 with the halo plane moved by the copy engine
    into the right neighbour's double-buffered slot (peer_halo.cu: stream
    memory-op flags, no SM, overlapping the interior launch) or, with
    SUNBW_PEER_HALO=0, by the communicator's send/recv: bit-identical to the
    oracle either way, and the split step's timing kinds (halo on the side
    stream, interior, plane 0) are reported."""
    monkeypatch.setenv("SUNBW_PEER_HALO", peer)
    nx, ny, nzl, steps = 128, 8, 4, 6
    nz = nzl * nranks
    y0 = oracle.bruss_ic(nx, ny, nz)
    params = S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz)
    k = kappas(nx, ny, nz)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=nz, kx=k[0], ky=k[1], kz=k[2],
                                          h=1e-3)

    def fn(c, r):
        P = S.Problem(c, params)
        n, off = 3 * P.local_cells, 3 * P.cell_offset
        y = torch.from_numpy(y0[off:off + n].copy()).cuda()
        yout = torch.empty_like(y)
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=1e-3, K=3, use_graph=False, fused=True,
                                                              timing=True))
        rc, _ = st.advance(steps, S.NVector(c, yout))
        c.stream.synchronize()
        kt = st.kernel_times()
        res = (rc, off, yout.cpu().numpy(), set(kt))
        st.destroy(); P.destroy()
        return res

    res = run_ranks(S, nranks, fn)
    assert all(r[0] == 0 for r in res)
    assert all({"halo", "fused_newton", "fused_plane0"} <= r[3] for r in res), res[0][3]
    y = np.concatenate([r[2] for r in sorted(res, key=lambda t: t[1])])
    assert_bits_equal(y, yref, f"P={nranks} peer={peer}")
