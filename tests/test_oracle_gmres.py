"""Pins for the oracle's GMRES (the SPGMR role; the paper's global
Newton + GMRES configuration with the block solve as preconditioner),
CPU only.  Independent checks: Krylov theory (with an exact preconditioner
one step suffices; on a normal operator with k distinct eigenvalues GMRES
terminates in k steps), the true residual ‖b − A x‖₂ computed with numpy,
and the direct block LU solve."""
import numpy as np
import pytest

import oracle
import synth


def rand_blocks(stream, G, m, shift):
    return synth.uniform(stream, G * m * m, -1, 1).numpy().reshape(G, m, m) + shift * np.eye(m)


def test_exact_preconditioner_one_step():
    G, m = 200, 3
    A = rand_blocks(1, G, m, 3.0)
    b = synth.uniform(2, G * m, -1, 1).numpy()
    LU, piv, _ = oracle.lu_factor(A)
    x, steps, res = oracle.gmres(A, b, (LU, piv), maxl=5, tol=1e-12)
    assert steps == 1
    xd = oracle.lu_solve(LU, piv, b)
    assert np.max(np.abs(x - xd)) <= 1e-14 * np.max(np.abs(xd)) * 10


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_distinct_eigenvalues_terminate_in_k_steps(k):
    # A = diag(λ_i) with k distinct values: the minimal polynomial has degree k
    G, m = 64, 3
    lam = np.array([1.0, 2.5, 4.0, 7.0, 11.0])[:k]
    idx = (np.arange(G * m) * 7) % k
    diag = lam[idx].reshape(G, m)
    A = np.zeros((G, m, m))
    for i in range(m):
        A[:, i, i] = diag[:, i]
    b = synth.uniform(3, G * m, 0.5, 1.5).numpy()
    x, steps, res = oracle.gmres(A, b, None, maxl=10, tol=1e-13)
    assert steps == k
    assert np.allclose(x, b / diag.reshape(-1), rtol=1e-12, atol=0)


def test_true_residual_and_direct_solution():
    G, m = 40, 3
    A = rand_blocks(4, G, m, 2.0)
    b = synth.uniform(5, G * m, -1, 1).numpy()
    x, steps, res = oracle.gmres(A, b, None, maxl=60, tol=1e-11)
    r_true = b - np.einsum("gij,gj->gi", A, x.reshape(G, m)).reshape(-1)
    nb = np.linalg.norm(b)
    assert np.linalg.norm(r_true) <= 1e-10 * nb
    assert abs(np.linalg.norm(r_true) - res) <= 1e-10 * nb       # estimate = true residual
    xd = np.linalg.solve(A, b.reshape(G, m, 1))[..., 0].reshape(-1)
    assert np.allclose(x, xd, rtol=1e-9, atol=1e-11)
    # residual estimates decrease monotonically with maxl
    prev = np.inf
    for maxl in (1, 2, 4, 8):
        _, _, r = oracle.gmres(A, b, None, maxl=maxl, tol=0.0)
        assert r <= prev * (1 + 1e-12)
        prev = r


def test_global_newton_matches_task_local_C1():
    nx = 64
    y0 = oracle.bruss_ic(nx)
    kw = dict(kind=0, K=3, nx=nx, kx=0.01 * nx, h=1e-3)
    rc0, y0r, st0, _ = oracle.sbdf_integrate(y0, 100, **kw)
    rc1, y1r, st1, _ = oracle.sbdf_integrate(y0, 100, linsol=1, maxl=5, lin_tol=1e-10, **kw)
    assert rc0 == 0 and rc1 == 0
    assert st1["lin_iters"] == 3 * 100                 # exact block preconditioner: 1 step each
    assert np.max(np.abs(y1r - y0r) / np.abs(y0r)) <= 1e-12
