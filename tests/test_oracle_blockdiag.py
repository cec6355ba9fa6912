"""Pins for the oracle's block-diagonal matrix and batched LU (O5-O7), CPU.

Independent checks: exact rational Cramer's rule on small-integer blocks
(brute force), LAPACK getrf via scipy.linalg.lu_factor (same partial
pivoting rule, same 0-based ipiv convention), printed examples, structural
special cases (identity, diagonal, permutation), batched independence.
"""
from fractions import Fraction as F
from itertools import permutations

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth


def det_exact(M):
    m = len(M)
    tot = F(0)
    for p in permutations(range(m)):
        sgn = 1
        for i in range(m):
            for j in range(i + 1, m):
                if p[i] > p[j]:
                    sgn = -sgn
        prod = F(sgn)
        for i in range(m):
            prod *= F(M[i][p[i]])
        tot += prod
    return tot


def cramer(M, b):
    d = det_exact(M)
    m = len(M)
    xs = []
    for k in range(m):
        Mk = [[(b[i] if j == k else M[i][j]) for j in range(m)] for i in range(m)]
        xs.append(det_exact(Mk) / d)
    return d, xs


def test_golden_diag_solve(golden):
    for ex in golden["lu_solve"]:
        LU, piv, flag = oracle.lu_factor(np.array([ex["M"]], dtype=np.float64))
        assert flag == 0
        x = oracle.lu_solve(LU, piv, np.array(ex["r"], dtype=np.float64))
        assert np.array_equal(x, ex["x"]), ex["cite"]


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_identity_and_permutation_exact(m):
    I = np.eye(m)[None].repeat(3, axis=0)
    LU, piv, flag = oracle.lu_factor(I)
    assert flag == 0 and np.array_equal(LU, I) and np.array_equal(piv, np.tile(np.arange(m), (3, 1)))
    b = synth.uniform(1, 3 * m, -1, 1).numpy()
    assert np.array_equal(oracle.lu_solve(LU, piv, b), b)
    # permutation matrices: P x = b  ->  x = P^T b exactly
    for perm in list(permutations(range(m)))[:6]:
        Pm = np.eye(m)[list(perm)]
        LU, piv, flag = oracle.lu_factor(Pm[None])
        x = oracle.lu_solve(LU, piv, b[:m])
        assert flag == 0 and np.array_equal(x, Pm.T @ b[:m])


@pytest.mark.parametrize("m", [2, 3, 4])
def test_small_integer_blocks_vs_exact_cramer(m):
    G = 400
    A = synth.small_int_blocks(7, G, m).numpy()
    b = synth.small_int_blocks(8, G, m, -9, 9).numpy()[:, :, 0].copy()
    LU, piv, flag = oracle.lu_factor(A)
    sing = [g for g in range(G) if det_exact(A[g].tolist()) == 0]
    assert flag == (sing[0] + 1 if sing else 0)
    x = oracle.lu_solve(LU, piv, b.reshape(-1)).reshape(G, m)
    checked = 0
    for g in range(G):
        if g in sing:
            continue
        d, xs = cramer(A[g].tolist(), b[g].tolist())
        ex = np.array([float(v) for v in xs])
        # backward-stable LU: forward error ≲ cond·u; small-integer blocks are mild
        cond = np.linalg.cond(A[g])
        assert np.all(np.abs(x[g] - ex) <= 64 * 2 ** -53 * cond * np.maximum(np.abs(ex).max(), 1)), g
        checked += 1
    assert checked > G // 2


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8])
def test_factors_match_lapack_getrf(m):
    G = 200
    A = synth.uniform(11, G * m * m, -1, 1).numpy().reshape(G, m, m)
    LU, piv, flag = oracle.lu_factor(A)
    assert flag == 0
    for g in range(G):
        lu_ref, piv_ref = scipy.linalg.lu_factor(A[g])
        assert np.array_equal(piv[g], piv_ref), g      # same pivot rule (first max)
        assert np.allclose(LU[g], lu_ref, rtol=1e-12, atol=1e-13), g


def test_singular_flag_first_block_and_independence():
    G, m = 10, 3
    A = synth.uniform(12, G * 9, -1, 1).numpy().reshape(G, 3, 3)
    A[4, :, 1] = 0.0            # zero column -> exactly zero pivot
    A[7] = 0.0
    _, _, flag = oracle.lu_factor(A)
    assert flag == 5
    # batched independence: perturbing block j changes only x_j
    B = synth.uniform(13, G * 9, -1, 1).numpy().reshape(G, 3, 3) + 3 * np.eye(3)
    b = synth.uniform(14, G * 3, -1, 1).numpy()
    x0 = oracle.lu_solve(*oracle.lu_factor(B)[:2], b)
    B2 = B.copy(); B2[6, 0, 2] += 0.5
    x1 = oracle.lu_solve(*oracle.lu_factor(B2)[:2], b)
    diff = np.nonzero(x0 != x1)[0] // 3
    assert set(diff.tolist()) == {6}


def test_round_trip_and_matvec():
    G, m = 1000, 3
    A = synth.uniform(15, G * 9, -1, 1).numpy().reshape(G, 3, 3) + 2 * np.eye(3)
    b = synth.uniform(16, G * 3, -1, 1).numpy()
    y = oracle.block_matvec(A, b)
    assert np.allclose(y.reshape(G, 3), np.einsum("gij,gj->gi", A, b.reshape(G, 3)), rtol=1e-15, atol=1e-15)
    LU, piv, _ = oracle.lu_factor(A)
    x = oracle.lu_solve(LU, piv, y)
    assert np.max(np.abs(x - b)) <= 1e-12                         # S:335 round trip
    assert np.allclose(x.reshape(G, 3), np.linalg.solve(A, y.reshape(G, 3, 1))[..., 0], rtol=1e-12, atol=1e-13)


def test_scale_add_identity():
    A = synth.uniform(17, 5 * 9, -2, 2).numpy().reshape(5, 3, 3)
    assert np.array_equal(oracle.scale_add_identity(0.0, A), np.tile(np.eye(3), (5, 1, 1)))
    Ad = synth.dyadic(17, 45).numpy().reshape(5, 3, 3)
    M = oracle.scale_add_identity(-0.5, Ad)
    assert np.array_equal(M, -0.5 * Ad + np.eye(3))                 # dyadic: exact


# ---------------------------------------------------------------------------
# Block inverse by symbolic Gauss-Jordan (the paper's task-local solver,
# P:389-390): pinned by the adjugate formula in exact rationals, numpy's
# LAPACK inverse, structural special cases and the exact-arithmetic identity
# A·A^{-1} = I.

def inv_exact(M):
    """Exact inverse by the adjugate (cofactor) formula, independent of GJ."""
    m = len(M)
    d = det_exact(M)
    inv = [[F(0)] * m for _ in range(m)]
    for i in range(m):
        for j in range(m):
            minor = [[M[r][c] for c in range(m) if c != i] for r in range(m) if r != j]
            inv[i][j] = (-1) ** (i + j) * det_exact(minor) / d
    return inv


def test_gj_identity_and_diagonal_exact():
    D = np.zeros((4, 3, 3))
    diag = [(1.0, 1.0, 1.0), (2.0, -4.0, 0.5), (3.0, 7.0, 1e-3), (-1.0, 10.0, 5e5)]
    for g, d in enumerate(diag):
        D[g] = np.diag(d)
    B, flag = oracle.gj_inverse(D)
    assert flag == 0
    for g, d in enumerate(diag):
        expect = np.diag([1.0 / x for x in d])          # RN(1/d): one rounding each
        assert np.array_equal(B[g], expect)


def test_gj_small_integer_blocks_vs_exact_rationals():
    rng = np.random.default_rng(11)
    checked = 0
    while checked < 300:
        M = rng.integers(-4, 5, (3, 3)).astype(float)
        M += np.diag(rng.integers(5, 9, 3))              # leading minors nonzero
        Mi = [[int(v) for v in row] for row in M]
        if det_exact(Mi) == 0 or Mi[0][0] == 0 or det_exact([r[:2] for r in Mi[:2]]) == 0:
            continue
        B, flag = oracle.gj_inverse(M[None])
        assert flag == 0
        ex = inv_exact(Mi)
        for i in range(3):
            for j in range(3):
                e = float(ex[i][j])
                # a handful of roundings on well-conditioned blocks
                assert abs(B[0, i, j] - e) <= 64 * 2 ** -53 * max(1.0, abs(e)), (M, i, j)
        checked += 1


def test_gj_random_blocks_vs_lapack_and_identity():
    G = 5000
    u = synth.uniform(synth.S_CELL, 9 * G, -1, 1).numpy().reshape(G, 3, 3)
    M = u + 4.0 * np.eye(3)[None]                         # diagonally dominant: no pivoting needed
    B, flag = oracle.gj_inverse(M)
    assert flag == 0
    ref = np.linalg.inv(M)
    assert np.max(np.abs(B - ref) / np.maximum(np.abs(ref), 1e-3)) <= 1e-13
    I = np.einsum("gij,gjk->gik", M, B)
    assert np.max(np.abs(I - np.eye(3)[None])) <= 1e-14


def test_gj_apply_is_left_to_right_matvec():
    G = 1000
    B = synth.uniform(3, 9 * G, -1, 1).numpy().reshape(G, 3, 3)
    b = synth.uniform(4, 3 * G, -1, 1).numpy()
    x = oracle.gj_apply(B, b).reshape(G, 3)
    bb = b.reshape(G, 3)
    for g in range(0, G, 97):
        for i in range(3):
            s = B[g, i, 0] * bb[g, 0]
            s = s + B[g, i, 1] * bb[g, 1]
            s = s + B[g, i, 2] * bb[g, 2]
            assert x[g, i] == s


def test_gj_zero_leading_pivot_flags_block():
    # nonsingular, but Gauss-Jordan without pivoting meets a zero pivot: the
    # method's documented limitation (the symbolic sequence has no pivoting)
    M = np.stack([np.eye(3), np.array([[0.0, 1, 0], [1, 0, 0], [0, 0, 1]]), np.eye(3)])
    _, flag = oracle.gj_inverse(M)
    assert flag == 2


def test_gj_newton_matrix_equals_lu_solution():
    # On Brusselator Newton matrices M = I - γJ the GJ inverse and the LU
    # solve give the same correction up to rounding
    G = 2000
    u = synth.uniform(synth.S_CELL, G, 0.5, 2.0).numpy()
    y = np.stack([u, 3.0 * u, 3.5 - 0.1 * u], 1).reshape(-1)
    J = oracle.bruss_jacobian(y)
    M = np.eye(3)[None] - 2e-3 / 3 * J
    B, flag = oracle.gj_inverse(M)
    LU, piv, f2 = oracle.lu_factor(M)
    assert flag == 0 and f2 == 0
    r = synth.uniform(7, 3 * G, -1, 1).numpy()
    x1 = oracle.gj_apply(B, r)
    x2 = oracle.lu_solve(LU, piv, r)
    assert np.max(np.abs(x1 - x2) / np.maximum(np.abs(x2), 1e-300)) <= 1e-12
