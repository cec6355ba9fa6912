"""Pins for the oracle's adaptive IMEX ARK (the paper's integrator, ARKODE
IMEX; tableau ARK3(2)4L[2]SA, DESIGN R26), CPU only.

Independent checks: the additive order conditions of the tableau through
order 3 (and order 2 of the embedding) in exact rational arithmetic on the
published coefficients and on the doubles the oracle uses; third-order
convergence against exp(λt) on the split linear test equation;
error-control behaviour (tolerance proportionality, step rejections,
recomputation after a failed stage solve)."""
import math
from fractions import Fraction as F

import numpy as np
import pytest

import oracle

G = F(1767732205903, 4055673282236)
C = [F(0), F(1767732205903, 2027836641118), F(3, 5), F(1)]
AE = [[0, 0, 0, 0], [F(1767732205903, 2027836641118), 0, 0, 0],
      [F(5535828885825, 10492691773637), F(788022342437, 10882634858940), 0, 0],
      [F(6485989280629, 16251701735622), F(-4246266847089, 9704473918619),
       F(10755448449292, 10357097424841), 0]]
AI = [[0, 0, 0, 0], [G, G, 0, 0],
      [F(2746238789719, 10658868560708), F(-640167445237, 6845629431997), G, 0],
      [F(1471266399579, 7840856788654), F(-4482444167858, 7529755066697),
       F(11266239266428, 11593286722821), G]]
B = [F(1471266399579, 7840856788654), F(-4482444167858, 7529755066697),
     F(11266239266428, 11593286722821), G]
D = [F(2756255671327, 12835298489170), F(-10771552573575, 22201958757719),
     F(9247589265047, 10645013368117), F(2193209047091, 5459859503100)]


def order_residuals(AE, AI, b, d, c):
    s = 4
    res = []
    for A in (AE, AI):
        res += [sum(A[i]) - c[i] for i in range(s)]
        res += [sum(b) - 1, sum(b[i] * c[i] for i in range(s)) - F(1, 2) if isinstance(b[0], F)
                else sum(b[i] * c[i] for i in range(s)) - 0.5]
        res.append(sum(b[i] * c[i] ** 2 for i in range(s)) - (F(1, 3) if isinstance(b[0], F) else 1 / 3))
    six = F(1, 6) if isinstance(b[0], F) else 1 / 6
    for A1 in (AE, AI):
        for A2 in (AE, AI):       # b A c with every pairing (additive coupling conditions)
            res.append(sum(b[i] * A1[i][j] * sum(A2[j]) for i in range(s) for j in range(s)) - six)
    res += [sum(d) - 1, sum(d[i] * c[i] for i in range(s)) - (F(1, 2) if isinstance(b[0], F) else 0.5)]
    return [abs(float(r)) for r in res]


def test_published_tableau_order_conditions_exact():
    assert max(order_residuals(AE, AI, B, D, C)) <= 1e-24
    assert AI[0][0] == 0 and all(AI[i][i] == G for i in range(1, 4))   # ESDIRK, explicit 1st stage
    assert B == AI[3]                                                  # stiffly accurate


def test_oracle_tableau_is_the_published_one():
    ae, ai, b, d, c = oracle.ark_tableau()
    assert max(order_residuals(ae.tolist(), ai.tolist(), b.tolist(), d.tolist(), c.tolist())) <= 2e-15
    for i in range(4):
        assert b[i] == float(B[i]) and d[i] == float(D[i]) and c[i] == float(C[i])
        for j in range(4):
            assert ae[i, j] == float(AE[i][j]) and ai[i, j] == float(AI[i][j])


@pytest.mark.parametrize("lamE,lamI", [(0.0, -10.0), (-1.0, 0.0), (-1.0, -10.0)])
def test_third_order_convergence(lamE, lamI):
    errs = []
    for k in range(4):
        N = 20 * 2 ** k
        rc, y, st = oracle.ark_integrate(np.ones(3), 1.0, h0=1.0 / N, fixed=True, kind=1, nx=1,
                                         lam_E=lamE, lam_I=lamI, maxnl=4, tol_nl=1e-4)
        assert rc == 0 and st["accepted"] == N
        errs.append(abs(y[0] - math.exp(lamE + lamI)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(2.7 < o < 3.3 for o in orders), orders


def test_error_control_tracks_tolerance():
    y0 = np.ones(3)
    exact = math.exp(-11.0 * 2.0)
    errs, steps = [], []
    for rtol in (1e-4, 1e-6, 1e-8):
        rc, y, st = oracle.ark_integrate(y0, 2.0, h0=1e-3, kind=1, nx=1, lam_E=-1.0, lam_I=-10.0,
                                         rtol=rtol, atol=rtol * 1e-3, tol_nl=1e-3, maxnl=4)
        assert rc == 0
        errs.append(abs(y[0] - exact))                 # the solution decays below atol: absolute error
        steps.append(st["accepted"])
    assert steps[0] < steps[1] < steps[2]
    # tolerance proportionality: 100x tighter tolerances give >= 10x smaller errors
    assert errs[0] > 10 * errs[1] > 100 * errs[2]
    assert errs[0] <= 1e-4 * 1.0                       # within rtol · max|y|


def test_brusselator_adaptive_run_and_retries():
    nx = 64
    y0 = oracle.bruss_ic(nx)
    rc, y, st = oracle.ark_integrate(y0, 1.0, h0=1e-4, nx=nx, kx=0.01 * nx)
    assert rc == 0 and abs(st["t"] - 1.0) < 1e-12
    # stiff startup: the controller rejects or retries some steps, then grows h
    assert st["rejected_err"] + st["rejected_nl"] > 0 and st["h_last"] > 1e-3
    # agrees with a fully converged small-step SBDF2 reference to tolerance level
    _, yb, _, _ = oracle.sbdf_integrate(y0, 4000, kind=0, newton_mode=2, nx=nx, kx=0.01 * nx,
                                        h=2.5e-4)
    assert np.max(np.abs(y - yb) / np.abs(yb)) < 1e-4
    # a Newton budget of one iteration forces stage failures -> h/4 recomputation
    rc, y1, st1 = oracle.ark_integrate(y0, 0.01, h0=1e-3, nx=nx, kx=0.01 * nx, maxnl=1, tol_nl=1e-12,
                                       max_steps=50)
    assert st1["rejected_nl"] > 0
