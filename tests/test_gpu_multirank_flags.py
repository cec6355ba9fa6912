"""Rank-consistent recoverable failures ("if any one solve fails then
the entire time step is recomputed"): a zero pivot on ONE rank only must send
every rank down the same path — the tolerance-mode SBDF driver returns the
same code everywhere, the adaptive ARK driver recomputes the step with h/4
everywhere.  Without the flag allreduce the ranks' collectives stop pairing
up and the run hangs.  P = 2 logical ranks on one GPU (fake communicator).

Construction: the linear test problem (kind 1, f_I = λ_I y, J = λ_I I) with a
per-rank λ_I; on rank 1, λ_I = 1/γ rounded so that RN(γ λ_I) = 1 exactly,
hence M = I - γJ = 0 (every pivot zero) on every block of that rank only.
"""
import numpy as np
import pytest
import torch

from gpu_util import needs_cuda
from test_gpu_bruss import run_ranks

pytestmark = [pytest.mark.gpu, needs_cuda]

ARK_GAMMA = 1767732205903.0 / 4055673282236.0     # a^I_ii of ARK3(2)4L[2]SA


@pytest.fixture(scope="module")
def S():
    from paper_2011_12984_b200 import sunbw
    return sunbw


def exact_inverse(g):
    """λ with RN(g·λ) == 1.0 (so RN(-g·λ) + 1 == 0)."""
    lam = 1.0 / g
    for _ in range(8):
        if g * lam == 1.0:
            return lam
        lam = np.nextafter(lam, np.inf if g * lam < 1.0 else -np.inf)
    raise AssertionError("no exact inverse found")


def test_tolerance_mode_singular_on_one_rank(S):
    G, h = 96, 1e-3
    lam_bad = exact_inverse(h)            # SBDF1 first step: γ = h

    def fn(c, r):
        params = S.bruss_params(dim=1, nx=2 * G, kind=1, lam_E=0.0, lam_I=lam_bad if r == 1 else -10.0)
        P = S.Problem(c, params)
        y = torch.full((3 * P.local_cells,), 0.5, dtype=torch.float64, device="cuda")
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=h, K=4, newton_mode=1, use_graph=False))
        rc, stats = st.advance(3)
        c.stream.synchronize()
        st.destroy(); P.destroy()
        return rc, stats["steps"]

    res = run_ranks(S, 2, fn)
    assert res[0] == res[1], res
    assert res[0][0] == S.SUNBW_RECOV_SINGULAR and res[0][1] == 0


def test_ark_singular_on_one_rank_retries_everywhere(S):
    G, h0 = 96, 1e-3
    lam_bad = exact_inverse(h0 * ARK_GAMMA)   # first attempt's stage matrix is 0 on rank 1

    def fn(c, r):
        params = S.bruss_params(dim=1, nx=2 * G, kind=1, lam_E=-1.0, lam_I=lam_bad if r == 1 else -10.0)
        P = S.Problem(c, params)
        y = torch.full((3 * P.local_cells,), 0.5, dtype=torch.float64, device="cuda")
        A = S.Ark(P, S.NVector(c, y), h0=h0, fixed=True, maxnl=4, tol_nl=1e-4)
        rc, st = A.evolve(4 * h0)
        c.stream.synchronize()
        A.destroy(); P.destroy()
        return rc, st["accepted"], st["rejected_nl"], st["newton_iters"]

    res = run_ranks(S, 2, fn)
    assert res[0] == res[1], res
    rc, acc, rej, _ = res[0]
    assert rc == 0 and rej == 1 and acc >= 4
