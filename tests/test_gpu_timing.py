"""Per-kernel timing of the stepper (BW_StepperOptions.timing): every kernel
(1), one pair per fused chain graph (1, graphs), every k-th step (k > 1,
eager steps — the N > 1 bench's mode)."""
import pytest
import torch

from gpu_util import needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda]


@pytest.mark.parametrize("timing,use_graph", [(1, False), (1, True), (5, False)])
def test_fused_step_kernel_times(timing, use_graph):
    from paper_2011_12984_b200 import sunbw as S
    ctx = S.Context(0)
    n = 128
    P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
    y = torch.empty(3 * n ** 3, dtype=torch.float64, device="cuda")
    S.BW_InitialCondition(P, S.NVector(ctx, y))
    st = S.Stepper(P, S.NVector(ctx, y), S.stepper_options(h=1e-3, K=3, use_graph=use_graph, timing=timing,
                                                            fused=True, numerics=1))
    warm, steps = 7, 24
    rc, _ = st.advance(warm)
    assert rc == 0
    st.kernel_times(reset=True)
    rc, _ = st.advance(steps)
    assert rc == 0
    kt = st.kernel_times(reset=True)
    ms, cnt = kt["fused_newton"]
    expect = steps if timing == 1 else len([s for s in range(warm, warm + steps) if s % timing == 0])
    assert cnt == expect, (cnt, expect)
    us = 1e3 * ms / cnt
    assert 5.0 < us < 500.0, us                     # a C3 step kernel: tens of microseconds
    st.destroy(); P.destroy(); ctx.destroy()
