"""The submodel multi-instance pattern (§6, fig:cvodestreams): k
independent integrator instances, each on its own CUDA stream over its own
group of cells, run concurrently from k host threads.  Reaction-only cells
are independent, so every cell's trajectory is bit-identical to the grouped
single-instance run (grouping invariance) and to the oracle."""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bits_equal, needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda]


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("fused", [False, True])
def test_instances_on_streams_match_grouped_run(k, fused):
    from paper_2011_12984_b200 import sunbw as S
    G, steps = 40_000, 10
    u = synth.uniform(synth.S_CELL, G, 0, 1).numpy()
    y0 = np.stack([1.0 + 0.1 * u, 3.5 + 0.1 * u, 3.0 + 0.1 * u], 1).reshape(-1)
    _, yref, _, _ = oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=G, reaction_only=True, h=1e-3)
    cuts = np.linspace(0, G, k + 1).astype(int)
    out, errs = [None] * k, []

    def body(i):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = S.Context(0, stream)
                g0, g1 = cuts[i], cuts[i + 1]
                P = S.Problem(ctx, S.bruss_params(dim=1, nx=int(g1 - g0), reaction_only=True))
                y = torch.from_numpy(y0[3 * g0:3 * g1].copy()).cuda()
                yo = torch.empty_like(y)
                st = S.Stepper(P, S.NVector(ctx, y), S.stepper_options(h=1e-3, K=3, fused=fused))
                rc, _ = st.advance(steps, S.NVector(ctx, yo))
                stream.synchronize()
                out[i] = (rc, yo.cpu().numpy())
                st.destroy(); P.destroy(); ctx.destroy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=body, args=(i,)) for i in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    assert all(o[0] == 0 for o in out)
    assert_bits_equal(np.concatenate([o[1] for o in out]), yref, f"{k} instances fused={fused}")
