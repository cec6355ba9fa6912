"""The NCCL communicator path on one GPU: unique id, ncclCommInitRank with
a single rank, and the partitioned reductions / driver running through it
(the multi-rank exchange logic itself is covered by the fake communicator,
NCCL forbids two ranks on one device)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bits_equal, needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda]


def test_nccl_single_rank_context(tmp_path):
    from paper_2011_12984_b200 import sunbw as S
    uid = S.nccl_unique_id()
    assert len(uid) == 128
    ctx = S.Context(0)
    ctx.init_nccl(uid, 0, 1)
    assert ctx.rank == 0 and ctx.nranks == 1
    n = 100_003
    x = synth.uniform(1, n, -1, 1, device="cuda")
    w = synth.uniform(3, n, 0.5, 1.5, device="cuda")
    vx, vw = S.NVector(ctx, x), S.NVector(ctx, w)
    assert vx.global_length() == n
    ref = oracle.wrms(x.cpu().numpy(), w.cpu().numpy())
    assert abs(S.N_VWrmsNorm(vx, vw) - ref) <= 1e-12 * ref
    # a short fused 3D run through the NCCL-backed context
    nx, ny, nz = 128, 4, 4
    y0 = oracle.bruss_ic(nx, ny, nz)
    _, yref, _, _ = oracle.sbdf_integrate(y0, 4, kind=0, K=3, nx=nx, ny=ny, nz=nz, kx=0.01 * nx,
                                          ky=0.01 * ny, kz=0.01 * nz, h=1e-3)
    P = S.Problem(ctx, S.bruss_params(dim=3, nx=nx, ny=ny, nz=nz))
    yd = torch.from_numpy(y0).cuda()
    yo = torch.empty_like(yd)
    st = S.Stepper(P, S.NVector(ctx, yd), S.stepper_options(h=1e-3, K=3, fused=True))
    rc, _ = st.advance(4, S.NVector(ctx, yo))
    assert rc == 0
    assert_bits_equal(yo, yref, "fused via NCCL context")
    st.destroy(); P.destroy(); ctx.destroy()
