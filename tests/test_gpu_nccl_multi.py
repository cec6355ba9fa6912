"""Two real NCCL ranks, one process per GPU (runs wherever >= 2 GPUs are
visible; skipped on a one-GPU box): a reduced C5 workload (z-slabs of
128 x 8 x 8 cells per rank, SBDF2 + K = 3, fused single-kernel step with the
halo over NVLink) through the C ABI, the gathered state bit-identical to the
one-rank oracle integration (exact numerics) or within 1e-9 (contracted).
Both halo mechanisms: the copy engine into the peer's IPC-mapped slot
(peer_halo.cu, default) and NCCL send/recv (SUNBW_PEER_HALO=0)."""
import os

import numpy as np
import pytest
import torch

import oracle
from gpu_util import needs_cuda

pytestmark = [pytest.mark.gpu, needs_cuda,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")]

NX, NY, NZL, STEPS = 128, 8, 8, 6


def _rank(rank, world, uid, numerics, peer, q):
    os.environ["SUNBW_PEER_HALO"] = peer
    import torch as T
    from paper_2011_12984_b200 import sunbw as S
    try:
        T.cuda.set_device(rank)
        ctx = S.Context(rank)
        ctx.init_nccl(uid, rank, world)
        nz = NZL * world
        y0 = oracle.bruss_ic(NX, NY, nz)
        P = S.Problem(ctx, S.bruss_params(dim=3, nx=NX, ny=NY, nz=nz))
        n, off = 3 * P.local_cells, 3 * P.cell_offset
        y = T.from_numpy(y0[off:off + n].copy()).cuda()
        yout = T.empty_like(y)
        st = S.Stepper(P, S.NVector(ctx, y), S.stepper_options(h=1e-3, K=3, use_graph=False, fused=True,
                                                                numerics=numerics))
        rc, stats = st.advance(STEPS, S.NVector(ctx, yout))
        T.cuda.synchronize()
        q.put((rank, rc, off, yout.cpu().numpy(), stats["last_nu"]))
        st.destroy(); P.destroy(); ctx.destroy()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None, None))


@pytest.mark.parametrize("peer", ["1", "0"])
@pytest.mark.parametrize("numerics", [0, 1])
def test_two_nccl_ranks_reduced_C5(numerics, peer):
    import torch.multiprocessing as mp
    from paper_2011_12984_b200 import sunbw as S
    world = 2
    uid = S.nccl_unique_id()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_rank, args=(r, world, uid, numerics, peer, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] == 0 for r in res), res
    nz = NZL * world
    y0 = oracle.bruss_ic(NX, NY, nz)
    k = (0.01 * NX, 0.01 * NY, 0.01 * nz)
    _, yref, stref, _ = oracle.sbdf_integrate(y0, STEPS, kind=0, K=3, nx=NX, ny=NY, nz=nz, kx=k[0], ky=k[1],
                                              kz=k[2], h=1e-3)
    y = np.concatenate([r[3] for r in sorted(res, key=lambda t: t[2])])
    if numerics == 0:
        assert np.array_equal(y.view(np.int64), yref.view(np.int64))
    else:
        assert float(np.max(np.abs(y - yref) / np.maximum(np.abs(yref), 1.0))) <= 1e-9
    assert res[0][4] == res[1][4]                     # same global nu on both ranks
