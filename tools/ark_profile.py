"""Fused ARK on C3 (128^3) for a short interval: the workload for ncu launch
lists / kernel captures of the ARK stage kernels (tools only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2011_12984_b200 import sunbw as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
ctx = S.Context(0)
P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
y = torch.empty(3 * n ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y))
A = S.Ark(P, S.NVector(ctx, y), h0=1e-4, max_steps=2000, fused=True)
rc, st = A.evolve(t_end)
torch.cuda.synchronize()
print(rc, st)
A.destroy(); P.destroy(); ctx.destroy()
