"""C3 (128^3) adaptive ARK to t = 0.01: composed vs fused stages, device-timed
(the bench's other_configs rows, standalone for A/B runs)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2011_12984_b200 import sunbw as S  # noqa: E402

n = 128
ctx = S.Context(0)
P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
y = torch.empty(3 * n ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y))
out = {}
for fused in ([False, True] if "--composed" in sys.argv else [True]):
    A = S.Ark(P, S.NVector(ctx, y), h0=1e-4, max_steps=2000, fused=fused)
    A.evolve(0.001)
    A.destroy()
    A = S.Ark(P, S.NVector(ctx, y), h0=1e-4, max_steps=2000, fused=fused)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc, st = A.evolve(0.01)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["fused" if fused else "composed"] = {"ms": round(ms, 2), "accepted": st["accepted"],
                                             "attempts": st["accepted"] + st["rejected_err"] + st["rejected_nl"],
                                             "newton_iters": st["newton_iters"],
                                             "us_per_attempt": round(1e3 * ms / (st["accepted"] + st["rejected_err"] + st["rejected_nl"]), 1)}
    A.destroy()
print(json.dumps(out))
