"""Step time of the fused C5 step with and without the per-kernel timing
events in the step graphs (tools only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2011_12984_b200 import sunbw as S  # noqa: E402

ctx = S.Context(0)
P = S.Problem(ctx, S.bruss_params(dim=3, nx=256, ny=256, nz=256))
y0 = torch.empty(3 * 256 ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y0))
for timing in (True, False, True, False):
    st = S.Stepper(P, S.NVector(ctx, y0), S.stepper_options(h=1e-3, K=3, use_graph=True, timing=timing,
                                                            fused=True, numerics=1))
    st.advance(10)
    for steps in (20, 200):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.advance(steps)
        e1.record()
        torch.cuda.synchronize()
        print(f"timing={timing} steps={steps}: {1e3 * e0.elapsed_time(e1) / steps:.1f} us/step")
    st.destroy()
