"""Kernel-to-kernel gaps of the graph-replayed fused C5 step with and without
the per-kernel timing events (CUPTI via torch.profiler; tools only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
from paper_2011_12984_b200 import sunbw as S  # noqa: E402

ctx = S.Context(0)
P = S.Problem(ctx, S.bruss_params(dim=3, nx=256, ny=256, nz=256))
y0 = torch.empty(3 * 256 ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y0))
for timing in (True, False):
    st = S.Stepper(P, S.NVector(ctx, y0), S.stepper_options(h=1e-3, K=3, use_graph=True, timing=timing,
                                                            fused=True, numerics=1))
    st.advance(10)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        st.advance(24)
        torch.cuda.synchronize()
    ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                 and "fused_newton" in e.name), key=lambda e: e.time_range.start)
    dur = [e.time_range.end - e.time_range.start for e in ev]
    gaps = [b.time_range.start - a.time_range.end for a, b in zip(ev, ev[1:])]
    print(f"timing={timing}: {len(ev)} kernels, mean {sum(dur) / len(dur):.1f} us, gaps "
          f"mean {sum(gaps) / len(gaps):.2f} us, min {min(gaps):.2f}, max {max(gaps):.2f}")
    st.destroy()
