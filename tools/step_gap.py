import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2011_12984_b200 import sunbw as S
torch.cuda.set_device(0)
ctx = S.Context(0)
n = 256
P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
y0 = torch.empty(3 * n**3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y0))
for timing, graph in [(True, False), (True, False), (False, False), (False, True), (True, True), (True, True)]:
    st = S.Stepper(P, S.NVector(ctx, y0), S.stepper_options(h=1e-3, K=3, use_graph=graph, timing=timing, fused=True))
    st.advance(10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st.advance(300); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 300
    kt = st.kernel_times(reset=True) if timing else {}
    print(f"timing={timing} graph={graph}: {ms*1e3:.1f} us/step", {k: round(v[0]/v[1]*1e3, 1) for k, v in kt.items()})
    st.destroy()
