"""Timeline evidence for the copy-engine halo: two in-process
ranks (fake communicator) on one GPU run the fused step on 256 x 256 x 64
z-slabs each; CUPTI (torch.profiler) records every kernel and copy with
device timestamps.  For each step the peer copy of the halo plane (1.57 MB,
copy engine) is matched with the interior kernel it must overlap; the JSON
line reports how many halo copies ran entirely inside an interior kernel.

usage: python tools/halo_overlap.py [steps] [planes]"""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import oracle  # noqa: E402
from paper_2011_12984_b200 import sunbw as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nzl = int(sys.argv[2]) if len(sys.argv) > 2 else 64
nranks, n = 2, 256
nz = nzl * nranks
params = S.bruss_params(dim=3, nx=n, ny=n, nz=nz)
comm = S.FakeComm(nranks)
out = [None] * nranks
ready = threading.Barrier(nranks)


def body(r):
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        c = S.Context(0, stream)
        c.set_fake_comm(comm, r)
        P = S.Problem(c, params)
        y = torch.empty(3 * P.local_cells, dtype=torch.float64, device="cuda")
        S.BW_InitialCondition(P, S.NVector(c, y))
        st = S.Stepper(P, S.NVector(c, y), S.stepper_options(h=1e-3, K=3, use_graph=False, fused=True,
                                                              numerics=1, timing=True))
        st.advance(3)
        st.kernel_times(reset=True)
        stream.synchronize()
        ready.wait()
        st.advance(steps)
        stream.synchronize()
        out[r] = st.kernel_times()
        st.destroy(); P.destroy(); c.destroy()


with profile(activities=[ProfilerActivity.CUDA]) as prof:
    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
comm.destroy()

evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = [(e.time_range.start, e.time_range.end, e.name) for e in evs if "k_fused_newton" in e.name]
copies = [(e.time_range.start, e.time_range.end, e.name) for e in evs
          if "Memcpy" in e.name or "memcpy" in e.name.lower()]
halo = [c for c in copies if "DtoD" in c[2] or "PtoP" in c[2] or "Device -> Device" in c[2]]
inside = 0
for (s0, e0, _) in halo:
    if any(ks <= s0 and e0 <= ke for (ks, ke, _) in kern):
        inside += 1
res = {"steps_per_rank": steps, "ranks": nranks, "slab": [n, n, nzl], "fused_kernels": len(kern),
       "halo_copies": len(halo), "halo_copies_inside_a_kernel": inside,
       "halo_copy_us_avg": round(sum(e - s for s, e, _ in halo) / max(1, len(halo)), 2),
       "kernel_us_avg": round(sum(e - s for s, e, _ in kern) / max(1, len(kern)), 2),
       "stepper_kernel_times_rank0": {k: [round(v[0], 3), v[1]] for k, v in out[0].items()},
       "copy_names": sorted({c[2] for c in copies})[:6]}
print(json.dumps(res))
