"""Timeline of the fused ARK on C3 (128^3) to t = 0.01 (tools only): CUPTI
(torch.profiler) kernel and memcpy records -> per kernel kind the count and
mean duration, and per attempt the GPU-busy time against the wall span
(host decision + launch bubbles between attempts)."""
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2011_12984_b200 import sunbw as S  # noqa: E402

n = int(os.environ.get("ARK_N", "128"))
t_end = float(os.environ.get("ARK_T", "0.01"))
ctx = S.Context(0)
P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
y = torch.empty(3 * n ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y))
A = S.Ark(P, S.NVector(ctx, y), h0=1e-4, max_steps=2000, fused=True)
A.evolve(0.001)
A.destroy()
A = S.Ark(P, S.NVector(ctx, y), h0=1e-4, max_steps=2000, fused=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rc, st = A.evolve(t_end)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)


def kind(name):
    m = re.search(r"k_ark_(tile|stage)<(\d+), (true|false)", name)
    if m:
        return ("final" if m.group(3) == "true" else f"stage{m.group(2)}") + f"_{m.group(1)}"
    if "Memcpy" in name or "memcpy" in name:
        return "memcpy"
    return re.sub(r"\(.*", "", name)[:60]


per = defaultdict(list)
for e in ev:
    per[kind(e.name)].append(e.time_range.end - e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
busy = sum(e.time_range.end - e.time_range.start for e in ev)
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    gaps.append((g, kind(a.name), kind(b.name)))
big = defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    key = f"{a} -> {b}"
    big[key][0] += 1
    big[key][1] += g
attempts = st["accepted"] + st["rejected_err"] + st["rejected_nl"]
out = {"t_end": t_end, "n": n, "stats": st, "attempts": attempts, "span_us": round(span, 1),
       "gpu_busy_us": round(busy, 1), "us_per_attempt": round(span / attempts, 1),
       "kernels": {k: {"count": len(v), "us_avg": round(sum(v) / len(v), 2), "us_total": round(sum(v), 1)}
                   for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))},
       "gaps": {k: {"count": c, "us_total": round(s, 1), "us_avg": round(s / c, 2)}
                for k, (c, s) in sorted(big.items(), key=lambda kv: -kv[1][1])[:12]}}
print(json.dumps(out, indent=1))
