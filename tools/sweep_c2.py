#!/usr/bin/env python
"""C2: the N_Vector op sweep (BASELINE.json configs[1]; the paper's E1,
P:222-251): each op on random fp64 data at lengths 1e3 .. 1e9 (half
decades), 50 timed calls after 5 warm-up calls, device-timed
with CUDA events around the public N_V* calls (reductions include their
host return, as the API defines).  GB/s from algorithmic bytes; rows whose
working set fits in L2 are labelled.  The serial oracle is timed beside
it on one host core up to 1e7 (the paper's GPU/serial crossover).

Writes one JSON object per line to stdout (and --out)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L2_BYTES = 126e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max", type=float, default=1e9)
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--ops", default=None, help="comma-separated subset of the op names")
    ap.add_argument("--min", type=float, default=1e3)
    args = ap.parse_args()

    import numpy as np
    import torch

    import synth
    from paper_2011_12984_b200 import sunbw as S

    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    ctx = S.Context(0)
    stream = torch.cuda.current_stream()
    lengths = [int(round(10 ** (3 + 0.5 * i))) for i in range(13)]
    lengths = [n for n in lengths if args.min <= n <= args.max]
    # (name, bytes per element, vectors needed, gpu call, oracle call)
    ops = ["LinearSum", "Scale", "Prod", "Div", "WrmsNorm", "DotProd", "LinearCombination8",
           "DotProdMulti8", "ScaleAddMulti8"]
    if args.ops:
        ops = [o for o in ops if o in args.ops.split(",")]
    bpe = {"LinearSum": 24, "Scale": 16, "Prod": 24, "Div": 24, "WrmsNorm": 16, "DotProd": 16,
           "LinearCombination8": 72, "DotProdMulti8": 72, "ScaleAddMulti8": 136}
    nvecs = {"LinearSum": 3, "Scale": 2, "Prod": 3, "Div": 3, "WrmsNorm": 2, "DotProd": 2,
             "LinearCombination8": 9, "DotProdMulti8": 9, "ScaleAddMulti8": 17}
    out = open(args.out, "w") if args.out else None
    free = torch.cuda.mem_get_info()[0]
    for n in lengths:
        maxv = max(nvecs[o] for o in ops if nvecs[o] * 8 * n < 0.8 * free)
        vecs = [synth.uniform(1 + j, n, -1.0, 1.0, device="cuda") if j != 1 else
                synth.uniform(2, n, 0.5, 1.5, device="cuda") for j in range(maxv)]
        hv = None
        if not args.no_oracle and n <= 1e7:
            hv = [v.cpu().numpy() for v in vecs[:17]]
        V = [S.NVector(ctx, t) for t in vecs]
        c8 = [(j + 1) / 8 for j in range(8)]
        a8 = [1 - j / 16 for j in range(8)]
        for op in ops:
            if nvecs[op] > maxv:
                continue
            x, y, z = V[0], V[1], V[2] if len(V) > 2 else None
            calls = {
                "LinearSum": lambda: S.N_VLinearSum(1.25, x, -0.75, y, z),
                "Scale": lambda: S.N_VScale(0.5, x, V[1]),
                "Prod": lambda: S.N_VProd(x, y, z),
                "Div": lambda: S.N_VDiv(x, y, z),
                "WrmsNorm": lambda: S.N_VWrmsNorm(x, y),
                "DotProd": lambda: S.N_VDotProd(x, y),
                "LinearCombination8": lambda: S.N_VLinearCombination(c8, V[1:9], x),
                "DotProdMulti8": lambda: S.N_VDotProdMulti(x, V[1:9]),
                "ScaleAddMulti8": lambda: S.N_VScaleAddMulti(a8, x, V[1:9], V[9:17]),
            }
            fn = calls[op]
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.reps
            gbs = bpe[op] * n / (us * 1e-6) / 1e9
            row = {"op": "N_V" + op, "n": n, "gpu_us": round(us, 2), "GB/s": round(gbs, 1),
                   "frac_of_peak": round(gbs / peak, 4), "l2_resident": bpe[op] * n < L2_BYTES}
            if hv is not None:
                import oracle
                O = {
                    "LinearSum": lambda: oracle.linear_sum(1.25, hv[0], -0.75, hv[1]),
                    "Scale": lambda: oracle.scale(0.5, hv[0]),
                    "Prod": lambda: oracle.prod(hv[0], hv[1]),
                    "Div": lambda: oracle.div(hv[0], hv[1]),
                    "WrmsNorm": lambda: oracle.wrms(hv[0], hv[1]),
                    "DotProd": lambda: oracle.dot(hv[0], hv[1]),
                    "LinearCombination8": lambda: oracle.linear_combination(c8, hv[1:9]),
                    "DotProdMulti8": lambda: oracle.dot_prod_multi(hv[0], hv[1:9]),
                    "ScaleAddMulti8": lambda: oracle.scale_add_multi(a8, hv[0], hv[1:9]),
                }
                reps = 50 if n <= 1e6 else 5
                t0 = time.perf_counter()
                for _ in range(reps):
                    O[op]()
                row["oracle_us_1core"] = round((time.perf_counter() - t0) * 1e6 / reps, 2)
                row["gpu_speedup"] = round(row["oracle_us_1core"] / us, 1)
            line = json.dumps(row)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
        del V, vecs
        torch.cuda.empty_cache()
    ctx.check("sweep")


if __name__ == "__main__":
    main()
