#!/usr/bin/env python
"""bench.py — advection–reaction time-stepping throughput on B200 (and the
N_Vector op bandwidths of the C2 sweep point), one JSON line on rank 0.

Workload (BASELINE.json configs[4], the weak-scaling config; at N = 1 it is
one GPU's slab): 3D Brusselator advection–reaction (DESIGN R19),
256^3 cells per GPU, z-slab partitioned, fp64, SBDF2 + modified Newton with
K = 3 block-LU iterations per step (DESIGN R14/R15), h = 1e-3.  A "step" is
one time step of the whole hot path: halo exchange, advection, the SBDF
right-hand side, error weights, Jacobian + M = I - γJ + LU, K × (reaction,
residual, block solve, update, WRMS) — fused per cell in one kernel
(--mode fused, default) or through the N_Vector/solver kernels one by one
(--mode composed).

Launch: python bench.py --gpus N --steps K --warmup W
        (N > 1 under torchrun: one rank per GPU, NCCL).
--impl reference: the serial CPU oracle (oracle/), as it stands, on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic HBM bytes per cell per launch, per kernel (DESIGN.md §6,
# SURVEY §8(d)); the fused Newton kernel reads y_n and the SBDF2 history H_n
# and writes y_{n+1} and H_{n+1} (R28; y_n's row/plane neighbours for the
# in-kernel advection are L2 hits, not counted)
BYTES_PER_CELL = {
    "advection": 48, "rhs_combine": 120, "ewt": 216, "predict": 48, "jacobian": 96,
    "scaleaddi": 144, "lu_setup": 148, "reaction": 48, "residual": 96, "lu_solve": 124,
    "update": 72, "wrms": 48, "fused_newton": 96, "halo": 0,
}
WRMS_FUSED_BYTES = 0        # the fused path's fold reads only per-CTA partials
NUM_SMS = 148
FP64_LANES_PER_SM = 64
FP64_SUSTAINED_TOPS = 12.3          # T fp64 op/s sustained by DFMA chains in the fused grid structure (r01i)


def sm_max_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("sm_max_mhz", 1965.0))
    except (OSError, ValueError):
        return 1965.0


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ distributed
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    return world, rank, local


def slab(rank: int, world: int, n_ax: int):
    """z-slab of rank `rank` in the weak-scaled C5 grid (n_ax^2 x n_ax*world):
    (first global plane, local planes, domain length Lz) — MPIPlusX layout."""
    return rank * n_ax, n_ax, float(world)


def broadcast_uid(uid, rank: int, dist):
    """NCCL unique id from rank 0 to every rank through the torch store."""
    box = [uid if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def max_over_ranks(ms: float, dist, world: int, device) -> float:
    """The job time is the slowest rank's (device-timed) time."""
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_reference(args, world, rank):
    """The serial CPU oracle, as it stands, on a bounded sample of the same
    workload: a 256 x 256 x nzs slab (periodic), same parameters, fixed K."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    nx = ny = 256
    nzs = args.ref_planes
    L = 1.0
    k = 0.01 / (L / nx)
    y0 = oracle.bruss_ic(nx, ny, nzs, L, L, L * nzs / 256)
    kw = dict(kind=0, K=3, nx=nx, ny=ny, nz=nzs, kx=k, ky=k, kz=k, h=1e-3)
    if args.warmup:
        oracle.sbdf_integrate(y0, args.warmup, **kw)
    t0 = time.perf_counter()
    rc, _, _, _ = oracle.sbdf_integrate(y0, args.steps, **kw)
    dt = time.perf_counter() - t0
    cells = nx * ny * nzs
    v = cells * args.steps / dt
    sample = f"{nx}x{ny}x{nzs} cells (1/{256 // nzs} of a 256^3 slab), {args.steps} SBDF2 steps, K=3"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "cell-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (paper IC, P:376-382)",
        "config": workload_config(world, "oracle (serial CPU, bounded sample: see cpu_baseline)"),
        "cpu_baseline": {"value": v, "unit": "cell-steps/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "cell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "rc": rc,
    }), flush=True)


METRIC = ("advection-reaction throughput, cell time-steps/s (3D Brusselator, 256^3 cells/GPU, "
          "SBDF2 + K=3 block-LU Newton, fp64)")


def workload_config(world, mode, n_ax=256, numerics=None):
    """The `config` object of both arms (BASELINE configs[4], one slab per GPU)."""
    return {"workload": "C5: 3D Brusselator advection-reaction, 256^3 cells per GPU "
                        "(configs[4]; N=1 is one slab)",
            "cells_per_gpu": n_ax ** 3, "global_grid": [n_ax, n_ax, n_ax * world],
            "K": 3, "h": 1e-3, "mode": mode, "numerics": numerics, "parallelism": f"z-slab x{world}",
            "l2": "inputs larger than L2 (state 403 MB per vector)"}


def cpu_baseline_sample(planes=64, steps=15):
    """Oracle on the GPU box's host, one core, bounded sample (~10 s)."""
    import oracle
    oracle.build()
    nx = ny = 256
    k = 0.01 * nx
    y0 = oracle.bruss_ic(nx, ny, planes, 1.0, 1.0, planes / 256)
    t0 = time.perf_counter()
    oracle.sbdf_integrate(y0, steps, kind=0, K=3, nx=nx, ny=ny, nz=planes, kx=k, ky=k, kz=k, h=1e-3)
    dt = time.perf_counter() - t0
    return {"value": nx * ny * planes * steps / dt, "unit": "cell-steps/s", "cores": 1,
            "kind": "oracle",
            "sample": f"256x256x{planes} cells, {steps} SBDF steps (K=3), 1 host thread, {dt:.1f} s"}


def nvector_ops(S, ctx, torch, peak, n=100_000_000, reps=20):
    """C2 sweep point at n = 1e8 through the public N_V* calls (inputs
    800 MB each, > L2).  Reductions include their host return."""
    import synth
    out = {}
    dev = "cuda"
    x = synth.uniform(1, n, -1, 1, device=dev)
    y = synth.uniform(2, n, -1, 1, device=dev)
    w = synth.uniform(3, n, 0.5, 1.5, device=dev)
    z = torch.empty_like(x)
    X = [synth.uniform(32 + j, n, -1, 1, device=dev) for j in range(8)]
    vx, vy, vw, vz = (S.NVector(ctx, t) for t in (x, y, w, z))
    vX = [S.NVector(ctx, t) for t in X]
    c = [(j + 1) / 8 for j in range(8)]
    ops = {
        "N_VLinearSum": (lambda: S.N_VLinearSum(1.25, vx, -0.75, vy, vz), 24),
        "N_VScale": (lambda: S.N_VScale(0.5, vx, vz), 16),
        "N_VProd": (lambda: S.N_VProd(vx, vy, vz), 24),
        "N_VWrmsNorm": (lambda: S.N_VWrmsNorm(vx, vw), 16),
        "N_VDotProd": (lambda: S.N_VDotProd(vx, vy), 16),
        "N_VLinearCombination_8": (lambda: S.N_VLinearCombination(c, vX, vz), 72),
        "N_VDotProdMulti_8": (lambda: S.N_VDotProdMulti(vx, vX), 72),
    }
    stream = torch.cuda.current_stream()
    for name, (fn, bpe) in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = bpe * n / (ms * 1e-3) / 1e9
        out[name] = {"us": round(ms * 1e3, 1), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)}
    ctx.check("nvector ops")
    del X, vX
    return out


def other_configs(S, ctx, torch):
    """The other BASELINE.json configs, measured briefly on this GPU (fixed
    K = 3, h = 1e-3, device-timed with CUDA events):
      C1: 1D Brusselator, 64 cells, t in [0, 1] (1000 steps) — launch-bound:
          composed step replayed from CUDA graphs, the fused step one launch
          per step (graph replay), and the fused multi-step kernel (the whole
          Advance in one launch);
      C3: 3D, 128^3 cells, fused single-kernel step (graph replay);
      C4: 1e7 independent reaction cells (batched block Newton only): fused
          steps, and one composed Newton iteration (f_I, residual LC, block
          solve, update, WRMS) with its algorithmic bytes (388 B/cell)."""
    out = {}
    stream = torch.cuda.current_stream()

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def stepper_rate(params, G, steps, **opt):
        P = S.Problem(ctx, params)
        y0 = torch.empty(3 * G, dtype=torch.float64, device="cuda")
        vy = S.NVector(ctx, y0)
        S.BW_InitialCondition(P, vy)
        st = S.Stepper(P, vy, S.stepper_options(h=1e-3, K=3, **opt))
        st.advance(5)                                   # warm-up, graph capture
        ms = timed(lambda: st.advance(steps))
        st.destroy(); P.destroy()
        return steps / (ms * 1e-3)

    c1 = S.bruss_params(dim=1, nx=64)
    out["C1_1D_64cells"] = {
        "composed_graph_steps_per_s": round(stepper_rate(c1, 64, 1000, use_graph=True), 1),
        "fused_steps_per_s": round(stepper_rate(c1, 64, 1000, use_graph=True, fused=True), 1),
        "fused_one_launch_per_step_graph_steps_per_s": round(
            stepper_rate(c1, 64, 1000, use_graph=True, fused=True, single_step_launches=True), 1),
        "note": "fused: the whole Advance in one launch with the state on chip (<= 512 cells)"}
    # the paper's own task-local block solve (symbolic Gauss-Jordan inverse,
    # P:389-390, DESIGN R29) in the fused step at the bench workload (C5 slab)
    c5 = S.bruss_params(dim=3, nx=256, ny=256, nz=256)
    r5 = stepper_rate(c5, 256 ** 3, 100, use_graph=True, fused=True, linsol=2)
    out["C5_block_inverse_GJ"] = {"fused_steps_per_s": round(r5, 1), "cell_steps_per_s": r5 * 256 ** 3,
                                  "note": "linsol=2: block inverse by symbolic Gauss-Jordan (ablation; "
                                          "the headline uses the LU solve)"}
    c3 = S.bruss_params(dim=3, nx=128, ny=128, nz=128)
    r3 = stepper_rate(c3, 128 ** 3, 200, use_graph=True, fused=True)
    out["C3_3D_128cubed"] = {"fused_steps_per_s": round(r3, 1), "cell_steps_per_s": r3 * 128 ** 3}
    # the paper's integrator (adaptive IMEX ARK3(2)4L[2]SA, f2; composed
    # kernels, host step-size decisions) on C3 to t = 0.01
    P = S.Problem(ctx, c3)
    y3 = torch.empty(3 * 128 ** 3, dtype=torch.float64, device="cuda")
    S.BW_InitialCondition(P, S.NVector(ctx, y3))
    A = S.Ark(P, S.NVector(ctx, y3), h0=1e-4, max_steps=2000)
    ms = timed(lambda: A.evolve(0.01))
    _, ast = A.evolve(0.01)                      # already at t_end: stats of the run
    A.destroy(); P.destroy()
    out["C3_adaptive_ARK"] = {"t_end": 0.01, "accepted_steps": ast["accepted"],
                              "rejected_steps": ast["rejected_err"] + ast["rejected_nl"],
                              "newton_iters": ast["newton_iters"], "ms": round(ms, 2),
                              "steps_per_s": round(ast["accepted"] / (ms * 1e-3), 1)}
    G4 = 10_000_000
    c4 = S.bruss_params(dim=1, nx=G4, reaction_only=True)
    r4 = stepper_rate(c4, G4, 100, use_graph=True, fused=True)
    # one composed Newton iteration on 1e7 cells through the public calls
    P = S.Problem(ctx, c4)
    z = torch.empty(3 * G4, dtype=torch.float64, device="cuda")
    S.BW_InitialCondition(P, S.NVector(ctx, z))
    d, fI, r, dl = (torch.empty_like(z) for _ in range(4))
    ewt = torch.full_like(z, 1e6)
    Md = torch.empty(G4, 3, 3, dtype=torch.float64, device="cuda")
    vz, vd, vf, vr, vdl, vw = (S.NVector(ctx, t) for t in (z, d, fI, r, dl, ewt))
    M = S.SUNMatrix(ctx, Md)
    S.BW_ReactionJacobian(P, vz, M)
    S.SUNMatScaleAddI(-2e-3 / 3, M)
    LS = S.SUNLinearSolver(vz, M)
    S.SUNLinSolSetup(LS, M)
    d.copy_(z)
    c3 = [1.0, 2e-3 / 3, -1.0]

    def newton_iter():
        S.BW_ReactionRHS(P, vz, vf)
        S.N_VLinearCombination(c3, [vd, vf, vz], vr)
        S.SUNLinSolSolve(LS, M, vdl, vr)
        S.N_VLinearSum(1.0, vz, 1.0, vdl, vz)
        S.N_VWrmsNorm(vdl, vw)

    newton_iter()
    reps = 20
    ms = timed(lambda: [newton_iter() for _ in range(reps)]) / reps
    out["C4_1e7_reaction_cells"] = {
        "fused_steps_per_s": round(r4, 1), "cell_steps_per_s": r4 * G4,
        "composed_newton_iter_us": round(ms * 1e3, 1),
        "composed_newton_iter_GB/s": round(388 * G4 / (ms * 1e-3) / 1e9, 1)}
    del LS, M
    P.destroy()
    ctx.check("other configs")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="sunbw", choices=["sunbw", "reference"])
    ap.add_argument("--mode", default="fused", choices=["fused", "composed"])
    ap.add_argument("--cells", type=int, default=256, help="cells per axis per GPU slab")
    ap.add_argument("--numerics", default="contracted", choices=["contracted", "exact"],
                    help="fused cell step: FMA-contracted (rel 1e-9 parity, DESIGN R30) or the "
                         "bit-exact RN sequence")
    ap.add_argument("--no-ops", action="store_true", help="skip the C2 N_Vector op point")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    ap.add_argument("--ref-planes", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "sunbw":
        args.warmup = 3

    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2011_12984_b200 import sunbw as S

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = S.Context(local)
    if world > 1:
        uid = broadcast_uid(S.nccl_unique_id() if rank == 0 else None, rank, dist)
        ctx.init_nccl(uid, rank, world)

    n_ax = args.cells
    G = n_ax ** 3
    z0, nzl, Lz = slab(rank, world, n_ax)
    params = S.bruss_params(dim=3, nx=n_ax, ny=n_ax, nz=n_ax * world, Lx=1.0, Ly=1.0, Lz=Lz)
    P = S.Problem(ctx, params)
    assert P.local_cells == G
    y0 = torch.empty(3 * G, dtype=torch.float64, device="cuda")
    vy0 = S.NVector(ctx, y0)
    S.BW_InitialCondition(P, vy0)
    yout = torch.empty_like(y0)
    vyout = S.NVector(ctx, yout)
    fused = args.mode == "fused"
    # graph replay of the step at N = 1; eager launches when NCCL is in the
    # step (halo on a side stream), which is not exercised under capture here
    numerics = 1 if (fused and args.numerics == "contracted") else 0
    st = S.Stepper(P, vy0, S.stepper_options(h=1e-3, K=3, use_graph=world == 1, timing=True, fused=fused,
                                             numerics=numerics))
    rc, _ = st.advance(args.warmup)
    assert rc == 0, rc
    st.kernel_times(reset=True)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rc, stats = st.advance(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = ctx.launches - l0
    assert rc == 0, rc
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local, dist, world, "cuda")
    value = world * G * args.steps / (ms * 1e-3)

    # per-kernel device times inside the timed region (CUDA events on the
    # context stream) -> roofline of the dominant kernel
    peak, peak_kind = measured_peak()
    kt = st.kernel_times(reset=True)
    kernels = {}
    for name, (kms, cnt) in kt.items():
        bpc = BYTES_PER_CELL.get(name, 0)
        if fused and name == "wrms":
            bpc = WRMS_FUSED_BYTES
        avg = kms / cnt
        ach = bpc * G / (avg * 1e-3) / 1e9 if bpc else 0.0
        kernels[name] = {"ms_total": round(kms, 3), "launches": cnt, "us_avg": round(avg * 1e3, 2),
                         "share": round(kms / ms_local, 4), "GB/s": round(ach, 1)}
    dom = max(kernels, key=lambda k: kernels[k]["ms_total"] if BYTES_PER_CELL.get(k) else -1)
    ach = kernels[dom]["GB/s"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if n_ax == 256 and os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(dom)        # ncu dram read+write per launch, same workload
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "kernel": dom,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, this workload)",
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                else "fallback (B200_PROFILING.md)",
                "bytes_per_launch": BYTES_PER_CELL[dom] * G}
    if fused and n_ax == 256 and os.path.exists(tpath):
        # the fused step is as much an fp64-ALU kernel as an HBM one
        # (DESIGN.md §6): its fp64-pipe instructions per cell (ncu, same
        # workload) against 148 SMs x 64 FP64 lanes x the max SM clock
        with open(tpath) as f:
            ops = json.load(f).get("fused_newton_fp64_per_cell")
        if ops:
            a64 = ops * G / (kernels[dom]["us_avg"] * 1e-6) / 1e12
            p64 = FP64_LANES_PER_SM * NUM_SMS * sm_max_mhz() * 1e6 / 1e12
            roofline["fp64"] = {"achieved": round(a64, 2), "peak": round(p64, 2), "unit": "Top/s",
                                "frac": round(a64 / p64, 4), "ops_per_cell": ops,
                                "peak_source": "148 SMs x 64 FP64 lanes/clk (profiles/r01d_fp64_latency.txt: "
                                               "0.49 fp64 warp-instr/clk/SMSP) x sm_max_mhz",
                                # context: what independent DFMA chains sustain in the
                                # same grid/tile/TMA structure (DESIGN §6 calibration)
                                "sustained": FP64_SUSTAINED_TOPS,
                                "frac_of_sustained": round(a64 / FP64_SUSTAINED_TOPS, 4),
                                "sustained_source": "profiles/r01i_tile_streams.txt "
                                                    "(tools/microbench/tile_streams.cu, 3 x 256 DFMA/cell)"}
    # bytes per step of this mode; the composed path's are SURVEY §8(d)'s
    # 820 + 388 K per cell, the fused step's 96 per cell (R28)
    step_bytes = sum(BYTES_PER_CELL[k] * G * v["launches"] for k, v in kernels.items()
                     if BYTES_PER_CELL.get(k)) / args.steps
    if fused:
        step_bytes = BYTES_PER_CELL["fused_newton"] * G

    # e2e through the public API with host buffers: pinned H2D of the initial
    # state, Advance(K), D2H of the final state (per-step bytes = state/K)
    host_in = y0.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    ydev = torch.empty_like(y0)
    vydev = S.NVector(ctx, ydev)
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    ydev.copy_(host_in, non_blocking=True)
    st.reset(vydev, 0.0)
    rc2, _ = st.advance(args.steps, vyout)
    host_out.copy_(yout, non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), dist, world, "cuda")
    state_bytes = 3 * G * 8
    e2e = {"value": world * G * args.steps / (e2e_ms * 1e-3), "unit": "cell-steps/s",
           "h2d_bytes_per_step": state_bytes / args.steps, "d2h_bytes_per_step": state_bytes / args.steps,
           "note": "pinned H2D of y0 + Advance(K) + D2H of y_K through the C ABI, timed with CUDA events"}

    ops = None
    if rank == 0 and world == 1 and not args.no_ops:
        st.destroy()
        P.destroy()
        del y0, yout, ydev
        torch.cuda.empty_cache()
        ops = nvector_ops(S, ctx, torch, peak)
    configs = None
    if rank == 0 and world == 1 and not args.no_ops:
        torch.cuda.empty_cache()
        configs = other_configs(S, ctx, torch)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "steps_per_s": args.steps / (ms * 1e-3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (paper's Gaussian IC, P:376-382, on the 3D grid)",
            "config": workload_config(world, args.mode, n_ax, args.numerics if fused else "exact"),
            "roofline": roofline, "step_bytes": step_bytes, "composed_equiv_bytes_per_step": (820 + 388 * 3) * G,
            "step_GB/s": round(step_bytes / (ms / args.steps * 1e-3) / 1e9, 1),
            "kernels": kernels, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "cpu_baseline": cpu, "nvector_ops_1e8": ops, "other_configs": configs,
            "newton_iters": stats["newton_iters"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
