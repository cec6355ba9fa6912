"""Diagnostic: how many cells of a C5 fused step take the exact (IEEE
division / pivoting) path.  Needs the SUNBW_FUSED_COUNT_EXACT=1 variant:
  python tools/build_variant.py var_cnt SUNBW_FUSED_COUNT_EXACT=1
  SUNBW_LIB=build/var_cnt/libsunbw.so python tools/count_exact.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_12984_b200 import sunbw as S  # noqa: E402

lib = S.lib()
f = lib.SUNBW_DebugExactCells
f.restype = ctypes.c_longlong
f.argtypes = [ctypes.c_int]
ctx = S.Context(0)
n = 256
P = S.Problem(ctx, S.bruss_params(dim=3, nx=n, ny=n, nz=n))
y0 = torch.empty(3 * n ** 3, dtype=torch.float64, device="cuda")
S.BW_InitialCondition(P, S.NVector(ctx, y0))
yout = torch.empty_like(y0)
st = S.Stepper(P, S.NVector(ctx, y0), S.stepper_options(h=1e-3, K=3, fused=True))
f(1)
for rep in range(4):
    rc, stats = st.advance(10, S.NVector(ctx, yout))
    print(f"advance {rep}: rc={rc} exact-path cells in 10 steps: {f(1)} of {10 * n ** 3}", flush=True)
