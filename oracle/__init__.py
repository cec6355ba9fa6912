"""Serial CPU oracle for the sunbw hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2011_12984_b200`` never imports it, and the two share
no code (the only module both sides use is ``synth``, the seeded input
generator, which holds none of the method's arithmetic).

The arithmetic lives in ``oracle.cpp`` (plain C++17, single thread, compiled
with ``-ffp-contract=off -fno-fast-math``); this module is ctypes marshalling
over numpy arrays.  Each function cites the passage it follows in
``oracle.cpp``.  Parity status per function is in DESIGN.md §4; every
function is pinned — the nonlinear Brusselator trajectory, for which the
paper prints no values, against an independent Radau IIA integration of
the semi-discrete equations (tests/test_oracle_bruss.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++), if missing or stale."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", *CXXFLAGS, "-o", _LIB, _SRC])
    return _LIB


_lib = None
_D = C.c_double
_I64 = C.c_int64
_P = C.c_void_p


class SbdfParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("newton_mode", C.c_int32), ("K", C.c_int32),
                ("reaction_only", C.c_int32),
                ("nx", _I64), ("ny", _I64), ("nz", _I64),
                ("kx", _D), ("ky", _D), ("kz", _D),
                ("A", _D), ("B", _D), ("eps", _D),
                ("lam_E", _D), ("lam_I", _D),
                ("h", _D), ("rtol", _D), ("atol", _D), ("tol_nl", _D),
                ("linsol", C.c_int32), ("maxl", C.c_int32), ("lin_tol", _D)]


class SbdfStats(C.Structure):
    _fields_ = [("steps", _I64), ("newton_iters", _I64), ("setups", _I64),
                ("solves", _I64), ("fails", _I64), ("singular", _I64),
                ("last_nu", _D), ("lin_iters", _I64)]


class ArkParams(C.Structure):
    _fields_ = [("prob", SbdfParams), ("h0", _D), ("t_end", _D), ("maxnl", C.c_int32),
                ("max_steps", C.c_int32), ("fixed", C.c_int32), ("pad_", C.c_int32)]


class ArkStats(C.Structure):
    _fields_ = [("accepted", _I64), ("rejected_err", _I64), ("rejected_nl", _I64),
                ("newton_iters", _I64), ("setups", _I64), ("t", _D), ("h_last", _D)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        sig = {
            "oracle_linear_sum": (None, [_I64, _D, _P, _D, _P, _P]),
            "oracle_scale": (None, [_I64, _D, _P, _P]),
            "oracle_prod": (None, [_I64, _P, _P, _P]),
            "oracle_div": (None, [_I64, _P, _P, _P]),
            "oracle_const": (None, [_I64, _D, _P]),
            "oracle_abs": (None, [_I64, _P, _P]),
            "oracle_inv": (None, [_I64, _P, _P]),
            "oracle_add_const": (None, [_I64, _P, _D, _P]),
            "oracle_dot": (_D, [_I64, _P, _P]),
            "oracle_wsqrsum": (_D, [_I64, _P, _P]),
            "oracle_wsqrsum_mask": (_D, [_I64, _P, _P, _P]),
            "oracle_wrms": (_D, [_I64, _P, _P]),
            "oracle_wrms_mask": (_D, [_I64, _P, _P, _P]),
            "oracle_max_norm": (_D, [_I64, _P]),
            "oracle_min": (_D, [_I64, _P]),
            "oracle_linear_combination": (None, [C.c_int, _P, _P, _I64, _P]),
            "oracle_scale_add_multi": (None, [C.c_int, _P, _P, _P, _P, _I64]),
            "oracle_dot_prod_multi": (None, [C.c_int, _P, _P, _I64, _P]),
            "oracle_scale_add_identity": (None, [_I64, C.c_int, _D, _P]),
            "oracle_lu_factor": (_I64, [_I64, C.c_int, _P, _P]),
            "oracle_gj_inverse": (_I64, [_I64, C.c_int, _P, _P]),
            "oracle_gj_apply": (None, [_I64, C.c_int, _P, _P, _P]),
            "oracle_lu_solve": (None, [_I64, C.c_int, _P, _P, _P, _P]),
            "oracle_block_matvec": (None, [_I64, C.c_int, _P, _P, _P]),
            "oracle_bruss_reaction": (None, [_I64, _P, _D, _D, _D, _P]),
            "oracle_bruss_jacobian": (None, [_I64, _P, _D, _P]),
            "oracle_advection": (None, [_I64, _I64, _I64, _D, _D, _D, _P, _P]),
            "oracle_bruss_ic": (None, [_I64, _I64, _I64, _D, _D, _D, _D, _D, _D, _P]),
            "oracle_sbdf_integrate": (C.c_int, [C.POINTER(SbdfParams), _P, _I64,
                                                C.POINTER(SbdfStats), _P, _I64]),
            "oracle_gmres": (C.c_int, [_I64, C.c_int, _P, _P, _P, _P, _P, C.c_int, _D,
                                       C.POINTER(_D)]),
            "oracle_ark_tableau": (None, [_P, _P, _P, _P, _P]),
            "oracle_ark_integrate": (C.c_int, [C.POINTER(ArkParams), _P, C.POINTER(ArkStats)]),
            "oracle_abi_version": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# ---------------------------------------------------------------- helpers
def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _ptr_array(arrs):
    arr = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return arr


# ---------------------------------------------------------- O1 streaming
def linear_sum(a, x, b, y):
    x, y = _f64(x), _f64(y)
    z = np.empty_like(x)
    lib().oracle_linear_sum(x.size, a, _ptr(x), b, _ptr(y), _ptr(z))
    return z


def scale(c, x):
    x = _f64(x); z = np.empty_like(x)
    lib().oracle_scale(x.size, c, _ptr(x), _ptr(z)); return z


def prod(x, y):
    x, y = _f64(x), _f64(y); z = np.empty_like(x)
    lib().oracle_prod(x.size, _ptr(x), _ptr(y), _ptr(z)); return z


def div(x, y):
    x, y = _f64(x), _f64(y); z = np.empty_like(x)
    lib().oracle_div(x.size, _ptr(x), _ptr(y), _ptr(z)); return z


def const(c, n):
    z = np.empty(n, dtype=np.float64)
    lib().oracle_const(n, c, _ptr(z)); return z


def abs_(x):
    x = _f64(x); z = np.empty_like(x)
    lib().oracle_abs(x.size, _ptr(x), _ptr(z)); return z


def inv(x):
    x = _f64(x); z = np.empty_like(x)
    lib().oracle_inv(x.size, _ptr(x), _ptr(z)); return z


def add_const(x, b):
    x = _f64(x); z = np.empty_like(x)
    lib().oracle_add_const(x.size, _ptr(x), b, _ptr(z)); return z


# --------------------------------------------------------- O2 reductions
def dot(x, y):
    x, y = _f64(x), _f64(y)
    return lib().oracle_dot(x.size, _ptr(x), _ptr(y))


def wsqrsum(x, w):
    x, w = _f64(x), _f64(w)
    return lib().oracle_wsqrsum(x.size, _ptr(x), _ptr(w))


def wsqrsum_mask(x, w, idv):
    x, w, idv = _f64(x), _f64(w), _f64(idv)
    return lib().oracle_wsqrsum_mask(x.size, _ptr(x), _ptr(w), _ptr(idv))


def wrms(x, w):
    x, w = _f64(x), _f64(w)
    return lib().oracle_wrms(x.size, _ptr(x), _ptr(w))


def wrms_mask(x, w, idv):
    x, w, idv = _f64(x), _f64(w), _f64(idv)
    return lib().oracle_wrms_mask(x.size, _ptr(x), _ptr(w), _ptr(idv))


def max_norm(x):
    x = _f64(x); return lib().oracle_max_norm(x.size, _ptr(x))


def min_(x):
    x = _f64(x); return lib().oracle_min(x.size, _ptr(x))


# ------------------------------------------------------------- O3 fused
def linear_combination(c, X):
    X = [_f64(v) for v in X]
    c = _f64(c)
    z = np.empty_like(X[0])
    lib().oracle_linear_combination(len(X), _ptr(c), _ptr_array(X), X[0].size, _ptr(z))
    return z


def scale_add_multi(a, x, Y):
    x = _f64(x); Y = [_f64(v) for v in Y]; a = _f64(a)
    Z = [np.empty_like(x) for _ in Y]
    lib().oracle_scale_add_multi(len(Y), _ptr(a), _ptr(x), _ptr_array(Y), _ptr_array(Z), x.size)
    return Z


def dot_prod_multi(x, Y):
    x = _f64(x); Y = [_f64(v) for v in Y]
    d = np.empty(len(Y))
    lib().oracle_dot_prod_multi(len(Y), _ptr(x), _ptr_array(Y), x.size, _ptr(d))
    return d


# ------------------------------------------------------- block diagonal
def scale_add_identity(c, A):
    """A: (G, m, m) -> c*A + I per block (new array)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    G, m, _ = A.shape
    lib().oracle_scale_add_identity(G, m, c, _ptr(A))
    return A


def lu_factor(A):
    """Returns (LU (G,m,m), piv (G,m) int32 LAPACK-style 0-based rows, flag)."""
    LU = np.array(A, dtype=np.float64, order="C", copy=True)
    G, m, _ = LU.shape
    piv = np.zeros((G, m), dtype=np.int32)
    flag = lib().oracle_lu_factor(G, m, _ptr(LU), _ptr(piv))
    return LU, piv, int(flag)


def gj_inverse(A):
    """Block inverses by symbolic Gauss-Jordan without pivoting:
    returns (Ainv (G,m,m), flag = 1 + first block with a zero pivot, else 0)."""
    A = _f64(A)
    G, m, _ = A.shape
    B = np.empty_like(A)
    flag = lib().oracle_gj_inverse(G, m, _ptr(A), _ptr(B))
    return B, int(flag)


def gj_apply(Ainv, b):
    Ainv = _f64(Ainv)
    G, m, _ = Ainv.shape
    b = _f64(b).reshape(G * m)
    x = np.empty_like(b)
    lib().oracle_gj_apply(G, m, _ptr(Ainv), _ptr(b), _ptr(x))
    return x


def lu_solve(LU, piv, b):
    LU = _f64(LU); piv = np.ascontiguousarray(piv, dtype=np.int32)
    G, m, _ = LU.shape
    b = _f64(b).reshape(G * m)
    x = np.empty_like(b)
    lib().oracle_lu_solve(G, m, _ptr(LU), _ptr(piv), _ptr(b), _ptr(x))
    return x


def gmres(A, b, P=None, maxl=10, tol=1e-10):
    """Right-preconditioned GMRES on a block-diagonal operator A (G, m, m);
    P: None (identity) or (LU, piv) from lu_factor.  Returns (x, steps, res)."""
    A = _f64(A); G, m, _ = A.shape
    b = _f64(b).reshape(G * m)
    x = np.empty_like(b)
    res = C.c_double(0.0)
    if P is None:
        plu, ppiv = None, None
    else:
        plu = _f64(P[0]); ppiv = np.ascontiguousarray(P[1], dtype=np.int32)
    steps = lib().oracle_gmres(G, m, _ptr(A), _ptr(plu) if plu is not None else None,
                               _ptr(ppiv) if ppiv is not None else None, _ptr(b), _ptr(x),
                               maxl, tol, C.byref(res))
    return x, steps, res.value


def block_matvec(A, x):
    A = _f64(A); G, m, _ = A.shape
    x = _f64(x).reshape(G * m)
    y = np.empty_like(x)
    lib().oracle_block_matvec(G, m, _ptr(A), _ptr(x), _ptr(y))
    return y


# ----------------------------------------------------------- Brusselator
BRUSS = dict(c=0.01, A=1.0, B=3.5, eps=5e-6, alpha=0.1)


def bruss_reaction(y, A=1.0, B=3.5, eps=5e-6):
    y = _f64(y); f = np.empty_like(y)
    lib().oracle_bruss_reaction(y.size // 3, _ptr(y), A, B, eps, _ptr(f)); return f


def bruss_jacobian(y, eps=5e-6):
    y = _f64(y); G = y.size // 3
    J = np.empty((G, 3, 3))
    lib().oracle_bruss_jacobian(G, _ptr(y), eps, _ptr(J)); return J


def advection(y, nx, ny=1, nz=1, kx=0.0, ky=0.0, kz=0.0):
    y = _f64(y); f = np.empty_like(y)
    lib().oracle_advection(nx, ny, nz, kx, ky, kz, _ptr(y), _ptr(f)); return f


def bruss_ic(nx, ny=1, nz=1, Lx=1.0, Ly=1.0, Lz=1.0, A=1.0, B=3.5, alpha=0.1):
    y = np.empty(3 * nx * ny * nz)
    lib().oracle_bruss_ic(nx, ny, nz, Lx, Ly, Lz, A, B, alpha, _ptr(y)); return y


def sbdf_integrate(y0, nsteps, *, kind=0, newton_mode=0, K=3, reaction_only=False,
                   nx=1, ny=1, nz=1, kx=0.0, ky=0.0, kz=0.0,
                   A=1.0, B=3.5, eps=5e-6, lam_E=0.0, lam_I=0.0,
                   h=1e-3, rtol=1e-6, atol=1e-9, tol_nl=1e-3, log_every=0,
                   linsol=0, maxl=5, lin_tol=1e-10):
    """Fixed-step IMEX SBDF1/SBDF2 with modified Newton (oracle.cpp O12/O13).

    Returns (rc, y, stats_dict, ylog or None)."""
    y = np.array(y0, dtype=np.float64, copy=True)
    P = SbdfParams(kind, newton_mode, K, int(bool(reaction_only)), nx, ny, nz,
                   kx, ky, kz, A, B, eps, lam_E, lam_I, h, rtol, atol, tol_nl,
                   linsol, maxl, lin_tol)
    st = SbdfStats()
    ylog = None
    if log_every > 0:
        ylog = np.zeros((nsteps // log_every, y.size))
    rc = lib().oracle_sbdf_integrate(C.byref(P), _ptr(y), nsteps, C.byref(st),
                                     _ptr(ylog) if ylog is not None else None,
                                     log_every)
    stats = {k: getattr(st, k) for k, _ in SbdfStats._fields_}
    return rc, y, stats, ylog


# ------------------------------------------------------- adaptive IMEX ARK
def ark_tableau():
    """(AE 4x4, AI 4x4, b, d, c) of ARK3(2)4L[2]SA as doubles."""
    AE, AI = np.zeros((4, 4)), np.zeros((4, 4))
    b, d, c = np.zeros(4), np.zeros(4), np.zeros(4)
    lib().oracle_ark_tableau(_ptr(AE), _ptr(AI), _ptr(b), _ptr(d), _ptr(c))
    return AE, AI, b, d, c


def ark_integrate(y0, t_end, *, h0=1e-4, maxnl=3, max_steps=100000, fixed=False, kind=0,
                  reaction_only=False, nx=1, ny=1, nz=1, kx=0.0, ky=0.0, kz=0.0, A=1.0, B=3.5,
                  eps=5e-6, lam_E=0.0, lam_I=0.0, rtol=1e-6, atol=1e-9, tol_nl=0.1):
    """Adaptive IMEX ARK3(2)4L[2]SA (oracle.cpp).  Returns (rc, y, stats)."""
    y = np.array(y0, dtype=np.float64, copy=True)
    P = SbdfParams(kind, 1, maxnl, int(bool(reaction_only)), nx, ny, nz, kx, ky, kz, A, B, eps,
                   lam_E, lam_I, h0, rtol, atol, tol_nl, 0, 1, 0.0)
    AP = ArkParams(P, h0, t_end, maxnl, max_steps, int(bool(fixed)), 0)
    st = ArkStats()
    rc = lib().oracle_ark_integrate(C.byref(AP), _ptr(y), C.byref(st))
    return rc, y, {k: getattr(st, k) for k, _ in ArkStats._fields_}
