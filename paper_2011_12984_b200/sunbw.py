"""Thin Python binding of libsunbw.so (include/sunbw.h), by ctypes.

Argument marshalling only: every step of the hot path runs in the
library's CUDA kernels.  Functions keep the C names; N_Vector / SUNMatrix /
SUNLinearSolver / problem / stepper handles are wrapped in small classes
that keep the backing torch tensors alive (the caller-owned memory of
N_VMake_B200, §3).  If the library is missing this module raises —
there is no fallback path of any kind.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SUNBW_LIB", os.path.join(_HERE, "libsunbw.so"))

_lib = None
_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_I64 = C.c_int64

SUNBW_POLICY_GRID_STRIDE = 0
SUNBW_POLICY_THREAD_DIRECT = 1
SUNBW_RECOV_SINGULAR, SUNBW_RECOV_NONCONV, SUNBW_RECOV_BAD_EWT = 1, 2, 3
(BW_K_HALO, BW_K_ADVECTION, BW_K_RHS_COMBINE, BW_K_EWT, BW_K_PREDICT, BW_K_JACOBIAN,
 BW_K_SCALEADDI, BW_K_LU_SETUP, BW_K_REACTION, BW_K_RESIDUAL, BW_K_LU_SOLVE, BW_K_UPDATE,
 BW_K_WRMS, BW_K_FUSED_NEWTON, BW_K_FUSED_PLANE0, BW_K_COUNT_) = range(16)
KERNEL_NAMES = ["halo", "advection", "rhs_combine", "ewt", "predict", "jacobian", "scaleaddi",
                "lu_setup", "reaction", "residual", "lu_solve", "update", "wrms", "fused_newton",
                "fused_plane0"]


class BW_BrussParams(C.Structure):
    _fields_ = [("dim", C.c_int32), ("kind", C.c_int32), ("reaction_only", C.c_int32),
                ("pad_", C.c_int32), ("nx", _I64), ("ny", _I64), ("nz", _I64),
                ("Lx", _D), ("Ly", _D), ("Lz", _D), ("c", _D), ("A", _D), ("B", _D),
                ("eps", _D), ("alpha", _D), ("lam_E", _D), ("lam_I", _D)]


class BW_StepperOptions(C.Structure):
    _fields_ = [("h", _D), ("newton_mode", C.c_int32), ("K", C.c_int32), ("tol_nl", _D),
                ("rtol", _D), ("atol", _D), ("use_graph", C.c_int32), ("timing", C.c_int32),
                ("fused", C.c_int32), ("fused_advection", C.c_int32),
                ("linsol", C.c_int32), ("maxl", C.c_int32), ("lin_tol", _D),
                ("single_step_launches", C.c_int32), ("numerics", C.c_int32)]


class BW_StepperStats(C.Structure):
    _fields_ = [("steps", _I64), ("newton_iters", _I64), ("setups", _I64), ("solves", _I64),
                ("fails", _I64), ("singular", _I64), ("last_nu", _D), ("t", _D),
                ("lin_iters", _I64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class BW_ArkOptions(C.Structure):
    _fields_ = [("h0", _D), ("rtol", _D), ("atol", _D), ("tol_nl", _D), ("maxnl", C.c_int32),
                ("max_steps", C.c_int32), ("fixed", C.c_int32), ("pad_", C.c_int32)]


class BW_ArkStats(C.Structure):
    _fields_ = [("accepted", _I64), ("rejected_err", _I64), ("rejected_nl", _I64),
                ("newton_iters", _I64), ("setups", _I64), ("t", _D), ("h_last", _D)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "SUNBW_ContextCreate": (_I, [_I, _P, C.POINTER(_P)]),
    "SUNBW_ContextSetStream": (_I, [_P, _P]),
    "SUNBW_ContextGetStream": (_P, [_P]),
    "SUNBW_ContextDestroy": (_I, [_P]),
    "SUNBW_GetLastError": (_I, [_P, _I]),
    "SUNBW_ErrorString": (C.c_char_p, [_I]),
    "SUNBW_ContextKernelLaunches": (_I64, [_P]),
    "SUNBW_NcclGetUniqueId": (_I, [_P]),
    "SUNBW_ContextInitNccl": (_I, [_P, _P, _I, _I]),
    "SUNBW_FakeCommCreate": (_I, [_I, C.POINTER(_P)]),
    "SUNBW_FakeCommDestroy": (_I, [_P]),
    "SUNBW_ContextSetFakeComm": (_I, [_P, _P, _I]),
    "SUNBW_ContextRank": (_I, [_P]),
    "SUNBW_ContextNRanks": (_I, [_P]),
    "SUNBW_SelfTestDivision": (_I, [_P, _I64, _P, _P, _P]),
    "SUNBW_ProbeLaunchLatency": (_I, [_P, _I64, _P]),
    "N_VNew_B200": (_P, [_P, _I64]),
    "N_VMake_B200": (_P, [_P, _I64, _P]),
    "N_VClone": (_P, [_P]),
    "N_VDestroy": (None, [_P]),
    "N_VGetDeviceArrayPointer_B200": (_P, [_P]),
    "N_VSetDeviceArrayPointer_B200": (_I, [_P, _P]),
    "N_VGetLength": (_I64, [_P]),
    "N_VGetLocalLength": (_I64, [_P]),
    "N_VSetKernelExecPolicy_B200": (_I, [_P, _I, _I, _I, _I]),
    "N_VLinearSum": (None, [_D, _P, _D, _P, _P]),
    "N_VScale": (None, [_D, _P, _P]),
    "N_VProd": (None, [_P, _P, _P]),
    "N_VDiv": (None, [_P, _P, _P]),
    "N_VConst": (None, [_D, _P]),
    "N_VAbs": (None, [_P, _P]),
    "N_VInv": (None, [_P, _P]),
    "N_VAddConst": (None, [_P, _D, _P]),
    "N_VDotProd": (_D, [_P, _P]),
    "N_VWrmsNorm": (_D, [_P, _P]),
    "N_VWrmsNormMask": (_D, [_P, _P, _P]),
    "N_VMaxNorm": (_D, [_P]),
    "N_VMin": (_D, [_P]),
    "N_VDotProdLocal": (_D, [_P, _P]),
    "N_VWSqrSumLocal": (_D, [_P, _P]),
    "N_VLinearCombination": (_I, [_I, _P, _P, _P]),
    "N_VScaleAddMulti": (_I, [_I, _P, _P, _P, _P]),
    "N_VDotProdMulti": (_I, [_I, _P, _P, _P]),
    "N_VLinearSumVectorArray": (_I, [_I, _D, _P, _D, _P, _P]),
    "N_VScaleVectorArray": (_I, [_I, _P, _P, _P]),
    "N_VConstVectorArray": (_I, [_I, _D, _P]),
    "N_VWrmsNormVectorArray": (_I, [_I, _P, _P, _P]),
    "N_VWrmsNormMaskVectorArray": (_I, [_I, _P, _P, _P, _P]),
    "N_VScaleAddMultiVectorArray": (_I, [_I, _I, _P, _P, _P, _P]),
    "N_VLinearCombinationVectorArray": (_I, [_I, _I, _P, _P, _P]),
    "SUNMatrix_B200BlockDiag": (_P, [_P, _I64, _I]),
    "SUNMatrix_B200BlockDiagMake": (_P, [_P, _I64, _I, _P]),
    "SUNMatrix_B200BlockDiag_Data": (_P, [_P]),
    "SUNMatrix_B200BlockDiag_NumBlocks": (_I64, [_P]),
    "SUNMatrix_B200BlockDiag_BlockSize": (_I, [_P]),
    "SUNMatScaleAddI": (_I, [_D, _P]),
    "SUNMatMatvec": (_I, [_P, _P, _P]),
    "SUNMatDestroy": (None, [_P]),
    "SUNLinSol_B200BatchedLU": (_P, [_P, _P]),
    "SUNLinSol_B200BatchedGJ": (_P, [_P, _P]),
    "SUNLinSolSetup": (_I, [_P, _P]),
    "SUNLinSolSolve": (_I, [_P, _P, _P, _P, _D]),
    "SUNLinSolLastFlag": (_I64, [_P]),
    "SUNLinSol_B200BatchedLU_SetDeferredCheck": (_I, [_P, _I]),
    "SUNLinSol_B200BatchedLU_Pivots": (_P, [_P]),
    "SUNLinSolFree": (None, [_P]),
    "SUNLinSol_B200SPGMR": (_P, [_P, _P, _I, _I]),
    "SUNLinSolNumIters": (_I64, [_P]),
    "SUNLinSolResNorm": (_D, [_P]),
    "BW_ProblemCreate": (_I, [_P, C.POINTER(BW_BrussParams), C.POINTER(_P)]),
    "BW_ProblemDestroy": (_I, [_P]),
    "BW_ProblemLocalCells": (_I64, [_P]),
    "BW_ProblemCellOffset": (_I64, [_P]),
    "BW_InitialCondition": (_I, [_P, _P]),
    "BW_AdvectionRHS": (_I, [_P, _P, _P]),
    "BW_ReactionRHS": (_I, [_P, _P, _P]),
    "BW_ReactionJacobian": (_I, [_P, _P, _P]),
    "BW_StepperCreate": (_I, [_P, _P, C.POINTER(BW_StepperOptions), C.POINTER(_P)]),
    "BW_StepperAdvance": (_I, [_P, _I64, _P, C.POINTER(BW_StepperStats)]),
    "BW_StepperReset": (_I, [_P, _P, _D]),
    "BW_StepperKernelTimes": (_I, [_P, _P, _P, _I]),
    "BW_StepperDestroy": (_I, [_P]),
    "BW_ArkCreate": (_I, [_P, _P, C.POINTER(BW_ArkOptions), C.POINTER(_P)]),
    "BW_ArkEvolve": (_I, [_P, _D, _P, C.POINTER(BW_ArkStats)]),
    "BW_ArkDestroy": (_I, [_P]),
}


def lib():
    """Loads libsunbw.so (raises if it was not built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                               "(the CUDA library is the only implementation)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


class SunbwError(RuntimeError):
    pass


def _check(rc, what):
    if rc < 0:
        raise SunbwError(f"{what}: {lib().SUNBW_ErrorString(rc).decode()} ({rc})")
    return rc


# ------------------------------------------------------------------ objects
class Context:
    """SUNBW_Context on `device`, bound to a CUDA stream (default: torch's
    current stream)."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = _P()
        _check(lib().SUNBW_ContextCreate(device, _P(self.stream.cuda_stream), C.byref(h)),
               "SUNBW_ContextCreate")
        self.handle = h.value
        self._keep = []

    def last_error(self, clear=True) -> int:
        return lib().SUNBW_GetLastError(self.handle, int(clear))

    def check(self, what="sunbw"):
        e = self.last_error(True)
        if e < 0:
            raise SunbwError(f"{what}: {lib().SUNBW_ErrorString(e).decode()} ({e})")

    @property
    def launches(self) -> int:
        return lib().SUNBW_ContextKernelLaunches(self.handle)

    @property
    def rank(self) -> int:
        return lib().SUNBW_ContextRank(self.handle)

    @property
    def nranks(self) -> int:
        return lib().SUNBW_ContextNRanks(self.handle)

    def init_nccl(self, uid: bytes, rank: int, nranks: int):
        buf = C.create_string_buffer(uid, 128)
        _check(lib().SUNBW_ContextInitNccl(self.handle, buf, rank, nranks), "SUNBW_ContextInitNccl")

    def set_fake_comm(self, comm: "FakeComm", rank: int):
        _check(lib().SUNBW_ContextSetFakeComm(self.handle, comm.handle, rank),
               "SUNBW_ContextSetFakeComm")

    def destroy(self):
        if getattr(self, "handle", None):
            lib().SUNBW_ContextDestroy(self.handle)
            self.handle = None


def selftest_division(ctx: "Context", a: torch.Tensor, b: torch.Tensor):
    """(quotient mismatches, pairs checked)."""
    out = (_I64 * 2)()
    _check(lib().SUNBW_SelfTestDivision(ctx.handle, a.numel(), _P(a.data_ptr()), _P(b.data_ptr()), out),
           "SUNBW_SelfTestDivision")
    return tuple(out)


def probe_launch_latency(ctx: "Context", n: int = 100_000):
    """(eager us/launch, graph us/node, host launch+sync round trip us)."""
    out = (C.c_double * 3)()
    _check(lib().SUNBW_ProbeLaunchLatency(ctx.handle, n, out), "SUNBW_ProbeLaunchLatency")
    return tuple(out)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().SUNBW_NcclGetUniqueId(buf), "SUNBW_NcclGetUniqueId")
    return buf.raw


class FakeComm:
    def __init__(self, nranks: int):
        h = _P()
        _check(lib().SUNBW_FakeCommCreate(nranks, C.byref(h)), "SUNBW_FakeCommCreate")
        self.handle = h.value
        self.nranks = nranks

    def destroy(self):
        if self.handle:
            lib().SUNBW_FakeCommDestroy(self.handle)
            self.handle = None


class NVector:
    """N_Vector wrapping a 1-D contiguous float64 CUDA tensor (N_VMake_B200)."""

    def __init__(self, ctx: Context, t: torch.Tensor):
        if not (t.is_cuda and t.dtype == torch.float64 and t.dim() == 1 and t.is_contiguous()):
            raise ValueError("N_VMake_B200 needs a contiguous 1-D float64 CUDA tensor")
        self.ctx, self.t = ctx, t
        h = lib().N_VMake_B200(ctx.handle, t.numel(), _P(t.data_ptr()) if t.numel() else None)
        if not h:
            ctx.check("N_VMake_B200")
            raise SunbwError("N_VMake_B200 failed")
        self.handle = h

    @property
    def _as_parameter_(self):
        return _P(self.handle)

    def __len__(self):
        return self.t.numel()

    def global_length(self) -> int:
        return lib().N_VGetLength(self.handle)

    def set_policy(self, policy=SUNBW_POLICY_GRID_STRIDE, block=0, grid=0, reduce_block=0):
        _check(lib().N_VSetKernelExecPolicy_B200(self.handle, policy, block, grid, reduce_block),
               "N_VSetKernelExecPolicy_B200")

    def __del__(self):
        try:
            if self.handle:
                lib().N_VDestroy(self.handle)
        except Exception:
            pass
        self.handle = None


def _vec_array(vs: Sequence[NVector]):
    return (_P * len(vs))(*[v.handle for v in vs])


def _dbl_array(xs):
    return (_D * len(xs))(*[float(x) for x in xs])


# -------------------------------------------------------- N_Vector ops (C names)
def N_VLinearSum(a, x, b, y, z): lib().N_VLinearSum(a, x, b, y, z)
def N_VScale(c, x, z): lib().N_VScale(c, x, z)
def N_VProd(x, y, z): lib().N_VProd(x, y, z)
def N_VDiv(x, y, z): lib().N_VDiv(x, y, z)
def N_VConst(c, z): lib().N_VConst(c, z)
def N_VAbs(x, z): lib().N_VAbs(x, z)
def N_VInv(x, z): lib().N_VInv(x, z)
def N_VAddConst(x, b, z): lib().N_VAddConst(x, b, z)
def N_VDotProd(x, y) -> float: return lib().N_VDotProd(x, y)
def N_VWrmsNorm(x, w) -> float: return lib().N_VWrmsNorm(x, w)
def N_VWrmsNormMask(x, w, idv) -> float: return lib().N_VWrmsNormMask(x, w, idv)
def N_VMaxNorm(x) -> float: return lib().N_VMaxNorm(x)
def N_VMin(x) -> float: return lib().N_VMin(x)
def N_VDotProdLocal(x, y) -> float: return lib().N_VDotProdLocal(x, y)
def N_VWSqrSumLocal(x, w) -> float: return lib().N_VWSqrSumLocal(x, w)


def N_VLinearCombination(c, X: Sequence[NVector], z: NVector) -> int:
    return lib().N_VLinearCombination(len(X), _dbl_array(c), _vec_array(X), z)


def N_VScaleAddMulti(a, x: NVector, Y: Sequence[NVector], Z: Sequence[NVector]) -> int:
    return lib().N_VScaleAddMulti(len(Y), _dbl_array(a), x, _vec_array(Y), _vec_array(Z))


def N_VDotProdMulti(x: NVector, Y: Sequence[NVector]):
    out = (_D * len(Y))()
    rc = lib().N_VDotProdMulti(len(Y), x, _vec_array(Y), out)
    if rc != 0:
        raise SunbwError(f"N_VDotProdMulti failed ({rc})")
    return list(out)


# ------------------------------------------------------ vector-array ops
def N_VLinearSumVectorArray(a, X, b, Y, Z) -> int:
    return lib().N_VLinearSumVectorArray(len(X), a, _vec_array(X), b, _vec_array(Y), _vec_array(Z))


def N_VScaleVectorArray(c, X, Z) -> int:
    return lib().N_VScaleVectorArray(len(X), _dbl_array(c), _vec_array(X), _vec_array(Z))


def N_VConstVectorArray(c, Z) -> int:
    return lib().N_VConstVectorArray(len(Z), c, _vec_array(Z))


def N_VWrmsNormVectorArray(X, W):
    out = (_D * len(X))()
    if lib().N_VWrmsNormVectorArray(len(X), _vec_array(X), _vec_array(W), out):
        raise SunbwError("N_VWrmsNormVectorArray failed")
    return list(out)


def N_VWrmsNormMaskVectorArray(X, W, idv):
    out = (_D * len(X))()
    if lib().N_VWrmsNormMaskVectorArray(len(X), _vec_array(X), _vec_array(W), idv, out):
        raise SunbwError("N_VWrmsNormMaskVectorArray failed")
    return list(out)


def _vec_array_2d(rows):
    inner = [_vec_array(r) for r in rows]
    arr = (_P * len(rows))(*[C.cast(r, _P) for r in inner])
    arr._keep = inner
    return arr


def N_VScaleAddMultiVectorArray(a, X, Y, Z) -> int:
    return lib().N_VScaleAddMultiVectorArray(len(X), len(a), _dbl_array(a), _vec_array(X),
                                             _vec_array_2d(Y), _vec_array_2d(Z))


def N_VLinearCombinationVectorArray(c, X, Z) -> int:
    return lib().N_VLinearCombinationVectorArray(len(Z), len(c), _dbl_array(c), _vec_array_2d(X),
                                                 _vec_array(Z))


# ------------------------------------------------------- block-diagonal + LU
class SUNMatrix:
    """Block-diagonal matrix wrapping a (G, m, m) float64 CUDA tensor."""

    def __init__(self, ctx: Context, t: torch.Tensor):
        if not (t.is_cuda and t.dtype == torch.float64 and t.dim() == 3 and t.is_contiguous()
                and t.shape[1] == t.shape[2]):
            raise ValueError("block-diagonal data must be a contiguous (G, m, m) float64 CUDA tensor")
        self.ctx, self.t = ctx, t
        G, m = t.shape[0], t.shape[1]
        h = lib().SUNMatrix_B200BlockDiagMake(ctx.handle, G, m, _P(t.data_ptr()) if G else None)
        if not h:
            raise SunbwError("SUNMatrix_B200BlockDiagMake failed (1 <= m <= 8)")
        self.handle = h

    @property
    def _as_parameter_(self):
        return _P(self.handle)

    def __del__(self):
        try:
            if self.handle:
                lib().SUNMatDestroy(self.handle)
        except Exception:
            pass
        self.handle = None


def SUNMatScaleAddI(c, A: SUNMatrix) -> int:
    return _check(lib().SUNMatScaleAddI(c, A), "SUNMatScaleAddI")


def SUNMatMatvec(A: SUNMatrix, x: NVector, y: NVector) -> int:
    return _check(lib().SUNMatMatvec(A, x, y), "SUNMatMatvec")


class SUNLinearSolver:
    """Batched block LU (default); with gj=True the paper's block inverse by
    symbolic Gauss-Jordan; with spgmr_maxl, SPGMR (GMRES with the
    block LU as optional preconditioner)."""

    def __init__(self, y: NVector, A: SUNMatrix, spgmr_maxl: int = 0, block_prec: bool = True,
                 gj: bool = False):
        if spgmr_maxl:
            h = lib().SUNLinSol_B200SPGMR(y, A, spgmr_maxl, int(block_prec))
        elif gj:
            h = lib().SUNLinSol_B200BatchedGJ(y, A)
        else:
            h = lib().SUNLinSol_B200BatchedLU(y, A)
        if not h:
            raise SunbwError("SUNLinearSolver construction failed")
        self.handle = h
        self.nblocks = A.t.shape[0]

    @property
    def _as_parameter_(self):
        return _P(self.handle)

    def pivots(self) -> torch.Tensor:
        """Copy of the packed pivot codes (int32 per block)."""
        n = self.nblocks
        if n == 0:
            return torch.empty(0, dtype=torch.int32)
        ptr = lib().SUNLinSol_B200BatchedLU_Pivots(self.handle)
        torch.cuda.synchronize()
        return _device_view(ptr, (n,), "<i4").cpu()

    def __del__(self):
        try:
            if self.handle:
                lib().SUNLinSolFree(self.handle)
        except Exception:
            pass
        self.handle = None


class _CudaArray:
    """A raw device pointer exposed through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _device_view(ptr: int, shape, typestr: str) -> torch.Tensor:
    """torch view of library-owned device memory (valid while the owner lives)."""
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device="cuda")


def SUNLinSolSetup(S: SUNLinearSolver, A: SUNMatrix) -> int:
    return _check(lib().SUNLinSolSetup(S, A), "SUNLinSolSetup")


def SUNLinSolSolve(S: SUNLinearSolver, A: SUNMatrix, x: NVector, b: NVector, tol=0.0) -> int:
    return _check(lib().SUNLinSolSolve(S, A, x, b, tol), "SUNLinSolSolve")


def SUNLinSolNumIters(S: SUNLinearSolver) -> int:
    return lib().SUNLinSolNumIters(S)


def SUNLinSolResNorm(S: SUNLinearSolver) -> float:
    return lib().SUNLinSolResNorm(S)


def SUNLinSolLastFlag(S: SUNLinearSolver) -> int:
    return lib().SUNLinSolLastFlag(S)


def SUNLinSol_B200BatchedLU_SetDeferredCheck(S: SUNLinearSolver, deferred: bool) -> int:
    return lib().SUNLinSol_B200BatchedLU_SetDeferredCheck(S, int(deferred))


# ------------------------------------------------------- problem + stepper
BRUSS_DEFAULTS = dict(c=0.01, A=1.0, B=3.5, eps=5e-6, alpha=0.1)


def bruss_params(dim=1, nx=64, ny=1, nz=1, Lx=1.0, Ly=1.0, Lz=1.0, kind=0, reaction_only=False,
                 lam_E=0.0, lam_I=0.0, **kw) -> BW_BrussParams:
    p = dict(BRUSS_DEFAULTS)
    p.update(kw)
    return BW_BrussParams(dim, kind, int(bool(reaction_only)), 0, nx, ny, nz, Lx, Ly, Lz,
                          p["c"], p["A"], p["B"], p["eps"], p["alpha"], lam_E, lam_I)


class Problem:
    def __init__(self, ctx: Context, params: BW_BrussParams):
        self.ctx, self.params = ctx, params
        h = _P()
        _check(lib().BW_ProblemCreate(ctx.handle, C.byref(params), C.byref(h)), "BW_ProblemCreate")
        self.handle = h.value

    @property
    def _as_parameter_(self):
        return _P(self.handle)

    @property
    def local_cells(self) -> int:
        return lib().BW_ProblemLocalCells(self.handle)

    @property
    def cell_offset(self) -> int:
        return lib().BW_ProblemCellOffset(self.handle)

    def destroy(self):
        if self.handle:
            lib().BW_ProblemDestroy(self.handle)
            self.handle = None


def BW_InitialCondition(P: Problem, y: NVector) -> int:
    return _check(lib().BW_InitialCondition(P, y), "BW_InitialCondition")


def BW_AdvectionRHS(P: Problem, y: NVector, fE: NVector) -> int:
    return _check(lib().BW_AdvectionRHS(P, y, fE), "BW_AdvectionRHS")


def BW_ReactionRHS(P: Problem, y: NVector, fI: NVector) -> int:
    return _check(lib().BW_ReactionRHS(P, y, fI), "BW_ReactionRHS")


def BW_ReactionJacobian(P: Problem, y: NVector, J: SUNMatrix) -> int:
    return _check(lib().BW_ReactionJacobian(P, y, J), "BW_ReactionJacobian")


def stepper_options(h=1e-3, newton_mode=0, K=3, tol_nl=1e-3, rtol=1e-6, atol=1e-9,
                    use_graph=True, timing=False, fused=False,
                    fused_advection=True, linsol=0, maxl=5, lin_tol=1e-10,
                    single_step_launches=False, numerics=0) -> BW_StepperOptions:
    """numerics (fused mode): 0 bit-exact, 1 contracted (FMA) cell step held
    to relative 1e-9 (DESIGN R30)."""
    return BW_StepperOptions(h, newton_mode, K, tol_nl, rtol, atol, int(use_graph), int(timing),
                             int(fused), int(fused_advection), linsol, maxl, lin_tol,
                             int(single_step_launches), int(numerics))


class Stepper:
    def __init__(self, P: Problem, y0: NVector, opts: BW_StepperOptions):
        self.P, self.opts = P, opts
        h = _P()
        _check(lib().BW_StepperCreate(P, y0, C.byref(opts), C.byref(h)), "BW_StepperCreate")
        self.handle = h.value

    @property
    def _as_parameter_(self):
        return _P(self.handle)

    def advance(self, nsteps: int, y_out: NVector | None = None):
        st = BW_StepperStats()
        rc = lib().BW_StepperAdvance(self.handle, nsteps, y_out if y_out is not None else None,
                                     C.byref(st))
        _check(rc, "BW_StepperAdvance")
        return rc, st.as_dict()

    def reset(self, y0: NVector, t0: float = 0.0):
        _check(lib().BW_StepperReset(self.handle, y0, t0), "BW_StepperReset")

    def kernel_times(self, reset=False):
        ms = (_D * BW_K_COUNT_)()
        cnt = (_I64 * BW_K_COUNT_)()
        _check(lib().BW_StepperKernelTimes(self.handle, ms, cnt, int(reset)), "BW_StepperKernelTimes")
        return {KERNEL_NAMES[k]: (ms[k], cnt[k]) for k in range(BW_K_COUNT_) if cnt[k]}

    def destroy(self):
        if self.handle:
            lib().BW_StepperDestroy(self.handle)
            self.handle = None


class Ark:
    """Adaptive IMEX ARK3(2)4L[2]SA integrator (BW_ArkCreate / BW_ArkEvolve)."""

    def __init__(self, P: Problem, y0: NVector, h0=1e-4, rtol=1e-6, atol=1e-9, tol_nl=0.1, maxnl=3,
                 max_steps=100000, fixed=False, fused=False):
        self.opts = BW_ArkOptions(h0, rtol, atol, tol_nl, maxnl, max_steps, int(bool(fixed)), int(bool(fused)))
        h = _P()
        _check(lib().BW_ArkCreate(P, y0, C.byref(self.opts), C.byref(h)), "BW_ArkCreate")
        self.handle = h.value

    def evolve(self, t_end: float, y_out: NVector | None = None):
        st = BW_ArkStats()
        rc = lib().BW_ArkEvolve(self.handle, t_end, y_out if y_out is not None else None, C.byref(st))
        _check(rc, "BW_ArkEvolve")
        return rc, st.as_dict()

    def destroy(self):
        if self.handle:
            lib().BW_ArkDestroy(self.handle)
            self.handle = None
