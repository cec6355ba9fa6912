// vecarray.cu — SUNDIALS "vector array" fused operations (N_V*VectorArray):
// one kernel launch applies a streaming op or a reduction to nvec vector
// tuples (blockIdx.y = vector index), instead of nvec launches.  These are
// the fused-op family the integrators use for stage/Krylov blocks (DESIGN
// R1).  Same rounding rules as the single-vector ops
// (explicit RN intrinsics: bit-identical to the serial definitions);
// reductions are deterministic two-level folds, one allreduce of nvec
// values when partitioned.

#include <cmath>
#include <vector>

#include "sunbw_device.cuh"
#include "sunbw_internal.h"

namespace {

using sunbw::d4;
using sunbw::ld4;
using sunbw::Split;
using sunbw::split_for;
using sunbw::st4;

constexpr int kMaxVA = 8;   // vectors per launch (larger nvec: several launches)

struct VAArgs {
  const double* X[kMaxVA];
  const double* Y[kMaxVA];
  double* Z[kMaxVA];
  double c[kMaxVA];
  Split sp[kMaxVA];
  double a, b;
};

// kind 0: Z = a X + b Y;  1: Z = c_j X;  2: Z = a (const)
template <int KIND>
__device__ __forceinline__ double va_op(const VAArgs& A, int j, double x, double y) {
  if (KIND == 0) return __dadd_rn(__dmul_rn(A.a, x), __dmul_rn(A.b, y));
  if (KIND == 1) return __dmul_rn(A.c[j], x);
  return A.a;
}

template <int KIND>
__global__ void __launch_bounds__(256) k_va_stream(VAArgs A, int64_t n) {
  const int j = blockIdx.y;
  const Split sp = A.sp[j];
  const double* X = A.X[j];
  const double* Y = A.Y[j];
  double* Z = A.Z[j];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < sp.head; i += nth)
    Z[i] = va_op<KIND>(A, j, KIND < 2 ? X[i] : 0.0, KIND == 0 ? Y[i] : 0.0);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth)
    Z[i] = va_op<KIND>(A, j, KIND < 2 ? X[i] : 0.0, KIND == 0 ? Y[i] : 0.0);
  for (int64_t v = tid; v < sp.nvec; v += nth) {
    const int64_t off = sp.head + 4 * v;
    d4 xv{}, yv{}, o;
    if (KIND < 2) xv = ld4(X + off);
    if (KIND == 0) yv = ld4(Y + off);
#pragma unroll
    for (int l = 0; l < 4; ++l) o.v[l] = va_op<KIND>(A, j, xv.v[l], yv.v[l]);
    st4(Z + off, o);
  }
}

// Σ (x_i w_i)^2 [id_i > 0] for vector j: one partial per (block, j)
template <bool MASK>
__global__ void __launch_bounds__(256) k_va_wsqr(VAArgs A, const double* id, int64_t n, double* partials) {
  __shared__ double sh[32];
  const int j = blockIdx.y, nv = gridDim.y;
  const double* X = A.X[j];
  const double* W = A.Y[j];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = tid;
  for (; i + nth < n; i += 2 * nth) {          // two independent chains
    const double p0 = __dmul_rn(X[i], W[i]), p1 = __dmul_rn(X[i + nth], W[i + nth]);
    if (!MASK || id[i] > 0.0) s0 = __fma_rn(p0, p0, s0);
    if (!MASK || id[i + nth] > 0.0) s1 = __fma_rn(p1, p1, s1);
  }
  if (i < n) {
    const double p0 = __dmul_rn(X[i], W[i]);
    if (!MASK || id[i] > 0.0) s0 = __fma_rn(p0, p0, s0);
  }
  double s = __dadd_rn(s0, s1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) sh[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sh[0];
    for (int q = 1; q < nw; ++q) t = __dadd_rn(t, sh[q]);
    partials[(int64_t)blockIdx.x * nv + j] = t;
  }
}

__global__ void k_va_fold(const double* partials, int nblocks, int nv, double* out) {
  const int j = threadIdx.x;
  if (j >= nv) return;
  double t = 0.0;
  for (int b = 0; b < nblocks; ++b) t = __dadd_rn(t, partials[(int64_t)b * nv + j]);
  out[j] = t;
}

__global__ void k_va_wrms_final(const double* sums, int nv, double nglobal, double* h_out) {
  const int j = threadIdx.x;
  if (j < nv) h_out[j] = __dsqrt_rn(__ddiv_rn(sums[j], nglobal));
}

int launch_stream(SUNBW_Context ctx, int kind, int nvec, int64_t n, VAArgs& A) {
  if (n <= 0 || nvec <= 0) return 0;
  int64_t items = 0;
  for (int j = 0; j < nvec; ++j) {
    const double* ptrs[3] = {A.Z[j], A.X[j], A.Y[j]};
    const int np = kind == 0 ? 3 : (kind == 1 ? 2 : 1);
    A.sp[j] = split_for(n, ptrs, np);
    int64_t it = A.sp[j].nvec > 0 ? A.sp[j].nvec : n;
    if (it > items) items = it;
  }
  int64_t need = (items + 255) / 256;
  int64_t cap = (int64_t)ctx->nsm * 8 / nvec + 1;
  dim3 grid((unsigned)(need < cap ? (need < 1 ? 1 : need) : cap), nvec);
  if (kind == 0) k_va_stream<0><<<grid, 256, 0, ctx->stream>>>(A, n);
  else if (kind == 1) k_va_stream<1><<<grid, 256, 0, ctx->stream>>>(A, n);
  else k_va_stream<2><<<grid, 256, 0, ctx->stream>>>(A, n);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

bool same_shape(N_Vector a, N_Vector b) {
  if (!a || !b) return false;
  if (a->ctx != b->ctx) { ctx_set_err(a->ctx, SUNBW_ERR_CONTEXT); return false; }
  if (a->local_len != b->local_len) { ctx_set_err(a->ctx, SUNBW_ERR_LENGTH); return false; }
  return true;
}

}  // namespace

extern "C" int N_VLinearSumVectorArray(int nvec, double a, N_Vector* X, double b, N_Vector* Y,
                                       N_Vector* Z) {
  if (nvec < 1 || !X || !Y || !Z) return -1;
  for (int j = 0; j < nvec; ++j)
    if (!same_shape(Z[0], X[j]) || !same_shape(Z[0], Y[j]) || !same_shape(Z[0], Z[j])) return -1;
  for (int j0 = 0; j0 < nvec; j0 += kMaxVA) {
    const int k = nvec - j0 < kMaxVA ? nvec - j0 : kMaxVA;
    VAArgs A{};
    A.a = a;
    A.b = b;
    for (int j = 0; j < k; ++j) { A.X[j] = X[j0 + j]->d; A.Y[j] = Y[j0 + j]->d; A.Z[j] = Z[j0 + j]->d; }
    if (launch_stream(Z[0]->ctx, 0, k, Z[0]->local_len, A)) return -1;
  }
  return 0;
}

extern "C" int N_VScaleVectorArray(int nvec, const double* c, N_Vector* X, N_Vector* Z) {
  if (nvec < 1 || !c || !X || !Z) return -1;
  for (int j = 0; j < nvec; ++j)
    if (!same_shape(Z[0], X[j]) || !same_shape(Z[0], Z[j])) return -1;
  for (int j0 = 0; j0 < nvec; j0 += kMaxVA) {
    const int k = nvec - j0 < kMaxVA ? nvec - j0 : kMaxVA;
    VAArgs A{};
    for (int j = 0; j < k; ++j) { A.X[j] = X[j0 + j]->d; A.Z[j] = Z[j0 + j]->d; A.c[j] = c[j0 + j]; }
    if (launch_stream(Z[0]->ctx, 1, k, Z[0]->local_len, A)) return -1;
  }
  return 0;
}

extern "C" int N_VConstVectorArray(int nvec, double c, N_Vector* Z) {
  if (nvec < 1 || !Z) return -1;
  for (int j = 0; j < nvec; ++j)
    if (!same_shape(Z[0], Z[j])) return -1;
  for (int j0 = 0; j0 < nvec; j0 += kMaxVA) {
    const int k = nvec - j0 < kMaxVA ? nvec - j0 : kMaxVA;
    VAArgs A{};
    A.a = c;
    for (int j = 0; j < k; ++j) A.Z[j] = Z[j0 + j]->d;
    if (launch_stream(Z[0]->ctx, 2, k, Z[0]->local_len, A)) return -1;
  }
  return 0;
}

static int wrms_array(int nvec, N_Vector* X, N_Vector* W, N_Vector id, double* nrm) {
  if (nvec < 1 || nvec > 64 || !X || !W || !nrm) return -1;
  for (int j = 0; j < nvec; ++j)
    if (!same_shape(X[0], X[j]) || !same_shape(X[0], W[j])) return -1;
  if (id && !same_shape(X[0], id)) return -1;
  SUNBW_Context ctx = X[0]->ctx;
  if (X[0]->global_len == 0) return ctx_set_err(ctx, SUNBW_ERR_EMPTY), -1;
  const int64_t n = X[0]->local_len;
  double* sums = ctx->d_red + 128;                      // nvec <= 64 slots
  for (int j0 = 0; j0 < nvec; j0 += kMaxVA) {
    const int k = nvec - j0 < kMaxVA ? nvec - j0 : kMaxVA;
    VAArgs A{};
    for (int j = 0; j < k; ++j) { A.X[j] = X[j0 + j]->d; A.Y[j] = W[j0 + j]->d; }
    int64_t need = (n + 511) / 512;
    int64_t cap = (int64_t)ctx->nsm * 8 / k + 1;
    int gx = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
    dim3 grid(gx, k);
    if (id) k_va_wsqr<true><<<grid, 256, 0, ctx->stream>>>(A, id->d, n, ctx->d_partials);
    else k_va_wsqr<false><<<grid, 256, 0, ctx->stream>>>(A, nullptr, n, ctx->d_partials);
    k_va_fold<<<1, 32, 0, ctx->stream>>>(ctx->d_partials, gx, k, sums + j0);
    ctx->launches += 2;
    if (ctx_check_launch(ctx)) return -1;
  }
  if (ctx->comm && ctx->comm->nranks > 1) {
    int e = ctx->comm->allreduce(sums, nvec, RED_SUM, ctx->stream);
    if (e) return ctx_set_err(ctx, e), -1;
  }
  k_va_wrms_final<<<1, 64, 0, ctx->stream>>>(sums, nvec, (double)X[0]->global_len, ctx->h_slot_dev);
  ctx->launches++;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA), -1;
  for (int j = 0; j < nvec; ++j) nrm[j] = ((volatile double*)ctx->h_slot)[j];
  return 0;
}

extern "C" int N_VWrmsNormVectorArray(int nvec, N_Vector* X, N_Vector* W, double* nrm) {
  return wrms_array(nvec, X, W, nullptr, nrm);
}

extern "C" int N_VWrmsNormMaskVectorArray(int nvec, N_Vector* X, N_Vector* W, N_Vector id, double* nrm) {
  if (!id) return -1;
  return wrms_array(nvec, X, W, id, nrm);
}

// Z_ij = a_j X_i + Y_ij  /  Z_i = Σ_j c_j X_ij : per output vector one
// fused multi-vector launch (2D pointer arrays are row-major [nvec][nsum])
extern "C" int N_VScaleAddMultiVectorArray(int nvec, int nsum, const double* a, N_Vector* X,
                                           N_Vector** Y, N_Vector** Z) {
  if (nvec < 1 || nsum < 1 || !a || !X || !Y || !Z) return -1;
  for (int i = 0; i < nvec; ++i)
    if (N_VScaleAddMulti(nsum, a, X[i], Y[i], Z[i])) return -1;
  return 0;
}

extern "C" int N_VLinearCombinationVectorArray(int nvec, int nsum, const double* c, N_Vector** X,
                                               N_Vector* Z) {
  if (nvec < 1 || nsum < 1 || !c || !X || !Z) return -1;
  for (int i = 0; i < nvec; ++i)
    if (N_VLinearCombination(nsum, c, X[i], Z[i])) return -1;
  return 0;
}
