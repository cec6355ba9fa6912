// nvector.cu — the N_Vector object and its sm_100a kernels.
//
// Streaming ops (§2, §4.1): one grid-stride kernel template,
// 256-bit (LDG.E.256 / STG.E.256) vector accesses on 32-byte-aligned runs,
// scalar head/tail, U independent 32-B loads per operand in flight per thread.
// Every arithmetic step is an explicit round-to-nearest intrinsic
// (__dmul_rn/__dadd_rn/__ddiv_rn), so no FMA contraction can change bits:
// results are bit-identical to the serial definition (DESIGN R2/R3).
//
// Reductions (§4.1): per-thread accumulation over the same
// vector runs, warp-shuffle tree, shared-memory tree across warps, one
// partial per CTA; then a single-CTA fold of the partials in a fixed order
// (deterministic, no atomics on the result path), the communicator's
// allreduce when partitioned (MPIPlusX, §4), and the finalisation
// (sqrt(s/N) for WRMS) written to device memory and the pinned host slot.
//
// Fused ops (SUNDIALS fused vector ops, DESIGN R1/R4): one pass over the
// inputs for up to 8 vectors per launch.

#include <cmath>
#include <cstring>

#include "sunbw_device.cuh"
#include "sunbw_internal.h"

namespace {

using sunbw::d4;
using sunbw::ld4;
using sunbw::st4;
using sunbw::Split;
using sunbw::split_for;
constexpr int kU = sunbw::kU;


// Kernels holding several 32-B vectors per operand in registers (reductions,
// fused multi-vector ops) are compiled for 256-thread CTAs: a 1024-thread
// bound would cap them at 64 registers and spill.  A larger policy block
// size is clamped for them.
constexpr int kMaxBlockWide = 256;

// launch configuration from the vector's execution policy
inline sunbw::LaunchCfg stream_cfg(SUNBW_Context ctx, const _N_Vector* pol,
                                   int64_t work_items, int max_block = 1024) {
  int block = pol ? pol->block : 256;
  if (block > max_block) block = max_block;
  int64_t need = (work_items + (int64_t)block * kU - 1) / ((int64_t)block * kU);
  if (need < 1) need = 1;
  int64_t grid;
  if (pol && pol->policy == SUNBW_POLICY_THREAD_DIRECT) {
    grid = (work_items + block - 1) / block;               // one item per thread
    if (grid < 1) grid = 1;
    if (grid > 0x7fffffff) grid = 0x7fffffff;
  } else {
    int64_t cap = pol && pol->grid > 0 ? pol->grid
                                       : (int64_t)ctx->nsm * (2048 / block);
    grid = need < cap ? need : cap;
  }
  return {block, (int)grid};
}

// ------------------------------------------------------------ streaming
template <int NIN, int NOUT>
struct SArgs {
  const double* in[NIN > 0 ? NIN : 1];
  double* out[NOUT];
};

struct OpLinearSum {
  double a, b;
  __device__ void operator()(const double* x, double* z) const {
    z[0] = __dadd_rn(__dmul_rn(a, x[0]), __dmul_rn(b, x[1]));
  }
};
struct OpScale {
  double c;
  __device__ void operator()(const double* x, double* z) const { z[0] = __dmul_rn(c, x[0]); }
};
struct OpProd {
  __device__ void operator()(const double* x, double* z) const { z[0] = __dmul_rn(x[0], x[1]); }
};
struct OpDiv {
  __device__ void operator()(const double* x, double* z) const { z[0] = __ddiv_rn(x[0], x[1]); }
};
struct OpConst {
  double c;
  __device__ void operator()(const double*, double* z) const { z[0] = c; }
};
struct OpAbs {
  __device__ void operator()(const double* x, double* z) const { z[0] = fabs(x[0]); }
};
struct OpInv {
  __device__ void operator()(const double* x, double* z) const { z[0] = __drcp_rn(x[0]); }
};
struct OpAddConst {
  double b;
  __device__ void operator()(const double* x, double* z) const { z[0] = __dadd_rn(x[0], b); }
};

template <class Op, int NIN, int NOUT>
__device__ __forceinline__ void stream_scalar(const SArgs<NIN, NOUT>& a, int64_t i, const Op& op) {
  double xin[NIN > 0 ? NIN : 1], zout[NOUT];
#pragma unroll
  for (int k = 0; k < NIN; ++k) xin[k] = a.in[k][i];
  op(xin, zout);
#pragma unroll
  for (int k = 0; k < NOUT; ++k) a.out[k][i] = zout[k];
}

template <class Op, int NIN, int NOUT>
__global__ void __launch_bounds__(1024) k_stream(SArgs<NIN, NOUT> a, int64_t n, Split sp, Op op) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < sp.head; i += nth) stream_scalar<Op, NIN, NOUT>(a, i, op);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) stream_scalar<Op, NIN, NOUT>(a, i, op);
  // single-input ops keep as many 32-B loads in flight per thread as the
  // two-input ones
  constexpr int U = NIN <= 1 ? 2 * kU : kU;
  for (int64_t v0 = tid; v0 < sp.nvec; v0 += nth * U) {
    d4 in[U][NIN > 0 ? NIN : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) {
#pragma unroll
        for (int k = 0; k < NIN; ++k) in[u][k] = ld4(a.in[k] + sp.head + 4 * v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) {
        d4 out[NOUT];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double xin[NIN > 0 ? NIN : 1], zout[NOUT];
#pragma unroll
          for (int k = 0; k < NIN; ++k) xin[k] = in[u][k].v[l];
          op(xin, zout);
#pragma unroll
          for (int k = 0; k < NOUT; ++k) out[k].v[l] = zout[k];
        }
#pragma unroll
        for (int k = 0; k < NOUT; ++k) st4(a.out[k] + sp.head + 4 * v, out[k]);
      }
    }
  }
}

template <class Op, int NIN, int NOUT>
int launch_stream(SUNBW_Context ctx, const _N_Vector* pol, int64_t n, SArgs<NIN, NOUT> a, Op op) {
  if (n <= 0) return 0;
  const double* ptrs[NIN + NOUT > 0 ? NIN + NOUT : 1];
  for (int k = 0; k < NIN; ++k) ptrs[k] = a.in[k];
  for (int k = 0; k < NOUT; ++k) ptrs[NIN + k] = a.out[k];
  Split sp = split_for(n, ptrs, NIN + NOUT);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  sunbw::LaunchCfg cfg = stream_cfg(ctx, pol, items);
  k_stream<Op, NIN, NOUT><<<cfg.grid, cfg.block, 0, ctx->stream>>>(a, n, sp, op);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

// ----------------------------------------------------------- reductions
// Per-element term and combine rule of each reduction kind.
template <int KIND>
struct RedTraits;
template <>
struct RedTraits<sunbw::RK_DOT> {
  static constexpr int NIN = 2;
  __device__ static double init() { return 0.0; }
  __device__ static double acc(double s, const double* x) { return __fma_rn(x[0], x[1], s); }
  __device__ static double comb(double a, double b) { return __dadd_rn(a, b); }
};
template <>
struct RedTraits<sunbw::RK_WSQR> {
  static constexpr int NIN = 2;
  __device__ static double init() { return 0.0; }
  __device__ static double acc(double s, const double* x) {
    double p = __dmul_rn(x[0], x[1]);
    return __fma_rn(p, p, s);
  }
  __device__ static double comb(double a, double b) { return __dadd_rn(a, b); }
};
template <>
struct RedTraits<sunbw::RK_WSQR_MASK> {
  static constexpr int NIN = 3;
  __device__ static double init() { return 0.0; }
  __device__ static double acc(double s, const double* x) {
    double p = __dmul_rn(x[0], x[1]);
    return x[2] > 0.0 ? __fma_rn(p, p, s) : s;
  }
  __device__ static double comb(double a, double b) { return __dadd_rn(a, b); }
};
template <>
struct RedTraits<sunbw::RK_MAXABS> {
  static constexpr int NIN = 1;
  __device__ static double init() { return 0.0; }
  __device__ static double acc(double s, const double* x) {
    double a = fabs(x[0]);
    return a > s ? a : s;                 // NaN never selected (R9)
  }
  __device__ static double comb(double a, double b) { return b > a ? b : a; }
};
template <>
struct RedTraits<sunbw::RK_MIN> {
  static constexpr int NIN = 1;
  __device__ static double init() { return INFINITY; }
  __device__ static double acc(double s, const double* x) { return x[0] < s ? x[0] : s; }
  __device__ static double comb(double a, double b) { return b < a ? b : a; }
};

template <class T>
__device__ __forceinline__ double block_reduce(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = T::comb(v, __shfl_xor_sync(0xffffffffu, v, o));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();                                   // sh reuse across calls
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < nw ? sh[l] : T::init();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = T::comb(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;                                          // valid in thread 0
}

struct RArgs {
  const double* in[3];
};

template <int KIND>
__global__ void __launch_bounds__(kMaxBlockWide) k_reduce(RArgs a, int64_t n, Split sp, double* partials) {
  using T = RedTraits<KIND>;
  constexpr int NIN = T::NIN;
  __shared__ double sh[32];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double s[kU][4];
#pragma unroll
  for (int u = 0; u < kU; ++u)
#pragma unroll
    for (int l = 0; l < 4; ++l) s[u][l] = T::init();
  double x[NIN];
  for (int64_t i = tid; i < sp.head; i += nth) {
#pragma unroll
    for (int k = 0; k < NIN; ++k) x[k] = a.in[k][i];
    s[0][0] = T::acc(s[0][0], x);
  }
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) {
#pragma unroll
    for (int k = 0; k < NIN; ++k) x[k] = a.in[k][i];
    s[0][1] = T::acc(s[0][1], x);
  }
  for (int64_t v0 = tid; v0 < sp.nvec; v0 += nth * kU) {
    d4 in[kU][NIN];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) {
#pragma unroll
        for (int k = 0; k < NIN; ++k) in[u][k] = ld4(a.in[k] + sp.head + 4 * v);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
#pragma unroll
          for (int k = 0; k < NIN; ++k) x[k] = in[u][k].v[l];
          s[u][l] = T::acc(s[u][l], x);
        }
      }
    }
  }
  double t = T::init();
#pragma unroll
  for (int u = 0; u < kU; ++u)
#pragma unroll
    for (int l = 0; l < 4; ++l) t = T::comb(t, s[u][l]);
  t = block_reduce<T>(t, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// Fold nparts partials (per output column j < nv, stride nv) in fixed order;
// optionally finalise.  One CTA.
template <class T>
__global__ void k_fold(const double* partials, int nparts, int nv, int fin, double nglobal,
                       double* d_out, double* h_out) {
  __shared__ double sh[32];
  for (int j = 0; j < nv; ++j) {
    double t = T::init();
    for (int p = threadIdx.x; p < nparts; p += blockDim.x) t = T::comb(t, partials[(int64_t)p * nv + j]);
    t = block_reduce<T>(t, sh);
    if (threadIdx.x == 0) {
      if (fin == sunbw::RF_WRMS) t = __dsqrt_rn(__ddiv_rn(t, nglobal));
      d_out[j] = t;
      if (h_out) h_out[j] = t;
    }
  }
}

template <class T>
__global__ void k_finalize(const double* in, int nv, int fin, double nglobal, double* d_out,
                           double* h_out) {
  int j = threadIdx.x;
  if (j >= nv) return;
  double t = in[j];
  if (fin == sunbw::RF_WRMS) t = __dsqrt_rn(__ddiv_rn(t, nglobal));
  d_out[j] = t;
  if (h_out) h_out[j] = t;
}

inline int reduce_grid(SUNBW_Context ctx, const _N_Vector* pol, int64_t items, int block) {
  int64_t need = (items + (int64_t)block * kU - 1) / ((int64_t)block * kU);
  if (need < 1) need = 1;
  int64_t cap = (int64_t)ctx->nsm * (2048 / block);
  if (pol && pol->grid > 0) cap = pol->grid;
  int64_t g = need < cap ? need : cap;
  if (g > SUNBW_Context_::kPartialsCap / 8) g = SUNBW_Context_::kPartialsCap / 8;
  return (int)g;
}

template <int KIND>
int launch_reduce(SUNBW_Context ctx, const _N_Vector* pol, int64_t n, RArgs a, sunbw::RedFinal fin,
                  int64_t nglobal, double* d_out, double* h_out, bool global) {
  using T = RedTraits<KIND>;
  int block = pol ? pol->reduce_block : 256;
  if (block > kMaxBlockWide) block = kMaxBlockWide;
  Split sp = split_for(n, a.in, T::NIN);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  int grid = reduce_grid(ctx, pol, items, block);
  if (n <= 0) grid = 1;
  k_reduce<KIND><<<grid, block, 0, ctx->stream>>>(a, n, sp, ctx->d_partials);
  ctx->launches++;
  bool comm = global && ctx->comm && ctx->comm->nranks > 1;
  RedOp rop = KIND == sunbw::RK_MAXABS ? RED_MAX : (KIND == sunbw::RK_MIN ? RED_MIN : RED_SUM);
  if (!comm) {
    k_fold<T><<<1, 256, 0, ctx->stream>>>(ctx->d_partials, grid, 1, (int)fin, (double)nglobal, d_out, h_out);
    ctx->launches++;
    return ctx_check_launch(ctx);
  }
  double* tmp = ctx->d_red + (SUNBW_Context_::kRedSlots - 16);
  k_fold<T><<<1, 256, 0, ctx->stream>>>(ctx->d_partials, grid, 1, sunbw::RF_NONE, 1.0, tmp, nullptr);
  ctx->launches++;
  if (ctx_check_launch(ctx)) return SUNBW_ERR_CUDA;
  int e = ctx->comm->allreduce(tmp, 1, rop, ctx->stream);
  if (e) return ctx_set_err(ctx, e);
  k_finalize<T><<<1, 32, 0, ctx->stream>>>(tmp, 1, (int)fin, (double)nglobal, d_out, h_out);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

// ------------------------------------------------------------------ fused
constexpr int kMaxNV = 8;

struct FusedArgs {
  const double* X[kMaxNV];
  double* Z[kMaxNV];
  double c[kMaxNV];
  const double* x;
  double* z;
};

// z = [z +] Σ_j c_j X_j, sequential in j (bit-identical to the definition).
template <int NV, bool ACC>
__device__ __forceinline__ double lc_elem(const double* xin, double zin, const double* c) {
  double acc = ACC ? __dadd_rn(zin, __dmul_rn(c[0], xin[0])) : __dmul_rn(c[0], xin[0]);
#pragma unroll
  for (int j = 1; j < NV; ++j) acc = __dadd_rn(acc, __dmul_rn(c[j], xin[j]));
  return acc;
}

template <int NV, bool ACC>
__global__ void __launch_bounds__(kMaxBlockWide) k_lincomb(FusedArgs a, int64_t n, Split sp) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double xin[NV];
  auto scalar = [&](int64_t i) {
#pragma unroll
    for (int j = 0; j < NV; ++j) xin[j] = a.X[j][i];
    double zi = ACC ? a.z[i] : 0.0;
    a.z[i] = lc_elem<NV, ACC>(xin, zi, a.c);
  };
  for (int64_t i = tid; i < sp.head; i += nth) scalar(i);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) scalar(i);
  for (int64_t v = tid; v < sp.nvec; v += nth) {
    d4 in[NV];
    d4 zin;
    const int64_t off = sp.head + 4 * v;
#pragma unroll
    for (int j = 0; j < NV; ++j) in[j] = ld4(a.X[j] + off);
    if (ACC) zin = ld4(a.z + off);
    d4 out;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
#pragma unroll
      for (int j = 0; j < NV; ++j) xin[j] = in[j].v[l];
      out.v[l] = lc_elem<NV, ACC>(xin, ACC ? zin.v[l] : 0.0, a.c);
    }
    st4(a.z + off, out);
  }
}

// Z_j = a_j x + Y_j
template <int NV>
__global__ void __launch_bounds__(kMaxBlockWide) k_scaleaddmulti(FusedArgs a, int64_t n, Split sp) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  auto scalar = [&](int64_t i) {
    double xi = a.x[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) a.Z[j][i] = __dadd_rn(__dmul_rn(a.c[j], xi), a.X[j][i]);
  };
  for (int64_t i = tid; i < sp.head; i += nth) scalar(i);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) scalar(i);
  for (int64_t v = tid; v < sp.nvec; v += nth) {
    const int64_t off = sp.head + 4 * v;
    d4 xv = ld4(a.x + off);
    d4 yv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) yv[j] = ld4(a.X[j] + off);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      d4 o;
#pragma unroll
      for (int l = 0; l < 4; ++l) o.v[l] = __dadd_rn(__dmul_rn(a.c[j], xv.v[l]), yv[j].v[l]);
      st4(a.Z[j] + off, o);
    }
  }
}

// partial dots d_j = x·Y_j, one partial per CTA per j (stride NV)
template <int NV>
__global__ void __launch_bounds__(kMaxBlockWide) k_dotmulti(FusedArgs a, int64_t n, Split sp, double* partials) {
  using T = RedTraits<sunbw::RK_DOT>;
  __shared__ double sh[32];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  double s[NV][2];
#pragma unroll
  for (int j = 0; j < NV; ++j) s[j][0] = s[j][1] = 0.0;
  auto scalar = [&](int64_t i) {
    double xi = a.x[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) s[j][0] = __fma_rn(xi, a.X[j][i], s[j][0]);
  };
  for (int64_t i = tid; i < sp.head; i += nth) scalar(i);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) scalar(i);
  for (int64_t v = tid; v < sp.nvec; v += nth) {
    const int64_t off = sp.head + 4 * v;
    d4 xv = ld4(a.x + off);
    d4 yv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) yv[j] = ld4(a.X[j] + off);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      s[j][0] = __fma_rn(xv.v[0], yv[j].v[0], s[j][0]);
      s[j][1] = __fma_rn(xv.v[1], yv[j].v[1], s[j][1]);
      s[j][0] = __fma_rn(xv.v[2], yv[j].v[2], s[j][0]);
      s[j][1] = __fma_rn(xv.v[3], yv[j].v[3], s[j][1]);
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double t = block_reduce<T>(__dadd_rn(s[j][0], s[j][1]), sh);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.x * NV + j] = t;
  }
}

int lincomb_chunk(SUNBW_Context ctx, const _N_Vector* pol, int64_t n, int nv, bool acc,
                  FusedArgs& a) {
  const double* ptrs[kMaxNV + 1];
  for (int j = 0; j < nv; ++j) ptrs[j] = a.X[j];
  ptrs[nv] = a.z;
  Split sp = split_for(n, ptrs, nv + 1);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  sunbw::LaunchCfg cfg = stream_cfg(ctx, pol, items * kU, kMaxBlockWide);   // one vector per thread-iteration
  dim3 g(cfg.grid), b(cfg.block);
  cudaStream_t s = ctx->stream;
#define LC_CASE(NV)                                                        \
  case NV:                                                                 \
    if (acc) k_lincomb<NV, true><<<g, b, 0, s>>>(a, n, sp);                \
    else k_lincomb<NV, false><<<g, b, 0, s>>>(a, n, sp);                   \
    break;
  switch (nv) {
    LC_CASE(1) LC_CASE(2) LC_CASE(3) LC_CASE(4) LC_CASE(5) LC_CASE(6) LC_CASE(7) LC_CASE(8)
    default: return SUNBW_ERR_ARG;
  }
#undef LC_CASE
  ctx->launches++;
  return ctx_check_launch(ctx);
}

int scaleaddmulti_chunk(SUNBW_Context ctx, const _N_Vector* pol, int64_t n, int nv, FusedArgs& a) {
  const double* ptrs[2 * kMaxNV + 1];
  for (int j = 0; j < nv; ++j) { ptrs[2 * j] = a.X[j]; ptrs[2 * j + 1] = a.Z[j]; }
  ptrs[2 * nv] = a.x;
  Split sp = split_for(n, ptrs, 2 * nv + 1);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  sunbw::LaunchCfg cfg = stream_cfg(ctx, pol, items * kU, kMaxBlockWide);
  dim3 g(cfg.grid), b(cfg.block);
  cudaStream_t s = ctx->stream;
#define SAM_CASE(NV) case NV: k_scaleaddmulti<NV><<<g, b, 0, s>>>(a, n, sp); break;
  switch (nv) {
    SAM_CASE(1) SAM_CASE(2) SAM_CASE(3) SAM_CASE(4) SAM_CASE(5) SAM_CASE(6) SAM_CASE(7) SAM_CASE(8)
    default: return SUNBW_ERR_ARG;
  }
#undef SAM_CASE
  ctx->launches++;
  return ctx_check_launch(ctx);
}

int dotmulti_chunk(SUNBW_Context ctx, const _N_Vector* pol, int64_t n, int nv, FusedArgs& a,
                   double* d_out_local) {
  const double* ptrs[kMaxNV + 1];
  for (int j = 0; j < nv; ++j) ptrs[j] = a.X[j];
  ptrs[nv] = a.x;
  Split sp = split_for(n, ptrs, nv + 1);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  int block = pol ? pol->reduce_block : 256;
  if (block > kMaxBlockWide) block = kMaxBlockWide;
  int grid = reduce_grid(ctx, pol, items * kU, block);
  dim3 g(grid), b(block);
  cudaStream_t s = ctx->stream;
#define DPM_CASE(NV) case NV: k_dotmulti<NV><<<g, b, 0, s>>>(a, n, sp, ctx->d_partials); break;
  switch (nv) {
    DPM_CASE(1) DPM_CASE(2) DPM_CASE(3) DPM_CASE(4) DPM_CASE(5) DPM_CASE(6) DPM_CASE(7) DPM_CASE(8)
    default: return SUNBW_ERR_ARG;
  }
#undef DPM_CASE
  k_fold<RedTraits<sunbw::RK_DOT>><<<1, 256, 0, s>>>(ctx->d_partials, grid, nv, sunbw::RF_NONE, 1.0,
                                                      d_out_local, nullptr);
  ctx->launches += 2;
  return ctx_check_launch(ctx);
}

__global__ void k_flag_nonpositive(const double* v, int* flag) {
  if (!(v[0] > 0.0)) *flag = 1;
}

}  // namespace

// =========================================================== internal API
namespace sunbw {

int linear_sum(SUNBW_Context ctx, int64_t n, double a, const double* x, double b,
               const double* y, double* z, const _N_Vector* pol) {
  SArgs<2, 1> s{{x, y}, {z}};
  return launch_stream(ctx, pol, n, s, OpLinearSum{a, b});
}
int scale(SUNBW_Context ctx, int64_t n, double c, const double* x, double* z, const _N_Vector* pol) {
  SArgs<1, 1> s{{x}, {z}};
  return launch_stream(ctx, pol, n, s, OpScale{c});
}
int abs_(SUNBW_Context ctx, int64_t n, const double* x, double* z, const _N_Vector* pol) {
  SArgs<1, 1> s{{x}, {z}};
  return launch_stream(ctx, pol, n, s, OpAbs{});
}
int add_const(SUNBW_Context ctx, int64_t n, const double* x, double b, double* z,
              const _N_Vector* pol) {
  SArgs<1, 1> s{{x}, {z}};
  return launch_stream(ctx, pol, n, s, OpAddConst{b});
}
int inv(SUNBW_Context ctx, int64_t n, const double* x, double* z, const _N_Vector* pol) {
  SArgs<1, 1> s{{x}, {z}};
  return launch_stream(ctx, pol, n, s, OpInv{});
}

int linear_combination(SUNBW_Context ctx, int64_t n, int nv, const double* c,
                       const double* const* X, double* z, const _N_Vector* pol) {
  if (nv < 1) return ctx_set_err(ctx, SUNBW_ERR_ARG);
  if (n <= 0) return 0;
  for (int j0 = 0; j0 < nv; j0 += kMaxNV) {
    int k = nv - j0 < kMaxNV ? nv - j0 : kMaxNV;
    FusedArgs a{};
    for (int j = 0; j < k; ++j) { a.X[j] = X[j0 + j]; a.c[j] = c[j0 + j]; }
    a.z = z;
    int e = lincomb_chunk(ctx, pol, n, k, j0 > 0, a);
    if (e) return e;
  }
  return 0;
}

int reduce(SUNBW_Context ctx, RedKind kind, RedFinal fin, int64_t n, int64_t nglobal,
           const double* x, const double* y, const double* id, double* d_out,
           double* h_out, bool global, const _N_Vector* pol) {
  RArgs a{{x, y, id}};
  switch (kind) {
    case RK_DOT: return launch_reduce<RK_DOT>(ctx, pol, n, a, fin, nglobal, d_out, h_out, global);
    case RK_WSQR: return launch_reduce<RK_WSQR>(ctx, pol, n, a, fin, nglobal, d_out, h_out, global);
    case RK_WSQR_MASK:
      return launch_reduce<RK_WSQR_MASK>(ctx, pol, n, a, fin, nglobal, d_out, h_out, global);
    case RK_MAXABS: return launch_reduce<RK_MAXABS>(ctx, pol, n, a, fin, nglobal, d_out, h_out, global);
    case RK_MIN: return launch_reduce<RK_MIN>(ctx, pol, n, a, fin, nglobal, d_out, h_out, global);
  }
  return SUNBW_ERR_ARG;
}

int dot_multi(SUNBW_Context ctx, int64_t n, int nv, const double* x, const double* const* Y,
              double* d_out, double* h_out, bool global, const _N_Vector* pol) {
  if (nv < 1 || nv > SUNBW_Context_::kRedSlots - 32) return ctx_set_err(ctx, SUNBW_ERR_ARG);
  for (int j0 = 0; j0 < nv; j0 += kMaxNV) {
    int k = nv - j0 < kMaxNV ? nv - j0 : kMaxNV;
    FusedArgs a{};
    for (int j = 0; j < k; ++j) a.X[j] = Y[j0 + j];
    a.x = x;
    int e = dotmulti_chunk(ctx, pol, n, k, a, d_out + j0);
    if (e) return e;
  }
  bool comm = global && ctx->comm && ctx->comm->nranks > 1;
  if (comm) {
    int e = ctx->comm->allreduce(d_out, nv, RED_SUM, ctx->stream);
    if (e) return ctx_set_err(ctx, e);
  }
  if (h_out) {
    k_finalize<RedTraits<RK_DOT>><<<1, 256, 0, ctx->stream>>>(d_out, nv, RF_NONE, 1.0, d_out, h_out);
    ctx->launches++;
  }
  return ctx_check_launch(ctx);
}

int flag_nonpositive(SUNBW_Context ctx, const double* d_val, int* d_flag) {
  k_flag_nonpositive<<<1, 1, 0, ctx->stream>>>(d_val, d_flag);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

}  // namespace sunbw

// ================================================================ C ABI
namespace {

int64_t global_length(SUNBW_Context ctx, int64_t local, int* err) {
  *err = 0;
  if (!ctx->comm || ctx->comm->nranks == 1) return local;
  // collective: sum of local lengths (exact in fp64 below 2^53)
  double* tmp = ctx->d_red + (SUNBW_Context_::kRedSlots - 8);
  double v = (double)local;
  if (cudaMemcpyAsync(tmp, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) {
    *err = SUNBW_ERR_CUDA;
    return -1;
  }
  int e = ctx->comm->allreduce(tmp, 1, RED_SUM, ctx->stream);
  if (e) { *err = e; return -1; }
  if (cudaMemcpyAsync(&v, tmp, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    *err = SUNBW_ERR_CUDA;
    return -1;
  }
  return (int64_t)v;
}

N_Vector make_vec(SUNBW_Context ctx, int64_t n, double* d, bool owned, int64_t nglob) {
  auto* v = new _N_Vector();
  v->ctx = ctx;
  v->local_len = n;
  v->global_len = nglob;
  v->d = d;
  v->owned = owned;
  return v;
}

bool compat(N_Vector a, N_Vector b) {
  if (!a || !b) return false;
  if (a->ctx != b->ctx) { ctx_set_err(a->ctx, SUNBW_ERR_CONTEXT); return false; }
  if (a->local_len != b->local_len) { ctx_set_err(a->ctx, SUNBW_ERR_LENGTH); return false; }
  return true;
}

}  // namespace

extern "C" N_Vector N_VNew_B200(SUNBW_Context ctx, int64_t n) {
  if (!ctx || n < 0) return nullptr;
  int err;
  int64_t ng = global_length(ctx, n, &err);
  if (err) { ctx_set_err(ctx, err); return nullptr; }
  double* d = nullptr;
  if (n > 0 && cudaMallocAsync(&d, sizeof(double) * n, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    ctx_set_err(ctx, SUNBW_ERR_MEM);
    return nullptr;
  }
  return make_vec(ctx, n, d, true, ng);
}

extern "C" N_Vector N_VMake_B200(SUNBW_Context ctx, int64_t n, double* d) {
  if (!ctx || n < 0 || (n > 0 && !d) || ((uintptr_t)d & 7)) return nullptr;
  int err;
  int64_t ng = global_length(ctx, n, &err);
  if (err) { ctx_set_err(ctx, err); return nullptr; }
  return make_vec(ctx, n, d, false, ng);
}

extern "C" N_Vector N_VClone(N_Vector w) {
  if (!w) return nullptr;
  double* d = nullptr;
  if (w->local_len > 0 &&
      cudaMallocAsync(&d, sizeof(double) * w->local_len, w->ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    ctx_set_err(w->ctx, SUNBW_ERR_MEM);
    return nullptr;
  }
  N_Vector v = make_vec(w->ctx, w->local_len, d, true, w->global_len);
  v->policy = w->policy; v->block = w->block; v->grid = w->grid; v->reduce_block = w->reduce_block;
  return v;
}

extern "C" void N_VDestroy(N_Vector v) {
  if (!v) return;
  if (v->owned && v->d) cudaFreeAsync(v->d, v->ctx->stream);
  delete v;
}

extern "C" double* N_VGetDeviceArrayPointer_B200(N_Vector v) { return v ? v->d : nullptr; }

extern "C" int N_VSetDeviceArrayPointer_B200(N_Vector v, double* d) {
  if (!v || v->owned || (v->local_len > 0 && !d) || ((uintptr_t)d & 7)) return SUNBW_ERR_ARG;
  v->d = d;
  return 0;
}

extern "C" int64_t N_VGetLength(N_Vector v) { return v ? v->global_len : -1; }
extern "C" int64_t N_VGetLocalLength(N_Vector v) { return v ? v->local_len : -1; }

extern "C" int N_VSetKernelExecPolicy_B200(N_Vector v, int policy, int block, int grid,
                                           int reduce_block) {
  if (!v) return SUNBW_ERR_ARG;
  if (policy != SUNBW_POLICY_GRID_STRIDE && policy != SUNBW_POLICY_THREAD_DIRECT) return SUNBW_ERR_ARG;
  if (block == 0) block = 256;
  if (reduce_block == 0) reduce_block = 256;
  if (block < 32 || block > 1024 || (block & 31) || reduce_block < 32 || reduce_block > 1024 ||
      (reduce_block & 31) || grid < 0)
    return SUNBW_ERR_ARG;
  v->policy = policy; v->block = block; v->grid = grid; v->reduce_block = reduce_block;
  return 0;
}

// ---------------------------------------------------------- streaming ABI
extern "C" void N_VLinearSum(double a, N_Vector x, double b, N_Vector y, N_Vector z) {
  if (!compat(x, y) || !compat(x, z)) return;
  sunbw::linear_sum(z->ctx, z->local_len, a, x->d, b, y->d, z->d, z);
}
extern "C" void N_VScale(double c, N_Vector x, N_Vector z) {
  if (!compat(x, z)) return;
  sunbw::scale(z->ctx, z->local_len, c, x->d, z->d, z);
}
extern "C" void N_VProd(N_Vector x, N_Vector y, N_Vector z) {
  if (!compat(x, y) || !compat(x, z)) return;
  SArgs<2, 1> s{{x->d, y->d}, {z->d}};
  launch_stream(z->ctx, z, z->local_len, s, OpProd{});
}
extern "C" void N_VDiv(N_Vector x, N_Vector y, N_Vector z) {
  if (!compat(x, y) || !compat(x, z)) return;
  SArgs<2, 1> s{{x->d, y->d}, {z->d}};
  launch_stream(z->ctx, z, z->local_len, s, OpDiv{});
}
extern "C" void N_VConst(double c, N_Vector z) {
  if (!z) return;
  SArgs<0, 1> s{{nullptr}, {z->d}};
  launch_stream(z->ctx, z, z->local_len, s, OpConst{c});
}
extern "C" void N_VAbs(N_Vector x, N_Vector z) {
  if (!compat(x, z)) return;
  sunbw::abs_(z->ctx, z->local_len, x->d, z->d, z);
}
extern "C" void N_VInv(N_Vector x, N_Vector z) {
  if (!compat(x, z)) return;
  sunbw::inv(z->ctx, z->local_len, x->d, z->d, z);
}
extern "C" void N_VAddConst(N_Vector x, double b, N_Vector z) {
  if (!compat(x, z)) return;
  sunbw::add_const(z->ctx, z->local_len, x->d, b, z->d, z);
}

// ---------------------------------------------------------- reduction ABI
namespace {

double host_reduce(N_Vector x, sunbw::RedKind kind, sunbw::RedFinal fin, const double* y,
                   const double* id, bool global) {
  SUNBW_Context ctx = x->ctx;
  bool needs_n = fin == sunbw::RF_WRMS || kind == sunbw::RK_MAXABS || kind == sunbw::RK_MIN;
  if (global && needs_n && x->global_len == 0) {      // N >= 1
    ctx_set_err(ctx, SUNBW_ERR_EMPTY);
    return NAN;
  }
  int e = sunbw::reduce(ctx, kind, fin, x->local_len, x->global_len, x->d, y, id, ctx->d_red,
                        ctx->h_slot_dev, global, x);
  if (e) return NAN;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    ctx_set_err(ctx, SUNBW_ERR_CUDA);
    return NAN;
  }
  return ((volatile double*)ctx->h_slot)[0];
}

}  // namespace

extern "C" double N_VDotProd(N_Vector x, N_Vector y) {
  if (!compat(x, y)) return NAN;
  return host_reduce(x, sunbw::RK_DOT, sunbw::RF_NONE, y->d, nullptr, true);
}
extern "C" double N_VDotProdLocal(N_Vector x, N_Vector y) {
  if (!compat(x, y)) return NAN;
  return host_reduce(x, sunbw::RK_DOT, sunbw::RF_NONE, y->d, nullptr, false);
}
extern "C" double N_VWSqrSumLocal(N_Vector x, N_Vector w) {
  if (!compat(x, w)) return NAN;
  return host_reduce(x, sunbw::RK_WSQR, sunbw::RF_NONE, w->d, nullptr, false);
}
extern "C" double N_VWrmsNorm(N_Vector x, N_Vector w) {
  if (!compat(x, w)) return NAN;
  return host_reduce(x, sunbw::RK_WSQR, sunbw::RF_WRMS, w->d, nullptr, true);
}
extern "C" double N_VWrmsNormMask(N_Vector x, N_Vector w, N_Vector id) {
  if (!compat(x, w) || !compat(x, id)) return NAN;
  return host_reduce(x, sunbw::RK_WSQR_MASK, sunbw::RF_WRMS, w->d, id->d, true);
}
extern "C" double N_VMaxNorm(N_Vector x) {
  if (!x) return NAN;
  return host_reduce(x, sunbw::RK_MAXABS, sunbw::RF_NONE, nullptr, nullptr, true);
}
extern "C" double N_VMin(N_Vector x) {
  if (!x) return NAN;
  return host_reduce(x, sunbw::RK_MIN, sunbw::RF_NONE, nullptr, nullptr, true);
}

// ---------------------------------------------------------------- fused ABI
extern "C" int N_VLinearCombination(int nv, const double* c, N_Vector* X, N_Vector z) {
  if (nv < 1 || !c || !X || !z) return -1;
  std::vector<const double*> ptrs(nv);
  for (int j = 0; j < nv; ++j) {
    if (!compat(z, X[j])) return -1;
    ptrs[j] = X[j]->d;
  }
  // with more than one chunk, z may only alias X[0] (later chunks re-read X)
  for (int j = kMaxNV; j < nv; ++j)
    if (X[j]->d == z->d) return ctx_set_err(z->ctx, SUNBW_ERR_ARG), -1;
  return sunbw::linear_combination(z->ctx, z->local_len, nv, c, ptrs.data(), z->d, z) ? -1 : 0;
}

extern "C" int N_VScaleAddMulti(int nv, const double* a, N_Vector x, N_Vector* Y, N_Vector* Z) {
  if (nv < 1 || !a || !x || !Y || !Z) return -1;
  for (int j = 0; j < nv; ++j)
    if (!compat(x, Y[j]) || !compat(x, Z[j])) return -1;
  for (int j0 = 0; j0 < nv; j0 += kMaxNV) {
    int k = nv - j0 < kMaxNV ? nv - j0 : kMaxNV;
    FusedArgs f{};
    for (int j = 0; j < k; ++j) { f.X[j] = Y[j0 + j]->d; f.Z[j] = Z[j0 + j]->d; f.c[j] = a[j0 + j]; }
    f.x = x->d;
    if (x->local_len > 0 && scaleaddmulti_chunk(x->ctx, x, x->local_len, k, f)) return -1;
  }
  return 0;
}

extern "C" int N_VDotProdMulti(int nv, N_Vector x, N_Vector* Y, double* dots) {
  if (nv < 1 || !x || !Y || !dots || nv > 64) return -1;
  std::vector<const double*> ptrs(nv);
  for (int j = 0; j < nv; ++j) {
    if (!compat(x, Y[j])) return -1;
    ptrs[j] = Y[j]->d;
  }
  SUNBW_Context ctx = x->ctx;
  if (sunbw::dot_multi(ctx, x->local_len, nv, x->d, ptrs.data(), ctx->d_red, ctx->h_slot_dev, true, x))
    return -1;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA), -1;
  for (int j = 0; j < nv; ++j) dots[j] = ((volatile double*)ctx->h_slot)[j];
  return 0;
}
