// blockdiag.cu — low-storage block-diagonal matrix and the batched LU solver.
//
// Matrix (§5): nblocks square m×m blocks sharing one pattern; the
// shared pattern of the Brusselator Newton matrix (§7) is a full 3×3
// block, so values are stored dense, [G][m][m], row-major within a block.
//
// Solver (the role of SUNLinearSolver_cuSolverSp_batchQR, §5, and of
// the demo's per-cell 3×3 block solves, §7): one thread owns one
// block in registers; a CTA stages its blocks through shared memory so that
// every global access is a fully coalesced, contiguous run (the 72-byte
// blocks would otherwise be read with a 72-byte lane stride).  Partial
// pivoting with the first-maximum rule; every operation an explicit RN
// intrinsic (no contraction), matching the serial definition bit for bit.
// No tensor cores: 3×3 blocks are not a dense contraction (north star).

#include <cstring>

#include "sunbw_device.cuh"
#include "sunbw_internal.h"
#include "pipeline.cuh"

namespace {

using sunbw::d4;
using sunbw::ld4;
using sunbw::Split;
using sunbw::split_for;
using sunbw::st4;

// blocks per CTA for block size M: keep the staged tile <= 16 KB
template <int M>
__host__ __device__ constexpr int bpc() {
  return M <= 4 ? 128 : (M <= 6 ? 64 : 32);
}

// cooperative contiguous copy global <-> shared (coalesced, 8 B per lane;
// 16 B when both sides are 16-B aligned)
__device__ __forceinline__ void tile_in(double* s, const double* g, int count) {
  if ((((uintptr_t)g) & 15) == 0) {
    const double2* g2 = (const double2*)g;
    double2* s2 = (double2*)s;
    int n2 = count >> 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) s2[i] = __ldcs(g2 + i);
    if ((count & 1) && threadIdx.x == 0) s[count - 1] = g[count - 1];
  } else {
    for (int i = threadIdx.x; i < count; i += blockDim.x) s[i] = __ldcs(g + i);
  }
}

__device__ __forceinline__ void tile_out(double* g, const double* s, int count) {
  if ((((uintptr_t)g) & 15) == 0) {
    double2* g2 = (double2*)g;
    const double2* s2 = (const double2*)s;
    int n2 = count >> 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) g2[i] = s2[i];
    if ((count & 1) && threadIdx.x == 0) g[count - 1] = s[count - 1];
  } else {
    for (int i = threadIdx.x; i < count; i += blockDim.x) g[i] = s[i];
  }
}

// In-register LU with partial pivoting of one M×M block (O6 definition):
// column k: r = first row of max |a_ik|, i >= k; swap rows; l = a_ik/a_kk;
// a_ij -= l a_kj.  A zero pivot marks the block singular and skips the
// column's elimination.  Returns the packed pivot code (3 bits per step).
template <int M>
__device__ __forceinline__ int lu_regs(double (&a)[M][M], bool& singular) {
  int code = 0;
  singular = false;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    int r = k;
    double best = fabs(a[k][k]);
#pragma unroll
    for (int i = k + 1; i < M; ++i) {
      double v = fabs(a[i][k]);
      if (v > best) { best = v; r = i; }
    }
    code |= r << (3 * k);
#pragma unroll
    for (int i = k + 1; i < M; ++i) {
      if (i == r) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
          double t = a[k][j];
          a[k][j] = a[i][j];
          a[i][j] = t;
        }
      }
    }
    double akk = a[k][k];
    if (akk == 0.0) {
      singular = true;
      continue;
    }
#pragma unroll
    for (int i = k + 1; i < M; ++i) {
      double l = __ddiv_rn(a[i][k], akk);
      a[i][k] = l;
#pragma unroll
      for (int j = k + 1; j < M; ++j) a[i][j] = __dsub_rn(a[i][j], __dmul_rn(l, a[k][j]));
    }
  }
  return code;
}

// x = U^{-1} L^{-1} P b (O7 definition), y in registers
template <int M>
__device__ __forceinline__ void lu_solve_regs(const double (&a)[M][M], int code, double (&y)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) {
    int r = (code >> (3 * k)) & 7;
#pragma unroll
    for (int i = k + 1; i < M; ++i) {
      if (i == r) {
        double t = y[k];
        y[k] = y[i];
        y[i] = t;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double s = y[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(a[i][j], y[j]));
    y[i] = s;
  }
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int j = i + 1; j < M; ++j) s = __dsub_rn(s, __dmul_rn(a[i][j], y[j]));
    y[i] = __ddiv_rn(s, a[i][i]);
  }
}

template <int M>
__global__ void __launch_bounds__(bpc<M>()) k_lu_factor(double* A, int32_t* piv, int64_t G,
                                                       unsigned long long* first_singular) {
  constexpr int MM = M * M;
  constexpr int B = bpc<M>();
  __shared__ double s[B * MM];
  for (int64_t g0 = (int64_t)blockIdx.x * B; g0 < G; g0 += (int64_t)gridDim.x * B) {
    int nb = (int)((G - g0) < B ? (G - g0) : B);
    double* gA = A + g0 * MM;
    __syncthreads();
    tile_in(s, gA, nb * MM);
    __syncthreads();
    int t = threadIdx.x;
    if (t < nb) {
      double a[M][M];
#pragma unroll
      for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) a[i][j] = s[t * MM + i * M + j];
      bool sing;
      int code = lu_regs<M>(a, sing);
#pragma unroll
      for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) s[t * MM + i * M + j] = a[i][j];
      piv[g0 + t] = code;
      if (sing) atomicMin(first_singular, (unsigned long long)(g0 + t + 1));
    }
    __syncthreads();
    tile_out(gA, s, nb * MM);
  }
}

template <int M>
__global__ void __launch_bounds__(bpc<M>()) k_lu_solve(const double* LU, const int32_t* piv,
                                                      const double* b, double* x, int64_t G) {
  constexpr int MM = M * M;
  constexpr int B = bpc<M>();
  __shared__ double s[B * MM];
  __shared__ double sb[B * M];
  for (int64_t g0 = (int64_t)blockIdx.x * B; g0 < G; g0 += (int64_t)gridDim.x * B) {
    int nb = (int)((G - g0) < B ? (G - g0) : B);
    __syncthreads();
    tile_in(s, LU + g0 * MM, nb * MM);
    tile_in(sb, b + g0 * M, nb * M);
    __syncthreads();
    int t = threadIdx.x;
    if (t < nb) {
      double a[M][M], y[M];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        y[i] = sb[t * M + i];
#pragma unroll
        for (int j = 0; j < M; ++j) a[i][j] = s[t * MM + i * M + j];
      }
      lu_solve_regs<M>(a, __ldcs(piv + g0 + t), y);
#pragma unroll
      for (int i = 0; i < M; ++i) sb[t * M + i] = y[i];
    }
    __syncthreads();
    tile_out(x + g0 * M, sb, nb * M);
  }
}

template <int M>
__global__ void __launch_bounds__(bpc<M>()) k_block_matvec(const double* A, const double* xv,
                                                          double* yv, int64_t G) {
  constexpr int MM = M * M;
  constexpr int B = bpc<M>();
  __shared__ double s[B * MM];
  __shared__ double sx[B * M];
  for (int64_t g0 = (int64_t)blockIdx.x * B; g0 < G; g0 += (int64_t)gridDim.x * B) {
    int nb = (int)((G - g0) < B ? (G - g0) : B);
    __syncthreads();
    tile_in(s, A + g0 * MM, nb * MM);
    tile_in(sx, xv + g0 * M, nb * M);
    __syncthreads();
    int t = threadIdx.x;
    double r[M];
    if (t < nb) {
#pragma unroll
      for (int i = 0; i < M; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(s[t * MM + i * M + j], sx[t * M + j]));
        r[i] = acc;
      }
    }
    __syncthreads();
    if (t < nb) {
#pragma unroll
      for (int i = 0; i < M; ++i) sx[t * M + i] = r[i];
    }
    __syncthreads();
    tile_out(yv + g0 * M, sx, nb * M);
  }
}

// A <- c A + I: streaming over the flat value array, 256-bit accesses
__global__ void __launch_bounds__(256) k_scale_add_identity(double* A, int64_t n, Split sp, int m,
                                                            double c) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int mm = m * m;
  auto elem = [&](int64_t e, double v) {
    int w = (int)(e % mm);
    double r = __dmul_rn(c, v);
    if (w / m == w % m) r = __dadd_rn(r, 1.0);
    return r;
  };
  for (int64_t i = tid; i < sp.head; i += nth) A[i] = elem(i, A[i]);
  for (int64_t i = sp.tail0 + tid; i < n; i += nth) A[i] = elem(i, A[i]);
  for (int64_t v0 = tid; v0 < sp.nvec; v0 += nth * 2) {
    d4 in[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) in[u] = ld4(A + sp.head + 4 * v);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int64_t v = v0 + u * nth;
      if (v < sp.nvec) {
        int64_t e0 = sp.head + 4 * v;
        d4 o;
#pragma unroll
        for (int l = 0; l < 4; ++l) o.v[l] = elem(e0 + l, in[u].v[l]);
        st4(A + e0, o);
      }
    }
  }
}

inline int grid_for(SUNBW_Context ctx, int64_t G, int B, int occ) {
  int64_t need = (G + B - 1) / B;
  int64_t cap = (int64_t)ctx->nsm * occ;
  int64_t g = need < cap ? need : cap;
  return g < 1 ? 1 : (int)g;
}

// ---- TMA-pipelined variants (pipeline.cuh): every operand tile of T
// blocks is one bulk copy; persistent CTAs, double-buffered.  Used when all
// operands are 16-B aligned (always for library-allocated storage).
template <int M>
__host__ __device__ constexpr int tpc() {
  return M <= 4 ? 128 : 32;
}
constexpr int kStagesLU = 2;

template <int M>
__global__ void __launch_bounds__(tpc<M>()) k_lu_factor_tma(sunbw::pipe::IO<1, 2> io, int64_t G,
                                                           unsigned long long* first_singular) {
  extern __shared__ __align__(128) unsigned char smem[];
  sunbw::pipe::run<tpc<M>(), kStagesLU>(
      io, G, smem, [&](int, int64_t g, const unsigned char** ip, unsigned char** op) {
        const double* ain = reinterpret_cast<const double*>(ip[0]);
        double a[M][M];
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int j = 0; j < M; ++j) a[i][j] = ain[i * M + j];
        bool sing;
        int code = lu_regs<M>(a, sing);
        double* aout = reinterpret_cast<double*>(op[0]);
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int j = 0; j < M; ++j) aout[i * M + j] = a[i][j];
        *reinterpret_cast<int32_t*>(op[1]) = code;
        if (sing) atomicMin(first_singular, (unsigned long long)(g + 1));
      });
}

template <int M>
__global__ void __launch_bounds__(tpc<M>()) k_lu_solve_tma(sunbw::pipe::IO<3, 1> io, int64_t G) {
  extern __shared__ __align__(128) unsigned char smem[];
  sunbw::pipe::run<tpc<M>(), kStagesLU>(
      io, G, smem, [&](int, int64_t, const unsigned char** ip, unsigned char** op) {
        const double* lu = reinterpret_cast<const double*>(ip[0]);
        const int code = *reinterpret_cast<const int32_t*>(ip[1]);
        const double* b = reinterpret_cast<const double*>(ip[2]);
        double a[M][M], y[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          y[i] = b[i];
#pragma unroll
          for (int j = 0; j < M; ++j) a[i][j] = lu[i * M + j];
        }
        lu_solve_regs<M>(a, code, y);
        double* x = reinterpret_cast<double*>(op[0]);
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = y[i];
      });
}

// ---- block inverse by symbolic Gauss-Jordan (the paper's task-local block
// solve; DESIGN R29).  On
// [A | I] without row exchanges; the identity block's structure is
// data-independent, so the "symbolic" skipping of its structural zeros and
// ones is resolved at compile time: at step k row k holds values in columns
// j <= k (B_kk was the structural 1, now p = RN(1/a_kk)), and every other
// row gets column k as -RN(f B_kk) and columns j < k as RN(B_ij - RN(f B_kj)).
template <int M>
__device__ __forceinline__ bool gj_regs(double (&a)[M][M], double (&B)[M][M]) {
  bool sing = false;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    sing |= a[k][k] == 0.0;
    const double p = __drcp_rn(a[k][k]);              // RN(1/a_kk) (IEEE 1/0 = inf)
#pragma unroll
    for (int j = k + 1; j < M; ++j) a[k][j] = __dmul_rn(a[k][j], p);
#pragma unroll
    for (int j = 0; j < k; ++j) B[k][j] = __dmul_rn(B[k][j], p);
    B[k][k] = p;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (i == k) continue;
      const double f = a[i][k];
#pragma unroll
      for (int j = k + 1; j < M; ++j) a[i][j] = __dsub_rn(a[i][j], __dmul_rn(f, a[k][j]));
#pragma unroll
      for (int j = 0; j < k; ++j) B[i][j] = __dsub_rn(B[i][j], __dmul_rn(f, B[k][j]));
      B[i][k] = -__dmul_rn(f, B[k][k]);
    }
  }
  return sing;
}

template <int M>
__global__ void __launch_bounds__(tpc<M>()) k_gj_inverse_tma(sunbw::pipe::IO<1, 1> io, int64_t G,
                                                            unsigned long long* first_singular) {
  extern __shared__ __align__(128) unsigned char smem[];
  sunbw::pipe::run<tpc<M>(), kStagesLU>(
      io, G, smem, [&](int, int64_t g, const unsigned char** ip, unsigned char** op) {
        const double* ain = reinterpret_cast<const double*>(ip[0]);
        double a[M][M], B[M][M];
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int j = 0; j < M; ++j) a[i][j] = ain[i * M + j];
        const bool sing = gj_regs<M>(a, B);
        double* bout = reinterpret_cast<double*>(op[0]);
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int j = 0; j < M; ++j) bout[i * M + j] = B[i][j];
        if (sing) atomicMin(first_singular, (unsigned long long)(g + 1));
      });
}

// plain one-thread-per-block variants (operands not 16-B aligned)
template <int M>
__global__ void k_gj_inverse(double* A, int64_t G, unsigned long long* first_singular) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    double a[M][M], B[M][M];
#pragma unroll
    for (int e = 0; e < M * M; ++e) a[e / M][e % M] = A[g * M * M + e];
    if (gj_regs<M>(a, B)) atomicMin(first_singular, (unsigned long long)(g + 1));
#pragma unroll
    for (int e = 0; e < M * M; ++e) A[g * M * M + e] = B[e / M][e % M];
  }
}
template <int M>
__global__ void k_gj_apply(const double* B, const double* b, double* x, int64_t G) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    double r[M], y[M];
#pragma unroll
    for (int i = 0; i < M; ++i) r[i] = b[g * M + i];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      double s = __dmul_rn(B[g * M * M + i * M], r[0]);
#pragma unroll
      for (int j = 1; j < M; ++j) s = __dadd_rn(s, __dmul_rn(B[g * M * M + i * M + j], r[j]));
      y[i] = s;
    }
#pragma unroll
    for (int i = 0; i < M; ++i) x[g * M + i] = y[i];
  }
}

// x = A^{-1} b: each row a left-to-right sum (R29); x may alias b
template <int M>
__global__ void __launch_bounds__(tpc<M>()) k_gj_apply_tma(sunbw::pipe::IO<2, 1> io, int64_t G) {
  extern __shared__ __align__(128) unsigned char smem[];
  sunbw::pipe::run<tpc<M>(), kStagesLU>(
      io, G, smem, [&](int, int64_t, const unsigned char** ip, unsigned char** op) {
        const double* B = reinterpret_cast<const double*>(ip[0]);
        const double* b = reinterpret_cast<const double*>(ip[1]);
        double r[M], x[M];
#pragma unroll
        for (int i = 0; i < M; ++i) r[i] = b[i];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double s = __dmul_rn(B[i * M], r[0]);
#pragma unroll
          for (int j = 1; j < M; ++j) s = __dadd_rn(s, __dmul_rn(B[i * M + j], r[j]));
          x[i] = s;
        }
        double* xo = reinterpret_cast<double*>(op[0]);
#pragma unroll
        for (int i = 0; i < M; ++i) xo[i] = x[i];
      });
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// persistent grid: resident CTAs per SM from the shared-memory footprint
inline int grid_tma(SUNBW_Context ctx, int64_t G, int T, int smem) {
  int64_t need = (G + T - 1) / T;
  int occ = (220 * 1024) / smem;
  if (occ > 2048 / T) occ = 2048 / T;
  if (occ < 1) occ = 1;
  int64_t cap = (int64_t)ctx->nsm * occ;
  int64_t g = need < cap ? need : cap;
  return g < 1 ? 1 : (int)g;
}

template <int M>
int launch_lu_factor(SUNBW_Context ctx, int64_t G, double* A, int32_t* piv, unsigned long long* d_first) {
  constexpr int T = tpc<M>();
  if (aligned16(A) && aligned16(piv)) {
    sunbw::pipe::IO<1, 2> io{{(const unsigned char*)A}, {M * M * 8}, {(unsigned char*)A, (unsigned char*)piv},
                             {M * M * 8, 4}};
    const int smem = 128 + T * (kStagesLU * M * M * 8 + M * M * 8 + 4);
    static bool attr = cudaFuncSetAttribute(k_lu_factor_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            smem) == cudaSuccess;
    if (!attr) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    k_lu_factor_tma<M><<<grid_tma(ctx, G, T, smem), T, smem, ctx->stream>>>(io, G, d_first);
  } else {
    k_lu_factor<M><<<grid_for(ctx, G, bpc<M>(), 16), bpc<M>(), 0, ctx->stream>>>(A, piv, G, d_first);
  }
  ctx->launches++;
  return ctx_check_launch(ctx);
}

template <int M>
int launch_lu_solve(SUNBW_Context ctx, int64_t G, const double* LU, const int32_t* piv, const double* b,
                    double* x) {
  constexpr int T = tpc<M>();
  if (aligned16(LU) && aligned16(piv) && aligned16(b) && aligned16(x)) {
    sunbw::pipe::IO<3, 1> io{{(const unsigned char*)LU, (const unsigned char*)piv, (const unsigned char*)b},
                             {M * M * 8, 4, M * 8},
                             {(unsigned char*)x},
                             {M * 8}};
    const int smem = 128 + T * (kStagesLU * (M * M * 8 + 4 + M * 8) + M * 8);
    static bool attr = cudaFuncSetAttribute(k_lu_solve_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            smem) == cudaSuccess;
    if (!attr) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    k_lu_solve_tma<M><<<grid_tma(ctx, G, T, smem), T, smem, ctx->stream>>>(io, G);
  } else {
    k_lu_solve<M><<<grid_for(ctx, G, bpc<M>(), 16), bpc<M>(), 0, ctx->stream>>>(LU, piv, b, x, G);
  }
  ctx->launches++;
  return ctx_check_launch(ctx);
}

constexpr int kOccGJ = 16;

template <int M>
int launch_gj_inverse(SUNBW_Context ctx, int64_t G, double* A, unsigned long long* d_first) {
  constexpr int T = tpc<M>();
  if (!aligned16(A)) {
    k_gj_inverse<M><<<grid_for(ctx, G, 128, kOccGJ), 128, 0, ctx->stream>>>(A, G, d_first);
    ctx->launches++;
    return ctx_check_launch(ctx);
  }
  sunbw::pipe::IO<1, 1> io{{(const unsigned char*)A}, {M * M * 8}, {(unsigned char*)A}, {M * M * 8}};
  const int smem = 128 + T * (kStagesLU * M * M * 8 + M * M * 8);
  static bool attr = cudaFuncSetAttribute(k_gj_inverse_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          smem) == cudaSuccess;
  if (!attr) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  k_gj_inverse_tma<M><<<grid_tma(ctx, G, T, smem), T, smem, ctx->stream>>>(io, G, d_first);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

template <int M>
int launch_gj_apply(SUNBW_Context ctx, int64_t G, const double* B, const double* b, double* x) {
  constexpr int T = tpc<M>();
  if (!(aligned16(B) && aligned16(b) && aligned16(x))) {
    k_gj_apply<M><<<grid_for(ctx, G, 128, kOccGJ), 128, 0, ctx->stream>>>(B, b, x, G);
    ctx->launches++;
    return ctx_check_launch(ctx);
  }
  sunbw::pipe::IO<2, 1> io{{(const unsigned char*)B, (const unsigned char*)b}, {M * M * 8, M * 8},
                           {(unsigned char*)x}, {M * 8}};
  const int smem = 128 + T * (kStagesLU * (M * M * 8 + M * 8) + M * 8);
  static bool attr = cudaFuncSetAttribute(k_gj_apply_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          smem) == cudaSuccess;
  if (!attr) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  k_gj_apply_tma<M><<<grid_tma(ctx, G, T, smem), T, smem, ctx->stream>>>(io, G);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

}  // namespace

// ============================================================ internal API
namespace sunbw {

#define DISPATCH_M(m, MACRO) \
  switch (m) {               \
    MACRO(1) MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) \
    default: return ctx_set_err(ctx, SUNBW_ERR_UNSUPPORTED); \
  }

// resident CTAs per SM for the staged (non-TMA) kernels
constexpr int kOccLU = 16;

// factor in place; d_first accumulates the first singular block (min)
int lu_factor_noreset(SUNBW_Context ctx, int64_t G, int m, double* A, int32_t* piv,
                      unsigned long long* d_first) {
  if (G <= 0) return 0;
#define LUF(M) \
  case M: return launch_lu_factor<M>(ctx, G, A, piv, d_first);
  DISPATCH_M(m, LUF)
#undef LUF
}

int lu_factor(SUNBW_Context ctx, int64_t G, int m, double* A, int32_t* piv,
              unsigned long long* d_first) {
  if (cudaMemsetAsync(d_first, 0xFF, sizeof(unsigned long long), ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  return lu_factor_noreset(ctx, G, m, A, piv, d_first);
}

int lu_solve(SUNBW_Context ctx, int64_t G, int m, const double* LU, const int32_t* piv,
             const double* b, double* x) {
  if (G <= 0) return 0;
#define LUS(M) \
  case M: return launch_lu_solve<M>(ctx, G, LU, piv, b, x);
  DISPATCH_M(m, LUS)
#undef LUS
}

// block inverses in place (symbolic Gauss-Jordan, R29); d_first as lu_factor
int gj_inverse(SUNBW_Context ctx, int64_t G, int m, double* A, unsigned long long* d_first, bool reset) {
  if (reset && cudaMemsetAsync(d_first, 0xFF, sizeof(unsigned long long), ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (G <= 0) return 0;
#define GJI(M) \
  case M: return launch_gj_inverse<M>(ctx, G, A, d_first);
  DISPATCH_M(m, GJI)
#undef GJI
}

int gj_apply(SUNBW_Context ctx, int64_t G, int m, const double* B, const double* b, double* x) {
  if (G <= 0) return 0;
#define GJA(M) \
  case M: return launch_gj_apply<M>(ctx, G, B, b, x);
  DISPATCH_M(m, GJA)
#undef GJA
}

int block_matvec(SUNBW_Context ctx, int64_t G, int m, const double* A, const double* x, double* y) {
  if (G <= 0) return 0;
#define MV(M) \
  case M: k_block_matvec<M><<<grid_for(ctx, G, bpc<M>(), kOccLU), bpc<M>(), 0, ctx->stream>>>(A, x, y, G); break;
  DISPATCH_M(m, MV)
#undef MV
  ctx->launches++;
  return ctx_check_launch(ctx);
}

int scale_add_identity(SUNBW_Context ctx, int64_t G, int m, double c, double* A) {
  int64_t n = G * m * m;
  if (n <= 0) return 0;
  const double* p = A;
  Split sp = split_for(n, &p, 1);
  int64_t items = sp.nvec > 0 ? sp.nvec : n;
  int64_t need = (items + 511) / 512;
  int64_t cap = (int64_t)ctx->nsm * 8;
  int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  k_scale_add_identity<<<grid, 256, 0, ctx->stream>>>(A, n, sp, m, c);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

}  // namespace sunbw

// ==================================================================== C ABI
extern "C" SUNMatrix SUNMatrix_B200BlockDiag(SUNBW_Context ctx, int64_t nblocks, int m) {
  if (!ctx || nblocks < 0 || m < 1 || m > 8) return nullptr;
  double* d = nullptr;
  if (nblocks > 0 &&
      cudaMallocAsync(&d, sizeof(double) * nblocks * m * m, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    ctx_set_err(ctx, SUNBW_ERR_MEM);
    return nullptr;
  }
  return new _SUNMatrix{ctx, nblocks, m, d, true};
}

extern "C" SUNMatrix SUNMatrix_B200BlockDiagMake(SUNBW_Context ctx, int64_t nblocks, int m,
                                                 double* d) {
  if (!ctx || nblocks < 0 || m < 1 || m > 8 || (nblocks > 0 && !d) || ((uintptr_t)d & 7))
    return nullptr;
  return new _SUNMatrix{ctx, nblocks, m, d, false};
}

extern "C" double* SUNMatrix_B200BlockDiag_Data(SUNMatrix A) { return A ? A->d : nullptr; }
extern "C" int64_t SUNMatrix_B200BlockDiag_NumBlocks(SUNMatrix A) { return A ? A->nblocks : -1; }
extern "C" int SUNMatrix_B200BlockDiag_BlockSize(SUNMatrix A) { return A ? A->m : -1; }

extern "C" int SUNMatScaleAddI(double c, SUNMatrix A) {
  if (!A) return SUNBW_ERR_ARG;
  return sunbw::scale_add_identity(A->ctx, A->nblocks, A->m, c, A->d);
}

extern "C" int SUNMatMatvec(SUNMatrix A, N_Vector x, N_Vector y) {
  if (!A || !x || !y) return SUNBW_ERR_ARG;
  if (x->ctx != A->ctx || y->ctx != A->ctx) return ctx_set_err(A->ctx, SUNBW_ERR_CONTEXT);
  if (x->local_len != A->nblocks * A->m || y->local_len != x->local_len)
    return ctx_set_err(A->ctx, SUNBW_ERR_LENGTH);
  if (x->d == y->d) return ctx_set_err(A->ctx, SUNBW_ERR_ARG);
  return sunbw::block_matvec(A->ctx, A->nblocks, A->m, A->d, x->d, y->d);
}

extern "C" void SUNMatDestroy(SUNMatrix A) {
  if (!A) return;
  if (A->owned && A->d) cudaFreeAsync(A->d, A->ctx->stream);
  delete A;
}

namespace {
struct LinSolImpl : _SUNLinearSolver {
  unsigned long long* d_first = nullptr;
};
}  // namespace

extern "C" SUNLinearSolver SUNLinSol_B200BatchedLU(N_Vector y, SUNMatrix A) {
  if (!y || !A || y->ctx != A->ctx || y->local_len != A->nblocks * A->m) return nullptr;
  auto* S = new LinSolImpl();
  S->ctx = A->ctx;
  S->nblocks = A->nblocks;
  S->m = A->m;
  if (cudaMalloc(&S->d_piv, sizeof(int32_t) * (A->nblocks > 0 ? A->nblocks : 1)) != cudaSuccess ||
      cudaMalloc(&S->d_first, sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    ctx_set_err(A->ctx, SUNBW_ERR_MEM);
    SUNLinSolFree(S);
    return nullptr;
  }
  return S;
}

// The paper's task-local block solve (DESIGN R29): Setup replaces
// every block by its inverse (symbolic Gauss-Jordan, no row exchanges; a
// zero pivot flags the block), Solve applies it.  Same handle type and
// Setup/Solve/LastFlag/Free calls as the batched LU.
extern "C" SUNLinearSolver SUNLinSol_B200BatchedGJ(N_Vector y, SUNMatrix A) {
  SUNLinearSolver S = SUNLinSol_B200BatchedLU(y, A);
  if (S) S->type = 2;
  return S;
}

extern "C" int SUNLinSolSetup(SUNLinearSolver S0, SUNMatrix A) {
  if (S0 && S0->type == 1) return sunbw::spgmr_setup(S0, A);
  auto* S = (LinSolImpl*)S0;
  if (!S || !A) return SUNBW_ERR_ARG;
  if (A->ctx != S->ctx) return ctx_set_err(S->ctx, SUNBW_ERR_CONTEXT);
  if (A->nblocks != S->nblocks || A->m != S->m) return ctx_set_err(S->ctx, SUNBW_ERR_LENGTH);
  int e = S->type == 2 ? sunbw::gj_inverse(S->ctx, S->nblocks, S->m, A->d, S->d_first)
                       : sunbw::lu_factor(S->ctx, S->nblocks, S->m, A->d, S->d_piv, S->d_first);
  if (e) return e;
  S->flag_pending = true;
  if (S->deferred) return 0;
  int64_t f = SUNLinSolLastFlag(S);
  if (f < 0) return (int)f;
  return f > 0 ? SUNBW_RECOV_SINGULAR : 0;
}

extern "C" int SUNLinSolSolve(SUNLinearSolver S, SUNMatrix A, N_Vector x, N_Vector b, double tol) {
  if (S && S->type == 1) return sunbw::spgmr_solve(S, A, x, b, tol);
  if (!S || !A || !x || !b) return SUNBW_ERR_ARG;
  if (x->ctx != S->ctx || b->ctx != S->ctx || A->ctx != S->ctx) return ctx_set_err(S->ctx, SUNBW_ERR_CONTEXT);
  if (x->local_len != S->nblocks * S->m || b->local_len != x->local_len)
    return ctx_set_err(S->ctx, SUNBW_ERR_LENGTH);
  if (S->type == 2) return sunbw::gj_apply(S->ctx, S->nblocks, S->m, A->d, b->d, x->d);
  return sunbw::lu_solve(S->ctx, S->nblocks, S->m, A->d, S->d_piv, b->d, x->d);
}

extern "C" int64_t SUNLinSolLastFlag(SUNLinearSolver S0) {
  if (S0 && S0->type == 1) return S0->last_flag;
  auto* S = (LinSolImpl*)S0;
  if (!S) return SUNBW_ERR_ARG;
  if (S->flag_pending) {
    unsigned long long v = 0;
    if (cudaMemcpyAsync(&v, S->d_first, sizeof(v), cudaMemcpyDeviceToHost, S->ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(S->ctx->stream) != cudaSuccess)
      return ctx_set_err(S->ctx, SUNBW_ERR_CUDA);
    S->last_flag = v == ~0ull ? 0 : (int64_t)v;
    S->flag_pending = false;
  }
  return S->last_flag;
}

extern "C" int SUNLinSol_B200BatchedLU_SetDeferredCheck(SUNLinearSolver S, int deferred) {
  if (!S) return SUNBW_ERR_ARG;
  S->deferred = deferred;
  return 0;
}

extern "C" int32_t* SUNLinSol_B200BatchedLU_Pivots(SUNLinearSolver S) { return S ? S->d_piv : nullptr; }

extern "C" void SUNLinSolFree(SUNLinearSolver S0) {
  if (S0 && S0->type == 1) return sunbw::spgmr_free(S0);
  auto* S = (LinSolImpl*)S0;
  if (!S) return;
  if (S->d_piv) cudaFree(S->d_piv);
  if (S->d_first) cudaFree(S->d_first);
  delete S;
}
