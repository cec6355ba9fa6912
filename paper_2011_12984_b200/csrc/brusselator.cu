// brusselator.cu — the paper's demonstration problem as sm_100a kernels.
//
// Brusselator advection–reaction (§7):
//   u_t = -c u_x + A - (w+1) u + v u^2
//   v_t = -c v_x + w u - v u^2
//   w_t = -c w_x + (B - w)/eps - w u
// with c = 0.01, A = 1, B = 3.5, eps = 5e-6, periodic on [0, b]
// (P:374), Gaussian initial bump, first-order upwind finite
// differences on n_x points split over n_px tasks.  The 3D variant
// (DESIGN R19) applies the same upwind difference along x, y and z.
//
// State is interleaved per cell (u,v,w) (DESIGN R12), so the implicit
// reaction couples only the 3 unknowns of a cell and the Newton matrix is
// block diagonal with 3×3 blocks.  The advection operator is
// explicit and needs one plane (3D) or one cell (1D) from the left
// neighbour's slab (the GPU-to-GPU halo of P:394 §7).

#include <cmath>

#include "sunbw_device.cuh"
#include "sunbw_internal.h"
#include "pipeline.cuh"

namespace {

struct Prob {
  SUNBW_Context ctx;
  BW_BrussParams p;
  int64_t nxl, nyl, nzl;     // local extents
  int64_t G;                 // local cells
  int64_t cell_off;          // first global cell
  int64_t part_off;          // first global index along the partitioned axis
  double kx, ky, kz;         // kappa = RN(c / RN(L/n)) per axis
  double* d_halo;            // left neighbour's last plane (P > 1)
  int64_t halo_len;          // doubles per plane
};

// --------------------------------------------------------------- staging
__device__ __forceinline__ void stage_in(double* s, const double* g, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) s[i] = __ldcs(g + i);
}
__device__ __forceinline__ void stage_out(double* g, const double* s, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) g[i] = s[i];
}

// Per-cell map with the AoS tiles staged through shared memory: every global
// access is a contiguous coalesced run.  F: (const double in[WIN],
// double out[WOUT]).
constexpr int kCells = 128;

template <class F, int WIN, int WOUT>
__global__ void __launch_bounds__(kCells) k_cellmap(const double* in, double* out, int64_t G, F f) {
  __shared__ double sin_[kCells * WIN];
  __shared__ double sout[kCells * WOUT];
  for (int64_t c0 = (int64_t)blockIdx.x * kCells; c0 < G; c0 += (int64_t)gridDim.x * kCells) {
    int nc = (int)((G - c0) < kCells ? (G - c0) : kCells);
    __syncthreads();
    stage_in(sin_, in + c0 * WIN, nc * WIN);
    __syncthreads();
    int t = threadIdx.x;
    if (t < nc) {
      double x[WIN], y[WOUT];
#pragma unroll
      for (int k = 0; k < WIN; ++k) x[k] = sin_[t * WIN + k];
      f(x, y);
#pragma unroll
      for (int k = 0; k < WOUT; ++k) sout[t * WOUT + k] = y[k];
    }
    __syncthreads();
    stage_out(out + c0 * WOUT, sout, nc * WOUT);
  }
}

// f_I (reaction terms), same operation order as the definition
struct FReaction {
  double A, B, eps;
  __device__ void operator()(const double* y, double* f) const {
    double u = y[0], v = y[1], w = y[2];
    double uu = __dmul_rn(u, u);
    double vuu = __dmul_rn(v, uu);
    double fu = __dadd_rn(__dsub_rn(A, __dmul_rn(__dadd_rn(w, 1.0), u)), vuu);
    double wu = __dmul_rn(w, u);
    double fv = __dsub_rn(wu, vuu);
    double fw = __dsub_rn(__ddiv_rn(__dsub_rn(B, w), eps), wu);
    f[0] = fu;
    f[1] = fv;
    f[2] = fw;
  }
};

// J = ∂f_I/∂(u,v,w) (P:369-371 differentiated), row-major 3×3
struct FJacobian {
  double inv_eps;   // RN(1/eps), host-computed
  __device__ void operator()(const double* y, double* a) const {
    double u = y[0], v = y[1], w = y[2];
    double uu = __dmul_rn(u, u);
    double uv2 = __dmul_rn(__dmul_rn(2.0, u), v);
    double w1 = __dadd_rn(w, 1.0);
    a[0] = __dsub_rn(uv2, w1);
    a[1] = uu;
    a[2] = -u;
    a[3] = __dsub_rn(w, uv2);
    a[4] = -uu;
    a[5] = u;
    a[6] = -w;
    a[7] = 0.0;
    a[8] = __dsub_rn(-inv_eps, u);
  }
};

// linear test problem: f_I = lam y, J = lam I
struct FLinear {
  double lam;
  __device__ void operator()(const double* y, double* f) const {
    f[0] = __dmul_rn(lam, y[0]);
    f[1] = __dmul_rn(lam, y[1]);
    f[2] = __dmul_rn(lam, y[2]);
  }
};
struct FLinearJac {
  double lam;
  __device__ void operator()(const double*, double* a) const {
#pragma unroll
    for (int e = 0; e < 9; ++e) a[e] = (e % 4 == 0) ? lam : 0.0;
  }
};

// IC: p = alpha exp(-e), e = Σ_axis (x-mu)^2 / (2 sigma^2)
struct ICParams {
  int64_t nx, ny, nz;        // global extents
  int64_t cell_off;          // first global cell of this slab
  double dx, dy, dz, mx, my, mz, tx, ty, tz;
  double A, BA, alpha;
};

__global__ void k_ic(double* y, int64_t G, ICParams q) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < G;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t gc = q.cell_off + c;
    int64_t i = gc % q.nx, j = (gc / q.nx) % q.ny, k = gc / (q.nx * q.ny);
    double xe = __dsub_rn(__dmul_rn((double)i, q.dx), q.mx);
    double e = __ddiv_rn(__dmul_rn(xe, xe), q.tx);
    if (q.ny > 1) {
      double ye = __dsub_rn(__dmul_rn((double)j, q.dy), q.my);
      e = __dadd_rn(e, __ddiv_rn(__dmul_rn(ye, ye), q.ty));
    }
    if (q.nz > 1) {
      double ze = __dsub_rn(__dmul_rn((double)k, q.dz), q.mz);
      e = __dadd_rn(e, __ddiv_rn(__dmul_rn(ze, ze), q.tz));
    }
    double p = __dmul_rn(q.alpha, exp(-e));
    y[3 * c] = __dadd_rn(q.A, p);
    y[3 * c + 1] = __dadd_rn(q.BA, p);
    y[3 * c + 2] = __dadd_rn(3.0, p);
  }
}

// 1D upwind advection, partitioned along x: f_i = kx (q_{i-1} - q_i); the
// i-1 neighbour of local cell 0 comes from `left` (halo, or own last cell).
__global__ void k_adv1d(const double* __restrict__ y, const double* __restrict__ left,
                        double* __restrict__ f, int64_t n, double kx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double q = y[e];
    double qm = e >= 3 ? y[e - 3] : left[e];
    f[e] = __dmul_rn(kx, __dsub_rn(qm, q));
  }
}

// 3D upwind advection on a z-slab: one CTA per (k, j) row of 3·nx values.
// Sum order x, then + y, then + z (DESIGN R19); x and y periodic inside the
// slab, the k-1 plane of local k = 0 from `below` (halo or own last plane).
struct Adv3 {
  int nx, ny, nzl;
  int ny_g, nz_g;            // global extents (terms of extent-1 axes vanish)
  double kx, ky, kz;
};

__global__ void __launch_bounds__(256) k_adv3d(const double* __restrict__ y,
                                               const double* __restrict__ below,
                                               double* __restrict__ f, Adv3 a) {
  const int rowlen = 3 * a.nx;
  const int64_t plane = (int64_t)rowlen * a.ny;
  const int nrows = a.ny * a.nzl;
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int j = r % a.ny, k = r / a.ny;
    const int64_t base = (int64_t)r * rowlen;
    const int64_t rowm = j > 0 ? base - rowlen : base + (int64_t)(a.ny - 1) * rowlen;
    const double* zrow = k > 0 ? y + base - plane : below + (int64_t)j * rowlen;
    for (int e = threadIdx.x; e < rowlen; e += blockDim.x) {
      const int i = e / 3;
      const int em = i > 0 ? e - 3 : e + rowlen - 3;
      double q = y[base + e];
      double acc = __dmul_rn(a.kx, __dsub_rn(y[base + em], q));
      if (a.ny_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.ky, __dsub_rn(y[rowm + e], q)));
      if (a.nz_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.kz, __dsub_rn(zrow[e], q)));
      f[base + e] = acc;
    }
  }
}

// Multi-row variant: a CTA of 256 threads takes RPB consecutive rows, each
// thread EPT values per row (3·nx <= 256·EPT); all of a thread's loads are
// issued before any value is used (RPB·EPT independent y_n loads in flight
// per thread instead of one).  Same arithmetic and order as k_adv3d.
template <int RPB, int EPT>
__global__ void __launch_bounds__(256) k_adv3d_r(const double* __restrict__ y,
                                                 const double* __restrict__ below,
                                                 double* __restrict__ f, Adv3 a) {
  const int rowlen = 3 * a.nx;
  const int64_t plane = (int64_t)rowlen * a.ny;
  const int nrows = a.ny * a.nzl;
  for (int r0 = blockIdx.x * RPB; r0 < nrows; r0 += gridDim.x * RPB) {
    double q[RPB][EPT], qx[RPB][EPT], qy[RPB][EPT], qz[RPB][EPT];
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr) {
      const int r = r0 + rr < nrows ? r0 + rr : nrows - 1;
      const int j = r % a.ny, k = r / a.ny;
      const int64_t base = (int64_t)r * rowlen;
      const int64_t rowm = j > 0 ? base - rowlen : base + (int64_t)(a.ny - 1) * rowlen;
      const double* zrow = k > 0 ? y + base - plane : below + (int64_t)j * rowlen;
#pragma unroll
      for (int c = 0; c < EPT; ++c) {
        int e = threadIdx.x + 256 * c;
        e = e < rowlen ? e : rowlen - 1;
        const int em = e >= 3 ? e - 3 : e + rowlen - 3;
        q[rr][c] = __ldg(y + base + e);
        qx[rr][c] = __ldg(y + base + em);
        qy[rr][c] = a.ny_g > 1 ? __ldg(y + rowm + e) : 0.0;
        qz[rr][c] = a.nz_g > 1 ? __ldg(zrow + e) : 0.0;
      }
    }
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr) {
      const int r = r0 + rr;
      if (r >= nrows) break;
      const int64_t base = (int64_t)r * rowlen;
#pragma unroll
      for (int c = 0; c < EPT; ++c) {
        const int e = threadIdx.x + 256 * c;
        if (e >= rowlen) break;
        double acc = __dmul_rn(a.kx, __dsub_rn(qx[rr][c], q[rr][c]));
        if (a.ny_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.ky, __dsub_rn(qy[rr][c], q[rr][c])));
        if (a.nz_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.kz, __dsub_rn(qz[rr][c], q[rr][c])));
        f[base + e] = acc;
      }
    }
  }
}

// Vectorised 3D variant for 3·nx % 4 == 0 (nx % 4 == 0) and 32-B aligned
// rows: thread v owns the 4 values [4v, 4v+4) of the row; the row is staged
// in shared memory for the x-neighbour (e-3 crosses 32-B vectors), the y-1
// row and the z-1 plane row are read as aligned 256-bit vectors (they are
// L2 hits: the row below was read ~one plane earlier).  Same arithmetic and
// order as k_adv3d.
__global__ void __launch_bounds__(256) k_adv3d_v4(const double* __restrict__ y,
                                                  const double* __restrict__ below,
                                                  double* __restrict__ f, Adv3 a) {
  __shared__ __align__(32) double srow[3 * 1024];
  const int rowlen = 3 * a.nx;
  const int nv = rowlen / 4;
  const int64_t plane = (int64_t)rowlen * a.ny;
  const int nrows = a.ny * a.nzl;
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int j = r % a.ny, k = r / a.ny;
    const int64_t base = (int64_t)r * rowlen;
    const double* yrow = y + base;
    const double* ym = j > 0 ? yrow - rowlen : yrow + (int64_t)(a.ny - 1) * rowlen;
    const double* zm = k > 0 ? yrow - plane : below + (int64_t)j * rowlen;
    __syncthreads();
    sunbw::d4 q[2], qy[2], qz[2];
    int cnt = 0;
    for (int v = threadIdx.x; v < nv && cnt < 2; v += blockDim.x, ++cnt) {
      q[cnt] = sunbw::ld4(yrow + 4 * v);
      if (a.ny_g > 1) qy[cnt] = sunbw::ld4(ym + 4 * v);
      if (a.nz_g > 1) qz[cnt] = sunbw::ld4(zm + 4 * v);
      *reinterpret_cast<sunbw::d4*>(srow + 4 * v) = q[cnt];
    }
    __syncthreads();
    cnt = 0;
    for (int v = threadIdx.x; v < nv && cnt < 2; v += blockDim.x, ++cnt) {
      sunbw::d4 o;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int e = 4 * v + l;
        const double qq = q[cnt].v[l];
        const double qx = srow[e >= 3 ? e - 3 : e + rowlen - 3];
        double acc = __dmul_rn(a.kx, __dsub_rn(qx, qq));
        if (a.ny_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.ky, __dsub_rn(qy[cnt].v[l], qq)));
        if (a.nz_g > 1) acc = __dadd_rn(acc, __dmul_rn(a.kz, __dsub_rn(qz[cnt].v[l], qq)));
        o.v[l] = acc;
      }
      sunbw::st4(f + base + 4 * v, o);
    }
  }
}

int grid_cells(SUNBW_Context ctx, int64_t G) {
  int64_t need = (G + kCells - 1) / kCells;
  int64_t cap = (int64_t)ctx->nsm * 16;
  int64_t g = need < cap ? need : cap;
  return g < 1 ? 1 : (int)g;
}

int check_vec(Prob* P, N_Vector v) {
  if (!v) return SUNBW_ERR_ARG;
  if (v->ctx != P->ctx) return ctx_set_err(P->ctx, SUNBW_ERR_CONTEXT);
  if (v->local_len != 3 * P->G) return ctx_set_err(P->ctx, SUNBW_ERR_LENGTH);
  return 0;
}

// TMA-pipelined per-cell map (pipeline.cuh): input and output tiles of 128
// cells move as single bulk copies, double-buffered, persistent CTAs
template <class F, int WIN, int WOUT>
__global__ void __launch_bounds__(kCells) k_cellmap_tma(sunbw::pipe::IO<1, 1> io, int64_t G, F f) {
  extern __shared__ __align__(128) unsigned char smem[];
  sunbw::pipe::run<kCells, 2>(io, G, smem,
                              [&](int, int64_t, const unsigned char** ip, unsigned char** op) {
                                const double* xi = reinterpret_cast<const double*>(ip[0]);
                                double x[WIN], y[WOUT];
#pragma unroll
                                for (int k = 0; k < WIN; ++k) x[k] = xi[k];
                                f(x, y);
                                double* yo = reinterpret_cast<double*>(op[0]);
#pragma unroll
                                for (int k = 0; k < WOUT; ++k) yo[k] = y[k];
                              });
}

template <class F, int WIN, int WOUT>
void launch_cellmap(SUNBW_Context ctx, const double* in, double* out, int64_t G, F f) {
  // output-heavy maps (the 72-B Jacobian blocks) measured faster staged
  if (WOUT <= WIN && (((uintptr_t)in | (uintptr_t)out) & 15) == 0) {
    sunbw::pipe::IO<1, 1> io{{(const unsigned char*)in}, {WIN * 8}, {(unsigned char*)out}, {WOUT * 8}};
    const int smem = 128 + kCells * (2 * WIN * 8 + WOUT * 8);
    int64_t need = (G + kCells - 1) / kCells;
    int occ = (220 * 1024) / smem;
    if (occ > 16) occ = 16;
    int64_t cap = (int64_t)ctx->nsm * occ;
    int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
    k_cellmap_tma<F, WIN, WOUT><<<grid, kCells, smem, ctx->stream>>>(io, G, f);
  } else {
    k_cellmap<F, WIN, WOUT><<<grid_cells(ctx, G), kCells, 0, ctx->stream>>>(in, out, G, f);
  }
}

}  // namespace

// ============================================================ internal API
namespace sunbw {

int bw_reaction(void* prob, const double* y, double* f) {
  auto* P = (Prob*)prob;
  SUNBW_Context ctx = P->ctx;
  if (P->G <= 0) return 0;
  if (P->p.kind == 1)
    launch_cellmap<FLinear, 3, 3>(ctx, y, f, P->G, FLinear{P->p.lam_I});
  else
    launch_cellmap<FReaction, 3, 3>(ctx, y, f, P->G, FReaction{P->p.A, P->p.B, P->p.eps});
  ctx->launches++;
  return ctx_check_launch(ctx);
}

int bw_jacobian(void* prob, const double* y, double* J) {
  auto* P = (Prob*)prob;
  SUNBW_Context ctx = P->ctx;
  if (P->G <= 0) return 0;
  if (P->p.kind == 1)
    launch_cellmap<FLinearJac, 3, 9>(ctx, y, J, P->G, FLinearJac{P->p.lam_I});
  else
    launch_cellmap<FJacobian, 3, 9>(ctx, y, J, P->G, FJacobian{1.0 / P->p.eps});
  ctx->launches++;
  return ctx_check_launch(ctx);
}

// halo exchange only (ring shift of the last plane to the right neighbour)
int bw_halo_stream(void* prob, const double* y, cudaStream_t stream) {
  auto* P = (Prob*)prob;
  SUNBW_Context ctx = P->ctx;
  if (ctx_nranks(ctx) == 1 || P->p.reaction_only || P->p.kind == 1) return 0;
  const double* last = y + 3 * P->G - P->halo_len;
  int e = ctx->comm->halo_shift(last, P->d_halo, (size_t)P->halo_len, stream);
  return e ? ctx_set_err(ctx, e) : 0;
}

int bw_halo(void* prob, const double* y) { return bw_halo_stream(prob, y, ((Prob*)prob)->ctx->stream); }

// stencil only (assumes bw_halo ran for this y when P > 1)
int bw_advection_stencil(void* prob, const double* y, double* f) {
  auto* P = (Prob*)prob;
  SUNBW_Context ctx = P->ctx;
  int64_t n = 3 * P->G;
  if (n <= 0) return 0;
  if (P->p.reaction_only) {
    if (cudaMemsetAsync(f, 0, sizeof(double) * n, ctx->stream) != cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    return 0;
  }
  if (P->p.kind == 1) return sunbw::scale(ctx, n, P->p.lam_E, y, f, nullptr);
  const double* left = ctx_nranks(ctx) > 1 ? P->d_halo : y + n - P->halo_len;
  if (P->p.dim == 1) {
    int64_t need = (n + 255) / 256, cap = (int64_t)ctx->nsm * 8;
    k_adv1d<<<(int)(need < cap ? need : cap), 256, 0, ctx->stream>>>(y, left, f, n, P->kx);
  } else {
    Adv3 a{(int)P->nxl, (int)P->nyl, (int)P->nzl, (int)P->p.ny, (int)P->p.nz, P->kx, P->ky, P->kz};
    int rows = (int)(P->nyl * P->nzl);
    const int rowlen = 3 * (int)P->nxl;
#ifndef SUNBW_ADV_VARIANT
#define SUNBW_ADV_VARIANT 0   // 0: per-element kernel (fastest measured); 1/2: vectorised
#endif
    const bool vec = SUNBW_ADV_VARIANT > 0 && rowlen % 4 == 0 && rowlen <= 2048 &&
                     (((uintptr_t)y | (uintptr_t)f | (uintptr_t)left) & 31) == 0;
#ifndef SUNBW_ADV_RPB
#define SUNBW_ADV_RPB 2
#endif
    if (SUNBW_ADV_RPB > 0 && rowlen <= 4 * 256 && !vec) {
      constexpr int R = SUNBW_ADV_RPB > 0 ? SUNBW_ADV_RPB : 1;
      const int ept = (rowlen + 255) / 256;
      const int64_t need = (rows + R - 1) / R, cap = (int64_t)ctx->nsm * 8 * 4;
      const int grid = (int)(need < cap ? need : cap);
      if (ept == 1) k_adv3d_r<R, 1><<<grid, 256, 0, ctx->stream>>>(y, left, f, a);
      else if (ept == 2) k_adv3d_r<R, 2><<<grid, 256, 0, ctx->stream>>>(y, left, f, a);
      else if (ept == 3) k_adv3d_r<R, 3><<<grid, 256, 0, ctx->stream>>>(y, left, f, a);
      else k_adv3d_r<R, 4><<<grid, 256, 0, ctx->stream>>>(y, left, f, a);
    } else if (vec) {
      int nv = rowlen / 4;
      int block = nv <= 256 ? ((nv + 31) / 32) * 32 : 256;
      int64_t cap = SUNBW_ADV_VARIANT == 1 ? (int64_t)ctx->nsm * (2048 / block) : rows;
      int grid = (int)(rows < cap ? rows : cap);
      k_adv3d_v4<<<grid, block, 0, ctx->stream>>>(y, left, f, a);
    } else {
      k_adv3d<<<rows, 256, 0, ctx->stream>>>(y, left, f, a);
    }
  }
  ctx->launches++;
  return ctx_check_launch(ctx);
}

int64_t bw_local_cells(void* prob) { return ((Prob*)prob)->G; }
BW_BrussParams bw_params(void* prob) { return ((Prob*)prob)->p; }

bool bw_small_geometry(void* prob, SmallGeom* g) {
  auto* P = (Prob*)prob;
  const BW_BrussParams& p = P->p;
  if (ctx_nranks(P->ctx) != 1 || P->G < 1 || P->G > kSmallCells) return false;
  g->nx = (int)P->nxl;
  g->ny = (int)P->nyl;
  g->nz = (int)P->nzl;
  g->kx = P->kx;
  g->ky = P->ky;
  g->kz = P->kz;
  g->expl = p.reaction_only ? 2 : (p.kind == 1 ? 1 : 0);
  g->lam_E = p.lam_E;
  return true;
}

void bw_ark_geometry(void* prob, ArkGeometry* g) {
  auto* P = (Prob*)prob;
  const BW_BrussParams& p = P->p;
  g->dim = p.dim;
  g->expl = p.reaction_only ? 2 : (p.kind == 1 ? 1 : 0);
  g->has_y = p.ny > 1;
  g->has_z = p.nz > 1;
  g->nx = P->nxl;
  g->ny = P->nyl;
  g->nzl = P->nzl;
  g->G = P->G;
  g->halo_len = P->halo_len;
  g->kx = P->kx;
  g->ky = P->ky;
  g->kz = P->kz;
  g->lam_E = p.lam_E;
}

bool bw_fused_advection(void* prob, const double* y, FusedAdvection* fa) {
  auto* P = (Prob*)prob;
  const BW_BrussParams& p = P->p;
  if (p.dim != 3 || p.kind != 0 || p.reaction_only || P->nxl % 128 != 0 || p.ny < 2 || p.nz < 2 ||
      P->G >= (int64_t(1) << 31))               // the kernel's tile indexing is 32-bit
    return false;
  fa->nx = P->nxl;
  fa->ny = P->nyl;
  fa->nzl = P->nzl;
  fa->kx = P->kx;
  fa->ky = P->ky;
  fa->kz = P->kz;
  fa->below = ctx_nranks(P->ctx) > 1 ? P->d_halo : y + 3 * P->G - P->halo_len;
  return true;
}

}  // namespace sunbw

// ==================================================================== C ABI
extern "C" int BW_ProblemCreate(SUNBW_Context ctx, const BW_BrussParams* p, void** out) {
  if (!ctx || !p || !out) return SUNBW_ERR_ARG;
  *out = nullptr;
  if ((p->dim != 1 && p->dim != 3) || p->nx < 1 || p->ny < 1 || p->nz < 1 || p->Lx <= 0 ||
      (p->dim == 1 && (p->ny != 1 || p->nz != 1)) || (p->kind != 0 && p->kind != 1) ||
      (p->kind == 0 && !(p->c > 0)))            // upwind direction fixed: c > 0 (R20)
    return SUNBW_ERR_ARG;
  if (p->dim == 3 && (p->Ly <= 0 || p->Lz <= 0 || p->nx > (1 << 20) || p->ny > (1 << 20)))
    return SUNBW_ERR_ARG;
  int R = ctx_nranks(ctx), r = ctx_rank(ctx);
  auto* P = new Prob();
  P->ctx = ctx;
  P->p = *p;
  if (p->dim == 1) {
    if (p->nx % R) { delete P; return SUNBW_ERR_ARG; }
    P->nxl = p->nx / R; P->nyl = 1; P->nzl = 1;
    P->part_off = r * P->nxl;
    P->cell_off = P->part_off;
    P->halo_len = 3;
  } else {
    if (p->nz % R) { delete P; return SUNBW_ERR_ARG; }
    P->nxl = p->nx; P->nyl = p->ny; P->nzl = p->nz / R;
    P->part_off = r * P->nzl;
    P->cell_off = P->part_off * p->nx * p->ny;
    P->halo_len = 3 * p->nx * p->ny;
  }
  P->G = P->nxl * P->nyl * P->nzl;
  // kappa = RN(c / RN(L/n)) (O9)
  P->kx = p->c / (p->Lx / (double)p->nx);
  P->ky = p->dim == 3 ? p->c / (p->Ly / (double)p->ny) : 0.0;
  P->kz = p->dim == 3 ? p->c / (p->Lz / (double)p->nz) : 0.0;
  P->d_halo = nullptr;
  if (R > 1 && cudaMalloc(&P->d_halo, sizeof(double) * P->halo_len) != cudaSuccess) {
    cudaGetLastError();
    delete P;
    return ctx_set_err(ctx, SUNBW_ERR_MEM);
  }
  *out = P;
  return 0;
}

extern "C" int BW_ProblemDestroy(void* prob) {
  auto* P = (Prob*)prob;
  if (!P) return SUNBW_ERR_ARG;
  if (P->d_halo) cudaFree(P->d_halo);
  delete P;
  return 0;
}

extern "C" int64_t BW_ProblemLocalCells(void* prob) { return prob ? ((Prob*)prob)->G : -1; }
extern "C" int64_t BW_ProblemCellOffset(void* prob) { return prob ? ((Prob*)prob)->cell_off : -1; }

extern "C" int BW_InitialCondition(void* prob, N_Vector y) {
  auto* P = (Prob*)prob;
  if (!P) return SUNBW_ERR_ARG;
  if (int e = check_vec(P, y)) return e;
  if (P->G <= 0) return 0;
  const BW_BrussParams& p = P->p;
  ICParams q;
  q.nx = p.nx; q.ny = p.ny; q.nz = p.nz; q.cell_off = P->cell_off;
  double Ly = p.dim == 3 ? p.Ly : 1.0, Lz = p.dim == 3 ? p.Lz : 1.0;
  q.dx = p.Lx / (double)p.nx; q.dy = Ly / (double)p.ny; q.dz = Lz / (double)p.nz;
  q.mx = p.Lx / 2.0; q.my = Ly / 2.0; q.mz = Lz / 2.0;
  double sx = p.Lx / 4.0, sy = Ly / 4.0, sz = Lz / 4.0;
  q.tx = 2.0 * (sx * sx); q.ty = 2.0 * (sy * sy); q.tz = 2.0 * (sz * sz);
  q.A = p.A; q.BA = p.B / p.A; q.alpha = p.alpha;
  SUNBW_Context ctx = P->ctx;
  int64_t need = (P->G + 255) / 256, cap = (int64_t)ctx->nsm * 8;
  k_ic<<<(int)(need < cap ? need : cap), 256, 0, ctx->stream>>>(y->d, P->G, q);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

extern "C" int BW_AdvectionRHS(void* prob, N_Vector y, N_Vector fE) {
  auto* P = (Prob*)prob;
  if (!P) return SUNBW_ERR_ARG;
  if (int e = check_vec(P, y)) return e;
  if (int e = check_vec(P, fE)) return e;
  if (y->d == fE->d) return ctx_set_err(P->ctx, SUNBW_ERR_ARG);
  if (int e = sunbw::bw_halo(P, y->d)) return e;
  return sunbw::bw_advection_stencil(P, y->d, fE->d);
}

extern "C" int BW_ReactionRHS(void* prob, N_Vector y, N_Vector fI) {
  auto* P = (Prob*)prob;
  if (!P) return SUNBW_ERR_ARG;
  if (int e = check_vec(P, y)) return e;
  if (int e = check_vec(P, fI)) return e;
  return sunbw::bw_reaction(P, y->d, fI->d);
}

extern "C" int BW_ReactionJacobian(void* prob, N_Vector y, SUNMatrix J) {
  auto* P = (Prob*)prob;
  if (!P || !J) return SUNBW_ERR_ARG;
  if (int e = check_vec(P, y)) return e;
  if (J->ctx != P->ctx) return ctx_set_err(P->ctx, SUNBW_ERR_CONTEXT);
  if (J->nblocks != P->G || J->m != 3) return ctx_set_err(P->ctx, SUNBW_ERR_LENGTH);
  return sunbw::bw_jacobian(P, y->d, J->d);
}
