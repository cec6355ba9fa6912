// ark_fused.cu — the adaptive IMEX ARK step of the paper's demonstration
// (ARKODE IMEX; tableau ARK3(2)4L[2]SA, DESIGN R26) with each
// stage fused into ONE kernel, the fast path of ark.cu's composed driver
// (BW_ArkOptions.fused; DESIGN R32).
//
// Stage i = 1..3 (a^I_11 = 0: stage 0 is Z_0 = y_n), one thread per cell:
//   for j < i:  FE_j = f_E(Z_j) (upwind stencil of Z_j, neighbours from
//               memory / the halo), FI_j = f_I(Z_j)
//   rhs = y_n + h Σ_{j<i} (aE_ij FE_j + aI_ij FI_j)
//   modified Newton on z - hγ f_I(z) = rhs from the predictor Z_{i-1}:
//   M = I - hγ J(Z_{i-1}), LU, Kr iterations r = rhs + hγ f_I(z) - z,
//   δ = M⁻¹r, z += δ, Σ(δ ewt(y_n))² per iteration  -> Z_i
// Final kernel: y_{n+1} = y_n + h Σ b_j (FE_j + FI_j), the embedded error
// e = h Σ (b_j - d_j)(FE_j + FI_j) and Σ(e ewt)².
// Only the stage states Z_1..Z_3 are stored (one vector each): FE_j and FI_j
// are recomputed from Z_j where they are needed, so a stage reads i state
// vectors and writes one, instead of the composed path's 2i+1 reads and
// separate LC / Jacobian / LU / solve / update / WRMS passes.
//
// Convergence (R31's scheme per stage): every stage kernel runs a
// predicted iteration count Kr_i and reports every iteration's global ν;
// the three stages and the final kernel are enqueued back to back and the
// host reads all ν's and the error norm with ONE synchronisation per
// attempt, then takes the oracle's decisions stage by stage (first k with
// ν_k <= tol_nl; a zero pivot or no convergence within maxnl recomputes the
// step with h/4).  A stage whose count differs from Kr_i is
// recomputed with the right count, together with the stages after it.
// The cell arithmetic is the contracted one of R30 (FMAs, reciprocal
// pivots; a cell whose Newton matrix would pivot or whose pivots leave the
// guarded range takes the pivoting IEEE-division path): parity to the
// oracle's composed ARK is the north star's 1e-9 on states with identical
// step / iteration counts (tests/test_gpu_ark.py).

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "sunbw_internal.h"
#include "cellstep.cuh"

namespace {

using namespace sunbw::cell;

constexpr int kThreads = 256;
constexpr int kMaxNL = 4;                // fused ARK: Newton iterations per stage <= 4
constexpr int kCols = kMaxNL + 1;        // partial columns: [unused, S_1..S_kMaxNL]
constexpr int kStages = 4;               // ARK3(2)4L[2]SA

// ARK3(2)4L[2]SA (Kennedy & Carpenter 2003), as in ark.cu / the oracle
const double kG = 1767732205903.0 / 4055673282236.0;
const double kAE[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 2027836641118.0, 0, 0, 0},
    {5535828885825.0 / 10492691773637.0, 788022342437.0 / 10882634858940.0, 0, 0},
    {6485989280629.0 / 16251701735622.0, -4246266847089.0 / 9704473918619.0,
     10755448449292.0 / 10357097424841.0, 0}};
const double kAI[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 4055673282236.0, 1767732205903.0 / 4055673282236.0, 0, 0},
    {2746238789719.0 / 10658868560708.0, -640167445237.0 / 6845629431997.0,
     1767732205903.0 / 4055673282236.0, 0},
    {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
     11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0}};
const double kB[4] = {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
                      11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0};
const double kD[4] = {2756255671327.0 / 12835298489170.0, -10771552573575.0 / 22201958757719.0,
                      9247589265047.0 / 10645013368117.0, 2193209047091.0 / 5459859503100.0};

struct Geom {
  int dim, expl, has_y, has_z;
  int64_t nx, ny, nzl, G;
  double kx, ky, kz, ks, lam_E;
};

struct Args {
  const double* y;              // y_n = Z_0
  const double* Z[3];           // Z_1..Z_3
  const double* below[4];       // per state: what sits under local cell/plane 0 (halo or own wrap)
  double* out;                  // Z_i (stage) or y_{n+1} (final)
  double cE[4], cI[4];          // stage: h aE_ij, h aI_ij;  final: h b_j, h b_j
  double cErr[4];               // final: h (b_j - d_j)
  double* partials;             // [grid][kCols]
  unsigned* counter;            // in-kernel fold (self-resetting)
  double* sums;                 // this launch's kCols local sums
  unsigned long long* first;    // first singular cell (1-based), this stage
  int krt;                      // Newton iterations of this launch
};

template <int KIND>
__device__ __forceinline__ void implicit_rhs(const FusedParams& p, const double (&q)[3], double (&fi)[3]) {
  if (KIND == 1) {
#pragma unroll
    for (int s = 0; s < 3; ++s) fi[s] = p.lam_I * q[s];
    return;
  }
  const double u = q[0], v = q[1], w = q[2], uu = u * u;
  fi[0] = __fma_rn(v, uu, __fma_rn(-(w + 1.0), u, p.A));                // A - (w+1)u + v u²
  fi[1] = __fma_rn(-v, uu, w * u);                                      // wu - v u²
  fi[2] = __fma_rn(-w, u + p.rcp_eps, p.beps);                          // (B - w)/ε - wu
}

// Contracted modified Newton on one cell (R30 arithmetic, γ = p.gamma):
// false (z untouched) if the Newton matrix needs a row exchange or a pivot
// leaves the guarded range — the caller then runs newton_exact.
template <int KIND>
__device__ __forceinline__ bool newton_ct(const FusedParams& p, const double (&d)[3], double (&z)[3],
                                          const double (&ew)[3], int krt, double (&nu)[kMaxNL]) {
  double a00, a01, a02, a10, a11, a12, a20, a21, a22;
  if (KIND == 1) {
    const double m = __fma_rn(-p.gamma, p.lam_I, 1.0);
    a00 = a11 = a22 = m;
    a01 = a02 = a10 = a12 = a20 = a21 = 0.0;
  } else {
    const double u = z[0], v = z[1], w = z[2];
    const double uu = u * u, uv2 = (u + u) * v, gu = p.gamma * u;
    a01 = -p.gamma * uu;
    a00 = __fma_rn(-p.gamma, uv2 - (w + 1.0), 1.0);
    a02 = gu;
    a10 = p.gamma * (uv2 - w);
    a11 = 1.0 - a01;
    a12 = -gu;
    a20 = p.gamma * w;
    a21 = 0.0;
    a22 = p.c22 + gu;
  }
  bool ok = !mag_gt(a10, a00) & !mag_gt(a20, a00) & safe_mag(a00);
  const double p0 = rcp_nr2(a00);
  const double l10 = a10 * p0, l20 = a20 * p0;
  a11 = __fma_rn(-l10, a01, a11);
  a12 = __fma_rn(-l10, a02, a12);
  a21 = __fma_rn(-l20, a01, a21);
  a22 = __fma_rn(-l20, a02, a22);
  ok = ok & !mag_gt(a21, a11) & safe_mag(a11);
  const double p1 = rcp_nr2(a11);
  const double l21 = a21 * p1;
  a22 = __fma_rn(-l21, a12, a22);
  ok = ok & safe_mag(a22);
  if (!ok) return false;
  const double p2 = rcp_nr2(a22);
#pragma unroll
  for (int it = 0; it < kMaxNL; ++it) {
    if (it >= krt) break;
    double f[3];
    implicit_rhs<KIND>(p, z, f);
    double r0 = __fma_rn(p.gamma, f[0], d[0] - z[0]);
    double r1 = __fma_rn(p.gamma, f[1], d[1] - z[1]);
    double r2 = __fma_rn(p.gamma, f[2], d[2] - z[2]);
    r1 = __fma_rn(-l10, r0, r1);
    r2 = __fma_rn(-l21, r1, __fma_rn(-l20, r0, r2));
    r2 = r2 * p2;
    r1 = __fma_rn(-a12, r2, r1) * p1;
    r0 = __fma_rn(-a02, r2, __fma_rn(-a01, r1, r0)) * p0;
    z[0] += r0;
    z[1] += r1;
    z[2] += r2;
    const double q0 = r0 * ew[0], q1 = r1 * ew[1], q2 = r2 * ew[2];
    nu[it] += __fma_rn(q2, q2, __fma_rn(q1, q1, q0 * q0));
  }
  return true;
}

// The same iteration with partial pivoting and IEEE divisions (the exact
// primitives of the composed path); returns false for a zero pivot.
template <int KIND>
__device__ __noinline__ bool newton_exact(const FusedParams& p, const double (&d)[3], double (&z)[3],
                                          const double (&ew)[3], int krt, double (&nu)[kMaxNL]) {
  double a[3][3], rp[3];
  newton_matrix<KIND>(p, z, a);
  bool singular = false;
  DivExact dv{true};
  const int code = lu3(a, rp, singular, dv);
  for (int it = 0; it < krt; ++it) {
    double f[3], r[3];
    reaction<KIND>(p, z, f, dv);
#pragma unroll
    for (int s = 0; s < 3; ++s) r[s] = __dadd_rn(__dadd_rn(d[s], __dmul_rn(p.gamma, f[s])), -z[s]);
    solve3(a, code, true, rp, r, dv);
    double w = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      z[s] = __dadd_rn(z[s], r[s]);
      const double q = r[s] * ew[s];
      w = __fma_rn(q, q, w);
    }
#pragma unroll
    for (int k = 0; k < kMaxNL; ++k)
      if (k == it) nu[k] += w;
  }
  return !singular;
}

// One cell of a stage (or of the final combination) from its loaded
// neighbourhood: ld(j, which, s) returns component s of state j at the cell
// (which = 0), its x- (1), y- (2) and z-neighbour (3) upwind; the result
// (Z_i or y_{n+1}) goes to o[3]; ν partials into nu.
// FULL3D: the tiled kernels' geometry (upwind advection on all three axes)
// known at compile time, no per-cell operator branches
template <int NS, bool FINAL, int KIND, bool FULL3D, class Ld>
__device__ __forceinline__ void ark_cell(const FusedParams& p, const Geom& g, const Args& a, const Ld& ld,
                                         double (&o)[3], double (&nu)[kMaxNL], int64_t c) {
  double yn[3], ew[3], acc[3] = {0.0, 0.0, 0.0}, err[3] = {0.0, 0.0, 0.0}, q[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    yn[s] = ld(0, 0, s);
    const double tt = __fma_rn(p.rtol, fabs(yn[s]), p.atol);
    ew[s] = safe_mag(tt) ? rcp_nr2(tt) : 1.0 / tt;                     // ewt(y_n) (R30 reciprocal)
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    double fe[3], fi[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) q[s] = ld(j, 0, s);
    if (!FULL3D && g.expl == 2) {
      fe[0] = fe[1] = fe[2] = 0.0;
    } else if (!FULL3D && g.expl == 1) {
#pragma unroll
      for (int s = 0; s < 3; ++s) fe[s] = g.lam_E * q[s];
    } else {
#pragma unroll
      for (int s = 0; s < 3; ++s) {                                    // upwind stencil, contracted
        double f = __fma_rn(-g.ks, q[s], g.kx * ld(j, 1, s));
        if (FULL3D || g.has_y) f = __fma_rn(g.ky, ld(j, 2, s), f);
        if (FULL3D || g.has_z) f = __fma_rn(g.kz, ld(j, 3, s), f);
        fe[s] = f;
      }
    }
    implicit_rhs<KIND>(p, q, fi);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      acc[s] = __fma_rn(a.cE[j], fe[s], __fma_rn(a.cI[j], fi[s], acc[s]));
      if (FINAL) err[s] = __fma_rn(a.cErr[j], fe[s] + fi[s], err[s]);
    }
  }
  if (FINAL) {
    double w = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      o[s] = yn[s] + acc[s];
      const double e = err[s] * ew[s];
      w = __fma_rn(e, e, w);
    }
    nu[0] += w;
  } else {
    double d[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      d[s] = yn[s] + acc[s];
      o[s] = q[s];                                                     // predictor Z_{i-1}
    }
    if (!newton_ct<KIND>(p, d, o, ew, a.krt, nu)) {
#pragma unroll
      for (int s = 0; s < 3; ++s) o[s] = q[s];
      if (!newton_exact<KIND>(p, d, o, ew, a.krt, nu)) atomicMin(a.first, (unsigned long long)(c + 1));
    }
  }
}

// CTA partials of nu (fixed order), then the last CTA to arrive folds every
// CTA's row into a.sums (deterministic: lane-strided + shuffle tree)
template <int NT>
__device__ __forceinline__ void ark_epilogue(const Args& a, bool fin, double (&nu)[kMaxNL],
                                             double (&red)[NT / 32][kCols], int& last) {
  const int t = threadIdx.x;
  const int KC = fin ? 1 : a.krt;
  const int w = t >> 5, l = t & 31;
#pragma unroll
  for (int k = 0; k < kMaxNL; ++k) {
    const double v = warp_sum(nu[k]);
    if (l == 0) red[w][k + 1] = v;
  }
  __syncthreads();
  if (t >= 1 && t <= KC) {
    double s = red[0][t];
    for (int q2 = 1; q2 < NT / 32; ++q2) s = __dadd_rn(s, red[q2][t]);
    a.partials[(int64_t)blockIdx.x * kCols + t] = s;
    __threadfence();
  }
  __syncthreads();
  if (t == 0) last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int col = 1 + w; col <= KC; col += NT / 32) {
    // lane-strided with four independent chains (loads in flight), then a
    // fixed combination and shuffle tree: deterministic
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    const int nb = (int)gridDim.x;
    int b = l;
    for (; b + 96 < nb; b += 128) {
      v0 = __dadd_rn(v0, __ldcg(a.partials + (int64_t)b * kCols + col));
      v1 = __dadd_rn(v1, __ldcg(a.partials + (int64_t)(b + 32) * kCols + col));
      v2 = __dadd_rn(v2, __ldcg(a.partials + (int64_t)(b + 64) * kCols + col));
      v3 = __dadd_rn(v3, __ldcg(a.partials + (int64_t)(b + 96) * kCols + col));
    }
    for (; b < nb; b += 32) v0 = __dadd_rn(v0, __ldcg(a.partials + (int64_t)b * kCols + col));
    double v = warp_sum(__dadd_rn(__dadd_rn(v0, v1), __dadd_rn(v2, v3)));
    if (l == 0) a.sums[col] = v;
  }
  if (t == 0) *a.counter = 0u;
}

// Plain variant (any geometry): one thread per cell, grid-stride, loads
// from global memory (neighbours through L1/L2).
template <int NS, bool FINAL, int KIND>
__global__ void __launch_bounds__(kThreads, 2) k_ark_stage(FusedParams p, Geom g, Args a) {
  __shared__ double red[kThreads / 32][kCols];
  __shared__ int last;
  double nu[kMaxNL];
#pragma unroll
  for (int k = 0; k < kMaxNL; ++k) nu[k] = 0.0;
  const int64_t plane = g.nx * g.ny;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < g.G; c += (int64_t)gridDim.x * kThreads) {
    const int64_t k = c / plane, rem = c - k * plane, jy = rem / g.nx, i = rem - jy * g.nx;
    auto ld = [&](int j, int which, int s) -> double {
      const double* Zj = j == 0 ? a.y : a.Z[j - 1];
      const double* b = a.below[j];
      switch (which) {
        case 0: return Zj[3 * c + s];
        case 1: return __ldg((i > 0 ? Zj + 3 * (c - 1) : (g.dim == 1 ? b : Zj + 3 * (c + g.nx - 1))) + s);
        case 2: return __ldg((jy > 0 ? Zj + 3 * (c - g.nx) : Zj + 3 * (c + (g.ny - 1) * g.nx)) + s);
        default: return __ldg((k > 0 ? Zj + 3 * (c - plane) : b + 3 * (jy * g.nx + i)) + s);
      }
    };
    double o[3];
    ark_cell<NS, FINAL, KIND, false>(p, g, a, ld, o, nu, c);
#pragma unroll
    for (int s = 0; s < 3; ++s) a.out[3 * c + s] = o[s];
  }
  ark_epilogue<kThreads>(a, FINAL, nu, red, last);
}

// Tiled variant (3D upwind advection, nx % 128 == 0, both transverse axes
// present): persistent CTAs of 128 threads walk 128-cell tiles; per state
// the tile, its row-below and plane-below tiles and the two cells before
// the row start arrive by bulk copies (TMA) into a 2-stage shared ring, the
// result tile leaves by one bulk store — the fused SBDF step's data path
// (fused.cu), so the stage runs at the memory system's pace instead of per-
// thread load latency.
constexpr int kTile = 128;
template <int NS, int KS>
struct __align__(128) ArkTileSmem {
  double in[KS][NS][3][kTile * 3];
  double xm[KS][NS][8];
  double out[2][kTile * 3];
  uint64_t full[KS];
  double red[kTile / 32][kCols];
  int last;
};

// KS: input stages in the shared ring (2: double-buffered; 1: more CTAs per SM)
template <int NS, bool FINAL, int KIND, int KS>
__global__ void __launch_bounds__(kTile) k_ark_tile(FusedParams p, Geom g, Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ArkTileSmem<NS, KS>& S = *reinterpret_cast<ArkTileSmem<NS, KS>*>(smem_raw);
  const int t = threadIdx.x;
  const int64_t ntiles = g.G / kTile, plane = g.nx * g.ny;
  constexpr uint32_t kTB = kTile * 3 * 8;
  auto issue = [&](int64_t tile, int st) {           // thread 0
    const uint32_t c0 = (uint32_t)(tile * kTile), nx = (uint32_t)g.nx, ny = (uint32_t)g.ny;
    const uint32_t r = c0 / nx, i0 = c0 - r * nx, jr = r % ny, k = r / ny;
    const int64_t xprev = i0 > 0 ? (int64_t)c0 - 1 : (int64_t)c0 + g.nx - 1;
    sunbw::pipe::mbar_expect_tx(&S.full[st], NS * (3 * kTB + 48));
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const double* Zj = j == 0 ? a.y : a.Z[j - 1];
      sunbw::pipe::bulk_g2s(S.in[st][j][0], Zj + 3 * (int64_t)c0, kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.in[st][j][1], jr > 0 ? Zj + 3 * ((int64_t)c0 - g.nx) : Zj + 3 * ((int64_t)c0 + (g.ny - 1) * g.nx),
                     kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.in[st][j][2], k > 0 ? Zj + 3 * ((int64_t)c0 - plane) : a.below[j] + 3 * ((int64_t)jr * g.nx + i0),
                     kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.xm[st][j], Zj + 3 * (xprev - 1), 48, &S.full[st]);
    }
  };
  if (t == 0) {
    for (int st = 0; st < KS; ++st) sunbw::pipe::mbar_init(&S.full[st], 1);
    sunbw::pipe::fence_mbar_init();
  }
  __syncthreads();
  if (t == 0)
    for (int st = 0; st < KS; ++st) {
      const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
      if (tile < ntiles) issue(tile, st);
    }
  double nu[kMaxNL];
#pragma unroll
  for (int k = 0; k < kMaxNL; ++k) nu[k] = 0.0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % KS, ob = it & 1;
    sunbw::pipe::mbar_wait(&S.full[st], (uint32_t)((it / KS) & 1));
    const double* sb = &S.in[st][0][0][3 * t];        // this cell in the stage's tiles
    const double* sx = t > 0 ? &S.in[st][0][0][3 * (t - 1)] : &S.xm[st][0][3];
    const int xs = t > 0 ? 3 * kTile * 3 : 8;          // stride between states of sx
    auto ld = [&](int j, int which, int s) -> double {
      switch (which) {
        case 0: return sb[j * (3 * kTile * 3) + s];
        case 1: return sx[j * xs + s];
        case 2: return sb[j * (3 * kTile * 3) + kTile * 3 + s];
        default: return sb[j * (3 * kTile * 3) + 2 * kTile * 3 + s];
      }
    };
    double o[3];
    ark_cell<NS, FINAL, KIND, true>(p, g, a, ld, o, nu, tile * kTile + t);
#pragma unroll
    for (int s = 0; s < 3; ++s) S.out[ob][3 * t + s] = o[s];
    sunbw::pipe::fence_async_smem();
    if (t == 0) sunbw::pipe::bulk_wait_read_all();          // out[ob] of two tiles ago has left
    __syncthreads();
    if (t == 0) {
      sunbw::pipe::bulk_s2g(a.out + tile * (kTile * 3), S.out[ob], kTB);
      sunbw::pipe::bulk_commit();
      const int64_t next = tile + KS * (int64_t)gridDim.x;
      if (next < ntiles) issue(next, st);
    }
  }
  if (t == 0) sunbw::pipe::bulk_wait_all();
  ark_epilogue<kTile>(a, FINAL, nu, S.red, S.last);
}

// flags (singular per stage, 0/1) into column 0 of each stage's sums, and
// the singular records reset for the next round
__global__ void k_ark_pack(unsigned long long* first, double* sums) {
  const int s = threadIdx.x;
  if (s < kStages) {
    sums[s * kCols] = first[s] != ~0ull ? 1.0 : 0.0;
    first[s] = ~0ull;
  }
}
// (global) sums -> [flag, ν_1..ν_4] per stage; the final's column 1 = dsm
__global__ void k_ark_finalize(const double* sums, double nglobal, double* res) {
  const int t = threadIdx.x;
  if (t < kStages * kCols) res[t] = (t % kCols) == 0 ? sums[t] : __dsqrt_rn(__ddiv_rn(sums[t], nglobal));
}
// one rank: both in one launch
__global__ void k_ark_pack_finalize(unsigned long long* first, double nglobal, double* res, double* sums) {
  const int t = threadIdx.x;
  if (t < kStages * kCols) {
    const int st = t / kCols;
    res[t] = (t % kCols) == 0 ? (first[st] != ~0ull ? 1.0 : 0.0) : __dsqrt_rn(__ddiv_rn(sums[t], nglobal));
  }
  __syncthreads();
  if (t < kStages) first[t] = ~0ull;
}

}  // namespace

namespace sunbw {

BW_BrussParams bw_params(void* prob);
FusedParams fused_params(const BW_BrussParams& bp, bool first, double h, double rtol, double atol);

struct ArkFused {
  SUNBW_Context ctx;
  void* prob;
  ArkGeometry geo;
  int64_t nglobal;
  double* Z[3] = {};
  double* halo[4] = {};          // P > 1: the left neighbour's last plane of each state
  double* partials = nullptr;
  double* sums = nullptr;        // [stage 0..3][kCols] (stage 3 = final)
  double* res = nullptr;
  unsigned* counter = nullptr;
  unsigned long long* first = nullptr;
  double* h_res = nullptr;       // pinned
  int kpred[3] = {0, 0, 0};
  int grid = 1;                  // plain kernels
  bool tiled = false;            // 3D upwind, nx % 128 == 0: the TMA-tiled kernels
  int tgrid[5] = {};             // tiled kernels' persistent grid per NS (1..4)
  int tgrid_ks[5] = {};          // ... computed for this ring depth
};

ArkFused* ark_fused_create(SUNBW_Context ctx, void* prob, int64_t nglobal) {
  auto* F = new ArkFused();
  F->ctx = ctx;
  F->prob = prob;
  bw_ark_geometry(prob, &F->geo);
  F->nglobal = nglobal;
  const int64_t n = 3 * F->geo.G > 0 ? 3 * F->geo.G : 1;
  const int64_t need = (F->geo.G + kThreads - 1) / kThreads, cap = (int64_t)ctx->nsm * 2;
  F->grid = (int)(need < 1 ? 1 : (need < cap ? need : cap));
  bool ok = true;
  for (auto& z : F->Z) ok = ok && cudaMalloc(&z, sizeof(double) * n) == cudaSuccess;
  if (ctx_nranks(ctx) > 1)
    for (auto& hb : F->halo) ok = ok && cudaMalloc(&hb, sizeof(double) * F->geo.halo_len) == cudaSuccess;
  const ArkGeometry& g = F->geo;
  F->tiled = g.dim == 3 && g.expl == 0 && g.has_y && g.has_z && g.nx % kTile == 0 && g.G % kTile == 0 &&
             g.G > 0 && g.G < (int64_t(1) << 31);
  ok = ok && cudaMalloc(&F->partials, sizeof(double) * (int64_t)ctx->nsm * 16 * kCols) == cudaSuccess &&
       cudaMalloc(&F->sums, sizeof(double) * kStages * kCols) == cudaSuccess &&
       cudaMalloc(&F->res, sizeof(double) * kStages * kCols) == cudaSuccess &&
       cudaMalloc(&F->counter, sizeof(unsigned)) == cudaSuccess &&
       cudaMalloc(&F->first, sizeof(unsigned long long) * kStages) == cudaSuccess &&
       cudaHostAlloc(&F->h_res, sizeof(double) * kStages * kCols, cudaHostAllocDefault) == cudaSuccess &&
       cudaMemsetAsync(F->counter, 0, sizeof(unsigned), ctx->stream) == cudaSuccess &&
       cudaMemsetAsync(F->first, 0xFF, sizeof(unsigned long long) * kStages, ctx->stream) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    ark_fused_destroy(F);
    return nullptr;
  }
  return F;
}

void ark_fused_destroy(ArkFused* F) {
  if (!F) return;
  for (auto z : F->Z)
    if (z) cudaFree(z);
  for (auto hb : F->halo)
    if (hb) cudaFree(hb);
  if (F->partials) cudaFree(F->partials);
  if (F->sums) cudaFree(F->sums);
  if (F->res) cudaFree(F->res);
  if (F->counter) cudaFree(F->counter);
  if (F->first) cudaFree(F->first);
  if (F->h_res) cudaFreeHost(F->h_res);
  delete F;
}

namespace {

template <int NS, bool FINAL, int KIND, int KS>
int launch_tiled_ks(ArkFused* F, const FusedParams& p, const Geom& g, const Args& a) {
  const int bytes = (int)sizeof(ArkTileSmem<NS, KS>);
  auto fn = k_ark_tile<NS, FINAL, KIND, KS>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return SUNBW_ERR_CUDA;
  if (F->tgrid_ks[NS] != KS) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTile, bytes) != cudaSuccess || occ < 1)
      return SUNBW_ERR_CUDA;
    const int64_t ntiles = g.G / kTile, cap = (int64_t)F->ctx->nsm * (occ < 16 ? occ : 16);
    F->tgrid[NS] = (int)(ntiles < cap ? ntiles : cap);
    F->tgrid_ks[NS] = KS;
  }
  fn<<<F->tgrid[NS], kTile, bytes, F->ctx->stream>>>(p, g, a);
  return 0;
}

// stages per ring: SUNBW_ARK_KS (1 or 2) overrides, for A/B measurements
int ark_ks(int NS) {
  static const int ov = [] {
    const char* e = std::getenv("SUNBW_ARK_KS");
    return e ? std::atoi(e) : 0;
  }();
  (void)NS;
  return ov == 1 || ov == 2 ? ov : 1;   // measured: single-buffered rings (more CTAs per SM) are faster
}

template <int NS, bool FINAL, int KIND>
int launch_tiled(ArkFused* F, const FusedParams& p, const Geom& g, const Args& a) {
  return ark_ks(NS) == 1 ? launch_tiled_ks<NS, FINAL, KIND, 1>(F, p, g, a)
                         : launch_tiled_ks<NS, FINAL, KIND, 2>(F, p, g, a);
}

template <int KIND>
int launch_stage(ArkFused* F, int NS, bool fin, const FusedParams& p, const Geom& g, const Args& a) {
  cudaStream_t s = F->ctx->stream;
  if (F->tiled) {
    if (fin) return launch_tiled<4, true, KIND>(F, p, g, a);
    if (NS == 1) return launch_tiled<1, false, KIND>(F, p, g, a);
    if (NS == 2) return launch_tiled<2, false, KIND>(F, p, g, a);
    return launch_tiled<3, false, KIND>(F, p, g, a);
  }
  if (fin) {
    k_ark_stage<4, true, KIND><<<F->grid, kThreads, 0, s>>>(p, g, a);
  } else if (NS == 1) {
    k_ark_stage<1, false, KIND><<<F->grid, kThreads, 0, s>>>(p, g, a);
  } else if (NS == 2) {
    k_ark_stage<2, false, KIND><<<F->grid, kThreads, 0, s>>>(p, g, a);
  } else {
    k_ark_stage<3, false, KIND><<<F->grid, kThreads, 0, s>>>(p, g, a);
  }
  return 0;
}

}  // namespace

// One attempted step of size h from y (y_{n+1} -> ynew).  *nl_ok = 0 if a
// stage solve failed (zero pivot, or no convergence within maxnl): the
// caller recomputes with h/4.  newton_iters / setups: the oracle's counts
// for this attempt (stages reached, iterations performed).
int ark_fused_attempt(ArkFused* F, const double* y, double* ynew, double h, double rtol, double atol,
                      double tol_nl, int maxnl, int* nl_ok, double* dsm, int64_t* newton_iters,
                      int64_t* setups) {
  SUNBW_Context ctx = F->ctx;
  if (maxnl < 1 || maxnl > kMaxNL) return ctx_set_err(ctx, SUNBW_ERR_ARG);
  const ArkGeometry& G0 = F->geo;
  const bool multi = ctx_nranks(ctx) > 1;
  FusedParams p = fused_params(bw_params(F->prob), false, h, rtol, atol);
  p.gamma = h * kG;
  p.m21 = -p.gamma * 0.0;
  p.c22 = 1.0 + p.gamma / p.eps;
  Geom g{G0.dim, G0.expl, G0.has_y, G0.has_z, G0.nx, G0.ny, G0.nzl, G0.G, G0.kx, G0.ky, G0.kz,
         G0.kx + (G0.has_y ? G0.ky : 0.0) + (G0.has_z ? G0.kz : 0.0), G0.lam_E};
  const double* states[4] = {y, F->Z[0], F->Z[1], F->Z[2]};
  auto below = [&](int j) -> const double* {
    return multi ? F->halo[j] : states[j] + 3 * G0.G - G0.halo_len;
  };
  auto exchange = [&](int j) -> int {           // halo of state j (P > 1; advection only)
    if (!multi || G0.expl != 0) return 0;
    return ctx->comm->halo_shift(states[j] + 3 * G0.G - G0.halo_len, F->halo[j], (size_t)G0.halo_len,
                                 ctx->stream);
  };
  int Kr[4] = {0, 0, 0, 0};
  for (int i = 1; i <= 3; ++i) Kr[i] = F->kpred[i - 1] >= 1 && F->kpred[i - 1] <= maxnl ? F->kpred[i - 1] : maxnl;
  if (int e = exchange(0)) return ctx_set_err(ctx, e);
  int start = 1;
  int64_t iters = 0;                             // iterations of the stages already accepted (< start)
  for (int round = 0; round < 8; ++round) {
    // (the singular records were reset by the previous round's pack; the
    // stage sums are overwritten by each launch's fold)
    for (int i = start; i <= 4; ++i) {           // stages start..3, then the final combination (i = 4)
      const bool fin = i == 4;
      Args a{};
      a.y = y;
      for (int j = 0; j < 3; ++j) a.Z[j] = F->Z[j];
      for (int j = 0; j < 4; ++j) a.below[j] = below(j);
      a.out = fin ? ynew : F->Z[i - 1];
      for (int j = 0; j < 4; ++j) {
        a.cE[j] = fin ? h * kB[j] : h * kAE[i][j];
        a.cI[j] = fin ? h * kB[j] : h * kAI[i][j];
        a.cErr[j] = h * (kB[j] - kD[j]);
      }
      a.partials = F->partials;
      a.counter = F->counter;
      a.sums = F->sums + (i - 1) * kCols;
      a.first = F->first + (i - 1);
      a.krt = fin ? 1 : Kr[i];
      if (G0.G > 0) {
        const int e = bw_params(F->prob).kind == 1 ? launch_stage<1>(F, i, fin, p, g, a)
                                                   : launch_stage<0>(F, i, fin, p, g, a);
        if (e) return ctx_set_err(ctx, e);
        ctx->launches++;
        if (ctx_check_launch(ctx)) return SUNBW_ERR_CUDA;
      }
      if (!fin)
        if (int e = exchange(i)) return ctx_set_err(ctx, e);
    }
    if (multi) {
      k_ark_pack<<<1, 32, 0, ctx->stream>>>(F->first, F->sums);
      if (int e = ctx->comm->allreduce(F->sums, kStages * kCols, RED_SUM, ctx->stream)) return ctx_set_err(ctx, e);
      k_ark_finalize<<<1, 32, 0, ctx->stream>>>(F->sums, (double)F->nglobal, F->res);
      ctx->launches += 2;
    } else {
      k_ark_pack_finalize<<<1, 32, 0, ctx->stream>>>(F->first, (double)F->nglobal, F->res, F->sums);
      ctx->launches++;
    }
    if (cudaMemcpyAsync(F->h_res, F->res, sizeof(double) * kStages * kCols, cudaMemcpyDeviceToHost,
                        ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    // the oracle's decisions, stage by stage, from the first recomputed one
    int redo = 0;
    for (int i = start; i <= 3 && !redo; ++i) {
      const double* r = F->h_res + (i - 1) * kCols;
      if (r[0] != 0.0) {                         // zero pivot: no iterations, step recomputed
        *setups += i;
        *newton_iters += iters;
        *nl_ok = 0;
        return 0;
      }
      int kstar = 0;
      for (int k = 1; k <= Kr[i] && !kstar; ++k)
        if (r[k] <= tol_nl) kstar = k;
      if (kstar == Kr[i]) {
        iters += Kr[i];
        F->kpred[i - 1] = Kr[i];
        continue;
      }
      if (kstar > 0) {
        Kr[i] = kstar;                           // converged earlier: redo from this stage
      } else if (Kr[i] < maxnl) {
        Kr[i] = maxnl;                           // not yet converged: redo with the maximum
      } else {                                   // no convergence within maxnl
        *setups += i;
        *newton_iters += iters + maxnl;
        F->kpred[i - 1] = maxnl;
        *nl_ok = 0;
        return 0;
      }
      redo = i;
    }
    if (!redo) {
      *setups += 3;
      *newton_iters += iters;
      *nl_ok = 1;
      *dsm = F->h_res[3 * kCols + 1];
      return 0;
    }
    start = redo;
  }
  return ctx_set_err(ctx, SUNBW_ERR_CUDA);       // unreachable (each stage redoes at most twice)
}

}  // namespace sunbw
