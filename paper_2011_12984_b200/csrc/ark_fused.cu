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
#include <utility>

#include "sunbw_internal.h"
#include "cellstep.cuh"

namespace {

using namespace sunbw::cell;

constexpr int kThreads = 256;
constexpr int kMaxNL = 4;                // fused ARK: Newton iterations per stage <= 4
constexpr int kCols = kMaxNL + 1;        // partial columns: [unused, S_1..S_kMaxNL]
constexpr int kStages = 4;               // ARK3(2)4L[2]SA

// ARK3(2)4L[2]SA (Kennedy & Carpenter 2003), as in ark.cu / the oracle, for
// the kernels (constant-folded from the same literals as ark.cu's host copy)
__constant__ double d_kG = 1767732205903.0 / 4055673282236.0;
__constant__ double d_kAE[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 2027836641118.0, 0, 0, 0},
    {5535828885825.0 / 10492691773637.0, 788022342437.0 / 10882634858940.0, 0, 0},
    {6485989280629.0 / 16251701735622.0, -4246266847089.0 / 9704473918619.0,
     10755448449292.0 / 10357097424841.0, 0}};
__constant__ double d_kAI[4][4] = {
    {0, 0, 0, 0},
    {1767732205903.0 / 4055673282236.0, 1767732205903.0 / 4055673282236.0, 0, 0},
    {2746238789719.0 / 10658868560708.0, -640167445237.0 / 6845629431997.0,
     1767732205903.0 / 4055673282236.0, 0},
    {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
     11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0}};
__constant__ double d_kB[4] = {1471266399579.0 / 7840856788654.0, -4482444167858.0 / 7529755066697.0,
                               11266239266428.0 / 11593286722821.0, 1767732205903.0 / 4055673282236.0};
__constant__ double d_kD[4] = {2756255671327.0 / 12835298489170.0, -10771552573575.0 / 22201958757719.0,
                               9247589265047.0 / 10645013368117.0, 2193209047091.0 / 5459859503100.0};

struct Geom {
  int dim, expl, has_y, has_z;
  int64_t nx, ny, nzl, G;
  double kx, ky, kz, ks, lam_E;
};

// Device-resident controller state of one Evolve call (DESIGN R33): the
// step size, time, current buffer, per-stage predicted iteration counts and
// the statistics live here; the stage kernels read what they need at entry
// and k_ark_control updates it after every round, so the host never waits
// for a decision.  A round = the stages start..3 and the final combination
// of one attempted step (start > 1: the stages of an attempt redone with a
// corrected iteration count).
struct ArkCtl {
  double t, h;                  // time; step size (the current attempt's, clipped)
  double h_unclipped;           // proposal before clipping to t_end
  double t_end, tol_nl;
  int clipped, cur;             // cur: y_n = ybuf[cur]
  int start;                    // first stage of this round (1..4)
  int Kr[4];                    // Newton iterations per stage in this round ([1..3])
  int kpred[3];                 // the last accepted count per stage (prediction)
  int done;                     // 0 running; 1 t_end reached; 2 max_steps; 3 h underflow; 4 internal
  int maxnl, max_steps, fixed, rounds_att;
  long long attempts, accepted, rej_err, rej_nl, newton_iters, setups, iters_att, rounds;
};

// The host loop of BW_ArkEvolve (ark.cu) for one attempted step: stop
// conditions, clipping to t_end, the stage iteration predictions.
__device__ void ark_begin_attempt(ArkCtl& C) {
  if (!(C.t_end - C.t > 1e-12 * fmax(1.0, fabs(C.t_end)))) { C.done = 1; return; }
  if (C.attempts++ >= C.max_steps) { C.done = 2; return; }
  C.h_unclipped = C.h;
  C.clipped = C.t + C.h > C.t_end;
  if (C.clipped) C.h = C.t_end - C.t;
  if (C.h < 1e-14 * (1.0 + C.t)) { C.done = 3; return; }
  C.start = 1;
  C.iters_att = 0;
  C.rounds_att = 0;
  for (int i = 1; i <= 3; ++i)
    C.Kr[i] = C.kpred[i - 1] >= 1 && C.kpred[i - 1] <= C.maxnl ? C.kpred[i - 1] : C.maxnl;
}

// After a round: the oracle's stage decisions (R31 per stage: the first k
// with ν_k <= tol_nl; a zero pivot or no convergence within maxnl fails the
// attempt), then — once the attempt is complete — the error test and
// step-size update of BW_ArkEvolve, and the next attempt's setup.
__device__ void ark_control(ArkCtl& C, const double* res) {
  if (C.done) return;
  C.rounds++;
  bool nl_fail = false;
  int redo = 0;
  for (int i = C.start; i <= 3 && !redo && !nl_fail; ++i) {
    const double* r = res + (i - 1) * kCols;
    if (r[0] != 0.0) {                           // zero pivot: no iterations, step recomputed
      C.setups += i;
      C.newton_iters += C.iters_att;
      nl_fail = true;
      break;
    }
    int kstar = 0;
    for (int k = 1; k <= C.Kr[i] && !kstar; ++k)
      if (r[k] <= C.tol_nl) kstar = k;
    if (kstar == C.Kr[i]) {
      C.iters_att += C.Kr[i];
      C.kpred[i - 1] = C.Kr[i];
      continue;
    }
    if (kstar > 0) {
      C.Kr[i] = kstar;                           // converged earlier: redo from this stage
    } else if (C.Kr[i] < C.maxnl) {
      C.Kr[i] = C.maxnl;                         // not yet converged: redo with the maximum
    } else {                                     // no convergence within maxnl
      C.setups += i;
      C.newton_iters += C.iters_att + C.maxnl;
      C.kpred[i - 1] = C.maxnl;
      nl_fail = true;
      break;
    }
    redo = i;
  }
  if (!nl_fail && redo) {                        // the same attempt, stages redo..3 again
    C.start = redo;
    if (++C.rounds_att > 8) C.done = 4;          // unreachable (each stage redoes at most twice)
    return;
  }
  if (nl_fail) {
    C.rej_nl++;
    C.h *= 0.25;
  } else {
    C.setups += 3;
    C.newton_iters += C.iters_att;
    double dsm = res[3 * kCols + 1];
    double fac = dsm > 0.0 ? 0.9 * pow(dsm, -1.0 / 3.0) : 5.0;
    if (C.fixed) { dsm = 0.0; fac = 1.0; }
    if (dsm <= 1.0) {
      C.cur ^= 1;
      C.t += C.h;
      C.accepted++;
      C.h *= fmin(5.0, fmax(0.2, fac));
      if (C.clipped) C.h = fmax(C.h, C.h_unclipped);
    } else {
      C.rej_err++;
      C.h *= fmin(1.0, fmax(0.2, fac));
    }
  }
  ark_begin_attempt(C);
}

// the host's view of ArkCtl::done after a round (mapped pinned memory)
__device__ __forceinline__ void ark_publish(const ArkCtl& C, volatile int* host_done) {
  *host_done = C.done;
  __threadfence_system();
}

struct Args {
  double* ybuf[2];              // y_n / y_{n+1} (ArkCtl::cur selects y_n)
  const double* Z[3];           // Z_1..Z_3
  const double* below0[2];      // what sits under local plane 0 of ybuf[b] (halo or own wrap)
  const double* below[4];       // [1..3]: what sits under local plane 0 of Z_j ([0] unused)
  double* zout;                 // stage i: Z_i
  ArkCtl* ctl;
  int stage;                    // 1..3, 4 = final
  // P = 1, final: the fold of all stage sums and k_ark_control run in the
  // launch's last CTA (no separate launches between rounds)
  int control;
  double* sums_all;             // [stage][kCols]
  unsigned long long* first_all;
  double* res;
  double nglobal;
  volatile int* host_done;
  double* partials;             // [grid][kCols]
  unsigned* counter;            // in-kernel fold (self-resetting)
  double* sums;                 // this launch's kCols local sums
  unsigned long long* first;    // first singular cell (1-based), this stage
};

// The round's values, resolved at kernel entry from *ctl into shared memory
// (read where they are used rather than held in registers across the tile
// loop: the kernels are register-bound at 5 CTAs per SM).
struct RoundRT {
  const double* y;              // y_n = Z_0
  const double* below0;         // its plane under local plane 0
  double* out;                  // Z_i (stage) or y_{n+1} (final)
  double gamma, m21, c22;       // hγ̂, RN(-γ·0), 1 + γ/ε
  double cc[12];                // [h aE_ij | h aI_ij | -] (stage), [h b_j | h b_j | h (b_j - d_j)] (final)
  int krt;                      // Newton iterations of this launch
};

// The round's parameters from the controller state: false if this launch
// has nothing to do (Evolve finished, or a stage before the round's start).
// h-dependent constants are formed here with the host's operations (γ = h·γ̂,
// 1 + γ/ε, h·a_ij), so they carry the same bits the host would pass.
// false if this launch has nothing to do (Evolve finished, or a stage
// before the round's start); else R (shared) is filled — the caller
// synchronises the CTA before the first use.
template <int NS, bool FINAL>
__device__ __forceinline__ bool ark_resolve(const Args& a, const FusedParams& p, RoundRT& R) {
  static_assert(FINAL ? NS == 4 : (NS >= 1 && NS <= 3), "stage i reads i states");
  const ArkCtl& C = *a.ctl;
  if (C.done != 0 || NS < C.start) return false;
  const int t = threadIdx.x;
  const double h = C.h;
  if (t == 0) {
    const bool c1 = C.cur != 0;
    R.y = c1 ? a.ybuf[1] : a.ybuf[0];
    R.below0 = c1 ? a.below0[1] : a.below0[0];
    R.out = FINAL ? (c1 ? a.ybuf[0] : a.ybuf[1]) : a.zout;
    R.gamma = h * d_kG;
    R.m21 = -R.gamma * 0.0;
    R.c22 = 1.0 + R.gamma / p.eps;
    R.krt = FINAL ? 1 : C.Kr[NS & 3];
  }
  if (t < 4) {
    R.cc[t] = FINAL ? h * d_kB[t] : h * d_kAE[NS & 3][t];
    R.cc[4 + t] = FINAL ? h * d_kB[t] : h * d_kAI[NS & 3][t];
    R.cc[8 + t] = h * (d_kB[t] - d_kD[t]);
  }
  return true;
}

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

// Contracted modified Newton on one cell (R30 arithmetic, γ = gam):
// false (z untouched) if the Newton matrix needs a row exchange or a pivot
// leaves the guarded range — the caller then runs newton_exact.
template <int KIND>
__device__ __forceinline__ bool newton_ct(const FusedParams& p, const double gam, const double c22,
                                          const double (&d)[3], double (&z)[3],
                                          const double (&ew)[3], int krt, double (&nu)[kMaxNL]) {
  double a00, a01, a02, a10, a11, a12, a20, a21, a22;
  if (KIND == 1) {
    const double m = __fma_rn(-gam, p.lam_I, 1.0);
    a00 = a11 = a22 = m;
    a01 = a02 = a10 = a12 = a20 = a21 = 0.0;
  } else {
    const double u = z[0], v = z[1], w = z[2];
    const double uu = u * u, uv2 = (u + u) * v, gu = gam * u;
    a01 = -gam * uu;
    a00 = __fma_rn(-gam, uv2 - (w + 1.0), 1.0);
    a02 = gu;
    a10 = gam * (uv2 - w);
    a11 = 1.0 - a01;
    a12 = -gu;
    a20 = gam * w;
    a21 = 0.0;
    a22 = c22 + gu;
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
    double r0 = __fma_rn(gam, f[0], d[0] - z[0]);
    double r1 = __fma_rn(gam, f[1], d[1] - z[1]);
    double r2 = __fma_rn(gam, f[2], d[2] - z[2]);
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
// primitives of the composed path); returns false for a zero pivot.  Its
// operands travel in one local record built only on this (rare) path, and
// the parameters by value, so the fast path's arrays stay in registers.
struct ExactIO {
  double d[3], z[3], ew[3], nu[kMaxNL];
};
template <int KIND>
__device__ __noinline__ bool newton_exact(const FusedParams p, ExactIO& io, int krt) {
  double a[3][3], rp[3];
  newton_matrix<KIND>(p, io.z, a);
  bool singular = false;
  DivExact dv{true};
  const int code = lu3(a, rp, singular, dv);
  for (int it = 0; it < krt; ++it) {
    double f[3], r[3];
    reaction<KIND>(p, io.z, f, dv);
#pragma unroll
    for (int s = 0; s < 3; ++s) r[s] = __dadd_rn(__dadd_rn(io.d[s], __dmul_rn(p.gamma, f[s])), -io.z[s]);
    solve3(a, code, true, rp, r, dv);
    double w = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      io.z[s] = __dadd_rn(io.z[s], r[s]);
      const double q = r[s] * io.ew[s];
      w = __fma_rn(q, q, w);
    }
    io.nu[it] = w;
  }
  return !singular;
}

// One cell of a stage (or of the final combination), in two phases so that
// the tiled kernel can release its input tiles between them:
// ark_gather reads the cell's loaded neighbourhood — ld(j, which, s) returns
// component s of state j at the cell (which = 0), its x- (1), y- (2) and
// z-neighbour (3) upwind — and reduces it to the stage right-hand side d,
// the predictor q = Z_{i-1} and ewt(y_n) (FINAL: the result o = y_{n+1} and
// the error-norm partial); ark_solve then runs the stage's Newton iterations
// on registers only.
// FULL3D: the tiled kernels' geometry (upwind advection on all three axes)
// known at compile time, no per-cell operator branches
template <int NS, bool FINAL, int KIND, bool FULL3D, class Ld>
__device__ __forceinline__ void ark_gather(const FusedParams& p, const Geom& g, const RoundRT& R, const Ld& ld,
                                           double (&d)[3], double (&q)[3], double (&ew)[3],
                                           double (&nu)[kMaxNL]) {
  double yn[3], acc[3] = {0.0, 0.0, 0.0}, err[3] = {0.0, 0.0, 0.0};
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
      acc[s] = __fma_rn(R.cc[j], fe[s], __fma_rn(R.cc[4 + j], fi[s], acc[s]));
      if (FINAL) err[s] = __fma_rn(R.cc[8 + j], fe[s] + fi[s], err[s]);
    }
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) d[s] = yn[s] + acc[s];                   // FINAL: y_{n+1}; stage: rhs
  if (FINAL) {
    double w = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double e = err[s] * ew[s];
      w = __fma_rn(e, e, w);
    }
    nu[0] += w;
  }
}

// Newton on one stage cell from the predictor q; the stage value to o.
template <int KIND>
__device__ __forceinline__ void ark_solve(const FusedParams& p, const RoundRT& R, const Args& a, const double (&d)[3],
                                          const double (&q)[3], const double (&ew)[3], double (&o)[3],
                                          double (&nu)[kMaxNL], int64_t c) {
#pragma unroll
  for (int s = 0; s < 3; ++s) o[s] = q[s];                             // predictor Z_{i-1}
  if (!newton_ct<KIND>(p, R.gamma, R.c22, d, o, ew, R.krt, nu)) {
    ExactIO io;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      io.d[s] = d[s];
      io.z[s] = q[s];
      io.ew[s] = ew[s];
    }
    FusedParams pe = p;
    pe.gamma = R.gamma;
    pe.m21 = R.m21;
    pe.c22 = R.c22;
    const bool ok = newton_exact<KIND>(pe, io, R.krt);
#pragma unroll
    for (int s = 0; s < 3; ++s) o[s] = io.z[s];
#pragma unroll
    for (int k = 0; k < kMaxNL; ++k)
      if (k < R.krt) nu[k] += io.nu[k];
    if (!ok) atomicMin(a.first, (unsigned long long)(c + 1));
  }
}

template <int NS, bool FINAL, int KIND, bool FULL3D, class Ld>
__device__ __forceinline__ void ark_cell(const FusedParams& p, const Geom& g, const RoundRT& R, const Args& a,
                                         const Ld& ld, double (&o)[3], double (&nu)[kMaxNL], int64_t c) {
  double d[3], q[3], ew[3];
  ark_gather<NS, FINAL, KIND, FULL3D>(p, g, R, ld, d, q, ew, nu);
  if (FINAL) {
#pragma unroll
    for (int s = 0; s < 3; ++s) o[s] = d[s];
  } else {
    ark_solve<KIND>(p, R, a, d, q, ew, o, nu, c);
  }
}

// CTA partials of nu (fixed order), then the last CTA to arrive folds every
// CTA's row into a.sums (deterministic: lane-strided + shuffle tree)
template <int NT>
__device__ __forceinline__ void ark_epilogue(const Args& a, bool fin, int krt, double (&nu)[kMaxNL],
                                             double (&red)[NT / 32][kCols], int& last) {
  const int t = threadIdx.x;
  const int KC = fin ? 1 : krt;
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
  if (!fin || !a.control) return;
  __syncthreads();                             // this CTA's sums are visible to it
  if (t < kStages * kCols) {                   // k_ark_pack_finalize
    const int st = t / kCols;
    a.res[t] = (t % kCols) == 0 ? (a.first_all[st] != ~0ull ? 1.0 : 0.0)
                                : __dsqrt_rn(__ddiv_rn(__ldcg(a.sums_all + t), a.nglobal));
  }
  __syncthreads();
  if (t < kStages) a.first_all[t] = ~0ull;
  if (t == 0) {
    ark_control(*a.ctl, a.res);
    ark_publish(*a.ctl, a.host_done);
  }
}

// Plain variant (any geometry): one thread per cell, grid-stride, loads
// from global memory (neighbours through L1/L2).
template <int NS, bool FINAL, int KIND>
__global__ void __launch_bounds__(kThreads, 2) k_ark_stage(FusedParams p, Geom g, Args a) {
  __shared__ RoundRT R;
  if (!ark_resolve<NS, FINAL>(a, p, R)) return;
  __syncthreads();
  __shared__ double red[kThreads / 32][kCols];
  __shared__ int last;
  double nu[kMaxNL];
#pragma unroll
  for (int k = 0; k < kMaxNL; ++k) nu[k] = 0.0;
  const int64_t plane = g.nx * g.ny;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < g.G; c += (int64_t)gridDim.x * kThreads) {
    const int64_t k = c / plane, rem = c - k * plane, jy = rem / g.nx, i = rem - jy * g.nx;
    auto ld = [&](int j, int which, int s) -> double {
      const double* Zj = j == 0 ? R.y : a.Z[j - 1];
      const double* b = j == 0 ? R.below0 : a.below[j];
      switch (which) {
        case 0: return Zj[3 * c + s];
        case 1: return __ldg((i > 0 ? Zj + 3 * (c - 1) : (g.dim == 1 ? b : Zj + 3 * (c + g.nx - 1))) + s);
        case 2: return __ldg((jy > 0 ? Zj + 3 * (c - g.nx) : Zj + 3 * (c + (g.ny - 1) * g.nx)) + s);
        default: return __ldg((k > 0 ? Zj + 3 * (c - plane) : b + 3 * (jy * g.nx + i)) + s);
      }
    };
    double o[3];
    ark_cell<NS, FINAL, KIND, false>(p, g, R, a, ld, o, nu, c);
#pragma unroll
    for (int s = 0; s < 3; ++s) R.out[3 * c + s] = o[s];
  }
  ark_epilogue<kThreads>(a, FINAL, R.krt, nu, red, last);
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
  RoundRT rt;
  int last;
};

// KS: input stages in the shared ring (2: double-buffered; 1: more CTAs per
// SM).  ER (early release): the input tiles are released — and the ring
// slot refilled with the tile KS ahead — as soon as every thread has reduced
// its neighbourhood to registers (ark_gather), so the copies run under the
// stage's Newton iterations instead of after them.
template <int NS, bool FINAL, int KIND, int KS, bool ER>
__global__ void __launch_bounds__(kTile) k_ark_tile(FusedParams p, Geom g, Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ArkTileSmem<NS, KS>& S = *reinterpret_cast<ArkTileSmem<NS, KS>*>(smem_raw);
  RoundRT& R = S.rt;                                      // filled by ark_resolve below
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
      const double* Zj = j == 0 ? R.y : a.Z[j - 1];
      sunbw::pipe::bulk_g2s(S.in[st][j][0], Zj + 3 * (int64_t)c0, kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.in[st][j][1], jr > 0 ? Zj + 3 * ((int64_t)c0 - g.nx) : Zj + 3 * ((int64_t)c0 + (g.ny - 1) * g.nx),
                     kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.in[st][j][2], k > 0 ? Zj + 3 * ((int64_t)c0 - plane) : (j == 0 ? R.below0 : a.below[j]) + 3 * ((int64_t)jr * g.nx + i0),
                     kTB, &S.full[st]);
      sunbw::pipe::bulk_g2s(S.xm[st][j], Zj + 3 * (xprev - 1), 48, &S.full[st]);
    }
  };
  if (t == 0) {
    for (int st = 0; st < KS; ++st) sunbw::pipe::mbar_init(&S.full[st], 1);
    sunbw::pipe::fence_mbar_init();
  }
  if (!ark_resolve<NS, FINAL>(a, p, R)) return;
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
    const int64_t next = tile + KS * (int64_t)gridDim.x;
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
    double d[3], q[3], ew[3], o[3];
    ark_gather<NS, FINAL, KIND, true>(p, g, R, ld, d, q, ew, nu);
    if (ER) {
      __syncthreads();                                 // every thread is done with in[st]
      if (t == 0 && next < ntiles) issue(next, st);
    }
    if (FINAL) {
#pragma unroll
      for (int s = 0; s < 3; ++s) o[s] = d[s];
    } else {
      ark_solve<KIND>(p, R, a, d, q, ew, o, nu, tile * kTile + t);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) S.out[ob][3 * t + s] = o[s];
    sunbw::pipe::fence_async_smem();
    if (t == 0) sunbw::pipe::bulk_wait_read_all();          // out[ob] of two tiles ago has left
    __syncthreads();
    if (t == 0) {
      sunbw::pipe::bulk_s2g(R.out + tile * (kTile * 3), S.out[ob], kTB);
      sunbw::pipe::bulk_commit();
      if (!ER && next < ntiles) issue(next, st);
    }
  }
  if (t == 0) sunbw::pipe::bulk_wait_all();
  ark_epilogue<kTile>(a, FINAL, R.krt, nu, S.red, S.last);
}

// flags (singular per stage, 0/1) into column 0 of each stage's sums, and
// the singular records reset for the next round
__global__ void k_ark_pack(const ArkCtl* C, unsigned long long* first, double* sums) {
  if (C->done) return;
  const int s = threadIdx.x;
  if (s < kStages) {
    sums[s * kCols] = first[s] != ~0ull ? 1.0 : 0.0;
    first[s] = ~0ull;
  }
}
// (global) sums -> [flag, ν_1..ν_4] per stage; the final's column 1 = dsm
__global__ void k_ark_finalize(const ArkCtl* C, const double* sums, double nglobal, double* res) {
  if (C->done) return;
  const int t = threadIdx.x;
  if (t < kStages * kCols) res[t] = (t % kCols) == 0 ? sums[t] : __dsqrt_rn(__ddiv_rn(sums[t], nglobal));
}
__global__ void k_ark_begin(ArkCtl* C, volatile int* host_done) {
  ark_begin_attempt(*C);
  ark_publish(*C, host_done);
}
__global__ void k_ark_control(ArkCtl* C, const double* res, volatile int* host_done) {
  ark_control(*C, res);
  ark_publish(*C, host_done);
}

// one rank: both in one launch
__global__ void k_ark_pack_finalize(const ArkCtl* C, unsigned long long* first, double nglobal, double* res,
                                    double* sums) {
  if (C->done) return;
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
  double* halo[4] = {};          // P > 1: the left neighbour's last plane of Z_1..Z_3 ([1..3])
  double* halo0[2] = {};         // P > 1: ... of each y buffer
  double* partials = nullptr;
  double* sums = nullptr;        // [stage 0..3][kCols] (stage 3 = final)
  double* res = nullptr;
  unsigned* counter = nullptr;
  unsigned long long* first = nullptr;
  ArkCtl* ctl = nullptr;         // device controller state
  ArkCtl* h_ctl = nullptr;       // pinned staging for the controller state
  int* h_done = nullptr;         // mapped pinned [2]: ArkCtl::done after round k in slot k & 1
  int* d_done = nullptr;         // ... its device address
  cudaEvent_t ev[2] = {};
  cudaStream_t cap = nullptr;    // P = 1: one round captured as a graph (per y buffer pair)
  cudaGraphExec_t gexec = nullptr;
  const double* gkey[2] = {};
  int64_t glaunches = 0;
  int kpred[3] = {0, 0, 0};
  int grid = 1;                  // plain kernels
  bool tiled = false;            // 3D upwind, nx % 128 == 0: the TMA-tiled kernels
  int tgrid[5] = {};             // tiled kernels' persistent grid per NS (1..4)
  int tgrid_ks[5] = {};          // ... computed for this ring configuration
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
  if (ctx_nranks(ctx) > 1) {
    for (int j = 1; j < 4; ++j) ok = ok && cudaMalloc(&F->halo[j], sizeof(double) * F->geo.halo_len) == cudaSuccess;
    for (auto& hb : F->halo0) ok = ok && cudaMalloc(&hb, sizeof(double) * F->geo.halo_len) == cudaSuccess;
  }
  const ArkGeometry& g = F->geo;
  F->tiled = g.dim == 3 && g.expl == 0 && g.has_y && g.has_z && g.nx % kTile == 0 && g.G % kTile == 0 &&
             g.G > 0 && g.G < (int64_t(1) << 31);
  ok = ok && cudaMalloc(&F->partials, sizeof(double) * (int64_t)ctx->nsm * 16 * kCols) == cudaSuccess &&
       cudaMalloc(&F->sums, sizeof(double) * kStages * kCols) == cudaSuccess &&
       cudaMalloc(&F->res, sizeof(double) * kStages * kCols) == cudaSuccess &&
       cudaMalloc(&F->counter, sizeof(unsigned)) == cudaSuccess &&
       cudaMalloc(&F->first, sizeof(unsigned long long) * kStages) == cudaSuccess &&
       cudaMalloc(&F->ctl, sizeof(ArkCtl)) == cudaSuccess &&
       cudaHostAlloc(&F->h_ctl, sizeof(ArkCtl), cudaHostAllocDefault) == cudaSuccess &&
       cudaHostAlloc(&F->h_done, 2 * sizeof(int), cudaHostAllocMapped) == cudaSuccess &&
       cudaHostGetDevicePointer((void**)&F->d_done, F->h_done, 0) == cudaSuccess &&
       cudaEventCreateWithFlags(&F->ev[0], cudaEventDisableTiming) == cudaSuccess &&
       cudaEventCreateWithFlags(&F->ev[1], cudaEventDisableTiming) == cudaSuccess &&
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
  for (auto hb : F->halo0)
    if (hb) cudaFree(hb);
  if (F->partials) cudaFree(F->partials);
  if (F->sums) cudaFree(F->sums);
  if (F->res) cudaFree(F->res);
  if (F->counter) cudaFree(F->counter);
  if (F->first) cudaFree(F->first);
  if (F->ctl) cudaFree(F->ctl);
  if (F->h_ctl) cudaFreeHost(F->h_ctl);
  if (F->h_done) cudaFreeHost(F->h_done);
  for (auto e : F->ev)
    if (e) cudaEventDestroy(e);
  if (F->gexec) cudaGraphExecDestroy(F->gexec);
  if (F->cap) cudaStreamDestroy(F->cap);
  delete F;
}

namespace {

template <class Kern>
int launch_ark(Kern fn, int grid, int block, int smem, cudaStream_t s, const FusedParams& p, const Geom& g,
               const Args& a) {
  fn<<<grid, block, smem, s>>>(p, g, a);
  return 0;
}

template <int NS, bool FINAL, int KIND, int KS, bool ER>
int launch_tiled_ks(ArkFused* F, const FusedParams& p, const Geom& g, const Args& a) {
  const int bytes = (int)sizeof(ArkTileSmem<NS, KS>);
  auto fn = k_ark_tile<NS, FINAL, KIND, KS, ER>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return SUNBW_ERR_CUDA;
  const int cfg = KS * 2 + (ER ? 1 : 0);
  if (F->tgrid_ks[NS] != cfg) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTile, bytes) != cudaSuccess || occ < 1)
      return SUNBW_ERR_CUDA;
    const int64_t ntiles = g.G / kTile, cap = (int64_t)F->ctx->nsm * (occ < 16 ? occ : 16);
    F->tgrid[NS] = (int)(ntiles < cap ? ntiles : cap);
    F->tgrid_ks[NS] = cfg;
  }
  return launch_ark(fn, F->tgrid[NS], kTile, bytes, F->ctx->stream, p, g, a);
}

// ring configuration per stage kind (NS = 1..3 stages, 4 = final):
// SUNBW_ARK_CFG = four digits, one per NS, each 1 = (KS 1), 2 = (KS 2),
// 3 = (KS 1, early release), 4 = (KS 2, early release) — for A/B runs
int ark_cfg(int NS) {
  static const char* ov = std::getenv("SUNBW_ARK_CFG");
  static const char kDefault[] = "3333";      // measured (r02 ARK A/B, DESIGN R33)
  const char* c = ov && std::strlen(ov) == 4 ? ov : kDefault;
  const int v = c[NS - 1] - '0';
  return v >= 1 && v <= 4 ? v : 1;
}

template <int NS, bool FINAL, int KIND>
int launch_tiled(ArkFused* F, const FusedParams& p, const Geom& g, const Args& a) {
  switch (ark_cfg(NS)) {
    case 2: return launch_tiled_ks<NS, FINAL, KIND, 2, false>(F, p, g, a);
    case 3: return launch_tiled_ks<NS, FINAL, KIND, 1, true>(F, p, g, a);
    case 4: return launch_tiled_ks<NS, FINAL, KIND, 2, true>(F, p, g, a);
    default: return launch_tiled_ks<NS, FINAL, KIND, 1, false>(F, p, g, a);
  }
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
    return launch_ark(k_ark_stage<4, true, KIND>, F->grid, kThreads, 0, s, p, g, a);
  } else if (NS == 1) {
    return launch_ark(k_ark_stage<1, false, KIND>, F->grid, kThreads, 0, s, p, g, a);
  } else if (NS == 2) {
    return launch_ark(k_ark_stage<2, false, KIND>, F->grid, kThreads, 0, s, p, g, a);
  } else {
    return launch_ark(k_ark_stage<3, false, KIND>, F->grid, kThreads, 0, s, p, g, a);
  }
  return 0;
}

}  // namespace

// BW_ArkEvolve's loop for the fused stages, driven from the device
// (DESIGN R33): every round — the stage kernels, the final combination, the
// fold (+ allreduce at P > 1) and k_ark_control — is enqueued without
// waiting for the previous one's decision; each kernel reads the round's
// h, current buffer, start stage and iteration counts from ArkCtl and exits
// at once if it has nothing to do.  At P = 1 a round is the four stage
// launches alone (the final launch's last CTA folds the norms and runs the
// controller).  The controller publishes ArkCtl::done to mapped pinned
// memory; the host keeps two rounds in flight, waits for the older one's
// event and reads the flag to know when the Evolve call has finished (at
// most one no-op round follows).
// *y / *ynew are swapped if the result ended in the second buffer.
int ark_fused_evolve(ArkFused* F, double** y, double** ynew, double* t, double* h, double t_end,
                     const BW_ArkOptions& opt, BW_ArkStats* st, int* rc) {
  SUNBW_Context ctx = F->ctx;
  if (opt.maxnl < 1 || opt.maxnl > kMaxNL) return ctx_set_err(ctx, SUNBW_ERR_ARG);
  const ArkGeometry& G0 = F->geo;
  const bool multi = ctx_nranks(ctx) > 1;
  cudaStream_t s = ctx->stream;                  // (switched to the capture stream while capturing)
  const FusedParams p = fused_params(bw_params(F->prob), false, 0.0, opt.rtol, opt.atol);  // γ, c22: per round
  const Geom g{G0.dim, G0.expl, G0.has_y, G0.has_z, G0.nx, G0.ny, G0.nzl, G0.G, G0.kx, G0.ky, G0.kz,
               G0.kx + (G0.has_y ? G0.ky : 0.0) + (G0.has_z ? G0.kz : 0.0), G0.lam_E};
  double* yb[2] = {*y, *ynew};
  auto wrap = [&](const double* v) { return v + 3 * G0.G - G0.halo_len; };
  ArkCtl& c = *F->h_ctl;
  std::memset(&c, 0, sizeof(c));
  c.t = *t;
  c.h = *h;
  c.t_end = t_end;
  c.tol_nl = opt.tol_nl;
  c.maxnl = opt.maxnl;
  c.max_steps = opt.max_steps;
  c.fixed = opt.fixed;
  for (int i = 0; i < 3; ++i) c.kpred[i] = F->kpred[i];
  if (cudaMemcpyAsync(F->ctl, &c, sizeof(ArkCtl), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  ((volatile int*)F->h_done)[0] = ((volatile int*)F->h_done)[1] = 0;
  k_ark_begin<<<1, 1, 0, s>>>(F->ctl, F->d_done);
  ctx->launches++;
  Args base{};
  for (int b = 0; b < 2; ++b) {
    base.ybuf[b] = yb[b];
    base.below0[b] = multi ? F->halo0[b] : wrap(yb[b]);
  }
  for (int j = 0; j < 3; ++j) {
    base.Z[j] = F->Z[j];
    base.below[j + 1] = multi ? F->halo[j + 1] : wrap(F->Z[j]);
  }
  base.ctl = F->ctl;
  base.partials = F->partials;
  base.counter = F->counter;
  base.control = multi ? 0 : 1;
  base.sums_all = F->sums;
  base.first_all = F->first;
  base.res = F->res;
  base.nglobal = (double)F->nglobal;
  base.host_done = F->d_done;
  const bool kind1 = bw_params(F->prob).kind == 1;
  auto exchange = [&](const double* v, double* dst) -> int {   // P > 1, advection only
    if (!multi || G0.expl != 0) return 0;
    return ctx->comm->halo_shift(wrap(v), dst, (size_t)G0.halo_len, s);
  };
  // slot: where this round's separate controller launch publishes done
  // (P > 1: each rank must stop after the same round, so the host reads the
  // state after round k - 1 — slot (k - 1) & 1 — not whatever is latest)
  auto round = [&](int slot) -> int {
    for (int b = 0; b < 2; ++b)
      if (int e = exchange(yb[b], F->halo0[b])) return e;
    for (int i = 1; i <= 4; ++i) {
      const bool fin = i == 4;
      Args a = base;
      a.stage = i;
      a.zout = fin ? nullptr : F->Z[i - 1];
      a.sums = F->sums + (i - 1) * kCols;
      a.first = F->first + (i - 1);
      if (G0.G > 0) {
        const int e = kind1 ? launch_stage<1>(F, i, fin, p, g, a) : launch_stage<0>(F, i, fin, p, g, a);
        if (e) return e;
        ctx->launches++;
        if (ctx_check_launch(ctx)) return SUNBW_ERR_CUDA;
      }
      if (!fin)
        if (int e = exchange(F->Z[i - 1], F->halo[i])) return e;
    }
    if (multi) {
      k_ark_pack<<<1, 32, 0, s>>>(F->ctl, F->first, F->sums);
      if (int e = ctx->comm->allreduce(F->sums, kStages * kCols, RED_SUM, s)) return e;
      k_ark_finalize<<<1, 32, 0, s>>>(F->ctl, F->sums, (double)F->nglobal, F->res);
      k_ark_control<<<1, 1, 0, s>>>(F->ctl, F->res, F->d_done + slot);
      ctx->launches += 3;
    } else if (G0.G == 0) {                      // (no final launch to carry the controller)
      k_ark_pack_finalize<<<1, 32, 0, s>>>(F->ctl, F->first, (double)F->nglobal, F->res, F->sums);
      k_ark_control<<<1, 1, 0, s>>>(F->ctl, F->res, F->d_done + slot);
      ctx->launches += 2;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : SUNBW_ERR_CUDA;
  };
  // P = 1: the round's four launches replayed from a graph (the kernels take
  // everything that changes between rounds from ArkCtl)
  const bool use_graph = !multi && G0.G > 0;
  if (use_graph && (!F->gexec || F->gkey[0] != yb[0] || F->gkey[1] != yb[1])) {
    if (F->gexec) cudaGraphExecDestroy(F->gexec);
    F->gexec = nullptr;
    if (!F->cap && cudaStreamCreateWithFlags(&F->cap, cudaStreamNonBlocking) != cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    cudaStream_t user = ctx->stream;
    const int64_t l0 = ctx->launches.load();
    cudaGraph_t gr = nullptr;
    int rc0 = 0;
    ctx->stream = s = F->cap;
    if (cudaStreamBeginCapture(F->cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      rc0 = SUNBW_ERR_CUDA;
    } else {
      rc0 = round(0);                            // (one rank: the final launch publishes in slot 0)
      if (cudaStreamEndCapture(F->cap, &gr) != cudaSuccess && !rc0) rc0 = SUNBW_ERR_CUDA;
    }
    ctx->stream = s = user;
    F->glaunches = ctx->launches.load() - l0;
    ctx->launches -= F->glaunches;
    if (!rc0 && cudaGraphInstantiate(&F->gexec, gr, 0) != cudaSuccess) rc0 = SUNBW_ERR_CUDA;
    if (gr) cudaGraphDestroy(gr);
    if (rc0) {
      cudaGetLastError();
      F->gexec = nullptr;
      return ctx_set_err(ctx, rc0 < 0 ? rc0 : SUNBW_ERR_CUDA);
    }
    F->gkey[0] = yb[0];
    F->gkey[1] = yb[1];
  }
  // each attempt takes at most 9 rounds (stages redone at most twice each)
  const int64_t max_rounds = 9 * ((int64_t)opt.max_steps + 1) + 2;
  for (int64_t k = 0;; ++k) {
    if (k > max_rounds) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    if (use_graph) {
      if (cudaGraphLaunch(F->gexec, s) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      ctx->launches += F->glaunches;
    } else if (int e = round((int)(k & 1))) {
      return ctx_set_err(ctx, e);
    }
    if (cudaEventRecord(F->ev[k & 1], s) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    if (k > 0) {
      if (cudaEventSynchronize(F->ev[(k - 1) & 1]) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      if (((volatile int*)F->h_done)[use_graph ? 0 : (int)((k - 1) & 1)]) break;
    }
  }
  if (cudaMemcpyAsync(&c, F->ctl, sizeof(ArkCtl), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (c.done == 4) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  *rc = c.done == 2 ? 1 : c.done == 3 ? 2 : 0;
  *t = c.t;
  *h = c.h;
  if (c.cur) std::swap(*y, *ynew);
  for (int i = 0; i < 3; ++i) F->kpred[i] = c.kpred[i];
  st->accepted += c.accepted;
  st->rejected_err += c.rej_err;
  st->rejected_nl += c.rej_nl;
  st->newton_iters += c.newton_iters;
  st->setups += c.setups;
  return 0;
}

}  // namespace sunbw
