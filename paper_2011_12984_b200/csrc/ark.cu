// ark.cu — adaptive IMEX additive Runge–Kutta driver: the integrator of the
// paper's demonstration (ARKODE IMEX: advection explicit, stiff
// reaction implicit), with temporal error control by global WRMS reductions
// and recomputation of a step with a smaller h when a nonlinear solve fails
// (P:394).  Tableau ARK3(2)4L[2]SA (Kennedy & Carpenter; DESIGN R26).
//
// Host control logic, device data (the paper's split): every vector
// operation is one of the library's kernels — the stage right-hand sides,
// the new solution and the embedded error are single N_VLinearCombination
// launches over up to 9 vectors; each stage is solved by modified Newton
// with the batched block LU (the task-local solver); the stage
// convergence and the error test are global reductions read on the host.
//
// Stage i (a^I_11 = 0):  Z_i = y_n + h Σ_{j<i}(aE_ij FE_j + aI_ij FI_j) + hγ f_I(Z_i)
// Newton on a stage: predictor Z_{i-1}, M = I − hγ J(Z_{i-1}), r = rhs + hγ
// f_I(Z) − Z, δ = M⁻¹ r, Z += δ, ν = WRMS(δ, ewt) ≤ tol_nl; no convergence
// in maxnl iterations (or a zero pivot) → recompute the step with h/4.
// Step: y_{n+1} = y_n + h Σ b_i(FE_i + FI_i); e = h Σ (b_i − d_i)(FE_i + FI_i);
// accept iff WRMS(e, ewt(y_n)) ≤ 1; h ← h·clamp(0.9·dsm^(−1/3), 0.2, 5)
// (rejection: upper clamp 1).

#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

#include "sunbw_internal.h"

namespace sunbw {
int bw_reaction(void* prob, const double* y, double* f);
int bw_jacobian(void* prob, const double* y, double* J);
int bw_halo(void* prob, const double* y);
int bw_advection_stencil(void* prob, const double* y, double* f);
int64_t bw_local_cells(void* prob);
}  // namespace sunbw

namespace {

// ARK3(2)4L[2]SA (Kennedy & Carpenter 2003), as in SUNDIALS ARKODE
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

struct Ark {
  void* prob;
  SUNBW_Context ctx;
  BW_ArkOptions opt;
  int64_t G, n, nglobal;
  double *y, *Z, *rhs, *ewt, *tmp, *r, *delta, *fI, *ynew, *err, *M;
  double* FE[4];
  double* FI[4];
  int32_t* piv;
  unsigned long long* d_first;
  double t = 0.0, h = 0.0;
  BW_ArkStats st{};
  sunbw::ArkFused* fused = nullptr;   // opt.fused: one kernel per stage (ark_fused.cu, R32)
};

double host_wrms(SUNBW_Context ctx, int64_t n, int64_t nglob, const double* x, const double* w, int* e) {
  *e = sunbw::reduce(ctx, sunbw::RK_WSQR, sunbw::RF_WRMS, n, nglob, x, w, nullptr, ctx->d_red,
                     ctx->h_slot_dev, true, nullptr);
  if (*e) return NAN;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    *e = ctx_set_err(ctx, SUNBW_ERR_CUDA);
    return NAN;
  }
  return ((volatile double*)ctx->h_slot)[0];
}

#define TRY(x)             \
  do {                     \
    int e_ = (x);          \
    if (e_ < 0) return e_; \
  } while (0)

// stage right-hand sides: f_E (with the halo exchange) and f_I
int eval_rhs(Ark* A, const double* Z, double* fe, double* fi) {
  TRY(sunbw::bw_halo(A->prob, Z));
  TRY(sunbw::bw_advection_stencil(A->prob, Z, fe));
  TRY(sunbw::bw_reaction(A->prob, Z, fi));
  return 0;
}

// one attempted step with A->h; *ok = 0 on a nonlinear failure
int attempt(Ark* A, int* nl_ok, double* dsm) {
  SUNBW_Context ctx = A->ctx;
  const int64_t n = A->n, G = A->G;
  const double h = A->h, hg = h * kG;
  TRY(sunbw::abs_(ctx, n, A->y, A->tmp, nullptr));
  TRY(sunbw::scale(ctx, n, A->opt.rtol, A->tmp, A->tmp, nullptr));
  TRY(sunbw::add_const(ctx, n, A->tmp, A->opt.atol, A->tmp, nullptr));
  TRY(sunbw::inv(ctx, n, A->tmp, A->ewt, nullptr));
  *nl_ok = 1;
  for (int i = 0; i < 4; ++i) {
    if (i == 0) {
      TRY(sunbw::scale(ctx, n, 1.0, A->y, A->Z, nullptr));
    } else {
      double c[9];
      const double* X[9];
      int k = 0;
      c[k] = 1.0;
      X[k++] = A->y;
      for (int j = 0; j < i; ++j) {
        c[k] = h * kAE[i][j];
        X[k++] = A->FE[j];
        c[k] = h * kAI[i][j];
        X[k++] = A->FI[j];
      }
      TRY(sunbw::linear_combination(ctx, n, k, c, X, A->rhs, nullptr));
      // modified Newton from Z_{i-1}
      TRY(sunbw::bw_jacobian(A->prob, A->Z, A->M));
      TRY(sunbw::scale_add_identity(ctx, G, 3, -hg, A->M));
      TRY(sunbw::lu_factor(ctx, G, 3, A->M, A->piv, A->d_first));
      A->st.setups++;
      // a zero pivot on any rank recomputes the step on every rank
      TRY(sunbw::or_flags_over_ranks(ctx, A->d_first, nullptr));
      unsigned long long f = 0;
      if (cudaMemcpyAsync(&f, A->d_first, sizeof(f), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
          cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      if (f != ~0ull) { *nl_ok = 0; return 0; }
      bool conv = false;
      const double c3[3] = {1.0, hg, -1.0};
      for (int it = 0; it < A->opt.maxnl; ++it) {
        TRY(sunbw::bw_reaction(A->prob, A->Z, A->fI));
        const double* X3[3] = {A->rhs, A->fI, A->Z};
        TRY(sunbw::linear_combination(ctx, n, 3, c3, X3, A->r, nullptr));
        TRY(sunbw::lu_solve(ctx, G, 3, A->M, A->piv, A->r, A->delta));
        TRY(sunbw::linear_sum(ctx, n, 1.0, A->Z, 1.0, A->delta, A->Z, nullptr));
        A->st.newton_iters++;
        int e = 0;
        double nu = host_wrms(ctx, n, A->nglobal, A->delta, A->ewt, &e);
        if (e) return e;
        if (nu <= A->opt.tol_nl) { conv = true; break; }   // same global ν on every rank
      }
      if (!conv) { *nl_ok = 0; return 0; }
    }
    TRY(eval_rhs(A, A->Z, A->FE[i], A->FI[i]));
  }
  double c[9], ce[8];
  const double* X[9];
  const double* Xe[8];
  c[0] = 1.0;
  X[0] = A->y;
  for (int i = 0; i < 4; ++i) {
    c[1 + 2 * i] = h * kB[i];
    X[1 + 2 * i] = A->FE[i];
    c[2 + 2 * i] = h * kB[i];
    X[2 + 2 * i] = A->FI[i];
    const double be = h * (kB[i] - kD[i]);
    ce[2 * i] = be;
    Xe[2 * i] = A->FE[i];
    ce[2 * i + 1] = be;
    Xe[2 * i + 1] = A->FI[i];
  }
  TRY(sunbw::linear_combination(ctx, n, 9, c, X, A->ynew, nullptr));
  TRY(sunbw::linear_combination(ctx, n, 8, ce, Xe, A->err, nullptr));
  int e = 0;
  *dsm = host_wrms(ctx, n, A->nglobal, A->err, A->ewt, &e);
  return e;
}

// BW_ArkEvolve's loop with host decisions (composed path): *rc = 0, 1
// (max_steps) or 2 (step size underflow); < 0 on errors.
int evolve_host(Ark* A, double t_end, int* rc) {
  int attempts = 0;
  while (t_end - A->t > 1e-12 * std::fmax(1.0, std::fabs(t_end))) {
    if (attempts++ >= A->opt.max_steps) { *rc = 1; break; }
    // a step shortened to land on t_end does not shrink the next proposal
    // (DESIGN R26): the unclipped h is restored after it if larger
    const double h_unclipped = A->h;
    const bool clipped = A->t + A->h > t_end;
    if (clipped) A->h = t_end - A->t;
    if (A->h < 1e-14 * (1.0 + A->t)) { *rc = 2; break; }
    int nl_ok = 1;
    double dsm = 0.0;
    int e = attempt(A, &nl_ok, &dsm);
    if (e < 0) return e;
    if (!nl_ok) {
      A->st.rejected_nl++;
      A->h *= 0.25;
      continue;
    }
    double fac = dsm > 0.0 ? 0.9 * std::pow(dsm, -1.0 / 3.0) : 5.0;
    if (A->opt.fixed) { dsm = 0.0; fac = 1.0; }
    if (dsm <= 1.0) {
      std::swap(A->y, A->ynew);
      A->t += A->h;
      A->st.accepted++;
      A->h *= std::fmin(5.0, std::fmax(0.2, fac));
      if (clipped) A->h = std::fmax(A->h, h_unclipped);
    } else {
      A->st.rejected_err++;
      A->h *= std::fmin(1.0, std::fmax(0.2, fac));
    }
  }
  return 0;
}

}  // namespace

extern "C" int BW_ArkCreate(void* prob, N_Vector y0, const BW_ArkOptions* opt, void** out) {
  if (!prob || !y0 || !opt || !out) return SUNBW_ERR_ARG;
  *out = nullptr;
  if (!(opt->h0 > 0) || opt->maxnl < 1 || opt->max_steps < 1 || (opt->fused != 0 && opt->fused != 1))
    return SUNBW_ERR_ARG;
  if (opt->fused && opt->maxnl > 4) return SUNBW_ERR_UNSUPPORTED;   // fused stages: maxnl <= 4
  SUNBW_Context ctx = y0->ctx;
  int64_t G = sunbw::bw_local_cells(prob);
  if (y0->local_len != 3 * G) return ctx_set_err(ctx, SUNBW_ERR_LENGTH);
  auto* A = new Ark();
  A->prob = prob;
  A->ctx = ctx;
  A->opt = *opt;
  A->G = G;
  A->n = 3 * G;
  A->nglobal = y0->global_len;
  A->h = opt->h0;
  const int64_t n = A->n > 0 ? A->n : 1;
  double** vecs[] = {&A->y, &A->Z, &A->rhs, &A->ewt, &A->tmp, &A->r, &A->delta, &A->fI, &A->ynew,
                     &A->err, &A->FE[0], &A->FE[1], &A->FE[2], &A->FE[3], &A->FI[0], &A->FI[1],
                     &A->FI[2], &A->FI[3]};
  bool ok = true;
  for (double** v : vecs) ok = ok && cudaMalloc(v, sizeof(double) * n) == cudaSuccess;
  ok = ok && cudaMalloc(&A->M, sizeof(double) * 9 * (G > 0 ? G : 1)) == cudaSuccess &&
       cudaMalloc(&A->piv, sizeof(int32_t) * (G > 0 ? G : 1)) == cudaSuccess &&
       cudaMalloc(&A->d_first, sizeof(unsigned long long)) == cudaSuccess;
  if (ok && opt->fused) ok = (A->fused = sunbw::ark_fused_create(ctx, prob, A->nglobal)) != nullptr;
  if (!ok ||
      cudaMemcpyAsync(A->y, y0->d, sizeof(double) * A->n, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    BW_ArkDestroy(A);
    return ctx_set_err(ctx, SUNBW_ERR_MEM);
  }
  *out = A;
  return 0;
}

extern "C" int BW_ArkEvolve(void* ark, double t_end, N_Vector y_out, BW_ArkStats* stats) {
  auto* A = (Ark*)ark;
  if (!A) return SUNBW_ERR_ARG;
  SUNBW_Context ctx = A->ctx;
  if (y_out && (y_out->ctx != ctx || y_out->local_len != A->n)) return ctx_set_err(ctx, SUNBW_ERR_LENGTH);
  int rc = 0;
  const int e = A->fused ? sunbw::ark_fused_evolve(A->fused, &A->y, &A->ynew, &A->t, &A->h, t_end, A->opt,
                                                   &A->st, &rc)   // the same loop, decided on the device (R33)
                         : evolve_host(A, t_end, &rc);
  if (e < 0) return e;
  if (y_out &&
      cudaMemcpyAsync(y_out->d, A->y, sizeof(double) * A->n, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  A->st.t = A->t;
  A->st.h_last = A->h;
  if (stats) *stats = A->st;
  return rc;
}

extern "C" int BW_ArkDestroy(void* ark) {
  auto* A = (Ark*)ark;
  if (!A) return SUNBW_ERR_ARG;
  cudaStreamSynchronize(A->ctx->stream);
  double* bufs[] = {A->y, A->Z, A->rhs, A->ewt, A->tmp, A->r, A->delta, A->fI, A->ynew, A->err,
                    A->FE[0], A->FE[1], A->FE[2], A->FE[3], A->FI[0], A->FI[1], A->FI[2], A->FI[3], A->M};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (A->piv) cudaFree(A->piv);
  if (A->d_first) cudaFree(A->d_first);
  sunbw::ark_fused_destroy(A->fused);
  delete A;
  return 0;
}
