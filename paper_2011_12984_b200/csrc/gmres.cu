// gmres.cu — SPGMR: right-preconditioned GMRES on the block-diagonal
// operator, the Krylov solver of the paper's "global" Newton configuration
// (§5 lists GMRES among the matrix-free solvers that run on the GPU
// vectors; §7: "the native SUNDIALS Newton SUNNonlinear and GMRES
// SUNLinearSolver with the problem-specific block linear solver method
// previously described serving as a preconditioner").
//
// Algorithm (textbook right-preconditioned GMRES): x0 = 0, β = ‖b‖₂,
// V₀ = b/β; step j: z = P⁻¹V_j (batched block LU), w = A z (block SpMV,
// P:313), h = w·[V₀..V_j] (ONE fused N_VDotProdMulti reduction), w ← w −
// Σ h_i V_i (ONE N_VLinearCombination), h_{j+1} = ‖w‖₂, V_{j+1} = w/h_{j+1},
// Givens rotations on the host; stop at |g_{j+1}| ≤ tol·β.  Then
// x = P⁻¹ Σ y_i V_i.  Classical Gram–Schmidt is what lets the fused
// multi-vector kernels carry the orthogonalisation (one pass over the basis
// per step); each step has two global reductions (the dots and the norm),
// the per-iteration synchronisation the paper's global solver pays.

#include <cmath>
#include <cstring>
#include <vector>

#include "sunbw_internal.h"

namespace {

struct Spgmr : _SUNLinearSolver {
  int maxl = 0;
  bool prec = false;
  int64_t n = 0;
  double* V = nullptr;          // (maxl + 1) Krylov vectors, contiguous
  double* z = nullptr;
  double* w = nullptr;
  double* Plu = nullptr;        // LU factors of the preconditioner blocks
  int32_t* Ppiv = nullptr;
  unsigned long long* d_first = nullptr;
  int64_t last_iters = 0;
  double last_res = 0.0;
};

int norm2(SUNBW_Context ctx, int64_t n, int64_t nglob, const double* v, double* out) {
  int e = sunbw::reduce(ctx, sunbw::RK_DOT, sunbw::RF_NONE, n, nglob, v, v, nullptr, ctx->d_red,
                        ctx->h_slot_dev, true, nullptr);
  if (e) return e;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  *out = std::sqrt(((volatile double*)ctx->h_slot)[0]);
  return 0;
}

int apply_prec(Spgmr* S, const double* v, double* out) {
  if (S->prec) return sunbw::lu_solve(S->ctx, S->nblocks, S->m, S->Plu, S->Ppiv, v, out);
  if (cudaMemcpyAsync(out, v, sizeof(double) * S->n, cudaMemcpyDeviceToDevice, S->ctx->stream) !=
      cudaSuccess)
    return ctx_set_err(S->ctx, SUNBW_ERR_CUDA);
  return 0;
}

}  // namespace

namespace sunbw {

SUNLinearSolver spgmr_create(SUNBW_Context ctx, int64_t G, int m, int maxl, bool block_prec) {
  if (!ctx || G < 0 || m < 1 || m > 8 || maxl < 1 || maxl > 60) return nullptr;
  auto* S = new Spgmr();
  S->type = 1;
  S->ctx = ctx;
  S->nblocks = G;
  S->m = m;
  S->maxl = maxl;
  S->prec = block_prec;
  S->n = G * m;
  const int64_t n = S->n > 0 ? S->n : 1;
  bool ok = cudaMalloc(&S->V, sizeof(double) * n * (maxl + 1)) == cudaSuccess &&
            cudaMalloc(&S->z, sizeof(double) * n) == cudaSuccess &&
            cudaMalloc(&S->w, sizeof(double) * n) == cudaSuccess &&
            cudaMalloc(&S->d_first, sizeof(unsigned long long)) == cudaSuccess;
  if (ok && block_prec)
    ok = cudaMalloc(&S->Plu, sizeof(double) * (G > 0 ? G : 1) * m * m) == cudaSuccess &&
         cudaMalloc(&S->Ppiv, sizeof(int32_t) * (G > 0 ? G : 1)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    spgmr_free(S);
    ctx_set_err(ctx, SUNBW_ERR_MEM);
    return nullptr;
  }
  return S;
}

// preconditioner setup from raw block values: copy + batched LU (the
// operator itself stays intact for the matrix-vector products)
// d_first_accum: accumulate the first singular block there (the driver's
// per-Advance flag) instead of resetting the solver's own flag
int spgmr_setup_raw(SUNLinearSolver S0, const double* A, unsigned long long* d_first_accum) {
  auto* S = (Spgmr*)S0;
  if (!S->prec) return 0;
  SUNBW_Context ctx = S->ctx;
  if (cudaMemcpyAsync(S->Plu, A, sizeof(double) * S->nblocks * S->m * S->m, cudaMemcpyDeviceToDevice,
                      ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (d_first_accum) return lu_factor_noreset(ctx, S->nblocks, S->m, S->Plu, S->Ppiv, d_first_accum);
  return lu_factor(ctx, S->nblocks, S->m, S->Plu, S->Ppiv, S->d_first);
}

int spgmr_setup(SUNLinearSolver S0, SUNMatrix A) {
  auto* S = (Spgmr*)S0;
  if (!S || !A) return SUNBW_ERR_ARG;
  if (A->ctx != S->ctx) return ctx_set_err(S->ctx, SUNBW_ERR_CONTEXT);
  if (A->nblocks != S->nblocks || A->m != S->m) return ctx_set_err(S->ctx, SUNBW_ERR_LENGTH);
  int e = spgmr_setup_raw(S, A->d, nullptr);
  if (e) return e;
  if (!S->prec) return 0;
  unsigned long long f = 0;
  if (cudaMemcpyAsync(&f, S->d_first, sizeof(f), cudaMemcpyDeviceToHost, S->ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(S->ctx->stream) != cudaSuccess)
    return ctx_set_err(S->ctx, SUNBW_ERR_CUDA);
  S->last_flag = f == ~0ull ? 0 : (int64_t)f;
  return S->last_flag ? SUNBW_RECOV_SINGULAR : 0;
}

int spgmr_solve_raw(SUNLinearSolver S0, const double* A, double* x, const double* b, double tol) {
  auto* S = (Spgmr*)S0;
  SUNBW_Context ctx = S->ctx;
  const int64_t n = S->n;
  const int64_t nglob = n;                  // global length only enters the norms via Σ
  const int maxl = S->maxl;
  auto Vj = [&](int j) { return S->V + (int64_t)j * n; };
  std::vector<double> H((maxl + 1) * maxl, 0.0), g(maxl + 1, 0.0), cs(maxl), sn(maxl);
  double beta = 0.0;
  int e = norm2(ctx, n, nglob, b, &beta);
  if (e) return e;
  if (beta == 0.0) {
    S->last_iters = 0;
    S->last_res = 0.0;
    if (n > 0 && cudaMemsetAsync(x, 0, sizeof(double) * n, ctx->stream) != cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    return 0;
  }
  if ((e = scale(ctx, n, 1.0 / beta, b, Vj(0), nullptr))) return e;
  g[0] = beta;
  int steps = 0;
  std::vector<const double*> X(maxl + 2);
  std::vector<double> c(maxl + 2);
  for (int j = 0; j < maxl; ++j) {
    if ((e = apply_prec(S, Vj(j), S->z))) return e;
    if ((e = block_matvec(ctx, S->nblocks, S->m, A, S->z, S->w))) return e;
    // h_ij = w · V_i, i <= j: one fused multi-dot (global)
    for (int i = 0; i <= j; ++i) X[i] = Vj(i);
    if ((e = dot_multi(ctx, n, j + 1, S->w, X.data(), ctx->d_red, ctx->h_slot_dev, true, nullptr)))
      return e;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    for (int i = 0; i <= j; ++i) H[i * maxl + j] = ((volatile double*)ctx->h_slot)[i];
    // w = w - Σ h_ij V_i: one fused linear combination (in place, w = X[0])
    X[0] = S->w;
    c[0] = 1.0;
    for (int i = 0; i <= j; ++i) { X[i + 1] = Vj(i); c[i + 1] = -H[i * maxl + j]; }
    if ((e = linear_combination(ctx, n, j + 2, c.data(), X.data(), S->w, nullptr))) return e;
    double hn = 0.0;
    if ((e = norm2(ctx, n, nglob, S->w, &hn))) return e;
    H[(j + 1) * maxl + j] = hn;
    if (hn != 0.0 && (e = scale(ctx, n, 1.0 / hn, S->w, Vj(j + 1), nullptr))) return e;
    for (int i = 0; i < j; ++i) {            // previous rotations on column j
      double a = H[i * maxl + j], cc = H[(i + 1) * maxl + j];
      H[i * maxl + j] = cs[i] * a + sn[i] * cc;
      H[(i + 1) * maxl + j] = -sn[i] * a + cs[i] * cc;
    }
    double a = H[j * maxl + j], cc = H[(j + 1) * maxl + j];
    double r = std::hypot(a, cc);
    cs[j] = a / r;
    sn[j] = cc / r;
    H[j * maxl + j] = r;
    H[(j + 1) * maxl + j] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    steps = j + 1;
    if (std::fabs(g[j + 1]) <= tol * beta || hn == 0.0) break;
  }
  std::vector<double> y(steps);
  for (int i = steps - 1; i >= 0; --i) {
    double s = g[i];
    for (int k = i + 1; k < steps; ++k) s -= H[i * maxl + k] * y[k];
    y[i] = s / H[i * maxl + i];
  }
  for (int i = 0; i < steps; ++i) X[i] = Vj(i);
  if ((e = linear_combination(ctx, n, steps, y.data(), X.data(), S->w, nullptr))) return e;
  if ((e = apply_prec(S, S->w, x))) return e;
  S->last_iters = steps;
  S->last_res = std::fabs(g[steps]);
  return steps;
}

int spgmr_solve(SUNLinearSolver S0, SUNMatrix A, N_Vector x, N_Vector b, double tol) {
  auto* S = (Spgmr*)S0;
  if (!S || !A || !x || !b) return SUNBW_ERR_ARG;
  if (A->ctx != S->ctx || x->ctx != S->ctx || b->ctx != S->ctx) return ctx_set_err(S->ctx, SUNBW_ERR_CONTEXT);
  if (x->local_len != S->n || b->local_len != S->n || A->nblocks != S->nblocks || A->m != S->m)
    return ctx_set_err(S->ctx, SUNBW_ERR_LENGTH);
  if (x->d == b->d) return ctx_set_err(S->ctx, SUNBW_ERR_ARG);
  int r = spgmr_solve_raw(S, A->d, x->d, b->d, tol > 0 ? tol : 1e-10);
  return r < 0 ? r : 0;
}

int64_t spgmr_last_iters(SUNLinearSolver S) { return ((Spgmr*)S)->last_iters; }

void spgmr_free(SUNLinearSolver S0) {
  auto* S = (Spgmr*)S0;
  if (!S) return;
  double* bufs[] = {S->V, S->z, S->w, S->Plu};
  for (double* p : bufs)
    if (p) cudaFree(p);
  if (S->Ppiv) cudaFree(S->Ppiv);
  if (S->d_first) cudaFree(S->d_first);
  delete S;
}

}  // namespace sunbw

extern "C" SUNLinearSolver SUNLinSol_B200SPGMR(N_Vector y, SUNMatrix A, int maxl, int block_prec) {
  if (!y || !A || y->ctx != A->ctx || y->local_len != A->nblocks * A->m) return nullptr;
  return sunbw::spgmr_create(A->ctx, A->nblocks, A->m, maxl, block_prec != 0);
}

extern "C" int64_t SUNLinSolNumIters(SUNLinearSolver S) {
  if (!S) return SUNBW_ERR_ARG;
  return S->type == 1 ? sunbw::spgmr_last_iters(S) : 0;
}

extern "C" double SUNLinSolResNorm(SUNLinearSolver S) {
  if (!S || S->type != 1) return 0.0;
  return ((Spgmr*)S)->last_res;
}
