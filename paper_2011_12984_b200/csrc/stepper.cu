// stepper.cu — fixed-step IMEX-BDF Newton driver (the integrator + task-local
// nonlinear solver of the paper's demonstration, §7).
//
// IMEX split: advection f_E explicit, stiff reaction f_I
// implicit.  Integrator (DESIGN R14): SBDF1 on the first step, SBDF2 after:
//   n = 0:  z - h f_I(z) = y_0 + h f_E(y_0)                       (γ = h)
//   n ≥ 1:  z - (2h/3) f_I(z) = 4/3 y_n - 1/3 y_{n-1}
//                               + 4h/3 f_E(y_n) - 2h/3 f_E(y_{n-1})  (γ = 2h/3)
// Nonlinear solver (DESIGN R15): modified Newton per cell,
// matrix M = I - γ J(z⁰) built and LU-factored once per step at the
// predictor z⁰ = y_n; each iteration r = d + γ f_I(z) - z, δ = M⁻¹ r,
// z += δ, ν = WRMS(δ, ewt), ewt = 1/(rtol |y_n| + atol).
//
// Composed mode: every stage is one of the library's N_Vector / matrix /
// solver kernels, enqueued on the context stream (the structure of
// fig:advrecatorg).  Fixed-K mode never synchronises inside a
// step; the step is captured once per buffer-rotation state into a CUDA
// graph and replayed (launch-bound small problems).  Tolerance
// mode synchronises once per Newton iteration for the host decision
// (reductions return to the host).
//
// Fused mode (the task-local solver as ONE kernel per step):
// after the halo + advection kernels, each thread owns one cell and runs the
// whole step — d, ewt, Jacobian, M, LU, K Newton iterations — in registers,
// with the same operation order as the composed path (bit-identical state);
// per-iteration WRMS and the ewt minimum leave as per-CTA partials folded by
// one small kernel.

#include <cmath>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "sunbw_internal.h"

namespace sunbw {
int bw_reaction(void* prob, const double* y, double* f);
int bw_jacobian(void* prob, const double* y, double* J);
int bw_halo(void* prob, const double* y);
int bw_halo_stream(void* prob, const double* y, cudaStream_t stream);
int bw_advection_stencil(void* prob, const double* y, double* f);
int64_t bw_local_cells(void* prob);
BW_BrussParams bw_params(void* prob);
int fused_newton(SUNBW_Context ctx, void* prob, int64_t G, bool first, int K, double h,
                 double rtol, double atol, const double* y, const double* fE, const double* hin,
                 double* hout, double* z, double* partials, unsigned long long* d_first,
                 int* nblocks_out, const FusedAdvection* adv, int64_t tile_begin, int64_t tile_end,
                 const FusedFold* fold, int solver, bool tol, TolDev* tdev = nullptr);
int fused_fold(SUNBW_Context ctx, const double* partials, int nblocks, int K, int64_t nglobal,
               double* d_min, double* d_nu, int* d_err);
int fused_finalize_pending(SUNBW_Context ctx, double* pending, int K, int64_t nglobal, double* d_min,
                           double* d_nu, int* d_err);
}  // namespace sunbw

namespace {

// local (singular, bad-ewt) flags as doubles, and back after the allreduce
__global__ void k_flags(const unsigned long long* first, const int* err, double* flags) {
  flags[0] = *first != ~0ull ? 1.0 : 0.0;
  flags[1] = (err && *err) ? 1.0 : 0.0;
}
__global__ void k_flags_back(const double* flags, unsigned long long* first, int* err) {
  if (flags[0] != 0.0 && *first == ~0ull) *first = 0;   // singular elsewhere: report block 0
  if (err && flags[1] != 0.0) *err = 1;
}

}  // namespace

int sunbw::or_flags_over_ranks(SUNBW_Context ctx, unsigned long long* d_first, int* d_err) {
  if (ctx_nranks(ctx) <= 1) return 0;
  double* flags = ctx->d_red + 96;
  k_flags<<<1, 1, 0, ctx->stream>>>(d_first, d_err, flags);
  ctx->launches++;
  int e = ctx->comm->allreduce(flags, 2, RED_MAX, ctx->stream);
  if (e) return ctx_set_err(ctx, e);
  k_flags_back<<<1, 1, 0, ctx->stream>>>(flags, d_first, d_err);
  ctx->launches++;
  return ctx_check_launch(ctx);
}

namespace {

constexpr int kMaxK = 32;
constexpr int kMaxKF = 8;      // fused mode: K <= 8

struct Stepper {
  void* prob;
  SUNBW_Context ctx;
  BW_StepperOptions opt;
  int64_t G, n, nglobal;
  double* y[3];
  double* fE[2];
  int iy = 0, iyp = 1, iz = 2, ife = 0, ifep = 1;
  double *d, *ewt, *tmp, *fI, *r, *delta, *M;
  int32_t* piv;
  unsigned long long* d_first;
  double* d_scal;        // [0] ewt min, [1..K] nu per iteration
  int* d_err;            // 1: non-positive ewt denominator seen
  double* d_partials;    // fused mode per-CTA partials
  double* h_tol = nullptr;   // fused tolerance mode: pinned [min, nu_1..nu_8 | first | err]
  unsigned long long* h_end = nullptr;   // pinned: end-of-Advance [first, err, nu]
  int k_pred = 0;            // fused tolerance mode: the last step's iteration count
  sunbw::TolDev* d_tdev = nullptr;   // fused tolerance mode driven from the device (R35)
  sunbw::TolDev* h_tdev = nullptr;   // pinned staging
  int* h_tdone = nullptr;            // mapped pinned: TolDev::done after the latest launch
  int* d_tdone = nullptr;
  cudaEvent_t tev[2] = {};
  int64_t tol_launches = 0;  // fused tolerance mode: step launches (recomputations included)
  unsigned* d_counter = nullptr;   // fused mode: arrival counter of the in-kernel fold
  SUNLinearSolver gm = nullptr;   // linsol 1: SPGMR, block-LU preconditioner
  // fused mode on P > 1 ranks: halo on a side stream overlapping the
  // interior tiles; reductions deferred to the end of Advance (fixed K)
  cudaStream_t side = nullptr;
  cudaEvent_t evA = nullptr, evB = nullptr;
  double* d_pending = nullptr;   // K + 2: local [min, sums], flag
  bool deferred = false;
  // fused fixed-K step of a one-CTA problem: many steps per launch
  bool small = false;
  sunbw::SmallGeom sg{};
  int64_t step = 0;
  double t = 0.0;
  BW_StepperStats st{};
  // graphs, keyed by rotation state (iy, ife): 3 × 2
  cudaStream_t cap_stream = nullptr;
  // keys 0..5: one step; 6..11: a chain of kChain steps starting at that
  // rotation state (the rotation's period), replayed while >= kChain remain
  cudaGraphExec_t gexec[12] = {};
  int64_t graph_launches[12] = {};
  // timing mode with graphs: the captured graph's event-record nodes (in
  // capture order, start/end pairs) get fresh pool events before each replay
  cudaGraph_t graph[12] = {};
  std::vector<cudaGraphNode_t> ev_nodes[12];
  std::vector<int> ev_node_kind[12];
  bool capturing = false;
  // timing
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_kind;          // per event pair: kind + kKindMod * (launches - 1)
  // fused single-kernel steps captured as a chain: one event pair around the
  // whole chain instead of one per kernel (an event-record node between two
  // step kernels costs ~7 us of idle GPU, tools/step_gaps_cupti.py)
  bool chain_timed = false;
  double k_ms[BW_K_COUNT_] = {};
  int64_t k_count[BW_K_COUNT_] = {};
};

int alloc(Stepper* S, double** p, int64_t count) {
  if (cudaMalloc(p, sizeof(double) * (count > 0 ? count : 1)) != cudaSuccess) {
    cudaGetLastError();
    return SUNBW_ERR_MEM;
  }
  return 0;
}

// ------------------------------------------------------------ timing hooks
// NVTX range per stage, named by the paper's four timing categories
// (advection incl. its communication, reaction, linear solve incl.
// the Jacobian and matrix setup, and "other" = integrator + nonlinear solver
// vector work); the fused kernel is all four in one launch.
const char* nvtx_category(int kind) {
  switch (kind) {
    case BW_K_HALO: case BW_K_ADVECTION: return "advection (incl. halo)";
    case BW_K_REACTION: return "reaction";
    case BW_K_JACOBIAN: case BW_K_SCALEADDI: case BW_K_LU_SETUP: case BW_K_LU_SOLVE: return "linear solve";
    case BW_K_FUSED_NEWTON: case BW_K_FUSED_PLANE0: return "fused step (all categories)";
    default: return "other";
  }
}

constexpr int kKindMod = 64;              // > BW_K_COUNT_
static_assert(BW_K_COUNT_ < kKindMod, "event kind encoding");

struct Timed {
  Stepper* S;
  int kind;
  bool on;
  cudaStream_t st;
  Timed(Stepper* s, int k, cudaStream_t stream = nullptr)
      : S(s), kind(k),
        on(s->opt.timing != 0 && !(s->chain_timed && k == BW_K_FUSED_NEWTON) &&
           (s->opt.timing <= 1 || s->capturing || s->step % s->opt.timing == 0)),
        st(stream ? stream : s->ctx->stream) {
    nvtxRangePushA(nvtx_category(k));
    if (!on) return;
    if (S->ev_used + 2 > S->ev_pool.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        S->ev_pool.push_back(e);
      }
    }
    cudaEventRecordWithFlags(S->ev_pool[S->ev_used], st,
                             S->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
  ~Timed() {
    nvtxRangePop();
    if (!on) return;
    cudaEventRecordWithFlags(S->ev_pool[S->ev_used + 1], st,
                             S->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    S->ev_kind.push_back(kind);
    S->ev_used += 2;
  }
};

void harvest_timing(Stepper* S) {
  for (size_t i = 0; i < S->ev_kind.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, S->ev_pool[2 * i], S->ev_pool[2 * i + 1]);
    const int kind = S->ev_kind[i] % kKindMod, launches = S->ev_kind[i] / kKindMod + 1;
    S->k_ms[kind] += ms;
    S->k_count[kind] += launches;
  }
  S->ev_kind.clear();
  S->ev_used = 0;
}

#define TRY(x)              \
  do {                      \
    int e_ = (x);           \
    if (e_ < 0) return e_;  \
  } while (0)

// ------------------------------------------------------------- one step
// Enqueues the whole step on ctx->stream.  Tolerance mode: returns > 0 on a
// recoverable failure (needs the host decision, so it synchronises).
int enqueue_step(Stepper* S, bool first) {
  SUNBW_Context ctx = S->ctx;
  const BW_StepperOptions& o = S->opt;
  const int64_t n = S->n, G = S->G;
  double* y = S->y[S->iy];
  double* yp = S->y[S->iyp];
  double* z = S->y[S->iz];
  double* fE = S->fE[S->ife];
  double* fEp = S->fE[S->ifep];
  const double h = o.h;
  const double gamma = first ? h : (2.0 * h) / 3.0;

  sunbw::FusedAdvection fa;
  const bool adv_in_kernel = o.fused && o.fused_advection && sunbw::bw_fused_advection(S->prob, y, &fa) &&
                             G % 128 == 0 && G <= INT32_MAX;
  // P > 1 with the single-kernel step: the halo plane travels on a side
  // stream while the interior tiles (local planes k >= 1) are computed; the
  // plane-0 tiles, which read it, run after the join (SURVEY §8(e) overlap)
  const bool split = adv_in_kernel && ctx_nranks(ctx) > 1 && S->side;
  // fused mode: fE[ife] / fE[ifep] hold the SBDF2 history H_{n+1} / H_n
  // (R28) and y[iyp] (y_{n-1}, unused) takes f_E,n when it is computed by
  // the separate stencil kernel
  double* fE_n = o.fused ? yp : fE;
  // fused step of a reaction-only problem: f_E ≡ 0 is not materialised
  const bool fzero = o.fused && !adv_in_kernel && sunbw::bw_params(S->prob).reaction_only;
  if (fzero) fE_n = nullptr;
  if (!split) {
    if (ctx_nranks(ctx) > 1) {   // one rank: periodic wrap in place, nothing to time
      Timed t(S, BW_K_HALO);
      TRY(sunbw::bw_halo(S->prob, y));
    }
    if (!adv_in_kernel && !fzero) {
      Timed t(S, BW_K_ADVECTION);
      TRY(sunbw::bw_advection_stencil(S->prob, y, fE_n));
    }
  }

  if (o.fused) {
    const int solver = o.numerics == 1 ? 2 : (o.linsol == 2 ? 1 : 0);
    // partials are folded by the step's last CTA unless a blocking
    // allreduce must sit between fold and finalisation (P > 1, not deferred)
    const bool fold_in_kernel = S->deferred || ctx_nranks(ctx) <= 1;
    // one launch sequence of the step with Kr Newton iterations (tolk: the
    // tolerance-mode kernel, every iteration's nu); with_halo: the P > 1
    // split around the side-stream halo
    auto run = [&](int Kr, bool tolk, bool with_halo) -> int {
      int nb = 0, nb2 = 0;
      sunbw::FusedFold fold{0, S->d_counter, S->deferred ? S->d_pending : nullptr, S->d_scal, S->d_scal + 1,
                            S->d_err, S->nglobal};
      const sunbw::FusedFold* fk = fold_in_kernel ? &fold : nullptr;
      if (split && with_halo && ctx->comm->peer) {
        // copy-engine halo (peer_halo.cu): no SM is needed for the transfer,
        // so it proceeds while the interior launch fills the GPU
        const int64_t tpp = fa.nx * fa.ny / 128;          // tiles per z-plane
        const size_t hl = (size_t)(3 * fa.nx * fa.ny);
        if (cudaEventRecord(S->evA, ctx->stream) != cudaSuccess ||
            cudaStreamWaitEvent(S->side, S->evA, 0) != cudaSuccess)
          return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        {
          Timed t(S, BW_K_HALO, S->side);
          TRY(sunbw::peer_halo_send(ctx->comm->peer, y + 3 * G - hl, hl, S->side) ? ctx_set_err(ctx, SUNBW_ERR_CUDA)
                                                                                   : 0);
        }
        if (cudaEventRecord(S->evB, S->side) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        {
          Timed t(S, BW_K_FUSED_NEWTON);
          TRY(sunbw::fused_newton(ctx, S->prob, G, first, Kr, h, o.rtol, o.atol, y, nullptr, fEp, fE, z,
                                  S->d_partials, S->d_first, &nb, &fa, tpp, -1, nullptr, solver, tolk));
        }
        sunbw::FusedAdvection fa0 = fa;
        if (sunbw::peer_halo_wait(ctx->comm->peer, ctx->stream, &fa0.below)) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        fold.prev_parts = nb;
        {
          Timed t(S, BW_K_FUSED_PLANE0);
          TRY(sunbw::fused_newton(ctx, S->prob, G, first, Kr, h, o.rtol, o.atol, y, nullptr, fEp, fE, z,
                                  S->d_partials + (int64_t)nb * (Kr + 1), S->d_first, &nb2, &fa0, 0, tpp,
                                  fk, solver, tolk));
        }
        if (sunbw::peer_halo_release(ctx->comm->peer, ctx->stream) ||
            cudaStreamWaitEvent(ctx->stream, S->evB, 0) != cudaSuccess)   // own send done before y is reused
          return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      } else if (split && with_halo) {
        const int64_t tpp = fa.nx * fa.ny / 128;          // tiles per z-plane
        if (cudaEventRecord(S->evA, ctx->stream) != cudaSuccess ||
            cudaStreamWaitEvent(S->side, S->evA, 0) != cudaSuccess)
          return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        {
          Timed t(S, BW_K_HALO, S->side);
          TRY(sunbw::bw_halo_stream(S->prob, y, S->side));
        }
        if (cudaEventRecord(S->evB, S->side) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        {
          Timed t(S, BW_K_FUSED_NEWTON);
          TRY(sunbw::fused_newton(ctx, S->prob, G, first, Kr, h, o.rtol, o.atol, y, nullptr, fEp, fE, z,
                                  S->d_partials, S->d_first, &nb, &fa, tpp, -1, nullptr, solver, tolk));
        }
        if (cudaStreamWaitEvent(ctx->stream, S->evB, 0) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        fold.prev_parts = nb;
        {
          Timed t(S, BW_K_FUSED_PLANE0);
          TRY(sunbw::fused_newton(ctx, S->prob, G, first, Kr, h, o.rtol, o.atol, y, nullptr, fEp, fE, z,
                                  S->d_partials + (int64_t)nb * (Kr + 1), S->d_first, &nb2, &fa, 0, tpp,
                                  fk, solver, tolk));
        }
      } else {
        Timed t(S, BW_K_FUSED_NEWTON);
        TRY(sunbw::fused_newton(ctx, S->prob, G, first, Kr, h, o.rtol, o.atol, y,
                                adv_in_kernel ? nullptr : fE_n, fEp, fE, z, S->d_partials, S->d_first, &nb,
                                adv_in_kernel ? &fa : nullptr, 0, -1, fk, solver, tolk));
      }
      if (!fold_in_kernel) {
        Timed t(S, BW_K_WRMS);
        TRY(sunbw::fused_fold(ctx, S->d_partials, nb + nb2, Kr, S->nglobal, S->d_scal, S->d_scal + 1,
                              S->d_err));
      }
      return 0;
    };
    if (o.newton_mode != 1) return run(o.K, false, true);

    // Tolerance mode, fused (DESIGN R31): the step kernel runs a
    // predicted number of iterations Kr (the last step's count) and reports
    // every iteration's global nu; the host takes the oracle's decision --
    // the first k with nu_k <= tol_nl -- and recomputes the step (its inputs
    // are untouched) when that k differs from Kr: with k if k < Kr, with the
    // maximum K if none of the Kr converged.  No convergence within K:
    // recoverable failure, as on the composed path.
    int Kr = S->k_pred > 0 && S->k_pred <= o.K ? S->k_pred : o.K;
    for (int attempt = 0; attempt < 3; ++attempt) {
      // every attempt repeats the halo exchange: the copy-engine halo's slot
      // is released to the sender after each plane-0 launch
      TRY(run(Kr, true, true));
      TRY(sunbw::or_flags_over_ranks(ctx, S->d_first, S->d_err));
      if (cudaMemcpyAsync(S->h_tol, S->d_scal, sizeof(double) * (Kr + 1), cudaMemcpyDeviceToHost,
                          ctx->stream) != cudaSuccess ||
          cudaMemcpyAsync(S->h_tol + kMaxKF + 1, S->d_first, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream) != cudaSuccess ||
          cudaMemcpyAsync(S->h_tol + kMaxKF + 2, S->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) !=
              cudaSuccess ||
          cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      S->tol_launches++;
      if (attempt > 0) S->st.setups++;   // a recomputation repeats the Setup (stats: setups per launch)
      const unsigned long long f = *(const unsigned long long*)(S->h_tol + kMaxKF + 1);
      if (*(const int*)(S->h_tol + kMaxKF + 2)) return SUNBW_RECOV_BAD_EWT;
      if (f != ~0ull) { S->st.singular = (int64_t)f; return SUNBW_RECOV_SINGULAR; }
      int kstar = 0;
      for (int k = 1; k <= Kr && !kstar; ++k)
        if (S->h_tol[k] <= o.tol_nl) kstar = k;            // same global nu on every rank (R17)
      if (kstar == Kr) {
        S->st.newton_iters += Kr;
        S->st.last_nu = S->h_tol[Kr];
        S->k_pred = Kr;
        return 0;
      }
      if (kstar > 0) {
        Kr = kstar;                  // converged earlier than predicted: redo with exactly kstar
      } else if (Kr == o.K) {
        S->st.newton_iters += o.K;
        S->st.last_nu = S->h_tol[o.K];
        return SUNBW_RECOV_NONCONV;
      } else {
        Kr = o.K;                    // not converged within Kr: redo with the maximum
      }
    }
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);   // unreachable: at most Kr -> K -> kstar
  }

  {
    Timed t(S, BW_K_RHS_COMBINE);
    if (first) {
      TRY(sunbw::linear_sum(ctx, n, 1.0, y, h, fE, S->d, nullptr));
    } else {
      // history terms first (R28): the fused kernel carries their sum
      const double c[4] = {-1.0 / 3.0, -((2.0 * h) / 3.0), 4.0 / 3.0, (4.0 * h) / 3.0};
      const double* X[4] = {yp, fEp, y, fE};
      TRY(sunbw::linear_combination(ctx, n, 4, c, X, S->d, nullptr));
    }
  }
  {
    Timed t(S, BW_K_EWT);
    TRY(sunbw::abs_(ctx, n, y, S->tmp, nullptr));
    TRY(sunbw::scale(ctx, n, o.rtol, S->tmp, S->tmp, nullptr));
    TRY(sunbw::add_const(ctx, n, S->tmp, o.atol, S->tmp, nullptr));
    TRY(sunbw::reduce(ctx, sunbw::RK_MIN, sunbw::RF_NONE, n, S->nglobal, S->tmp, nullptr, nullptr,
                      S->d_scal, nullptr, true, nullptr));
    TRY(sunbw::flag_nonpositive(ctx, S->d_scal, S->d_err));
    TRY(sunbw::inv(ctx, n, S->tmp, S->ewt, nullptr));
  }
  { Timed t(S, BW_K_PREDICT); TRY(sunbw::scale(ctx, n, 1.0, y, z, nullptr)); }
  { Timed t(S, BW_K_JACOBIAN); TRY(sunbw::bw_jacobian(S->prob, z, S->M)); }
  { Timed t(S, BW_K_SCALEADDI); TRY(sunbw::scale_add_identity(ctx, G, 3, -gamma, S->M)); }
  {
    Timed t(S, BW_K_LU_SETUP);
    if (S->gm)   // global Newton: M stays the GMRES operator, its LU preconditions
      TRY(sunbw::spgmr_setup_raw(S->gm, S->M, S->d_first));
    else if (o.linsol == 2)   // the paper's block inverse (R29)
      TRY(sunbw::gj_inverse(ctx, G, 3, S->M, S->d_first, false));
    else
      TRY(sunbw::lu_factor_noreset(ctx, G, 3, S->M, S->piv, S->d_first));
  }

  const bool tol = o.newton_mode == 1;
  if (tol) {
    // the host needs the singular flag and the ewt check before iterating;
    // every rank must take the same branch (the collectives below pair up)
    TRY(sunbw::or_flags_over_ranks(ctx, S->d_first, S->d_err));
    unsigned long long f = 0;
    int err = 0;
    if (cudaMemcpyAsync(S->h_end, S->d_first, sizeof(f), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(S->h_end + 1, S->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    std::memcpy(&f, S->h_end, sizeof(f));
    std::memcpy(&err, S->h_end + 1, sizeof(int));
    if (err) return SUNBW_RECOV_BAD_EWT;
    if (f != ~0ull) { S->st.singular = (int64_t)f; return SUNBW_RECOV_SINGULAR; }
  }
  const double c3[3] = {1.0, gamma, -1.0};
  for (int it = 0; it < o.K; ++it) {
    { Timed t(S, BW_K_REACTION); TRY(sunbw::bw_reaction(S->prob, z, S->fI)); }
    {
      Timed t(S, BW_K_RESIDUAL);
      const double* X3[3] = {S->d, S->fI, z};
      TRY(sunbw::linear_combination(ctx, n, 3, c3, X3, S->r, nullptr));
    }
    {
      Timed t(S, BW_K_LU_SOLVE);
      if (S->gm) {
        int steps = sunbw::spgmr_solve_raw(S->gm, S->M, S->delta, S->r, o.lin_tol);
        TRY(steps);
        S->st.lin_iters += steps;
      } else if (o.linsol == 2) {
        TRY(sunbw::gj_apply(ctx, G, 3, S->M, S->r, S->delta));
      } else {
        TRY(sunbw::lu_solve(ctx, G, 3, S->M, S->piv, S->r, S->delta));
      }
    }
    { Timed t(S, BW_K_UPDATE); TRY(sunbw::linear_sum(ctx, n, 1.0, z, 1.0, S->delta, z, nullptr)); }
    {
      Timed t(S, BW_K_WRMS);
      TRY(sunbw::reduce(ctx, sunbw::RK_WSQR, sunbw::RF_WRMS, n, S->nglobal, S->delta, S->ewt, nullptr,
                        S->d_scal + 1 + it, tol ? ctx->h_slot_dev : nullptr, true, nullptr));
    }
    S->st.newton_iters++;
    S->st.solves++;
    if (tol) {
      if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      double nu = ((volatile double*)ctx->h_slot)[0];
      S->st.last_nu = nu;
      if (nu <= o.tol_nl) return 0;        // all ranks see the same global ν (R17)
    }
  }
  return tol ? SUNBW_RECOV_NONCONV : 0;
}

void rotate(Stepper* S) {
  int oy = S->iy, oyp = S->iyp, oz = S->iz;
  S->iy = oz; S->iyp = oy; S->iz = oyp;
  std::swap(S->ife, S->ifep);
}

int graph_key(const Stepper* S) { return S->iy * 2 + S->ife; }

constexpr int kChain = 6;

// capture `nsteps` SBDF2 steps (fixed-K) from the current rotation state into
// graph `key` (the rotation state is restored afterwards)
int capture_step(Stepper* S, int key, int nsteps = 1) {
  SUNBW_Context ctx = S->ctx;
  if (!S->cap_stream &&
      cudaStreamCreateWithFlags(&S->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  cudaStream_t user = ctx->stream;
  ctx->stream = S->cap_stream;
  int64_t l0 = ctx->launches.load();
  int64_t it0 = S->st.newton_iters, so0 = S->st.solves;
  const size_t ev0 = S->ev_used, kind0 = S->ev_kind.size();
  cudaGraph_t g = nullptr;
  int rc = 0;
  if (cudaStreamBeginCapture(S->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    rc = SUNBW_ERR_CUDA;
  } else {
    S->capturing = true;
    const int iy = S->iy, iyp = S->iyp, iz = S->iz, ife = S->ife, ifep = S->ifep;
    // one kernel per step (fused with the in-kernel advection, one rank,
    // fixed K): time the chain as a whole; the kernels follow each other
    // with ~0.3 us gaps, so the pair's time / nsteps is the kernel's launch
    // duration to within that.  The pair is reserved (and its kind entered)
    // before the steps are enqueued, so it keeps its place in the pool.
    sunbw::FusedAdvection fa;
    bool chain = S->opt.timing && S->opt.fused && S->opt.newton_mode == 0 && S->opt.fused_advection &&
                 ctx_nranks(ctx) <= 1 && nsteps > 1 && S->G % 128 == 0 && S->G <= INT32_MAX &&
                 sunbw::bw_fused_advection(S->prob, S->y[S->iy], &fa);
    size_t slot = 0;
    if (chain) {
      while (S->ev_used + 2 > S->ev_pool.size() && chain) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { rc = SUNBW_ERR_CUDA; chain = false; break; }
        S->ev_pool.push_back(e);
      }
    }
    if (chain) {
      slot = S->ev_used;
      S->ev_used += 2;
      S->ev_kind.push_back(BW_K_FUSED_NEWTON + kKindMod * (nsteps - 1));
      cudaEventRecordWithFlags(S->ev_pool[slot], S->cap_stream, cudaEventRecordExternal);
      S->chain_timed = true;
    }
    for (int k = 0; k < nsteps && !rc; ++k) {
      rc = enqueue_step(S, false);
      rotate(S);
    }
    if (chain) {
      S->chain_timed = false;
      cudaEventRecordWithFlags(S->ev_pool[slot + 1], S->cap_stream, cudaEventRecordExternal);
    }
    S->iy = iy; S->iyp = iyp; S->iz = iz; S->ife = ife; S->ifep = ifep;
    S->capturing = false;
    if (cudaStreamEndCapture(S->cap_stream, &g) != cudaSuccess) rc = rc ? rc : SUNBW_ERR_CUDA;
  }
  ctx->stream = user;
  if (!rc && g && S->opt.timing) {
    // event-record nodes in capture order: match each node's event with the
    // pool entries the capture consumed
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    const size_t nev = S->ev_used - ev0;
    std::vector<cudaGraphNode_t> ordered(nev, nullptr);
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      cudaGraphNodeGetType(nd, &ty);
      if (ty != cudaGraphNodeTypeEventRecord) continue;
      cudaEvent_t ev;
      cudaGraphEventRecordNodeGetEvent(nd, &ev);
      for (size_t i = 0; i < nev; ++i)
        if (S->ev_pool[ev0 + i] == ev) ordered[i] = nd;
    }
    for (cudaGraphNode_t nd : ordered)
      if (!nd) rc = SUNBW_ERR_CUDA;
    S->ev_nodes[key] = ordered;
    S->ev_node_kind[key].assign(S->ev_kind.begin() + kind0, S->ev_kind.end());
    S->ev_used = ev0;                      // the capture's events measured nothing
    S->ev_kind.resize(kind0);
  }
  S->st.newton_iters = it0;
  S->st.solves = so0;
  S->graph_launches[key] = ctx->launches.load() - l0;
  ctx->launches -= S->graph_launches[key];
  if (rc) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return ctx_set_err(ctx, rc < 0 ? rc : SUNBW_ERR_CUDA);
  }
  if (cudaGraphInstantiate(&S->gexec[key], g, 0) != cudaSuccess) {
    cudaGraphDestroy(g);
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  }
  S->graph[key] = g;                       // kept: its event nodes are updated per replay
  return 0;
}

// Captures (and uploads) the step graph of every rotation state (3 state
// buffers x 2 history buffers = 6 keys, the rotation's period) at the first
// graph step, so that no capture or first-launch upload lands inside a later
// Advance call (a timed region).
int capture_all_keys(Stepper* S) {
  const int iy = S->iy, iyp = S->iyp, iz = S->iz, ife = S->ife, ifep = S->ifep;
  int rc = 0;
  for (int r = 0; r < 6 && !rc; ++r) {
    const int key = graph_key(S);
    for (int c = 0; c < 2 && !rc; ++c) {          // the single step, then the chain
      const int gk = key + 6 * c;
      if (S->gexec[gk]) continue;
      rc = capture_step(S, gk, c ? kChain : 1);
      if (!rc && cudaGraphUpload(S->gexec[gk], S->ctx->stream) != cudaSuccess)
        rc = ctx_set_err(S->ctx, SUNBW_ERR_CUDA);
    }
    rotate(S);
  }
  S->iy = iy; S->iyp = iyp; S->iz = iz; S->ife = ife; S->ifep = ifep;
  return rc;
}

}  // namespace

// ==================================================================== C ABI
extern "C" int BW_StepperCreate(void* prob, N_Vector y0, const BW_StepperOptions* opt, void** out) {
  if (!prob || !y0 || !opt || !out) return SUNBW_ERR_ARG;
  *out = nullptr;
  if (opt->K < 1 || opt->K > kMaxK || !(opt->h > 0) || (opt->newton_mode != 0 && opt->newton_mode != 1))
    return SUNBW_ERR_ARG;
  if (opt->linsol < 0 || opt->linsol > 2 || (opt->linsol == 1 && (opt->maxl < 1 || opt->maxl > 60)))
    return SUNBW_ERR_ARG;
  if (opt->numerics < 0 || opt->numerics > 1) return SUNBW_ERR_ARG;
  if (opt->fused && (opt->K > 8 || opt->linsol == 1)) return SUNBW_ERR_UNSUPPORTED;
  // fused tolerance mode: the contracted cell step (R30, R31)
  if (opt->fused && opt->newton_mode == 1 && opt->numerics != 1) return SUNBW_ERR_UNSUPPORTED;
  if (opt->fused && opt->numerics == 1 && opt->linsol != 0) return SUNBW_ERR_UNSUPPORTED;
  SUNBW_Context ctx = y0->ctx;
  int64_t G = sunbw::bw_local_cells(prob);
  if (y0->local_len != 3 * G) return ctx_set_err(ctx, SUNBW_ERR_LENGTH);
  auto* S = new Stepper();
  S->prob = prob;
  S->ctx = ctx;
  S->opt = *opt;
  if (ctx->comm && !ctx->comm->capturable()) S->opt.use_graph = 0;
  if (S->opt.newton_mode == 1 || S->opt.linsol == 1) S->opt.use_graph = 0;   // host decisions
  S->G = G;
  S->n = 3 * G;
  S->nglobal = y0->global_len;
  int64_t n = S->n;
  int e = 0;
  for (int i = 0; i < 3 && !e; ++i) e = alloc(S, &S->y[i], n);
  for (int i = 0; i < 2 && !e; ++i) e = alloc(S, &S->fE[i], n);
  if (!e && !opt->fused) {
    e = alloc(S, &S->d, n);
    if (!e) e = alloc(S, &S->ewt, n);
    if (!e) e = alloc(S, &S->tmp, n);
    if (!e) e = alloc(S, &S->fI, n);
    if (!e) e = alloc(S, &S->r, n);
    if (!e) e = alloc(S, &S->delta, n);
    if (!e) e = alloc(S, &S->M, 9 * G);
    if (!e && cudaMalloc(&S->piv, sizeof(int32_t) * (G > 0 ? G : 1)) != cudaSuccess) e = SUNBW_ERR_MEM;
  }
  if (!e && opt->linsol == 1) {
    S->gm = sunbw::spgmr_create(ctx, G, 3, opt->maxl, true);
    if (!S->gm) e = SUNBW_ERR_MEM;
  }
  if (!e && opt->fused && opt->newton_mode == 0 && !opt->single_step_launches)
    S->small = sunbw::bw_small_geometry(prob, &S->sg);
  if (!e && opt->fused && ctx_nranks(ctx) > 1) {
    S->deferred = opt->newton_mode == 0;
    if (cudaStreamCreateWithFlags(&S->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->evA, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->evB, cudaEventDisableTiming) != cudaSuccess)
      e = SUNBW_ERR_CUDA;
    if (!e) e = alloc(S, &S->d_pending, kMaxK + 2);
    // copy-engine halo for the fused step (collective; falls back to NCCL
    // send/recv when peer mappings are unavailable on any rank)
    sunbw::FusedAdvection fa;
    if (!e && opt->fused_advection && sunbw::bw_fused_advection(prob, y0->d, &fa))
      ctx->comm->peer_setup((size_t)(3 * fa.nx * fa.ny), ctx->stream);
  }
  if (!e) e = alloc(S, &S->d_scal, kMaxK + 8);
  if (!e) e = alloc(S, &S->d_partials, (int64_t)(ctx->nsm * 16) * (kMaxK + 1));
  if (!e && cudaMalloc(&S->d_first, sizeof(unsigned long long)) != cudaSuccess) e = SUNBW_ERR_MEM;
  if (!e && cudaMalloc(&S->d_err, sizeof(int)) != cudaSuccess) e = SUNBW_ERR_MEM;
  if (!e && cudaMalloc(&S->d_counter, sizeof(unsigned)) != cudaSuccess) e = SUNBW_ERR_MEM;
  if (!e && cudaHostAlloc(&S->h_end, 4 * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess)
    e = SUNBW_ERR_MEM;
  if (!e && opt->fused && opt->newton_mode == 1 &&
      cudaHostAlloc(&S->h_tol, sizeof(double) * (kMaxKF + 4), cudaHostAllocDefault) != cudaSuccess)
    e = SUNBW_ERR_MEM;
  sunbw::FusedAdvection fa_t;
  const bool adv_fused = opt->fused && opt->fused_advection && sunbw::bw_fused_advection(prob, y0->d, &fa_t) &&
                         G % 128 == 0 && G <= INT32_MAX;
  if (!e && opt->fused && opt->newton_mode == 1 && ctx_nranks(ctx) == 1 && adv_fused &&
      (cudaMalloc(&S->d_tdev, sizeof(sunbw::TolDev)) != cudaSuccess ||
       cudaHostAlloc(&S->h_tdev, sizeof(sunbw::TolDev), cudaHostAllocDefault) != cudaSuccess ||
       cudaHostAlloc(&S->h_tdone, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
       cudaHostGetDevicePointer((void**)&S->d_tdone, S->h_tdone, 0) != cudaSuccess ||
       cudaEventCreateWithFlags(&S->tev[0], cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&S->tev[1], cudaEventDisableTiming) != cudaSuccess))
    e = SUNBW_ERR_MEM;
  if (e) {
    cudaGetLastError();
    BW_StepperDestroy(S);
    return ctx_set_err(ctx, e);
  }
  if (cudaMemcpyAsync(S->y[S->iy], y0->d, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(S->d_first, 0xFF, sizeof(unsigned long long), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(S->d_err, 0, sizeof(int), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(S->d_counter, 0, sizeof(unsigned), ctx->stream) != cudaSuccess) {
    BW_StepperDestroy(S);
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  }
  *out = S;
  return 0;
}

// Fused tolerance mode, one rank, in-kernel advection, after the first
// step (R35): up to n steps with the decisions on the device.  Each launch is
// one attempt of the current step (the kernel takes its buffers and
// iteration count from TolDev, its last CTA decides); the host keeps two
// launches in flight and stops enqueuing once the mapped done flag is set
// (at most one no-op launch follows).  *done = steps completed; *rc = the
// recoverable code of a failed step (the Advance ends there), else 0.
int tol_device_advance(Stepper* S, int64_t n, int64_t* done, int* rc) {
  SUNBW_Context ctx = S->ctx;
  const BW_StepperOptions& o = S->opt;
  sunbw::FusedAdvection fa;
  if (!sunbw::bw_fused_advection(S->prob, S->y[S->iy], &fa)) return ctx_set_err(ctx, SUNBW_ERR_ARG);
  sunbw::TolDev& T = *S->h_tdev;
  std::memset(&T, 0, sizeof(T));
  for (int i = 0; i < 3; ++i) T.y[i] = S->y[i];
  for (int i = 0; i < 2; ++i) T.H[i] = S->fE[i];
  T.iy = S->iy; T.iyp = S->iyp; T.iz = S->iz; T.ife = S->ife; T.ifep = S->ifep;
  T.K = o.K;
  T.Kr = S->k_pred > 0 && S->k_pred <= o.K ? S->k_pred : o.K;
  T.k_pred = S->k_pred;
  T.nsteps = n;
  T.tol_nl = o.tol_nl;
  T.below_off = (long long)(fa.below - S->y[S->iy]);
  T.host_done = S->d_tdone;
  *(volatile int*)S->h_tdone = 0;
  if (cudaMemcpyAsync(S->d_tdev, &T, sizeof(T), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  const int64_t max_launches = 3 * n + 2;            // <= 3 attempts per step
  for (int64_t k = 0;; ++k) {
    if (k > max_launches) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    int nb = 0;
    sunbw::FusedFold fold{0, S->d_counter, nullptr, S->d_scal, S->d_scal + 1, S->d_err, S->nglobal};
    {
      Timed t(S, BW_K_FUSED_NEWTON);
      // (pointer arguments: placeholders of the right shape; the kernel takes
      // the current ones from TolDev)
      TRY(sunbw::fused_newton(ctx, S->prob, S->G, false, o.K, o.h, o.rtol, o.atol, S->y[S->iy], nullptr,
                              S->fE[S->ifep], S->fE[S->ife], S->y[S->iz], S->d_partials, S->d_first, &nb, &fa, 0,
                              -1, &fold, 2, true, S->d_tdev));
    }
    if (cudaEventRecord(S->tev[k & 1], ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
    if (k > 0) {
      if (cudaEventSynchronize(S->tev[(k - 1) & 1]) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      if (*(volatile int*)S->h_tdone) break;
    }
  }
  if (cudaMemcpyAsync(&T, S->d_tdev, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (T.rc < 0) return ctx_set_err(ctx, T.rc);
  S->iy = T.iy; S->iyp = T.iyp; S->iz = T.iz; S->ife = T.ife; S->ifep = T.ifep;
  S->k_pred = T.k_pred;
  S->tol_launches += T.attempts;
  S->step += T.steps_done;
  S->t += (double)T.steps_done * o.h;
  S->st.steps += T.steps_done;
  S->st.setups += T.steps_done + T.setups_extra;
  S->st.newton_iters += T.newton_iters;
  if (T.steps_done > 0 || T.rc == SUNBW_RECOV_NONCONV) S->st.last_nu = T.last_nu;
  if (T.rc > 0) {
    S->st.fails++;
    if (T.rc == SUNBW_RECOV_SINGULAR) S->st.singular = (int64_t)T.singular;
  }
  *done = T.steps_done;
  *rc = T.rc;
  return 0;
}

extern "C" int BW_StepperAdvance(void* stepper, int64_t nsteps, N_Vector y_out, BW_StepperStats* stats) {
  auto* S = (Stepper*)stepper;
  if (!S || nsteps < 0) return SUNBW_ERR_ARG;
  SUNBW_Context ctx = S->ctx;
  if (y_out && (y_out->ctx != ctx || y_out->local_len != S->n)) return ctx_set_err(ctx, SUNBW_ERR_LENGTH);
  int rc = 0;
  if (S->deferred &&
      cudaMemsetAsync(S->d_pending + S->opt.K + 1, 0, sizeof(double), ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (S->small && nsteps > 0) {
    // the whole Advance in one launch (state on chip); bit-identical to the
    // per-step kernels
    {
      Timed t(S, BW_K_FUSED_NEWTON);
      TRY(sunbw::fused_multistep(ctx, S->prob, S->sg, S->G, S->step == 0, nsteps, S->opt.K,
                                 S->opt.numerics == 1 ? 2 : (S->opt.linsol == 2 ? 1 : 0),
                                 S->opt.h, S->opt.rtol, S->opt.atol, S->y[S->iy], S->fE[S->ifep], S->y[S->iz],
                                 S->fE[S->ife], S->d_scal, S->d_err, S->d_first, S->nglobal));
    }
    rotate(S);
    S->step += nsteps;
    S->t += (double)nsteps * S->opt.h;
    S->st.steps += nsteps;
    S->st.setups += nsteps;
    S->st.newton_iters += nsteps * S->opt.K;
  }
  const int64_t nloop = S->small ? 0 : nsteps;  // per-step launches
  for (int64_t s = 0; s < nloop;) {
    bool first = S->step == 0;
    if (!first && S->d_tdev) {                      // the rest of the Advance on the device (R35)
      int64_t nd = 0;
      TRY(tol_device_advance(S, nloop - s, &nd, &rc));
      s += nd;
      break;
    }
    int nin = 1;                                  // steps done by this iteration
    if (S->opt.use_graph && !first) {
      int key = graph_key(S);
      if (!S->gexec[key]) {
        int e = capture_all_keys(S);
        if (e) return e;
      }
      if (nloop - s >= kChain && S->gexec[key + 6]) {   // kChain steps in one graph launch
        key += 6;
        nin = kChain;
      }
      if (S->opt.timing && !S->ev_nodes[key].empty()) {
        const std::vector<cudaGraphNode_t>& nodes = S->ev_nodes[key];
        while (S->ev_used + nodes.size() > S->ev_pool.size()) {
          for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            S->ev_pool.push_back(e);
          }
        }
        for (size_t j = 0; j < nodes.size(); ++j)
          if (cudaGraphExecEventRecordNodeSetEvent(S->gexec[key], nodes[j], S->ev_pool[S->ev_used + j]) !=
              cudaSuccess)
            return ctx_set_err(ctx, SUNBW_ERR_CUDA);
        S->ev_used += nodes.size();
        S->ev_kind.insert(S->ev_kind.end(), S->ev_node_kind[key].begin(), S->ev_node_kind[key].end());
      }
      if (cudaGraphLaunch(S->gexec[key], ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
      ctx->launches += S->graph_launches[key];
      S->st.newton_iters += (int64_t)nin * S->opt.K;
      S->st.solves += S->opt.fused ? 0 : (int64_t)nin * S->opt.K;
    } else {
      int64_t it0 = S->st.newton_iters;
      rc = enqueue_step(S, first);
      if (S->opt.fused && S->opt.newton_mode == 0) S->st.newton_iters = it0 + S->opt.K;
      if (rc < 0) return rc;
      if (rc > 0) { S->st.fails++; break; }
    }
    for (int k = 0; k < nin; ++k) {
      S->st.setups++;
      rotate(S);
      S->step++;
      S->t += S->opt.h;
      S->st.steps++;
    }
    s += nin;
  }
  // end of the call: one synchronisation for the deferred checks
  unsigned long long f = 0;
  int err = 0;
  double nu = 0.0;
  if (S->deferred && nsteps > 0) {
    int e = sunbw::fused_finalize_pending(ctx, S->d_pending, S->opt.K, S->nglobal, S->d_scal,
                                          S->d_scal + 1, S->d_err);
    if (e) return e;
  }
  if (S->opt.newton_mode == 0 && ctx_nranks(ctx) > 1) {
    // every rank returns the same code: OR the local flags over the ranks
    TRY(sunbw::or_flags_over_ranks(ctx, S->d_first, S->d_err));
  }
  if (S->opt.newton_mode == 0) {
    // into pinned memory: asynchronous copies, one synchronisation below
    // (pageable destinations would each block in a staging copy)
    if (cudaMemcpyAsync(S->h_end, S->d_first, sizeof(f), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(S->h_end + 1, S->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(S->h_end + 2, S->d_scal + S->opt.K, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream) !=
            cudaSuccess)
      return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  }
  if (y_out &&
      cudaMemcpyAsync(y_out->d, S->y[S->iy], sizeof(double) * S->n, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  if (S->opt.newton_mode == 0) {
    std::memcpy(&f, S->h_end, sizeof(f));
    std::memcpy(&err, S->h_end + 1, sizeof(int));
    std::memcpy(&nu, S->h_end + 2, sizeof(double));
  }
  // timing events are read lazily (BW_StepperKernelTimes, or the next call
  // once many are pending): no host work after the step kernels here
  if (S->opt.timing && S->ev_used > 4096) harvest_timing(S);
  if (S->opt.newton_mode == 0 && nsteps > 0) {
    S->st.last_nu = nu;
    if (f != ~0ull) { S->st.singular = (int64_t)f; rc = rc ? rc : SUNBW_RECOV_SINGULAR; }
    if (err) rc = rc ? rc : SUNBW_RECOV_BAD_EWT;
  }
  S->st.t = S->t;
  if (stats) *stats = S->st;
  return rc;
}

extern "C" int BW_StepperReset(void* stepper, N_Vector y0, double t0) {
  auto* S = (Stepper*)stepper;
  if (!S || !y0) return SUNBW_ERR_ARG;
  SUNBW_Context ctx = S->ctx;
  if (y0->ctx != ctx || y0->local_len != S->n) return ctx_set_err(ctx, SUNBW_ERR_LENGTH);
  S->iy = 0; S->iyp = 1; S->iz = 2; S->ife = 0; S->ifep = 1;   // graphs stay valid per key
  if (cudaMemcpyAsync(S->y[S->iy], y0->d, sizeof(double) * S->n, cudaMemcpyDeviceToDevice,
                      ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(S->d_first, 0xFF, sizeof(unsigned long long), ctx->stream) != cudaSuccess ||
      cudaMemsetAsync(S->d_err, 0, sizeof(int), ctx->stream) != cudaSuccess)
    return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  S->step = 0;
  S->t = t0;
  S->st = BW_StepperStats{};
  return 0;
}

extern "C" int BW_StepperKernelTimes(void* stepper, double* ms, int64_t* launches, int reset) {
  auto* S = (Stepper*)stepper;
  if (!S) return SUNBW_ERR_ARG;
  if (S->opt.timing && !S->ev_kind.empty()) {
    if (cudaStreamSynchronize(S->ctx->stream) != cudaSuccess) return ctx_set_err(S->ctx, SUNBW_ERR_CUDA);
    harvest_timing(S);
  }
  for (int k = 0; k < BW_K_COUNT_; ++k) {
    if (ms) ms[k] = S->k_ms[k];
    if (launches) launches[k] = S->k_count[k];
    if (reset) { S->k_ms[k] = 0; S->k_count[k] = 0; }
  }
  return 0;
}

extern "C" int BW_StepperDestroy(void* stepper) {
  auto* S = (Stepper*)stepper;
  if (!S) return SUNBW_ERR_ARG;
  cudaStreamSynchronize(S->ctx->stream);
  for (auto& g : S->gexec)
    if (g) cudaGraphExecDestroy(g);
  for (auto& g : S->graph)
    if (g) cudaGraphDestroy(g);
  if (S->cap_stream) cudaStreamDestroy(S->cap_stream);
  for (auto e : S->ev_pool) cudaEventDestroy(e);
  double* bufs[] = {S->y[0], S->y[1], S->y[2], S->fE[0], S->fE[1], S->d, S->ewt, S->tmp,
                    S->fI, S->r, S->delta, S->M, S->d_scal, S->d_partials};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (S->piv) cudaFree(S->piv);
  if (S->d_first) cudaFree(S->d_first);
  if (S->d_counter) cudaFree(S->d_counter);
  if (S->d_err) cudaFree(S->d_err);
  if (S->gm) sunbw::spgmr_free(S->gm);
  if (S->side) cudaStreamDestroy(S->side);
  if (S->evA) cudaEventDestroy(S->evA);
  if (S->evB) cudaEventDestroy(S->evB);
  if (S->d_pending) cudaFree(S->d_pending);
  if (S->h_tol) cudaFreeHost(S->h_tol);
  if (S->d_tdev) cudaFree(S->d_tdev);
  if (S->h_tdev) cudaFreeHost(S->h_tdev);
  if (S->h_tdone) cudaFreeHost(S->h_tdone);
  for (auto ev : S->tev)
    if (ev) cudaEventDestroy(ev);
  if (S->h_end) cudaFreeHost(S->h_end);
  delete S;
  return 0;
}
