// sunbw_internal.h — private declarations shared by the libsunbw sources.
// (Never included by the oracle; the oracle shares nothing with this tree.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "sunbw.h"

#define SUNBW_MAX_SM 256

// ------------------------------------------------------------ communicator
enum RedOp { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

struct PeerHalo;   // peer_halo.cu

struct Comm {
  int rank = 0, nranks = 1;
  PeerHalo* peer = nullptr;            // copy-engine halo into the right neighbour (peer_halo.cu)
  virtual ~Comm();
  // collective: make `peer` ready for halos of up to `count` doubles;
  // 0 = ready, > 0 = not available (the caller uses halo_shift)
  virtual int peer_setup(size_t count, cudaStream_t s) { (void)count; (void)s; return 1; }
  // in-place allreduce of `count` doubles in device memory, on stream s
  virtual int allreduce(double* d_buf, int count, RedOp op, cudaStream_t s) = 0;
  // ring shift: send `count` doubles to rank+1, receive from rank-1
  virtual int halo_shift(const double* d_send, double* d_recv, size_t count,
                         cudaStream_t s) = 0;
  virtual bool capturable() const = 0;   // may run inside CUDA graph capture
};

namespace sunbw {
bool peer_halo_supported();
PeerHalo* peer_halo_alloc(size_t cap, int* err);
void peer_halo_free(PeerHalo* h);
double* peer_halo_base(PeerHalo* h);
size_t peer_halo_capacity(const PeerHalo* h);
void peer_halo_connect(PeerHalo* h, double* right_base, double* left_base);
void peer_halo_set_ipc(PeerHalo* h, void* right_map, void* left_map);
// sender (side stream): wait until the right neighbour freed the slot, copy
// `send` into it, raise its arrival flag
int peer_halo_send(PeerHalo* h, const double* send, size_t count, cudaStream_t side);
// receiver (main stream): wait for this exchange's data; *recv = the slot
int peer_halo_wait(PeerHalo* h, cudaStream_t main, const double** recv);
// receiver (main stream, after the consumer kernel): free the slot
int peer_halo_release(PeerHalo* h, cudaStream_t main);
}  // namespace sunbw

Comm* make_nccl_comm(const void* uid, int rank, int nranks, int* err);
Comm* make_fake_comm_member(void* shared, int rank, int* err);

// ----------------------------------------------------------------- context
struct SUNBW_Context_ {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nsm = 148;
  int err = 0;                          // sticky error
  std::atomic<int64_t> launches{0};
  Comm* comm = nullptr;                 // nullptr: single rank
  // reduction scratch (stable addresses: usable inside graph capture)
  double* d_partials = nullptr;         // kPartialsCap doubles
  double* d_red = nullptr;              // kRedSlots doubles (device results)
  double* h_slot = nullptr;             // pinned-mapped host slot
  double* h_slot_dev = nullptr;         // its device alias
  unsigned long long* d_flag = nullptr; // LU singular-block min
  static constexpr int kPartialsCap = 1 << 16;
  static constexpr int kRedSlots = 256;
};

int  ctx_set_err(SUNBW_Context ctx, int code);
int  ctx_check_launch(SUNBW_Context ctx);   // cudaGetLastError -> sticky
inline int ctx_rank(SUNBW_Context c) { return c->comm ? c->comm->rank : 0; }
inline int ctx_nranks(SUNBW_Context c) { return c->comm ? c->comm->nranks : 1; }

// ---------------------------------------------------------------- N_Vector
struct _N_Vector {
  SUNBW_Context ctx;
  int64_t local_len;
  int64_t global_len;
  double* d;
  bool owned;
  int policy = SUNBW_POLICY_GRID_STRIDE;
  int block = 256;
  int grid = 0;
  int reduce_block = 256;
};

// ---------------------------------------------------------- block matrix
struct _SUNMatrix {
  SUNBW_Context ctx;
  int64_t nblocks;
  int m;
  double* d;
  bool owned;
};

struct _SUNLinearSolver {
  int type = 0;                 // 0: batched block LU, 1: SPGMR (gmres.cu), 2: batched GJ inverse
  SUNBW_Context ctx;
  int64_t nblocks;
  int m;
  int32_t* d_piv;
  int deferred = 0;
  int64_t last_flag = 0;
  bool flag_pending = false;
};

// ------------------------------------------- internal (device-result) API
// Launch-level entry points used by the driver; they never synchronise.
// Results land in device memory so that a step can be graph-captured.
namespace sunbw {

struct LaunchCfg {
  int block;
  int grid;
};

// streaming
int linear_sum(SUNBW_Context, int64_t n, double a, const double* x, double b,
               const double* y, double* z, const _N_Vector* pol);
int scale(SUNBW_Context, int64_t n, double c, const double* x, double* z,
          const _N_Vector* pol);
int abs_(SUNBW_Context, int64_t n, const double* x, double* z, const _N_Vector* pol);
int add_const(SUNBW_Context, int64_t n, const double* x, double b, double* z,
              const _N_Vector* pol);
int inv(SUNBW_Context, int64_t n, const double* x, double* z, const _N_Vector* pol);
// fused z = Σ c_j X_j (nv any)
int linear_combination(SUNBW_Context, int64_t n, int nv, const double* c,
                       const double* const* X, double* z, const _N_Vector* pol);

// reductions.  kind: see RedKind.  Writes the GLOBAL result (after the
// communicator's allreduce and the finalisation) to d_out[0..nv) and, if
// h_out_dev != nullptr, also to that (mapped host) address.
enum RedKind { RK_DOT = 0, RK_WSQR = 1, RK_WSQR_MASK = 2, RK_MAXABS = 3, RK_MIN = 4 };
enum RedFinal { RF_NONE = 0, RF_WRMS = 1 };
int reduce(SUNBW_Context, RedKind kind, RedFinal fin, int64_t n_local,
           int64_t n_global, const double* x, const double* y, const double* id,
           double* d_out, double* h_out_dev, bool global, const _N_Vector* pol);
int dot_multi(SUNBW_Context, int64_t n_local, int nv, const double* x,
              const double* const* Y, double* d_out, double* h_out_dev,
              bool global, const _N_Vector* pol);

// kernel: d_flag |= (d_val[0] <= 0) for the ewt check
int flag_nonpositive(SUNBW_Context, const double* d_val, int* d_flag);

// block diagonal
int scale_add_identity(SUNBW_Context, int64_t G, int m, double c, double* A);
int lu_factor(SUNBW_Context, int64_t G, int m, double* A, int32_t* piv,
              unsigned long long* d_first_singular);
int lu_solve(SUNBW_Context, int64_t G, int m, const double* LU,
             const int32_t* piv, const double* b, double* x);
int block_matvec(SUNBW_Context, int64_t G, int m, const double* A,
                 const double* x, double* y);

int lu_factor_noreset(SUNBW_Context, int64_t G, int m, double* A, int32_t* piv,
                      unsigned long long* d_first);
// block inverses in place by symbolic Gauss-Jordan (R29) and their apply;
// reset = false accumulates the first singular block into d_first
int gj_inverse(SUNBW_Context, int64_t G, int m, double* A, unsigned long long* d_first, bool reset = true);
int gj_apply(SUNBW_Context, int64_t G, int m, const double* Ainv, const double* b, double* x);

// SPGMR (gmres.cu): dispatched from the SUNLinSol* entry points
SUNLinearSolver spgmr_create(SUNBW_Context ctx, int64_t G, int m, int maxl, bool block_prec);
int spgmr_setup_raw(SUNLinearSolver S, const double* A, unsigned long long* d_first_accum);
int spgmr_setup(SUNLinearSolver S, SUNMatrix A);
int spgmr_solve(SUNLinearSolver S, SUNMatrix A, N_Vector x, N_Vector b, double tol);
void spgmr_free(SUNLinearSolver S);
// device-pointer form used by the driver: operator A (G blocks of 3x3),
// solves A x = b to relative residual tol; returns Arnoldi steps or < 0
int spgmr_solve_raw(SUNLinearSolver S, const double* A, double* x, const double* b, double tol);
int64_t spgmr_last_iters(SUNLinearSolver S);

// geometry for the fused step kernel's in-kernel 3D advection
struct FusedAdvection {
  int64_t nx, ny, nzl;       // local slab extents (nx % 128 == 0)
  double kx, ky, kz;
  const double* below;       // the plane under local plane 0 (halo or own last)
};
// fills *fa and returns true when the problem's advection can be fused into
// the Newton kernel (3D Brusselator, nx % 128 == 0, ny > 1, nz > 1)
bool bw_fused_advection(void* prob, const double* y, FusedAdvection* fa);

// In-kernel fold of the fused step's per-CTA partials: the last CTA of the
// step's final launch (self-resetting arrival counter) folds every partial
// of the step in fixed order and writes either the finalised values (d_min,
// d_nu, d_err; no communicator) or the local pending record (pending != 0).
// Geometry of a problem small enough for one CTA (one rank): the fused
// multi-step kernel keeps the whole state on chip and runs many steps per
// launch (launch-bound small problems).
constexpr int kSmallCells = 512;
struct SmallGeom {
  int nx, ny, nz;            // global = local extents (one rank)
  double kx, ky, kz;         // upwind coefficients (terms of extent-1 axes vanish)
  int expl;                  // 0: upwind advection, 1: f_E = λ_E y, 2: f_E = 0
  double lam_E;
};
bool bw_small_geometry(void* prob, SmallGeom* g);
int fused_multistep(SUNBW_Context ctx, void* prob, const SmallGeom& gm, int64_t G, bool first, int64_t nsteps,
                    int K, int solver, double h, double rtol, double atol, const double* y, const double* hin,
                    double* y_out, double* hout, double* d_scal, int* d_err, unsigned long long* d_first,
                    int64_t nglobal);

// OR the local recoverable-failure flags over the ranks (the ensemble
// of task-local solves succeeds or fails as one): afterwards *d_first is
// unchanged, or 0 if a singular block was flagged only on another rank, and
// *d_err (may be nullptr) is 1 if any rank set it.  No-op on one rank.
int or_flags_over_ranks(SUNBW_Context ctx, unsigned long long* d_first, int* d_err);

// Geometry and explicit operator of a problem for the fused ARK stage
// kernels (ark_fused.cu): local extents, which axes carry an advection term,
// and the explicit operator kind (0 upwind advection, 1 f_E = λ_E y, 2 f_E = 0)
struct ArkGeometry {
  int dim, expl, has_y, has_z;
  int64_t nx, ny, nzl, G, halo_len;
  double kx, ky, kz, lam_E;
};
void bw_ark_geometry(void* prob, ArkGeometry* g);
// the fused ARK stages and their device-driven Evolve loop (ark_fused.cu)
struct ArkFused;
ArkFused* ark_fused_create(SUNBW_Context ctx, void* prob, int64_t nglobal);
void ark_fused_destroy(ArkFused* F);
int ark_fused_evolve(ArkFused* F, double** y, double** ynew, double* t, double* h, double t_end,
                     const BW_ArkOptions& opt, BW_ArkStats* st, int* rc);

// Fused tolerance mode driven from the device (DESIGN R35; one rank, in-
// kernel advection): the rotation of the state buffers, the iteration count
// of the next launch and the step's decision live here; the step kernel
// reads them at entry and its last CTA takes the oracle's decision (R31)
// after folding the norms, so the host enqueues launches without waiting.
struct TolDev {
  double* y[3];              // state buffers (S->y)
  double* H[2];              // SBDF2 history buffers (S->fE)
  int iy, iyp, iz, ife, ifep;
  int Kr, K, k_pred;
  int done, rc;              // rc: 0 or SUNBW_RECOV_*
  int attempt;               // launches of the current step so far
  long long nsteps, steps_done, newton_iters, setups_extra, attempts;
  unsigned long long singular;
  double last_nu, tol_nl;
  long long below_off;       // y + below_off: the plane under local plane 0 (own wrap)
  volatile int* host_done;   // mapped pinned: done after the latest launch
};

struct FusedFold {
  int prev_parts;            // partial rows written by earlier launches of this step
  unsigned* counter;         // zero-initialised
  double* pending;           // K + 2: [min, sums], flag  (deferred mode)
  double* d_min;
  double* d_nu;
  int* d_err;
  int64_t nglobal;
};

}  // namespace sunbw

#define SUNBW_CUDA_TRY(ctx, expr)                                \
  do {                                                           \
    cudaError_t e_ = (expr);                                     \
    if (e_ != cudaSuccess) return ctx_set_err((ctx), SUNBW_ERR_CUDA); \
  } while (0)
