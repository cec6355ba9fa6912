// context.cu — execution context, sticky errors, communicators.
//
// The context carries what SUNDIALS splits between SUNMemoryHelper, the
// vector's stream setter and the MPIPlusX communicator (§3,
// P:214-215 §4.1, §4): the CUDA stream every object runs on, the
// scratch for block reductions, the pinned-mapped host slot through which a
// reduction returns its scalar (§4.1), and the communicator that
// finishes reductions and exchanges halos.

#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "sunbw_internal.h"

// ------------------------------------------------------------------ errors
int ctx_set_err(SUNBW_Context ctx, int code) {
  if (ctx && code < 0 && ctx->err == 0) ctx->err = code;
  static const bool debug = [] {
    const char* e = std::getenv("SUNBW_DEBUG");
    return e && e[0] == '1';
  }();
  if (debug && code < 0) {                         // diagnostics: the pending CUDA error, if any
    const cudaError_t ce = cudaPeekAtLastError();
    std::fprintf(stderr, "[sunbw] error %d (cuda: %s)\n", code, cudaGetErrorString(ce));
  }
  return code;
}

int ctx_check_launch(SUNBW_Context ctx) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  return 0;
}

extern "C" const char* SUNBW_ErrorString(int code) {
  switch (code) {
    case SUNBW_SUCCESS: return "success";
    case SUNBW_RECOV_SINGULAR: return "recoverable: singular block (zero pivot)";
    case SUNBW_RECOV_NONCONV: return "recoverable: Newton iteration did not converge";
    case SUNBW_RECOV_BAD_EWT: return "recoverable: non-positive error-weight denominator";
    case SUNBW_ERR_ARG: return "invalid argument";
    case SUNBW_ERR_LENGTH: return "vector length mismatch";
    case SUNBW_ERR_CONTEXT: return "objects belong to different contexts";
    case SUNBW_ERR_CUDA: return "CUDA error";
    case SUNBW_ERR_COMM: return "communicator (NCCL) error";
    case SUNBW_ERR_EMPTY: return "reduction over an empty vector";
    case SUNBW_ERR_MEM: return "allocation failure";
    case SUNBW_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown error";
  }
}

// ----------------------------------------------------------------- context
extern "C" int SUNBW_ContextCreate(int device, void* stream, SUNBW_Context* out) {
  if (!out) return SUNBW_ERR_ARG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return SUNBW_ERR_CUDA;
  auto* c = new SUNBW_Context_();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    delete c;
    return SUNBW_ERR_CUDA;
  }
  c->nsm = nsm;
  bool ok = cudaMalloc(&c->d_partials, sizeof(double) * SUNBW_Context_::kPartialsCap) == cudaSuccess &&
            cudaMalloc(&c->d_red, sizeof(double) * SUNBW_Context_::kRedSlots) == cudaSuccess &&
            cudaMalloc(&c->d_flag, sizeof(unsigned long long) * 4) == cudaSuccess &&
            cudaHostAlloc(&c->h_slot, sizeof(double) * 64, cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer((void**)&c->h_slot_dev, c->h_slot, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    SUNBW_ContextDestroy(c);
    return SUNBW_ERR_MEM;
  }
  *out = c;
  return 0;
}

extern "C" int SUNBW_ContextSetStream(SUNBW_Context ctx, void* stream) {
  if (!ctx) return SUNBW_ERR_ARG;
  ctx->stream = (cudaStream_t)stream;
  return 0;
}

extern "C" void* SUNBW_ContextGetStream(SUNBW_Context ctx) {
  return ctx ? (void*)ctx->stream : nullptr;
}

extern "C" int SUNBW_ContextDestroy(SUNBW_Context ctx) {
  if (!ctx) return SUNBW_ERR_ARG;
  cudaStreamSynchronize(ctx->stream);
  delete ctx->comm;
  if (ctx->d_partials) cudaFree(ctx->d_partials);
  if (ctx->d_red) cudaFree(ctx->d_red);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  if (ctx->h_slot) cudaFreeHost(ctx->h_slot);
  delete ctx;
  return 0;
}

extern "C" int SUNBW_GetLastError(SUNBW_Context ctx, int clear) {
  if (!ctx) return SUNBW_ERR_ARG;
  int e = ctx->err;
  if (clear) ctx->err = 0;
  return e;
}

extern "C" int64_t SUNBW_ContextKernelLaunches(SUNBW_Context ctx) {
  return ctx ? ctx->launches.load() : -1;
}

extern "C" int SUNBW_ContextRank(SUNBW_Context ctx) { return ctx ? ctx_rank(ctx) : -1; }
extern "C" int SUNBW_ContextNRanks(SUNBW_Context ctx) { return ctx ? ctx_nranks(ctx) : -1; }

Comm::~Comm() { sunbw::peer_halo_free(peer); }

// -------------------------------------------------------------------- NCCL
// Reductions finish with ncclAllReduce over NVLink (MPIPlusX global step,
// P:133-135 §4); the advection halo is a ring shift with ncclSend/Recv (the
// GPU-to-GPU point-to-point exchange of P:394 §7).
namespace {

ncclRedOp_t to_nccl(RedOp op) {
  return op == RED_SUM ? ncclSum : (op == RED_MAX ? ncclMax : ncclMin);
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  int allreduce(double* d, int count, RedOp op, cudaStream_t s) override {
    if (nranks == 1) return 0;
    return ncclAllReduce(d, d, count, ncclDouble, to_nccl(op), comm, s) == ncclSuccess
               ? 0 : SUNBW_ERR_COMM;
  }
  int halo_shift(const double* send, double* recv, size_t count, cudaStream_t s) override {
    int right = (rank + 1) % nranks, left = (rank + nranks - 1) % nranks;
    if (ncclGroupStart() != ncclSuccess) return SUNBW_ERR_COMM;
    ncclResult_t a = ncclSend(send, count, ncclDouble, right, comm, s);
    ncclResult_t b = ncclRecv(recv, count, ncclDouble, left, comm, s);
    ncclResult_t c = ncclGroupEnd();
    return (a == ncclSuccess && b == ncclSuccess && c == ncclSuccess) ? 0 : SUNBW_ERR_COMM;
  }
  bool capturable() const override { return true; }
  // one process per GPU: IPC handles of every rank's halo buffers, all-
  // gathered over NCCL, the neighbours' opened here; all ranks agree on the
  // outcome (allreduce of the local result) before anyone uses it
  int peer_setup(size_t count, cudaStream_t s) override {
    if (nranks == 1) return 1;
    if (peer && sunbw::peer_halo_capacity(peer) >= count) return 0;
    sunbw::peer_halo_free(peer);
    peer = nullptr;
    int ok = sunbw::peer_halo_supported() ? 1 : 0, err = 0;
    PeerHalo* h = ok ? sunbw::peer_halo_alloc(count, &err) : nullptr;
    ok = h != nullptr;
    cudaIpcMemHandle_t mine{};
    if (ok) ok = cudaIpcGetMemHandle(&mine, sunbw::peer_halo_base(h)) == cudaSuccess;
    std::vector<char> all(sizeof(cudaIpcMemHandle_t) * nranks);
    char *d_all = nullptr, *d_mine = nullptr;
    double* d_ok = nullptr;
    if (cudaMalloc(&d_all, all.size()) != cudaSuccess || cudaMalloc(&d_mine, sizeof(mine)) != cudaSuccess ||
        cudaMalloc(&d_ok, sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return 1;
    }
    const double okd = ok ? 1.0 : 0.0;
    cudaMemcpyAsync(d_mine, &mine, sizeof(mine), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_ok, &okd, sizeof(double), cudaMemcpyHostToDevice, s);
    bool nccl_ok = ncclAllGather(d_mine, d_all, sizeof(mine), ncclChar, comm, s) == ncclSuccess &&
                   ncclAllReduce(d_ok, d_ok, 1, ncclDouble, ncclMin, comm, s) == ncclSuccess;
    double all_ok = 0.0;
    cudaMemcpyAsync(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&all_ok, d_ok, sizeof(double), cudaMemcpyDeviceToHost, s);
    nccl_ok = nccl_ok && cudaStreamSynchronize(s) == cudaSuccess;
    cudaFree(d_all);
    cudaFree(d_mine);
    cudaFree(d_ok);
    void *rmap = nullptr, *lmap = nullptr;
    const int right = (rank + 1) % nranks, left = (rank + nranks - 1) % nranks;
    int open_ok = 1;
    if (nccl_ok && all_ok == 1.0) {
      cudaIpcMemHandle_t hr, hl;
      std::memcpy(&hr, all.data() + right * sizeof(hr), sizeof(hr));
      std::memcpy(&hl, all.data() + left * sizeof(hl), sizeof(hl));
      open_ok = cudaIpcOpenMemHandle(&rmap, hr, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (open_ok) lmap = rmap;
      if (open_ok && left != right)
        open_ok = cudaIpcOpenMemHandle(&lmap, hl, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (!open_ok) cudaGetLastError();
    }
    // second agreement: every rank opened its neighbours
    double o2 = (nccl_ok && all_ok == 1.0 && open_ok) ? 1.0 : 0.0, all2 = 0.0;
    double* d2 = nullptr;
    if (cudaMalloc(&d2, sizeof(double)) == cudaSuccess) {
      cudaMemcpyAsync(d2, &o2, sizeof(double), cudaMemcpyHostToDevice, s);
      if (ncclAllReduce(d2, d2, 1, ncclDouble, ncclMin, comm, s) == ncclSuccess) {
        cudaMemcpyAsync(&all2, d2, sizeof(double), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) all2 = 0.0;
      }
      cudaFree(d2);
    }
    if (all2 != 1.0) {
      if (rmap) cudaIpcCloseMemHandle(rmap);
      if (lmap && lmap != rmap) cudaIpcCloseMemHandle(lmap);
      sunbw::peer_halo_free(h);
      cudaGetLastError();
      return 1;
    }
    sunbw::peer_halo_connect(h, (double*)rmap, (double*)lmap);
    sunbw::peer_halo_set_ipc(h, rmap, lmap);
    peer = h;
    return 0;
  }
};

}  // namespace

Comm* make_nccl_comm(const void* uid, int rank, int nranks, int* err) {
  auto* c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  if (ncclCommInitRank(&c->comm, nranks, id, rank) != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    *err = SUNBW_ERR_COMM;
    return nullptr;
  }
  *err = 0;
  return c;
}

extern "C" int SUNBW_NcclGetUniqueId(void* out) {
  if (!out) return SUNBW_ERR_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SUNBW_ERR_COMM;
  std::memcpy(out, &id, 128);
  return 0;
}

extern "C" int SUNBW_ContextInitNccl(SUNBW_Context ctx, const void* uid, int rank, int nranks) {
  if (!ctx || !uid || nranks < 1 || rank < 0 || rank >= nranks) return SUNBW_ERR_ARG;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return ctx_set_err(ctx, SUNBW_ERR_CUDA);
  int err = 0;
  Comm* c = make_nccl_comm(uid, rank, nranks, &err);
  if (!c) return ctx_set_err(ctx, err);
  delete ctx->comm;
  ctx->comm = c;
  return 0;
}

// ---------------------------------------------------------- fake communicator
// P logical ranks inside one process (one host thread per rank, one GPU):
// the analog of SPEC's in-process ranks.  NCCL forbids two ranks on
// one device, so multi-rank logic is tested through this instead.
namespace {

__global__ void k_fold_ranks(const double* const* bufs, int nranks, int count,
                             int op, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double acc = bufs[0][i];
  for (int r = 1; r < nranks; ++r) {     // ascending rank order (DESIGN R7)
    double v = bufs[r][i];
    if (op == RED_SUM) acc = __dadd_rn(acc, v);
    else if (op == RED_MAX) acc = (v > acc) ? v : acc;
    else acc = (v < acc) ? v : acc;
  }
  out[i] = acc;
}

struct FakeShared {
  int nranks;
  std::vector<double*> peer_base;       // per rank: its PeerHalo buffer (in-process)
  std::vector<int> peer_ok;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<const double*> ptr;
  std::vector<cudaEvent_t> ev;
  const double** d_ptrs = nullptr;      // device copy of ptr[] per rank slot
  explicit FakeShared(int n) : nranks(n), peer_base(n, nullptr), peer_ok(n, 0), ptr(n), ev(n, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct FakeMember : Comm {
  FakeShared* sh;
  cudaEvent_t ev = nullptr;
  double* d_tmp = nullptr;
  const double** d_ptrs = nullptr;
  int cap = 0;
  ~FakeMember() override {
    if (ev) cudaEventDestroy(ev);
    if (d_tmp) cudaFree(d_tmp);
    if (d_ptrs) cudaFree(d_ptrs);
  }
  int publish(const double* p, cudaStream_t s) {
    if (cudaEventRecord(ev, s) != cudaSuccess) return SUNBW_ERR_CUDA;
    sh->ptr[rank] = p;
    sh->ev[rank] = ev;
    return 0;
  }
  int allreduce(double* d, int count, RedOp op, cudaStream_t s) override {
    if (nranks == 1) return 0;
    if (count > cap) {
      if (d_tmp) cudaFree(d_tmp);
      cap = count < 64 ? 64 : count;
      if (cudaMalloc(&d_tmp, sizeof(double) * cap) != cudaSuccess) return SUNBW_ERR_MEM;
    }
    if (publish(d, s)) return SUNBW_ERR_CUDA;
    sh->barrier();                                   // all partials published
    for (int q = 0; q < nranks; ++q)
      if (q != rank) cudaStreamWaitEvent(s, sh->ev[q], 0);
    std::vector<const double*> ptrs(sh->ptr);
    cudaMemcpyAsync(d_ptrs, ptrs.data(), sizeof(double*) * nranks, cudaMemcpyHostToDevice, s);
    k_fold_ranks<<<(count + 127) / 128, 128, 0, s>>>(d_ptrs, nranks, count, (int)op, d_tmp);
    cudaEventRecord(ev, s);
    sh->barrier();                                   // everyone enqueued its fold
    for (int q = 0; q < nranks; ++q)
      if (q != rank) cudaStreamWaitEvent(s, sh->ev[q], 0);
    sh->barrier();                                   // waits enqueued before reuse
    cudaMemcpyAsync(d, d_tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
    return cudaGetLastError() == cudaSuccess ? 0 : SUNBW_ERR_CUDA;
  }
  int halo_shift(const double* send, double* recv, size_t count, cudaStream_t s) override {
    int left = (rank + nranks - 1) % nranks;
    if (publish(send, s)) return SUNBW_ERR_CUDA;
    sh->barrier();
    cudaStreamWaitEvent(s, sh->ev[left], 0);
    const double* src = sh->ptr[left];
    cudaMemcpyAsync(recv, src, sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
    sh->barrier();                                   // all reads of ev[] done
    cudaEventRecord(ev, s);
    sh->ev[rank] = ev;
    sh->barrier();
    int right = (rank + 1) % nranks;                 // it read my send buffer
    cudaStreamWaitEvent(s, sh->ev[right], 0);
    sh->barrier();
    return cudaGetLastError() == cudaSuccess ? 0 : SUNBW_ERR_CUDA;
  }
  bool capturable() const override { return false; }
  // in-process ranks on one device: the neighbours' buffers are plain
  // device pointers of this context
  int peer_setup(size_t count, cudaStream_t s) override {
    (void)s;
    if (nranks == 1) return 1;
    if (peer && sunbw::peer_halo_capacity(peer) >= count) return 0;
    sunbw::peer_halo_free(peer);
    peer = nullptr;
    int err = 0;
    PeerHalo* h = sunbw::peer_halo_supported() ? sunbw::peer_halo_alloc(count, &err) : nullptr;
    sh->peer_base[rank] = h ? sunbw::peer_halo_base(h) : nullptr;
    sh->peer_ok[rank] = h != nullptr;
    sh->barrier();
    bool all = true;
    for (int q = 0; q < nranks; ++q) all = all && sh->peer_ok[q];
    const int right = (rank + 1) % nranks, left = (rank + nranks - 1) % nranks;
    double *rb = sh->peer_base[right], *lb = sh->peer_base[left];
    sh->barrier();                                   // everyone read the table
    if (!all) {
      sunbw::peer_halo_free(h);
      return 1;
    }
    sunbw::peer_halo_connect(h, rb, lb);
    peer = h;
    return 0;
  }
};

}  // namespace

extern "C" int SUNBW_FakeCommCreate(int nranks, void** out) {
  if (!out || nranks < 1) return SUNBW_ERR_ARG;
  *out = new FakeShared(nranks);
  return 0;
}

extern "C" int SUNBW_FakeCommDestroy(void* comm) {
  delete (FakeShared*)comm;
  return 0;
}

Comm* make_fake_comm_member(void* shared, int rank, int* err) {
  auto* sh = (FakeShared*)shared;
  auto* m = new FakeMember();
  m->sh = sh;
  m->rank = rank;
  m->nranks = sh->nranks;
  if (cudaEventCreateWithFlags(&m->ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&m->d_ptrs, sizeof(double*) * sh->nranks) != cudaSuccess) {
    delete m;
    *err = SUNBW_ERR_CUDA;
    return nullptr;
  }
  *err = 0;
  return m;
}

extern "C" int SUNBW_ContextSetFakeComm(SUNBW_Context ctx, void* comm, int rank) {
  if (!ctx || !comm) return SUNBW_ERR_ARG;
  auto* sh = (FakeShared*)comm;
  if (rank < 0 || rank >= sh->nranks) return SUNBW_ERR_ARG;
  int err = 0;
  Comm* c = make_fake_comm_member(comm, rank, &err);
  if (!c) return ctx_set_err(ctx, err);
  delete ctx->comm;
  ctx->comm = c;
  return 0;
}

// ------------------------------------------------- launch-latency probe
// Launch overhead dominates small problems (~8 us per kernel on
// V100): the device time per back-to-back empty kernel launched eagerly, per
// empty kernel node replayed from one CUDA graph, and the host round trip of
// one launch + stream synchronisation.
namespace {
__global__ void k_empty() {}
}  // namespace

extern "C" int SUNBW_ProbeLaunchLatency(SUNBW_Context ctx, int64_t n, double* out3) {
  if (!ctx || n < 1 || n > 10000000 || !out3) return SUNBW_ERR_ARG;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  int rc = 0;
  float ms = 0.f;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    rc = SUNBW_ERR_CUDA;
    goto done;
  }
  // (a) eager launches, device time per launch
  for (int i = 0; i < 100; ++i) k_empty<<<1, 32, 0, s>>>();
  cudaEventRecord(e0, s);
  for (int64_t i = 0; i < n; ++i) k_empty<<<1, 32, 0, s>>>();
  cudaEventRecord(e1, s);
  if (cudaEventSynchronize(e1) != cudaSuccess) { rc = SUNBW_ERR_CUDA; goto done; }
  cudaEventElapsedTime(&ms, e0, e1);
  out3[0] = 1e3 * ms / (double)n;
  {
    // (b) one graph of min(n, 10000) kernel nodes, replayed until n nodes ran
    const int64_t nodes = n < 10000 ? n : 10000, reps = (n + nodes - 1) / nodes;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { rc = SUNBW_ERR_CUDA; goto done; }
    for (int64_t i = 0; i < nodes; ++i) k_empty<<<1, 32, 0, s>>>();
    if (cudaStreamEndCapture(s, &g) != cudaSuccess || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess ||
        cudaGraphUpload(ge, s) != cudaSuccess || cudaGraphLaunch(ge, s) != cudaSuccess) {
      rc = SUNBW_ERR_CUDA;
      goto done;
    }
    cudaEventRecord(e0, s);
    for (int64_t r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) { rc = SUNBW_ERR_CUDA; goto done; }
    cudaEventElapsedTime(&ms, e0, e1);
    out3[1] = 1e3 * ms / (double)(reps * nodes);
  }
  {
    // (c) host round trip: launch + synchronise, mean over min(n, 2000)
    const int64_t m = n < 2000 ? n : 2000;
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < m; ++i) {
      k_empty<<<1, 32, 0, s>>>();
      cudaStreamSynchronize(s);
    }
    const auto t1 = std::chrono::steady_clock::now();
    out3[2] = std::chrono::duration<double, std::micro>(t1 - t0).count() / (double)m;
  }
  ctx->launches += n + 100;
done:
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (cudaGetLastError() != cudaSuccess && !rc) rc = SUNBW_ERR_CUDA;
  return rc ? ctx_set_err(ctx, rc) : 0;
}
