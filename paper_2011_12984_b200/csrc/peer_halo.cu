// peer_halo.cu — the advection halo (§7: "point-to-point communication
// is required for evaluating the explicit advection operator; ... this
// communication occurs directly between GPUs") as a copy-engine transfer
// into the right neighbour's memory, instead of NCCL send/recv kernels.
//
// Why: the fused step kernel is a persistent grid that fills every SM; an
// NCCL send/recv kernel enqueued beside it on a side stream cannot become
// resident until the interior launch drains, so the halo would sit on the
// critical path before the plane-0 launch.  A cudaMemcpyAsync between peer
// device buffers runs on a copy engine (over NVLink between GPUs, or inside
// one GPU for the in-process test ranks) and needs no SM.
//
// Protocol (one direction, c > 0 upwind: rank r sends its last plane to
// r+1), sequence number s = 1, 2, ... per exchange, slot s & 1 of the
// receiver's double-buffered halo:
//   sender, side stream:  wait  ack(own)        >= s - 2   (slot free)
//                         copy  last plane  ->  right.slot[s & 1]
//                         write right.arrived[s & 1] = s
//   receiver, main stream: wait arrived[s & 1]  >= s        (before plane 0)
//                          ... plane-0 tiles read slot[s & 1] ...
//                          write left.ack = s               (after plane 0)
// The waits and writes are stream memory operations (cuStreamWaitValue32 /
// cuStreamWriteValue32, resolved through cudaGetDriverEntryPoint), so the
// whole exchange is enqueued without host synchronisation.  The write after
// the copy carries the default memory barrier: the data is visible before
// the flag.
//
// Setup: every rank allocates [slot 0 | slot 1 | flags]; the neighbours'
// addresses come from the in-process fake communicator directly, or (one
// process per GPU) from CUDA IPC handles all-gathered over NCCL and opened
// with cudaIpcOpenMemHandle.

#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "sunbw_internal.h"

namespace {

using PfnWait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PfnWrite = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct MemOps {
  PfnWait wait = nullptr;
  PfnWrite write = nullptr;
  bool ok = false;
};

const MemOps& memops() {
  static const MemOps m = [] {
    MemOps r;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&r.wait, cudaEnableDefault, &q1) ==
            cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&r.write, cudaEnableDefault, &q2) ==
            cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess)
      r.ok = r.wait && r.write;
    return r;
  }();
  return m;
}

constexpr size_t kFlagBytes = 256;

}  // namespace

struct PeerHalo {
  size_t cap = 0;                      // doubles per slot
  double* local = nullptr;             // [slot0 | slot1 | flags]
  unsigned* flags = nullptr;           // local: [arrived0, arrived1, ack, pad]
  double* r_slots = nullptr;           // right neighbour's slots
  unsigned* r_flags = nullptr;         // right neighbour's flags (arrived)
  unsigned* l_flags = nullptr;         // left neighbour's flags (ack)
  void* ipc_r = nullptr;               // IPC mappings to close (multi-process)
  void* ipc_l = nullptr;
  uint32_t seq = 0;
  ~PeerHalo() {
    if (ipc_r) cudaIpcCloseMemHandle(ipc_r);
    if (ipc_l && ipc_l != ipc_r) cudaIpcCloseMemHandle(ipc_l);
    if (local) cudaFree(local);
  }
};

namespace sunbw {

bool peer_halo_supported() {
  const char* e = std::getenv("SUNBW_PEER_HALO");
  if (e && e[0] == '0') return false;
  return memops().ok;
}

PeerHalo* peer_halo_alloc(size_t cap, int* err) {
  auto* h = new PeerHalo();
  h->cap = cap;
  const size_t bytes = 2 * cap * sizeof(double) + kFlagBytes;
  if (cudaMalloc(&h->local, bytes) != cudaSuccess || cudaMemset(h->local, 0, bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    h->local = nullptr;
    delete h;
    *err = SUNBW_ERR_MEM;
    return nullptr;
  }
  h->flags = (unsigned*)(h->local + 2 * cap);
  *err = 0;
  return h;
}

void peer_halo_free(PeerHalo* h) { delete h; }

double* peer_halo_base(PeerHalo* h) { return h ? h->local : nullptr; }

// neighbours' [slots | flags] base addresses (already mapped into this process)
void peer_halo_connect(PeerHalo* h, double* right_base, double* left_base) {
  h->r_slots = right_base;
  h->r_flags = (unsigned*)(right_base + 2 * h->cap);
  h->l_flags = (unsigned*)(left_base + 2 * h->cap);
}

void peer_halo_set_ipc(PeerHalo* h, void* right_map, void* left_map) {
  h->ipc_r = right_map;
  h->ipc_l = left_map;
}

size_t peer_halo_capacity(const PeerHalo* h) { return h ? h->cap : 0; }

int peer_halo_send(PeerHalo* h, const double* send, size_t count, cudaStream_t side) {
  if (count > h->cap) return SUNBW_ERR_ARG;
  const MemOps& m = memops();
  const uint32_t s = ++h->seq, slot = s & 1;
  if (s > 2 && m.wait((CUstream)side, (CUdeviceptr)(h->flags + 2), s - 2, CU_STREAM_WAIT_VALUE_GEQ) !=
                   CUDA_SUCCESS)
    return SUNBW_ERR_CUDA;
  if (cudaMemcpyAsync(h->r_slots + slot * h->cap, send, count * sizeof(double), cudaMemcpyDeviceToDevice,
                      side) != cudaSuccess)
    return SUNBW_ERR_CUDA;
  if (m.write((CUstream)side, (CUdeviceptr)(h->r_flags + slot), s, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    return SUNBW_ERR_CUDA;
  return 0;
}

int peer_halo_wait(PeerHalo* h, cudaStream_t main, const double** recv) {
  const uint32_t s = h->seq, slot = s & 1;
  if (memops().wait((CUstream)main, (CUdeviceptr)(h->flags + slot), s, CU_STREAM_WAIT_VALUE_GEQ) !=
      CUDA_SUCCESS)
    return SUNBW_ERR_CUDA;
  *recv = h->local + slot * h->cap;
  return 0;
}

int peer_halo_release(PeerHalo* h, cudaStream_t main) {
  if (memops().write((CUstream)main, (CUdeviceptr)(h->l_flags + 2), h->seq, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    return SUNBW_ERR_CUDA;
  return 0;
}

}  // namespace sunbw
