// pipeline.cuh — TMA bulk-copy tile pipeline for per-cell (per-block) maps.
//
// The AoS arrays of the hot path (3-double cell states, 9-double 3×3
// blocks, int32 pivot codes) are contiguous per tile of T cells, so each
// operand tile is ONE bulk copy (cp.async.bulk, the TMA engine; 16-B aligned,
// size a multiple of 16 B).  A persistent CTA of T threads walks its tiles
// with a STAGES-deep shared-memory ring: the producer thread (thread 0)
// issues the next tiles' copies, an mbarrier per stage counts the arriving
// bytes, the T threads compute one cell each from shared memory, write the
// results to an output tile and thread 0 sends it back with a bulk
// shared→global copy.  A ragged last tile is handled with plain loads.
#pragma once

#include <stdint.h>

namespace sunbw {
namespace pipe {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// The same copies with an L2 eviction-priority hint (createpolicy): data
// read again soon by another tile (evict_last), or at its last use / never
// read again in this launch (evict_first).
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Operand description: global base and bytes per cell.  All bases must be
// 16-B aligned and T * bytes_per_cell a multiple of 16.
template <int NIN, int NOUT>
struct IO {
  const unsigned char* in[NIN];
  int in_bpc[NIN];
  unsigned char* out[NOUT];
  int out_bpc[NOUT];
};

template <int NIN, int NOUT>
__host__ __device__ constexpr int smem_bytes(int T, int stages, const int (&in_bpc)[NIN],
                                             const int (&out_bpc)[NOUT]) {
  int s = 0;
  for (int i = 0; i < NIN; ++i) s += in_bpc[i];
  int o = 0;
  for (int i = 0; i < NOUT; ++i) o += out_bpc[i];
  return 128 + T * (stages * s + o);
}

// Runs body(t, cell, in_ptrs, out_ptrs) for every cell, where in_ptrs[i] /
// out_ptrs[i] point at the cell's bytes (in shared memory for full tiles,
// in global memory for the ragged tail).  Dynamic shared memory layout:
// [mbarriers | stage 0 inputs | ... | outputs].
template <int T, int STAGES, int NIN, int NOUT, class Body>
__device__ __forceinline__ void run(const IO<NIN, NOUT>& io, int64_t n, unsigned char* smem, Body body) {
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  unsigned char* base = smem + 128;
  int in_tile = 0, out_tile = 0;
  int in_off[NIN], out_off[NOUT];
#pragma unroll
  for (int i = 0; i < NIN; ++i) { in_off[i] = in_tile; in_tile += T * io.in_bpc[i]; }
#pragma unroll
  for (int i = 0; i < NOUT; ++i) { out_off[i] = out_tile; out_tile += T * io.out_bpc[i]; }
  unsigned char* outbuf = base + STAGES * in_tile;
  const int t = threadIdx.x;
  const int64_t full_tiles = n / T;

  auto issue = [&](int64_t tile, int stage) {
    mbar_expect_tx(&full[stage], (uint32_t)in_tile);
#pragma unroll
    for (int i = 0; i < NIN; ++i)
      bulk_g2s(base + stage * in_tile + in_off[i], io.in[i] + tile * T * io.in_bpc[i],
               (uint32_t)(T * io.in_bpc[i]), &full[stage]);
  };
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0)
    for (int s = 0; s < STAGES; ++s) {
      int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < full_tiles) issue(tile, s);
    }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < full_tiles; tile += gridDim.x, ++it) {
    const int stage = it % STAGES;
    mbar_wait(&full[stage], (uint32_t)((it / STAGES) & 1));
    if (t == 0) bulk_wait_read_all();          // previous output tile has left smem
    __syncthreads();
    const unsigned char* ip[NIN];
    unsigned char* op[NOUT];
#pragma unroll
    for (int i = 0; i < NIN; ++i) ip[i] = base + stage * in_tile + in_off[i] + t * io.in_bpc[i];
#pragma unroll
    for (int i = 0; i < NOUT; ++i) op[i] = outbuf + out_off[i] + t * io.out_bpc[i];
    body(t, tile * T + t, ip, op);
    fence_async_smem();
    __syncthreads();                           // stage read, outputs written
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < NOUT; ++i)
        bulk_s2g(io.out[i] + tile * T * io.out_bpc[i], outbuf + out_off[i], (uint32_t)(T * io.out_bpc[i]));
      bulk_commit();
      int64_t next = tile + (int64_t)STAGES * gridDim.x;
      if (next < full_tiles) issue(next, stage);
    }
  }
  if (t == 0) bulk_wait_all();
  // ragged tail: plain global accesses, by the CTA that would own the tile
  const int64_t tail0 = full_tiles * T;
  if (tail0 < n && blockIdx.x == (int)(full_tiles % gridDim.x)) {
    const int64_t c = tail0 + t;
    if (c < n) {
      const unsigned char* ip[NIN];
      unsigned char* op[NOUT];
#pragma unroll
      for (int i = 0; i < NIN; ++i) ip[i] = io.in[i] + c * io.in_bpc[i];
#pragma unroll
      for (int i = 0; i < NOUT; ++i) op[i] = io.out[i] + c * io.out_bpc[i];
      body(t, c, ip, op);
    }
  }
}

}  // namespace pipe
}  // namespace sunbw
