// Memory-side ceiling of the fused step's data movement, without its
// arithmetic (diagnostic for DESIGN §11): the same persistent grid (740 CTAs
// x 128 threads), 128-cell AoS tiles moved by bulk copies into a 2-stage
// mbarrier ring and out by bulk stores from double-buffered shared tiles.
//   mode 0: y_n + H_n in, y_{n+1} + H_{n+1} out          (4 streams, 96 B/cell)
//   mode 1: mode 0 + the row-below and plane-below tiles  (the fused step's pattern)
//   mode 2: mode 1 with a dependent fp64 chain of `chain` ops per cell
//   mode 3: mode 1 in the packed working layout [y | H] per tile: one 6 KB
//           bulk load + the two neighbour y tiles, one 6 KB bulk store
//           (3 address streams instead of 5)
//   mode 4: mode 3 without the neighbour tiles (2 streams)
//   mode 5: mode 1 with L2 cache hints: the own y tile evict_last (it is read
//           again as a neighbour), neighbour tiles evict_first (last use),
//           H and both stores evict_first
// Prints us per launch and algorithmic GB/s (96 B/cell) per mode.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kCells = 128, kTile = kCells * 3;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
               "l"(s), "r"(n), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void g2s_h(void* d, const void* s, uint32_t n, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sa(d)),
      "l"(s), "r"(n), "r"(sa(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void s2g_h(void* d, const void* s, uint32_t n, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(d), "r"(sa(s)),
               "r"(n), "l"(pol) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sa(s)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

struct __align__(128) Smem {
  double in[2][4][kTile];
  double out[2][2][kTile];
  uint64_t full[2];
};

__global__ void __launch_bounds__(kCells, 5) k_tiles(const double* y, const double* h, double* z, double* ho,
                                                      int64_t ntiles, int64_t row_tiles, int64_t plane_tiles,
                                                      int mode, int chain) {
  extern __shared__ __align__(128) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x;
  const bool packed = mode == 3 || mode == 4;
  const bool hints = mode == 5;
  const uint64_t PL = pol_last(), PF = pol_first();
  auto issue = [&](int64_t tile, int st) {
    const bool nb = mode >= 1 && mode != 4;
    if (packed) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&S.full[st])),
                   "r"((nb ? 4 : 2) * kTile * 8) : "memory");
      g2s(S.in[st][0], y + tile * 2 * kTile, 2 * kTile * 8, &S.full[st]);
      if (nb) {
        const int64_t ym = tile >= row_tiles ? tile - row_tiles : tile;
        const int64_t zm = tile >= plane_tiles ? tile - plane_tiles : tile + ntiles - plane_tiles;
        g2s(S.in[st][2], y + ym * 2 * kTile, kTile * 8, &S.full[st]);
        g2s(S.in[st][3], y + zm * 2 * kTile, kTile * 8, &S.full[st]);
      }
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&S.full[st])),
                 "r"((nb ? 4 : 2) * kTile * 8) : "memory");
    if (hints) {
      const int64_t ym = tile >= row_tiles ? tile - row_tiles : tile;
      const int64_t zm = tile >= plane_tiles ? tile - plane_tiles : tile + ntiles - plane_tiles;
      g2s_h(S.in[st][0], y + tile * kTile, kTile * 8, &S.full[st], PL);
      g2s_h(S.in[st][1], h + tile * kTile, kTile * 8, &S.full[st], PF);
      g2s_h(S.in[st][2], y + ym * kTile, kTile * 8, &S.full[st], PL);
      g2s_h(S.in[st][3], y + zm * kTile, kTile * 8, &S.full[st], PF);
      return;
    }
    g2s(S.in[st][0], y + tile * kTile, kTile * 8, &S.full[st]);
    g2s(S.in[st][1], h + tile * kTile, kTile * 8, &S.full[st]);
    if (nb) {
      const int64_t ym = tile >= row_tiles ? tile - row_tiles : tile;
      const int64_t zm = tile >= plane_tiles ? tile - plane_tiles : tile + ntiles - plane_tiles;
      g2s(S.in[st][2], y + ym * kTile, kTile * 8, &S.full[st]);
      g2s(S.in[st][3], y + zm * kTile, kTile * 8, &S.full[st]);
    }
  };
  if (t == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&S.full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int s = 0; s < 2; ++s)
      if (blockIdx.x + s * (int64_t)gridDim.x < ntiles) issue(blockIdx.x + s * (int64_t)gridDim.x, s);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
                     sa(&S.full[st])), "r"((uint32_t)((it >> 1) & 1)) : "memory");
    const int ob = it & 1;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      double a = S.in[st][0][3 * t + s], b = S.in[st][1][3 * t + s];
      if (mode >= 1 && mode != 4) a = __dadd_rn(a, __dadd_rn(S.in[st][2][3 * t + s], S.in[st][3][3 * t + s]));
      if (mode == 2)
        for (int c = 0; c < chain; ++c) a = __fma_rn(a, 0.999999, b);
      S.out[ob][0][3 * t + s] = a;
      S.out[ob][1][3 * t + s] = b;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      if (packed) {
        s2g(z + tile * 2 * kTile, S.out[ob][0], 2 * kTile * 8);
      } else if (hints) {
        s2g_h(z + tile * kTile, S.out[ob][0], kTile * 8, PF);
        s2g_h(ho + tile * kTile, S.out[ob][1], kTile * 8, PF);
      } else {
        s2g(z + tile * kTile, S.out[ob][0], kTile * 8);
        s2g(ho + tile * kTile, S.out[ob][1], kTile * 8);
      }
      const int64_t nx = tile + 2 * (int64_t)gridDim.x;
      if (nx < ntiles) issue(nx, st);
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// mode 6: the SBDF2 step without the history vector — y_n and y_{n-1} each
// with their row-below and plane-below tiles in (the history term is
// recomputed from y_{n-1} and its stencil), y_{n+1} out (3 streams + 4
// neighbour tiles, 72 B/cell algorithmic); chain > 0 adds the dependent
// DFMA chains of mode 2.  L2 hints as in mode 5.
struct __align__(128) Smem6 {
  double in[2][6][kTile];
  double xm[2][2][8];
  double out[2][kTile];
  uint64_t full[2];
};
__global__ void __launch_bounds__(kCells, 5) k_tiles6(const double* y, const double* yp, double* z, int64_t ntiles,
                                                       int64_t row_tiles, int64_t plane_tiles, int chain) {
  extern __shared__ __align__(128) unsigned char raw[];
  Smem6& S = *reinterpret_cast<Smem6*>(raw);
  const int t = threadIdx.x;
  const uint64_t PL = pol_last(), PF = pol_first();
  auto issue = [&](int64_t tile, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&S.full[st])),
                 "r"(6 * kTile * 8 + 2 * 48) : "memory");
    const int64_t ym = tile >= row_tiles ? tile - row_tiles : tile;
    const int64_t zm = tile >= plane_tiles ? tile - plane_tiles : tile + ntiles - plane_tiles;
    const int64_t xp = tile > 0 ? tile * kTile - 6 : 0;
    g2s_h(S.in[st][0], y + tile * kTile, kTile * 8, &S.full[st], PL);
    g2s_h(S.in[st][1], y + ym * kTile, kTile * 8, &S.full[st], PL);
    g2s_h(S.in[st][2], y + zm * kTile, kTile * 8, &S.full[st], PF);
    g2s(S.xm[st][0], y + xp, 48, &S.full[st]);
    g2s_h(S.in[st][3], yp + tile * kTile, kTile * 8, &S.full[st], PL);
    g2s_h(S.in[st][4], yp + ym * kTile, kTile * 8, &S.full[st], PL);
    g2s_h(S.in[st][5], yp + zm * kTile, kTile * 8, &S.full[st], PF);
    g2s(S.xm[st][1], yp + xp, 48, &S.full[st]);
  };
  if (t == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&S.full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0)
    for (int s = 0; s < 2; ++s)
      if (blockIdx.x + s * (int64_t)gridDim.x < ntiles) issue(blockIdx.x + s * (int64_t)gridDim.x, s);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
                     sa(&S.full[st])), "r"((uint32_t)((it >> 1) & 1)) : "memory");
    const int ob = it & 1;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      double a = __dadd_rn(S.in[st][0][3 * t + s], __dadd_rn(S.in[st][1][3 * t + s], S.in[st][2][3 * t + s]));
      double b = __dadd_rn(S.in[st][3][3 * t + s], __dadd_rn(S.in[st][4][3 * t + s], S.in[st][5][3 * t + s]));
      a = __dadd_rn(a, t > 0 ? S.in[st][0][3 * (t - 1) + s] : S.xm[st][0][3 + s]);
      b = __dadd_rn(b, t > 0 ? S.in[st][3][3 * (t - 1) + s] : S.xm[st][1][3 + s]);
      for (int c = 0; c < chain; ++c) a = __fma_rn(a, 0.999999, b);
      S.out[ob][3 * t + s] = __dadd_rn(a, b);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      s2g_h(z + tile * kTile, S.out[ob], kTile * 8, PF);
      const int64_t nx = tile + 2 * (int64_t)gridDim.x;
      if (nx < ntiles) issue(nx, st);
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int64_t n = 256, G = n * n * n, ntiles = G / kCells;
  double *y, *h, *z, *ho;
  const size_t bytes = (size_t)G * 3 * 8;
  // packed modes use y and z as [y | H] arrays of 2x the size
  cudaMalloc(&y, 2 * bytes); cudaMalloc(&h, bytes); cudaMalloc(&z, 2 * bytes); cudaMalloc(&ho, bytes);
  cudaMemset(y, 0, 2 * bytes); cudaMemset(h, 0, bytes);
  const int smem = sizeof(Smem);
  cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 5;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int only = argc > 1 ? atoi(argv[1]) : -1;
  struct { int mode, chain; } cases[] = {{0, 0}, {1, 0}, {3, 0}, {4, 0}, {5, 0}, {1, 0}, {5, 0}, {2, 32}, {2, 64}};
  for (auto c : cases) {
    if (only >= 0 && c.mode != only) continue;
    for (int w = 0; w < 3; ++w)
      k_tiles<<<grid, kCells, smem>>>(y, h, z, ho, ntiles, 2, 512, c.mode, c.chain);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r)
      k_tiles<<<grid, kCells, smem>>>((r & 1) ? z : y, (r & 1) ? ho : h, (r & 1) ? y : z, (r & 1) ? h : ho, ntiles,
                                      2, 512, c.mode, c.chain);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("mode %d chain %3d (3 chains/thread): %7.1f us/launch  %6.0f GB/s algorithmic (96 B/cell)  err=%s\n",
           c.mode, c.chain, us, 96.0 * G / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  {
    const int smem6 = sizeof(Smem6);
    cudaFuncSetAttribute(k_tiles6, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
    for (int chain : {0, 32}) {
      if (only >= 0 && only != 6) break;
      for (int w = 0; w < 3; ++w) k_tiles6<<<grid, kCells, smem6>>>(y, h, z, ntiles, 2, 512, chain);
      cudaEventRecord(e0);
      const int reps = 20;
      // rotation y_{n-1} <- y_n <- y_{n+1} over three buffers
      double* buf[3] = {h, y, z};
      for (int r = 0; r < reps; ++r)
        k_tiles6<<<grid, kCells, smem6>>>(buf[(r + 1) % 3], buf[r % 3], buf[(r + 2) % 3], ntiles, 2, 512, chain);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("mode 6 chain %3d (no history vector): %7.1f us/launch  %6.0f GB/s algorithmic (72 B/cell)  "
             "err=%s\n", chain, us, 72.0 * G / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
