// fp64 dependent-chain latency and throughput on B200 (diagnostic for the
// fused Newton kernel's latency-bound profile).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, double a, double b, int n, long long* cyc, int op) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  if (op == 0) {
    for (int i = 0; i < n; ++i) x = __fma_rn(x, a, b);
  } else if (op == 1) {
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  } else if (op == 2) {
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
  } else if (op == 3) {
    for (int i = 0; i < n; ++i) x = __drcp_rn(x);
  } else {
    for (int i = 0; i < n; ++i) x = __ddiv_rn(b, x);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 1024 * sizeof(double)); cudaMalloc(&c, sizeof(long long));
  double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0 + i * 1e-6;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[] = {"DFMA", "DADD", "DMUL", "drcp_rn", "ddiv_rn"};
  for (int op = 0; op < 5; ++op) {
    for (int threads : {32, 1024}) {
      int n = 4096;
      chain<<<1, threads>>>(d, 0.999999, 1e-7, n, c, op);
      cudaDeviceSynchronize();
      chain<<<1, threads>>>(d, 0.999999, 1e-7, n, c, op);
      long long cyc; cudaMemcpy(&cyc, c, sizeof(cyc), cudaMemcpyDeviceToHost);
      printf("%-8s threads=%4d  %.2f cycles per dependent op (per warp)\n", names[op], threads, (double)cyc / n);
    }
  }
  return 0;
}
