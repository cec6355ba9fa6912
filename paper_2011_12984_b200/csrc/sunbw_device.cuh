// sunbw_device.cuh — device helpers shared by the libsunbw kernels:
// 256-bit global accesses and the head/vector/tail split of a range.
#pragma once

#include <stdint.h>

namespace sunbw {

constexpr int kU = 2;   // 32-B vectors in flight per operand per thread (streaming)

struct __align__(32) d4 {
  double v[4];
};

// 256-bit load (LDG.E.256 on sm_100a), not allocated in L1: streamed data
__device__ __forceinline__ d4 ld4(const double* p) {
  d4 r;
  asm("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
      : "l"(p));
  return r;
}

// 256-bit store (STG.E.256).  "memory" clobber: no load is moved past it,
// which keeps element-wise aliasing (z == x) correct.
__device__ __forceinline__ void st4(double* p, const d4& r) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]),
               "d"(r.v[2]), "d"(r.v[3])
               : "memory");
}

// [0,n) = scalar head | nvec 32-byte vectors | scalar tail.  The vector body
// is used only if every pointer has the same offset mod 32 B; otherwise the
// whole range is the scalar "head" (still coalesced, 8 B per lane).
struct Split {
  int64_t head, nvec, tail0;
};

inline Split split_for(int64_t n, const double* const* ptrs, int np) {
  Split s{n, 0, n};
  if (n <= 0 || np == 0) return {0, 0, 0};
  uintptr_t off = (uintptr_t)ptrs[0] & 31;
  for (int i = 1; i < np; ++i)
    if (((uintptr_t)ptrs[i] & 31) != off) return s;
  if (off & 7) return s;
  int64_t head = off ? (int64_t)((32 - off) / 8) : 0;
  if (head > n) head = n;
  int64_t nvec = (n - head) / 4;
  return {head, nvec, head + nvec * 4};
}

}  // namespace sunbw
