// Shared device definitions for the B200 hot path (sm_100a, fp64 CUDA cores).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/uc_b200.h"

namespace uc {

// ---------------------------------------------------------------------------
// 3-point Gauss-Legendre rule, bit-identical to numpy's leggauss(3) as used by
// undercool/mesh.py:52-61.  Note w0 = 0.5555555555555557 (not 5/9).
// L0[q] = (1 - x_q)/2 and L1[q] = (1 + x_q)/2 are the Q1 basis values at the
// points (mesh.py:63-79), also (x_q + 1)/2 for the Gauss coordinates
// (mesh.py:119-128).
// ---------------------------------------------------------------------------
#define UC_GW0 0x1.1c71c71c71c73p-1
#define UC_GW1 0x1.c71c71c71c71cp-1
#define UC_LA 0x1.c64bf7a1fb924p-1
#define UC_LB 0x1.cda042f0236e0p-4

__host__ __device__ __forceinline__ constexpr double gw(int q) { return q == 1 ? UC_GW1 : UC_GW0; }
// value of the 1D Q1 basis j (0 or 1) at Gauss point q (0..2)
__host__ __device__ __forceinline__ constexpr double lq(int j, int q) {
  return j == 0 ? (q == 0 ? UC_LA : (q == 1 ? 0.5 : UC_LB))
                : (q == 0 ? UC_LB : (q == 1 ? 0.5 : UC_LA));
}
// sign of the 1D Q1 basis derivative (times 1/h)
__host__ __device__ __forceinline__ constexpr double dsg(int j) { return j == 0 ? -1.0 : 1.0; }

// sqrt(machine eps) of newton.py:26
#define UC_EPS0 0x1.0000000000000p-26

// ---------------------------------------------------------------------------
// Grid (structured Q1 mesh, x fastest) with an owned slab of node planes
// along the slowest axis.
// ---------------------------------------------------------------------------
struct Grid {
  int dim;
  int64_t nn[3];   // nodes per axis (nn[2] = 1 in 2D)
  int64_t ne[3];   // elements per axis (ne[2] = 1 in 2D)
  int64_t plane;   // nodes per plane orthogonal to the slow axis
  int64_t nslow;   // nodes along the slow axis
  int64_t eslow;   // elements along the slow axis
  int64_t lo, hi;  // owned node planes [lo, hi)
  int64_t nloc;    // owned nodes per field = (hi - lo) * plane
  double h[3];     // spacing
  double ih[3];    // 1/h as the reference's 0.5*(2/h)
};

// Division by a run-time constant via multiply-high (CUTLASS FastDivmod
// scheme): n / d == umulhi(n, m) >> s for 0 <= n < 2^31.
struct FastDiv {
  uint32_t d, m, s;
  static FastDiv make(uint32_t d) {
    FastDiv f{d, 0u, 0u};
    if (d <= 1) return f;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    const uint64_t p = 31 + l;
    f.m = (uint32_t)(((1ull << p) + d - 1) / d);
    f.s = (uint32_t)(p - 32);
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return d <= 1 ? n : (__umulhi(n, m) >> s);
  }
};

// Field view: owned block-ordered array plus optional ghost planes.
struct FieldView {
  const double* owned;   // [2][nloc]
  const double* glo;     // [2][plane] plane lo-1 (NULL on a single GPU)
  const double* ghi;     // [2][plane] plane hi
};

__device__ __forceinline__ double fetch(const FieldView& v, const Grid& g, int f, int64_t p,
                                        int64_t lat) {
  if (p < g.lo) return v.glo[f * g.plane + lat];
  if (p >= g.hi) return v.ghi[f * g.plane + lat];
  return v.owned[f * g.nloc + (p - g.lo) * g.plane + lat];
}

#define UC_CUDA_OK(expr)                                                     \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return ::uc::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
  } while (0)

int set_cuda_error(cudaError_t e, const char* what, const char* file, int line);
int set_error(int code, const char* fmt, ...);

// numpy-faithful two-rounding elementwise ops (no FMA contraction)
__device__ __forceinline__ double axpy_rn(double a, double s, double b) {
  return __dadd_rn(a, __dmul_rn(s, b));
}

// TMA bulk copies (cp.async.bulk) completing on a shared-memory mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  for (unsigned spin = 0; !done; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
    if (spin > (1u << 26)) __trap();  // a copy that never completes (a fault): fail, do not hang
  }
}

}  // namespace uc
