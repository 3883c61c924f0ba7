// common.cuh -- shared device helpers of libbnn (CUDA path only; never included by the oracle).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define BNN_DEV __device__ __forceinline__
#define BNN_FULL_MASK 0xffffffffu

namespace bnn {

constexpr int kWarp = 32;

// Eq. (2) bit placement with B = 32 (R2): element j of a 32-group lands on bit 31 - j.
// __ballot_sync puts lane j on bit j, so the packed word of 32 lane-bits is brev(ballot).
BNN_DEV uint32_t ballot_pack(bool bit) { return __brev(__ballot_sync(BNN_FULL_MASK, bit)); }

BNN_DEV int popc(uint32_t v) { return __popc(v); }

// u8 x s8 4-way dot product (IDP4A.U8.S8): a holds 4 unsigned bytes, b 4 signed bytes.
BNN_DEV int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Division by a runtime-invariant divisor d (1 <= d < 2^31) for numerators n < 2^31, as a
// multiply-high + add + shift (Granlund-Montgomery): l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1, q = (umulhi(m, n) + n) >> l.  Built on the host (launch arguments) or once
// per thread (luma_band_kernel).
struct FastDiv {
  uint32_t d, m, l;
  __host__ __device__ FastDiv() : d(1), m(1), l(0) {}
  __host__ __device__ explicit FastDiv(uint32_t div) : d(div) {
    l = 0;
    while ((1ull << l) < div) ++l;
    m = (uint32_t)((((1ull << l) - div) << 32) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(m, n) + n) >> l; }
};

// For u8 x: (x > t) <=> (x > u8_threshold(t)) exactly (R14): x integer, so x > t <=> x > floor(t);
// clamped to [-1, 255]; NaN t (never true) -> 255.
BNN_DEV int u8_threshold(float t) {
  if (!(t == t)) return 255;
  if (t < -1.0f) return -1;
  if (t >= 255.0f) return 255;
  return (int)floorf(t);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-serialization
// attribute may start while its predecessor runs; every thread calls griddep_wait() before touching
// memory the predecessor writes or reads (activations), griddep_launch() lets the successor start
// its prologue early.  Both are no-ops for kernels launched without the attribute.
BNN_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
BNN_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

BNN_DEV int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
BNN_DEV int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

}  // namespace bnn
