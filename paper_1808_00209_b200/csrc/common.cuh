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

BNN_DEV int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
BNN_DEV int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

}  // namespace bnn
