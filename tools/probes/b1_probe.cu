// mma.sync .b1 probe for sm_100a (B200): the north_star's "optional mma.sync .b1 XOR-popc variant,
// kept only if it assembles for sm_100a and beats the integer-pipe kernel".
//
// ptxas accepts mma.sync.m16n8k256 / m8n8k128 .b1 (.xor.popc and .and.popc) for sm_100a but lowers
// them to bit-plane splits (LOP3) + MOVM.U4TO8 + legacy IMMA.16832.U8.U8 (cuobjdump -sass).
// This measures what that costs, chip-wide, against the literal Eq. (4) mix on the integer pipe:
//   BMMA_XOR  : d = popc(a ^ b) summed, m16n8k256, 4 independent accumulator chains per warp
//   BMMA_AND  : the same with .and.popc (XOR = 2 AND emulations on sm_90; here both are emulated)
//   BMMA_M8   : m8n8k128 .xor.popc
//   XPA       : acc += popc(x ^ w) on 32-bit words (LOP3 + POPC + IADD), 8 chains per thread
// and checks one m16n8k256 xor.popc fragment against a CPU popcount (fragment layouts of the PTX ISA:
// A row-major 16x256 bits = 4 x b32 per thread, B col-major 256x8 bits = 2 x b32, C/D 16x8 s32 = 4).
// Rates are binary MACs per second (one MAC = one bit position of one output element).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o b1_probe b1_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

__device__ __forceinline__ void bmma_xor(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void bmma_and(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void bmma_m8(int (&d)[2], uint32_t a, uint32_t b) {
  asm volatile("mma.sync.aligned.m8n8k128.row.col.s32.b1.b1.s32.xor.popc {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+r"(d[0]), "+r"(d[1])
               : "r"(a), "r"(b));
}

template <int MODE>
__global__ void k_bmma(int* out, uint32_t seed) {
  uint32_t a[4][4], b[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int i = 0; i < 4; ++i) a[c][i] = seed * (threadIdx.x + 7 * i + 1) + c;
    b[c][0] = seed ^ (threadIdx.x * 0x9E3779B9u + c);
    b[c][1] = ~b[c][0] + c;
  }
  int d[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // new operand bits every iteration (as from shared memory in a conv), so the compiler cannot hoist
      // the bit-plane split / MOVM expansion out of the loop
#pragma unroll
      for (int i = 0; i < 4; ++i) a[c][i] += 0x01010101u;
      b[c][0] += 0x00010001u;
      b[c][1] ^= a[c][0];
      if (MODE == 0) bmma_xor(d[c], a[c], b[c]);
      else if (MODE == 1) bmma_and(d[c], a[c], b[c]);
      else {
        int e[2] = {d[c][0], d[c][1]};
        bmma_m8(e, a[c][0], b[c][0]);
        d[c][0] = e[0];
        d[c][1] = e[1];
      }
    }
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_xpa(int* out, uint32_t seed) {
  uint32_t x[8], w = seed ^ threadIdx.x;
  int acc[8] = {};
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] += __popc(x[i] ^ w);
      x[i] += 0x01010101u;  // keep the chains live (IADD; same count as the real loop's address math)
    }
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one m16n8k256 xor.popc on known fragments (C = 0) for the correctness check
__global__ void k_check(const uint32_t* A, const uint32_t* B, int* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  // A 16 x 256 bits row-major as 16 rows x 8 words; fragment a0..a3 = (row g, k-word t), (row g+8, t),
  // (row g, t+4), (row g+8, t+4); B 256 x 8 bits col-major as 8 cols x 8 words: b0 = (col g, word t),
  // b1 = (col g, word t+4); D 16 x 8: d0,d1 = (row g, cols 2t, 2t+1), d2,d3 = (row g+8, ...)
  uint32_t a[4] = {A[g * 8 + t], A[(g + 8) * 8 + t], A[g * 8 + t + 4], A[(g + 8) * 8 + t + 4]};
  uint32_t b[2] = {B[g * 8 + t], B[g * 8 + t + 4]};
  int d[4] = {0, 0, 0, 0};
  bmma_xor(d, a, b);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s  SMs=%d  cc=%d.%d  max clock %d MHz\n", p.name, p.multiProcessorCount, p.major, p.minor,
         clk_khz / 1000);
  const int sms = p.multiProcessorCount, threads = 256, blocks = sms * 8;
  int* out;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(int));

  // correctness of one fragment
  uint32_t hA[128], hB[64];
  uint32_t s = 12345;
  for (int i = 0; i < 128; ++i) hA[i] = (s = s * 1664525u + 1013904223u);
  for (int i = 0; i < 64; ++i) hB[i] = (s = s * 1664525u + 1013904223u);
  uint32_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, 128 * sizeof(int));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k_check<<<1, 32>>>(dA, dB, dD);
  int hD[128];
  cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 8; ++c) {
      int ref = 0;
      for (int w = 0; w < 8; ++w) ref += __builtin_popcount(hA[r * 8 + w] ^ hB[c * 8 + w]);
      bad += ref != hD[r * 8 + c];
    }
  printf("m16n8k256 xor.popc fragment check: %s (%d of 128 wrong)\n", bad ? "FAIL" : "exact", bad);

  const double macs_warp_iter[3] = {4.0 * 16 * 8 * 256, 4.0 * 16 * 8 * 256, 4.0 * 8 * 8 * 128};
  const char* names[3] = {"BMMA m16n8k256 xor.popc", "BMMA m16n8k256 and.popc", "BMMA m8n8k128 xor.popc"};
  for (int m = 0; m < 3; ++m) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k_bmma<0><<<blocks, threads>>>(out, 7);
      else if (m == 1) k_bmma<1><<<blocks, threads>>>(out, 7);
      else k_bmma<2><<<blocks, threads>>>(out, 7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    const double macs = macs_warp_iter[m] * ITERS * blocks * (threads / 32);
    printf("%-26s %8.3f ms  %8.2f T binary-MAC/s\n", names[m], t, macs / (t * 1e-3) / 1e12);
  }
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_xpa<<<blocks, threads>>>(out, 7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    const double macs = 32.0 * 8 * ITERS * (double)blocks * threads;
    printf("%-26s %8.3f ms  %8.2f T binary-MAC/s\n", "XOR+POPC+IADD (int pipe)", t, macs / (t * 1e-3) / 1e12);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
