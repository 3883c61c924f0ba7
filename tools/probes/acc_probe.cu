// Accumulation-precision probe for tcgen05.mma kind::mxf4 on sm_100a: is D = C + A.B exact when the fp32
// accumulator C is large (C0 = 1.5 * 2^e) and the products are small integers?  (If the tensor core kept
// only ~14 significant bits when it aligns the products to the accumulator, the low bits would be lost.)
// A: e2m1 {0, 1.0} (0x0 / 0x2), B: e2m1 {+-2, +-6, +-4, +-1, 0} -- the conv1 operand values.  C is written
// with tcgen05.st, then `reps` MMAs accumulate onto it (accumulate = 1 from the first); D must equal
// C0 + reps * (exact integer dot product) bit for bit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o acc_probe acc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase));
}

constexpr int M = 128, N = 128, KB = 32;
__global__ void __launch_bounds__(128) k_acc(const uint8_t* A, const uint8_t* B, float c0, int reps, float* D) {
  __shared__ __align__(1024) uint8_t sA[M * KB];
  __shared__ __align__(1024) uint8_t sB[N * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * KB; i += 128) {
    const int r = i / KB, b = i % KB, c = b / 16, o = b % 16;
    sA[c * (M / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + o] = A[i];
  }
  for (int i = tid; i < N * KB; i += 128) {
    const int r = i / KB, b = i % KB, c = b / 16, o = b % 16;
    sB[c * (N / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + o] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase, lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t sfa = tmem + N, sfb = tmem + N + 8;
  {
    const uint32_t v = 0x7F7F7F7Fu, c = __float_as_uint(c0);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfa + lane_off), "r"(v));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfb + lane_off), "r"(v));
    for (int c8 = 0; c8 < N; c8 += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tmem + lane_off + c8), "r"(c));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint64_t ad = make_desc(smem_u32(sA), M / 8 * 128, 128), bd = make_desc(smem_u32(sB), N / 8 * 128, 128);
    for (int r = 0; r < reps; ++r)
      asm volatile(
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], 1;\n\t" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc_mxf4(M, N)), "r"(sfa), "r"(sfb));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c8 = 0; c8 < N; c8 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + lane_off + c8));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[(warp * 32 + (tid & 31)) * N + c8 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

static int val(uint8_t c) {
  const int mag[8] = {0, 1, 2, 3, 4, 6, 8, 12};  // e2m1 x 2 (codes: 0, 0.5, 1, 1.5, 2, 3, 4, 6)
  return ((c & 8) ? -1 : 1) * mag[c & 7];        // in units of 0.5
}

int main() {
  const int K = 64;
  const uint8_t bvals[9] = {0x4, 0xC, 0x7, 0xF, 0x6, 0xE, 0x2, 0xA, 0x0};  // +-2, +-6, +-4, +-1, 0
  int first_bad_e = 99;  // smallest C0 exponent with an inexact result (any trial)
  for (int trial = 0; trial < 3; ++trial) {
    std::vector<uint8_t> ca(M * K), cb(N * K), hA(M * 32), hB(N * 32);
    srand(100 + trial);
    for (auto& v : ca) v = (rand() & 1) ? 0x2 : 0x0;
    for (auto& v : cb) v = bvals[rand() % (trial == 0 ? 2 : 9)];
    for (int r = 0; r < M; ++r)
      for (int b = 0; b < 32; ++b) hA[r * 32 + b] = ca[r * K + 2 * b] | (ca[r * K + 2 * b + 1] << 4);
    for (int r = 0; r < N; ++r)
      for (int b = 0; b < 32; ++b) hB[r * 32 + b] = cb[r * K + 2 * b] | (cb[r * K + 2 * b + 1] << 4);
    uint8_t *dA, *dB;
    float* dD;
    cudaMalloc(&dA, M * 32); cudaMalloc(&dB, N * 32); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA.data(), M * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * 32, cudaMemcpyHostToDevice);
    for (int e = 0; e <= 24; e += (e < 14 ? 7 : 1)) {
      for (int sgn = 1; sgn >= -1; sgn -= 2) {
        const float c0 = e == 0 ? 0.0f : sgn * 1.5f * (float)(1 << e);
        for (int reps : {1, 3}) {
          k_acc<<<1, 128>>>(dA, dB, c0, reps, dD);
          if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
          std::vector<float> hD(M * N);
          cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
          long long bad = 0, maxdev = 0;
          for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
              long long s2 = 0;  // exact sum in units of 0.25 (0.5 x 0.5)
              for (int k = 0; k < K; ++k) s2 += (long long)val(ca[m * K + k]) * val(cb[n * K + k]);
              const double want = (double)c0 + reps * s2 / 4.0;  // exact in double
              const double got = hD[m * N + n];
              if (got != want) {
                ++bad;
                long long dev = (long long)((got - want) * 4);
                if (dev < 0) dev = -dev;
                if (dev > maxdev) maxdev = dev;
              }
            }
          // representable? the exact result needs |c0| + ... within fp32's 24-bit mantissa at ulp <= 0.25 / 1
          printf("trial %d  C0 = %+.0f (1.5 * 2^%d)  reps %d: %s (%lld of %d differ, max |dev| %lld quarter-units)\n", trial,
                 c0, e, reps, bad ? "INEXACT" : "exact", bad, M * N, maxdev);
          if (bad && e < first_bad_e) first_bad_e = e;
        }
      }
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
  }
  if (first_bad_e == 99) printf("exact for every tested C0 (up to 1.5*2^24)\n");
  else printf("exact for every C0 up to 1.5*2^%d; first inexact results at 1.5*2^%d\n", first_bad_e - 1, first_bad_e);
  return 0;
}
