// tcgen05.mma kind::i8 probe for sm_100a: (1) correctness of a hand-built SWIZZLE_NONE K-major
// smem descriptor + instruction descriptor against a CPU GEMM, (2) cycles per MMA for
// M = 128, N in {32, 64, 128, 256}, K = 32 (int8), both operands in shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SWIZZLE_NONE K-major canonical layout ((8,m),2):((16B,SBO),LBO)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
  return (2u << 4)                 // c_format = S32
       | (1u << 7)                 // a_format = signed 8
       | (1u << 10)                // b_format = signed 8
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

template <int N>
__global__ void __launch_bounds__(128) k_umma(const int8_t* A, const int8_t* B, int32_t* D, int reps,
                                              long long* cycles) {
  constexpr int M = 128, K = 32;
  __shared__ __align__(1024) int8_t sA[M * K];
  __shared__ __align__(1024) int8_t sB[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical layout: element (r, k) at (k/16)*LBO + (r/8)*SBO + (r%8)*16 + k%16
  const uint32_t A_SBO = 128, A_LBO = (M / 8) * 128;
  const uint32_t B_SBO = 128, B_LBO = (N / 8) * 128;
  for (int i = tid; i < M * K; i += 128) {
    int r = i / K, k = i % K;
    sA[(k / 16) * A_LBO + (r / 8) * A_SBO + (r % 8) * 16 + k % 16] = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    int r = i / K, k = i % K;
    sB[(k / 16) * B_LBO + (r / 8) * B_SBO + (r % 8) * 16 + k % 16] = B[i];
  }
  if (warp == 0) {
    constexpr uint32_t cols = N < 32 ? 32 : N;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    const uint64_t ad = make_desc(smem_u32(sA), A_LBO, A_SBO);
    const uint64_t bd = make_desc(smem_u32(sB), B_LBO, B_SBO);
    constexpr uint32_t idesc = make_idesc_i8(M, N);
    t0 = clock64();
    for (int r = 0; r < reps; ++r) mma_i8(tmem, ad, bd, idesc, r > 0 ? 1u : 0u);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  mbar_wait(&bar, 0);
  // each warp reads its 32 lanes; N columns in chunks of 32
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    if (blockIdx.x == 0)
      for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    constexpr uint32_t cols = N < 32 ? 32 : N;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(cols));
  }
}

template <int N>
void run(int reps, int blocks) {
  const int M = 128, K = 32;
  std::vector<int8_t> hA(M * K), hB(N * K);
  srand(7 + N);
  for (auto& v : hA) v = (int8_t)((rand() % 7) - 3);
  for (auto& v : hB) v = (int8_t)((rand() % 7) - 3);
  int8_t *dA, *dB; int32_t* dD; long long* dc;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, blocks * 8);
  cudaMemcpy(dA, hA.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K, cudaMemcpyHostToDevice);
  k_umma<N><<<blocks, 128>>>(dA, dB, dD, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e)); exit(1); }
  std::vector<int32_t> hD(M * N);
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  std::vector<long long> cyc(blocks);
  cudaMemcpy(cyc.data(), dc, blocks * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[n * K + k];
      if (hD[m * N + n] != s * reps) { if (bad < 5) printf("  mismatch m=%d n=%d got %d want %d\n", m, n, hD[m * N + n], s * reps); ++bad; }
    }
  double mean = 0; for (auto c : cyc) mean += c; mean /= blocks;
  printf("N=%3d reps=%5d blocks=%4d: %s  cycles/MMA=%.2f  MAC/clk/SM=%.0f\n", N, reps, blocks, bad ? "WRONG" : "exact",
         mean / reps, 128.0 * N * 32 * reps / mean * (blocks > 148 ? 1 : 1));
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<32>(1, 1);
  run<64>(1, 1);
  run<128>(1, 1);
  run<256>(1, 1);
  for (int b : {1, 148}) {
    run<32>(4096, b);
    run<64>(4096, b);
    run<128>(4096, b);
    run<256>(4096, b);
  }
  return 0;
}
