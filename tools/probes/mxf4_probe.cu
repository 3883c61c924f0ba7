// tcgen05.mma kind::mxf4 (block-scaled packed e2m1) probe for sm_100a.
// Checks (1) a +/-1/0 e2m1 GEMM M128 x N x K64 with all scale factors = 1.0 (UE8M0 0x7F filled into
// TMEM) against a CPU dot product, with a standard K-major SWIZZLE_NONE layout and with the
// "overlapping chunks" layout (LBO = 16 B: K-chunk 1 of row m is the 16 bytes right after K-chunk 0,
// i.e. the next pixel); (2) cycles per MMA for N = 32 / 128 / 256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mxf4_probe mxf4_probe.cu
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
// block-scaled instruction descriptor: a/b format E2M1 (=1 for MXF4), scale E8M0, K64
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase));
}

// A: M x 64 e2m1 codes (one per byte in `A`, values 0x2 / 0xA / 0x0), packed two per byte, low nibble first.
template <int N>
__global__ void __launch_bounds__(128) k_mxf4(const uint8_t* A, const uint8_t* B, float* D, int reps, int overlap,
                                               long long* cycles) {
  constexpr int M = 128, KB = 32;  // bytes per row (64 elements)
  __shared__ __align__(1024) uint8_t sA[M * KB + 4096];
  __shared__ __align__(1024) uint8_t sB[N * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // standard: (r, chunk c) at c*LBO + (r/8)*128 + (r%8)*16, LBO = M/8*128
  // overlap:  row r chunk 0 at 16*r (rows contiguous, 16 B each), chunk 1 = row r + 1's chunk 0
  for (int i = tid; i < M * KB; i += 128) {
    const int r = i / KB, b = i % KB, c = b / 16, o = b % 16;
    if (!overlap) sA[c * (M / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + o] = A[i];
  }
  if (overlap)  // pixel stream: P[p] = 16 bytes; row r = (P[r], P[r+1])
    for (int i = tid; i < (M + 1) * 16; i += 128) sA[i] = A[(i / 16 < M ? (i / 16) * KB : (M - 1) * KB + 16) + i % 16];
  for (int i = tid; i < N * KB; i += 128) {
    const int r = i / KB, b = i % KB, c = b / 16, o = b % 16;
    sB[c * (N / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + o] = B[i];
  }
  constexpr uint32_t COLS = (2 * N + 16 <= 64) ? 64 : ((N + 16 <= 128) ? 128 : ((N + 16 <= 256) ? 256 : 512));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(COLS));
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
  const uint32_t tmem = tbase;
  const uint32_t sfa = tmem + N, sfb = tmem + N + 8;  // columns after the accumulator
  {  // all scale factors = 1.0 (UE8M0 0x7F), 8 columns each, every lane
    const uint32_t v = 0x7F7F7F7Fu;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfa + lane_off), "r"(v));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfb + lane_off), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint64_t ad = overlap ? make_desc(smem_u32(sA), 16, 128) : make_desc(smem_u32(sA), M / 8 * 128, 128);
    const uint64_t bd = make_desc(smem_u32(sB), N / 8 * 128, 128);
    constexpr uint32_t idesc = idesc_mxf4(M, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(sfa), "r"(sfb), "r"(r > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (blockIdx.x == 0)
      for (int j = 0; j < 8; ++j) D[(warp * 32 + (tid & 31)) * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS));
}

static int val(uint8_t code) { return code == 0x2 ? 1 : (code == 0xA ? -1 : 0); }

template <int N>
void run(int reps, int blocks, int overlap) {
  const int M = 128, K = 64;
  std::vector<uint8_t> codes_a(M * K), codes_b(N * K), hA(M * 32), hB(N * 32);
  srand(11 + N + overlap);
  const uint8_t pick[3] = {0x2, 0xA, 0x0};
  for (auto& v : codes_a) v = pick[rand() % 3];
  for (auto& v : codes_b) v = pick[rand() % 3];
  if (overlap)  // row r's second half must equal row r+1's first half (pixel stream)
    for (int r = 0; r < M; ++r)
      for (int k = 32; k < 64; ++k) codes_a[r * K + k] = (r + 1 < M) ? codes_a[(r + 1) * K + k - 32] : codes_a[r * K + k];
  for (int r = 0; r < M; ++r)
    for (int b = 0; b < 32; ++b) hA[r * 32 + b] = codes_a[r * K + 2 * b] | (codes_a[r * K + 2 * b + 1] << 4);
  for (int r = 0; r < N; ++r)
    for (int b = 0; b < 32; ++b) hB[r * 32 + b] = codes_b[r * K + 2 * b] | (codes_b[r * K + 2 * b + 1] << 4);
  uint8_t *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, M * 32); cudaMalloc(&dB, N * 32); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, blocks * 8);
  cudaMemcpy(dA, hA.data(), M * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * 32, cudaMemcpyHostToDevice);
  k_mxf4<N><<<blocks, 128>>>(dA, dB, dD, reps, overlap, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e)); exit(1); }
  std::vector<float> hD(M * N);
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  std::vector<long long> cyc(blocks);
  cudaMemcpy(cyc.data(), dc, blocks * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  const int rows = overlap ? M - 1 : M;  // the last overlapped row reads past the stream
  for (int m = 0; m < rows; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int k = 0; k < K; ++k) s += val(codes_a[m * K + k]) * val(codes_b[n * K + k]);
      if (hD[m * N + n] != (float)(s * reps)) {
        if (bad < 4) printf("  mismatch m=%d n=%d got %f want %d\n", m, n, hD[m * N + n], s * reps);
        ++bad;
      }
    }
  double mean = 0; for (auto c : cyc) mean += c; mean /= blocks;
  printf("mxf4 N=%3d overlap=%d reps=%5d blocks=%3d: %s  cycles/MMA=%.2f  MAC/clk/SM=%.0f\n", N, overlap, reps, blocks,
         bad ? "WRONG" : "exact", mean / reps, 128.0 * N * 64 * reps / mean);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<32>(1, 1, 0);
  run<32>(1, 1, 1);
  run<128>(1, 1, 0);
  run<128>(1, 1, 1);
  run<256>(1, 1, 0);
  for (int ov : {0, 1}) {
    run<32>(4096, 148, ov);
    run<64>(4096, 148, ov);
    run<128>(4096, 148, ov);
    run<256>(4096, 148, ov);
  }
  return 0;
}
