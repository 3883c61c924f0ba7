// MMA issue-rate probe (sm_100a): how fast can ONE thread keep the tensor pipe fed with kind::mxf4 M128 N128 K64
// MMAs when the descriptors change per MMA the way the conv kernels' do?  One CTA per SM, one thread issues
// `tiles` tiles of T MMAs (+ one commit per tile), cycles per MMA printed.  Operand contents are irrelevant
// (timing only).  Variants:
//   0  constant A / B descriptors and D (the mxf4_probe loop)
//   1  conv2-like: A start = buffer (tile % 4) + offset (sp, t), LBO 160 / SBO 320; B block per MMA; D set tile % 3
//   2  as 1 with a dense A layout (LBO 2048, SBO 128)
//   3  as 1, all 18 x 4 A descriptors and 18 B descriptors precomputed before the loop (64-bit adds only)
//   4  as 1 with a tcgen05.commit after every MMA
//   5  A descriptor = base descriptor of buffer (tile % 4) + a constant (start address >> 4) per MMA, B = base + constant
//   6  as 5 with the tile loop unrolled by 12 (buffer and accumulator set compile-time constants)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe issue_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], 1;" ::"r"(d), "l"(a),
      "l"(b), "n"(idesc_mxf4(128, 128)), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar));
}

constexpr int T = 18, SP = 3, KS = 6;
constexpr uint32_t ROWB = 160, PLANE = 36 * ROWB + 64, ABYTES = 2 * PLANE, BBLK = 2 * 128 * 16;

__global__ void __launch_bounds__(128, 1) k_issue(int variant, int tiles, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                 // 4 A buffers
  uint8_t* sB = sm + 4 * ABYTES;    // 18 B blocks
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)(4 * ABYTES + T * BBLK) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x22222222u * (i & 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase, sfa = tmem + 384, sfb = tmem + 392;
  {
    const uint32_t lo = (uint32_t)(warp * 32) << 16, v = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfa + lo), "r"(v));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sfb + lo), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB), barp = smem_u32(&bar);
    uint64_t adp[4][T], bdp[T];
    for (int ab = 0; ab < 4; ++ab)
      for (int m = 0; m < T; ++m) {
        const int sp = m / KS, t = m % KS;
        adp[ab][m] = make_desc(a0 + ab * ABYTES + (t & 1) * PLANE + 2 * sp * ROWB + (t >> 1) * 16, ROWB, 2 * ROWB);
      }
    for (int m = 0; m < T; ++m) bdp[m] = make_desc(b0 + m * BBLK, 128 * 16, 128);
    const long long t0 = clock64();
    if (variant == 0) {
      const uint64_t ad = make_desc(a0, 2048, 128), bd = make_desc(b0, 2048, 128);
      for (int it = 0; it < tiles; ++it) {
#pragma unroll
        for (int m = 0; m < T; ++m) mma(tmem, ad, bd, sfa, sfb);
        commit(barp);
      }
    } else if (variant == 3) {
      int ab = 0, cb = 0;
      for (int it = 0; it < tiles; ++it) {
#pragma unroll
        for (int m = 0; m < T; ++m) mma(tmem + cb * 128, adp[ab][m], bdp[m], sfa, sfb);
        commit(barp);
        ab = (ab + 1) & 3;
        cb = cb == 2 ? 0 : cb + 1;
      }
    } else if (variant == 5) {
      uint64_t abd[4];
      for (int ab = 0; ab < 4; ++ab) abd[ab] = make_desc(a0 + ab * ABYTES, ROWB, 2 * ROWB);
      const uint64_t bbase = make_desc(b0, 128 * 16, 128);
      int ab = 0, cb = 0;
      for (int it = 0; it < tiles; ++it) {
        const uint64_t ab0 = abd[ab];
        const uint32_t d = tmem + cb * 128;
#pragma unroll
        for (int sp = 0; sp < SP; ++sp)
#pragma unroll
          for (int t = 0; t < KS; ++t)
            mma(d, ab0 + (((t & 1) * PLANE + 2 * sp * ROWB + (t >> 1) * 16) >> 4), bbase + (((sp * KS + t) * BBLK) >> 4), sfa, sfb);
        commit(barp);
        ab = (ab + 1) & 3;
        cb = cb == 2 ? 0 : cb + 1;
      }
    } else if (variant == 6) {
      const uint64_t abase0 = make_desc(a0, ROWB, 2 * ROWB), bbase = make_desc(b0, 128 * 16, 128);
      for (int it = 0; it < tiles; it += 12) {
#pragma unroll
        for (int u = 0; u < 12; ++u) {
          const uint64_t ab0 = abase0 + (((u & 3) * ABYTES) >> 4);
          const uint32_t d = tmem + (u % 3) * 128;
#pragma unroll
          for (int sp = 0; sp < SP; ++sp)
#pragma unroll
            for (int t = 0; t < KS; ++t)
              mma(d, ab0 + (((t & 1) * PLANE + 2 * sp * ROWB + (t >> 1) * 16) >> 4), bbase + (((sp * KS + t) * BBLK) >> 4), sfa, sfb);
          commit(barp);
        }
      }
    } else {
      const bool dense = variant == 2;
      int ab = 0, cb = 0;
      for (int it = 0; it < tiles; ++it) {
        const uint32_t abase = a0 + ab * ABYTES;
#pragma unroll
        for (int sp = 0; sp < SP; ++sp)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const uint64_t ad = dense ? make_desc(abase + (sp * KS + t) * 256, 2048, 128)
                                      : make_desc(abase + (t & 1) * PLANE + 2 * sp * ROWB + (t >> 1) * 16, ROWB, 2 * ROWB);
            const uint64_t bd = make_desc(b0 + (sp * KS + t) * BBLK, 128 * 16, 128);
            mma(tmem + cb * 128, ad, bd, sfa, sfb);
            if (variant == 4) commit(barp);
          }
        commit(barp);
        ab = (ab + 1) & 3;
        cb = cb == 2 ? 0 : cb + 1;
      }
    }
    // drain: a commit on a second barrier completes after every MMA issued above
    uint32_t done = 0;
    const uint32_t bar2p = smem_u32(&bar2);
    commit(bar2p);
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar2p));
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int smem = 4 * ABYTES + T * BBLK;
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* dc;
  cudaMalloc(&dc, 148 * 8);
  const int tiles = 1992;
  for (int v = 0; v <= 6; ++v) {
    k_issue<<<148, 128, smem>>>(v, tiles, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("variant %d: %s\n", v, cudaGetErrorString(e)); return 1; }
    long long h[148];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    printf("variant %d: %.1f clk per MMA (%d tiles x %d MMAs, 148 CTAs)\n", v, mean / (tiles * T), tiles, T);
  }
  return 0;
}
