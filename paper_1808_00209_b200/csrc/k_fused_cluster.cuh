// k_fused_cluster.cuh -- the whole vehicle-shaped network for a small batch in ONE thread-block cluster
// (pack -> conv1 + pool -> conv2 + pool -> FC1-3 + argmax with the activations kept on
// chip; the paper's batch-1 protocol, Table 1; its fusion idea).
//
// One cluster of up to 16 CTAs (one per SM, 16 warps each) runs every layer of one image after the other.
// There is no global-memory activation and no software grid barrier: each CTA keeps a FULL copy of the
// conv1 map (48 x 48 words) and of the conv2 map (24 x 24 words) in its shared memory, producers write
// every CTA's copy through distributed shared memory (lanes 0..15 of the producing warp each address one
// CTA), and the hardware cluster barrier (barrier.cluster arrive.release / wait.acquire) separates the
// phases.  Everything a phase reads is on chip before the phase starts:
//   prologue  one thread per CTA issues the bulk copy (mbarrier complete_tx) of the CTA's block of FC1 weight
//             rows (outputs [rank m1, rank m1 + m1)); CTA 0's threads issue 4-byte cp.async copies of the FC2 /
//             FC3 weights -- they land while conv1 / conv2 run;
//   phase 0   bulk copy of the raw image rows this CTA's conv1 rows need (pooled rows [rank RP, +RP) and the
//             K1 - 1 halo rows), clamped to the image; rows outside it are never read (R4 padding);
//   phase 1   the staged rows are thresholded (SIGN / THRESH_RGB, Eq. 1, R14) into a 0/1 byte image with zero
//             rows / columns around the image (the -1 padding, R4), then conv1 (+ 2x2 OR-pool) over this CTA's
//             pooled rows: warp = pooled pixel, lane = output channel; the K x K x c patch bits of the 4 window
//             pixels are branch-free byte reads + ballots, acc = K^2 c - 2 popc(patch ^ w) (Eq. 4); the word is
//             stored into every CTA's map (st.shared::cluster, lane l -> CTA l);
//   phase 2   conv2 (+ pool) from the local conv1 copy: warp = pooled pixel (all 4 window pixels), lane = output
//             channel, the (K2 x K2) 32-channel input words are warp-broadcast reads, each kernel row's K2 XOR
//             words go through the carry-save popcount (3 POPC instead of 5 for K2 = 5); stored like phase 1;
//   phase 3   FC1: warp = one of the CTA's m1 outputs (weights in shared memory), lanes stride the local conv2
//             copy; the bit goes to CTA 0 with one DSMEM atomicOr;
//   phase 4   CTA 0: FC2 -> FC3 integer logits (weights in shared memory) -> argmax (first maximum, R19).
// All integer; results equal the layer-by-layer path.  Same topology checks as fused_small_kernel.
#pragma once
#include <cooperative_groups.h>

#include "k_conv.cuh"  // csa_popc
#include "k_conv_tc4_pool.cuh"  // the pool-in-N conv2 operand layout, weight image and epilogue
#include "k_conv1_fp4.cuh"     // the conv1 strip layout, threshold masks, e2m1 nibbles, weight image
#include "k_fused_small.cuh"
#include "tc.cuh"

namespace bnn {

constexpr int kClusterMax = 16;

// shared-memory layout of fused_cluster_kernel (32-bit words; every block 16-byte aligned), for a cluster of
// `ncta` CTAs -- the host sizes it for the smallest cluster it may get (8)
struct FusedClusterLayout {
  int y1, y2, h1, h2, logit, raw, bim, f1w, f2w, f3w, tf, tcb, tca, tcl, c1b, c1c, c1a, c1r, total;  // word offsets
  int rp, raw_rows, m1, pb;  // pooled rows per CTA, staged raw rows, FC1 rows per CTA, bit-image row pitch (bytes)
  int nbox;                  // conv1 raw boxes per CTA (tensor-core conv1)
  __host__ __device__ FusedClusterLayout(int H, int W, int C, int K1, int ncta, int l1, int l2, int l3) {
    auto up4 = [](int v) { return (v + 3) & ~3; };
    const int H1 = H / 2, W1 = W / 2, H2 = H1 / 2, W2 = W1 / 2;
    rp = (H1 + ncta - 1) / ncta;
    raw_rows = 2 * rp + K1 - 1;
    m1 = (l1 + ncta - 1) / ncta;
    const int dw1 = H2 * W2, dw2 = (l1 + 31) / 32, dw3 = (l2 + 31) / 32;
    y1 = 0;
    y2 = y1 + up4(H1 * W1);
    h1 = y2 + up4(H2 * W2);
    h2 = h1 + kFusedMaxL / 32;
    logit = h2 + kFusedMaxL / 32;
    raw = logit + 32;
    pb = (W + K1 - 1) * C;
    bim = raw + up4((raw_rows * W * C + 3) / 4);
    f1w = bim + up4((raw_rows * pb + 3) / 4);
    f2w = f1w + up4(m1 * dw1);
    f3w = f2w + up4(l2 * dw2);
    tf = f3w + up4(l3 * dw3);                 // FC1 thr [m1], flip [m1]; FC2 thr [l2], flip [l2] (int)
    // tensor-core conv2 (K2 = 5, 32 channels): weight image, A operand (both 1024-byte aligned), LUT + start values
    tcb = (tf + up4(2 * (m1 + l2)) + 255) & ~255;
    tca = tcb + (int)(ConvTc4PoolCfg<5>::B_BYTES / 4);
    tcl = tca + ((int)(ConvTc4PoolCfg<5>::A_BYTES / 4) + 255) / 256 * 256;
    // tensor-core conv1 (K1 = 5, 3 channels): weight image, offset-MMA constants, A strips, raw box
    c1b = (tcl + 256 * (1 + ConvTc4PoolCfg<5>::LUTC) + 32 + 255) & ~255;
    c1c = c1b + (int)(Conv1Fp4Cfg<5>::B_BYTES / 4);
    c1a = c1c + (int)(Conv1Fp4Cfg<5>::CONST_BYTES / 4);
    c1r = c1a + (int)((Conv1Fp4Cfg<5>::A_BYTES / 4 + 31) & ~31u);
    // raw boxes of this CTA's conv1 tiles (ceil(tiles / ncta), prefetched one image ahead)
    const int t1 = ((H1 + Conv1Fp4Cfg<5>::PH - 1) / Conv1Fp4Cfg<5>::PH) * ((W1 + Conv1Fp4Cfg<5>::PW - 1) / Conv1Fp4Cfg<5>::PW);
    nbox = (t1 + ncta - 1) / ncta;
    total = c1r + nbox * (int)(Conv1Fp4Cfg<5>::RAW_BYTES / 4) + 32;
  }
};

// TC2: conv2 (K2 = 5, 32 -> 32 channels, pool 2) on the tensor cores -- one 16 x 8 pooled-pixel tile per CTA, the
// pool window folded into N exactly as conv_tc4_pool_kernel (18 mxf4 MMAs of M128 N128 K64 into TMEM), the A operand
// expanded from the CTA's local conv1 copy, the start values C0 - (thr' + 1) and the s16 sign gather of that
// kernel; each pooled word is stored into every CTA's conv2 map
// TC1: conv1 (K1 = 5, 3 input channels, SIGN / THRESH_RGB) on the tensor cores as conv1_fp4_pool_kernel computes it --
// one 16 x 8 pooled-pixel tile per CTA and round (18 tiles for 96 x 96), the raw box staged by word loads, strips of
// {0, 1} e2m1 built from the threshold masks, the offset MMA (C0) + 3 mxf4 MMAs, the s16 sign gather
template <int K2, bool TC2 = false, bool TC1 = false>
__global__ void __launch_bounds__(kFusedWarps * 32, 1) fused_cluster_kernel(const FusedSmallArgs A) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) uint32_t cl_smem[];
  __shared__ uint64_t w_bar, raw_bar, tc_wbar, tc_mma;
  __shared__ uint32_t tmem_s;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), ncta = (int)cl.num_blocks();
  // several clusters (1-D grid of whole clusters): cluster cid serves images cid, cid + ncl, ... (no shared state)
  const int cid = (int)(blockIdx.x / (unsigned)ncta), ncl = (int)(gridDim.x / (unsigned)ncta);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = rank * kFusedWarps + warp, nw = ncta * kFusedWarps;
  const int H1 = A.H >> 1, W1 = A.W >> 1, H2 = H1 >> 1, W2 = W1 >> 1;
  const int C = A.C, K = A.K1, R = (K - 1) / 2;
  const FusedClusterLayout Lo(A.H, A.W, C, K, ncta, A.l1, A.l2, A.l3);
  const int dw1 = H2 * W2, dw2 = (A.l1 + 31) / 32, dw3 = (A.l2 + 31) / 32;
  uint32_t* y1 = cl_smem + Lo.y1;  // [H1 * W1] conv1 map (full copy)
  uint32_t* y2 = cl_smem + Lo.y2;  // [H2 * W2] conv2 map (full copy; OR-accumulated)
  uint32_t* h1 = cl_smem + Lo.h1;  // FC1 bits (CTA 0's copy is the target)
  uint32_t* h2 = cl_smem + Lo.h2;  // FC2 bits (CTA 0)
  int32_t* s_logit = reinterpret_cast<int32_t*>(cl_smem + Lo.logit);
  const uint8_t* raw = reinterpret_cast<const uint8_t*>(cl_smem + Lo.raw);
  uint8_t* bim = reinterpret_cast<uint8_t*>(cl_smem + Lo.bim);  // [raw_rows][pb] 0/1 bytes, zero outside the image
  const uint32_t* f1w = cl_smem + Lo.f1w;  // FC1 rows [rank m1, rank m1 + m1)
  const uint32_t* f2w = cl_smem + Lo.f2w;  // (CTA 0)
  const uint32_t* f3w = cl_smem + Lo.f3w;  // (CTA 0)
  // lane l < ncta addresses CTA l's copies (DSMEM); every lane addresses CTA 0's FC1 bits
  const uint32_t y1_c = tc::mapa(tc::smem_addr(y1), lane < ncta ? lane : 0);  // CTA lane's maps (shared::cluster)
  const uint32_t y2_c = tc::mapa(tc::smem_addr(y2), lane < ncta ? lane : 0);
  uint32_t* h1_0 = cl.map_shared_rank(h1, 0);
  const int o1 = rank * Lo.m1, n1 = max(0, min(Lo.m1, A.l1 - o1));  // this CTA's FC1 outputs
  int32_t* s_t1 = reinterpret_cast<int32_t*>(cl_smem + Lo.tf);  // FC1 thresholds / flips of this CTA's outputs,
  int32_t* s_f1 = s_t1 + Lo.m1;                                 // FC2's (CTA 0): read per output by one lane,
  int32_t* s_t2 = s_f1 + Lo.m1;                                 // so they are loaded once, up front
  int32_t* s_f2 = s_t2 + A.l2;
  const int py0 = rank * Lo.rp, py1 = min(H1, py0 + Lo.rp);  // this CTA's pooled conv1 rows
  const int gy0 = 2 * py0 - R;                                 // image row of staged raw row 0
  const int rlo = max(0, gy0), rhi = min(A.H, 2 * py1 + K - 1 - R);  // staged image rows [rlo, rhi)
  const int rowb = A.W * C;
  // tensor-core conv1: the raw boxes (IR rows x RAW_W bytes from image row oy0 - R, byte ox0 C - XOFF) of this
  // CTA's tiles of image im, by 16-byte cp.async (zero fill outside the image; rows and boxes are 16-byte aligned)
  auto prefetch_boxes = [&](int im) {
    using C1 = Conv1Fp4Cfg<5>;
    constexpr int CPR = C1::RAW_W / 16, CPB = C1::IR * CPR;  // 16-byte chunks per box row / box
    const int t1x = (W1 + C1::PW - 1) / C1::PW, ntile1 = ((H1 + C1::PH - 1) / C1::PH) * t1x;
    const uint8_t* xi = A.x + (int64_t)im * A.H * A.W * C;
    uint8_t* boxes = reinterpret_cast<uint8_t*>(cl_smem + Lo.c1r);
    for (int k = threadIdx.x; k < Lo.nbox * CPB; k += blockDim.x) {
      const int sel = k / CPB, kk = k - sel * CPB, tile = rank + sel * ncta;
      if (tile >= ntile1) continue;
      const int ty = tile / t1x, tx = tile - ty * t1x, rr = kk / CPR, ch = kk - rr * CPR;
      const int gy = ty * C1::TH - C1::R + rr, xb = tx * C1::TW * 3 - C1::XOFF + 16 * ch;
      const bool ok = gy >= 0 && gy < A.H && xb >= 0 && xb + 16 <= A.W * C;
      const uint8_t* src = ok ? xi + (int64_t)gy * A.W * C + xb : A.x;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tc::smem_addr(boxes + sel * C1::RAW_BYTES + rr * C1::RAW_W + 16 * ch)),
                   "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_raw = [&](int img) {  // phase 0: the raw rows of this CTA's conv1 rows (one thread)
    const uint32_t bytes = (uint32_t)((rhi - rlo) * rowb);
    tc::mbar_arrive_expect_tx(&raw_bar, bytes);
    tc::stage_chunks(cl_smem + Lo.raw + ((rlo - gy0) * rowb) / 4, A.x + ((int64_t)img * A.H + rlo) * rowb, bytes, &raw_bar);
  };

  // Prologue: one batch of independent loads and asynchronous copies, then one relaxed cluster barrier (no
  // memory fence: nothing written here is read remotely before the phase barriers).  Thread 0 starts the first
  // image's raw rows and this CTA's FC1 weight rows (bulk copies); CTA 0 starts the FC2 / FC3 weights (cp.async).
  if (rank == 0) fused_trace(A, 64, 0);  // kernel entry
  if (threadIdx.x == 0) {
    tc::mbar_init(&w_bar, 1);
    tc::mbar_init(&raw_bar, 1);
    tc::fence_mbar_init();
    if (!TC1 && cid < A.n && rhi > rlo) stage_raw(cid);
    if constexpr (TC2 || TC1) {
      tc::mbar_init(&tc_wbar, 1);
      tc::mbar_init(&tc_mma, 1);
      tc::fence_mbar_init();
      // weight images, waited before the first MMA
      tc::mbar_arrive_expect_tx(&tc_wbar, (TC2 ? ConvTc4PoolCfg<5>::B_BYTES : 0u) + (TC1 ? Conv1Fp4Cfg<5>::B_BYTES : 0u));
      if (TC2) tc::stage_chunks(cl_smem + Lo.tcb, A.w2img, ConvTc4PoolCfg<5>::B_BYTES, &tc_wbar);
      if (TC1) tc::stage_chunks(cl_smem + Lo.c1b, A.w1img, Conv1Fp4Cfg<5>::B_BYTES, &tc_wbar);
    }
    const uint32_t b1 = (uint32_t)n1 * dw1 * 4;  // dw1 % 4 == 0 (host check)
    tc::mbar_arrive_expect_tx(&w_bar, b1);
    if (b1) tc::stage_chunks(cl_smem + Lo.f1w, A.f1 + (int64_t)o1 * dw1, b1, &w_bar);
  }
  if constexpr (TC1) {
    if (cid < A.n) prefetch_boxes(cid);
  }
  if (rank == 0) {
    for (int j = threadIdx.x; j < A.l2 * dw2; j += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_addr(cl_smem + Lo.f2w + j)), "l"(A.f2 + j) : "memory");
    for (int j = threadIdx.x; j < A.l3 * dw3; j += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_addr(cl_smem + Lo.f3w + j)), "l"(A.f3 + j) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // conv2 weights of this lane's output channel, in registers for the whole kernel
  constexpr int KK2 = K2 * K2;
  uint32_t w2[KK2];
#pragma unroll
  for (int i = 0; i < KK2; ++i) w2[i] = __ldg(A.w2 + (int64_t)lane * KK2 + i);
  const int th2 = A.thr2 != nullptr ? A.thr2[lane] : 0;
  const bool fl2 = A.flip2 != nullptr && A.flip2[lane] != 0;
  // conv1: patch bit b = 32 w + lane <-> (ky, kx, c), b = (ky K + kx) C + c (MSB-first)
  const int nb = K * K * C, S1 = nb;
  // Small parameters are loaded into registers here and consumed (or stored to shared memory) at their first use,
  // so no load -> use stall sits in the prologue of this latency-critical kernel.
  float Tf[4] = {0.f, 0.f, 0.f, 0.f};  // input thresholds: t[c] = u8_threshold(-T[c]) at the image's conv1 phase
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (c < C && A.T != nullptr) Tf[c] = A.T[c];
  int t[4] = {0, 0, 0, 0};
  int off_[3];  // patch bit 32 w + lane: byte offset in the bit image from the window's top-left corner
  bool use_[3];
  uint32_t wreg[3];
#pragma unroll
  for (int w = 0; w < 3; ++w) {
    const int b = 32 * w + lane;
    use_[w] = b < nb;
    const int tap = use_[w] ? b / C : 0, c = use_[w] ? b - tap * C : 0;
    off_[w] = (tap / K) * Lo.pb + (tap % K) * C + c;
    wreg[w] = __ldg(A.w1p + lane * 3 + w);
  }
  const int th1 = A.thr1 != nullptr ? A.thr1[lane] : 0;
  const bool fl1 = A.flip1 != nullptr && A.flip1[lane] != 0;
  // FC1 / FC2 thresholds and flips (thread j < n1, CTA 0's threads j, j + 512 < l2 <= 1024): stored to shared memory
  // after image 0's conv1 phase (read per output by one lane in phases 3 / 4)
  const int pt1 = (threadIdx.x < n1 && A.thr_f1 != nullptr) ? A.thr_f1[o1 + threadIdx.x] : 0;
  const int pf1 = (threadIdx.x < n1 && A.flip_f1 != nullptr) ? A.flip_f1[o1 + threadIdx.x] : 0;
  int pt2[2] = {0, 0}, pf2[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = threadIdx.x + h * (int)blockDim.x;
    if (rank == 0 && j < A.l2) {
      pt2[h] = A.thr_f2 != nullptr ? A.thr_f2[j] : 0;
      pf2[h] = A.flip_f2 != nullptr ? A.flip_f2[j] : 0;
    }
  }
  auto store_fc_params = [&]() {
    if (threadIdx.x < n1) {
      s_t1[threadIdx.x] = pt1;
      s_f1[threadIdx.x] = pf1;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = threadIdx.x + h * (int)blockDim.x;
      if (rank == 0 && j < A.l2) {
        s_t2[j] = pt2[h];
        s_f2[j] = pf2[h];
      }
    }
  };
  for (int j = threadIdx.x; j < kFusedMaxL / 32; j += blockDim.x) h1[j] = 0u;
  using TP = ConvTc4PoolCfg<5>;
  const int tiles2_x = (W1 + TP::TW - 1) / TP::TW, tiles2 = ((H1 + TP::TH - 1) / TP::TH) * tiles2_x;
  const bool has_tile2 = TC2 && rank < tiles2;
  uint32_t* s_lut2 = cl_smem + Lo.tcl;            // LUTC interleaved copies of the bits -> e2m1 table
  float* s_init2 = reinterpret_cast<float*>(s_lut2 + 256 * TP::LUTC);  // C0 - (thr' + 1) per TMEM column
  if constexpr (TC1) {  // the offset MMA's constant operands: A = 1.0 everywhere, B = 6.0 at element 0 of a chunk row
    uint8_t* sC1 = reinterpret_cast<uint8_t*>(cl_smem + Lo.c1c);
    for (int i = threadIdx.x; i < (int)(Conv1Fp4Cfg<5>::CONST_BYTES / 16); i += blockDim.x)
      *reinterpret_cast<uint4*>(sC1 + 16 * i) = i < (int)(Conv1Fp4Cfg<5>::CONST_BYTES / 32)
                                                    ? make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u)
                                                    : make_uint4(0x7u, 0u, 0u, 0u);
  }
  if constexpr (TC2 || TC1) {
    if (warp == 0) {
      tc::tmem_alloc<256>(&tmem_s);
      tc::fence_before();  // (the address is read after the cluster barrier below)
    }
    if (threadIdx.x < 256) {
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) v |= (((threadIdx.x >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
#pragma unroll
      for (int c = 0; c < TP::LUTC; ++c) s_lut2[TP::LUTC * threadIdx.x + c] = v;
    }
  }
  // conv2 start values C0 - (thr' + 1) per TMEM column (as conv_tc4_pool_kernel: 32 valid channels): loaded here,
  // stored with the FC parameters
  const int pt_c2 = (TC2 && threadIdx.x < 32 && A.thr2 != nullptr) ? A.thr2[tc4_col_channel(threadIdx.x)] : 0;
  const int pf_c2 = (TC2 && threadIdx.x < 32 && A.flip2 != nullptr) ? A.flip2[tc4_col_channel(threadIdx.x)] : 0;
  auto store_c2_init = [&]() {
    if (TC2 && threadIdx.x < 32) {
      constexpr int S_TOT = 25 * 32;
      int tt = max(-S_TOT - 1, min(S_TOT, pt_c2));
      if (pf_c2 != 0) tt = max(-S_TOT - 1, min(S_TOT, -tt - 1));
      s_init2[threadIdx.x] = 12582912.0f - (float)(tt + 1);
    }
  };
  if (rank == 0) fused_trace(A, 64, 1);
  // every CTA of the cluster is running and has zeroed h1 (the first DSMEM atomics into it follow two phase
  // barriers later); the barrier's wait side synchronises the CTA (mbarrier initialisation, staged values)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");

  uint32_t mma_ph = 0;  // parity of the next tc_mma completion (conv1 tiles, then the conv2 tile, per image)
  for (int img = cid, it = 0; img < A.n; img += ncl, ++it) {  // it: this cluster's image count (phases, first use)
    if (rank == 0) fused_trace(A, img, 0);
#pragma unroll
    for (int c = 0; c < 4; ++c) t[c] = (c < C && A.T != nullptr) ? u8_threshold(-Tf[c]) : 0;
    if constexpr (TC1) {
      using C1 = Conv1Fp4Cfg<5>;
      tc::fence_after();
      const uint32_t tmem = tmem_s;
      const int t1x = (W1 + C1::PW - 1) / C1::PW, ntile1 = ((H1 + C1::PH - 1) / C1::PH) * t1x;
      uint8_t* sA1 = reinterpret_cast<uint8_t*>(cl_smem + Lo.c1a);
      asm volatile("cp.async.wait_all;" ::: "memory");  // this image's raw boxes (prefetched)
      __syncthreads();
      // builder constants (k_conv1_fp4.cuh, kBinRgb): per-channel 16-bit-lane threshold terms
      uint32_t Ev[3], Od[3];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        Ev[m] = (uint32_t)(0x7FFF - t[m]) | ((uint32_t)(0x7FFF - t[(m + 2) % 3]) << 16);
        Od[m] = (uint32_t)(0x7FFF - t[(m + 1) % 3]) | ((uint32_t)(0x7FFF - t[m]) << 16);
      }
      const bool zero_ok = t[0] >= 0 && t[1] >= 0 && t[2] >= 0;  // an all-zero byte thresholds to b = 0 (-1)
      for (int tile = rank, sel = 0; tile < ntile1; tile += ncta, ++sel) {
        const int ty = tile / t1x, tx = tile - ty * t1x, oy0 = ty * C1::TH, ox0 = tx * C1::TW;
        const uint8_t* box = reinterpret_cast<const uint8_t*>(cl_smem + Lo.c1r) + sel * C1::RAW_BYTES;
        // strips: item = (strip row r, 4 pooled columns j)
        if (threadIdx.x < C1::GROUPS) {
          constexpr int IPR = C1::PW / C1::SPI;
          const int r = threadIdx.x / IPR, j = threadIdx.x % IPR;
          const uint8_t* src = box + r * C1::RAW_W + C1::WB + 6 * C1::SPI * j;
          uint32_t M[C1::NWI];
#pragma unroll
          for (int w = 0; w < C1::NWI; ++w) M[w] = thresh_mask4(reinterpret_cast<const uint32_t*>(src)[w], Ev[(C1::C0 + w) % 3], Od[(C1::C0 + w) % 3]);
          if (!zero_ok) {  // out-of-image bytes must be b = 0 whatever the threshold
            const int gy = oy0 - C1::R + r;
            const bool row_ok = gy >= 0 && gy < A.H;
#pragma unroll
            for (int w = 0; w < C1::NWI; ++w)
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int xb = ox0 * 3 - C1::XOFF + C1::WB + 6 * C1::SPI * j + 4 * w + b;
                if (!row_ok || xb < 0 || xb >= rowb) M[w] &= ~(0xFFu << (8 * b));
              }
          }
          uint8_t* a = sA1 + r * C1::ROWP + C1::SPI * j * 16;
#pragma unroll
          for (int st = 0; st < C1::SPI; ++st) {
            const int o = C1::E + 6 * st, qw = o >> 2, sh = 8 * (o & 3);
            uint32_t m[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
              const int w = qw + k;
              const uint32_t lo = w < C1::NWI ? M[w] : 0u, hi = w + 1 < C1::NWI ? M[w + 1] : 0u;
              m[k] = (k < C1::NWS) ? (sh ? __funnelshift_r(lo, hi, sh) : lo) : 0u;
            }
            uint32_t v[4];
            conv1_nibbles<C1::SB>(m, v);
            *reinterpret_cast<uint4*>(a + st * 16) = make_uint4(v[0], v[1], v[2], v[3]);
          }
        }
        if (warp < 4 && it == 0 && tile == rank) {  // block scales (TMEM lane quarter = warp): 1.0, 1.0, 2^20
          const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
          tc::tmem_st8_same(lb + 128, 0x7F7F7F7Fu);
          tc::tmem_st8_same(lb + 136, 0x7F7F7F7Fu);
          tc::tmem_st8_same(lb + 144, 0x93939393u);
          tc::tmem_st_wait();
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (threadIdx.x == 0) {
          if (it == 0 && tile == rank) tc::mbar_wait(&tc_wbar, 0);  // the weight images landed
          constexpr uint32_t idesc = tc::idesc_mxf4(128, C1::N);
          const uint64_t adc = tc::desc_kmajor(tc::smem_addr(cl_smem + Lo.c1c), 128 * 16, 128);
          const uint64_t bdc = tc::desc_kmajor(tc::smem_addr(cl_smem + Lo.c1c) + C1::CONST_BYTES / 2, C1::N * 16, 128);
          const uint64_t ad0 = tc::desc_kmajor(tc::smem_addr(sA1), C1::ROWP, 2 * C1::ROWP);
          const uint64_t bd0 = tc::desc_kmajor(tc::smem_addr(cl_smem + Lo.c1b), C1::N * 16, 128);
          tc::mma_mxf4(tmem, adc, bdc, idesc, tmem + 128, tmem + 144, 0u);  // D = C0
#pragma unroll
          for (int pp = 0; pp < C1::NMMA; ++pp)
            tc::mma_mxf4(tmem, ad0 + (uint64_t)((pp * 2 * C1::ROWP) >> 4), bd0 + (uint64_t)((pp * 2 * C1::N * 16) >> 4), idesc,
                         tmem + 128, tmem + 136, 1u);
          tc::commit(&tc_mma);
        }
        if (warp < 4) {  // epilogue: pooled bit = max_q V_q >= 0 (k_conv1_fp4.cuh), thread = pooled pixel of the tile
          tc::mbar_wait(&tc_mma, mma_ph);
          __syncwarp();
          tc::fence_after();
          const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
          uint32_t a[16], b[16], c[16], d[16];
          tc::tmem_ld16_p16(lb + 0 * 32, a);
          tc::tmem_ld16_p16(lb + 1 * 32, b);
          tc::tmem_ld16_p16(lb + 2 * 32, c);
          tc::tmem_ld16_p16(lb + 3 * 32, d);
          tc::tmem_ld_wait();
          uint32_t neg = 0;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            uint32_t x;
            asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(x) : "r"(a[jj]), "r"(b[jj]), "r"(c[jj]));
            x = x & d[jj] & 0x80008000u;
            neg = __umulhi(neg, 0x80000000u) + x;
          }
          const int m = warp * 32 + lane, py = (oy0 >> 1) + m / C1::PW, px = (ox0 >> 1) + m % C1::PW;
          if (py < H1 && px < W1) {
            const uint32_t word = ~neg, addr = tc::smem_addr(y1 + py * W1 + px);
            for (int r = 0; r < ncta; ++r)
              asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(tc::mapa(addr, (uint32_t)r)), "r"(word));
          }
          tc::fence_before();
        }
        mma_ph ^= 1u;
        __syncthreads();  // (strips and the accumulator are reused by the next tile)
      }
      if (img + ncl < A.n) prefetch_boxes(img + ncl);  // lands during conv2 / FC
    } else {
    // ---- phase 0: raw rows of this CTA's conv1 rows
    if (threadIdx.x == 0 && rhi > rlo && it > 0) stage_raw(img);
    if (rhi > rlo) tc::mbar_wait(&raw_bar, (uint32_t)(it & 1));
    if (rank == 0) fused_trace(A, img, 5);
    // ---- phase 1a: the 0/1 byte image of the staged rows (zero outside the image: the -1 padding, R4)
    for (int r = warp; r < Lo.raw_rows; r += kFusedWarps) {  // warp = row, lane = bit-image column (pixel)
      const int gy = gy0 + r;
      const bool row_in = gy >= 0 && gy < A.H;
      for (int xx = lane; xx < A.W + K - 1; xx += 32) {
        const int gx = xx - R;
        const bool in = row_in && gx >= 0 && gx < A.W;
#pragma unroll
        for (int c = 0; c < 4; ++c)  // (t[] stays in registers: compile-time indices)
          if (c < C) bim[r * Lo.pb + xx * C + c] = (in && (int)raw[(gy - gy0) * rowb + gx * C + c] > t[c]) ? 1 : 0;
      }
    }
    __syncthreads();
    // ---- phase 1b: conv1 + pool over pooled rows [py0, py1) -> every CTA's y1
#pragma unroll 2
    for (int u = py0 * W1 + warp; u < py1 * W1; u += kFusedWarps) {
      const int py = u / W1, px = u - py * W1;
      const uint8_t* win = bim + (2 * py - R - gy0) * Lo.pb + 2 * px * C;  // window corner of offset q = 0
      uint32_t v[12];  // all 12 patch bytes of the 4 offsets first (independent loads), then the ballots
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 3; ++w) v[3 * q + w] = win[(q >> 1) * Lo.pb + (q & 1) * C + off_[w]];
      bool any = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int pc = 0;
#pragma unroll
        for (int w = 0; w < 3; ++w) pc += popc(ballot_pack(use_[w] && v[3 * q + w] != 0) ^ wreg[w]);
        any |= (S1 - 2 * pc > th1) != fl1;
      }
      const uint32_t word = ballot_pack(any);
      // (no "memory" clobber: the next pixel's loads may move above the store; the cluster barrier orders it.
      // Writing the own copy first and broadcasting 16-byte pieces after the loop measured the same.)
      if (lane < ncta) asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(y1_c + 4 * u), "r"(word));
    }
    }
    if (rank == 0) fused_trace(A, img, 6);  // (thread 0: its own warp's pixels done)
    if (it == 0) {  // (the phase barrier below publishes them)
      store_fc_params();
      store_c2_init();
    }
    cl.sync();
    if (rank == 0) fused_trace(A, img, 1);
    // ---- phase 2: conv2 + pool from the local y1 -> every CTA's y2
    if constexpr (TC2) {
      tc::fence_after();
      const uint32_t tmem = tmem_s;
      if (has_tile2) {
        const int ty = rank / tiles2_x, tx = rank - ty * tiles2_x, oy0 = ty * TP::TH, ox0 = tx * TP::TW;
        uint8_t* sA2 = reinterpret_cast<uint8_t*>(cl_smem + Lo.tca);
        // start values of the 4 x 32 accumulator columns (warps 0-3: TMEM lane quarters); block scales 1.0
        if (warp < 4) {
          const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
          uint32_t iv[16];
#pragma unroll
          for (int cb = 0; cb < 32; cb += 16) {
#pragma unroll
            for (int k = 0; k < 16; ++k) iv[k] = __float_as_uint(s_init2[cb + k]);
#pragma unroll
            for (int q = 0; q < 4; ++q) tmem_st16(lb + (uint32_t)(q * 32 + cb), iv);
          }
          if (it == 0) {
            tc::tmem_st8_same(lb + 128, 0x7F7F7F7Fu);
            tc::tmem_st8_same(lb + 136, 0x7F7F7F7Fu);
          }
          tc::tmem_st_wait();
        }
        // A operand: the tile's halo pixels (IR x IC) as e2m1 in two column-parity planes (k_conv_tc4_pool.cuh)
        const uint32_t* my_lut = s_lut2 + (lane & (TP::LUTC - 1));
        for (int p = threadIdx.x; p < TP::NPIX; p += blockDim.x) {
          const int r = p / TP::IC, c = p - r * TP::IC;
          const int gy = oy0 - TP::R + r, gx = ox0 - TP::R + c;
          const uint32_t w = (gy >= 0 && gy < H1 && gx >= 0 && gx < W1) ? y1[gy * W1 + gx] : 0u;  // outside: -1 (R4)
          uint32_t o4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) o4[k] = my_lut[TP::LUTC * ((w >> (24 - 8 * k)) & 0xFFu)];
          *reinterpret_cast<uint4*>(sA2 + (c & 1) * TP::PLANE + r * TP::ROWB + (c >> 1) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (threadIdx.x == 0) {
          if (it == 0) tc::mbar_wait(&tc_wbar, 0);  // the weight image landed
          constexpr uint32_t idesc = tc::idesc_mxf4(128, 128);
          const uint64_t adesc0 = tc::desc_kmajor(tc::smem_addr(sA2), TP::ROWB, 2 * TP::ROWB);
          const uint64_t bdesc0 = tc::desc_kmajor(tc::smem_addr(cl_smem + Lo.tcb), 128 * 16, 128);
#pragma unroll
          for (int sp = 0; sp < TP::SP; ++sp)
#pragma unroll
            for (int t = 0; t < TP::KS; ++t)
              tc::mma_mxf4(tmem, adesc0 + (uint64_t)(((t & 1) * TP::PLANE + (2 * sp) * TP::ROWB + (t >> 1) * 16) >> 4),
                           bdesc0 + (uint64_t)(((sp * TP::KS + t) * 2 * 128 * 16) >> 4), idesc, tmem + 128, tmem + 136, 1u);
          tc::commit(&tc_mma);
        }
        // epilogue (warps 0-3, thread = pooled pixel of the tile): pooled bit = NOT(all four acc'_q < 0)
        if (warp < 4) {
          tc::mbar_wait(&tc_mma, mma_ph);
          __syncwarp();
          tc::fence_after();
          const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
          uint32_t a[16], b[16], c[16], d[16];
          tc::tmem_ld16_p16(lb + 0 * 32, a);
          tc::tmem_ld16_p16(lb + 1 * 32, b);
          tc::tmem_ld16_p16(lb + 2 * 32, c);
          tc::tmem_ld16_p16(lb + 3 * 32, d);
          tc::tmem_ld_wait();
          uint32_t neg = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            uint32_t x;
            asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(x) : "r"(a[j]), "r"(b[j]), "r"(c[j]));
            x = x & d[j] & 0x80008000u;
            neg = __umulhi(neg, 0x80000000u) + x;
          }
          const int m = warp * 32 + lane, py = (oy0 >> 1) + m / TP::PW, px = (ox0 >> 1) + m % TP::PW;
          if (py < H2 && px < W2) {
            const uint32_t word = ~neg, addr = tc::smem_addr(y2 + py * W2 + px);
            for (int r = 0; r < ncta; ++r)
              asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(tc::mapa(addr, (uint32_t)r)), "r"(word));
          }
          tc::fence_before();  // (TMEM reads done before the next image's start values)
        }
        mma_ph ^= 1u;
      }
    } else {
      constexpr int RR = (K2 - 1) / 2;
      const int S2 = KK2 * 32;
      for (int u = gw; u < H2 * W2; u += nw) {
        const int py = u / W2, px = u - py * W2;
        bool any = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
          int acc = 0;
#pragma unroll
          for (int ky = 0; ky < K2; ++ky) {  // one kernel row's K2 XOR words through the carry-save popcount (f3)
            uint32_t xr[K2];
#pragma unroll
            for (int kx = 0; kx < K2; ++kx) {
              const int gy = oy + ky - RR, gx = ox + kx - RR;
              const uint32_t x = (gy >= 0 && gy < H1 && gx >= 0 && gx < W1) ? y1[gy * W1 + gx] : 0u;
              xr[kx] = x ^ w2[ky * K2 + kx];
            }
            acc += csa_popc<K2>(xr);
          }
          any |= (S2 - 2 * acc > th2) != fl2;
        }
        const uint32_t word = ballot_pack(any);
        if (lane < ncta) asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(y2_c + 4 * u), "r"(word));
      }
    }
    cl.sync();
    if (rank == 0) fused_trace(A, img, 2);
    // ---- phase 3: FC1 outputs [o1, o1 + n1) from the local y2 (weights in shared memory), bits into CTA 0's h1
    if (it == 0) tc::mbar_wait(&w_bar, 0);
    {
      const int64_t d1 = (int64_t)dw1 * 32;
      for (int k = warp; k < n1; k += kFusedWarps) {
        const uint32_t* wr = f1w + (int64_t)k * dw1;
        int s = 0;
#pragma unroll 6
        for (int j = lane; j < dw1; j += 32) s += popc(y2[j] ^ wr[j]);
        s = __reduce_add_sync(BNN_FULL_MASK, s);
        const int o = o1 + k, acc = (int)d1 - 2 * s;  // Eq. (4)
        const int tt = s_t1[k];
        const bool f = s_f1[k] != 0;
        if (lane == 0 && ((acc > tt) != f)) atomicOr(h1_0 + (o >> 5), 1u << (31 - (o & 31)));
      }
    }
    cl.sync();
    if (rank == 0) fused_trace(A, img, 3);
    // ---- phase 4 (CTA 0): FC2 -> FC3 integer logits -> argmax
    if (rank == 0) {
      if (it == 0) asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's FC2 / FC3 weight copies
      fused_dense_smem(h1, A.l1, f2w, A.l2, s_t2, s_f2, h2, nullptr);
      __syncthreads();
      fused_trace(A, img, 7);
      fused_dense_smem(h2, A.l2, f3w, A.l3, nullptr, nullptr, nullptr, s_logit);
      __syncthreads();
      if (warp == 0) {
        const bool ok = lane < A.l3;
        const int v = ok ? s_logit[lane] : 0;
        if (ok && A.logits != nullptr) A.logits[(int64_t)img * A.l3 + lane] = v;
        int bv = ok ? v : INT_MIN, bi = ok ? lane : INT_MAX;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
          const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, sh);
          const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, sh);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0 && A.cls != nullptr) A.cls[img] = bi;  // first maximum wins (R19)
      }
      for (int j = threadIdx.x; j < dw2; j += blockDim.x) h1[j] = 0u;  // next image's FC1 bits
      __syncthreads();
      fused_trace(A, img, 4);
    }
  }
  if (rank == 0) fused_trace(A, 64, 2);
  cl.sync();  // no CTA exits while another may still address its shared memory
  if (rank == 0) fused_trace(A, 64, 3);
  if constexpr (TC2 || TC1) {
    if (warp == 0) tc::tmem_dealloc<256>(tmem_s);
  }
}

}  // namespace bnn
