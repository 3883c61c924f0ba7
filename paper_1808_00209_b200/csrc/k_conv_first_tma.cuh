// k_conv_first_tma.cuh -- pooled first conv layer on u8 RGB input with the THRESH_RGB binarization
// fused (Section 3.1 preprocessing, PAPER.md:141-145 / 178-179, then Eq. 3 + Eq. 1 + 2x2 pool,
// PAPER.md:212-218, 242-244), fed by TMA.
//
// Same MMA structure as conv_first_tc_pool_kernel (k_conv_first_tc.cuh: 128 pooled pixels per
// tile, strips of K taps x 3 channels as int8 +/-1, two parity planes, 4 accumulator blocks one per
// 2x2 pool offset), but every per-pixel instruction that kernel spent is gone or halved:
//   * the raw u8 halo box (IR rows x 80 B, starting 16 B left of the tile: the innermost TMA box
//     coordinate must be 16-byte aligned) is one cp.async.bulk.tensor per tile into an NRAW-deep ring;
//     out-of-image bytes arrive as 0, which thresholds to -1 = the binary padding whenever every
//     channel threshold t_c >= 0 (else a uniform slow path patches them);
//   * the threshold x > t_c (R14) runs 4 bytes at a time: the even / odd bytes are spread into two
//     16-bit-lane words (PRMT), x + (0x7FFF - t_c) sets lane bit 15 iff x > t_c, and one PRMT with
//     sign replication gathers the four results as 0xFF / 0x00 bytes; ~M | 0x01 gives int8 +/-1.
//     The 16-byte strip of output column x is the thresholded row bytes [3x, 3x + 15), so a thread
//     thresholds 6 words and cuts 4 strips from them with funnel shifts;
//   * the per-channel threshold and flip are folded into the MMA: flipped channels get negated
//     weights (NOT(acc > t) == (-acc) > -t-1), and byte 15 of every strip (unused by the 15 taps x
//     channels) is forced to -1 while the weights carry thr'+1 there (split over kernel rows 0 and
//     1), so TMEM holds acc - thr' - 1 and the pooled bit is simply max_q(acc'_q) >= 0;
//   * the epilogue runs on all 8 warps (warp w: pixel quarter w%4, channel half w/4): one VIMNMX
//     and one VIMNMX3 per channel for the 4-way max, one funnel shift for the sign bit, one u16
//     store of 16 channel bits per pixel.
#pragma once
#include <cuda.h>

#include "k_conv_first_tc.cuh"

namespace bnn {

template <int K, bool FP4 = false, bool DB = false>
struct FirstTmaCfg {
  static constexpr int CIN = 3, NT = 32, R = (K - 1) / 2, PH = 16, PW = 8, TH = 2 * PH, TW = 2 * PW;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1;
  // TMA needs a 16-byte aligned innermost box coordinate (measured: tools/probes/tma_probe.cu), so the
  // box starts XOFF = 16 bytes before the tile's first output column (ox0 * 3, a multiple of 48) and
  // the strip of pooled column px starts at box byte DELTA + 6 px; builders read aligned words.
  static constexpr int XOFF = 16, DELTA = XOFF - 3 * R, E = DELTA & 3;
  static constexpr int C0 = (DELTA - E + 32 * 3 - XOFF) % 3;  // channel of box byte DELTA - E
  static constexpr int RAW_W = 80;  // box row bytes (>= DELTA + IC * 3; 80 B pitch spreads smem banks)
  static constexpr uint32_t RAW_BYTES = IR * RAW_W;
  static constexpr uint32_t RAW_STRIDE = (RAW_BYTES + 127) / 128 * 128;  // TMA destinations 128-B aligned
  static constexpr int NRAW = 8;  // raw-box ring: TMA prefetch distance NRAW - 1 tiles (HBM latency x bandwidth)
  static constexpr int KS = K + 1;        // strip rows per MMA group = taps per strip (pool offsets 0/1)
  static constexpr int SB = KS * CIN;     // data bytes of a strip (18 for K = 5); bytes SB..31 = -1
  static constexpr int N = 4 * NT;        // MMA N: (dy, dx) pool offsets x NT channels
  static constexpr int SRR = IR;          // strip rows
  // i8: a strip row is 32 int8 = two 16-byte K chunks (planes), one MMA (K = 32) per strip row;
  // FP4: a strip row is 32 e2m1 nibbles = one 16-byte chunk, one MMA (K = 64) per pair of strip rows
  // int8 strip-row pitch: one core matrix (PW = 8 strips x 16 B) + 16 B of padding, so the builders'
  // 16-byte stores of rows r and r+1 land in different banks (a 128-B pitch made every STS.128 of a
  // quarter-warp a 2-way bank conflict: ncu, half of the shared-memory store wavefronts); the MMA's
  // core matrices stay contiguous 128 B (SBO = 2 pitches)
  static constexpr uint32_t ROWP = FP4 ? PW * 16 : PW * 16 + 16;
  static constexpr uint32_t PLANE = SRR * ROWP;
  static constexpr uint32_t A_BYTES = FP4 ? PLANE : 2 * PLANE;
  static constexpr int NMMA = FP4 ? KS / 2 : KS;
  static constexpr uint32_t B_BYTES = NMMA * 2 * N * 16;
  // FP4: + block-scale columns; DB (int8 only): two accumulator sets, so tile it+1's MMAs run while
  // tile it is drained
  static constexpr uint32_t TMEM_COLS = (FP4 || DB) ? 256 : 128;
  static_assert(!(FP4 && DB), "e2m1 + double buffering needs > 256 TMEM columns");
  static constexpr int GROUPS = IR * (PW / 2);  // 2-strip work items
  static_assert(!FP4 || (KS % 2 == 0 && KS * (32 - SB) >= K * K * CIN / 6 + 3), "fp4 bias slots");
  static_assert(SB <= 31 && DELTA >= 0 && DELTA - E + 12 * (PW / 2 - 1) + 32 <= RAW_W && (TW * CIN) % 16 == 0 &&
                E + 6 + SB <= 32, "config");
};

BNN_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// 4 u8 -> 4 int8 (+1 if x > t else -1); E / O hold 0x7FFF - t for the even / odd byte lanes
BNN_DEV uint32_t thresh4(uint32_t x, uint32_t E, uint32_t O) {
  const uint32_t ev = prmt(x, 0u, 0x4240u) + E;
  const uint32_t od = prmt(x, 0u, 0x4341u) + O;
  const uint32_t m = prmt(ev, od, 0xFBD9u);  // sign of lane bit 15 -> 0xFF / 0x00 per byte
  return ~m | 0x01010101u;
}

// 4 u8 -> per-byte mask 0xFF where x > t (the sign-replicating PRMT of thresh4)
BNN_DEV uint32_t thresh_mask4(uint32_t x, uint32_t E, uint32_t O) {
  const uint32_t ev = prmt(x, 0u, 0x4240u) + E;
  const uint32_t od = prmt(x, 0u, 0x4341u) + O;
  return prmt(ev, od, 0xFBD9u);
}

BNN_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          tc::smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tc::smem_addr(bar))
      : "memory");
}

// mbarrier wait of the staging / epilogue warps: sleeping (suspend-time hint) unless exp bit 16
BNN_DEV void wait_x(int exp, uint64_t* bar, uint32_t phase) {
  if (exp & 16) tc::mbar_wait(bar, phase);
  else tc::mbar_wait_sleep(bar, phase);
}

BNN_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_addr(bar)), "r"(bytes) : "memory");
}

// thr'+1 of output channel o: thr' = flip ? -t-1 : t, clamped to [-S_TOT-1, S_TOT] (the same
// decisions: |acc| <= S_TOT); invalid channels get 1 (acc' = -1 -> bit 0)
template <int K, bool REAL = false>
BNN_DEV int first_tma_bias(const ConvArgs& A, int o) {
  constexpr int S_TOT = K * K * 3 * (REAL ? 255 : 1);
  if (o >= A.c_out) return 1;
  const bool f = A.flip != nullptr && A.flip[o] != 0;
  int tt = A.thr != nullptr ? A.thr[o] : 0;
  tt = max(-S_TOT - 1, min(S_TOT, tt));
  if (f) tt = max(-S_TOT - 1, min(S_TOT, -tt - 1));
  return tt + 1;
}

// e2m1 code of a small integer (|v| in {0, 1, 2, 3, 4, 6})
BNN_DEV uint32_t e2m1_int(int v) {
  const int a = v < 0 ? -v : v;
  const uint32_t c = a == 0 ? 0x0u : a == 1 ? 0x2u : a == 2 ? 0x4u : a == 3 ? 0x5u : a == 4 ? 0x6u : 0x7u;
  return (v < 0 && a != 0) ? (c | 0x8u) : c;
}
// FP4 bias: v = thr'+1 spread over bias slot k (0, 1, ...) as 6, 6, ..., remainder (5 = 4 + 1)
BNN_DEV int fp4_bias_part(int v, int k) {
  const int a = v < 0 ? -v : v, sg = v < 0 ? -1 : 1;
  const int full = a / 6, r = a % 6;
  int part = 0;
  if (k < full) part = 6;
  else if (k == full) part = (r == 5) ? 4 : r;
  else if (k == full + 1 && r == 5) part = 1;
  return sg * part;
}

// The shared-memory image of the weight operand for channel group g ([mma][K chunk][n][16 B]):
// column n = q * NT + o holds W[o] shifted by the pool offset q = (dy, dx): strip row s, tap t of the
// 6-tap strip -> W[o][s - dy][t - dx] (zero outside the kernel), +/-1 negated for flipped channels.
// i8: byte SB of strip row 0 carries the bias thr'+1 against the strips' -1; FP4 (e2m1 nibbles, K
// chunk = one strip row): the bias is spread over the nibbles SB..31 of the strip rows (values in
// {6, 4, 3, 2, 1}, all against -1).  Written by the kernel itself, or once per net by
// prep_first_tma_kernel (then bulk-copied per CTA).
// REAL (mode NONE, u8 pixels as the unsigned A operand, zero padding R5): strip bytes SB and SB+1 are
// A = 1 and A = 255, and B carries -(thr'+1) = r + 255 q there (|r| <= 127, |q| <= 75) in strip row 0.
template <int K, bool FP4, bool REAL = false>
BNN_DEV void stage_b_first_tma(const ConvArgs& A, int g, uint8_t* dst, int i0, int step) {
  using C = FirstTmaCfg<K, FP4>;
  constexpr int N = C::N, NT = C::NT, CIN = C::CIN;
  for (int i = i0; i < C::NMMA * 2 * N; i += step) {
    const int n = i % N, kc = (i / N) & 1, mi = i / (2 * N);
    const int q = n / NT, o = g * NT + n % NT, dy = q >> 1, dx = q & 1;
    const bool ok = o < A.c_out;
    const bool f = ok && A.flip != nullptr && A.flip[o] != 0;
    const int bias = first_tma_bias<K, REAL>(A, o);
    uint32_t w4[4] = {0u, 0u, 0u, 0u};
    if (FP4) {
      const int srow = 2 * mi + kc, ky = srow - dy;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        int v = 0;
        if (e < C::SB) {
          const int tap = e / CIN, c = e % CIN, kx = tap - dx;
          if (ok && c < A.c_in && ky >= 0 && ky < K && kx >= 0 && kx < K) {
            const uint32_t wv = __ldg(A.wt + ((int64_t)o * K + ky) * K + kx);
            v = ((wv >> (31 - c)) & 1u) ? 1 : -1;
            if (f) v = -v;
          }
        } else {
          v = fp4_bias_part(bias, srow * (32 - C::SB) + (e - C::SB));
        }
        w4[e >> 3] |= e2m1_int(v) << (4 * (e & 7));
      }
    } else {
      const int srow = mi, ky = srow - dy;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int el = kc * 16 + e, tap = el / CIN, c = el % CIN, kx = tap - dx;
        int v = 0;
        if (ok && el < C::SB && c < A.c_in && ky >= 0 && ky < K && kx >= 0 && kx < K) {  // c >= c_in: zero (GRAY)
          const uint32_t wv = __ldg(A.wt + ((int64_t)o * K + ky) * K + kx);
          v = ((wv >> (31 - c)) & 1u) ? 1 : -1;
          if (f) v = -v;
        }
        if (REAL) {
          const int nb = -bias, q = (nb >= 0 ? nb + 127 : nb - 127) / 255, r = nb - 255 * q;
          if (srow == 0 && el == C::SB) v = r;
          if (srow == 0 && el == C::SB + 1) v = q;
        } else if (srow == 0 && el == C::SB) {
          v = bias;
        }
        w4[e >> 2] |= ((uint32_t)v & 0xFFu) << (8 * (e & 3));
      }
    }
    *reinterpret_cast<uint4*>(dst + ((size_t)(mi * 2 + kc) * N + n) * 16) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

template <int K, bool FP4>
__global__ void prep_first_tma_kernel(const ConvArgs A, uint8_t* out) {
  stage_b_first_tma<K, FP4>(A, blockIdx.x, out + (size_t)blockIdx.x * FirstTmaCfg<K, FP4>::B_BYTES, threadIdx.x, blockDim.x);
}

// Warp roles (no block-wide barrier in the tile loop; mbarriers carry every hand-off):
//   warp 0, one thread : TMA producer (raw box of tile it+NRAW-1 into the ring) and MMA issuer
//   warps 1-5          : builders (144 two-strip items of a tile)
//   warps 6-9          : epilogue (TMEM lane quarter warp % 4, all 32 channels of a pooled pixel)
// raw_full[s]   TMA complete_tx              -> builders          raw_empty[s] builders (5) -> producer
// a_full[b]     builders (5)                 -> MMA issuer        mma_done[b]  MMA commit   -> epilogue, builders (A[b] reuse)
// acc_empty[b]  epilogue (4)                 -> MMA issuer (one or two TMEM accumulator sets)
constexpr int kFirstTmaThreads = 320;

template <int K, bool FP4, bool DB = false, bool REAL = false>
__global__ void __launch_bounds__(kFirstTmaThreads, (FP4 || DB) ? 2 : 3)
conv_first_tma_pool_kernel(const ConvArgs A, const __grid_constant__ CUtensorMap xmap, const float* __restrict__ Tt) {
  griddep_launch();
  using C = FirstTmaCfg<K, FP4, DB>;
  constexpr int R = C::R, PW = C::PW, TH = C::TH, TW = C::TW, RAW_W = C::RAW_W;
  constexpr int KS = C::KS, N = C::N, NT = C::NT, CIN = C::CIN, NB = 5;  // builder warps
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sRaw = dsm;                                   // NRAW x RAW_STRIDE
  uint8_t* sA = sRaw + C::NRAW * C::RAW_STRIDE;          // 2 x A_BYTES: [chunk][strip row][px][16 B]
  uint8_t* sB = sA + 2 * C::A_BYTES;                     // [strip row][chunk][n][16 B]
  __shared__ int32_t s_bias[NT];  // thr' + 1 (for the debug acc output)
  __shared__ uint64_t raw_full[C::NRAW], raw_empty[C::NRAW], a_full[2], mma_done[2], acc_empty[2], w_bar, scale_bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int stride = gridDim.x, ntiles = (int)A.total_tiles;  // < 2^31 (host check)

  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < C::NRAW; ++i) {
      tc::mbar_init(&raw_full[i], 1);
      tc::mbar_init(&raw_empty[i], NB);
    }
    tc::mbar_init(&a_full[0], NB);
    tc::mbar_init(&a_full[1], NB);
    tc::mbar_init(&mma_done[0], 1);
    tc::mbar_init(&mma_done[1], 1);
    tc::mbar_init(&acc_empty[0], 4);
    tc::mbar_init(&acc_empty[1], 4);
    tc::mbar_init(&w_bar, 1);
    tc::mbar_init(&scale_bar, 4);
    tc::fence_mbar_init();
  }
  __syncthreads();

  auto tile_origin = [&](int tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };

  static_assert(!(REAL && FP4), "real u8 pixels need the int8 operand");
  if (tid < NT) s_bias[tid] = first_tma_bias<K, REAL>(A, g * NT + tid);
  if (A.bimg != nullptr) {
    if (tid == 0) tc::stage_image(sB, A.bimg + (size_t)g * C::B_BYTES, C::B_BYTES, &w_bar);
  } else {
    stage_b_first_tma<K, FP4, REAL>(A, g, sB, tid, kFirstTmaThreads);
  }
  griddep_wait();  // the image buffer and the output buffer belong to the predecessors' stream order
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ------------------------------------------------------------ producer + MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = FP4 ? tc::idesc_mxf4(128, N) : tc::idesc_i8(128, N, !REAL);  // REAL: u8 A
      const uint32_t sfa = tmem + N, sfb = tmem + N + 8;  // FP4 block scales (all 1.0)
      auto issue_raw = [&](int tile, int slot) {
        int img, oy0, ox0;
        tile_origin(tile, img, oy0, ox0);
        mbar_expect_tx(&raw_full[slot], C::RAW_BYTES);
        tma_load_3d(sRaw + slot * C::RAW_STRIDE, &xmap, ox0 * CIN - C::XOFF, oy0 - R, img, &raw_full[slot]);
      };
#pragma unroll 1
      for (int j = 0; j < C::NRAW - 1; ++j)
        if ((int)blockIdx.x + j * stride < ntiles) issue_raw(blockIdx.x + j * stride, j);
      if (A.bimg != nullptr) tc::mbar_wait(&w_bar, 0);  // weight image landed
      if (FP4) tc::mbar_wait(&scale_bar, 0);            // block scales written by the epilogue warps
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += stride, ++it) {
        const int buf = it & 1;
        if (tile + (C::NRAW - 1) * stride < ntiles) {
          const int slot2 = (it + C::NRAW - 1) % C::NRAW;  // last used by tile it-1
          if (it >= 1) tc::mbar_wait(&raw_empty[slot2], (uint32_t)(((it - 1) / C::NRAW) & 1));
          issue_raw(tile + (C::NRAW - 1) * stride, slot2);
        }
        tc::mbar_wait(&a_full[buf], (uint32_t)((it >> 1) & 1));         // strips of tile it staged
        trace_ev(A, it, 0);
        if (DB) {
          if (it >= 2) tc::mbar_wait(&acc_empty[buf], (uint32_t)(((it - 2) >> 1) & 1));  // tile it-2 drained
        } else if (it >= 1) {
          tc::mbar_wait(&acc_empty[0], (uint32_t)((it - 1) & 1));  // tile it-1 drained
        }
        const uint32_t d_tmem = tmem + (DB ? (uint32_t)(buf * N) : 0u);
        trace_ev(A, it, 1);
        tc::fence_after();
        // descriptors: base + constant start-address offsets (>> 4) -- no per-MMA descriptor arithmetic chain in
        // front of the MMA (tools/probes/issue_probe.cu)
        const uint32_t a0 = tc::smem_addr(sA + buf * C::A_BYTES), b0 = tc::smem_addr(sB);
        if (FP4) {
          // MMA p: strip rows 2p, 2p+1 (+ 2 * pooled row): LBO = one strip row, SBO = 2 strip rows
          const uint64_t ab = tc::desc_kmajor(a0, PW * 16, 2 * PW * 16), bb = tc::desc_kmajor(b0, N * 16, 128);
#pragma unroll
          for (int p = 0; p < C::NMMA; ++p)
            tc::mma_mxf4(d_tmem, ab + (uint64_t)((2 * p * PW * 16) >> 4), bb + (uint64_t)((p * 2 * N * 16) >> 4), idesc, sfa,
                         sfb, p > 0 ? 1u : 0u);
        } else {
          // MMA s: strip row s + 2 * (pooled row), both K chunks (LBO = one chunk plane, SBO = 2 strip rows)
          const uint64_t ab = tc::desc_kmajor(a0, C::PLANE, 2 * C::ROWP), bb = tc::desc_kmajor(b0, N * 16, 128);
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            if ((exp_bits(A) & 8) && s > 0) break;
            tc::mma_i8(d_tmem, ab + (uint64_t)((s * C::ROWP) >> 4), bb + (uint64_t)((s * 2 * N * 16) >> 4), idesc,
                       s > 0 ? 1u : 0u);
          }
        }
        tc::commit(&mma_done[buf]);
        trace_ev(A, it, 2);
      }
    }
    __syncwarp();
  } else if (warp <= NB) {
    // ------------------------------------------------------------ builders
    int t[CIN];
    bool zero_ok = true;  // an all-zero (out-of-image) byte thresholds to -1 for every channel
#pragma unroll
    for (int c = 0; c < CIN; ++c) {
      t[c] = (Tt != nullptr) ? u8_threshold(-Tt[c]) : 0;
      zero_ok = zero_ok && t[c] >= 0;
    }
    uint32_t E[3], O[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      E[m] = (uint32_t)(0x7FFF - t[m]) | ((uint32_t)(0x7FFF - t[(m + 2) % 3]) << 16);
      O[m] = (uint32_t)(0x7FFF - t[(m + 1) % 3]) | ((uint32_t)(0x7FFF - t[m]) << 16);
    }
    const int bt = tid - 32;  // item: strip row r = bt / 4, pooled columns 2j, 2j+1 with j = bt % 4
    const int r = bt >> 2, j = bt & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += stride, ++it) {
      const int buf = it & 1, slot = it % C::NRAW;
      wait_x(exp_bits(A), &raw_full[slot], (uint32_t)((it / C::NRAW) & 1));
      if (it >= 2) wait_x(exp_bits(A), &mma_done[buf], (uint32_t)(((it - 2) >> 1) & 1));  // A[buf] read by MMA(it-2)
      if (tid == 32) trace_ev(A, it, 12);
      if (bt < C::GROUPS && !(exp_bits(A) & 4)) {
        // 2 strips (pooled columns 2j, 2j+1) of strip row r: box bytes [DELTA + 12 j, + 6 + SB)
        constexpr int WB = C::DELTA - C::E;  // 4-byte aligned word base of item 0
        const uint32_t* src = reinterpret_cast<const uint32_t*>(sRaw + slot * C::RAW_STRIDE + r * RAW_W + WB + 12 * j);
        // M[w]: 0xFF where the byte is +1 (x > t_c, R14), 0x00 where -1
        uint32_t M[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) M[w] = REAL ? src[w] : thresh_mask4(src[w], E[(C::C0 + w) % 3], O[(C::C0 + w) % 3]);
        if (!REAL && !zero_ok) {  // out-of-image bytes must be -1 whatever the threshold (uniform branch)
          int img, oy0, ox0;
          tile_origin(tile, img, oy0, ox0);
          const int gy = oy0 - R + r;
          const bool row_ok = gy >= 0 && gy < A.H;
#pragma unroll
          for (int w = 0; w < 8; ++w)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int xb = ox0 * CIN - C::XOFF + WB + 12 * j + 4 * w + b;  // image row byte
              if (!row_ok || xb < 0 || xb >= A.W * CIN) M[w] &= ~(0xFFu << (8 * b));
            }
        }
        uint8_t* a = sA + buf * C::A_BYTES;
        if (FP4) {
          // bytes -> e2m1 nibbles (+1 = 0x2, -1 = 0xA): bit 3 of each byte's nibble = "is -1"
          uint32_t NW[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t h[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t x = ~M[2 * q + u] & 0x08080808u;
              h[u] = prmt(x | (x >> 4), 0u, 0x4420u);  // nibbles of bytes 0-3 in bits 0-15
            }
            NW[q] = prmt(h[0], h[1], 0x5410u) | 0x22222222u;
          }
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            constexpr int e0 = C::E;
            const int o = e0 + 6 * s, qw = o >> 3, sh = 4 * (o & 7);
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int w = qw + k;
              const uint32_t lo = w < 4 ? NW[w] : 0xAAAAAAAAu, hi = w + 1 < 4 ? NW[w + 1] : 0xAAAAAAAAu;
              v[k] = sh ? __funnelshift_r(lo, hi, sh) : lo;
              const int n0 = 8 * k;  // nibbles >= SB: -1 (bias slots)
              if (n0 >= C::SB) v[k] = 0xAAAAAAAAu;
              else if (n0 + 8 > C::SB) v[k] = (v[k] & ~(0xFFFFFFFFu << (4 * (C::SB - n0)))) | (0xAAAAAAAAu << (4 * (C::SB - n0)));
            }
            const int px = 2 * j + s;
            *reinterpret_cast<uint4*>(a + (size_t)(r * PW + px) * 16) = make_uint4(v[0], v[1], v[2], v[3]);
          }
        } else {
          uint32_t T[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) T[w] = REAL ? M[w] : (~M[w] | 0x01010101u);  // raw u8 / int8 +1 / -1
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            constexpr int e0 = C::E;
            const int o = e0 + 6 * s, qw = o >> 2, sh = 8 * (o & 3);
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int w = qw + k;
              const uint32_t lo = w < 8 ? T[w] : 0xFFFFFFFFu, hi = w + 1 < 8 ? T[w + 1] : 0xFFFFFFFFu;
              v[k] = sh ? __funnelshift_r(lo, hi, sh) : lo;
              // bytes >= SB of the strip: -1 (bias slots / unused K); REAL: 1, 255, then 0
              const int b0 = 4 * k;
              const uint32_t keep = b0 >= C::SB ? 0u : (b0 + 4 > C::SB ? 0xFFFFFFFFu >> (8 * (b0 + 4 - C::SB)) : 0xFFFFFFFFu);
              uint32_t pat = 0xFFFFFFFFu;
              if (REAL) {
                pat = 0u;
#pragma unroll
                for (int jb = 0; jb < 4; ++jb)
                  pat |= (b0 + jb == C::SB ? 0x01u : (b0 + jb == C::SB + 1 ? 0xFFu : 0u)) << (8 * jb);
              }
              v[k] = (v[k] & keep) | (pat & ~keep);
            }
            const int px = 2 * j + s;
            *reinterpret_cast<uint4*>(a + r * C::ROWP + px * 16) = make_uint4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<uint4*>(a + C::PLANE + r * C::ROWP + px * 16) = make_uint4(v[4], v[5], v[6], v[7]);
          }
        }
      }
      tc::fence_async_smem();  // generic-proxy strip writes -> the MMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        trace_ev(A, it, 2 + warp);  // builder warps 1-5 -> events 3-7
        tc::mbar_arrive(&a_full[buf]);
        tc::mbar_arrive(&raw_empty[slot]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int m_py = (quarter * 32 + lane) / PW, m_pxl = (quarter * 32 + lane) % PW;  // pooled pixel in the tile
    const int Ho = A.H >> 1, Wo = A.W >> 1;
    const int nvalid = min(32, A.c_out - g * NT);
    const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
    const int t_off = (m_py * Wo + m_pxl) * A.cwo + g;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    if (FP4) {  // block scales of the A (lanes = rows) and B operands: 1.0
      tc::tmem_st8_same(lane_base + (uint32_t)N, 0x7F7F7F7Fu);
      tc::tmem_st8_same(lane_base + (uint32_t)(N + 8), 0x7F7F7F7Fu);
      tc::tmem_st_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&scale_bar);
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += stride, ++it) {
      const int buf = it & 1;
      int img, oy0, ox0;
      tile_origin(tile, img, oy0, ox0);
      wait_x(exp_bits(A), &mma_done[buf], (uint32_t)((it >> 1) & 1));
      if (lane == 0) trace_ev(A, it, 2 + warp);  // epilogue warps 6-9 -> events 8-11
      __syncwarp();
      tc::fence_after();
      const uint32_t acc_base = lane_base + (DB ? (uint32_t)(buf * N) : 0u);
      const int py = (oy0 >> 1) + m_py, px = (ox0 >> 1) + m_pxl;
      const bool in = py < Ho && px < Wo;
      if (A.acc != nullptr) {  // debug output: the 4 window pixels' true sums
#pragma unroll 1
        for (int q = 0; q < 4; ++q)
#pragma unroll 1
          for (int cb = 0; cb < NT; cb += 16) {
            int vv[16];
            tc::tmem_ld16(acc_base + (uint32_t)(q * NT + cb), vv);
            tc::tmem_ld_wait();
            const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
            if (in && oy < A.H && ox < A.W) {
              int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT + cb;
              for (int c = 0; c < 16 && g * NT + cb + c < A.c_out; ++c) {
                const int o = g * NT + cb + c;
                const int a = (FP4 ? (int)__int_as_float(vv[c]) : vv[c]) + s_bias[cb + c];
                dst[c] = (A.flip != nullptr && A.flip[o] != 0) ? -a : a;
              }
            }
          }
      }
      uint32_t neg = 0, negp[4] = {0u, 0u, 0u, 0u};
      bool packed = false;
      if constexpr (!FP4 && !REAL) {
        // 16-bit packed drain: acc' = acc - thr' - 1 is in [-151, 151], so the low halves of the int32
        // accumulators are exact s16 values; .pack::16b loads two channels per register, VIMNMX3 /
        // VIMNMX .S16x2 take the 4-way pool max of two channels per instruction, and the sign bits
        // of 4 channels are gathered by one PRMT (bytes 1 / 3 hold them as bit 7) and one multiply
        // (bits 7, 15, 23, 31 -> 31..28, MSB-first) instead of one funnel shift per channel
        if (!(exp_bits(A) & 3)) {
          packed = true;
#pragma unroll
          for (int cb = 0; cb < NT; cb += 16) {
            uint32_t a[8], b[8], c[8], d[8];
            tc::tmem_ld8_p16(acc_base + (uint32_t)(0 * NT + cb), a);
            tc::tmem_ld8_p16(acc_base + (uint32_t)(1 * NT + cb), b);
            tc::tmem_ld8_p16(acc_base + (uint32_t)(2 * NT + cb), c);
            tc::tmem_ld8_p16(acc_base + (uint32_t)(3 * NT + cb), d);
            tc::tmem_ld_wait();
            uint32_t m[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) m[jj] = __vmaxs2(__vimax3_s16x2(a[jj], b[jj], c[jj]), d[jj]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t w = __byte_perm(m[2 * i], m[2 * i + 1], 0x1357);  // ch 4i+3, 4i+2, 4i+1, 4i
              const uint32_t y = (w & 0x80808080u) * 0x00204081u;              // signs -> bits 28..31
              neg |= (y >> 28) << (28 - cb - 4 * i);
            }
          }
        }
      }
      if (!packed && !(exp_bits(A) & 2))
#pragma unroll
      for (int cb = 0; cb < NT; cb += 16) {
        int a[16], b[16], c[16];
        if (exp_bits(A) & 1) {
          tc::tmem_ld16(acc_base + (uint32_t)(0 * NT + cb), a);
          tc::tmem_ld16(acc_base + (uint32_t)(1 * NT + cb), b);
          tc::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) neg = __funnelshift_l((uint32_t)__vimax3_s32(a[k], b[k], a[k] ^ k), neg, 1);
          continue;
        }
        tc::tmem_ld16(acc_base + (uint32_t)(0 * NT + cb), a);
        tc::tmem_ld16(acc_base + (uint32_t)(1 * NT + cb), b);
        tc::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = max(a[k], b[k]);
        tc::tmem_ld16(acc_base + (uint32_t)(2 * NT + cb), b);
        tc::tmem_ld16(acc_base + (uint32_t)(3 * NT + cb), c);
        tc::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // 4 independent 8-channel shift chains (ILP), merged below
          uint32_t& nk = negp[(cb + k) >> 3];
          nk = __funnelshift_l((uint32_t)__vimax3_s32(a[k], b[k], c[k]), nk, 1);
        }
      }
      if (!packed) neg = (negp[0] << 24) | (negp[1] << 16) | (negp[2] << 8) | negp[3];
      tc::fence_before();
      __syncwarp();
      if (tid == 6 * 32) trace_ev(A, it, 13);
      if (lane == 0) tc::mbar_arrive(&acc_empty[DB ? buf : 0]);  // TMEM may be overwritten by later MMAs
      if (A.y != nullptr && in)
        A.y[(((int64_t)img * Ho + (oy0 >> 1)) * Wo + (ox0 >> 1)) * A.cwo + t_off] = ~neg & vmask;
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

}  // namespace bnn
