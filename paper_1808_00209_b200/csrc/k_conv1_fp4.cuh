// k_conv1_fp4.cuh -- the pooled first conv layer on a u8 3-channel image, binarized in the kernel
// (Section 2.3 preprocessing; Eq. 1 + Eq. 3 + 2x2 pool, PAPER.md:108-110,
// 212-218, 242-244), on tcgen05 kind::mxf4 with the activations as {0, 1} operands.
//
// Why this shape: the int8 TMA kernel (k_conv_first_tma.cuh) re-reads 8 KB of shared-
// memory operands per 128x128x32 MMA (6 per tile = 48 KB), i.e. the tensor core alone keeps the SM's
// 128 B/clk shared-memory path busy.  e2m1 operands halve the bytes per MAC and the MMA count (3 per
// tile, K = 64), and the whole SM runs ONE CTA with deep rings instead of 2 CTAs with 2 accumulators.
//
// Arithmetic (exact, R24): with x = 2b - 1 for the binarized input bit b in {0, 1} (b = 0 is also
// the -1 padding of R4 / R6),
//     acc_o = sum w x = sum (2w) b - S_o,        S_o = sum of the layer's weights of channel o,
// so A holds b (e2m1 0x2 = 1.0, 0x0 = 0.0), B holds 2w (0x4 / 0xC) and the constant -S_o - thr' - 1
// rides in B "bias slots" that A fills with 1.0.  TMEM then holds V_q = acc~_q - thr' - 1 for the
// four pool offsets q = (dy, dx) in N (B holds W shifted by q), and the pooled bit is
// max_q V_q >= 0 (thr' / flip folding as k_conv_first_tma.cuh, R23).  Every value is an integer with
// |V| <= 2 * 75 + 151.  Every tile's first MMA (constant operands, block scale 2^20) writes C0 = 1.5 * 2^23
// into the accumulators; fp32 holds every integer there and the tensor core's accumulation is exact
// (tools/probes/acc_probe.cu), so the low 16 bits of a result are V as an s16 and the epilogue drains two
// channels per register.
//
// Building A from the u8 bytes: the 16-bit-lane threshold gives per-byte masks (0xFF where x > t_c,
// R14); a strip of 18 bytes (6 taps x 3 channels) becomes 4 e2m1 words with two LOP per 8 bytes:
//     nibble word = (m[2w] & 0x02020202) | (m[2w+1] & 0x20202020)
// i.e. nibble 2k <- byte k of mask word 2w, nibble 2k+1 <- byte k of mask word 2w+1 (a fixed
// permutation of the strip's elements, strip_elem(); B uses the same one).
//
// Roles (20 warps, one CTA per SM, no block barrier in the tile loop; mbarriers carry every hand-off):
//   warp 0        : MMA issuer (all lanes loop; one elected lane issues 3 MMAs + 2 commits per tile on
//                   precomputed descriptors / barrier addresses -- with one CTA per SM this single-thread
//                   loop must stay short: measured 1,080 clk per tile when it also issued the TMA)
//   warp 1 lane 0 : TMA producer (raw box of tile it, up to NRAW tiles ahead)
//   warps 2-7     : builders, two groups of 3 (tile parity); item = (strip row, 4 pooled columns)
//   warps 8-19    : epilogue, three groups of 4 (group = accumulator set = tile % 3; lane quarter = warp % 4)
// raw_full[NRAW] TMA tx -> builders          raw_empty[NRAW] builder group (NB warps) -> producer
// a_full[NA]     builder group (NB) -> MMA   a_free[NA]      MMA commit -> builders (A buffer reuse)
// acc_full[NACC] MMA commit -> epilogue      acc_empty[NACC] epilogue group (4) -> MMA
#pragma once
#include <cuda.h>

#include "k_conv_first_tma.cuh"

namespace bnn {

template <int K>
struct Conv1Fp4Cfg {
  static constexpr int CIN = 3, NT = 32, R = (K - 1) / 2, PH = 16, PW = 8, TH = 2 * PH, TW = 2 * PW;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1;
  static constexpr int XOFF = 16, DELTA = XOFF - 3 * R;  // box byte of pooled column 0's strip
  static constexpr int WB = DELTA & ~3, E = DELTA & 3;  // item word base, strip 0 byte offset in it
  static constexpr int C0 = (WB - XOFF + 3 * 32) % 3;   // channel of box byte WB (box byte 16 = channel 0)
  static constexpr int RAW_W = 80;
  static constexpr uint32_t RAW_BYTES = IR * RAW_W;
  static constexpr uint32_t RAW_BYTES_LBP = (IR + 2) * RAW_W;  // kBinLbp box: one more row above and below
  static constexpr uint32_t RAW_STRIDE = (RAW_BYTES_LBP + 127) / 128 * 128;
  // kBinLbp per builder group: luma of box pixels k = 2 .. IC + 3 (LW columns) x IR + 2 rows, and the
  // synthetic box (IR rows x RAW_W bytes) of neighbour bits
  static constexpr int LW = IC + 2, LP = (LW + 3) / 4 * 4;
  static constexpr int KL0 = (XOFF / 3) - R - 1;  // box pixel k sits at box byte 1 + 3 k (image column ox0 - 5 + k)
  static_assert(XOFF == 16, "box pixel k <-> box byte 1 + 3 k, image column ox0 - 5 + k");
  static constexpr uint32_t LUMA_BYTES = (IR + 2) * LP, SYN_BYTES = IR * RAW_W;
  static constexpr uint32_t LBP_BYTES = 2 * (LUMA_BYTES + SYN_BYTES);
#ifndef BNN_C1_NRAW
#define BNN_C1_NRAW 8
#endif
  static constexpr int NRAW = BNN_C1_NRAW;  // raw-box ring depth (TMA loads in flight)
  static constexpr int KS = K + 1;     // strip rows of one pooled row's window (dy = 0, 1)
  static constexpr int SB = KS * CIN;  // data bytes of a strip (6 taps x 3 channels for K = 5)
  static constexpr int NWS = (SB + 3) / 4;                // mask words of a strip
  static constexpr int SPI = 4;                            // strips (pooled columns) per builder item
  static constexpr int NWI = (E + 6 * (SPI - 1) + SB + 3) / 4;  // mask words an item loads
  static constexpr int N = 4 * NT;
  static constexpr int NMMA = KS / 2;  // K = 64 e2m1 = 2 strip rows per MMA
  // strip-row pitch: one core matrix (8 strips x 16 B) + 16 B, so the quarter-warp STS.128 of rows
  // r and r+1 fall in different banks (LBO = ROWP, SBO = 2 ROWP; core matrices stay contiguous)
  static constexpr uint32_t ROWP = PW * 16 + 16;
  static constexpr uint32_t A_BYTES = IR * ROWP;
#ifndef BNN_C1_NA
#define BNN_C1_NA 4
#endif
#ifndef BNN_C1_NBG
#define BNN_C1_NBG 2
#endif
  static constexpr int NA = BNN_C1_NA;     // A buffers (power of 2)
  static constexpr int NBG = BNN_C1_NBG;   // builder groups (group = tile % NBG)
  static constexpr int NACC = 3;   // TMEM accumulator sets (3 x 128 columns + block scales)
  static constexpr uint32_t B_BYTES = NMMA * 2 * N * 16;
  static constexpr uint32_t TMEM_COLS = 512;
  // block scales: SFA at SF_COL and SFB at SF_COL + 8 (all 1.0); SFB of the offset MMA at SF_COL + 16 (2^20)
  static constexpr uint32_t SF_COL = NACC * N;
  // the offset MMA's constant operands: A = 1.0 everywhere (128 rows x 2 chunks), B = 6.0 at element 0 of
  // each 32-element block, scaled by 2^20: D = 2 * 6 * 2^20 = C0 = 1.5 * 2^23 in every accumulator
  static constexpr uint32_t CONST_BYTES = 2 * 2 * 128 * 16;
  static constexpr int GROUPS = IR * (PW / SPI);  // items per tile
  static constexpr int NB = (GROUPS + 31) / 32;    // builder warps per group (2 groups: tile parity)
  static constexpr int NE = NACC;                  // epilogue groups of 4 warps (group = accumulator set)
  static constexpr int THREADS = 32 * (2 + NBG * NB + 4 * NE);
#ifndef BNN_C1_TMA_W
#define BNN_C1_TMA_W 1
#endif
  // warp of the TMA producer (the builders take warps 1 .. 1 + NBG NB except it): 4 puts it on the MMA warp's SM
  // sub-partition (warp % 4 == 0) so that no ALU-heavy builder warp competes with the MMA thread for issue slots
  static constexpr int TMA_W = BNN_C1_TMA_W;
  static_assert(TMA_W >= 1 && TMA_W < 2 + NBG * NB, "TMA warp among the first 2 + NBG NB warps");
  static constexpr bool LDS64 = WB % 8 == 0 && (6 * SPI) % 8 == 0;  // item words 8-byte aligned: LDS.64
  static constexpr uint32_t SMEM = NRAW * RAW_STRIDE + NA * A_BYTES + B_BYTES + CONST_BYTES + LBP_BYTES + 1024;
  static_assert(KS % 2 == 0 && GROUPS <= NB * 32, "config");
  static_assert(WB + 4 * NWI + 6 * SPI * (PW / SPI - 1) <= RAW_W && E + 6 * (SPI - 1) + SB <= 4 * NWI,
                "item words inside the box row");
  static_assert(NWS <= 5, "strip <= 20 bytes");
};

// Element of strip row data carried by nibble n (0..31) of the e2m1 strip built by the kernel:
// >= 0 strip byte e (tap e / 3, channel e % 3), -1 a bias slot (A = 1.0), -2 unused (B = 0).
template <int SB>
__host__ __device__ constexpr int conv1_strip_elem(int n) {
  constexpr int nws = (SB + 3) / 4;
  const int w = n / 8, k = (n % 8) / 2, odd = n & 1;
  if (2 * w + 1 < nws) {
    const int e = 8 * w + (odd ? 4 + k : k);
    return e < SB ? e : -2;
  }
  if (2 * w < nws) {
    if (odd) return -1;
    const int e = 8 * w + k;
    return e < SB ? e : -2;
  }
  return -1;
}

// number of bias slots (A = 1.0) in one strip row
template <int SB>
__host__ __device__ constexpr int conv1_bias_slots() {
  int c = 0;
  for (int n = 0; n < 32; ++n) c += conv1_strip_elem<SB>(n) == -1 ? 1 : 0;
  return c;
}

// Output channel held by TMEM column c (0..31) of each pool-offset block: the epilogue ANDs the four offsets'
// sign bits of the s16 pair (c = 2j, 2j + 1) in register j and shifts them into one word with IMAD.HI, which
// leaves column 2j at bit j and column 2j + 1 at bit 16 + j; channel o must land on bit 31 - o (Eq. 2).
__host__ __device__ constexpr int conv1_col_channel(int c) { return (c & 1) ? 15 - (c >> 1) : 31 - (c >> 1); }

// thr' + 1 + S~_o (the bias the MMA subtracts) of output channel o; invalid channels: 1 (V = -1)
template <int K>
BNN_DEV int conv1_fp4_bias(const ConvArgs& A, int o) {
  if (o >= A.c_out) return 1;
  const bool f = A.flip != nullptr && A.flip[o] != 0;
  int s = 0;
  for (int t = 0; t < K * K; ++t) {
    const uint32_t wv = __ldg(A.wt + (int64_t)o * K * K + t);
    for (int c = 0; c < A.c_in && c < 3; ++c) s += ((wv >> (31 - c)) & 1u) ? 1 : -1;
  }
  if (f) s = -s;
  return first_tma_bias<K>(A, o) + s;
}

// The shared-memory image of B for channel group g: [mma p][K chunk kc][n = q * NT + o][16 B]; strip row
// s = 2p + kc, column n holds 2 w~[o][s - dy][t - dx] (q = (dy, dx)) at the data nibbles and the parts of
// -(thr' + 1 + S~_o) at the bias slots.  Written once per net (prep_conv1_fp4_kernel) or by the kernel.
template <int K>
BNN_DEV void stage_b_conv1_fp4(const ConvArgs& A, int g, uint8_t* dst, int i0, int step) {
  using C = Conv1Fp4Cfg<K>;
  constexpr int N = C::N, NT = C::NT, CIN = C::CIN, NSLOT = conv1_bias_slots<C::SB>();  // bias slots per strip row
  static_assert(NSLOT * C::KS * 6 >= 2 * K * K * CIN + 1, "bias slots must hold |thr' + 1 + S| <= 2 K^2 C + 1");
  for (int i = i0; i < C::NMMA * 2 * N; i += step) {
    const int n = i % N, kc = (i / N) & 1, p = i / (2 * N), s = 2 * p + kc;
    const int q = n / NT, o = g * NT + conv1_col_channel(n % NT), dy = q >> 1, dx = q & 1, ky = s - dy;
    const bool ok = o < A.c_out;
    const bool f = ok && A.flip != nullptr && A.flip[o] != 0;
    const int bias = -conv1_fp4_bias<K>(A, o);
    uint32_t w4[4] = {0u, 0u, 0u, 0u};
    int slot = s * NSLOT;  // running bias-slot index of this strip row
#pragma unroll
    for (int nb = 0; nb < 32; ++nb) {
      const int e = conv1_strip_elem<C::SB>(nb);
      int v = 0;
      if (e >= 0) {
        const int tap = e / CIN, c = e % CIN, kx = tap - dx;
        if (ok && c < A.c_in && ky >= 0 && ky < K && kx >= 0 && kx < K) {
          const uint32_t wv = __ldg(A.wt + ((int64_t)o * K + ky) * K + kx);
          v = ((wv >> (31 - c)) & 1u) ? 2 : -2;
          if (f) v = -v;
        }
      } else if (e == -1) {
        v = fp4_bias_part(bias, slot++);
      }
      w4[nb >> 3] |= e2m1_int(v) << (4 * (nb & 7));
    }
    *reinterpret_cast<uint4*>(dst + ((size_t)(p * 2 + kc) * N + n) * 16) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

template <int K>
__global__ void prep_conv1_fp4_kernel(const ConvArgs A, uint8_t* out) {
  stage_b_conv1_fp4<K>(A, blockIdx.x, out + (size_t)blockIdx.x * Conv1Fp4Cfg<K>::B_BYTES, threadIdx.x, blockDim.x);
}

// nibble word of a strip from its mask words (see the header): pairs, a single word, or bias only
template <int SB>
BNN_DEV void conv1_nibbles(const uint32_t (&m)[5], uint32_t (&v)[4]) {
  constexpr int nws = (SB + 3) / 4;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    if (2 * w + 1 < nws) v[w] = (m[2 * w] & 0x02020202u) | (m[2 * w + 1] & 0x20202020u);
    else if (2 * w < nws) v[w] = (m[2 * w] & 0x02020202u) | 0x20202020u;
    else v[w] = 0x22222222u;
  }
}

// Input binarization of the builders (Section 2.3):
//   kBinRgb  : per-channel thresholds, bit_c = x_c > t_c (THRESH_RGB / SIGN, and 0/1 images with t = 0)
//   kBinGray : THRESH_GRAY fused: Y = (299 R + 587 G + 114 B + 500) div 1000 (R15) from the raw RGB box,
//              bit = Y > t, i.e. 299 R + 587 G + 114 B >= 1000 (t + 1) - 500 (two DP2A per pixel); the
//              layer's c_in = 1 (channels 1, 2 of each strip tap carry zero weights)
//   kBinLbp  : LBP fused (R16): the box holds one extra row above and below; each builder group first
//              computes the luma of the box pixels (shared memory), then the three neighbour bits of every
//              tile pixel (replicate border) as 0xFF / 0x00 bytes in a synthetic box that the item build reads
constexpr int kBinRgb = 0, kBinGray = 1, kBinLbp = 2;

// PAIR (cta_group::2, (2, 1, 1) clusters, one CTA per SM): the two CTAs of a TPC run one M = 256 MMA per K
// step -- rank r's tile is A rows [128 r, 128 r + 128) and it holds B columns [64 r, 64 r + 64) (pool offsets
// 2r, 2r + 1) of the weight image and of the offset MMA's constant, so each SM reads 4 + 2 KB of operands
// per MMA instead of 4 + 4 KB, and the leader's (rank 0) single MMA thread issues once per two tiles.  Its
// a_full / acc_empty barriers count both CTAs' builders / epilogues (remote arrivals); a_free / acc_full
// commits are multicast to both CTAs.  Pair p runs tile pairs (2 t, 2 t + 1), t = p, p + npairs, ...; the
// second half of an odd last pair is built from tile 0's box and not stored.
template <int K, bool SPIN = false, int BIN = kBinRgb, bool PAIR = false>
__global__ void __launch_bounds__(Conv1Fp4Cfg<K>::THREADS, 1)
conv1_fp4_pool_kernel(const ConvArgs A, const __grid_constant__ CUtensorMap xmap, const float* __restrict__ Tt) {
  griddep_launch();
  using C = Conv1Fp4Cfg<K>;
  constexpr int R = C::R, PW = C::PW, TH = C::TH, TW = C::TW, RAW_W = C::RAW_W, N = C::N, NT = C::NT, IR_ = C::IR;
  constexpr int CIN = C::CIN, NB = C::NB, NA = C::NA, NACC = C::NACC, NRAW = C::NRAW, NE = C::NE;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sRaw = dsm;                           // NRAW x RAW_STRIDE
  uint8_t* sA = sRaw + NRAW * C::RAW_STRIDE;     // NA x A_BYTES: [strip row][px][16 B]
  uint8_t* sB = sA + NA * C::A_BYTES;            // B_BYTES
  uint8_t* sC = sB + C::B_BYTES;                 // CONST_BYTES: offset MMA's A, then its B
  uint8_t* sLbp = sC + C::CONST_BYTES;           // kBinLbp: per builder group [luma | synthetic box]
  __shared__ int32_t s_bias[NT];  // thr' + 1 (debug acc output)
  __shared__ uint64_t raw_full[NRAW], raw_empty[NRAW], a_full[NA], a_free[NA], acc_full[NACC], acc_empty[NACC];
  __shared__ uint64_t w_bar, scale_bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int ntiles = (int)A.total_tiles;
  // tile schedule: single CTA: blockIdx.x, + gridDim.x; pair: 2 t + rank over tile pairs t = pair, + npairs
  const int rank = PAIR ? (int)tc::cluster_rank() : 0;
  const int first = PAIR ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int stride = PAIR ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int tile_end = PAIR ? ntiles + (ntiles & 1) : ntiles;  // a pair runs both halves of the last pair

  if (warp == 0) {
    if constexpr (PAIR) tc::tmem_alloc_pair<C::TMEM_COLS>(&tmem_base_s);
    else tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NRAW; ++i) {
      tc::mbar_init(&raw_full[i], 1);
      tc::mbar_init(&raw_empty[i], NB);
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      tc::mbar_init(&a_full[i], PAIR ? 2 * NB : NB);
      tc::mbar_init(&a_free[i], 1);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], PAIR ? 8 : 4);  // the 4 warps of epilogue group i (of both CTAs)
    }
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

  if (tid < NT) s_bias[tid] = first_tma_bias<K>(A, g * NT + tid);
  if (PAIR) {  // this CTA's half of N of every (MMA, K chunk) block of the image (the host requires the image)
    if (tid == 0) {
      constexpr uint32_t HB = (N / 2) * 16;
      tc::mbar_arrive_expect_tx(&w_bar, C::B_BYTES / 2);
      const uint8_t* src = A.bimg + (size_t)g * C::B_BYTES + rank * HB;
      for (int blk = 0; blk < C::NMMA * 2; ++blk) tc::bulk_g2s(sB + blk * HB, src + (size_t)blk * N * 16, HB, &w_bar);
      tc::mbar_wait(&w_bar, 0);  // the leader's MMAs read this half after the cluster barrier below
    }
    if (warp < 4) {  // block scales of both CTAs before the cluster barrier (warp w: TMEM lanes 32 w ..)
      tc::fence_after();
      const uint32_t lb = tmem_base_s + ((uint32_t)(warp * 32) << 16);
      tc::tmem_st8_same(lb + C::SF_COL, 0x7F7F7F7Fu);
      tc::tmem_st8_same(lb + C::SF_COL + 8, 0x7F7F7F7Fu);
      tc::tmem_st8_same(lb + C::SF_COL + 16, 0x93939393u);  // 2^20
      tc::tmem_st_wait();
    }
  } else if (A.bimg != nullptr) {
    if (tid == 0) tc::stage_image(sB, A.bimg + (size_t)g * C::B_BYTES, C::B_BYTES, &w_bar);
  } else {
    stage_b_conv1_fp4<K>(A, g, sB, tid, C::THREADS);
  }
  for (int i = tid; i < (int)(C::CONST_BYTES / 16); i += C::THREADS) {
    const bool a_part = i < (int)(C::CONST_BYTES / 32);  // A: e2m1 1.0 everywhere; B: 6.0 at element 0 of a row chunk
    *reinterpret_cast<uint4*>(sC + 16 * i) = a_part ? make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u)
                                                    : make_uint4(0x7u, 0u, 0u, 0u);
  }
  griddep_wait();  // the image and output buffers belong to the predecessors' stream order
  tc::fence_async_smem();
  tc::fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // both CTAs' barriers, B halves and block scales are set
  else __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_s;

  const int my_tiles = (tile_end - first + stride - 1) / stride;
  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (converged warp, elected lane;
    // in a pair the leader issues for both CTAs)
    // (a whole-warp loop with elected-lane issue measured faster than a lane-0 loop unrolled over buffers / sets,
    // 0.537 vs 0.60 ms per 16384 images, and than waiting for tile it + 1 between tile it's MMAs, 0.60 ms)
    if (!PAIR || rank == 0) {
      constexpr uint32_t idesc = tc::idesc_mxf4(PAIR ? 256 : 128, N);
      constexpr uint32_t NB16 = (PAIR ? N / 2 : N) * 16;  // LBO of B: the CTA's N columns x 16 B
      const uint32_t sfa = tmem + C::SF_COL, sfb = tmem + C::SF_COL + 8, sfb_c = tmem + C::SF_COL + 16;
      const uint64_t adesc_c = tc::desc_kmajor(tc::smem_addr(sC), 128 * 16, 128);
      const uint64_t bdesc_c = tc::desc_kmajor(tc::smem_addr(sC) + C::CONST_BYTES / 2, NB16, 128);
      const uint32_t a_full0 = tc::smem_addr(&a_full[0]), a_free0 = tc::smem_addr(&a_free[0]);
      const uint32_t acc_full0 = tc::smem_addr(&acc_full[0]), acc_empty0 = tc::smem_addr(&acc_empty[0]);
      // strip rows 2p, 2p + 1 (+ 2 per pooled row): LBO = one strip row, SBO = two; buffer ab at + ab A_BYTES
      const uint64_t adesc0 = tc::desc_kmajor(tc::smem_addr(sA), C::ROWP, 2 * C::ROWP);
      uint64_t bdesc[C::NMMA];
#pragma unroll
      for (int p = 0; p < C::NMMA; ++p) bdesc[p] = tc::desc_kmajor(tc::smem_addr(sB) + (uint32_t)(p * 2 * NB16), NB16, 128);
      if (!PAIR) {
        if (A.bimg != nullptr) tc::mbar_wait(&w_bar, 0);
        tc::mbar_wait(&scale_bar, 0);  // block scales written by epilogue group 0
      }
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t sfb_, uint32_t acc) {
        if constexpr (PAIR) tc::mma_mxf4_pair_elect(d, ad, bd, idesc, sfa, sfb_, acc);
        else tc::mma_mxf4_elect(d, ad, bd, idesc, sfa, sfb_, acc);
      };
      uint32_t ab = 0, cb = 0, ph_full = 0, ph_empty = 0;
#pragma unroll 1
      for (int it = 0; it < my_tiles; ++it) {
        trace_ev(A, it, 0);
        tc::mbar_wait_at(a_full0 + 8 * ab, (ph_full >> ab) & 1u);
        ph_full ^= 1u << ab;
        trace_ev(A, it, 1);
        if (it >= NACC) {  // the set's previous tile has been drained
          tc::mbar_wait_at(acc_empty0 + 8 * cb, (ph_empty >> cb) & 1u);
          ph_empty ^= 1u << cb;
        }
        trace_ev(A, it, 2);
        tc::fence_after();
        const uint32_t d_tmem = tmem + cb * N;
        const uint64_t ad = adesc0 + (uint64_t)(ab * (C::A_BYTES >> 4));
        mma(d_tmem, adesc_c, bdesc_c, sfb_c, 0u);  // D = C0 (the offset MMA)
#pragma unroll
        for (int p = 0; p < C::NMMA; ++p) mma(d_tmem, ad + (uint64_t)(p * ((2 * C::ROWP) >> 4)), bdesc[p], sfb, 1u);
        if constexpr (PAIR) {
          tc::commit_pair_elect(a_free0 + 8 * ab);
          tc::commit_pair_elect(acc_full0 + 8 * cb);
        } else {
          tc::commit_elect(a_free0 + 8 * ab);
          tc::commit_elect(acc_full0 + 8 * cb);
        }
        trace_ev(A, it, 3);
        ab = (ab + 1) & (NA - 1);
        cb = (cb + 1 == NACC) ? 0 : cb + 1;
      }
    }
  } else if (warp == C::TMA_W) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t raw_full0 = tc::smem_addr(&raw_full[0]), raw_empty0 = tc::smem_addr(&raw_empty[0]);
      const uint32_t raw0 = tc::smem_addr(sRaw);
      uint32_t slot = 0, ph = 0;
#pragma unroll 1
      for (int it = 0; it < my_tiles; ++it) {
        if (it >= NRAW) {  // the slot's previous tile (it - NRAW) has been built
          tc::mbar_wait_at(raw_empty0 + 8 * slot, (ph >> slot) & 1u);
          ph ^= 1u << slot;
        }
        int img, oy0, ox0;
        const int tile = first + it * stride;
        tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);  // (an odd pair's empty half: any valid box)
        const uint32_t bar = raw_full0 + 8 * slot;
        constexpr uint32_t box_bytes = BIN == kBinLbp ? C::RAW_BYTES_LBP : C::RAW_BYTES;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(box_bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                raw0 + slot * C::RAW_STRIDE),
            "l"(reinterpret_cast<uint64_t>(&xmap)), "r"(ox0 * CIN - C::XOFF), "r"(oy0 - R - (BIN == kBinLbp ? 1 : 0)),
            "r"(img), "r"(bar)
            : "memory");
        slot = (slot + 1 == NRAW) ? 0 : slot + 1;
      }
    }
    __syncwarp();
  } else if (warp < 2 + C::NBG * NB) {
    // ------------------------------------------------------------ builders (group = tile parity)
    const int bw = C::TMA_W == 1 ? warp - 2 : (warp < C::TMA_W ? warp - 1 : warp - 2);  // builder warp index
    const int grp = bw / NB, bt = (bw - grp * NB) * 32 + lane;
    int t[CIN];
    bool zero_ok = true;  // an all-zero (out-of-image) byte thresholds to b = 0 (-1) for every channel
#pragma unroll
    for (int c = 0; c < CIN; ++c) {
      t[c] = (Tt != nullptr && (BIN == kBinRgb || c == 0)) ? u8_threshold(-Tt[c]) : 0;
      zero_ok = zero_ok && t[c] >= 0;
    }
    const int gray_lim = 1000 * (t[0] + 1) - 500;  // kBinGray: luma bit <=> s >= gray_lim (t in [-1, 255])
    uint32_t Ev[3], Od[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      Ev[m] = (uint32_t)(0x7FFF - t[m]) | ((uint32_t)(0x7FFF - t[(m + 2) % 3]) << 16);
      Od[m] = (uint32_t)(0x7FFF - t[(m + 1) % 3]) | ((uint32_t)(0x7FFF - t[m]) << 16);
    }
    constexpr int IPR = PW / C::SPI;  // items per strip row
    const int r = bt / IPR, j = bt % IPR;  // item: strip row r, pooled columns SPI j .. SPI j + SPI - 1
    const uint32_t item_off = (uint32_t)(r * RAW_W + C::WB + 6 * C::SPI * j);
    uint8_t* const a_item = sA + r * C::ROWP + C::SPI * j * 16;
    const uint32_t a_full_leader = PAIR ? tc::mapa(tc::smem_addr(&a_full[0]), 0) : 0u;
    int it = grp;
#pragma unroll 1
    for (int tile = first + grp * stride; tile < tile_end; tile += C::NBG * stride, it += C::NBG) {
      const int slot = it % NRAW, ab = it % NA;
      wait_x(SPIN ? 16 : 0, &raw_full[slot], (uint32_t)((it / NRAW) & 1));
      if (it >= NA) wait_x(SPIN ? 16 : 0, &a_free[ab], (uint32_t)(((it / NA) - 1) & 1));
      if (bt == 0) trace_ev(A, it, 4);
      const uint8_t* box = sRaw + slot * C::RAW_STRIDE;
      if constexpr (BIN == kBinLbp) {
        // phase 1: luma of box pixel (row rr, column k = kk + 2); box pixel k starts at box byte 1 + 3 k
        uint8_t* lum = sLbp + grp * (C::LUMA_BYTES + C::SYN_BYTES);
        uint8_t* syn = lum + C::LUMA_BYTES;
        for (int idx = bt; idx < (IR_ + 2) * C::LW; idx += NB * 32) {
          const int rr = idx / C::LW, kk = idx - rr * C::LW, k = kk + C::KL0;
          const uint8_t* p = box + rr * RAW_W + 1 + 3 * k;
          const uint32_t sy = 299u * p[0] + 587u * p[1] + 114u * p[2];
          lum[rr * C::LP + kk] = (uint8_t)((sy + 500u) / 1000u);  // R15
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NB * 32) : "memory");
        // phase 2: neighbour bits (R16: TL, R, BL; strict >; replicate border) of tile pixel (strip row r2,
        // column k = kk + 3), channel j at synthetic box byte 1 + 3 k + j; out-of-image pixels stay -1
        int img, oy0, ox0;
        tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
        for (int idx = bt; idx < IR_ * (C::LW - 2); idx += NB * 32) {
          const int r2 = idx / (C::LW - 2), kc = idx - r2 * (C::LW - 2) + 1, k = kc + C::KL0;
          const int gy = oy0 - R + r2, gx = ox0 - 5 + k;
          uint32_t b3 = 0u;
          if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) {
            const int rr = r2 + 1;
            const int ru = gy > 0 ? rr - 1 : rr, rd = gy + 1 < A.H ? rr + 1 : rr;
            const int kl = gx > 0 ? kc - 1 : kc, kr = gx + 1 < A.W ? kc + 1 : kc;
            const int y = lum[rr * C::LP + kc];
            b3 = (lum[ru * C::LP + kl] > y ? 0xFFu : 0u) | (lum[rr * C::LP + kr] > y ? 0xFF00u : 0u) |
                 (lum[rd * C::LP + kl] > y ? 0xFF0000u : 0u);
          }
          uint8_t* q = syn + r2 * RAW_W + 1 + 3 * k;
          q[0] = (uint8_t)b3;
          q[1] = (uint8_t)(b3 >> 8);
          q[2] = (uint8_t)(b3 >> 16);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NB * 32) : "memory");
      }
      if (bt < C::GROUPS && !(exp_bits(A) & 2)) {  // (diagnostics build: exp bit 2 skips the build)
        const uint8_t* src = (BIN == kBinLbp ? sLbp + grp * (C::LUMA_BYTES + C::SYN_BYTES) + C::LUMA_BYTES : box) + item_off;
        uint32_t X[C::NWI];
        if constexpr (C::LDS64) {
#pragma unroll
          for (int w = 0; w < C::NWI; w += 2) {
            const uint2 v = *reinterpret_cast<const uint2*>(src + 4 * w);
            X[w] = v.x;
            if (w + 1 < C::NWI) X[w + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int w = 0; w < C::NWI; ++w) X[w] = reinterpret_cast<const uint32_t*>(src)[w];
        }
        uint32_t M[C::NWI];  // 0xFF where the byte is b = 1 (x > t_c, R14)
        if constexpr (BIN == kBinLbp) {
#pragma unroll
          for (int w = 0; w < C::NWI; ++w) M[w] = X[w];  // the synthetic box holds the bits as bytes
        } else if constexpr (BIN == kBinRgb) {
#pragma unroll
          for (int w = 0; w < C::NWI; ++w) M[w] = thresh_mask4(X[w], Ev[(C::C0 + w) % 3], Od[(C::C0 + w) % 3]);
        } else {
          // pixel m of the item starts at item byte E + 3 m (a strip start is a pixel start); its channel-0
          // byte carries the luma bit, channels 1 and 2 stay 0 (zero weights)
          constexpr int NPIX_I = (6 * (C::SPI - 1) + C::SB) / 3;
#pragma unroll
          for (int w = 0; w < C::NWI; ++w) M[w] = 0u;
#pragma unroll
          for (int m = 0; m < NPIX_I; ++m) {
            const int i = C::E + 3 * m, wi = i >> 2, oi = i & 3;
            const uint32_t rgb = __byte_perm(X[wi], wi + 1 < C::NWI ? X[wi + 1] : 0u,
                                             (uint32_t)(oi | ((oi + 1) << 4) | ((oi + 2) << 8)));
            const uint32_t sy = __dp2a_hi(114u, rgb, __dp2a_lo((587u << 16) | 299u, rgb, 0u));  // 299R + 587G + 114B
            M[wi] |= ((int)sy >= gray_lim ? 0xFFu : 0u) << (8 * oi);
          }
        }
        if (BIN != kBinLbp && !zero_ok) {  // out-of-image bytes must be b = 0 whatever the threshold (uniform branch)
          int img, oy0, ox0;
          tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
          const int gy = oy0 - R + r;
          const bool row_ok = gy >= 0 && gy < A.H;
#pragma unroll
          for (int w = 0; w < C::NWI; ++w)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int xb = ox0 * CIN - C::XOFF + C::WB + 6 * C::SPI * j + 4 * w + b;  // image row byte
              if (!row_ok || xb < 0 || xb >= A.W * CIN) M[w] &= ~(0xFFu << (8 * b));
            }
        }
        uint8_t* a = a_item + ab * C::A_BYTES;
#pragma unroll
        for (int st = 0; st < C::SPI; ++st) {
          const int o = C::E + 6 * st, qw = o >> 2, sh = 8 * (o & 3);
          uint32_t m[5];
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int w = qw + k;
            const uint32_t lo = w < C::NWI ? M[w] : 0u, hi = w + 1 < C::NWI ? M[w + 1] : 0u;
            m[k] = (k < C::NWS) ? (sh ? __funnelshift_r(lo, hi, sh) : lo) : 0u;
          }
          uint32_t v[4];
          conv1_nibbles<C::SB>(m, v);
          *reinterpret_cast<uint4*>(a + st * 16) = make_uint4(v[0], v[1], v[2], v[3]);
        }
      }
      tc::fence_async_smem();  // generic-proxy strip writes -> the MMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        if (bt == 0) trace_ev(A, it, 5);
        if (bt == 32 * (NB - 1)) trace_ev(A, it, 6);
        if constexpr (PAIR) tc::mbar_arrive_cluster(a_full_leader + 8 * ab);
        else tc::mbar_arrive(&a_full[ab]);
        tc::mbar_arrive(&raw_empty[slot]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (group = accumulator set)
    const int ew = warp - 2 - C::NBG * NB, grp = ew >> 2, quarter = warp & 3;
    const int m_row = quarter * 32 + lane, m_py = m_row / PW, m_pxl = m_row % PW;  // pooled pixel of the tile
    const int Ho = A.H >> 1, Wo = A.W >> 1;
    const int nvalid = min(32, A.c_out - g * NT);
    const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t acc_base = lane_base + (uint32_t)(grp * N);  // this group's accumulator set
    const uint32_t empty_bar = PAIR ? tc::mapa(tc::smem_addr(&acc_empty[grp]), 0) : tc::smem_addr(&acc_empty[grp]);
    const bool want_acc = A.acc != nullptr;
    uint32_t* const ybase = A.y;
    if (!PAIR && grp == 0) {  // block scales of A (lanes = rows) and B: 1.0 (E8M0 127)
      tc::tmem_st8_same(lane_base + C::SF_COL, 0x7F7F7F7Fu);
      tc::tmem_st8_same(lane_base + C::SF_COL + 8, 0x7F7F7F7Fu);
      tc::tmem_st8_same(lane_base + C::SF_COL + 16, 0x93939393u);  // 2^20
      tc::tmem_st_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&scale_bar);
    }
    // every tile's first MMA writes C0 = 1.5 * 2^23 (the offset MMA): fp32 still holds every integer there and
    // the tensor core's accumulation is exact (tools/probes/acc_probe.cu), so the bit pattern of a result is
    // 0x4B400000 + V and its low 16 bits ARE V as an s16 (|V| <= 301): .pack::16b loads give 2 channels
    // per register and the pool max runs on s16 pairs
    constexpr uint32_t C0_BITS = 0x4B400000u;
    uint32_t ph = 0;
#pragma unroll 1
    for (int tile = first + grp * stride, it = grp; tile < tile_end; tile += NE * stride, it += NE, ph ^= 1u) {
      int img, oy0, ox0;
      tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
      const int py = (oy0 >> 1) + m_py, px = (ox0 >> 1) + m_pxl;
      const bool in = py < Ho && px < Wo && tile < ntiles;
      wait_x(SPIN ? 16 : 0, &acc_full[grp], ph);
      if (lane == 0 && quarter == 0) trace_ev(A, it, 7);
      __syncwarp();
      tc::fence_after();
      if (want_acc) {  // debug output: the 4 window pixels' true sums
#pragma unroll 1
        for (int q = 0; q < 4; ++q)
#pragma unroll 1
          for (int c0 = 0; c0 < NT; c0 += 16) {
            int vv[16];
            tc::tmem_ld16(acc_base + (uint32_t)(q * NT + c0), vv);
            tc::tmem_ld_wait();
            const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
            if (in && oy < A.H && ox < A.W) {
              int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT + c0;  // dst[oc - c0]
              for (int c = 0; c < 16; ++c) {  // TMEM column c0 + c holds channel conv1_col_channel(c0 + c)
                const int oc = conv1_col_channel(c0 + c), o = g * NT + oc;
                if (o >= A.c_out) continue;
                const int a = (vv[c] - (int)C0_BITS) + s_bias[oc];
                dst[oc - c0] = (A.flip != nullptr && A.flip[o] != 0) ? -a : a;
              }
            }
          }
      }
      if (exp_bits(A) & 1) {  // diagnostics build: exp bit 1 releases the set without draining it
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) tc::mbar_arrive_cluster(empty_bar);
          else tc::mbar_arrive_at(empty_bar);
        }
        continue;
      }
      uint32_t a[16], b[16], c[16], d[16];
      tc::tmem_ld16_p16(acc_base + (uint32_t)(0 * NT), a);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(1 * NT), b);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(2 * NT), c);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(3 * NT), d);
      tc::tmem_ld_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0 && quarter == 0) trace_ev(A, it, 8);
      if (lane == 0) {  // all values are in registers: the MMA may overwrite
        if (PAIR) tc::mbar_arrive_cluster(empty_bar);
        else tc::mbar_arrive_at(empty_bar);
      }
      // pooled bit = max_q V_q >= 0, i.e. NOT(all four V_q < 0): two LOP3 AND the sign bits (15, 31) of an s16
      // pair over the offsets and one LEA.HI, (neg >> 1) + x, shifts them into the word (3 ops per 2 channels);
      // the B column order (conv1_col_channel) makes the result MSB-first
      uint32_t neg = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint32_t x;
        asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(x) : "r"(a[j]), "r"(b[j]), "r"(c[j]));  // a & b & c
        x = x & d[j] & 0x80008000u;
        neg = __umulhi(neg, 0x80000000u) + x;  // (neg >> 1) + x: ptxas emits LEA.HI
      }
      if (ybase != nullptr && in) ybase[(((int64_t)img * Ho + py) * Wo + px) * A.cwo + g] = ~neg & vmask;
    }
  }
  if constexpr (PAIR) {
    tc::fence_before();
    tc::cluster_sync();  // the leader's last MMAs and commits touched this CTA's TMEM and barriers
    if (warp == 0) tc::tmem_dealloc_pair<C::TMEM_COLS>(tmem);
  } else {
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

}  // namespace bnn
