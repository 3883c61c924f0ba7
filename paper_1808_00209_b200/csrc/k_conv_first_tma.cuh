// k_conv_first_tma.cuh -- pooled first conv layer on u8 RGB input with the THRESH_RGB binarization
// fused (Section 3.1 preprocessing, PAPER.md:141-145 / 178-179, then Eq. 3 + Eq. 1 + 2x2 pool,
// PAPER.md:212-218, 242-244), fed by TMA.
//
// Same MMA structure as conv_first_tc_pool_kernel (k_conv_first_tc.cuh: 128 pooled pixels per
// tile, strips of K taps x 3 channels as int8 +/-1, two parity planes, 4 accumulator blocks one per
// 2x2 pool offset), but every per-pixel instruction that kernel spent is gone or halved:
//   * the raw u8 halo box (IR rows x 80 B, starting 16 B left of the tile: the innermost TMA box
//     coordinate must be 16-byte aligned) is one cp.async.bulk.tensor per tile into a 3-deep ring;
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

template <int K, int NT>
struct FirstTmaCfg {
  static constexpr int CIN = 3, R = (K - 1) / 2, PH = 16, PW = 8, TH = 2 * PH, TW = 2 * PW;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1;
  // TMA needs a 16-byte aligned innermost box coordinate (measured: tools/probes/tma_probe.cu), so the
  // box starts XOFF = 16 bytes before the tile's first output column (ox0 * 3, a multiple of 48) and
  // strip x starts at box byte DELTA + 3x; the builders read aligned words from DELTA - E.
  static constexpr int XOFF = 16, DELTA = XOFF - 3 * R, E = DELTA & 3;
  static constexpr int C0 = (DELTA - E + 32 * 3 - XOFF) % 3;  // channel of box byte DELTA - E
  static constexpr int RAW_W = 80;  // box row bytes (>= DELTA + IC * 3 + 4; 80 B pitch spreads smem banks)
  static constexpr uint32_t RAW_BYTES = IR * RAW_W;
  static constexpr uint32_t RAW_STRIDE = (RAW_BYTES + 127) / 128 * 128;  // TMA destinations 128-B aligned
  static constexpr int NRAW = 3;
  static constexpr int S = K * CIN;
  static constexpr int NMMA = (K + 1) / 2;
  static constexpr int SRR = TH + 2 * NMMA - 1;  // strip rows per parity plane
  static constexpr uint32_t A_BYTES = 2 * SRR * PW * 16;
  static constexpr uint32_t B_BYTES = NMMA * 2 * NT * 16;
  static constexpr uint32_t TMEM_COLS = (4 * NT <= 128) ? 128 : 256;
  static constexpr int GROUPS = IR * (TW / 4);  // 4-strip work items
  static_assert(S < 16 && DELTA >= 0 && DELTA - E + 12 * (TW / 4 - 1) + 28 <= RAW_W && (TW * CIN) % 16 == 0 && TW % 4 == 0 && NT % 32 == 0 && NT <= 64, "config");
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

BNN_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          tc::smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tc::smem_addr(bar))
      : "memory");
}

BNN_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_addr(bar)), "r"(bytes) : "memory");
}

template <int K, int NT>
__global__ void __launch_bounds__(256, 4)
conv_first_tma_pool_kernel(const ConvArgs A, const __grid_constant__ CUtensorMap xmap, const float* __restrict__ Tt) {
  using C = FirstTmaCfg<K, NT>;
  constexpr int R = C::R, PW = C::PW, TH = C::TH, TW = C::TW, RAW_W = C::RAW_W;
  constexpr int NMMA = C::NMMA, SRR = C::SRR, CIN = C::CIN;
  __shared__ __align__(128) uint8_t sRaw[C::NRAW][C::RAW_STRIDE];
  __shared__ __align__(128) uint8_t sA[2][C::A_BYTES];
  __shared__ __align__(128) uint8_t sB[C::B_BYTES];
  __shared__ int32_t s_bias[NT];  // thr' + 1 (for the debug acc output)
  __shared__ uint32_t s_lut[16];
  __shared__ uint64_t raw_bar[C::NRAW], mma_bar[2];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int64_t stride = gridDim.x;
  constexpr int S_TOT = K * K * CIN;  // |acc| <= S_TOT

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

  if (tid < 16) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= (((tid >> (3 - k)) & 1) ? 0x01u : 0xFFu) << (8 * k);
    s_lut[tid] = v;
  }
  for (int i = tid; i < 2 * (int)C::A_BYTES / 16; i += 256) reinterpret_cast<uint4*>(&sA[0][0])[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < C::NRAW; ++i) tc::mbar_init(&raw_bar[i], 1);
    tc::mbar_init(&mma_bar[0], 1);
    tc::mbar_init(&mma_bar[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();

  auto tile_origin = [&](int64_t tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };
  auto issue_raw = [&](int64_t tile, int slot) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    mbar_expect_tx(&raw_bar[slot], C::RAW_BYTES);
    tma_load_3d(&sRaw[slot][0], &xmap, ox0 * CIN - C::XOFF, oy0 - R, img, &raw_bar[slot]);
  };
  if (tid == 0) {
    if (blockIdx.x < A.total_tiles) issue_raw(blockIdx.x, 0);
    if (blockIdx.x + stride < A.total_tiles) issue_raw(blockIdx.x + stride, 1);
  }

  // weights: int8 +/-1 (negated for flipped channels), bias thr'+1 in byte 15 of kernel rows 0 and 1
  for (int i = tid; i < NMMA * 2 * NT; i += 256) {
    const int n = i % NT, ky = i / NT;
    const int o = g * NT + n;
    const bool ok = o < A.c_out;
    const bool f = ok && A.flip != nullptr && A.flip[o] != 0;
    uint32_t bits = 0;
    if (ok && ky < K) {
#pragma unroll
      for (int kx = 0; kx < K; ++kx)
        bits |= (__ldg(A.wt + ((int64_t)o * K + ky) * K + kx) >> (32 - CIN)) << (32 - (kx + 1) * CIN);
    }
    uint32_t o4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t m = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) m |= ((4 * q + b < C::S && ok && ky < K) ? 0xFFu : 0u) << (8 * b);
      o4[q] = s_lut[(bits >> (28 - 4 * q)) & 0xFu] & m;
      if (f) o4[q] ^= m & 0xFEFEFEFEu;  // +1 <-> -1 on the valid bytes
    }
    // thr' = flip ? -t-1 : t, clamped to [-S_TOT-1, S_TOT] (same decisions: |acc| <= S_TOT)
    int tt = (ok && A.thr != nullptr) ? A.thr[o] : 0;
    tt = max(-S_TOT - 1, min(S_TOT, tt));
    if (f) tt = max(-S_TOT - 1, min(S_TOT, -tt - 1));
    const int v = ok ? tt + 1 : 1;  // invalid channels: acc' = -1 -> bit 0
    const int b0 = v / 2, b1 = v - v / 2;
    if (ky == 0) { o4[3] = (o4[3] & 0x00FFFFFFu) | ((uint32_t)(b0 & 0xFF) << 24); if (n < NT) s_bias[n] = v; }
    if (ky == 1) o4[3] = (o4[3] & 0x00FFFFFFu) | ((uint32_t)(b1 & 0xFF) << 24);
    *reinterpret_cast<uint4*>(sB + ((size_t)ky * NT + n) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_s;
  constexpr uint32_t idesc = tc::idesc_i8(128, NT, true);

  // 4 strips (columns 4j..4j+3) of strip row r from the raw row bytes [12j, 12j + 24)
  auto build = [&](int slot, int buf, int r, int j, int img, int oy0, int ox0) {
    // box byte b = image row byte ox0*3 - XOFF + b; strip x starts at box byte DELTA + 3x
    constexpr int WB = C::DELTA - C::E;  // 4-byte aligned word base of group 0
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&sRaw[slot][r * RAW_W + WB + 12 * j]);
    uint32_t T[7];
#pragma unroll
    for (int w = 0; w < 7; ++w) T[w] = thresh4(src[w], E[(C::C0 + w) % 3], O[(C::C0 + w) % 3]);
    if (!zero_ok) {  // out-of-image bytes must be -1 whatever the threshold (uniform branch)
      const int gy = oy0 - R + r;
      const bool row_ok = gy >= 0 && gy < A.H;
#pragma unroll
      for (int w = 0; w < 7; ++w)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int xb = ox0 * CIN - C::XOFF + WB + 12 * j + 4 * w + b;  // image row byte
          if (!row_ok || xb < 0 || xb >= A.W * CIN) T[w] |= 0xFFu << (8 * b);
        }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      constexpr int e = C::E;
      const int o = e + 3 * s, q = o >> 2, sh = 8 * (o & 3);
      uint32_t v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = sh ? __funnelshift_r(T[q + k], T[q + k + 1], sh) : T[q + k];
      const int x = 4 * j + s;
      *reinterpret_cast<uint4*>(&sA[buf][(size_t)(((x & 1) * SRR + r) * PW + (x >> 1)) * 16]) =
          make_uint4(v[0], v[1], v[2], v[3] | 0xFF000000u);
    }
  };

  // epilogue of one tile: warp w -> pooled pixels 32 (w % 4) .., channel half w / 4 of each 32
  const int quarter = warp & 3, half = warp >> 2;
  const int m_px = quarter * 32 + lane;  // pooled pixel of the tile this thread drains
  const int Ho = A.H >> 1, Wo = A.W >> 1;
  const int64_t t_off = ((int64_t)(m_px / PW) * Wo + m_px % PW) * A.cwo;
  auto epilogue = [&](int img, int oy0, int ox0, int buf, uint32_t phase) {
    __syncwarp();  // tcgen05.ld is .sync.aligned: the warp must be converged (warp 4 diverged in build)
    tc::mbar_wait(&mma_bar[buf], phase);
    __syncwarp();
    tc::fence_after();
    const int py = (oy0 >> 1) + m_px / PW, px = (ox0 >> 1) + m_px % PW;
    const bool in = py < Ho && px < Wo;
    uint32_t* ybase = A.y + (((int64_t)img * Ho + (oy0 >> 1)) * Wo + (ox0 >> 1)) * A.cwo + t_off;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
    for (int cb = 16 * half; cb < NT && ((g * NT + cb) >> 5) < A.cwo; cb += 32) {
      if (A.acc != nullptr) {  // debug output: the 4 window pixels' true sums
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          int vv[16];
          tc::tmem_ld16(lane_base + (uint32_t)(q * NT + cb), vv);
          tc::tmem_ld_wait();
          const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
          if (in && oy < A.H && ox < A.W) {
            int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT + cb;
            for (int c = 0; c < 16 && g * NT + cb + c < A.c_out; ++c) {
              const int o = g * NT + cb + c;
              const int a = vv[c] + s_bias[cb + c];
              dst[c] = (A.flip != nullptr && A.flip[o] != 0) ? -a : a;
            }
          }
        }
      }
      int a[16], b[16], c[16];
      tc::tmem_ld16(lane_base + (uint32_t)(0 * NT + cb), a);
      tc::tmem_ld16(lane_base + (uint32_t)(1 * NT + cb), b);
      tc::tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = max(a[k], b[k]);
      tc::tmem_ld16(lane_base + (uint32_t)(2 * NT + cb), b);
      tc::tmem_ld16(lane_base + (uint32_t)(3 * NT + cb), c);
      tc::tmem_ld_wait();
      uint32_t neg = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) neg = __funnelshift_l((uint32_t)__vimax3_s32(a[k], b[k], c[k]), neg, 1);
      const int valid = min(16, A.c_out - (g * NT + cb));
      uint32_t bits = ~neg & 0xFFFFu;
      bits &= valid >= 16 ? 0xFFFFu : (valid <= 0 ? 0u : (0xFFFFu << (16 - valid)) & 0xFFFFu);
      if (A.y != nullptr && in) {
        uint16_t* y16 = reinterpret_cast<uint16_t*>(ybase + ((g * NT + cb) >> 5));
        y16[((cb & 31) == 0) ? 1 : 0] = (uint16_t)bits;  // channels 0-15 = high half of the LE word
      }
    }
    tc::fence_before();
  };

  int it = 0;
  int64_t prev = -1;
  int p_img = 0, p_oy0 = 0, p_ox0 = 0;  // origin of the previous tile (drained this iteration)
  for (int64_t tile = blockIdx.x; tile < A.total_tiles; tile += stride, ++it) {
    const int buf = it & 1, slot = it % C::NRAW;
    if (tid == 0 && tile + 2 * stride < A.total_tiles) issue_raw(tile + 2 * stride, (it + 2) % C::NRAW);
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    if (tid < C::GROUPS) {
      tc::mbar_wait(&raw_bar[slot], (uint32_t)((it / C::NRAW) & 1));
      if (it >= 2) tc::mbar_wait(&mma_bar[buf], (uint32_t)(((it - 2) >> 1) & 1));
      build(slot, buf, tid >> 2, tid & 3, img, oy0, ox0);
      tc::fence_async_smem();
    }
    // single TMEM accumulator set: drain tile it-1 before tile it's MMAs
    if (prev >= 0) epilogue(p_img, p_oy0, p_ox0, buf ^ 1, (uint32_t)(((it - 1) >> 1) & 1));
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      const uint32_t a0 = tc::smem_addr(&sA[buf][0]), b0 = tc::smem_addr(sB);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int dy = q >> 1, dx = q & 1;
#pragma unroll
        for (int p = 0; p < NMMA; ++p) {
          const uint64_t ad = tc::desc_kmajor(a0 + (uint32_t)(((dx * SRR + dy + 2 * p) * PW) * 16), PW * 16, 2 * PW * 16);
          const uint64_t bd = tc::desc_kmajor(b0 + (uint32_t)(p * 2 * NT * 16), NT * 16, 128);
          tc::mma_i8(tmem + (uint32_t)(q * NT), ad, bd, idesc, p > 0 ? 1u : 0u);
        }
      }
      tc::commit(&mma_bar[buf]);
    }
    prev = tile;
    p_img = img; p_oy0 = oy0; p_ox0 = ox0;
  }
  if (prev >= 0) epilogue(p_img, p_oy0, p_ox0, (it - 1) & 1, (uint32_t)(((it - 1) >> 1) & 1));
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

}  // namespace bnn
