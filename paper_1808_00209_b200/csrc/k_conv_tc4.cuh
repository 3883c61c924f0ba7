// k_conv_tc4.cuh -- binary convolution on the tensor cores with packed 4-bit operands
// (tcgen05.mma kind::mxf4, block-scaled e2m1, all scales 1.0).
//
// Same implicit GEMM as conv_tc_kernel (k_conv_tc.cuh) -- M = 128 output pixels (16 x 8), N = NT
// output channels, taps = descriptor offsets over a staged halo -- but +/-1 is stored as e2m1
// (+1.0 = 0x2, -1.0 = 0xA, pad channel 0.0 = 0x0), two per byte, so a 32-channel word of a pixel is
// 16 bytes (one K-chunk of a core matrix) and one MMA (K = 64) covers TWO taps: A row m takes its
// K-chunk 0 from tap u's pixel and its K-chunk 1 from tap u+1's pixel; the descriptor's LBO is just
// the distance between those two pixels in the halo (16 B for horizontal neighbours; validated
// with overlapping core matrices by tools/probes/mxf4_probe.cu).  The vehicle conv2 (K = 5,
// 32 channels) is 13 MMAs per 128 pixels instead of 25 int8 MMAs, and reads ~half the shared memory
// (the N = 32 MMAs are shared-memory-bound, 46 clk each either way).  Products of +/-1 with scale
// 1.0 summed in fp32 are exact integers (|acc| <= 2^24), so Eq. (3) stays bit-exact (R24).
#pragma once
#include "k_conv_tc.cuh"

namespace bnn {

template <int K, int CW, int NT>
struct ConvTc4Cfg {
  static constexpr int R = (K - 1) / 2, TH = 16, TW = 8;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1, NPIX = IR * IC, KK = K * K;
  static constexpr int U = CW * KK;            // 32-channel chunks (word j, tap t), j-major
  static constexpr int NMMA = (U + 1) / 2;     // two chunks per MMA
  static constexpr uint32_t A_BYTES = CW * NPIX * 16 + 256;  // + slack for the dummy chunk of odd U
  static constexpr uint32_t B_BYTES = NMMA * 2 * NT * 16;
  static constexpr uint32_t TMEM_COLS = (2 * NT + 16 <= 64) ? 64 : ((2 * NT + 16 <= 128) ? 128 : ((2 * NT + 16 <= 256) ? 256 : 512));
  static constexpr uint32_t SMEM = B_BYTES + 2 * A_BYTES + NT * 4 + 256 * 4 + 16;
};

// 8 channel bits (MSB = first channel) -> 8 e2m1 codes, two per byte, first channel in the low nibble
BNN_DEV void expand_word_fp4(uint32_t w, const uint32_t* lut256, uint32_t (&o)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = lut256[(w >> (24 - 8 * q)) & 0xFFu];
}

template <int K, int CW, int NT>
__global__ void __launch_bounds__(256, 3)
conv_tc4_kernel(const ConvArgs A) {
  using C = ConvTc4Cfg<K, CW, NT>;
  constexpr int R = C::R, TH = C::TH, TW = C::TW, IC = C::IC, NPIX = C::NPIX, KK = C::KK, U = C::U;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sB = dsm;                                           // [mma][chunk][NT][16]
  uint8_t* sA = dsm + C::B_BYTES;                              // 2 x [j][NPIX][16] (+ slack)
  float* s_thr = reinterpret_cast<float*>(sA + 2 * C::A_BYTES);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_thr + NT);  // 256 entries
  // warp roles: warps 4-7 expand the A halo (4 words / pixel -> e2m1) of tile it into A[it % 2], warp 4
  // lane 0 also issues the MMAs; warps 0-3 drain the accumulators of tile it from TMEM buffer it % 2.
  // a_full[b]: loaders (4) -> issuer; a_free[b]: commit -> loaders; acc_full[b]: commit -> epilogue;
  // acc_empty[b]: epilogue (4) -> issuer.  No block-wide barrier in the tile loop.
  __shared__ uint64_t a_full[2], a_free[2], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ uint32_t s_flip[NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  {
    uint32_t v = 0;  // tid = 8 channel bits
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((tid >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
    s_lut[tid] = v;
  }
  if (tid < NT) {
    const int o = g * NT + tid;
    // fp32 threshold: acc is an exact integer in fp32; thr clamped to +-2^24 keeps the compare exact
    const int t = (o < A.c_out && A.thr != nullptr) ? max(-(1 << 24), min(1 << 24, A.thr[o])) : 0;
    s_thr[tid] = (float)t;
  }
  if (warp < NT / 32) {
    const int o = g * NT + warp * 32 + lane;
    const uint32_t fm = ballot_pack(o < A.c_out && A.flip != nullptr && A.flip[o] != 0);
    if (lane == 0) s_flip[warp] = fm;
  }
  for (int i = tid; i < 2 * (int)C::A_BYTES / 16; i += 256) reinterpret_cast<uint4*>(sA)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&a_full[b], 4);
      tc::mbar_init(&a_free[b], 1);
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 4);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t tmem = tmem_base_s;
  const uint32_t sfa = tmem + 2 * NT, sfb = tmem + 2 * NT + 8;  // scale factors: all 1.0 (UE8M0 0x7F)
  if (warp < 4) {
    tc::tmem_st8_same(sfa + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st8_same(sfb + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st_wait();
  }
  // weights: chunk u = (j, t) j-major -> MMA u/2, K-chunk u%2; pad channels -> 0.0; dummy chunk -> 0
  for (int i = tid; i < C::NMMA * 2 * NT; i += 256) {
    const int n = i % NT, u = i / NT;
    const int o = g * NT + n;
    uint32_t o4[4] = {0u, 0u, 0u, 0u};
    if (u < U && o < A.c_out) {
      const int j = u / KK, t = u - j * KK;
      expand_word_fp4(__ldg(A.wt + ((int64_t)o * KK + t) * A.cw + j), s_lut, o4);
      const int valid = min(32, A.c_in - 32 * j);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t m = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) m |= (8 * q + e < valid ? 0xFu : 0u) << (4 * e);
        o4[q] &= m;
      }
    }
    *reinterpret_cast<uint4*>(sB + ((size_t)(u >> 1) * 2 + (u & 1)) * NT * 16 + n * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  constexpr uint32_t idesc = tc::idesc_mxf4(128, NT);

  auto tile_origin = [&](int64_t tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };
  auto epilogue = [&](int64_t tile, int buf, uint32_t phase) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    tc::mbar_wait_sleep(&acc_full[buf], phase);
    tc::fence_after();
    const int m = warp * 32 + lane;
    const int oy = oy0 + m / TW, ox = ox0 + m % TW;
    const bool in = oy < A.H && ox < A.W;
#pragma unroll 1
    for (int c0 = 0; c0 < NT && g * NT + c0 < A.c_out; c0 += 32) {
      int v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(buf * NT + c0), v);
      tc::tmem_ld_wait();
      uint32_t word = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) word = __funnelshift_l(__float_as_uint(s_thr[c0 + c] - __int_as_float(v[c])), word, 1);
      const int nvalid = A.c_out - (g * NT + c0);
      const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
      word = (word ^ s_flip[c0 / 32]) & vmask;
      if (A.acc != nullptr && in) {
        int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT + c0;
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nvalid) dst[c] = (int32_t)__int_as_float(v[c]);
      }
      const int wo = (g * NT + c0) >> 5;
      if (A.y != nullptr) {
        if (A.pool == 2) {
          uint32_t p = word | __shfl_xor_sync(BNN_FULL_MASK, word, 1);
          p |= __shfl_xor_sync(BNN_FULL_MASK, p, 8);
          const int Ho = A.H >> 1, Wo = A.W >> 1;
          if ((lane & 9) == 0 && (oy >> 1) < Ho && (ox >> 1) < Wo)
            A.y[(((int64_t)img * Ho + (oy >> 1)) * Wo + (ox >> 1)) * A.cwo + wo] = p;
        } else if (in) {
          A.y[(((int64_t)img * A.H + oy) * A.W + ox) * A.cwo + wo] = word;
        }
      }
    }
    tc::fence_before();
  };

  constexpr int PF = (CW * NPIX + 127) / 128;  // words per loader thread (warps 4-7)
  const int lt = tid - 128;
  uint32_t pref[PF];
  auto load_tile = [&](int64_t tile) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    const uint32_t* xin = A.x + (int64_t)img * A.H * A.W * A.cw;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = lt + q * 128;
      uint32_t w = 0u;  // outside the map: all -1 (R4)
      if (i < CW * NPIX) {
        const int p = i % NPIX, j = i / NPIX;
        const int r = p / IC, c = p - r * IC;
        const int gy = oy0 - R + r, gx = ox0 - R + c;
        if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) w = __ldg(xin + ((int64_t)gy * A.W + gx) * A.cw + j);
      }
      pref[q] = w;
    }
  };

  if (warp >= 4) {
    // ------------------------------------------------------------ loaders (+ MMA issuer: tid 128)
    if (blockIdx.x < A.total_tiles) load_tile(blockIdx.x);
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < A.total_tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      if (it >= 2) tc::mbar_wait_sleep(&a_free[buf], (uint32_t)(((it - 2) >> 1) & 1));  // A[buf] read by MMA(it-2)
      uint8_t* a = sA + buf * C::A_BYTES;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = lt + q * 128;
        if (i < CW * NPIX) {
          uint32_t o4[4];
          expand_word_fp4(pref[q], s_lut, o4);
          *reinterpret_cast<uint4*>(a + (size_t)i * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);  // [j][p]
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&a_full[buf]);
      if (tile + gridDim.x < A.total_tiles) load_tile(tile + gridDim.x);
      if (tid == 128) {
        tc::mbar_wait(&a_full[buf], (uint32_t)((it >> 1) & 1));
        if (it >= 2) tc::mbar_wait(&acc_empty[buf], (uint32_t)(((it - 2) >> 1) & 1));  // tile it-2 drained
        tc::fence_after();
        const uint64_t ad_base = tc::desc_kmajor(tc::smem_addr(a), 0, IC * 16), bd_base = tc::desc_kmajor(tc::smem_addr(sB), NT * 16, 128);
        const uint32_t d_tmem = tmem + (uint32_t)(buf * NT);
#pragma unroll
        for (int i = 0; i < C::NMMA; ++i) {
          // chunk u -> byte offset of its pixel for output pixel 0: plane j, halo (t / K, t % K)
          const int u0 = 2 * i, u1 = (2 * i + 1 < U) ? 2 * i + 1 : 2 * i;  // odd U: dummy (weights 0)
          const int off0 = ((u0 / KK) * NPIX + ((u0 % KK) / K) * IC + (u0 % KK) % K) * 16;
          const int off1 = ((u1 / KK) * NPIX + ((u1 % KK) / K) * IC + (u1 % KK) % K) * 16;
          const uint32_t lbo = (off1 > off0) ? (uint32_t)(off1 - off0) : 16u;
          // base descriptor (LBO 0) + constant start offset and LBO fields: no per-MMA descriptor arithmetic chain
          // in front of the MMA (tools/probes/issue_probe.cu)
          const uint64_t ad = ad_base + (uint64_t)(off0 >> 4) + ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16);
          const uint64_t bd = bd_base + (uint64_t)((i * 2 * NT * 16) >> 4);
          tc::mma_mxf4(d_tmem, ad, bd, idesc, sfa, sfb, i > 0 ? 1u : 0u);
        }
        tc::commit(&a_free[buf]);
        tc::commit(&acc_full[buf]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < A.total_tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      epilogue(tile, buf, (uint32_t)((it >> 1) & 1));
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[buf]);
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

}  // namespace bnn
