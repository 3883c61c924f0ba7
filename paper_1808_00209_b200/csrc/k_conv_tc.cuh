// k_conv_tc.cuh -- binary convolution on the 5th-generation tensor cores (tcgen05.mma kind::i8).
//
// Eq. (3) is a dense contraction over K*K*C_in +/-1 products, so besides the
// XOR-popcount integer path (Eq. 4) it can run as an int8 GEMM whose int32 result is exact
// (|acc| <= K*K*C_in << 2^31).  B200 has no binary (b1) tcgen05 kind, so bits are expanded in
// shared memory to int8 (+1 -> 0x01, -1 -> 0xFF; pad channels of the weights -> 0x00 so they add 0,
// out-of-map input words are 0 -> all -1 = the R4 padding).
//
// Implicit GEMM, no im2col: one CTA tile is M = 128 output pixels (16 rows x 8 columns) x
// N = NT output channels.  The expanded halo tile (16+K-1) x (8+K-1) pixels x 32 channels is laid
// out as two 16-channel planes of 16-byte pixel rows, which is exactly the SWIZZLE_NONE K-major
// UMMA layout: an 8-pixel output row is one 8 x 16 B core matrix, SBO = one halo row, LBO = one
// plane.  Tap (ky, kx) is just the descriptor start address moved by (ky * IC + kx) * 16 bytes,
// so the K*K*CW MMAs of a tile read the same staged halo.  Weights are expanded once per CTA.
// Accumulators live in TMEM (two buffers: the MMAs of tile i run while the epilogue of tile i-1
// reads the other buffer with tcgen05.ld); the epilogue is lane = pixel: 32 channel sums per
// thread -> threshold -> one packed word, 2x2 OR-pool with two shuffles.
#pragma once
#include "k_conv.cuh"
#include "tc.cuh"

namespace bnn {

template <int K, int CW, int NT>
struct ConvTcCfg {
  static constexpr int R = (K - 1) / 2, TH = 16, TW = 8;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1, NPIX = IR * IC, KK = K * K;
  static constexpr uint32_t A_BYTES = CW * 2 * NPIX * 16;
  static constexpr uint32_t B_BYTES = KK * CW * NT * 32;
  static constexpr uint32_t TMEM_COLS = (2 * NT <= 32) ? 32 : (2 * NT <= 64 ? 64 : (2 * NT <= 128 ? 128 : (2 * NT <= 256 ? 256 : 512)));
  static constexpr uint32_t SMEM = B_BYTES + 2 * A_BYTES + NT * 4 + 16 * 4 + 16;
};

// bits 31..0 of a packed word (channels 0..31, MSB first) -> 32 int8 (+1 / -1) as 8 u32, via a
// 16-entry nibble table in shared memory.
BNN_DEV void expand_word(uint32_t w, const uint32_t* lut, uint32_t (&o)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = lut[(w >> (28 - 4 * q)) & 0xFu];
}

// Epilogue of one 128-pixel tile (16 rows x 8 columns), run by warps 0-3: warp w owns TMEM lanes
// 32w..32w+31 = output pixels m of the tile.  Waits for the tile's MMAs, reads 32 channel sums at a
// time (tcgen05.ld 32x32b.x32), thresholds them into one packed word per pixel (Eq. 1 + Eq. 2),
// ORs 2x2 pixels for the fused pool (lanes m^1 and m^8 are the neighbours), stores.
// col_base: first TMEM column of the tile's accumulator; warp = TMEM lane quarter (0..3);
// (oy0, ox0): output origin of this 16 x 8 block.
template <int NT>
BNN_DEV void tc_epilogue(const ConvArgs& A, uint32_t tmem, uint32_t col_base, uint32_t phase, uint64_t* bar, int g,
                         int img, int oy0, int ox0, int warp, int lane, const int32_t* s_thr, const uint32_t* s_flip) {
  constexpr int TW = 8;
  tc::mbar_wait(bar, phase);
  tc::fence_after();
  const int m = warp * 32 + lane;  // TMEM lane = A row = output pixel of the tile
  const int oy = oy0 + m / TW, ox = ox0 + m % TW;
  const bool in = oy < A.H && ox < A.W;
#pragma unroll 1
  for (int c0 = 0; c0 < NT && g * NT + c0 < A.c_out; c0 += 32) {
    int v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + col_base + (uint32_t)c0, v);
    int th[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int4 t4 = reinterpret_cast<const int4*>(s_thr + c0)[q];
      th[4 * q] = t4.x; th[4 * q + 1] = t4.y; th[4 * q + 2] = t4.z; th[4 * q + 3] = t4.w;
    }
    tc::tmem_ld_wait();
    // bit_c = v_c > thr_c  <=>  thr_c - v_c < 0: shift the sign bits in, channel 0 ends at bit 31
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) word = __funnelshift_l((uint32_t)(th[c] - v[c]), word, 1);
    const int nvalid = A.c_out - (g * NT + c0);
    const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
    word = (word ^ s_flip[c0 / 32]) & vmask;
    if (A.acc != nullptr && in) {
      int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT + c0;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nvalid) dst[c] = v[c];
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
}

template <int K, int CW, int NT>
__global__ void __launch_bounds__(256, 3)
conv_tc_kernel(const ConvArgs A) {
  using C = ConvTcCfg<K, CW, NT>;
  constexpr int R = C::R, TH = C::TH, TW = C::TW, IC = C::IC, NPIX = C::NPIX, KK = C::KK;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sB = dsm;                                           // [t][j][sub][NT][16]
  uint8_t* sA = dsm + C::B_BYTES;                              // 2 x [j][sub][NPIX][16]
  int32_t* s_thr = reinterpret_cast<int32_t*>(sA + 2 * C::A_BYTES);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_thr + NT);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ uint32_t s_flip[NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;  // output-channel tile
  if (tid < 16) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= (((tid >> (3 - k)) & 1) ? 0x01u : 0xFFu) << (8 * k);
    s_lut[tid] = v;
  }
  if (tid < NT) {
    const int o = g * NT + tid;
    // clamped to +-2^30: |acc| <= 2^20 here, so thr - acc never overflows and the compare is unchanged
    s_thr[tid] = (o < A.c_out && A.thr != nullptr) ? max(-(1 << 30), min(1 << 30, A.thr[o])) : 0;
  }
  if (warp < NT / 32) {
    const int o = g * NT + warp * 32 + lane;
    const uint32_t fm = ballot_pack(o < A.c_out && A.flip != nullptr && A.flip[o] != 0);
    if (lane == 0) s_flip[warp] = fm;
  }
  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  // expand the CTA's weights once: B[t][j][sub][n] (pad channels of the last word -> 0)
  for (int i = tid; i < KK * CW * NT; i += 256) {
    const int n = i % NT, tj = i / NT;
    const int j = tj % CW, t = tj / CW;
    const int o = g * NT + n;
    uint32_t o8[8];
    const uint32_t w = (o < A.c_out) ? __ldg(A.wt + ((int64_t)o * KK + t) * A.cw + j) : 0u;
    expand_word(w, s_lut, o8);
    const int valid = min(32, A.c_in - 32 * j);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c0 = 4 * q;
      uint32_t m = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) m |= (c0 + b < valid ? 0xFFu : 0u) << (8 * b);
      o8[q] &= m;
    }
    uint4* dst0 = reinterpret_cast<uint4*>(sB + ((size_t)(t * CW + j) * 2 + 0) * NT * 16 + n * 16);
    uint4* dst1 = reinterpret_cast<uint4*>(sB + ((size_t)(t * CW + j) * 2 + 1) * NT * 16 + n * 16);
    *dst0 = make_uint4(o8[0], o8[1], o8[2], o8[3]);
    *dst1 = make_uint4(o8[4], o8[5], o8[6], o8[7]);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_s;
  constexpr uint32_t idesc = tc::idesc_i8(128, NT);

  auto tile_origin = [&](int64_t tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };

  auto epilogue = [&](int64_t tile, int buf, uint32_t phase) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    tc_epilogue<NT>(A, tmem, (uint32_t)(buf * NT), phase, &bar[buf], g, img, oy0, ox0, warp, lane, s_thr, s_flip);
  };

  // The packed input words of the next tile are loaded into registers (pref) right after the
  // MMAs of the current tile are issued, so their global latency hides behind the epilogue.
  constexpr int PF = (CW * NPIX + 255) / 256;
  uint32_t pref[PF];
  auto load_tile = [&](int64_t tile) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    const uint32_t* xin = A.x + (int64_t)img * A.H * A.W * A.cw;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = tid + q * 256;
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
  if (blockIdx.x < A.total_tiles) load_tile(blockIdx.x);

  int it = 0;
  int64_t prev = -1;
  for (int64_t tile = blockIdx.x; tile < A.total_tiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    if (it >= 2) tc::mbar_wait(&bar[buf], (uint32_t)(((it - 2) >> 1) & 1));  // A[buf] free again
    uint8_t* a = sA + buf * C::A_BYTES;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = tid + q * 256;
      if (i < CW * NPIX) {
        const int p = i % NPIX, j = i / NPIX;
        uint32_t o8[8];
        expand_word(pref[q], s_lut, o8);
        *reinterpret_cast<uint4*>(a + ((size_t)(j * 2 + 0) * NPIX + p) * 16) = make_uint4(o8[0], o8[1], o8[2], o8[3]);
        *reinterpret_cast<uint4*>(a + ((size_t)(j * 2 + 1) * NPIX + p) * 16) = make_uint4(o8[4], o8[5], o8[6], o8[7]);
      }
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 128) {  // warp 4 issues; warps 0-3 go straight to the previous tile's epilogue
      // descriptor start addresses advance in 16-byte units: compile-time offsets per (tap, word)
      const uint64_t ad0 = tc::desc_kmajor(tc::smem_addr(a), NPIX * 16, IC * 16);
      const uint64_t bd0 = tc::desc_kmajor(tc::smem_addr(sB), NT * 16, 128);
      const uint32_t d_tmem = tmem + (uint32_t)(buf * NT);
#pragma unroll
      for (int t = 0; t < KK; ++t) {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const uint64_t a_off = (uint64_t)((j * 2) * NPIX + (t / K) * IC + (t % K));
          const uint64_t b_off = (uint64_t)(((t * CW + j) * 2) * NT);
          tc::mma_i8(d_tmem, ad0 + a_off, bd0 + b_off, idesc, (t | j) ? 1u : 0u);
        }
      }
      tc::commit(&bar[buf]);
    }
    if (tile + gridDim.x < A.total_tiles) load_tile(tile + gridDim.x);
    if (prev >= 0 && warp < 4) epilogue(prev, buf ^ 1, (uint32_t)(((it - 1) >> 1) & 1));
    prev = tile;
  }
  if (prev >= 0 && warp < 4) epilogue(prev, (it - 1) & 1, (uint32_t)(((it - 1) >> 1) & 1));
  // drain: the other buffer's last commit may be unobserved by warps >= 4; wait before dealloc
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

}  // namespace bnn
