// k_conv_tc4_big.cuh -- wide binary conv layers (many input-channel words, e.g. the CIFAR BinaryNet
// and the config-3 sweep) on the tensor cores, tcgen05.mma kind::mxf4 (packed e2m1, unit scales).
//
// Same implicit GEMM as conv_tc4_kernel (M = 128 output pixels = 16 x 8, taps = descriptor offsets,
// two taps per K = 64 MMA), but the K dimension K*K*C_in is streamed: a stage holds CG input words
// (32 CG channels) of the halo and the matching K*K x CG x NT weight chunks, both expanded from
// packed bits in shared memory; two stages ping-pong so the MMAs of stage s run while stage s + 1
// is expanded.  N = NT = 128 output channels per CTA (an MMA at N = 128 is compute-bound: 64 clk for
// 128 x 128 x 64 MACs, 16K MAC/clk/SM).  Accumulators are double-buffered in TMEM so the epilogue of
// tile i overlaps the MMAs of tile i + 1.
#pragma once
#include "k_conv_tc4.cuh"

namespace bnn {

// P = images per tile.  P = 2 serves maps exactly 8 wide (CIFAR conv5/6 at 8 x 8): the tile is 8 rows x
// (2 images x 8 columns), the two images' halos sit side by side in each halo row (ICI = 8 + K - 1
// columns each), so core-matrix group g = 2 r + h (row r, image h) starts at g * ICI * 16 bytes --
// the same linear SBO the P = 1 layout has -- and no tile rows are wasted on an 8 x 8 map.
template <int K, int CG, int NT, int P = 1>
struct ConvTc4BigCfg {
  static constexpr int R = (K - 1) / 2, TH = 16 / P, TW = 8;
  static constexpr int ICI = TW + K - 1;           // halo columns per image
  static constexpr int IR = TH + K - 1, IC = P * ICI, NPIX = IR * IC, KK = K * K;
  static constexpr int U = CG * KK;            // chunks per stage (word j, tap t), j-major
  static constexpr int NMMA = (U + 1) / 2;
  static constexpr uint32_t A_BYTES = CG * NPIX * 16 + 256;
  static constexpr uint32_t B_BYTES = NMMA * 2 * NT * 16;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = (2 * NT + 16 <= 64) ? 64 : ((2 * NT + 16 <= 128) ? 128 : ((2 * NT + 16 <= 256) ? 256 : 512));
  static constexpr uint32_t SMEM = 2 * STAGE_BYTES + NT * 4 + 256 * 4 + 16;
  static constexpr int PF = (CG * NPIX + 255) / 256;
};

// One stage's weight operand ([mma][K chunk][NT][16 B]) for channel group g, stage st: chunk
// u = (jl, t) -> MMA u / 2, K-chunk u % 2; pad channels, words >= cw, the dummy chunk -> 0.  All of a
// thread's weight words are loaded first (independent loads in flight), then expanded.
template <int K, int CG, int NT>
BNN_DEV void stage_b_tc4_big(const ConvArgs& A, int g, int st, uint8_t* b, const uint32_t* lut, int tid, int nthr) {
  using C = ConvTc4BigCfg<K, CG, NT>;
  constexpr int KK = C::KK, U = C::U;
  constexpr int PB = (C::NMMA * 2 * NT + 255) / 256;
  const int j0 = st * CG;
  for (int base = 0; base < C::NMMA * 2 * NT; base += PB * nthr) {
    uint32_t wv[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int i = base + tid + q * nthr;
      const int n = i % NT, u = i / NT;
      const int o = g * NT + n;
      wv[q] = 0u;
      if (i < C::NMMA * 2 * NT && u < U && o < A.c_out) {
        const int jl = u / KK, t = u - jl * KK, j = j0 + jl;
        if (j < A.cw) wv[q] = __ldg(A.wt + ((int64_t)o * KK + t) * A.cw + j);
      }
    }
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int i = base + tid + q * nthr;
      if (i >= C::NMMA * 2 * NT) break;
      const int n = i % NT, u = i / NT;
      uint32_t o4[4] = {0u, 0u, 0u, 0u};
      const int jl = u / KK, j = j0 + jl;
      const int o = g * NT + n;
      if (u < U && o < A.c_out && j < A.cw) {
        expand_word_fp4(wv[q], lut, o4);
        const int valid = min(32, A.c_in - 32 * j);
        if (valid < 32) {
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint32_t mk = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) mk |= (8 * qq + e < valid ? 0xFu : 0u) << (4 * e);
            o4[qq] &= mk;
          }
        }
      }
      *reinterpret_cast<uint4*>(b + ((size_t)(u >> 1) * 2 + (u & 1)) * NT * 16 + n * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
  }
}

// The whole layer's weight operand, stage by stage ([group][stage] x B_BYTES), built once per call
// so the conv kernel stages it with one bulk copy per stage instead of re-expanding it per tile.
template <int K, int CG, int NT>
__global__ void __launch_bounds__(256) prep_tc4_big_kernel(const ConvArgs A, uint8_t* out) {
  __shared__ uint32_t lut[256];
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((threadIdx.x >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
    lut[threadIdx.x] = v;
  }
  __syncthreads();
  const int st = blockIdx.x, g = blockIdx.y, nstage = gridDim.x;
  stage_b_tc4_big<K, CG, NT>(A, g, st, out + ((size_t)g * nstage + st) * ConvTc4BigCfg<K, CG, NT>::B_BYTES, lut,
                             threadIdx.x, 256);
}

template <int K, int CG, int NT, int P = 1>
__global__ void __launch_bounds__(256, 1)
conv_tc4_big_kernel(const ConvArgs A) {
  using C = ConvTc4BigCfg<K, CG, NT, P>;
  constexpr int R = C::R, TH = C::TH, TW = C::TW, IC = C::IC, ICI = C::ICI, NPIX = C::NPIX, KK = C::KK, U = C::U, PF = C::PF;
  extern __shared__ __align__(1024) uint8_t dsm[];
  float* s_thr = reinterpret_cast<float*>(dsm + 2 * C::STAGE_BYTES);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_thr + NT);
  __shared__ uint64_t bar_stage[2], bar_acc[2], w_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ uint32_t s_flip[NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((tid >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
    s_lut[tid] = v;
  }
  if (tid < NT) {
    const int o = g * NT + tid;
    const int t = (o < A.c_out && A.thr != nullptr) ? max(-(1 << 24), min(1 << 24, A.thr[o])) : 0;
    s_thr[tid] = (float)t;
  }
  if (warp < NT / 32) {
    const int o = g * NT + warp * 32 + lane;
    const uint32_t fm = ballot_pack(o < A.c_out && A.flip != nullptr && A.flip[o] != 0);
    if (lane == 0) s_flip[warp] = fm;
  }
  for (int i = tid; i < 2 * (int)C::STAGE_BYTES / 16; i += 256) reinterpret_cast<uint4*>(dsm)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar_stage[0], 1);
    tc::mbar_init(&bar_stage[1], 1);
    tc::mbar_init(&bar_acc[0], 1);
    tc::mbar_init(&bar_acc[1], 1);
    tc::mbar_init(&w_bar[0], 1);
    tc::mbar_init(&w_bar[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t tmem = tmem_base_s;
  const uint32_t sfa = tmem + 2 * NT, sfb = tmem + 2 * NT + 8;
  if (warp < 4) {
    tc::tmem_st8_same(sfa + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st8_same(sfb + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  constexpr uint32_t idesc = tc::idesc_mxf4(128, NT);
  const int nstage = (A.cw + CG - 1) / CG;

  auto tile_origin = [&](int64_t tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    img *= P;  // first image of the tile
    oy0 = ty * TH;
    ox0 = tx * TW;
  };
  auto epilogue = [&](int64_t tile, int buf, uint32_t phase) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    tc::mbar_wait(&bar_acc[buf], phase);
    tc::fence_after();
    const int m = warp * 32 + lane;
    const int grp = m / TW, ih = grp % P;  // core-matrix group = (row, image)
    img += ih;
    const int oy = oy0 + grp / P, ox = ox0 + m % TW;
    const bool in = oy < A.H && ox < A.W && img < A.n;
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
          p |= __shfl_xor_sync(BNN_FULL_MASK, p, 8 * P);  // the next output row of the same image
          const int Ho = A.H >> 1, Wo = A.W >> 1;
          if ((lane & (1 | 8 * P)) == 0 && img < A.n && (oy >> 1) < Ho && (ox >> 1) < Wo)
            A.y[(((int64_t)img * Ho + (oy >> 1)) * Wo + (ox >> 1)) * A.cwo + wo] = p;
        } else if (in) {
          A.y[(((int64_t)img * A.H + oy) * A.W + ox) * A.cwo + wo] = word;
        }
      }
    }
    tc::fence_before();
  };

  // A words of the next stage are loaded into registers one stage ahead (their global-load latency
  // overlaps the current stage's MMAs instead of stalling the expansion)
  uint32_t pref[PF];
  auto load_a = [&](int64_t tile, int st) {
    int img, oy0, ox0;
    tile_origin(tile, img, oy0, ox0);
    const uint32_t* xin = A.x + (int64_t)img * A.H * A.W * A.cw;
    const int j0 = st * CG;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = tid + q * 256;
      uint32_t w = 0u;  // outside the map / beyond c_in: -1 bits (weights there are 0 for words >= cw)
      if (i < CG * NPIX) {
        const int p = i % NPIX, jl = i / NPIX, j = j0 + jl;
        const int r = p / IC, cc = p - r * IC, ih = cc / ICI, c = cc - ih * ICI;
        const int gy = oy0 - R + r, gx = ox0 - R + c;
        if (j < A.cw && gy >= 0 && gy < A.H && gx >= 0 && gx < A.W && img + ih < A.n)
          w = __ldg(xin + ((int64_t)ih * A.H * A.W + (int64_t)gy * A.W + gx) * A.cw + j);
      }
      pref[q] = w;
    }
  };
  uint32_t stage_uses = 0;
  int it = 0;
  int64_t prev = -1;
  if ((int64_t)blockIdx.x < A.total_tiles) load_a(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < A.total_tiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    for (int st = 0; st < nstage; ++st, ++stage_uses) {
      const int s = stage_uses & 1;
      if (stage_uses >= 2) tc::mbar_wait(&bar_stage[s], ((stage_uses - 2) >> 1) & 1);
      uint8_t* a = dsm + s * C::STAGE_BYTES;
      uint8_t* b = a + C::A_BYTES;
      if (A.bimg != nullptr && tid == 0)
        tc::stage_image(b, A.bimg + ((size_t)g * nstage + st) * C::B_BYTES, C::B_BYTES, &w_bar[s]);
      // A: halo words j0 .. j0+CG-1 -> planes [jl][p] (16 B = 32 channels as e2m1)
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = tid + q * 256;
        if (i < CG * NPIX) {
          uint32_t o4[4];
          expand_word_fp4(pref[q], s_lut, o4);
          *reinterpret_cast<uint4*>(a + (size_t)i * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
      }
      if (st + 1 < nstage) load_a(tile, st + 1);
      else if (tile + (int64_t)gridDim.x < A.total_tiles) load_a(tile + gridDim.x, 0);
      if (A.bimg != nullptr) {
        // B: this stage's pre-expanded weight image, one bulk copy (issued before the A expansion)
      } else {
        stage_b_tc4_big<K, CG, NT>(A, g, st, b, s_lut, tid, 256);
      }
      tc::fence_async_smem();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      if (tid == 128) {
        if (A.bimg != nullptr) tc::mbar_wait(&w_bar[s], (stage_uses >> 1) & 1);  // weight stage landed
        const uint64_t ad_base = tc::desc_kmajor(tc::smem_addr(a), 0, ICI * 16), bd_base = tc::desc_kmajor(tc::smem_addr(b), NT * 16, 128);
        const uint32_t d_tmem = tmem + (uint32_t)(buf * NT);
#pragma unroll
        for (int i = 0; i < C::NMMA; ++i) {
          const int u0 = 2 * i, u1 = (2 * i + 1 < U) ? 2 * i + 1 : 2 * i;
          const int off0 = ((u0 / KK) * NPIX + ((u0 % KK) / K) * IC + (u0 % KK) % K) * 16;
          const int off1 = ((u1 / KK) * NPIX + ((u1 % KK) / K) * IC + (u1 % KK) % K) * 16;
          const uint32_t lbo = (off1 > off0) ? (uint32_t)(off1 - off0) : 16u;
          // base descriptor (LBO 0) + constant start offset and LBO fields: no per-MMA descriptor arithmetic chain
          // in front of the MMA (tools/probes/issue_probe.cu)
          const uint64_t ad = ad_base + (uint64_t)(off0 >> 4) + ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16);
          const uint64_t bd = bd_base + (uint64_t)((i * 2 * NT * 16) >> 4);
          tc::mma_mxf4(d_tmem, ad, bd, idesc, sfa, sfb, (st > 0 || i > 0) ? 1u : 0u);
        }
        tc::commit(&bar_stage[s]);
        if (st == nstage - 1) tc::commit(&bar_acc[buf]);
      }
      // the previous tile's epilogue overlaps this tile's first stage
      if (st == 0 && prev >= 0 && warp < 4) epilogue(prev, buf ^ 1, (uint32_t)(((it - 1) >> 1) & 1));
    }
    prev = tile;
  }
  if (prev >= 0 && warp < 4) epilogue(prev, (it - 1) & 1, (uint32_t)(((it - 1) >> 1) & 1));
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

}  // namespace bnn
