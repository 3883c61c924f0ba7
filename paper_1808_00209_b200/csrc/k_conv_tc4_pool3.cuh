// k_conv_tc4_pool3.cuh -- the pooled 32-channel binary conv (Eq. 3 + Eq. 1 + 2x2 max-pool, PAPER.md:212-218,
// 242-244; the vehicle conv2) with the pool window folded into the MMA N exactly as conv_tc4_pool_kernel
// (k_conv_tc4_pool.cuh: same weight image, same A layout, same start values C0 - (thr' + 1) and s16 drain),
// restructured as ONE CTA per SM with three TMEM accumulator sets.
//
// Why (tools/trace_conv2.py): with one accumulator per CTA (2 CTAs per SM) every tile's chain is
// MMAs -> commit -> drain + re-arm of the start values (~700 clk) -> release -> next MMAs, and the two CTAs'
// MMA phases did not cover each other's drains: 3,300 clk per CTA tile against 18 x 64 = 1,152 clk of MMA.
// Here the MMA thread runs up to two tiles ahead of the epilogue (sets it % 3), four A buffers let two loader
// groups (tile parity) expand one tile while the MMAs read another, so the tensor pipe sees back-to-back tiles.
//
// Roles (21 warps):
//   warp 0        : MMA issuer (one lane): 18 MMAs + 2 commits per tile
//   warps 1-8     : loaders, two groups of 4 (group = it % 2): the tile's input words (prefetched into registers
//                   one tile ahead) expanded to e2m1 through the LUT into A buffer it % 4
//   warps 9-20    : epilogue, three groups of 4 (group = accumulator set = it % 3; lane quarter = warp % 4)
// a_full[4]   loader group (4 warps) -> MMA       a_free[4]    MMA commit -> loaders (A buffer reuse)
// acc_full[3] MMA commit -> epilogue group        acc_empty[3] epilogue group (4 warps, start values re-armed)
//                                                              -> MMA
// PAIR (cta_group::2, (2, 1, 1) clusters): as in k_conv_tc4_pool.cuh -- rank r's tile is A rows [128 r, +128), it
// holds B columns [64 r, +64), the leader's thread issues M = 256 MMAs, a_full / acc_empty count both CTAs'
// arrivals, a_free / acc_full commits are multicast.
#pragma once
#include "k_conv_tc4_pool.cuh"

namespace bnn {

template <int K, bool PAIR = false>
struct ConvTc4Pool3Cfg {
  using P = ConvTc4PoolCfg<K, PAIR>;
#ifndef BNN_C2_NLG
#define BNN_C2_NLG 3
#endif
  static constexpr int NLG = BNN_C2_NLG;  // loader groups (tile % NLG): each prefetches its next tile one round ahead
  static constexpr int NA = NLG + 2, NACC = 3, NL = 4;  // A buffers, accumulator sets, warps per loader group
  static constexpr int NE = NACC;                          // epilogue groups of 4 warps
  static constexpr int THREADS = 32 * (1 + NLG * NL + 4 * NE);
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t SF_COL = NACC * P::N;  // block scales (all 1.0): SFA at SF_COL, SFB at SF_COL + 8
  static constexpr uint32_t SMEM = P::B_SMEM + NA * P::A_BYTES + 256 * 4 * (1 + P::LUTC) + P::NT * 4 + 64;
};

template <int K, bool PAIR = false>
__global__ void __launch_bounds__(ConvTc4Pool3Cfg<K, PAIR>::THREADS, 1)
conv_tc4_pool3_kernel(const ConvArgs A) {
  griddep_launch();
  using CF = ConvTc4Pool3Cfg<K, PAIR>;
  using C = typename CF::P;
  constexpr int R = C::R, PW = C::PW, TH = C::TH, TW = C::TW, IC = C::IC, NPIX = C::NPIX, KS = C::KS;
  constexpr int N = C::N, NT = C::NT, NL = CF::NL, NA = CF::NA, NACC = CF::NACC, NLG = CF::NLG, NE = CF::NE;
  constexpr int PF = (NPIX + NL * 32 - 1) / (NL * 32);
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sB = dsm;                                                   // [mma][K-chunk][N (or N/2)][16]
  uint8_t* sA = dsm + C::B_SMEM;                                       // NA x [plane][row][colhalf][16]
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(sA + NA * C::A_BYTES);  // 256 entries (weight staging)
  uint32_t* s_lutr = s_lut + 256;                                      // LUTC interleaved copies (loaders)
  float* s_init = reinterpret_cast<float*>(s_lutr + 256 * C::LUTC);    // C0 - (thr' + 1) per TMEM column
  __shared__ uint64_t a_full[NA], a_free[NA], acc_full[NACC], acc_empty[NACC], w_bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int ntiles = (int)A.total_tiles;  // < 2^31 - 1 (host check)
  const int rank = PAIR ? (int)tc::cluster_rank() : 0;
  const int first = PAIR ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int stride = PAIR ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int tile_end = PAIR ? ntiles + (ntiles & 1) : ntiles;  // a pair runs both halves of the last pair
  const int S_TOT = K * K * A.c_in;                            // |acc| <= S_TOT
  if (tid < 256) {
    fill_lut_fp4(s_lut, tid);
#pragma unroll
    for (int c = 0; c < C::LUTC; ++c) s_lutr[C::LUTC * tid + c] = s_lut[tid];
  }
  if (tid < NT) {
    const int o = g * NT + tc4_col_channel(tid);
    const bool ok = o < A.c_out;
    const bool f = ok && A.flip != nullptr && A.flip[o] != 0;
    int tt = (ok && A.thr != nullptr) ? A.thr[o] : 0;
    tt = max(-S_TOT - 1, min(S_TOT, tt));
    if (f) tt = max(-S_TOT - 1, min(S_TOT, -tt - 1));
    s_init[tid] = 12582912.0f - (float)(ok ? tt + 1 : 1);  // C0 - (thr' + 1), C0 = 1.5 * 2^23 (see k_conv_tc4_pool.cuh)
  }
  if (warp == 0) {
    if constexpr (PAIR) tc::tmem_alloc_pair<CF::TMEM_COLS>(&tmem_base_s);
    else tc::tmem_alloc<CF::TMEM_COLS>(&tmem_base_s);
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      tc::mbar_init(&a_full[i], PAIR ? 2 * NL : NL);
      tc::mbar_init(&a_free[i], 1);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], PAIR ? 8 : 4);
    }
    tc::mbar_init(&w_bar, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_s;

  // weight operand: this CTA's columns of the per-net image (or staged from the packed weights)
  if (PAIR || A.bimg != nullptr) {
    if (tid == 0) {
      constexpr uint32_t HB = (PAIR ? N / 2 : N) * 16;
      tc::mbar_arrive_expect_tx(&w_bar, C::B_SMEM);
      const uint8_t* src = A.bimg + (size_t)g * C::B_BYTES + rank * HB;
      for (int blk = 0; blk < C::NMMA * 2; ++blk) tc::bulk_g2s(sB + blk * HB, src + (size_t)blk * N * 16, HB, &w_bar);
      tc::mbar_wait(&w_bar, 0);
    }
  } else if (tid < 256) {
    stage_b_tc4_pool<K>(A, g, sB, s_lut, tid, 256);  // (s_lut is complete: filled before the barrier above)
  }
  // start values of all accumulator sets and the block scales (warps 1-4 cover the four TMEM lane quarters)
  if (warp >= 1 && warp <= 4) {
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t initv[16];
#pragma unroll
    for (int cb = 0; cb < NT; cb += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) initv[k] = __float_as_uint(s_init[cb + k]);
#pragma unroll
      for (int set = 0; set < NACC; ++set)
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(lb + (uint32_t)(set * N + q * NT + cb), initv);
    }
    tc::tmem_st8_same(lb + CF::SF_COL, 0x7F7F7F7Fu);
    tc::tmem_st8_same(lb + CF::SF_COL + 8, 0x7F7F7F7Fu);
    tc::tmem_st_wait();
  }
  griddep_wait();  // the input map is the predecessor's output; y is ordered after its readers
  tc::fence_async_smem();
  tc::fence_before();
  if constexpr (PAIR) tc::cluster_sync();
  else __syncthreads();
  tc::fence_after();

  auto tile_origin = [&](int tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };
  const int my_tiles = (tile_end - first + stride - 1) / stride;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (the leader's in a pair)
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = tc::idesc_mxf4(PAIR ? 256 : 128, N);
      constexpr uint32_t NB16 = (PAIR ? N / 2 : N) * 16;  // B: the CTA's N columns x 16 B per K chunk
      const uint32_t sfa = tmem + CF::SF_COL, sfb = tmem + CF::SF_COL + 8;
      // descriptors as base + constant start-address offsets (>> 4; no carry out of the 14-bit field below 256 KB):
      // recomputing desc_kmajor per MMA put a shift / mask / R2UR chain in front of every MMA and halved the issue
      // rate (tools/probes/issue_probe.cu: 128 vs 64 clk per MMA)
      const uint64_t adesc0 = tc::desc_kmajor(tc::smem_addr(sA), C::ROWB, 2 * C::ROWB);
      const uint64_t bdesc0 = tc::desc_kmajor(tc::smem_addr(sB), NB16, 128);
      const uint32_t a_full0 = tc::smem_addr(&a_full[0]), a_free0 = tc::smem_addr(&a_free[0]);
      const uint32_t acc_full0 = tc::smem_addr(&acc_full[0]), acc_empty0 = tc::smem_addr(&acc_empty[0]);
      // tile it is ready when its A buffer is built (a_full[it % NA], phase (it / NA) & 1) and its accumulator set has
      // been drained (acc_empty[it % 3], phase (it / 3 - 1) & 1)
#pragma unroll 1
      for (int it = 0; it < my_tiles; ++it) {
        const int ab = it % NA, cb = it % NACC;
        trace_ev(A, it, 0);
        tc::mbar_wait_at(a_full0 + 8 * ab, (uint32_t)((it / NA) & 1));
        trace_ev(A, it, 1);
        if (it >= NACC) tc::mbar_wait_at(acc_empty0 + 8 * cb, (uint32_t)((it / NACC - 1) & 1));
        trace_ev(A, it, 2);
        tc::fence_after();
        const uint64_t abuf = adesc0 + (uint64_t)(ab * (C::A_BYTES >> 4));
        const uint32_t d_tmem = tmem + (uint32_t)cb * N;
#pragma unroll
        for (int sp = 0; sp < C::SP; ++sp)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const uint64_t ad = abuf + (uint64_t)(((t & 1) * C::PLANE + (2 * sp) * C::ROWB + (t >> 1) * 16) >> 4);
            const uint64_t bd = bdesc0 + (uint64_t)(((sp * KS + t) * 2 * NB16) >> 4);
            if constexpr (PAIR) tc::mma_mxf4_pair(d_tmem, ad, bd, idesc, sfa, sfb, 1u);
            else tc::mma_mxf4(d_tmem, ad, bd, idesc, sfa, sfb, 1u);
          }
        if constexpr (PAIR) {
          tc::commit_pair(a_free0 + 8 * ab);
          tc::commit_pair(acc_full0 + 8 * cb);
        } else {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a_free0 + 8 * ab));
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_full0 + 8 * cb));
        }
        trace_ev(A, it, 3);
      }
    }
    __syncwarp();
  } else if (warp <= NLG * NL) {
    // ------------------------------------------------------------ loaders (group = tile parity)
    const int grp = (warp - 1) / NL, lt = tid - 32 - grp * NL * 32;
    const uint32_t a_full_leader = PAIR ? tc::mapa(tc::smem_addr(&a_full[0]), 0) : 0u;
    const uint32_t* my_lut = s_lutr + (lane & (C::LUTC - 1));
    uint32_t pref[PF];
    auto load = [&](int tile) {
      int img, oy0, ox0;
      tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
      const uint32_t* xin = A.x + (int64_t)img * A.H * A.W;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int p = lt + q * NL * 32;
        uint32_t w = 0u;  // outside the map: all -1 (R4)
        if (p < NPIX && tile < ntiles) {
          const int r = p / IC, c = p - r * IC;
          const int gy = oy0 - R + r, gx = ox0 - R + c;
          if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) w = __ldg(xin + (int64_t)gy * A.W + gx);
        }
        pref[q] = w;
      }
    };
    int it = grp;
    if (it < my_tiles) load(first + it * stride);
#pragma unroll 1
    for (; it < my_tiles; it += NLG) {
      const int ab = it % NA;
      if (it >= NA) tc::mbar_wait_sleep(&a_free[ab], (uint32_t)(((it / NA) - 1) & 1));  // A[ab] read by MMA(it - NA)
      if (lt == 0) trace_ev(A, it, 4);
      uint8_t* a = sA + ab * C::A_BYTES;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int p = lt + q * NL * 32;
        if (p < NPIX) {
          const int r = p / IC, c = p - r * IC;
          uint32_t o4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) o4[k] = my_lut[C::LUTC * ((pref[q] >> (24 - 8 * k)) & 0xFFu)];
          *reinterpret_cast<uint4*>(a + (c & 1) * C::PLANE + r * C::ROWB + (c >> 1) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(a_full_leader + 8 * ab);
        else tc::mbar_arrive(&a_full[ab]);
        if (lt == 0) trace_ev(A, it, 5);
      }
      if (it + NLG < my_tiles) load(first + (it + NLG) * stride);
    }
  } else {
    // ------------------------------------------------------------ epilogue (group = accumulator set)
    const int ew = warp - 1 - NLG * NL, grp = ew >> 2, quarter = warp & 3;
    const int m_py = (quarter * 32 + lane) / PW, m_pxl = (quarter * 32 + lane) % PW;
    const int Ho = A.H >> 1, Wo = A.W >> 1;
    const int nvalid = min(32, A.c_out - g * NT);
    const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
    const int t_off = (m_py * Wo + m_pxl) * A.cwo + g;
    const uint32_t acc_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * N);
    const uint32_t empty_bar = PAIR ? tc::mapa(tc::smem_addr(&acc_empty[grp]), 0) : tc::smem_addr(&acc_empty[grp]);
    static_assert(NT == 32, "two 16-column start-value blocks");
    uint32_t ph = 0;
#pragma unroll 1
    for (int it = grp; it < my_tiles; it += NE, ph ^= 1u) {
      const int tile = first + it * stride;
      int img, oy0, ox0;
      tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
      tc::mbar_wait_sleep(&acc_full[grp], ph);
      if (lane == 0 && quarter == 0) trace_ev(A, it, 6);
      __syncwarp();
      tc::fence_after();
      const int py = (oy0 >> 1) + m_py, px = (ox0 >> 1) + m_pxl;
      const bool in = py < Ho && px < Wo && tile < ntiles;
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
              int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT;
              for (int c = 0; c < 16; ++c) {
                const int oc = tc4_col_channel(cb + c), o = g * NT + oc;
                if (o >= A.c_out) continue;
                const int a = (int)(__int_as_float(vv[c]) - s_init[cb + c]);
                dst[oc] = (A.flip != nullptr && A.flip[o] != 0) ? -a : a;
              }
            }
          }
      }
      uint32_t a[16], b[16], c[16], d[16];
      tc::tmem_ld16_p16(acc_base + (uint32_t)(0 * NT), a);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(1 * NT), b);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(2 * NT), c);
      tc::tmem_ld16_p16(acc_base + (uint32_t)(3 * NT), d);
      tc::tmem_ld_wait();
#pragma unroll
      for (int cb = 0; cb < NT; cb += 16) {  // the set's start values for its next tile
        uint32_t iv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) iv[k] = __float_as_uint(s_init[cb + k]);
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(acc_base + (uint32_t)(q * NT + cb), iv);
      }
      tc::tmem_st_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(empty_bar);
        else tc::mbar_arrive_at(empty_bar);
        if (quarter == 0) trace_ev(A, it, 7);
      }
      // pooled bit = NOT(all four acc'_q < 0) (k_conv_tc4_pool.cuh)
      uint32_t neg = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint32_t x;
        asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(x) : "r"(a[j]), "r"(b[j]), "r"(c[j]));
        x = x & d[j] & 0x80008000u;
        neg = __umulhi(neg, 0x80000000u) + x;
      }
      if (A.y != nullptr && in)
        A.y[(((int64_t)img * Ho + (oy0 >> 1)) * Wo + (ox0 >> 1)) * A.cwo + t_off] = ~neg & vmask;
    }
  }
  if constexpr (PAIR) {
    tc::fence_before();
    tc::cluster_sync();
    if (warp == 0) tc::tmem_dealloc_pair<CF::TMEM_COLS>(tmem);
  } else {
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<CF::TMEM_COLS>(tmem);
  }
}

}  // namespace bnn
