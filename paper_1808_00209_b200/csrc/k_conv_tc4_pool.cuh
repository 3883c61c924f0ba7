// k_conv_tc4_pool.cuh -- binary conv + threshold + 2x2 OR-pool on the tensor cores with the pool
// window folded into the MMA's N dimension (Eq. 3, Eq. 1, Section 3 max-pool; PAPER.md:212-218,
// 242-244, 327-330), for 32-channel packed inputs (the vehicle conv2 and CIFAR-like 32-channel maps).
//
// M = 128 POOLED pixels (16 x 8, a 32 x 16 conv region), N = 4 x 32: column q*32 + o is output
// channel o at pool offset q = (dy, dx), computed with the weights shifted by (dy, dx) over a
// (K+1) x (K+1) tap window.  A K-chunk is one (window row s, window column t) position = 32 input
// channels as 16 bytes of e2m1; for pooled pixel (pr, pc) it is the input pixel (2pr + s, 2pc + t),
// which sits in parity plane (t & 1) at column half pc + t/2, so 8 consecutive pooled columns are 8
// consecutive 16-byte rows (one core matrix), SBO = 2 input rows, and one MMA (K = 64) pairs window
// rows s and s+1 (LBO = one input row).  K = 5: 3 row pairs x 6 columns = 18 MMAs of N = 128 per
// 512 conv pixels, where the unpooled kernel (k_conv_tc4.cuh) needs 52 MMAs of N = 32 at the same
// ~46-64 cycle issue cost.
//
// Threshold and flip: flipped channels get negated weights (NOT(acc > t) == (-acc) > -t-1), and the
// accumulator is initialised to -(thr'+1) (tcgen05.st) before the first MMA of a tile, so TMEM ends
// with acc - thr' - 1 and the pooled bit is max_q(acc'_q) >= 0: a 4-way max (VIMNMX + VIMNMX3 on the
// fp32 bit patterns -- the integer order of IEEE bit patterns is correct about the sign) and one
// funnel shift per channel.  fp32 sums of +/-1 products and an integer start value are exact
// (|acc| <= 2^24, R24).  The epilogue runs on all 8 warps (pixel quarter x channel half) and stores
// 16 channel bits per pixel as one u16.
#pragma once
#include "k_conv_tc4.cuh"

namespace bnn {

template <int K, bool PAIR = false>
struct ConvTc4PoolCfg {
  static constexpr int R = (K - 1) / 2, PH = 16, PW = 8, TH = 2 * PH, TW = 2 * PW, NT = 32, N = 4 * NT;
  static constexpr int IR = TH + K - 1, IC = TW + K - 1, CH = (IC + 1) / 2, NPIX = IR * IC;
  static constexpr int KS = K + 1;                 // window rows / columns
  static constexpr int SP = KS / 2;                // row pairs per MMA column
  static constexpr int NMMA = SP * KS;
  // PLANE: one parity plane + 64 B, so a loader quarter-warp's 16-byte stores to the even (plane 0)
  // and odd (plane 1) columns of a row hit disjoint banks (an unpadded plane is a multiple of 128 B:
  // every STS.128 was a 2-way conflict, ncu)
  static constexpr uint32_t ROWB = CH * 16, PLANE = IR * ROWB + 64;
  static constexpr uint32_t A_BYTES = 2 * PLANE;
  static constexpr uint32_t B_BYTES = NMMA * 2 * N * 16;   // the weight image of one channel group
  static constexpr uint32_t B_SMEM = PAIR ? B_BYTES / 2 : B_BYTES;  // a CTA pair holds half of N per CTA
  static constexpr uint32_t TMEM_COLS = 256;       // N accumulator columns + block scales
  static constexpr int PF = (NPIX + 255) / 256;
  static constexpr int LUTC = 8;  // interleaved LUT copies (lane & 7): fewer bank conflicts in the loaders
  static constexpr uint32_t SMEM = B_SMEM + 2 * A_BYTES + 256 * 4 * (1 + LUTC) + NT * 4 + 64;
  static_assert(KS % 2 == 0 && PW + (KS - 1) / 2 <= CH, "window");
};

BNN_DEV void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// Output channel of TMEM column c (0..31) of each pool-offset block: the epilogue's LEA.HI shift leaves
// column 2j at bit j and column 2j + 1 at bit 16 + j of the packed word; channel o belongs at bit 31 - o.
__host__ __device__ constexpr int tc4_col_channel(int c) { return (c & 1) ? 15 - (c >> 1) : 31 - (c >> 1); }

// The shared-memory image of the weight operand for channel group g ([mma][K chunk][N][16 B]):
// MMA i = (row pair sp, window column t), K-chunk kc -> window row s = 2 sp + kc; column
// n = q * NT + o: W[o][s - dy][t - dx] as e2m1 (0 outside the kernel / pad channels), negated
// (+1 <-> -1 = nibble ^ 8) for flipped channels.  lut: the 256-entry bits -> e2m1 table.
template <int K>
BNN_DEV void stage_b_tc4_pool(const ConvArgs& A, int g, uint8_t* dst, const uint32_t* lut, int i0, int step) {
  using C = ConvTc4PoolCfg<K>;
  constexpr int N = C::N, NT = C::NT, KS = C::KS;
  for (int i = i0; i < C::NMMA * 2 * N; i += step) {
    const int n = i % N, kc = (i / N) & 1, mi = i / (2 * N);
    const int sp = mi / KS, t = mi % KS, s = 2 * sp + kc;
    const int q = n / NT, o = g * NT + tc4_col_channel(n % NT), dy = q >> 1, dx = q & 1;
    const int ky = s - dy, kx = t - dx;
    uint32_t o4[4] = {0u, 0u, 0u, 0u};
    if (o < A.c_out && ky >= 0 && ky < K && kx >= 0 && kx < K) {
      expand_word_fp4(__ldg(A.wt + ((int64_t)o * K + ky) * K + kx), lut, o4);
      const bool f = A.flip != nullptr && A.flip[o] != 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t m = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) m |= (8 * w + e < A.c_in ? 0xFu : 0u) << (4 * e);
        o4[w] &= m;
        if (f) o4[w] ^= m & 0x88888888u;
      }
    }
    *reinterpret_cast<uint4*>(dst + ((size_t)(mi * 2 + kc) * N + n) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
  }
}

BNN_DEV void fill_lut_fp4(uint32_t* lut, int tid) {
  uint32_t v = 0;  // tid = 8 channel bits -> 8 e2m1 codes (first channel low nibble)
#pragma unroll
  for (int k = 0; k < 8; ++k) v |= (((tid >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
  lut[tid] = v;
}

template <int K>
__global__ void __launch_bounds__(256) prep_tc4_pool_kernel(const ConvArgs A, uint8_t* out) {
  __shared__ uint32_t lut[256];
  fill_lut_fp4(lut, threadIdx.x);
  __syncthreads();
  stage_b_tc4_pool<K>(A, blockIdx.x, out + (size_t)blockIdx.x * ConvTc4PoolCfg<K>::B_BYTES, lut, threadIdx.x, 256);
}

// Warp roles (mbarrier hand-offs only, like conv_first_tma_pool_kernel):
//   warp 0, one thread : MMA issuer
//   warps 1-4          : loaders (global words of tile it+1 prefetched into registers, then
//                        expanded to e2m1 in the A buffer of tile it)
//   warps 5-8          : epilogue (TMEM lane quarter warp % 4, all 32 channels; re-arms the
//                        accumulator start values after draining)
// a_full[b]: loaders (4) -> issuer; mma_done[b]: commit -> epilogue, loaders (A[b] reuse);
// acc_empty: epilogue (4) -> issuer (single accumulator set).
//
// PAIR (cta_group::2, launched as (2, 1, 1) clusters): the two CTAs of a cluster sit on the two SMs of a TPC
// and run ONE M = 256 MMA per (row pair, column): rank r's 128 pooled pixels are A rows [128 r, 128 r + 128)
// and it holds B columns [64 r, 64 r + 64) (pool offsets 2r, 2r + 1) of the weight image at the same shared
// offsets, so each SM reads 4 KB of A + 2 KB of B per MMA instead of 4 + 4 KB (an N = 128 SS MMA is bound by
// the shared-memory operand path).  The leader (rank 0) issues every MMA and waits on its
// a_full (both CTAs' loaders arrive: 8) and acc_empty (both epilogues: 8); commits are multicast to the
// barriers of both CTAs; each TMEM holds its own 128 rows x all 128 columns, so the epilogue is unchanged.
// Pair p takes tile pairs (2 t, 2 t + 1), t = p, p + npairs, ...; a tile >= ntiles (odd count) is computed
// on zeros and not stored.
constexpr int kTc4PoolThreads = 288;

template <int K, bool PAIR = false>
__global__ void __launch_bounds__(kTc4PoolThreads, 2)
conv_tc4_pool_kernel(const ConvArgs A) {
  griddep_launch();
  using C = ConvTc4PoolCfg<K, PAIR>;
  constexpr int R = C::R, PW = C::PW, TH = C::TH, TW = C::TW, IC = C::IC, NPIX = C::NPIX, KS = C::KS;
  constexpr int N = C::N, NT = C::NT, NL = 4;  // loader warps
  constexpr int PF = (NPIX + NL * 32 - 1) / (NL * 32);
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sB = dsm;                                              // [mma][K-chunk][N][16]
  uint8_t* sA = dsm + C::B_SMEM;                                  // 2 x [plane][row][colhalf][16]
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(sA + 2 * C::A_BYTES);  // 256 entries (weight staging)
  uint32_t* s_lutr = s_lut + 256;                                      // LUTC interleaved copies (loaders)
  float* s_init = reinterpret_cast<float*>(s_lutr + 256 * C::LUTC);   // C0 - (thr' + 1) per TMEM column
  __shared__ uint64_t a_full[2], mma_done[2], acc_empty, w_bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int ntiles = (int)A.total_tiles;  // < 2^31 (host check)
  // tile schedule: single CTA: blockIdx.x, + gridDim.x; pair: 2 t + rank over tile pairs t = pair, + npairs
  const int rank = PAIR ? (int)tc::cluster_rank() : 0;
  const int first = PAIR ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int stride = PAIR ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int tile_end = PAIR ? ntiles + (ntiles & 1) : ntiles;  // a pair runs both halves of the last pair
  const int S_TOT = K * K * A.c_in;  // |acc| <= S_TOT
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
    // start value C0 - (thr' + 1), C0 = 1.5 * 2^23: the result's fp32 bit pattern is 0x4B400000 + acc' and its
    // low 16 bits are acc' as an s16 (exact: tools/probes/acc_probe.cu); invalid channels: acc' = -1 -> bit 0
    s_init[tid] = 12582912.0f - (float)(ok ? tt + 1 : 1);
  }
  if (warp == 0) {
    if constexpr (PAIR) tc::tmem_alloc_pair<C::TMEM_COLS>(&tmem_base_s);
    else tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  }
  if (tid == 0) {
    tc::mbar_init(&a_full[0], PAIR ? 2 * NL : NL);
    tc::mbar_init(&a_full[1], PAIR ? 2 * NL : NL);
    tc::mbar_init(&mma_done[0], 1);
    tc::mbar_init(&mma_done[1], 1);
    tc::mbar_init(&acc_empty, PAIR ? 8 : 4);
    tc::mbar_init(&w_bar, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t tmem = tmem_base_s;
  const uint32_t sfa = tmem + N, sfb = tmem + N + 8;  // block scales: all 1.0 (UE8M0 0x7F)

  if (PAIR) {  // this CTA's half of N of every (MMA, K chunk) block of the image (the host requires the image)
    if (tid == 0) {
      constexpr uint32_t HB = (N / 2) * 16;
      tc::mbar_arrive_expect_tx(&w_bar, C::B_SMEM);
      const uint8_t* src = A.bimg + (size_t)g * C::B_BYTES + rank * HB;
      for (int blk = 0; blk < C::NMMA * 2; ++blk) tc::bulk_g2s(sB + blk * HB, src + (size_t)blk * N * 16, HB, &w_bar);
      tc::mbar_wait(&w_bar, 0);  // the leader's MMAs read this CTA's half after the cluster barrier below
    }
  } else if (A.bimg != nullptr) {
    if (tid == 0) tc::stage_image(sB, A.bimg + (size_t)g * C::B_BYTES, C::B_BYTES, &w_bar);
  } else {
    if (tid < 256) stage_b_tc4_pool<K>(A, g, sB, s_lut, tid, 256);
  }
  // accumulator start values of the first tile and the block scales (epilogue warps 5-8 own
  // lane quarters 1, 2, 3, 0)
  if (warp >= 5) {
    const int quarter = warp & 3;
    const uint32_t lb = tmem + ((uint32_t)(quarter * 32) << 16);
    uint32_t initv[16];
#pragma unroll
    for (int cb = 0; cb < NT; cb += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) initv[k] = __float_as_uint(s_init[cb + k]);
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_st16(lb + (uint32_t)(q * NT + cb), initv);
    }
    tc::tmem_st8_same(sfa + ((uint32_t)(quarter * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st8_same(sfb + ((uint32_t)(quarter * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st_wait();
  }
  griddep_wait();  // the input map is the predecessor's output; y is ordered after its readers
  tc::fence_async_smem();
  tc::fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // both CTAs' barriers, B halves, start values and scales are set
  else __syncthreads();
  tc::fence_after();

  auto tile_origin = [&](int tile, int& img, int& oy0, int& ox0) {
    int ty, tx;
    tile_coords(A, tile, img, ty, tx);
    oy0 = ty * TH;
    ox0 = tx * TW;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = tc::idesc_mxf4(PAIR ? 256 : 128, N);
      constexpr uint32_t NB16 = (PAIR ? N / 2 : N) * 16;  // B: the CTA's N columns x 16 B per K chunk
      if (!PAIR && A.bimg != nullptr) tc::mbar_wait(&w_bar, 0);  // weight image landed
      int it = 0;
      for (int tile = first; tile < tile_end; tile += stride, ++it) {
        const int buf = it & 1;
        trace_ev(A, it, 0);
        if constexpr (PAIR) {
          tc::mbar_wait_cluster_at(tc::smem_addr(&a_full[buf]), (uint32_t)((it >> 1) & 1));
          trace_ev(A, it, 1);
          if (it >= 1) tc::mbar_wait_cluster_at(tc::smem_addr(&acc_empty), (uint32_t)((it - 1) & 1));
        } else {
          tc::mbar_wait(&a_full[buf], (uint32_t)((it >> 1) & 1));
          trace_ev(A, it, 1);
          if (it >= 1) tc::mbar_wait(&acc_empty, (uint32_t)((it - 1) & 1));  // drained and re-armed
        }
        trace_ev(A, it, 2);
        tc::fence_after();
        // (descriptors rebuilt per MMA: the base + constant-offset form that runs the issue probe and the other kernels
        // at the 64-clk floor made this 2-CTA/SM kernel slower in the bench step, 0.54 -> 0.79 ms per 16384 images)
        const uint32_t a0 = tc::smem_addr(sA + buf * C::A_BYTES), b0 = tc::smem_addr(sB);
#pragma unroll
        for (int sp = 0; sp < C::SP; ++sp)
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const uint32_t off = (uint32_t)((t & 1) * C::PLANE + (2 * sp) * C::ROWB + (t >> 1) * 16);
            const uint64_t ad = tc::desc_kmajor(a0 + off, C::ROWB, 2 * C::ROWB);
            const uint64_t bd = tc::desc_kmajor(b0 + (uint32_t)((sp * KS + t) * 2) * NB16, NB16, 128);
            if constexpr (PAIR) tc::mma_mxf4_pair(tmem, ad, bd, idesc, sfa, sfb, 1u);
            else tc::mma_mxf4(tmem, ad, bd, idesc, sfa, sfb, 1u);
          }
        if constexpr (PAIR) tc::commit_pair(tc::smem_addr(&mma_done[buf]));
        else tc::commit(&mma_done[buf]);
        trace_ev(A, it, 3);
      }
    }
    __syncwarp();
  } else if (warp <= NL) {
    // ------------------------------------------------------------ loaders
    const int lt = tid - 32;
    uint32_t pref[PF];
#define BNN_TC4P_LOAD(TILE)                                                                          \
  do {                                                                                               \
    int img_, oy0_, ox0_;                                                                            \
    tile_origin((TILE), img_, oy0_, ox0_);                                                           \
    const uint32_t* xin = A.x + (int64_t)img_ * A.H * A.W;                                           \
    _Pragma("unroll") for (int q = 0; q < PF; ++q) {                                                 \
      const int p = lt + q * NL * 32;                                                                \
      uint32_t w = 0u; /* outside the map: all -1 (R4) */                                            \
      if (p < NPIX && (TILE) < ntiles) {                                                             \
        const int r = p / IC, c = p - r * IC;                                                        \
        const int gy = oy0_ - R + r, gx = ox0_ - R + c;                                              \
        if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) w = __ldg(xin + (int64_t)gy * A.W + gx);     \
      }                                                                                              \
      pref[q] = w;                                                                                   \
    }                                                                                                \
  } while (0)
    const uint32_t a_full_leader = PAIR ? tc::mapa(tc::smem_addr(&a_full[0]), 0) : 0u;
    if (first < tile_end) BNN_TC4P_LOAD(first);
    int it = 0;
    for (int tile = first; tile < tile_end; tile += stride, ++it) {
      const int buf = it & 1;
      if (it >= 2) tc::mbar_wait_sleep(&mma_done[buf], (uint32_t)(((it - 2) >> 1) & 1));  // A[buf] read by MMA(it-2)
      if (lt == 0) trace_ev(A, it, 4);
      uint8_t* a = sA + buf * C::A_BYTES;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int p = lt + q * NL * 32;
        if (p < NPIX) {
          const int r = p / IC, c = p - r * IC;
          uint32_t o4[4];
          const uint32_t* my_lut = s_lutr + (lane & (C::LUTC - 1));
#pragma unroll
          for (int k = 0; k < 4; ++k) o4[k] = my_lut[C::LUTC * ((pref[q] >> (24 - 8 * k)) & 0xFFu)];
          *reinterpret_cast<uint4*>(a + (c & 1) * C::PLANE + r * C::ROWB + (c >> 1) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(a_full_leader + 8 * buf);
        else tc::mbar_arrive(&a_full[buf]);
        if (lt == 0) trace_ev(A, it, 5);
      }
      if (tile + stride < tile_end) BNN_TC4P_LOAD(tile + stride);
    }
#undef BNN_TC4P_LOAD
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int m_py = (quarter * 32 + lane) / PW, m_pxl = (quarter * 32 + lane) % PW;
    const int Ho = A.H >> 1, Wo = A.W >> 1;
    const int nvalid = min(32, A.c_out - g * NT);
    const uint32_t vmask = nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
    const int t_off = (m_py * Wo + m_pxl) * A.cwo + g;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    static_assert(NT == 32, "two 16-column start-value blocks");
    const uint32_t acc_empty_leader = PAIR ? tc::mapa(tc::smem_addr(&acc_empty), 0) : 0u;
    int it = 0;
    for (int tile = first; tile < tile_end; tile += stride, ++it) {
      const int buf = it & 1;
      int img, oy0, ox0;
      tile_origin(tile < ntiles ? tile : 0, img, oy0, ox0);
      tc::mbar_wait_sleep(&mma_done[buf], (uint32_t)((it >> 1) & 1));
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
            tc::tmem_ld16(lane_base + (uint32_t)(q * NT + cb), vv);
            tc::tmem_ld_wait();
            const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
            if (in && oy < A.H && ox < A.W) {
              int32_t* dst = A.acc + (((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * NT;
              for (int c = 0; c < 16; ++c) {  // TMEM column cb + c holds channel tc4_col_channel(cb + c)
                const int oc = tc4_col_channel(cb + c), o = g * NT + oc;
                if (o >= A.c_out) continue;
                const int a = (int)(__int_as_float(vv[c]) - s_init[cb + c]);
                dst[oc] = (A.flip != nullptr && A.flip[o] != 0) ? -a : a;
              }
            }
          }
      }
      // acc' of the 4 pool offsets as s16 pairs (low halves of C0 + acc', .pack::16b), then the next tile's
      // start values, then release: the MMA may run while the sign bits are gathered
      uint32_t a[16], b[16], c[16], d[16];
      tc::tmem_ld16_p16(lane_base + (uint32_t)(0 * NT), a);
      tc::tmem_ld16_p16(lane_base + (uint32_t)(1 * NT), b);
      tc::tmem_ld16_p16(lane_base + (uint32_t)(2 * NT), c);
      tc::tmem_ld16_p16(lane_base + (uint32_t)(3 * NT), d);
      tc::tmem_ld_wait();
#pragma unroll
      for (int cb = 0; cb < NT; cb += 16) {  // start values (broadcast shared loads: few live registers)
        uint32_t iv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) iv[k] = __float_as_uint(s_init[cb + k]);
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(lane_base + (uint32_t)(q * NT + cb), iv);
      }
      tc::tmem_st_wait();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(acc_empty_leader);
        else tc::mbar_arrive(&acc_empty);
        if (quarter == 0) trace_ev(A, it, 7);
      }
      // pooled bit = NOT(all four acc'_q < 0): two LOP3 AND the s16 sign bits, LEA.HI shifts them into the
      // word; the B column order (tc4_col_channel) makes it MSB-first
      uint32_t neg = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint32_t x;
        asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(x) : "r"(a[j]), "r"(b[j]), "r"(c[j]));  // a & b & c
        x = x & d[j] & 0x80008000u;
        neg = __umulhi(neg, 0x80000000u) + x;
      }
      if (A.y != nullptr && in)
        A.y[(((int64_t)img * Ho + (oy0 >> 1)) * Wo + (ox0 >> 1)) * A.cwo + t_off] = ~neg & vmask;
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
