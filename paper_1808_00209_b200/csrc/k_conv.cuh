// k_conv.cuh -- direct (im2col-free) binary convolution on the integer pipe, fused with the
// Eq. (1) threshold, the Eq. (2) pack and an optional 2x2 OR max-pool.
//
// Eq. (3) with Eq. (4):
//   acc[n,y,x,o] = K*K*C_in - 2 * sum_{ky,kx,w} popc( X[n, y+ky-R, x+kx-R, w] ^ Wt[o, ky, kx, w] )
// Out-of-map words are 0 (= -1, R4); pad bits are 0 in both operands and contribute 0.
//
// Thread mapping ("lane = output channel"): a warp owns one group of 32 output channels
// and a PR x PC block of output pixels; every input word it needs is a warp-broadcast
// shared-memory read, every weight word a conflict-free per-lane read.  A thread keeps
// PR*PC accumulators and a register row of PC+K-1 input words, so each loaded word feeds
// up to K popcounts (and each weight word PR*PC).  The epilogue turns 32 lane-bits into
// one packed word with brev(ballot) -- the packed output for the next layer falls out
// of the warp directly -- and ORs 2x2 pixels for the fused max-pool.
//
// The paper's own design (Alg. 1 im2col with B = 25 + smem-tiled GEMM)
// is prior art: here the patch is never materialised; the halo tile is staged once in
// shared memory (zero-filled = -1 padding, the analogue of Alg. 1's zero-initialised
// sh_block) and the K x K taps are walked from registers.
#pragma once
#include "common.cuh"

namespace bnn {

struct ConvArgs {
  const uint32_t* x;   // packed [n, H, W, cw]
  const uint32_t* wt;  // packed [c_out, K, K, cw]
  const int32_t* thr;  // [c_out] or null
  const uint8_t* flip; // [c_out] or null
  uint32_t* y;         // packed [n, H/pool, W/pool, cwo] or null
  int32_t* acc;        // [n, H, W, c_out] or null
  int n, H, W, cw, c_in, c_out, cwo, pool;
  int tiles_x, tiles_y;
  int64_t total_tiles;  // < 2^31 (checked by the host)
  int tiles_per_cta;
  FastDiv fd_img, fd_tx;  // division by tiles_x * tiles_y and by tiles_x
  const uint8_t* bimg;    // pre-expanded shared-memory image of the weight operand (per channel group) or null
  int exp;                // timing-experiment bits (bnn_set_option "first_exp"; 0 in production: results exact)
  unsigned long long* trace;  // bnn_set_trace buffer (CTA (0,0) role timestamps) or null
  int trace_cap;
};

// Timing-experiment bits of the TMA first layer (bnn_set_option "first_exp"): compiled only into the
// diagnostics build (-DBNN_TRACE, libbnn_trace.so).  In libbnn.so this is the constant 0, so none of the
// experiment branches exist in the production kernel and no option can make it skip work.
template <typename Args>
BNN_DEV constexpr int exp_bits(const Args& A) {
#ifdef BNN_TRACE
  return A.exp;
#else
  return ((void)A, 0);
#endif
}

// Role timestamp of tile iteration `it`, event `ev` (< 16) of CTA (0, 0), SM clock (bnn_set_trace)
template <typename Args>
BNN_DEV void trace_ev(const Args& A, int it, int ev) {
#ifdef BNN_TRACE
  if (A.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && it * 16 + ev < A.trace_cap)
    A.trace[it * 16 + ev] = clock64();
#endif
}

// tile index -> (image, tile row, tile column), two multiply-high divisions
template <typename Args>
BNN_DEV void tile_coords(const Args& A, int64_t tile, int& img, int& ty, int& tx) {
  const uint32_t t = (uint32_t)tile;
  const uint32_t im = A.fd_img.div(t);
  const uint32_t rem = t - im * (uint32_t)(A.tiles_x * A.tiles_y);
  const uint32_t y = A.fd_tx.div(rem);
  img = (int)im;
  ty = (int)y;
  tx = (int)(rem - y * (uint32_t)A.tiles_x);
}

// Epilogue shared by the binary conv kernels: threshold + pack (+ OR-pool) + stores.
// a[r][p] holds the exact integer accumulator of output pixel (oy0+r, ox0+p), channel o.
template <int PR, int PC>
BNN_DEV void conv_epilogue(const ConvArgs& A, int img, int oy0, int ox0, int g, int lane, const int (&a)[PR][PC],
                           int t, bool f) {
  const int o = g * 32 + lane;
  const bool valid = o < A.c_out;
  uint32_t word[PR][PC];
#pragma unroll
  for (int r = 0; r < PR; ++r)
#pragma unroll
    for (int p = 0; p < PC; ++p) {
      const int oy = oy0 + r, ox = ox0 + p;
      if (A.acc != nullptr && valid && oy < A.H && ox < A.W)
        A.acc[(((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + o] = a[r][p];
      word[r][p] = ballot_pack(valid && ((a[r][p] > t) != f));
    }
  if (A.y == nullptr) return;
  if (A.pool == 2) {
    static_assert(PR % 2 == 0 && PC % 2 == 0, "pool needs even blocks");
    const int Ho = A.H >> 1, Wo = A.W >> 1;
#pragma unroll
    for (int r = 0; r < PR; r += 2)
#pragma unroll
      for (int p = 0; p < PC; p += 2) {
        const uint32_t pw = word[r][p] | word[r][p + 1] | word[r + 1][p] | word[r + 1][p + 1];
        const int q = (r / 2) * (PC / 2) + p / 2;
        const int py = (oy0 + r) >> 1, px = (ox0 + p) >> 1;
        if (lane == q && py < Ho && px < Wo) A.y[(((int64_t)img * Ho + py) * Wo + px) * A.cwo + g] = pw;
      }
  } else {
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) {
        const int q = r * PC + p;
        const int oy = oy0 + r, ox = ox0 + p;
        if (lane == q && oy < A.H && ox < A.W) A.y[(((int64_t)img * A.H + oy) * A.W + ox) * A.cwo + g] = word[r][p];
      }
  }
}

// Generic binary conv: one CTA = WY x WX warps = one group of 32 output channels
// (blockIdx.y) x a TH x TW output tile, TH = WY*PR, TW = WX*PC; the input words are
// walked in chunks of CWC words per pixel.  When the whole weight slab fits one chunk it is
// staged once and the CTA loops over tiles_per_cta consecutive tiles.
// Carry-save (Harley-Seal style) popcount of K words: full adders built from LOP3
// (sum = a ^ b ^ c, carry = maj(a, b, c)) compress the K XOR words of one kernel row before the
// POPC pipe (16 lanes/clk/SM) sees them; LOP3 issues at 64/clk/SM.  K = 5: 3 POPC + 6 LOP3 instead
// of 5 POPC; K = 3: 2 + 2 instead of 3; K = 7: 3 + 8 instead of 7.  The count is exactly sum popc(x).
BNN_DEV void full_add(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}
template <int K>
BNN_DEV int csa_popc(const uint32_t (&x)[K]) {
  if constexpr (K == 1) {
    return popc(x[0]);
  } else if constexpr (K == 3) {
    uint32_t s, c;
    full_add(x[0], x[1], x[2], s, c);
    return popc(s) + 2 * popc(c);
  } else if constexpr (K == 5) {
    uint32_t s1, c1, s2, c2;
    full_add(x[0], x[1], x[2], s1, c1);
    full_add(s1, x[3], x[4], s2, c2);
    return popc(s2) + 2 * popc(c1 ^ c2) + 4 * popc(c1 & c2);
  } else {
    static_assert(K == 7, "csa_popc: K in {1, 3, 5, 7}");
    uint32_t s1, c1, s2, c2, s3, c3, cs, cc;
    full_add(x[0], x[1], x[2], s1, c1);
    full_add(s1, x[3], x[4], s2, c2);
    full_add(s2, x[5], x[6], s3, c3);
    full_add(c1, c2, c3, cs, cc);
    return popc(s3) + 2 * popc(cs) + 4 * popc(cc);
  }
}

template <int K, int PR, int PC, int WY, int WX, int CWC, bool CSA = false>
__global__ void __launch_bounds__(WY * WX * 32)
conv_bin_kernel(const ConvArgs A) {
  constexpr int R = (K - 1) / 2;
  constexpr int KK = K * K;
  constexpr int TH = WY * PR, TW = WX * PC;
  constexpr int IR = TH + K - 1;
  constexpr int IC = TW + K - 1;
  constexpr int ICP = (IC + 3) & ~3;
  constexpr int NV = (PC + K - 1 + 3) / 4;  // uint4 loads per register row
  constexpr int NT = WY * WX * 32;

  __shared__ __align__(16) uint32_t in_s[CWC * IR * ICP];
  __shared__ __align__(16) uint32_t w_s[CWC * KK * 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WX, wx = warp % WX;
  const int g = blockIdx.y;
  const int o = g * 32 + lane;
  const bool ovalid = o < A.c_out;
  const int thr_o = (A.thr != nullptr && ovalid) ? A.thr[o] : 0;
  const bool flip_o = (A.flip != nullptr && ovalid) ? (A.flip[o] != 0) : false;
  const int nbits = KK * A.c_in;
  const bool single = A.cw <= CWC;

  auto stage_w = [&](int c0, int nc) {
    for (int i = tid; i < 32 * KK * nc; i += NT) {
      const int ci = i % nc;
      const int rest = i / nc;
      const int t = rest % KK;
      const int l = rest / KK;
      const int oo = g * 32 + l;
      w_s[(ci * KK + t) * 32 + l] = (oo < A.c_out) ? __ldg(A.wt + ((int64_t)oo * KK + t) * A.cw + c0 + ci) : 0u;
    }
  };

  if (single) stage_w(0, A.cw);

  const int64_t t_begin = (int64_t)blockIdx.x * A.tiles_per_cta;
  const int64_t t_end = min(t_begin + A.tiles_per_cta, A.total_tiles);

  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    int img, ty, tx;
    tile_coords(A, tile, img, ty, tx);
    const int oy0 = ty * TH, ox0 = tx * TW;

    int acc[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) acc[r][p] = 0;

    for (int c0 = 0; c0 < A.cw; c0 += CWC) {
      const int nc = min(CWC, A.cw - c0);
      __syncthreads();  // previous readers of in_s / w_s are done
      if (!single) stage_w(c0, nc);
      const uint32_t* xin = A.x + (int64_t)img * A.H * A.W * A.cw;
      for (int i = tid; i < IR * IC * nc; i += NT) {
        const int ci = i % nc;
        const int rest = i / nc;
        const int col = rest % IC;
        const int row = rest / IC;
        const int gy = oy0 - R + row, gx = ox0 - R + col;
        uint32_t v = 0u;  // outside the map: bit 0 = -1 (R4)
        if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) v = __ldg(xin + ((int64_t)gy * A.W + gx) * A.cw + c0 + ci);
        in_s[(ci * IR + row) * ICP + col] = v;
      }
      __syncthreads();

      for (int ci = 0; ci < nc; ++ci) {
#pragma unroll
        for (int ky = 0; ky < K; ++ky) {
          uint32_t wr[K];
#pragma unroll
          for (int kx = 0; kx < K; ++kx) wr[kx] = w_s[(ci * KK + ky * K + kx) * 32 + lane];
#pragma unroll
          for (int r = 0; r < PR; ++r) {
            const uint4* src = reinterpret_cast<const uint4*>(in_s + (ci * IR + wy * PR + r + ky) * ICP + wx * PC);
            uint32_t rw[4 * NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const uint4 q = src[v];
              rw[4 * v] = q.x; rw[4 * v + 1] = q.y; rw[4 * v + 2] = q.z; rw[4 * v + 3] = q.w;
            }
            if constexpr (CSA) {
#pragma unroll
              for (int p = 0; p < PC; ++p) {
                uint32_t xk[K];
#pragma unroll
                for (int kx = 0; kx < K; ++kx) xk[kx] = rw[p + kx] ^ wr[kx];
                acc[r][p] += csa_popc<K>(xk);
              }
            } else {
#pragma unroll
              for (int kx = 0; kx < K; ++kx)
#pragma unroll
                for (int p = 0; p < PC; ++p) acc[r][p] += popc(rw[p + kx] ^ wr[kx]);
            }
          }
        }
      }
    }

    int a[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) a[r][p] = nbits - 2 * acc[r][p];
    conv_epilogue<PR, PC>(A, img, oy0 + wy * PR, ox0 + wx * PC, g, lane, a, thr_o, flip_o);
  }
}

// First binary layer with few input channels (c_in < 32, one word per pixel): the K x K x c_in
// patch of each output pixel is packed DENSELY into ceil(K*K*c_in/32) words (<= 8) in shared
// memory, and the weights are repacked the same way in registers, so conv1 of the vehicle net
// (K = 5, c_in = 3: 75 bits) costs 3 popcounts per output instead of 25.  Bit i of the patch
// (i = (ky*K + kx)*c_in + c) sits at word i/32, bit 31 - i%32 -- an internal order; the
// result is the same Eq. (3) sum (R2: the integer result is layout-invariant).
template <int K, int PR, int PC, int WY, int WX>
__global__ void __launch_bounds__(WY * WX * 32)
conv_patch_kernel(const ConvArgs A) {
  constexpr int R = (K - 1) / 2;
  constexpr int KK = K * K;
  constexpr int TH = WY * PR, TW = WX * PC;
  constexpr int IR = TH + K - 1;
  constexpr int IC = TW + K - 1;
  constexpr int NT = WY * WX * 32;
  constexpr int PWMAX = 8;
  constexpr int TWP = TW;  // patch plane pitch (TW is a multiple of 8)

  __shared__ uint32_t in_s[IR * IC];
  __shared__ __align__(16) uint32_t patch_s[PWMAX * TH * TWP];
  __shared__ uint32_t wp_s[PWMAX * 32 * (NT / 32)];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WX, wx = warp % WX;
  const int g = blockIdx.y;
  const int o = g * 32 + lane;
  const bool ovalid = o < A.c_out;
  const int thr_o = (A.thr != nullptr && ovalid) ? A.thr[o] : 0;
  const bool flip_o = (A.flip != nullptr && ovalid) ? (A.flip[o] != 0) : false;
  const int cin = A.c_in;
  const int nbits = KK * cin;
  const int npw = (nbits + 31) / 32;
  const uint32_t keep = 32 - cin;  // top cin bits of a pixel word

  // Repack this lane's weights densely (same bit order as the patch).  Each warp builds
  // its own copy in its slice of wp_s, then moves it to registers.
  {
    uint32_t* mine = wp_s + warp * (PWMAX * 32);
    uint64_t bits = 0;
    int nb = 0, pw = 0;
    for (int t = 0; t < KK; ++t) {
      const uint32_t wv = ovalid ? (__ldg(A.wt + (int64_t)o * KK + t) >> keep) : 0u;
      bits = (bits << cin) | wv;
      nb += cin;
      if (nb >= 32) { mine[pw * 32 + lane] = (uint32_t)(bits >> (nb - 32)); ++pw; nb -= 32; bits &= (nb ? ((1ull << nb) - 1) : 0ull); }
    }
    if (nb > 0) { mine[pw * 32 + lane] = (uint32_t)(bits << (32 - nb)); ++pw; }
    __syncwarp();
  }
  uint32_t wreg[PWMAX];
#pragma unroll
  for (int j = 0; j < PWMAX; ++j) wreg[j] = (j < npw) ? wp_s[warp * (PWMAX * 32) + j * 32 + lane] : 0u;

  const int64_t t_begin = (int64_t)blockIdx.x * A.tiles_per_cta;
  const int64_t t_end = min(t_begin + A.tiles_per_cta, A.total_tiles);

  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    int img, ty, tx;
    tile_coords(A, tile, img, ty, tx);
    const int oy0 = ty * TH, ox0 = tx * TW;

    __syncthreads();  // previous tile's readers are done
    const uint32_t* xin = A.x + (int64_t)img * A.H * A.W;
    for (int i = tid; i < IR * IC; i += NT) {
      const int col = i % IC, row = i / IC;
      const int gy = oy0 - R + row, gx = ox0 - R + col;
      in_s[i] = (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) ? __ldg(xin + (int64_t)gy * A.W + gx) : 0u;
    }
    __syncthreads();
    // build the dense patch words of every output pixel of the tile
    for (int pix = tid; pix < TH * TW; pix += NT) {
      const int py = pix / TW, px = pix - py * TW;
      uint64_t bits = 0;
      int nb = 0, pw = 0;
      for (int ky = 0; ky < K; ++ky)
        for (int kx = 0; kx < K; ++kx) {
          bits = (bits << cin) | (in_s[(py + ky) * IC + px + kx] >> keep);
          nb += cin;
          if (nb >= 32) {
            patch_s[(pw * TH + py) * TWP + px] = (uint32_t)(bits >> (nb - 32));
            ++pw;
            nb -= 32;
            bits &= (nb ? ((1ull << nb) - 1) : 0ull);
          }
        }
      if (nb > 0) patch_s[(pw * TH + py) * TWP + px] = (uint32_t)(bits << (32 - nb));
    }
    __syncthreads();

    int acc[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) acc[r][p] = 0;
#pragma unroll
    for (int j = 0; j < PWMAX; ++j) {
      if (j < npw) {
#pragma unroll
        for (int r = 0; r < PR; ++r) {
          const uint4* src = reinterpret_cast<const uint4*>(patch_s + (j * TH + wy * PR + r) * TWP + wx * PC);
#pragma unroll
          for (int v = 0; v < PC / 4; ++v) {
            const uint4 q = src[v];
            acc[r][4 * v] += popc(q.x ^ wreg[j]);
            acc[r][4 * v + 1] += popc(q.y ^ wreg[j]);
            acc[r][4 * v + 2] += popc(q.z ^ wreg[j]);
            acc[r][4 * v + 3] += popc(q.w ^ wreg[j]);
          }
        }
      }
    }
    int a[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) a[r][p] = nbits - 2 * acc[r][p];
    conv_epilogue<PR, PC>(A, img, oy0 + wy * PR, ox0 + wx * PC, g, lane, a, thr_o, flip_o);
  }
}

// First binary layer with few input channels, "strip" layout.  For every input row r of the
// halo tile and output column x, the K horizontal taps x-R..x+R of c_in bits each form one
// S = K*c_in bit strip (built with K warp shuffles per row, one lane per column).  A patch word
// then stacks rpw = 32/S strips of consecutive rows (top-aligned), so the K x K x c_in patch of
// an output pixel is ceil(K/rpw) words (vehicle conv1: 15-bit strips, 2 rows/word, 3 words) and
// costs a few shifts per pixel instead of a per-bit loop.  The weights are repacked the same way
// in registers.  With SRC_U8 the kernel reads the u8 image and applies the Section 2.3 threshold
// (bit_c = x_c > -T_c, or x_c > 0 for SIGN) itself, so the input never makes a packed round trip
// through HBM.
template <int K, int PR, int PC, int WY, int WX, bool SRC_U8>
__global__ void __launch_bounds__(WY * WX * 32)
conv_strip_kernel(const ConvArgs A, const uint8_t* __restrict__ xu8, const float* __restrict__ Tt) {
  constexpr int R = (K - 1) / 2;
  constexpr int TH = WY * PR, TW = WX * PC;
  constexpr int IR = TH + K - 1;
  constexpr int IC = TW + K - 1;
  constexpr int NT = WY * WX * 32;
  constexpr int NWARP = WY * WX;
  static_assert(IC <= 32, "one lane per halo column");

  __shared__ uint32_t strips[IR * TW];
  __shared__ __align__(16) uint32_t patch[K * TH * TW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WX, wx = warp % WX;
  const int g = blockIdx.y;
  const int o = g * 32 + lane;
  const bool ovalid = o < A.c_out;
  const int thr_o = (A.thr != nullptr && ovalid) ? A.thr[o] : 0;
  const bool flip_o = (A.flip != nullptr && ovalid) ? (A.flip[o] != 0) : false;
  const int cin = A.c_in;
  const int S = K * cin;
  const int rpw = 32 / S;
  const int nw = (K + rpw - 1) / rpw;
  const int nbits = K * K * cin;

  // thresholds for the fused u8 path: bit_c = x_c > t_c
  int ti[4] = {0, 0, 0, 0};  // u8 bit_c = x_c > ti_c  (SIGN: x > 0)
  if (SRC_U8 && Tt != nullptr) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < cin) ti[c] = u8_threshold(-Tt[c]);
  }

  // this lane's weights in the strip layout
  uint32_t wreg[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    wreg[j] = 0u;
    if (j < nw && ovalid) {
      for (int t = 0; t < rpw; ++t) {
        const int ky = j * rpw + t;
        if (ky >= K) break;
        uint32_t ws = 0;
#pragma unroll
        for (int kx = 0; kx < K; ++kx)
          ws |= (__ldg(A.wt + (int64_t)o * K * K + ky * K + kx) >> (32 - cin)) << (cin * (K - 1 - kx));
        wreg[j] |= ws << (32 - (t + 1) * S);
      }
    }
  }

  const int64_t t_begin = (int64_t)blockIdx.x * A.tiles_per_cta;
  const int64_t t_end = min(t_begin + A.tiles_per_cta, A.total_tiles);

  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    int img, ty, tx;
    tile_coords(A, tile, img, ty, tx);
    const int oy0 = ty * TH, ox0 = tx * TW;

    // phase A: one warp per halo row: lane = halo column -> c_in-bit code -> K-tap strips
    for (int r = warp; r < IR; r += NWARP) {
      const int gy = oy0 - R + r, gx = ox0 - R + lane;
      uint32_t code = 0u;  // outside the map: all bits 0 = -1 (R4)
      if (lane < IC && gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) {
        const int64_t pix = ((int64_t)img * A.H + gy) * A.W + gx;
        if (SRC_U8) {
          const uint8_t* px = xu8 + pix * cin;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < cin) code |= (uint32_t)((int)px[c] > ti[c]) << (cin - 1 - c);
        } else {
          code = __ldg(A.x + pix) >> (32 - cin);
        }
      }
      uint32_t strip = 0u;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) strip |= __shfl_sync(BNN_FULL_MASK, code, (lane + kx) & 31) << (cin * (K - 1 - kx));
      if (lane < TW) strips[r * TW + lane] = strip;
    }
    __syncthreads();
    // phase B: patch words = rpw strips of consecutive rows, top-aligned
    for (int it = tid; it < nw * TH * TW; it += NT) {
      const int j = it / (TH * TW);
      const int pix = it - j * (TH * TW);
      const int py = pix / TW, px = pix - py * TW;
      uint32_t word = 0u;
      for (int t = 0; t < rpw; ++t) {
        const int row = j * rpw + t;
        if (row < K) word |= strips[(py + row) * TW + px] << (32 - (t + 1) * S);
      }
      patch[it] = word;
    }
    __syncthreads();

    int acc[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) acc[r][p] = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j < nw) {
#pragma unroll
        for (int r = 0; r < PR; ++r) {
          const uint4* src = reinterpret_cast<const uint4*>(patch + (j * TH + wy * PR + r) * TW + wx * PC);
#pragma unroll
          for (int v = 0; v < PC / 4; ++v) {
            const uint4 q = src[v];
            acc[r][4 * v] += popc(q.x ^ wreg[j]);
            acc[r][4 * v + 1] += popc(q.y ^ wreg[j]);
            acc[r][4 * v + 2] += popc(q.z ^ wreg[j]);
            acc[r][4 * v + 3] += popc(q.w ^ wreg[j]);
          }
        }
      }
    }
    int a[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) a[r][p] = nbits - 2 * acc[r][p];
    conv_epilogue<PR, PC>(A, img, oy0 + wy * PR, ox0 + wx * PC, g, lane, a, thr_o, flip_o);
  }
}

// First binary layer, "lane = pixel" mapping (the fast path for c_in <= 10).
// With only NW (1..7) patch words per output, the lane = channel kernels above spend most of
// their issue slots on the per-pixel epilogue (ballot, brev, addressing).  Here each thread owns
// two vertically adjacent output pixels and walks the 32 output channels of its group: the
// channel's NW weight words and its integer limit arrive with one broadcast LDS.128, and
//   bit = (K*K*c_in - 2 acc > thr)  <=>  acc <= lim,  lim = floor((K*K*c_in - thr - 1) / 2)
// sets bit 31 - c of the output word with one predicated OR -- the packed word is built in a
// register, the flip mask is one XOR, the 2x2 OR-pool is one OR plus one shuffle.
// Patch layout: strips of K taps (S = K*c_in bits) stacked RPW = ceil(K/NW) rows per word.
template <int K, int NW, bool SRC_U8>
__global__ void __launch_bounds__(256)
conv_first_lp_kernel(const ConvArgs A, const uint8_t* __restrict__ xu8, const float* __restrict__ Tt) {
  constexpr int NWARP = 8, PRW = 2;
  constexpr int TH = NWARP * PRW, TW = 32;
  constexpr int R = (K - 1) / 2;
  constexpr int IR = TH + K - 1, IC = TW + K - 1;
  constexpr int RPW = (K + NW - 1) / NW;
  constexpr int WS = (NW + 1 + 3) & ~3;  // words per channel slot: NW weight words + limit
  constexpr int NT = NWARP * 32;

  __shared__ uint32_t codes[IR * IC];
  __shared__ uint32_t strips[IR * TW];
  __shared__ __align__(16) int32_t wsm[32 * WS];
  __shared__ uint32_t flipmask_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int cin = A.c_in;
  const int S = K * cin;
  const int nbits = K * K * cin;

  if (warp == 0) {
    const int o = g * 32 + lane;
    const bool ovalid = o < A.c_out;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      uint32_t word = 0u;
#pragma unroll
      for (int t = 0; t < RPW; ++t) {
        const int ky = j * RPW + t;
        if (ky < K && ovalid) {
          uint32_t ws = 0u;
#pragma unroll
          for (int kx = 0; kx < K; ++kx)
            ws |= (__ldg(A.wt + (int64_t)o * K * K + ky * K + kx) >> (32 - cin)) << (cin * (K - 1 - kx));
          word |= ws << (32 - (t + 1) * S);
        }
      }
      wsm[lane * WS + j] = (int32_t)word;
    }
    int lim = -1;  // invalid channel: acc >= 0 > lim, bit stays 0
    if (ovalid) {
      const int64_t thr = (A.thr != nullptr) ? (int64_t)A.thr[o] : 0;
      int64_t v = ((int64_t)nbits - thr - 1) >> 1;  // floor division
      v = v < -1 ? -1 : (v > nbits ? nbits : v);
      lim = (int)v;
    }
    wsm[lane * WS + NW] = lim;
    const uint32_t fm = ballot_pack(ovalid && A.flip != nullptr && A.flip[o] != 0);
    if (lane == 0) flipmask_s = fm;
  }

  int ti[4] = {0, 0, 0, 0};  // u8 bit_c = x_c > ti_c  (SIGN: x > 0)
  if (SRC_U8 && Tt != nullptr) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < cin) ti[c] = u8_threshold(-Tt[c]);
  }
  __syncthreads();
  const uint32_t flipmask = flipmask_s;

  const int64_t t_begin = (int64_t)blockIdx.x * A.tiles_per_cta;
  const int64_t t_end = min(t_begin + A.tiles_per_cta, A.total_tiles);

  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    int img, ty, tx;
    tile_coords(A, tile, img, ty, tx);
    const int oy0 = ty * TH, ox0 = tx * TW;

    __syncthreads();  // previous tile's readers of codes / strips are done
    for (int i = tid; i < IR * IC; i += NT) {
      const int r = i / IC, cc = i - r * IC;
      const int gy = oy0 - R + r, gx = ox0 - R + cc;
      uint32_t code = 0u;  // outside the map: -1 (R4)
      if (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) {
        const int64_t pix = ((int64_t)img * A.H + gy) * A.W + gx;
        if (SRC_U8) {
          const uint8_t* px = xu8 + pix * cin;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < cin) code |= (uint32_t)((int)px[c] > ti[c]) << (cin - 1 - c);
        } else {
          code = __ldg(A.x + pix) >> (32 - cin);
        }
      }
      codes[i] = code;
    }
    __syncthreads();
    for (int i = tid; i < IR * TW; i += NT) {
      const int r = i / TW, x = i - r * TW;
      uint32_t strip = 0u;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) strip |= codes[r * IC + x + kx] << (cin * (K - 1 - kx));
      strips[i] = strip;
    }
    __syncthreads();

    // this thread's two pixels: tile rows 2*warp and 2*warp + 1, column lane
    uint32_t s[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) s[i] = strips[(PRW * warp + i) * TW + lane];
    uint32_t p0[NW], p1[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      p0[j] = 0u;
      p1[j] = 0u;
#pragma unroll
      for (int t = 0; t < RPW; ++t) {
        const int ky = j * RPW + t;
        if (ky < K) {
          p0[j] |= s[ky] << (32 - (t + 1) * S);
          p1[j] |= s[ky + 1] << (32 - (t + 1) * S);
        }
      }
    }
    const int oy = oy0 + PRW * warp, ox = ox0 + lane;
    const bool in0 = oy < A.H && ox < A.W, in1 = (oy + 1) < A.H && ox < A.W;
    uint32_t w0 = 0u, w1 = 0u;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      int wv[WS];
#pragma unroll
      for (int q = 0; q < WS / 4; ++q) {
        const int4 v = reinterpret_cast<const int4*>(wsm + c * WS)[q];
        wv[4 * q] = v.x; wv[4 * q + 1] = v.y; wv[4 * q + 2] = v.z; wv[4 * q + 3] = v.w;
      }
      int a0 = 0, a1 = 0;
#pragma unroll
      for (int j = 0; j < NW; ++j) {
        a0 += popc(p0[j] ^ (uint32_t)wv[j]);
        a1 += popc(p1[j] ^ (uint32_t)wv[j]);
      }
      const int lim = wv[NW];
      if (a0 <= lim) w0 |= 1u << (31 - c);
      if (a1 <= lim) w1 |= 1u << (31 - c);
      if (A.acc != nullptr && g * 32 + c < A.c_out) {
        if (in0) A.acc[(((int64_t)img * A.H + oy) * A.W + ox) * A.c_out + g * 32 + c] = nbits - 2 * a0;
        if (in1) A.acc[(((int64_t)img * A.H + oy + 1) * A.W + ox) * A.c_out + g * 32 + c] = nbits - 2 * a1;
      }
    }
    w0 ^= flipmask;
    w1 ^= flipmask;
    if (A.y != nullptr) {
      if (A.pool == 2) {
        uint32_t v = w0 | w1;
        v |= __shfl_xor_sync(BNN_FULL_MASK, v, 1);
        const int Ho = A.H >> 1, Wo = A.W >> 1;
        const int py = oy >> 1, px = ox >> 1;
        if ((lane & 1) == 0 && py < Ho && px < Wo) A.y[(((int64_t)img * Ho + py) * Wo + px) * A.cwo + g] = v;
      } else {
        if (in0) A.y[(((int64_t)img * A.H + oy) * A.W + ox) * A.cwo + g] = w0;
        if (in1) A.y[(((int64_t)img * A.H + oy + 1) * A.W + ox) * A.cwo + g] = w1;
      }
    }
  }
}

// Real-valued first layer ("no input binarization"): acc = sum w * x with
// w in {+1,-1} and ZERO padding (R5).  u8 input: exact int32 via IDP4A.U8.S8 on a per-pixel
// byte patch staged in shared memory.  f32 input: fp32 FFMA in (ky, kx, c) order (R18).
struct RealConvArgs {
  const void* x;  // [n, H, W, c_in] u8 or f32
  const uint32_t* wt;
  const int32_t* thr;
  const uint8_t* flip;
  uint32_t* y;
  void* acc;  // int32 (u8) or float (f32)
  int n, H, W, c_in, c_out, cwo, pool;
  int tiles_x, tiles_y;
  int64_t total_tiles;
  int tiles_per_cta;
  FastDiv fd_img, fd_tx;
};

template <int K, int PR, int PC, int WY, int WX>
__global__ void __launch_bounds__(WY * WX * 32)
conv_real_u8_kernel(const RealConvArgs A) {
  constexpr int R = (K - 1) / 2;
  constexpr int KK = K * K;
  constexpr int TH = WY * PR, TW = WX * PC;
  constexpr int IR = TH + K - 1;
  constexpr int IC = TW + K - 1;
  constexpr int NT = WY * WX * 32;
  constexpr int NWMAX = (KK * 32 + 3) / 4;  // words of 4 bytes for c_in <= 32
  (void)NWMAX;
  extern __shared__ __align__(16) uint32_t dyn_s[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WX, wx = warp % WX;
  const int g = blockIdx.y;
  const int o = g * 32 + lane;
  const bool ovalid = o < A.c_out;
  const int thr_o = (A.thr != nullptr && ovalid) ? A.thr[o] : 0;
  const bool flip_o = (A.flip != nullptr && ovalid) ? (A.flip[o] != 0) : false;
  const int cin = A.c_in;
  const int nb = KK * cin;        // bytes per patch
  const int nw = (nb + 3) / 4;    // words per patch
  const int npix = TH * TW;

  uint8_t* in_s = reinterpret_cast<uint8_t*>(dyn_s);                      // IR*IC*cin bytes (padded to 16)
  const int in_bytes = ((IR * IC * cin) + 15) & ~15;
  uint32_t* patch_s = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(dyn_s) + in_bytes);  // [nw][npix]
  uint32_t* w_s = patch_s + nw * npix;                                     // [nw][32 * groups-in-cta=1]

  // s8 weights (+1 -> 0x01, -1 -> 0xff) in the same (ky, kx, c) byte order as the patch.
  for (int i = tid; i < nw * 32; i += NT) {
    const int j = i / 32, l = i % 32;
    const int oo = g * 32 + l;
    uint32_t word = 0;
    for (int b = 0; b < 4; ++b) {
      const int e = 4 * j + b;
      uint32_t byte = 0;
      if (e < nb && oo < A.c_out) {
        const int t = e / cin, c = e - t * cin;
        const uint32_t wv = __ldg(A.wt + (int64_t)oo * KK + t);
        byte = ((wv >> (31 - c)) & 1u) ? 0x01u : 0xffu;
      }
      word |= byte << (8 * b);
    }
    w_s[j * 32 + l] = word;
  }

  const int64_t t_begin = (int64_t)blockIdx.x * A.tiles_per_cta;
  const int64_t t_end = min(t_begin + A.tiles_per_cta, A.total_tiles);
  const uint8_t* xall = reinterpret_cast<const uint8_t*>(A.x);

  for (int64_t tile = t_begin; tile < t_end; ++tile) {
    int img, ty, tx;
    tile_coords(A, tile, img, ty, tx);
    const int oy0 = ty * TH, ox0 = tx * TW;
    __syncthreads();
    const uint8_t* xin = xall + (int64_t)img * A.H * A.W * cin;
    for (int i = tid; i < IR * IC * cin; i += NT) {
      const int c = i % cin;
      const int rest = i / cin;
      const int col = rest % IC, row = rest / IC;
      const int gy = oy0 - R + row, gx = ox0 - R + col;
      in_s[i] = (gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) ? xin[((int64_t)gy * A.W + gx) * cin + c] : (uint8_t)0;
    }
    __syncthreads();
    for (int i = tid; i < nw * npix; i += NT) {
      const int pix = i % npix, j = i / npix;
      const int py = pix / TW, px = pix - py * TW;
      uint32_t word = 0;
      for (int b = 0; b < 4; ++b) {
        const int e = 4 * j + b;
        uint32_t byte = 0;
        if (e < nb) {
          const int t = e / cin, c = e - t * cin;
          const int ky = t / K, kx = t - ky * K;
          byte = in_s[((py + ky) * IC + px + kx) * cin + c];
        }
        word |= byte << (8 * b);
      }
      patch_s[j * npix + pix] = word;
    }
    __syncthreads();

    int acc[PR][PC];
#pragma unroll
    for (int r = 0; r < PR; ++r)
#pragma unroll
      for (int p = 0; p < PC; ++p) acc[r][p] = 0;
    for (int j = 0; j < nw; ++j) {
      const uint32_t wv = w_s[j * 32 + lane];
#pragma unroll
      for (int r = 0; r < PR; ++r) {
        const uint4* src = reinterpret_cast<const uint4*>(patch_s + j * npix + (wy * PR + r) * TW + wx * PC);
#pragma unroll
        for (int v = 0; v < PC / 4; ++v) {
          const uint4 q = src[v];
          acc[r][4 * v] = dp4a_us(q.x, wv, acc[r][4 * v]);
          acc[r][4 * v + 1] = dp4a_us(q.y, wv, acc[r][4 * v + 1]);
          acc[r][4 * v + 2] = dp4a_us(q.z, wv, acc[r][4 * v + 2]);
          acc[r][4 * v + 3] = dp4a_us(q.w, wv, acc[r][4 * v + 3]);
        }
      }
    }
    ConvArgs E;
    E.x = nullptr; E.wt = nullptr; E.thr = nullptr; E.flip = nullptr;
    E.y = A.y; E.acc = reinterpret_cast<int32_t*>(A.acc);
    E.n = A.n; E.H = A.H; E.W = A.W; E.cw = 1; E.c_in = cin; E.c_out = A.c_out; E.cwo = A.cwo; E.pool = A.pool;
    conv_epilogue<PR, PC>(E, img, oy0 + wy * PR, ox0 + wx * PC, g, lane, acc, thr_o, flip_o);
  }
}

// f32 real first layer: simple and exact-order (fp32 add/sub over (ky, kx, c)); not on the
// benchmark path (the paper's NONE mode feeds u8 pixels).  One warp per (output pixel after
// pooling, channel group); lane = channel; the pool x pool sub-pixels are ORed.
__global__ void conv_real_f32_kernel(const RealConvArgs A, int K) {
  const int R = (K - 1) / 2;
  const int P = A.pool;
  const int Ho = A.H / P, Wo = A.W / P;
  const int64_t total = (int64_t)A.n * Ho * Wo * A.cwo * 32;
  const float* x = reinterpret_cast<const float*>(A.x);
  float* accf = reinterpret_cast<float*>(A.acc);
  const int lane = threadIdx.x & 31;
  for (int64_t i = gtid(); i - lane < total; i += gstride()) {
    const bool in_range = i < total;
    const int64_t opix = in_range ? i / (A.cwo * 32) : 0;
    const int g = in_range ? (int)((i / 32) % A.cwo) : 0;
    const int o = g * 32 + lane;
    const int img = (int)(opix / ((int64_t)Ho * Wo));
    const int rem = (int)(opix - (int64_t)img * Ho * Wo);
    const int py = rem / Wo, px = rem - py * Wo;
    const bool valid = in_range && o < A.c_out;
    const float t = (valid && A.thr) ? (float)A.thr[o] : 0.f;
    const bool f = (valid && A.flip) ? (A.flip[o] != 0) : false;
    uint32_t word = 0;
    for (int sy = 0; sy < P; ++sy)
      for (int sx = 0; sx < P; ++sx) {
        const int yy = py * P + sy, xx = px * P + sx;
        float s = 0.f;
        if (valid) {
          for (int ky = 0; ky < K; ++ky)
            for (int kx = 0; kx < K; ++kx) {
              const int gy = yy + ky - R, gx = xx + kx - R;
              if (gy < 0 || gy >= A.H || gx < 0 || gx >= A.W) continue;  // zero padding (R5)
              const uint32_t wv = __ldg(A.wt + ((int64_t)o * K + ky) * K + kx);
              const float* pp = x + (((int64_t)img * A.H + gy) * A.W + gx) * A.c_in;
              for (int c = 0; c < A.c_in; ++c) {
                const float v = pp[c];
                s = ((wv >> (31 - c)) & 1u) ? s + v : s - v;
              }
            }
          if (accf) accf[(((int64_t)img * A.H + yy) * A.W + xx) * A.c_out + o] = s;
        }
        word |= ballot_pack(valid && ((s > t) != f));
      }
    if (in_range && lane == 0 && A.y) A.y[opix * A.cwo + g] = word;
  }
}

}  // namespace bnn
