// k_pack.cuh -- sign-and-pack kernels (bnn_pack): Eq. (1) + Eq. (2) and the Section 2.3
// input-binarization modes.
// HBM-bound: one pass over the input, one packed word per pixel (or per 32 channels).
#pragma once
#include "common.cuh"

namespace bnn {

enum PackMode { kSign = 0, kThreshRGB = 1, kThreshGray = 2, kLBP = 3 };

// bit = x > t, evaluated exactly for every input dtype (R14: X + T > 0 <=> X > -T).
template <typename T> BNN_DEV bool gt_thr(T v, float t) { return (float)v > t; }
template <> BNN_DEV bool gt_thr<int32_t>(int32_t v, float t) { return (double)v > (double)t; }
template <typename T> BNN_DEV bool gt_zero(T v) { return v > (T)0; }

// Generic path: one thread per (pixel, output word); any c, any dtype, SIGN / THRESH_RGB.
template <typename T>
__global__ void pack_generic_kernel(const T* __restrict__ x, int64_t npix, int c, int cw, int mode,
                                    const float* __restrict__ Tt, uint32_t* __restrict__ y) {
  const int64_t total = npix * cw;
  for (int64_t i = gtid(); i < total; i += gstride()) {
    const int64_t p = i / cw;
    const int wi = (int)(i - p * cw);
    const T* px = x + p * c;
    const int c0 = wi * 32, c1 = min(c, c0 + 32);
    uint32_t word = 0;
    for (int ch = c0; ch < c1; ++ch) {
      bool b = (mode == kThreshRGB) ? gt_thr<T>(px[ch], -Tt[ch]) : gt_zero<T>(px[ch]);
      word |= (uint32_t)b << (31 - (ch - c0));
    }
    y[i] = word;
  }
}

// Fast path for the paper's input: u8 RGB (c = 3), SIGN or THRESH_RGB.  Each thread packs
// 4 pixels: three aligned 32-bit loads (12 bytes) -> one 16-byte store of 4 words.
__global__ void pack_u8c3_kernel(const uint8_t* __restrict__ x, int64_t npix, int mode,
                                 const float* __restrict__ Tt, uint32_t* __restrict__ y) {
  float t0 = 0.f, t1 = 0.f, t2 = 0.f;
  if (mode == kThreshRGB) { t0 = -Tt[0]; t1 = -Tt[1]; t2 = -Tt[2]; }
  const int64_t nq = npix / 4;
  const uint32_t* x32 = reinterpret_cast<const uint32_t*>(x);
  for (int64_t q = gtid(); q < nq; q += gstride()) {
    const uint32_t a = __ldg(x32 + 3 * q), b = __ldg(x32 + 3 * q + 1), c = __ldg(x32 + 3 * q + 2);
    uint32_t by[12];
#pragma unroll
    for (int j = 0; j < 4; ++j) { by[j] = (a >> (8 * j)) & 0xffu; by[4 + j] = (b >> (8 * j)) & 0xffu; by[8 + j] = (c >> (8 * j)) & 0xffu; }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o[j] = ((uint32_t)((float)by[3 * j] > t0) << 31) | ((uint32_t)((float)by[3 * j + 1] > t1) << 30) |
             ((uint32_t)((float)by[3 * j + 2] > t2) << 29);
    }
    reinterpret_cast<uint4*>(y)[q] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  // tail pixels (npix % 4)
  for (int64_t p = nq * 4 + gtid(); p < npix; p += gstride()) {
    const uint8_t* px = x + 3 * p;
    y[p] = ((uint32_t)((float)px[0] > t0) << 31) | ((uint32_t)((float)px[1] > t1) << 30) |
           ((uint32_t)((float)px[2] > t2) << 29);
  }
}

// Integer Rec.601 luma (R15).
BNN_DEV int luma_u8(const uint8_t* p) { return (299 * (int)p[0] + 587 * (int)p[1] + 114 * (int)p[2] + 500) / 1000; }

// THRESH_GRAY and LBP (u8, c = 3): one thread per pixel.
__global__ void pack_luma_kernel(const uint8_t* __restrict__ x, int n, int h, int w, int mode,
                                 const float* __restrict__ Tt, uint32_t* __restrict__ y) {
  const int64_t npix = (int64_t)n * h * w;
  const float t = (mode == kThreshGray) ? -Tt[0] : 0.f;
  for (int64_t p = gtid(); p < npix; p += gstride()) {
    const int64_t img = p / ((int64_t)h * w);
    const int rem = (int)(p - img * h * w);
    const int yy = rem / w, xx = rem - yy * w;
    const uint8_t* base = x + img * (int64_t)h * w * 3;
    const int Y = luma_u8(base + (int64_t)rem * 3);
    uint32_t word;
    if (mode == kThreshGray) {
      word = (uint32_t)((float)Y > t) << 31;
    } else {
      // clockwise from top-left: n0 = (-1,-1), n3 = (0,+1), n6 = (+1,-1)   (R16)
      const int ym = max(yy - 1, 0), yp = min(yy + 1, h - 1);
      const int xm = max(xx - 1, 0), xp = min(xx + 1, w - 1);
      const int n0 = luma_u8(base + ((int64_t)ym * w + xm) * 3);
      const int n3 = luma_u8(base + ((int64_t)yy * w + xp) * 3);
      const int n6 = luma_u8(base + ((int64_t)yp * w + xm) * 3);
      word = ((uint32_t)(n0 > Y) << 31) | ((uint32_t)(n3 > Y) << 30) | ((uint32_t)(n6 > Y) << 29);
    }
    y[p] = word;
  }
}

// THRESH_GRAY and LBP feeding the TMA first layer: the same bits as pack_luma_kernel, written as a
// u8 [n, h, w, 3] image of 0 (-1) / 1 (+1) bytes that conv_first_tma_pool_kernel thresholds with
// x > 0 (an out-of-image byte 0 is the -1 padding, R4).  GRAY: channel 0 = Y > -T, channels 1-2 = 0
// (their weights are zero for a c_in = 1 layer); LBP: channel j = n_{3j} > Y (R16, replicate border).
// Four pixels of a row per thread (w % 4 == 0, 4-byte aligned image): aligned word loads of the
// centre row (+ the right neighbour) and, for LBP, of the rows above / below (+ the left neighbour),
// three word stores of the 12 output bytes -- 27,648 B per 96 x 96 image instead of 36,864 B of
// packed words.
BNN_DEV int luma3(uint32_t b0, uint32_t b1, uint32_t b2) { return (299 * (int)b0 + 587 * (int)b1 + 114 * (int)b2 + 500) / 1000; }
BNN_DEV uint32_t byte_of(const uint32_t (&v)[4], int i) { return (v[i >> 2] >> (8 * (i & 3))) & 0xFFu; }

__global__ void luma_u8img4_kernel(const uint8_t* __restrict__ x, int n, int h, int w, int mode,
                                   const float* __restrict__ Tt, uint8_t* __restrict__ y) {
  const int64_t ngroups = (int64_t)n * h * (w >> 2);
  const float t = (mode == kThreshGray) ? -Tt[0] : 0.f;
  const int wg = w >> 2;
  for (int64_t q = gtid(); q < ngroups; q += gstride()) {
    const int64_t row = q / wg;  // image * h + yy
    const int x0 = (int)(q - row * wg) * 4;
    const int64_t img = row / h;
    const int yy = (int)(row - img * h);
    const uint8_t* base = x + img * (int64_t)h * w * 3;
    const uint32_t* rc = reinterpret_cast<const uint32_t*>(base + ((int64_t)yy * w + x0) * 3);
    uint32_t c[4] = {rc[0], rc[1], rc[2], 0u};  // pixels x0..x0+3 (12 bytes)
    if (x0 + 4 < w) c[3] = rc[3];               // bytes 12..14: pixel x0+4
    int Y[5];
#pragma unroll
    for (int i = 0; i < 4; ++i) Y[i] = luma3(byte_of(c, 3 * i), byte_of(c, 3 * i + 1), byte_of(c, 3 * i + 2));
    uint32_t o[3] = {0u, 0u, 0u};
    if (mode == kThreshGray) {
#pragma unroll
      for (int i = 0; i < 4; ++i) o[(3 * i) >> 2] |= (uint32_t)((float)Y[i] > t) << (8 * ((3 * i) & 3));
    } else {
      Y[4] = (x0 + 4 < w) ? luma3(byte_of(c, 12), byte_of(c, 13), byte_of(c, 14)) : Y[3];  // R of the last
      int U[5], D[5];  // rows above / below at x0-1 .. x0+3 (clamped rows and columns)
      const int ym = max(yy - 1, 0), yp = min(yy + 1, h - 1);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint8_t* rb = base + ((int64_t)(r == 0 ? ym : yp) * w + x0) * 3;
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(rb);
        uint32_t v[4] = {x0 > 0 ? rw[-1] : 0u, rw[0], rw[1], rw[2]};  // bytes of pixels x0-1 (1..3) .. x0+3
        int* L = r == 0 ? U : D;
#pragma unroll
        for (int i = 0; i < 4; ++i) L[i + 1] = luma3(byte_of(v, 4 + 3 * i), byte_of(v, 5 + 3 * i), byte_of(v, 6 + 3 * i));
        L[0] = x0 > 0 ? luma3(byte_of(v, 1), byte_of(v, 2), byte_of(v, 3)) : L[1];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // clockwise from top-left: n0 = (-1,-1), n3 = (0,+1), n6 = (+1,-1)   (R16)
        const uint32_t b0 = U[i] > Y[i], b1 = Y[i + 1] > Y[i], b2 = D[i] > Y[i];
        o[(3 * i) >> 2] |= b0 << (8 * ((3 * i) & 3));
        o[(3 * i + 1) >> 2] |= b1 << (8 * ((3 * i + 1) & 3));
        o[(3 * i + 2) >> 2] |= b2 << (8 * ((3 * i + 2) & 3));
      }
    }
    uint32_t* yo = reinterpret_cast<uint32_t*>(y + ((img * h + yy) * (int64_t)w + x0) * 3);
    yo[0] = o[0];
    yo[1] = o[1];
    yo[2] = o[2];
  }
}

// The same output, one CTA per band of kLumaBand image rows: the band's rows and the rows above / below
// (replicated at the image border) are staged in shared memory with coalesced word loads, every luma value is
// computed ONCE (four pixels per lane from three aligned words) into a row of bytes whose border columns
// replicate the edge columns, and the LBP neighbour bits (R16: TL, R, BL, strict >, replicate border) of four
// pixels are three SIMD byte compares (vcmpgtu4) of shifted words; 12 output bytes per lane, three word
// stores.  Warp = row, lane = 4-pixel group: no divisions.  The grid-stride kernel above re-reads every row
// three times with dependent 4-byte loads (config 2: 0.118 ms per 4096 images, ~1 TB/s).
constexpr int kLumaBand = 32;

__host__ __device__ constexpr size_t luma_band_smem(int w) {
  return (size_t)(kLumaBand + 2) * (size_t)w * 3 + (size_t)(kLumaBand + 2) * (size_t)(w + 8);
}

__global__ void __launch_bounds__(256) luma_band_kernel(const uint8_t* __restrict__ x, int n, int h, int w, int mode,
                                                        const float* __restrict__ Tt, uint8_t* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t lb_smem[];
  constexpr int BH = kLumaBand, NWARP = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bands = (h + BH - 1) / BH;
  const int64_t img = blockIdx.x / bands;
  const int y0 = (int)(blockIdx.x - img * bands) * BH, nrows = min(BH, h - y0);
  const int rw = w * 3 / 4, wg = w >> 2;  // words per image row, 4-pixel groups per row (w % 4 == 0)
  const int lw = w + 8;                   // luma row pitch: column c at byte c + 4 (c = -1 .. w)
  uint32_t* raw = reinterpret_cast<uint32_t*>(lb_smem);      // staged row r = image row y0 - 1 + r (clamped)
  uint8_t* lum = lb_smem + (size_t)(BH + 2) * w * 3;          // [BH + 2][lw]
  const uint8_t* base = x + img * (int64_t)h * w * 3;
  // asynchronous copies (LDGSTS): every load of the band is in flight at once (a load -> shared store loop
  // serialises on the load latency)
  const bool v16 = (rw % 4) == 0;  // 16-byte chunks (rows and images 16-byte aligned)
  for (int r = warp; r < nrows + 2; r += NWARP) {
    const int gy = min(max(y0 - 1 + r, 0), h - 1);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(base + (int64_t)gy * w * 3);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(raw + r * rw);
    if (v16) {
      for (int c = lane; c < rw / 4; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(src + 4 * c) : "memory");
    } else {
      for (int c = lane; c < rw; c += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4 * c), "l"(src + c) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  __syncthreads();
  // (row, 4-pixel group) units flattened over the block: every lane busy (w / 4 = 24 groups per row would leave
  // a quarter of a row-per-warp mapping idle); the row by a multiply-high division
  const FastDiv fdg((uint32_t)wg);
  for (int k = threadIdx.x; k < (nrows + 2) * wg; k += blockDim.x) {
    const int r = (int)fdg.div((uint32_t)k), g = k - r * wg;
    uint8_t* lr = lum + r * lw;
    {
      const uint32_t v[4] = {raw[r * rw + 3 * g], raw[r * rw + 3 * g + 1], raw[r * rw + 3 * g + 2], 0u};
      // R15: Y = (299 R + 587 G + 114 B + 500) div 1000; the sum as two DP2A (bytes of the word pairs), the division
      // as a multiply-high by ceil(2^32 / 1000) (exact for numerators < 2^22)
      uint32_t yw = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t rgb = __byte_perm(v[(3 * i) >> 2], v[((3 * i) >> 2) + 1], (uint32_t)(((3 * i) & 3) | ((((3 * i) & 3) + 1) << 4) | ((((3 * i) & 3) + 2) << 8)));
        const uint32_t sy = __dp2a_hi(114u, rgb, __dp2a_lo((587u << 16) | 299u, rgb, 500u));
        yw |= __umulhi(sy, 4294968u) << (8 * i);
      }
      *reinterpret_cast<uint32_t*>(lr + 4 + 4 * g) = yw;
      if (g == 0) lr[3] = (uint8_t)yw;                        // column -1 = column 0
      if (g == wg - 1) lr[w + 4] = (uint8_t)(yw >> 24);       // column w = column w - 1
    }
  }
  __syncthreads();
  const int tg = (mode == kThreshGray) ? u8_threshold(-Tt[0]) : 0;  // Y > -T <=> Y > tg (R14), tg in [-1, 255]
  const uint32_t t4 = (uint32_t)(tg < 0 ? 0 : tg) * 0x01010101u;
  for (int k = threadIdx.x; k < nrows * wg; k += blockDim.x) {
    const int r = (int)fdg.div((uint32_t)k), g = k - r * wg;
    const uint8_t* lc = lum + (r + 1) * lw;
    {
      const int b = 4 + 4 * g;  // byte of pixel 4 g in its luma row
      const uint32_t C = *reinterpret_cast<const uint32_t*>(lc + b);
      uint32_t m0, m1, m2;
      if (mode == kThreshGray) {
        m0 = tg < 0 ? 0xFFFFFFFFu : __vcmpgtu4(C, t4);
        m1 = m2 = 0u;
      } else {  // clockwise from top-left: n0 = (-1,-1), n3 = (0,+1), n6 = (+1,-1)   (R16)
        const uint32_t* up = reinterpret_cast<const uint32_t*>(lc - lw + b - 4);
        const uint32_t* dn = reinterpret_cast<const uint32_t*>(lc + lw + b - 4);
        const uint32_t* ce = reinterpret_cast<const uint32_t*>(lc + b);
        const uint32_t TL = __funnelshift_r(up[0], up[1], 24), BL = __funnelshift_r(dn[0], dn[1], 24);
        const uint32_t Rn = __funnelshift_r(ce[0], ce[1], 8);
        m0 = __vcmpgtu4(TL, C);
        m1 = __vcmpgtu4(Rn, C);
        m2 = __vcmpgtu4(BL, C);
      }
      m0 &= 0x01010101u;
      m1 &= 0x01010101u;
      m2 &= 0x01010101u;
      // output byte 3 i + j = bit j of pixel i
      const uint32_t o0 = (m0 & 0xFFu) | ((m1 & 0xFFu) << 8) | ((m2 & 0xFFu) << 16) | ((m0 & 0xFF00u) << 16);
      const uint32_t o1 = ((m1 >> 8) & 0xFFu) | ((m2 & 0xFF00u)) | ((m0 & 0xFF0000u)) | ((m1 & 0xFF0000u) << 8);
      const uint32_t o2 = ((m2 >> 16) & 0xFFu) | ((m0 >> 16) & 0xFF00u) | ((m1 >> 8) & 0xFF0000u) | (m2 & 0xFF000000u);
      uint32_t* yo = reinterpret_cast<uint32_t*>(y + ((img * h + y0 + r) * (int64_t)w + 4 * g) * 3);
      yo[0] = o0;
      yo[1] = o1;
      yo[2] = o2;
    }
  }
}

}  // namespace bnn
