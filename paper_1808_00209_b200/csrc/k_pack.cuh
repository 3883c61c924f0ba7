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

}  // namespace bnn
