/*
 * bnn_oracle.c -- CPU ORACLE (test infrastructure only; see bnn_oracle.h).
 *
 * Plain, slow, obviously-correct definitions on unpacked +/-1 values.
 * Every function cites the passage of PAPER.md it writes out.  No packing,
 * XOR or popcount appears anywhere in the arithmetic: the oracle multiplies
 * and adds +/-1 values, which is what Eq. (3) states.  The only bit-level
 * code is orc_pack / orc_unpack, which evaluate Eq. (2) arithmetically
 * (powers of two), so that packed GPU words can be compared.
 */
#include "bnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Eq. (1). */
int orc_sign(double x) { return x > 0.0 ? +1 : -1; }

/* Eq. (2), term by term:
 *   word_j = sum_{i=jB+1}^{(j+1)B} (1 + x_i) * 2^(B-2-mod(i-1,B)).
 * (1+x_i) is 0 or 2, so the term is 0 or 2^(B-1-mod(i-1,B)); we evaluate it as
 * the product (1+x_i) * 2^(B-2-m) and, for m = B-1 where the exponent is -1,
 * as (1+x_i)/2 (reading R1).  With B = 32 the word is placed at the top of a
 * 32-bit word as Eq. (2) fixes the element order within B bits; for B < 32 the
 * word holds B bits in its low B positions (the representation Alg. 1 builds with
 * "s << B-1-i").  D not divisible by B: the last word holds the
 * remaining elements at positions B-1, B-2, ... (reading R12). */
int64_t orc_pack(const int8_t* x, int64_t D, int B, uint32_t* words) {
  if (B < 1 || B > 32 || D < 0) return -1;
  int64_t nw = (D + B - 1) / B;
  for (int64_t j = 0; j < nw; ++j) {
    uint64_t v = 0; /* sums of terms stay below 2^32 */
    for (int64_t i = j * B + 1; i <= (j + 1) * B && i <= D; ++i) {
      int m = (int)((i - 1) % B);
      int one_plus_x = 1 + x[i - 1]; /* 0 or 2 */
      int e = B - 2 - m;             /* exponent of Eq. (2) */
      uint64_t term;
      if (e >= 0)
        term = (uint64_t)one_plus_x * ((uint64_t)1 << e);
      else
        term = (uint64_t)(one_plus_x / 2); /* 2^-1 * (1+x_i) */
      v += term;
    }
    words[j] = (uint32_t)v;
  }
  return nw;
}

/* Inverse of Eq. (2): element i <- bit B-1-mod(i-1,B) of word ceil(i/B);
 * bit value 1 <-> +1. */
int orc_unpack(const uint32_t* words, int64_t D, int B, int8_t* x) {
  if (B < 1 || B > 32 || D < 0) return -1;
  int64_t nw = (D + B - 1) / B;
  for (int64_t j = 0; j < nw; ++j) {
    uint64_t v = words[j];
    uint64_t valid = 0;
    for (int64_t i = j * B + 1; i <= (j + 1) * B && i <= D; ++i) {
      int p = B - 1 - (int)((i - 1) % B);
      uint64_t bit = (v / ((uint64_t)1 << p)) % 2;
      x[i - 1] = bit ? +1 : -1;
      valid += (uint64_t)1 << p;
    }
    /* every bit outside the valid positions must be 0 */
    uint64_t rest = v;
    for (int p = 0; p < 32; ++p) {
      uint64_t bit = (rest / ((uint64_t)1 << p)) % 2;
      uint64_t is_valid = (valid / ((uint64_t)1 << p)) % 2;
      if (bit && !is_valid) return -2;
    }
  }
  return 0;
}

/* Reading R15 (grayscale conversion is unspecified in PAPER.md:179, 378). */
int orc_luma(int r, int g, int b) { return (299 * r + 587 * g + 114 * b + 500) / 1000; }

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Section 2.3, PAPER.md:141-145 (thresholding: X -> sign(X + T), T in R^{1x1xC})
 * and PAPER.md:178-179 (LBP on the grayscale image, radius 1, three pixels at a
 * clockwise stride of 3, 1 if they exceed the centre). */
int orc_binarize_input(const double* x, int h, int w, int c, int mode, const double* T, int8_t* out) {
  if (h < 0 || w < 0 || c < 1) return -1;
  if (mode == ORC_SIGN) {
    for (int64_t i = 0; i < (int64_t)h * w * c; ++i) out[i] = (int8_t)orc_sign(x[i]);
    return c;
  }
  if (mode == ORC_THRESH_RGB) {
    if (!T) return -1;
    for (int y = 0; y < h; ++y)
      for (int xx = 0; xx < w; ++xx)
        for (int ch = 0; ch < c; ++ch) {
          int64_t i = ((int64_t)y * w + xx) * c + ch;
          out[i] = (int8_t)orc_sign(x[i] + T[ch]); /* R14: exact sign of X + T */
        }
    return c;
  }
  if (mode == ORC_THRESH_GRAY || mode == ORC_LBP) {
    if (c != 3) return -1;
    int* Y = (int*)malloc(sizeof(int) * (size_t)h * (size_t)w + 1);
    if (!Y) return -1;
    for (int y = 0; y < h; ++y)
      for (int xx = 0; xx < w; ++xx) {
        const double* p = x + ((int64_t)y * w + xx) * 3;
        Y[(int64_t)y * w + xx] = orc_luma((int)p[0], (int)p[1], (int)p[2]);
      }
    if (mode == ORC_THRESH_GRAY) {
      if (!T) { free(Y); return -1; }
      for (int64_t i = 0; i < (int64_t)h * w; ++i) out[i] = (int8_t)orc_sign((double)Y[i] + T[0]);
      free(Y);
      return 1;
    }
    /* LBP: neighbours n0..n7 clockwise from the top-left (reading R16). */
    static const int dy[8] = {-1, -1, -1, 0, +1, +1, +1, 0};
    static const int dx[8] = {-1, 0, +1, +1, +1, 0, -1, -1};
    for (int y = 0; y < h; ++y)
      for (int xx = 0; xx < w; ++xx) {
        int centre = Y[(int64_t)y * w + xx];
        for (int j = 0; j < 3; ++j) {
          int n = 3 * j; /* clockwise stride of 3: n0, n3, n6 */
          int yy = clampi(y + dy[n], 0, h - 1), xn = clampi(xx + dx[n], 0, w - 1);
          int v = Y[(int64_t)yy * w + xn];
          out[((int64_t)y * w + xx) * 3 + j] = (int8_t)(v > centre ? +1 : -1);
        }
      }
    free(Y);
    return 3;
  }
  return -1;
}

/* Eq. (3), with -1 outside the map (reading R4). */
void orc_conv_binary(const int8_t* x, int h, int w, int c_in, const int8_t* wt, int c_out, int k,
                     int64_t* acc) {
  int R = (k - 1) / 2;
  for (int y = 0; y < h; ++y)
    for (int xx = 0; xx < w; ++xx)
      for (int o = 0; o < c_out; ++o) {
        int64_t s = 0;
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx)
            for (int c = 0; c < c_in; ++c) {
              int yy = y + ky - R, xs = xx + kx - R;
              int v = (yy >= 0 && yy < h && xs >= 0 && xs < w) ? x[((int64_t)yy * w + xs) * c_in + c] : -1;
              int wv = wt[(((int64_t)o * k + ky) * k + kx) * c_in + c];
              s += (int64_t)wv * v;
            }
        acc[((int64_t)y * w + xx) * c_out + o] = s;
      }
}

/* Eq. (3), one output (same loops as orc_conv_binary). */
int64_t orc_conv_binary_point(const int8_t* x, int h, int w, int c_in, const int8_t* wt_o, int k, int y, int xx) {
  int R = (k - 1) / 2;
  int64_t s = 0;
  for (int ky = 0; ky < k; ++ky)
    for (int kx = 0; kx < k; ++kx)
      for (int c = 0; c < c_in; ++c) {
        int yy = y + ky - R, xs = xx + kx - R;
        int v = (yy >= 0 && yy < h && xs >= 0 && xs < w) ? x[((int64_t)yy * w + xs) * c_in + c] : -1;
        s += (int64_t)wt_o[((int64_t)ky * k + kx) * c_in + c] * v;
      }
  return s;
}

/* Eq. (3) on a real-valued first layer with zero padding (reading R5). */
void orc_conv_real(const double* x, int h, int w, int c_in, const int8_t* wt, int c_out, int k,
                   double* acc) {
  int R = (k - 1) / 2;
  for (int y = 0; y < h; ++y)
    for (int xx = 0; xx < w; ++xx)
      for (int o = 0; o < c_out; ++o) {
        double s = 0.0;
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx)
            for (int c = 0; c < c_in; ++c) {
              int yy = y + ky - R, xs = xx + kx - R;
              double v = (yy >= 0 && yy < h && xs >= 0 && xs < w) ? x[((int64_t)yy * w + xs) * c_in + c] : 0.0;
              int wv = wt[(((int64_t)o * k + ky) * k + kx) * c_in + c];
              s += (double)wv * v;
            }
        acc[((int64_t)y * w + xx) * c_out + o] = s;
      }
}

/* Eq. (1) with per-channel threshold/flip (reading R9; thr = 0, flip = 0 is Eq. 1). */
void orc_binarize_i64(const int64_t* acc, int64_t count, int c, const int32_t* thr,
                      const uint8_t* flip, int8_t* out) {
  for (int64_t i = 0; i < count; ++i) {
    int ch = (int)(i % c);
    int64_t t = thr ? (int64_t)thr[ch] : 0;
    int f = flip ? (flip[ch] != 0) : 0;
    int s = orc_sign((double)(acc[i] - t)); /* acc > t  <=>  sign(acc - t) = +1 */
    out[i] = (int8_t)(f ? -s : s);
  }
}

void orc_binarize_f64(const double* acc, int64_t count, int c, const int32_t* thr,
                      const uint8_t* flip, int8_t* out) {
  for (int64_t i = 0; i < count; ++i) {
    int ch = (int)(i % c);
    double t = thr ? (double)thr[ch] : 0.0;
    int f = flip ? (flip[ch] != 0) : 0;
    int s = acc[i] > t ? +1 : -1;
    out[i] = (int8_t)(f ? -s : s);
  }
}

/* 2x2 stride-2 max-pooling (Table 2). */
void orc_maxpool2(const int8_t* x, int h, int w, int c, int8_t* y) {
  int ho = h / 2, wo = w / 2;
  for (int i = 0; i < ho; ++i)
    for (int j = 0; j < wo; ++j)
      for (int ch = 0; ch < c; ++ch) {
        int m = -2;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) {
            int v = x[((int64_t)(2 * i + a) * w + (2 * j + b)) * c + ch];
            if (v > m) m = v;
          }
        y[((int64_t)i * wo + j) * c + ch] = (int8_t)m;
      }
}

/* Fully connected layer: acc[l] = W[l] . x. */
void orc_dense(const int8_t* x, int64_t d, const int8_t* W, int l, int64_t* acc) {
  for (int o = 0; o < l; ++o) {
    int64_t s = 0;
    for (int64_t i = 0; i < d; ++i) s += (int64_t)W[(int64_t)o * d + i] * x[i];
    acc[o] = s;
  }
}

int orc_argmax_i64(const int64_t* v, int l) {
  int best = 0;
  for (int i = 1; i < l; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

void orc_affine(const int64_t* acc, int l, const float* scale, const float* bias, double* score64,
                float* score32) {
  for (int o = 0; o < l; ++o) {
    if (score64) score64[o] = (double)scale[o] * (double)acc[o] + (double)bias[o];
    if (score32) score32[o] = fmaf(scale[o], (float)acc[o], bias[o]);
  }
}

int orc_argmax_f32(const float* v, int l) {
  int best = 0;
  for (int i = 1; i < l; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

/* Section 2 pipeline in Table 2's order. */
int orc_forward(const double* x, int h, int w, int c, int mode, const double* T, const orc_layer* layers,
                int n_layers, int64_t* logits, int32_t* cls) {
  if (n_layers < 1 || layers[n_layers - 1].kind != 2) return -1;
  /* current activation: either real (first layer, mode NONE) or +/-1 */
  int8_t* act = NULL;
  int ch = c, H = h, W = w;
  int64_t flat = 0; /* > 0 once we are in the dense part */
  int li = 0;
  if (mode == ORC_NONE) {
    const orc_layer* L = &layers[0];
    if (L->kind != 1) return -1;
    double* accr = (double*)malloc(sizeof(double) * (size_t)H * W * L->c_out);
    int8_t* b = (int8_t*)malloc((size_t)H * W * L->c_out);
    if (!accr || !b) { free(accr); free(b); return -1; }
    orc_conv_real(x, H, W, c, L->wt, L->c_out, L->k, accr);
    orc_binarize_f64(accr, (int64_t)H * W * L->c_out, L->c_out, L->thr, L->flip, b);
    free(accr);
    ch = L->c_out;
    if (L->pool == 2) {
      int8_t* p = (int8_t*)malloc((size_t)(H / 2) * (W / 2) * ch);
      orc_maxpool2(b, H, W, ch, p);
      free(b);
      b = p;
      H /= 2; W /= 2;
    }
    act = b;
    li = 1;
  } else {
    act = (int8_t*)malloc((size_t)H * W * (c > 3 ? c : 3));
    if (!act) return -1;
    ch = orc_binarize_input(x, H, W, c, mode, T, act);
    if (ch < 0) { free(act); return -1; }
  }
  for (; li < n_layers; ++li) {
    const orc_layer* L = &layers[li];
    int last = (li == n_layers - 1);
    if (L->kind == 1) {
      if (flat) { free(act); return -1; }
      int64_t n = (int64_t)H * W * L->c_out;
      int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
      int8_t* b = (int8_t*)malloc((size_t)n);
      orc_conv_binary(act, H, W, ch, L->wt, L->c_out, L->k, acc);
      orc_binarize_i64(acc, n, L->c_out, L->thr, L->flip, b);
      free(acc);
      free(act);
      ch = L->c_out;
      if (L->pool == 2) {
        int8_t* p = (int8_t*)malloc((size_t)(H / 2) * (W / 2) * ch);
        orc_maxpool2(b, H, W, ch, p);
        free(b);
        b = p;
        H /= 2; W /= 2;
      }
      act = b;
    } else if (L->kind == 2) {
      if (!flat) flat = (int64_t)H * W * ch; /* HWC flatten (reading R11) */
      int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)L->l);
      orc_dense(act, flat, L->wt, L->l, acc);
      if (last) {
        for (int i = 0; i < L->l; ++i) logits[i] = acc[i];
        *cls = orc_argmax_i64(acc, L->l);
        free(acc);
        free(act);
        return 0;
      }
      int8_t* b = (int8_t*)malloc((size_t)L->l);
      orc_binarize_i64(acc, L->l, L->l, L->thr, L->flip, b);
      free(acc);
      free(act);
      act = b;
      flat = L->l;
    } else {
      free(act);
      return -1;
    }
  }
  free(act);
  return -1;
}
