/*
 * bnn_oracle.h -- CPU ORACLE for the binarized-CNN forward pass of
 * Khan, Huttunen, Boutellier, "Binarized Convolutional Neural Networks for
 * Efficient Inference on GPUs" (EUSIPCO 2018, arXiv 1808.00209).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1808_00209_b200/csrc, include/bnn.h); neither side includes the other.
 *
 * Everything here is the plain definition, written on UNPACKED +/-1 values
 * (int8_t, -1 or +1), int64 accumulators and double for the real-valued
 * first layer.  No bit tricks, no blocking, no reordering.
 * Citations are "PAPER.md:<line>" (section / equation) into the paper text;
 * the readings of ambiguous passages are the numbered readings of DESIGN.md §3.
 *
 * Layouts: images and feature maps are HWC (one image); conv weights are
 * [c_out][k][k][c_in] (OHWI); dense weights are [l][d] with d in HWC flatten
 * order (reading R11).
 *
 * Parity pins: see DESIGN.md §4.  orc_forward's end-to-end accuracy against
 * the paper's Table 3 is "parity unpinned" (needs the paper's dataset/weights).
 */
#ifndef BNN_ORACLE_H
#define BNN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Input-binarization modes, PAPER.md:141-145 (Thresholding) and 178-179 (LBP). */
enum { ORC_SIGN = 0, ORC_THRESH_RGB = 1, ORC_THRESH_GRAY = 2, ORC_LBP = 3, ORC_NONE = -1 };

/* Eq. (1): sign(x) = -1 if x <= 0, +1 if x > 0. */
int orc_sign(double x);

/* Eq. (2): packing of a +/-1 vector of length D into words of
 * B <= 32 bits, evaluated arithmetically as sum_i (1+x_i) 2^(B-2-mod(i-1,B))
 * (reading R1: the factor (1+x_i) in {0,2} makes element i land on bit
 * B-1-mod(i-1,B); x_p is a vector of integers, not of +/-1).  A final partial
 * word holds D mod B elements at its top B-bit positions (reading R12), all
 * other bits 0.  Returns the number of words ceil(D/B), or -1 on bad B. */
int64_t orc_pack(const int8_t* x, int64_t D, int B, uint32_t* words);

/* Inverse of Eq. (2): bit B-1-mod(i-1,B) of word ceil(i/B) -> x_i.  Returns 0,
 * -1 on bad B, or -2 if any bit outside the valid positions is set. */
int orc_unpack(const uint32_t* words, int64_t D, int B, int8_t* x);

/* Integer Rec.601 luma, reading R15: (299 R + 587 G + 114 B + 500) div 1000. */
int orc_luma(int r, int g, int b);

/* Section 2.3 input binarization.
 *   x: one HWC image as doubles (exact conversions of u8 / i8 / f32 / i32 data).
 *   ORC_SIGN:        out[h][w][c] = sign(x)                        (c channels)
 *   ORC_THRESH_RGB:  out[h][w][c] = sign(x + T[c])   (R13/R14)      (c channels)
 *   ORC_THRESH_GRAY: out[h][w][0] = sign(luma + T[0]) (c must be 3; R15)
 *   ORC_LBP:         out[h][w][j] = +1 iff luma(neighbour n_{3j}) > luma(centre),
 *                    neighbours n0..n7 clockwise from top-left, replicate border
 *                    (R16; c must be 3)
 * Returns the number of output channels, or -1 on a bad argument. */
int orc_binarize_input(const double* x, int h, int w, int c, int mode, const double* T, int8_t* out);

/* Eq. (3), binary layer: cross-correlation of a +/-1 map
 * x[h][w][c_in] with +/-1 kernels wt[c_out][k][k][c_in], stride 1, same size,
 * odd k, radius R=(k-1)/2, positions outside the map take the value -1
 * (reading R4: Alg. 1 binarizes a zero-initialised buffer with "> 0").
 *   acc[y][x][o] = sum_{ky,kx,c} wt[o][ky][kx][c] * xp[y+ky-R][x+kx-R][c]      */
void orc_conv_binary(const int8_t* x, int h, int w, int c_in, const int8_t* wt, int c_out, int k,
                     int64_t* acc);

/* Eq. (3), binary layer, ONE output: acc[y][x][o] of orc_conv_binary, for sampled parity at
 * sizes where the whole map is too slow.  wt_o: the kernel of channel o, [k][k][c_in]. */
int64_t orc_conv_binary_point(const int8_t* x, int h, int w, int c_in, const int8_t* wt_o, int k, int y, int xx);

/* Eq. (3) for the real-valued first layer ("No input binarization", PAPER.md:380,
 * Table 1 "BCNN" row PAPER.md:291): same sum on real x with zero padding (R5). */
void orc_conv_real(const double* x, int h, int w, int c_in, const int8_t* wt, int c_out, int k,
                   double* acc);

/* Eq. (1) applied per channel with an optional integer threshold and flip
 * (reading R9/R-BN): out = ((acc > thr[ch]) != flip[ch]) ? +1 : -1.
 * thr == NULL means thr = 0 and flip == NULL means flip = 0, which is exactly
 * Eq. (1) (acc = 0 -> -1).  ch = index mod c. */
void orc_binarize_i64(const int64_t* acc, int64_t count, int c, const int32_t* thr,
                      const uint8_t* flip, int8_t* out);
void orc_binarize_f64(const double* acc, int64_t count, int c, const int32_t* thr,
                      const uint8_t* flip, int8_t* out);

/* 2x2 / stride-2 max-pooling of a +/-1 map (Table 2 rows "Max-Pooling",
 * PAPER.md:327,330): y[i][j][c] = max of the four x values.  h, w even. */
void orc_maxpool2(const int8_t* x, int h, int w, int c, int8_t* y);

/* Fully connected layer: acc[l] = sum_d W[l][d] * x[d]. */
void orc_dense(const int8_t* x, int64_t d, const int8_t* W, int l, int64_t* acc);

/* First maximum wins (reading R19). */
int orc_argmax_i64(const int64_t* v, int l);

/* Float output scaling of the last layer (SURVEY f4 variant): BinaryNet's output batch
 * normalisation folded to a per-class affine map (BinaryNet is the paper's ref. for BNNs,
 * PAPER.md:74) and XNOR-Net's per-output scaling factor alpha (bias 0) both take the form
 *   score[o] = scale[o] * acc[o] + bias[o].
 * score64: the value in double (the tolerance comparison, 1e-5 relative per north_star);
 * score32: the same value in fp32 with ONE rounding (fmaf; exact float(acc) for |acc| < 2^24),
 * the precision the argmax decision is taken in on both sides (R25).  Either may be NULL. */
void orc_affine(const int64_t* acc, int l, const float* scale, const float* bias, double* score64,
                float* score32);

/* First maximum wins over fp32 scores (R19, R25). */
int orc_argmax_f32(const float* v, int l);

/* A network for orc_forward.  kind 1 = conv (k, c_out, pool in {1,2}),
 * kind 2 = dense (l).  Hidden layers are binarized with thr/flip (NULL = Eq. 1);
 * the last layer must be dense and returns integer logits. */
typedef struct {
  int kind, k, c_out, pool, l;
  const int8_t* wt;
  const int32_t* thr;
  const uint8_t* flip;
} orc_layer;

/* Whole forward pass for ONE image (Section 2 pipeline, Table 2 layer order
 * PAPER.md:325-331):  input binarization (mode; ORC_NONE = real first layer)
 * -> [conv -> binarize -> (pool)]* -> flatten HWC -> [dense -> binarize]* -> dense
 * -> int64 logits, argmax.  x: the image as doubles.  Returns 0 or -1.
 * logits must hold the last layer's l values. */
int orc_forward(const double* x, int h, int w, int c, int mode, const double* T, const orc_layer* layers,
                int n_layers, int64_t* logits, int32_t* cls);

#ifdef __cplusplus
}
#endif
#endif
