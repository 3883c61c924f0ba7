/*
 * bnn.h -- C ABI of libbnn.so, the B200 (sm_100a) bit-packed XNOR-popcount forward
 * pass of the binarized CNN of Khan, Huttunen, Boutellier, "Binarized Convolutional
 * Neural Networks for Efficient Inference on GPUs" (EUSIPCO 2018, arXiv 1808.00209).
 *
 * Citations are PAPER.md:<line> (section / equation) of the paper text; "R<n>" are the
 * numbered readings of ambiguous passages in DESIGN.md §3.
 *
 * ---------------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ---------------------------------------------------------------------------------
 * Memory.   Every tensor pointer is a DEVICE pointer (cudaMalloc / PyTorch caching
 *           allocator) owned by the caller, except where an argument is documented
 *           as HOST.  The library never frees caller memory.  Tensors are dense,
 *           row-major, NHWC.  Pointers must be 16-byte aligned (else BNN_E_ALIGN).
 * Packed.   A packed tensor stores +/-1 values as uint32 words (Eq. 2, PAPER.md:186-195,
 *           with B = 32 along the channel axis, R2): channel c of a pixel -> word c/32,
 *           bit 31 - (c mod 32) (MSB-first); bit 1 <-> +1, bit 0 <-> -1; bits past the
 *           last channel ("pad bits") are 0.  A packed [n,h,w,c] tensor has
 *           ceil(c/32) words per pixel ("cw").
 * Streams.  Every call enqueues work on `stream` (NULL = legacy default stream) and
 *           returns before it completes, except bnn_forward_host (documented below).
 *           No call synchronizes the device on the hot path.
 * Errors.   Every call returns a bnn_status.  Arguments, shapes and alignment are
 *           validated before anything is launched; a launch failure is reported as
 *           BNN_E_CUDA.  No exception or abort crosses the ABI.  bnn_last_error()
 *           returns a thread-local, human-readable message for the last non-OK status
 *           of the calling thread.
 * Threads.  All functions are reentrant.  A bnn_net is immutable after creation but
 *           owns one workspace: calls on one net must be serialized by the caller
 *           (same stream, or external ordering).
 */
#ifndef BNN_H
#define BNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BNN_API __attribute__((visibility("default")))
#else
#define BNN_API
#endif

/* Same type as cudaStream_t; declared here so the header needs no CUDA headers. */
typedef struct CUstream_st* bnn_stream_t;

typedef enum {
  BNN_OK = 0,
  BNN_E_ARG = 1,         /* bad parameter (null pointer, negative size, bad enum)      */
  BNN_E_SHAPE = 2,       /* shapes do not chain / do not match                          */
  BNN_E_UNSUPPORTED = 3, /* valid but not implemented (e.g. even k, k > 7)              */
  BNN_E_ALIGN = 4,       /* pointer not 16-byte aligned                                  */
  BNN_E_CONFIG = 5,      /* mode / dtype combination not allowed                        */
  BNN_E_PADBITS = 6,     /* a packed weight word has nonzero pad bits                   */
  BNN_E_CUDA = 7,        /* CUDA runtime error (launch, allocation, copy)               */
  BNN_E_NOMEM = 8        /* host allocation failed                                      */
} bnn_status;

typedef enum {
  BNN_BITS = 0, /* packed uint32 words (see above)       */
  BNN_U8 = 1,   /* uint8                                 */
  BNN_F32 = 2,  /* float32                               */
  BNN_I32 = 3,  /* int32                                 */
  BNN_I8 = 4    /* int8                                  */
} bnn_dtype;

/* Input binarization, Section 2.3. */
typedef enum {
  BNN_SIGN = 0,        /* bit = x > 0                        (Eq. 1; also packs weights)    */
  BNN_THRESH_RGB = 1,  /* bit_c = x_c + T_c > 0, evaluated as x_c > -T_c in fp32 (R13, R14) */
  BNN_THRESH_GRAY = 2, /* Y = luma(R,G,B) (R15), bit = Y + T_0 > 0; 3 channels -> 1         */
  BNN_LBP = 3,         /* Y = luma; bit_j = Y(n_{3j}) > Y(centre), j = 0,1,2, neighbours
                          clockwise from top-left, replicate border (R16); 3 -> 3           */
  BNN_MODE_NONE = -1   /* no input binarization: the first conv reads real pixels (R5)     */
} bnn_pack_mode;

/* Thread-local text of the last non-OK status returned to this thread ("" if none). */
BNN_API const char* bnn_last_error(void);

/* ABI version (major * 100 + minor). */
BNN_API int bnn_version(void);

/* Process-wide tuning / test knobs (not thread-safe against concurrent launches):
 *   "conv_algo"     first-layer kernel choice for c_in < 32: 0 = automatic (default);
 *                   1 = generic one-word-per-tap conv; 2 = dense-patch kernel; 3 = strip
 *                   kernel (lane = channel); 4 = strip kernel (lane = pixel).
 *   "tiles_per_cta" 0 = automatic (default); k > 0 = every conv CTA walks k output tiles.
 *   "gemv_max_n"    dense layers over n <= value images use the GEMV kernel (default 255).
 *   "conv_tc"       1 (default): binary convs run on tcgen05 tensor cores where an instantiation
 *                   exists; 0: XOR-popcount integer pipe only (Eq. 4).
 *   "conv_tc_fp4"   1 (default): tensor-core convs use packed e2m1 operands (kind::mxf4); 0: int8.
 *   "conv_pool_tc"  1 (default): pooled 32-channel convs fold the 2x2 window into the MMA N.
 *   "conv_pair"     1 (default): inside a net, conv1_fp4 and the pooled 32-channel conv run as CTA pairs
 *                   (cta_group::2, M = 256: each SM stages half of the weight operand); 0: one CTA per
 *                   M = 128 tile.
 *   "first_pool_tc" 1 (default): pooled first layers use the pool-window-ordered kernels.
 *   "first_tma"     1 (default): pooled u8 RGB / SIGN first layers use the TMA-fed kernel.
 *   "first_fp4"     1 (default): binarized pooled u8 first layers run conv1_fp4_pool_kernel (kind::mxf4,
 *                   {0,1} activations, one CTA per SM); 0: the int8 TMA kernel (kind::i8).
 *   "luma_fused"    1 (default): a THRESH_GRAY net's first layer computes the luma from the raw RGB box itself
 *                   (no intermediate image); 2: LBP nets too (slower than the pre-pass, a comparison path);
 *                   0: both go through luma_u8img4_kernel's 0/1 image.
 *   "luma_band"     1 (default): the GRAY / LBP pre-pass of the TMA first layer stages bands of image rows in
 *                   shared memory and computes each luma once (luma_band_kernel); 0: luma_u8img4_kernel.
 *   "first_real_tma" 1 (default): pooled real-u8 first layers (mode NONE, c_in = 3) use the same TMA
 *                   kernel with the pixels as the unsigned int8 operand; 0: the register-staged kernel.
 *   "first_db"      1 (default): that (int8) kernel double-buffers its TMEM accumulators (2 CTAs/SM);
 *                   0: one accumulator set (3 CTAs/SM).
 *   "first_exp"     diagnostics build only (libbnn_trace.so, tools/time_first_exp.py): timing experiments
 *                   that skip work.  libbnn.so does not know the key (BNN_E_ARG) and its kernels contain
 *                   none of the experiment branches.
 *   "csa"           1 (default): the XOR-popcount conv compresses each kernel row's K XOR words
 *                   with carry-save adders (LOP3) before POPC; 0: one POPC per word (Eq. 4 as printed).
 *   "big_img"       1 (default): the streamed wide-channel conv expands its weights once per call
 *                   (stream-ordered scratch) and bulk-copies a stage per step; 0: expands per tile.
 *   "streams"       2 (default): bnn_forward alternates chunks over the caller's stream and an
 *                   internal second stream (own workspace; joined back before returning); 1: one.
 *   "dense_tc"      1 (default): dense layers over n >= 256 images run on tensor cores.
 *   "dense_tma"     1 (default): such a layer's activation stages arrive by TMA (4-deep ring); 0: register
 *                   prefetch one stage ahead.
 *   "dense_ksplit"  1 (default): such a layer splits K over up to 4 CTA groups (+ a reduction kernel)
 *                   when its 128-image tile grid would leave SMs idle; 0: no split.
 *   "pdl"           1 (default): forward-path kernels use programmatic dependent launch.
 *   "fused_max_n"   forward chunks of n <= value images (default 12; 0 = off) of a vehicle-shaped net run as
 *                   one whole-network kernel (a 16-CTA thread-block cluster; `fused_cluster` 0: cooperative grid).
 *   "fused_multi"   1 (default): that kernel runs one cluster per image of the chunk (up to the clusters the device
 *                   holds at once; a cluster serves images i, i + clusters, ...); 0: one cluster for the whole chunk.
 *   "fused_cs"      0 (default): 16-CTA clusters while the chunk's images fit in one wave of them (7 on a B200), else
 *                   8-CTA clusters; 8: always 8-CTA clusters.
 *   "fused_tc"      1 (default): that cluster kernel runs conv2 (k = 5, 32 -> 32 channels) and, for a 5x5x3 conv1,
 *                   conv1 on the tensor cores; 0: the integer pipe.
 *   "alg1"          0 (default); 1: bnn_forward runs the paper's own design instead -- Alg. 1
 *                   im2col + packing (B = k*k), tiled XOR-popcount GEMM, int32 max-pool, 64-segment
 *                   FC -- as a comparison baseline (u8 SIGN / THRESH_RGB nets,
 *                   k <= 5, no thresholds / flips; else BNN_E_UNSUPPORTED).
 * Results are bit-identical for every setting (tiling / kernel-choice invariance is a parity test):
 * no option of libbnn.so can make a call return a non-exact result.
 * Returns BNN_OK or BNN_E_ARG for an unknown key. */
BNN_API int bnn_set_option(const char* key, int value);

/* Tracing (diagnostics, not the hot path): registers a DEVICE buffer of `cap` uint64 (NULL / 0
 * disables).  While set, the pool-in-N TMA first-layer kernel records, for CTA (0,0), the SM clock
 * of 16 role events per tile iteration it at buf[16 * it + ev]: 0/1/2 MMA issuer after the A-ready
 * wait / before issuing / after commit; 3-7 builder warps 1-5 at A ready; 8-11 epilogue warps after
 * the accumulator-ready wait; 12 builder warp 1 after the A-buffer-free wait; 13 epilogue warp at
 * accumulator release.
 * Process-wide; not thread-safe against concurrent launches.  Recording is compiled only into the
 * diagnostics build (`python -m paper_1808_00209_b200._build --trace` -> libbnn_trace.so); the
 * production library returns BNN_E_UNSUPPORTED for a non-NULL buffer.  Errors: BNN_E_ARG. */
BNN_API bnn_status bnn_set_trace(unsigned long long* buf, int cap);

/* ---------------------------------------------------------------------------------
 * bnn_pack -- sign-and-pack (Eq. 1 + Eq. 2; Section 2.3 input binarization).
 *   x    : [n, h, w, c] of dtype dt (BNN_U8, BNN_I8, BNN_F32, BNN_I32).
 *   mode : BNN_SIGN / BNN_THRESH_RGB / BNN_THRESH_GRAY / BNN_LBP.
 *   T    : device float[c] for THRESH_RGB, float[1] for THRESH_GRAY, NULL otherwise.
 *   y    : packed [n, h, w, ceil(c_out/32)], c_out = c (SIGN, RGB), 1 (GRAY), 3 (LBP).
 * GRAY and LBP require c == 3 (RGB order) and dt == BNN_U8 (integer luma, R15).
 * Packing weights: a [c_out, k, k, c_in] +/-1 tensor is n = c_out, h = w = k, c = c_in;
 * a dense [l, d] matrix is n = l, h = w = 1, c = d.
 * Errors: BNN_E_ARG, BNN_E_CONFIG, BNN_E_ALIGN, BNN_E_CUDA.
 * ------------------------------------------------------------------------------- */
BNN_API bnn_status bnn_pack(const void* x, bnn_dtype dt, int n, int h, int w, int c, int mode, const float* T,
                    uint32_t* y, bnn_stream_t stream);

/* ---------------------------------------------------------------------------------
 * bnn_conv2d -- binary convolution, Eq. (3) computed with
 * Eq. (4), fused with the Eq. (1) threshold + Eq. (2) pack and an
 * optional 2x2 OR max-pool (Table 2).
 *
 * Stride 1, "same" output size, odd k in {1, 3, 5, 7}, no bias (R7).
 *   x_dt == BNN_BITS : x packed [n, h, w, ceil(c_in/32)]; positions outside the map are
 *                      -1 (R4).  acc[o] = k*k*c_in - 2 * sum popc(x XOR wt)  (exact).
 *   x_dt == BNN_U8 / BNN_F32 : "no input binarization" first layer:
 *                      x real [n, h, w, c_in] with c_in <= 32, zero padding (R5);
 *                      acc = sum (+/-x) is exact int32 for u8 and fp32 for f32 (R18).
 *   wt   : packed [c_out, k, k, ceil(c_in/32)] (pad bits must be 0).
 *   thr  : int32[c_out] or NULL (= 0); flip : uint8[c_out] or NULL (= 0):
 *          bit_o = (acc_o > thr_o) XOR flip_o  (thr = flip = 0 is Eq. 1; acc = 0 -> -1).
 *          For F32 input the compare is acc > (float)thr_o.
 *   pool : 1 (none) or 2 (2x2 stride-2 OR of the thresholded bits; h, w even) (R9).
 *   y    : packed [n, h/pool, w/pool, ceil(c_out/32)] or NULL.
 *   acc  : NULL, or the pre-threshold accumulators [n, h, w, c_out] (int32; float32
 *          for F32 input) -- a debug / parity output.  At least one of y, acc non-NULL.
 * Errors: BNN_E_ARG, BNN_E_SHAPE (odd h/w with pool 2), BNN_E_UNSUPPORTED (k),
 *         BNN_E_CONFIG (real input with c_in > 32), BNN_E_ALIGN, BNN_E_CUDA.
 * ------------------------------------------------------------------------------- */
BNN_API bnn_status bnn_conv2d(const void* x, bnn_dtype x_dt, int n, int h, int w, int c_in, const uint32_t* wt,
                      int c_out, int k, const int32_t* thr, const uint8_t* flip, int pool, uint32_t* y,
                      void* acc, bnn_stream_t stream);

/* ---------------------------------------------------------------------------------
 * bnn_maxpool -- 2x2 stride-2 max-pooling of a packed map as a word-wise OR
 * (max over {-1,+1} is OR of the bits; Table 2).
 *   x : packed [n, h, w, ceil(c/32)], h and w even; y : packed [n, h/2, w/2, ceil(c/32)].
 * Errors: BNN_E_ARG, BNN_E_SHAPE, BNN_E_ALIGN, BNN_E_CUDA.
 * ------------------------------------------------------------------------------- */
BNN_API bnn_status bnn_maxpool(const uint32_t* x, int n, int h, int w, int c, uint32_t* y, bnn_stream_t stream);

/* ---------------------------------------------------------------------------------
 * bnn_dense -- binary fully connected layer (Section 3.2) over a batch:
 *   acc[i, o] = d - 2 * sum_j popc(x[i, j] XOR wt[o, j])   (Eq. 4, exact)
 *   x   : packed [n, ceil(d/32)] (an NHWC map with c % 32 == 0 is already this, d = h*w*c,
 *         HWC flatten order R11).     wt : packed [l, ceil(d/32)].
 *   thr, flip : as bnn_conv2d, per output.
 *   y   : packed [n, ceil(l/32)] thresholded outputs, or NULL.
 *   acc : int32 [n, l] or NULL (the logits of a last layer).
 *   cls : int32 [n] argmax over l (first maximum wins, R19), or NULL; needs acc semantics
 *         only, l <= 1024.
 * Exact for every d: the tensor-core kernel (fp32 accumulators) is used only while d <= 2^24,
 * wider layers run on the XOR-popcount kernel (int32 accumulators).
 * Errors: BNN_E_ARG, BNN_E_ALIGN, BNN_E_CUDA.
 * ------------------------------------------------------------------------------- */
BNN_API bnn_status bnn_dense(const uint32_t* x, int n, int64_t d, const uint32_t* wt, int l, const int32_t* thr,
                     const uint8_t* flip, uint32_t* y, int32_t* acc, int32_t* cls, bnn_stream_t stream);

/* ---------------------------------------------------------------------------------
 * bnn_affine -- float output scaling of a last layer's integer logits (SURVEY f4 variant:
 * BinaryNet's output batch-normalisation folded to a per-class affine map -- BinaryNet is the
 * paper's BNN reference, PAPER.md:74 -- and XNOR-Net's per-output scaling factor, bias 0):
 *   score[i, o] = fmaf(scale[o], (float)acc[i, o], bias[o])    (fp32, ONE rounding; |acc| < 2^24)
 *   cls[i]      = first maximum of score[i, :]  (R19; the decision is taken on the fp32 scores, R25)
 *   acc : DEVICE int32 [n, l];  scale, bias : DEVICE float32 [l] (finite);  1 <= l <= 1024.
 *   score : DEVICE float32 [n, l] or NULL;  cls : DEVICE int32 [n] or NULL (not both NULL).
 * Errors: BNN_E_ARG, BNN_E_ALIGN, BNN_E_CUDA.
 * ------------------------------------------------------------------------------- */
BNN_API bnn_status bnn_affine(const int32_t* acc, int n, int l, const float* scale, const float* bias, float* score,
                              int32_t* cls, bnn_stream_t stream);

/* ---------------------------------------------------------------------------------
 * Network handle: the whole forward pass of Section 2 / Table 2:
 *   [input binarization] -> conv (+threshold, +pool) ... -> dense ... -> int32 logits.
 * ------------------------------------------------------------------------------- */
typedef struct bnn_net bnn_net;

typedef struct {
  int kind;            /* 1 = conv, 2 = dense                                        */
  int k;               /* conv kernel size (odd)                                     */
  int c_out;           /* conv output channels                                       */
  int pool;            /* conv: 1 or 2                                               */
  int l;               /* dense outputs                                              */
  const uint32_t* wt;  /* DEVICE packed weights (conv [c_out,k,k,cw]; dense [l,dw])  */
  const int32_t* thr;  /* DEVICE int32 per output, or NULL                           */
  const uint8_t* flip; /* DEVICE uint8 per output, or NULL                           */
} bnn_layer;

/* Creates a net for [*, h, w, c] images of dtype in_dt (BNN_U8 or BNN_F32).
 *   mode : a bnn_pack_mode; BNN_MODE_NONE makes layer 0 a real-input conv.
 *   T    : DEVICE thresholds for THRESH_RGB (c floats) / THRESH_GRAY (1 float), else NULL.
 *   layers / n_layers : HOST array, copied.  Weights, thr, flip and T are DEVICE memory owned
 *          by the caller and must outlive the net.  The last layer must be dense; its
 *          outputs are the logits.  conv -> dense requires the conv output channels to be
 *          a multiple of 32 (the packed NHWC map is then the HWC-flattened packed vector).
 *   max_batch : chunk size; bnn_forward processes any n in chunks of at most this many
 *          images, so the device workspace is sized for max_batch images (<= 65536).
 * Validates the chaining, the weight pad bits (one blocking copy of the weights to the
 * host) and allocates the workspace.  Errors: BNN_E_ARG, BNN_E_SHAPE, BNN_E_CONFIG,
 * BNN_E_UNSUPPORTED, BNN_E_PADBITS, BNN_E_CUDA, BNN_E_NOMEM. */
BNN_API bnn_status bnn_net_create(int h, int w, int c, bnn_dtype in_dt, int mode, const float* T, const bnn_layer* layers,
                          int n_layers, int max_batch, bnn_net** out);

/* images: DEVICE [n, h, w, c] of the net's dtype -> logits DEVICE int32 [n, l_last] (may be
 * NULL), cls DEVICE int32 [n] (argmax, first maximum wins; may be NULL).  Asynchronous. */
BNN_API bnn_status bnn_forward(bnn_net* net, const void* images, int n, int32_t* logits, int32_t* cls,
                       bnn_stream_t stream);

/* bnn_forward followed by bnn_affine on the last layer's logits: images DEVICE -> logits DEVICE
 * int32 [n, l_last] (required: the integer logits are kept), scores DEVICE float32 [n, l_last]
 * (may be NULL), cls DEVICE int32 [n] = first maximum of the fp32 scores (may be NULL; not both
 * NULL).  scale / bias: DEVICE float32 [l_last].  Asynchronous.  Errors as bnn_forward and
 * bnn_affine (BNN_E_UNSUPPORTED for l_last > 1024). */
BNN_API bnn_status bnn_forward_scores(bnn_net* net, const void* images, int n, const float* scale, const float* bias,
                                      int32_t* logits, float* scores, int32_t* cls, bnn_stream_t stream);

/* End-to-end variant: HOST images (pinned for full speed; pageable works) -> HOST logits /
 * cls.  Copies chunks host->device, runs the forward pass and copies results back,
 * overlapping copies with compute on an internal copy stream.  SYNCHRONOUS: returns after
 * the results are in host memory.  Errors as bnn_forward. */
BNN_API bnn_status bnn_forward_host(bnn_net* net, const void* h_images, int n, int32_t* h_logits, int32_t* h_cls,
                            bnn_stream_t stream);

/* Latency path for small batches (BASELINE config 1; the paper's protocol PAPER.md:135-137 times
 * the kernels of one image after its copy to the device).  bnn_net_staging allocates (once) device
 * staging buffers owned by the net for up to max_staged (<= 256) images and returns them: the
 * caller writes images to *in ([max_staged, h, w, c] of the net's dtype) and reads *logits
 * ([max_staged, l_last] int32) / *cls ([max_staged] int32).  bnn_forward_staged(net, n, stream)
 * runs the forward pass of the first n staged images; the first call for a given n captures the
 * whole pass into a CUDA graph, later calls replay it as ONE graph launch.  Asynchronous.
 * Errors: BNN_E_ARG (n > max_staged or no staging), BNN_E_CUDA. */
BNN_API bnn_status bnn_net_staging(bnn_net* net, int max_staged, void** in, int32_t** logits, int32_t** cls);
BNN_API bnn_status bnn_forward_staged(bnn_net* net, int n, bnn_stream_t stream);

/* Name of the CUDA kernel family bnn_forward uses for `layer` when running n images (e.g.
 * "conv_tc_kernel", "conv_first_tc_kernel", "conv_bin_kernel", "dense_kernel"); "" if out of range.
 * For measurement labelling (bench.py roofline) and tests. */
BNN_API const char* bnn_net_layer_kernel(const bnn_net* net, int layer, int n);

/* Number of kernel launches one bnn_forward of n images enqueues (for launch accounting). */
BNN_API int bnn_forward_launches(const bnn_net* net, int n);

/* Per-stage device timing of bnn_forward (CUDA events recorded on the forward stream around
 * every launch; stage 0 = input pack, stage i+1 = layer i, stage n_layers+1 = argmax).
 * bnn_net_profile(net, 1) resets the totals and starts recording; (net, 0) stops.
 * bnn_net_profile_read waits for the recorded events, adds their durations to the totals and
 * writes, for each of the first `cap` stages, the total milliseconds and launch count since the
 * last reset.  Returns the number of stages (n_layers + 2) or a negative bnn_status. */
BNN_API int bnn_net_profile(bnn_net* net, int enable);
BNN_API int bnn_net_profile_read(bnn_net* net, double* ms, int64_t* launches, int cap);

BNN_API void bnn_net_destroy(bnn_net* net);

#ifdef __cplusplus
}
#endif
#endif /* BNN_H */
