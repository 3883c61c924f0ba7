// k_dense.cuh -- binary fully connected layer as a packed XOR-popcount GEMM over the batch
// (Section 3.2; Eq. 4), the 2x2 OR max-pool
// (Table 2) and the argmax of the logits.
//
// Dense mapping: lane = output neuron (a group of 32 outputs per blockIdx.y), each warp owns
// PI images, activations are warp-broadcast 16-byte smem reads, weights per-lane smem reads.
// The paper's 64-segment shared-memory reduction without synchronisation is
// pre-Volta warp-synchronous code; here every output is one thread's register sum, no
// cross-thread reduction is needed at all for batch >= 1.
#pragma once
#include <climits>
#include "common.cuh"

namespace bnn {

struct DenseArgs {
  const uint32_t* x;   // packed [n, dw]
  const uint32_t* wt;  // packed [l, dw]
  const int32_t* thr;
  const uint8_t* flip;
  uint32_t* y;    // packed [n, lw] or null
  int32_t* acc;   // [n, l] or null
  int32_t* cls;   // [n] or null (only when l <= 32: one group holds all outputs)
  int n, l, lw;
  int64_t d, dw;
  int ks;        // dense_tc4: K split over gridDim.z (1 = none)
  float* part;   // ks > 1: partial sums [ks][ntiles * 128][gridDim.y * NT] (stream-ordered scratch)
  const uint8_t* bimg;  // dense_tc4: pre-expanded e2m1 weight image [group][stage][word][NT][16 B] or null
};

template <int PI, int NWARP, int DC>
__global__ void __launch_bounds__(NWARP * 32)
dense_kernel(const DenseArgs A) {
  griddep_launch();
  griddep_wait();
  constexpr int NT = NWARP * 32;
  constexpr int NIMG = PI * NWARP;
  constexpr int XP = DC + 4;  // row pitch of the activation tile (keeps 16 B alignment)
  __shared__ __align__(16) uint32_t xs[NIMG * XP];
  __shared__ __align__(16) uint32_t ws[DC * 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  const int o = g * 32 + lane;
  const bool ovalid = o < A.l;
  const int img0 = blockIdx.x * NIMG;

  int acc[PI];
#pragma unroll
  for (int i = 0; i < PI; ++i) acc[i] = 0;

  for (int64_t c0 = 0; c0 < A.dw; c0 += DC) {
    const int nc = (int)min((int64_t)DC, A.dw - c0);
    const int ncp = (nc + 3) & ~3;
    __syncthreads();
    for (int i = tid; i < NIMG * ncp; i += NT) {
      const int j = i % ncp, im = i / ncp;
      const int gi = img0 + im;
      xs[im * XP + j] = (j < nc && gi < A.n) ? __ldg(A.x + (int64_t)gi * A.dw + c0 + j) : 0u;
    }
    for (int i = tid; i < 32 * ncp; i += NT) {
      const int j = i % ncp, l = i / ncp;
      const int oo = g * 32 + l;
      ws[j * 32 + l] = (j < nc && oo < A.l) ? __ldg(A.wt + (int64_t)oo * A.dw + c0 + j) : 0u;
    }
    __syncthreads();
    for (int j = 0; j < ncp; j += 4) {
      const uint32_t w0 = ws[j * 32 + lane], w1 = ws[(j + 1) * 32 + lane];
      const uint32_t w2 = ws[(j + 2) * 32 + lane], w3 = ws[(j + 3) * 32 + lane];
#pragma unroll
      for (int i = 0; i < PI; ++i) {
        const uint4 q = *reinterpret_cast<const uint4*>(xs + (warp * PI + i) * XP + j);
        acc[i] += popc(q.x ^ w0) + popc(q.y ^ w1) + popc(q.z ^ w2) + popc(q.w ^ w3);
      }
    }
  }

  const int t = (A.thr != nullptr && ovalid) ? A.thr[o] : 0;
  const bool f = (A.flip != nullptr && ovalid) ? (A.flip[o] != 0) : false;
#pragma unroll
  for (int i = 0; i < PI; ++i) {
    const int gi = img0 + warp * PI + i;
    const bool img_ok = gi < A.n;
    const int a = (int)A.d - 2 * acc[i];
    if (A.acc != nullptr && img_ok && ovalid) A.acc[(int64_t)gi * A.l + o] = a;
    const uint32_t word = ballot_pack(ovalid && ((a > t) != f));
    if (A.y != nullptr && img_ok && lane == 0) A.y[(int64_t)gi * A.lw + g] = word;
    if (A.cls != nullptr) {
      // argmax across the lanes, first maximum wins (R19)
      int bv = ovalid ? a : INT_MIN, bi = ovalid ? o : INT_MAX;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, s);
        const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, s);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (img_ok && lane == 0) A.cls[gi] = bi;
    }
  }
}

// Small-batch dense (GEMV, the paper's batch-1 case, Section 3.2): one CTA per (image, group of
// 32 outputs), warp w computes output g*32 + w with its lanes striding over the dw words (16-byte
// loads when dw % 4 == 0) and one __reduce_add_sync; warp 0 then thresholds, packs (brev(ballot))
// and takes the argmax.  No image slots are wasted at n = 1 (the GEMM kernel computes 64 per CTA).
__global__ void __launch_bounds__(1024)
dense_gemv_kernel(const DenseArgs A) {
  griddep_launch();
  griddep_wait();
  __shared__ int part[32];
  const int img = blockIdx.x, g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int o = g * 32 + warp;
  int acc = 0;
  if (o < A.l) {
    const uint32_t* xr = A.x + (int64_t)img * A.dw;
    const uint32_t* wr = A.wt + (int64_t)o * A.dw;
    if ((A.dw & 3) == 0) {
      const uint4* x4 = reinterpret_cast<const uint4*>(xr);
      const uint4* w4 = reinterpret_cast<const uint4*>(wr);
      for (int64_t j = lane; j < (A.dw >> 2); j += 32) {
        const uint4 a = __ldg(x4 + j), b = __ldg(w4 + j);
        acc += popc(a.x ^ b.x) + popc(a.y ^ b.y) + popc(a.z ^ b.z) + popc(a.w ^ b.w);
      }
    } else {
      for (int64_t j = lane; j < A.dw; j += 32) acc += popc(__ldg(xr + j) ^ __ldg(wr + j));
    }
  }
  acc = __reduce_add_sync(BNN_FULL_MASK, acc);
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (warp != 0) return;
  const int oo = g * 32 + lane;
  const bool ovalid = oo < A.l && lane < (int)(blockDim.x >> 5);
  const int a = ovalid ? (int)A.d - 2 * part[lane] : 0;
  if (A.acc != nullptr && ovalid) A.acc[(int64_t)img * A.l + oo] = a;
  const int t = (A.thr != nullptr && ovalid) ? A.thr[oo] : 0;
  const bool f = (A.flip != nullptr && ovalid) ? (A.flip[oo] != 0) : false;
  const uint32_t word = ballot_pack(ovalid && ((a > t) != f));
  if (A.y != nullptr && lane == 0) A.y[(int64_t)img * A.lw + g] = word;
  if (A.cls != nullptr) {
    int bv = ovalid ? a : INT_MIN, bi = ovalid ? oo : INT_MAX;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, s);
      const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, s);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) A.cls[img] = bi;
  }
}

// argmax over int32 logits [n, l], first maximum wins (R19).  One warp per image.
__global__ void argmax_kernel(const int32_t* __restrict__ logits, int n, int l, int32_t* __restrict__ cls) {
  griddep_launch();
  griddep_wait();
  const int lane = threadIdx.x & 31;
  for (int64_t img = gtid() >> 5; img < n; img += gstride() >> 5) {
    int bv = INT_MIN, bi = INT_MAX;
    for (int o = lane; o < l; o += 32) {
      const int v = logits[img * l + o];
      if (v > bv) { bv = v; bi = o; }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, s);
      const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, s);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) cls[img] = bi;
  }
}

// Float output scaling of the last layer (BinaryNet's output batch-norm folded to a
// per-class affine map, XNOR-Net's per-output alpha): score = fmaf(scale[o], (float)acc, bias[o]) --
// one rounding, exact float(acc) for |acc| < 2^24 (precondition) -- and the first maximum of the fp32
// scores (R19, R25).  One warp per image, scale / bias staged in shared memory (l <= 1024).
__global__ void affine_argmax_kernel(const int32_t* __restrict__ acc, int n, int l, const float* __restrict__ scale,
                                     const float* __restrict__ bias, float* __restrict__ score,
                                     int32_t* __restrict__ cls) {
  griddep_launch();
  __shared__ float s_sc[1024], s_b[1024];
  for (int o = threadIdx.x; o < l; o += blockDim.x) {
    s_sc[o] = scale[o];
    s_b[o] = bias[o];
  }
  __syncthreads();
  griddep_wait();
  const int lane = threadIdx.x & 31;
  for (int64_t img = gtid() >> 5; img < n; img += gstride() >> 5) {
    float bv = 0.f;
    int bi = INT_MAX;
    for (int o = lane; o < l; o += 32) {
      const float v = __fmaf_rn(s_sc[o], (float)acc[img * l + o], s_b[o]);
      if (score != nullptr) score[img * l + o] = v;
      if (bi == INT_MAX || v > bv) { bv = v; bi = o; }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const float ov = __shfl_xor_sync(BNN_FULL_MASK, bv, s);
      const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, s);
      if (oi != INT_MAX && (bi == INT_MAX || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    if (lane == 0 && cls != nullptr) cls[img] = bi;
  }
}

// 2x2 stride-2 OR pooling of a packed map (max over {-1,+1} == OR of the bits).
__global__ void maxpool_or_kernel(const uint32_t* __restrict__ x, int n, int H, int W, int cw,
                                  uint32_t* __restrict__ y) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)n * Ho * Wo * cw;
  for (int64_t i = gtid(); i < total; i += gstride()) {
    const int wi = (int)(i % cw);
    const int64_t pix = i / cw;
    const int img = (int)(pix / ((int64_t)Ho * Wo));
    const int rem = (int)(pix - (int64_t)img * Ho * Wo);
    const int oy = rem / Wo, ox = rem - oy * Wo;
    const uint32_t* b = x + (((int64_t)img * H + 2 * oy) * W + 2 * ox) * cw + wi;
    y[i] = __ldg(b) | __ldg(b + cw) | __ldg(b + (int64_t)W * cw) | __ldg(b + (int64_t)W * cw + cw);
  }
}

}  // namespace bnn
