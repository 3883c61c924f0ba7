// k_fused_small.cuh -- the whole vehicle-shaped network in ONE kernel launch for small batches
// (the paper's batch-1 protocol, Table 1).
//
// Topology (checked by the host): conv1 on a u8 image (c <= 4 channels, SIGN / THRESH_RGB input
// binarization, K^2 c <= 96, 32 outputs, 2x2 pool) -> conv2 (32 -> 32 channels, K <= 5, 2x2 pool)
// -> dense -> dense -> dense (<= 32 integer logits) -> argmax.  At batch 1 the layers are far too
// small to fill a B200 with one kernel each (the multi-kernel graph is launch- and prologue-bound),
// so one cooperative grid (one 512-thread CTA per SM) runs them all with two grid barriers:
//   phase 1  warp = one conv1 pooled pixel, lane = output channel.  The 4 K x K x c patches of its
//            2x2 window are built with ballots (lane j thresholds the input element of patch bit j,
//            Eq. 1 / R14), then Eq. (4) acc = K^2 c - 2 popc(patch ^ w) per lane, threshold/flip,
//            OR over the window (R9), brev(ballot) packs the 32 channel bits (Eq. 2);
//   phase 2  warp = one conv2 pooled pixel, lane = output channel, 25 weight words per lane in
//            registers, the (K+1)^2 input words are warp-broadcast loads;
//   phase 3  CTA b = image b: FC1 / FC2 with one warp per output (lanes stride the words, one
//            __reduce_add_sync), bits gathered in shared memory; FC3 integer logits + argmax (R19).
// Out-of-map taps are -1 (bit 0, R4).  Everything is integer; results equal the layer-by-layer path.
#pragma once
#include "common.cuh"

namespace bnn {

struct FusedSmallArgs {
  const uint8_t* x;  // u8 [n, H, W, C]
  const float* T;    // [C] input thresholds (THRESH_RGB) or null (SIGN: x > 0)
  int n, H, W, C;
  int K1, K2;
  const uint32_t* w1;  // packed [32, K1, K1, 1]
  const uint32_t* w1p; // [32, 3]: conv1 weights re-packed densely along the K1 x K1 x C patch
  const int32_t* thr1;
  const uint8_t* flip1;
  const uint32_t* w2;  // packed [32, K2, K2, 1]
  const int32_t* thr2;
  const uint8_t* flip2;
  const uint32_t *f1, *f2, *f3;  // dense weights [l, dw]
  const int32_t *thr_f1, *thr_f2;
  const uint8_t *flip_f1, *flip_f2;
  int l1, l2, l3;
  uint32_t* y1;  // [n, H/2, W/2] packed conv1 output (32 channels = 1 word)
  uint32_t* y2;  // [n, H/4, W/4]
  uint32_t* h1;  // [n, ceil(l1/32)] packed FC1 output
  int32_t* logits;  // [n, l3] or null
  int32_t* cls;     // [n] or null
  unsigned* barrier;  // [2]: grid-barrier count, FC1-done count (zero at launch; the tail CTA re-arms them)
  unsigned long long* trace;  // diagnostics build (bnn_set_trace, trace_layer 2): CTA 0's phase globaltimer stamps
  const uint8_t* w2img;       // conv2's pool-in-N e2m1 weight image (prep_tc4_pool_kernel) for the cluster kernel's
                              // tensor-core conv2 phase, or null
  const uint8_t* w1img;       // conv1's e2m1 weight image (prep_conv1_fp4_kernel) for its tensor-core conv1 phase, or null
};

// phase timestamp (ns, %globaltimer) ev of image img into A.trace[img * 8 + ev] (diagnostics build only)
BNN_DEV void fused_trace(const FusedSmallArgs& A, int img, int ev) {
#ifdef BNN_TRACE
  if (A.trace != nullptr && threadIdx.x == 0 && img <= 64) {  // (img 64: kernel-level stamps)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.trace[img * 8 + ev] = t;
  }
#else
  (void)A, (void)img, (void)ev;
#endif
}

constexpr int kFusedWarps = 16;
constexpr int kFusedMaxL = 1024;  // l1, l2 <= this (shared-memory bit buffers)

BNN_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all CTAs of the (cooperatively launched, hence co-resident) grid arrive; `target` = k * gridDim.x
BNN_DEV void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire_u32(ctr) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// One dense layer for one image inside a CTA: x = packed [dw] in shared memory, out bits -> s_out
// (packed, zero-initialised by the caller) or logits.  Warp w takes outputs w, w + 16, ...; the
// weight loads of up to 8 of its outputs are issued together (the batch-1 chain is latency-bound).
// The same for weights, thresholds and flips already in shared memory (fused_cluster_kernel's FC2 / FC3):
// lane = output (a warp covers 32 outputs), each lane loops over the dw input words, and the warp's 32 sign
// bits are one ballot stored as one word (Eq. 2, MSB-first) -- no cross-lane reductions, no atomics.
BNN_DEV void fused_dense_smem(const uint32_t* xs, int64_t d, const uint32_t* w, int l, const int32_t* thr,
                              const int32_t* flip, uint32_t* s_out, int32_t* s_logit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dw = (int)((d + 31) / 32);
  for (int o0 = warp * 32; o0 < l; o0 += kFusedWarps * 32) {
    const int o = o0 + lane;
    const bool ok = o < l;
    int s = 0;
    if (ok)
      for (int j = 0; j < dw; ++j) s += popc(xs[j] ^ w[(int64_t)o * dw + j]);
    const int acc = (int)d - 2 * s;  // Eq. (4)
    if (s_logit != nullptr) {
      if (ok) s_logit[o] = acc;
    } else {
      const uint32_t word = ballot_pack(ok && ((acc > (thr != nullptr ? thr[o] : 0)) != (flip != nullptr && flip[o] != 0)));
      if (lane == 0) s_out[o0 >> 5] = word;
    }
  }
}

BNN_DEV void fused_dense(const uint32_t* xs, int64_t d, const uint32_t* __restrict__ w, int l, const int32_t* thr,
                         const uint8_t* flip, uint32_t* s_out, int32_t* s_logit) {
  constexpr int OB = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dw = (int)((d + 31) / 32);
  for (int o0 = warp; o0 < l; o0 += kFusedWarps * OB) {
    int s[OB];
#pragma unroll
    for (int k = 0; k < OB; ++k) s[k] = 0;
#pragma unroll 6
    for (int j = lane; j < dw; j += 32) {  // unrolled: 48 weight loads in flight per lane
      const uint32_t xv = xs[j];
#pragma unroll
      for (int k = 0; k < OB; ++k) {
        const int o = o0 + k * kFusedWarps;
        if (o < l) s[k] += popc(xv ^ __ldg(w + (int64_t)o * dw + j));
      }
    }
#pragma unroll
    for (int k = 0; k < OB; ++k) {
      const int o = o0 + k * kFusedWarps;
      const int sum = __reduce_add_sync(BNN_FULL_MASK, s[k]);
      if (o < l && lane == 0) {
        const int acc = (int)d - 2 * sum;  // Eq. (4)
        if (s_logit != nullptr) {
          s_logit[o] = acc;
        } else {
          const int t = thr != nullptr ? thr[o] : 0;
          const bool f = flip != nullptr && flip[o] != 0;
          if ((acc > t) != f) atomicOr(&s_out[o >> 5], 1u << (31 - (o & 31)));
        }
      }
    }
  }
}

// conv1 weights [32, K, K, 1 word (C bits)] -> 3 words per output channel, patch bit b =
// (ky K + kx) C + c at word b / 32, bit 31 - b % 32 (pad bits 0); run once per net.
__global__ void prep_fused_w1_kernel(const uint32_t* __restrict__ w1, int K, int C, uint32_t* __restrict__ out) {
  const int o = threadIdx.x;  // 32 threads
  const int nb = K * K * C;
  for (int w = 0; w < 3; ++w) {
    uint32_t v = 0;
    for (int j = 0; j < 32; ++j) {
      const int b = 32 * w + j;
      if (b < nb) {
        const int tp = b / C, c = b - tp * C;
        v |= ((w1[(int64_t)o * K * K + tp] >> (31 - c)) & 1u) << (31 - j);
      }
    }
    out[o * 3 + w] = v;
  }
}

template <int K2>
__global__ void __launch_bounds__(kFusedWarps * 32, 1) fused_small_kernel(const FusedSmallArgs A) {
  __shared__ uint32_t s_h1[kFusedMaxL / 32], s_h2[kFusedMaxL / 32];
  __shared__ int32_t s_logit[32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kFusedWarps + warp, nw = (int64_t)gridDim.x * kFusedWarps;
  const int H1 = A.H >> 1, W1 = A.W >> 1, H2 = H1 >> 1, W2 = W1 >> 1;
  const int lw1 = (A.l1 + 31) / 32;

  // conv2 / FC buffers written with atomicOr below start at zero
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)A.n * H2 * W2; i += (int64_t)gridDim.x * blockDim.x) A.y2[i] = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)A.n * lw1; i += (int64_t)gridDim.x * blockDim.x) A.h1[i] = 0u;
  // conv2 weights of this lane's output channel, loaded while phase 1 runs
  constexpr int KK2 = K2 * K2;
  uint32_t w2[KK2];
#pragma unroll
  for (int i = 0; i < KK2; ++i) w2[i] = __ldg(A.w2 + (int64_t)lane * KK2 + i);
  const int th2 = A.thr2 != nullptr ? A.thr2[lane] : 0;
  const bool fl2 = A.flip2 != nullptr && A.flip2[lane] != 0;

  // ---- phase 1: conv1 + input binarization + pool
  {
    const int K = A.K1, R = (K - 1) / 2, C = A.C, nb = K * K * C, S = nb;
    const int Ho = H1, Wo = W1;
    int t[4] = {0, 0, 0, 0};
    for (int c = 0; c < C; ++c) t[c] = A.T != nullptr ? u8_threshold(-A.T[c]) : 0;
    // patch bit b = 32 w + lane of word w <-> (ky, kx, c), b = (ky K + kx) C + c (MSB-first)
    int dy_[3], dx_[3], ch_[3], tw_[3];
    bool use_[3];
    uint32_t wreg[3];
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      const int b = 32 * w + lane;
      use_[w] = b < nb;
      const int tap = b / C, c = b - tap * C;
      dy_[w] = tap / K - R;
      dx_[w] = tap % K - R;
      ch_[w] = c;
      tw_[w] = c == 0 ? t[0] : (c == 1 ? t[1] : (c == 2 ? t[2] : t[3]));
      // this lane's channel o = lane: word w of its weight patch (pre-packed by prep_fused_w1_kernel)
      const uint32_t v = __ldg(A.w1p + lane * 3 + w);
      wreg[w] = v;
    }
    const int th = A.thr1 != nullptr ? A.thr1[lane] : 0;
    const bool fl = A.flip1 != nullptr && A.flip1[lane] != 0;
    const int64_t units = (int64_t)A.n * Ho * Wo;
    for (int64_t u = gw; u < units; u += nw) {
      const int img = (int)(u / (Ho * Wo));
      const int rem = (int)(u - (int64_t)img * Ho * Wo);
      const int py = rem / Wo, px = rem - py * Wo;
      const uint8_t* xi = A.x + (int64_t)img * A.H * A.W * C;
      bool any = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
        int pc = 0;
#pragma unroll
        for (int w = 0; w < 3; ++w) {
          const int gy = oy + dy_[w], gx = ox + dx_[w];
          bool bit = false;
          if (use_[w] && gy >= 0 && gy < A.H && gx >= 0 && gx < A.W) bit = (int)__ldg(xi + ((int64_t)gy * A.W + gx) * C + ch_[w]) > tw_[w];
          pc += popc(ballot_pack(bit) ^ wreg[w]);
        }
        const int acc = S - 2 * pc;
        any |= (acc > th) != fl;
      }
      const uint32_t word = ballot_pack(any);
      if (lane == 0) A.y1[u] = word;
    }
  }
  grid_barrier(A.barrier, gridDim.x);

  // ---- phase 2: conv2 (32 -> 32 channels) + pool; warp = one (pooled pixel, pool offset), the 4
  // offsets' packed bits meet in y2 through atomicOr (the OR-pool, R9)
  {
    constexpr int K = K2, R = (K - 1) / 2;
    const int S = KK2 * 32;
    const int64_t units = (int64_t)A.n * H2 * W2 * 4;
    for (int64_t u = gw; u < units; u += nw) {
      const int64_t pix = u >> 2;
      const int q = (int)(u & 3);
      const int img = (int)(pix / (H2 * W2));
      const int rem = (int)(pix - (int64_t)img * H2 * W2);
      const int py = rem / W2, px = rem - py * W2;
      const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
      const uint32_t* yi = A.y1 + (int64_t)img * H1 * W1;
      int acc = 0;
#pragma unroll
      for (int ky = 0; ky < K; ++ky)
#pragma unroll
        for (int kx = 0; kx < K; ++kx) {
          const int gy = oy + ky - R, gx = ox + kx - R;
          const uint32_t v = (gy >= 0 && gy < H1 && gx >= 0 && gx < W1) ? __ldcg(yi + gy * W1 + gx) : 0u;
          acc += popc(v ^ w2[ky * K + kx]);
        }
      const uint32_t word = ballot_pack(((S - 2 * acc) > th2) != fl2);
      if (lane == 0 && word != 0u) atomicOr(A.y2 + pix, word);
    }
  }
  grid_barrier(A.barrier, 2 * gridDim.x);

  // ---- phase 3a: FC1, warp = one (image, output); lanes stride the words
  const int64_t d1 = (int64_t)H2 * W2 * 32;
  const int dw1 = (int)(d1 / 32);
  {
    const int64_t units = (int64_t)A.n * A.l1;
    for (int64_t u = gw; u < units; u += nw) {
      const int img = (int)(u / A.l1), o = (int)(u - (int64_t)img * A.l1);
      const uint32_t* xr = A.y2 + (int64_t)img * dw1;
      const uint32_t* wr = A.f1 + (int64_t)o * dw1;
      int sacc = 0;
#pragma unroll 8
      for (int j = lane; j < dw1; j += 32) sacc += popc(__ldcg(xr + j) ^ __ldg(wr + j));
      sacc = __reduce_add_sync(BNN_FULL_MASK, sacc);
      const int acc = (int)d1 - 2 * sacc;  // Eq. (4)
      const int t = A.thr_f1 != nullptr ? A.thr_f1[o] : 0;
      const bool f = A.flip_f1 != nullptr && A.flip_f1[o] != 0;
      if (lane == 0 && ((acc > t) != f)) atomicOr(A.h1 + (int64_t)img * lw1 + (o >> 5), 1u << (31 - (o & 31)));
    }
  }
  // the last CTA to finish FC1 runs the tail (threadfence reduction pattern)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(A.barrier + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // every other CTA is past both grid barriers and the FC1 count: re-arm the counters for the next launch
  if (threadIdx.x == 0) {
    A.barrier[0] = 0u;
    A.barrier[1] = 0u;
  }
  // ---- phase 3b: FC2 -> FC3 integer logits -> argmax, per image in this CTA
  for (int img = 0; img < A.n; ++img) {
    for (int j = threadIdx.x; j < kFusedMaxL / 32; j += blockDim.x) {
      s_h1[j] = j < lw1 ? __ldcg(A.h1 + (int64_t)img * lw1 + j) : 0u;
      s_h2[j] = 0;
    }
    __syncthreads();
    fused_dense(s_h1, A.l1, A.f2, A.l2, A.thr_f2, A.flip_f2, s_h2, nullptr);
    __syncthreads();
    fused_dense(s_h2, A.l2, A.f3, A.l3, nullptr, nullptr, nullptr, s_logit);
    __syncthreads();
    if (warp == 0) {
      const bool ok = lane < A.l3;
      const int v = ok ? s_logit[lane] : 0;
      if (ok && A.logits != nullptr) A.logits[(int64_t)img * A.l3 + lane] = v;
      int bv = ok ? v : INT_MIN, bi = ok ? lane : INT_MAX;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, s);
        const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, s);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0 && A.cls != nullptr) A.cls[img] = bi;  // first maximum wins (R19)
    }
    __syncthreads();
  }
}

}  // namespace bnn
