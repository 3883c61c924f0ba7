// k_alg1.cuh -- the paper's own GPU design, kept as a prior-art comparison pipeline:
// Im2col3d with fused patch extraction + packing (Algorithm 1, B = K*K = 25 bits
// per channel), GEMM-conv with XOR-popcount (Eq. 4: smem-tiled, one output
// element per thread), real-valued 2x2 max-pool, and the fully connected layer with 64 segments per
// weight vector (the reduction here is barrier-synchronised -- the paper's
// warp-synchronous version is unsafe under independent thread scheduling).  Table 2 (PAPER.md:
// 320-331) lists exactly these kernels.  The feature maps between the kernels are int32 in HBM, as
// in the paper; binarization is "> 0" inside the next Im2col3d (Alg. 1 line 7).  Results are the
// same integers as the fused path (sign(max) == max(sign), R9), so the forward pass is bit-exact.
#pragma once
#include "common.cuh"

namespace bnn {

constexpr int kAlg1S = 2;  // thread-block rows (S = 2)

// Algorithm 1 for one layer.  Block = S x W threads (W = image width <= 512); the block's region
// (S + 2R) x (W + 2R) of one channel is staged in zero-initialised shared memory (horizontal padding
// implicit, vertical halo loaded when inside the image), then every thread extracts its K x K patch
// with the integer counter k (no division / modulo) and packs s = (v > 0) << (B - 1 - i).
// src: u8 [n, H, W, C] binarized with x > t_c (layer 0, written to smem as +/-1) or int32 maps
// [n, H, W, C].  out: [n, H, W, C] words, B = K*K valid bits (MSB-first).
template <bool U8>
__global__ void alg1_im2col_pack_kernel(const void* __restrict__ src, const float* __restrict__ T, int H, int W, int C,
                                        int K, uint32_t* __restrict__ out) {
  extern __shared__ int sh_block[];
  const int R = (K - 1) / 2, B = K * K, SW = W + 2 * R;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int img = blockIdx.y, y0 = blockIdx.x * kAlg1S;
  const int nthr = blockDim.x * blockDim.y, tid = ty * blockDim.x + tx;
  for (int c = 0; c < C; ++c) {
    int t = 0;
    if (U8) t = T != nullptr ? u8_threshold(-T[c]) : 0;
    for (int i = tid; i < (kAlg1S + 2 * R) * SW; i += nthr) sh_block[i] = 0;  // zero = -1 after "> 0"
    __syncthreads();
    for (int i = tid; i < (kAlg1S + 2 * R) * W; i += nthr) {  // top halo, middle rows, bottom halo
      const int r = i / W, x = i - r * W, gy = y0 - R + r;
      if (gy >= 0 && gy < H) {
        const int64_t off = (((int64_t)img * H + gy) * W + x) * C + c;
        int v;
        if (U8) v = ((int)static_cast<const uint8_t*>(src)[off] > t) ? 1 : -1;
        else v = static_cast<const int32_t*>(src)[off];
        sh_block[r * SW + x + R] = v;
      }
    }
    __syncthreads();
    const int y = y0 + ty;
    if (y < H && tx < W) {
      // ExtractPacked (Algorithm 1): the patch of output pixel (y, tx) starts at smem (ty, tx)
      uint32_t v = 0;
      int k = 0;
      for (int i = 0; i < B; ++i) {
        if (i - k * K == K) ++k;
        const int idx = SW * (ty + k) + tx + i - k * K;
        const uint32_t s = sh_block[idx] > 0 ? 1u : 0u;
        v |= s << (31 - i);  // the paper's B - 1 - i, placed at the top of the 32-bit word
      }
      out[(((int64_t)img * H + y) * W + tx) * C + c] = v;
    }
    __syncthreads();
  }
}

// GEMM-conv: F[p, o] = sum_c (B - 2 popc(P[p, c] ^ Wp[o, c])) for the M = n*H*W patch rows, with
// 16 x 16 tiles of P and Wp^T staged in shared memory.  Output int32 [M, C_out].
constexpr int kAlg1Tile = 16;
__global__ void alg1_gemm_conv_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ Wp, int64_t M, int C,
                                      int C_out, int B, int32_t* __restrict__ F) {
  __shared__ uint32_t sP[kAlg1Tile][kAlg1Tile + 1], sW[kAlg1Tile][kAlg1Tile + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t row = (int64_t)blockIdx.x * kAlg1Tile + ty;
  const int col = blockIdx.y * kAlg1Tile + tx;
  int acc = 0;
  for (int c0 = 0; c0 < C; c0 += kAlg1Tile) {
    sP[ty][tx] = (row < M && c0 + tx < C) ? P[row * C + c0 + tx] : 0u;
    const int wo = blockIdx.y * kAlg1Tile + ty;
    sW[ty][tx] = (wo < C_out && c0 + tx < C) ? Wp[(int64_t)wo * C + c0 + tx] : 0u;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kAlg1Tile; ++j) acc += popc(sP[ty][j] ^ sW[tx][j]);
    __syncthreads();
  }
  if (row < M && col < C_out) F[row * C_out + col] = C * B - 2 * acc;  // Eq. (4) summed over the C words
}

// Real-valued 2x2 stride-2 max-pool of int32 maps [n, H, W, C] -> [n, H/2, W/2, C] (Table 2).
__global__ void alg1_maxpool_kernel(const int32_t* __restrict__ F, int64_t n, int H, int W, int C, int32_t* __restrict__ G) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = n * Ho * Wo * C;
  for (int64_t i = gtid(); i < total; i += gstride()) {
    const int c = (int)(i % C);
    int64_t p = i / C;
    const int x = (int)(p % Wo);
    p /= Wo;
    const int y = (int)(p % Ho);
    const int64_t img = p / Ho;
    const int32_t* f = F + ((img * H + 2 * y) * W + 2 * x) * C + c;
    G[i] = max(max(f[0], f[C]), max(f[(int64_t)W * C], f[(int64_t)W * C + C]));
  }
}

// Packing before the fully connected layer ("including packing", Table 2): int32 [n, D] -> bits > 0.
__global__ void alg1_pack_kernel(const int32_t* __restrict__ G, int64_t n, int64_t D, uint32_t* __restrict__ x) {
  const int64_t dw = (D + 31) / 32;
  for (int64_t i = gtid(); i < n * dw; i += gstride()) {
    const int64_t img = i / dw, w = i - img * dw;
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t d = w * 32 + b;
      if (d < D && G[img * D + d] > 0) v |= 1u << (31 - b);
    }
    x[i] = v;
  }
}

// Fully connected layer: block = (output neuron, image), 64 threads each sum a
// segment of the XOR-popcount dot product into shared memory, then a tree reduction.  Hidden layers
// write sign bits (> 0) packed with atomicOr into a zeroed [n, ceil(l/32)] buffer; the last layer
// writes int32 logits.
__global__ void alg1_fc_kernel(const uint32_t* __restrict__ x, int64_t d, const uint32_t* __restrict__ Wt, int l,
                               uint32_t* __restrict__ y, int32_t* __restrict__ logits) {
  __shared__ int part[64];
  const int o = blockIdx.x, img = blockIdx.y, t = threadIdx.x;
  const int64_t dw = (d + 31) / 32;
  const uint32_t* xr = x + (int64_t)img * dw;
  const uint32_t* wr = Wt + (int64_t)o * dw;
  int s = 0;
  for (int64_t j = t; j < dw; j += 64) s += popc(xr[j] ^ wr[j]);
  part[t] = s;
  __syncthreads();
  for (int h = 32; h > 0; h >>= 1) {
    if (t < h) part[t] += part[t + h];
    __syncthreads();
  }
  if (t == 0) {
    const int acc = (int)d - 2 * part[0];
    if (logits != nullptr) logits[(int64_t)img * l + o] = acc;
    else if (acc > 0) atomicOr(y + (int64_t)img * ((l + 31) / 32) + (o >> 5), 1u << (31 - (o & 31)));
  }
}

// Conv weights [c_out, K, K, cw] (packed along channels) -> Alg. 1 layout Wp[o, c] = the K x K
// window of channel c packed like the patches (bit 31 - i, i = ky * K + kx).
__global__ void alg1_prep_weights_kernel(const uint32_t* __restrict__ wt, int c_out, int K, int C, uint32_t* __restrict__ Wp) {
  const int cw = (C + 31) / 32;
  for (int64_t i = gtid(); i < (int64_t)c_out * C; i += gstride()) {
    const int o = (int)(i / C), c = (int)(i - (int64_t)o * C);
    uint32_t v = 0;
    for (int t = 0; t < K * K; ++t) {
      const uint32_t word = wt[((int64_t)o * K * K + t) * cw + c / 32];
      v |= ((word >> (31 - c % 32)) & 1u) << (31 - t);
    }
    Wp[i] = v;
  }
}

}  // namespace bnn
