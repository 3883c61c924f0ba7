// k_fused_cluster.cuh -- the whole vehicle-shaped network for a small batch in ONE thread-block cluster
// (pack -> conv1 + pool -> conv2 + pool -> FC1-3 + argmax with the activations kept on
// chip; the paper's batch-1 protocol, Table 1; its fusion idea).
//
// One cluster of up to 16 CTAs (one per SM, 16 warps each) runs every layer of one image after the other.
// There is no global-memory activation and no software grid barrier: each CTA keeps a FULL copy of the
// conv1 map (48 x 48 words) and of the conv2 map (24 x 24 words) in its shared memory, the producer of a
// word stores it into every CTA's copy through distributed shared memory (lanes 0..15 of the producing
// warp each write one CTA), and the hardware cluster barrier (barrier.cluster arrive.release /
// wait.acquire) separates the phases:
//   phase 1  conv1 (+ SIGN / THRESH_RGB input binarization, 2x2 OR-pool): warp = pooled pixel, lane =
//            output channel; the K x K x c patch bits of the 4 window pixels come from ballots of the
//            thresholded input bytes (Eq. 1, R14), acc = K^2 c - 2 popc(patch ^ w) (Eq. 4);
//   phase 2  conv2 (+ pool): warp = pooled pixel (all 4 window pixels), lane = output channel, the
//            (K2 x K2) 32-channel input words are warp-broadcast reads of the local conv1 copy;
//   phase 3  FC1: warp = output (cluster-wide), lanes stride the local conv2 copy; the bit goes to CTA 0
//            with one DSMEM atomicOr;
//   phase 4  CTA 0: FC2 -> FC3 integer logits -> argmax (first maximum, R19).
// All integer; results equal the layer-by-layer path.  Same topology checks as fused_small_kernel.
#pragma once
#include <cooperative_groups.h>

#include "k_fused_small.cuh"

namespace bnn {

constexpr int kClusterMax = 16;

// dynamic shared memory of fused_cluster_kernel for an H x W image
__host__ __device__ constexpr size_t fused_cluster_smem(int H, int W) {
  return (size_t)((H / 2) * (W / 2) + (H / 4) * (W / 4) + 2 * (kFusedMaxL / 32) + 32) * 4;
}

template <int K2>
__global__ void __launch_bounds__(kFusedWarps * 32, 1) fused_cluster_kernel(const FusedSmallArgs A) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) uint32_t cl_smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), ncta = (int)cl.num_blocks();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = rank * kFusedWarps + warp, nw = ncta * kFusedWarps;
  const int H1 = A.H >> 1, W1 = A.W >> 1, H2 = H1 >> 1, W2 = W1 >> 1;
  const int lw1 = (A.l1 + 31) / 32;
  uint32_t* y1 = cl_smem;                          // [H1 * W1] conv1 map (full copy)
  uint32_t* y2 = y1 + H1 * W1;                     // [H2 * W2] conv2 map (full copy)
  uint32_t* h1 = y2 + H2 * W2;                     // FC1 bits (CTA 0's copy is the target)
  uint32_t* h2 = h1 + kFusedMaxL / 32;             // FC2 bits (CTA 0)
  int32_t* s_logit = reinterpret_cast<int32_t*>(h2 + kFusedMaxL / 32);
  // lane l < ncta addresses CTA l's copies (DSMEM); every lane addresses CTA 0's FC1 bits
  uint32_t* y1_l = cl.map_shared_rank(y1, lane < ncta ? lane : 0);
  uint32_t* y2_l = cl.map_shared_rank(y2, lane < ncta ? lane : 0);
  uint32_t* h1_0 = cl.map_shared_rank(h1, 0);

  // conv2 weights of this lane's output channel, in registers for the whole kernel
  constexpr int KK2 = K2 * K2;
  uint32_t w2[KK2];
#pragma unroll
  for (int i = 0; i < KK2; ++i) w2[i] = __ldg(A.w2 + (int64_t)lane * KK2 + i);
  const int th2 = A.thr2 != nullptr ? A.thr2[lane] : 0;
  const bool fl2 = A.flip2 != nullptr && A.flip2[lane] != 0;
  // conv1: patch bit b = 32 w + lane <-> (ky, kx, c), b = (ky K + kx) C + c (MSB-first)
  const int K = A.K1, R = (K - 1) / 2, C = A.C, nb = K * K * C, S1 = nb;
  int t[4] = {0, 0, 0, 0};
  for (int c = 0; c < C; ++c) t[c] = A.T != nullptr ? u8_threshold(-A.T[c]) : 0;
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
    wreg[w] = __ldg(A.w1p + lane * 3 + w);
  }
  const int th1 = A.thr1 != nullptr ? A.thr1[lane] : 0;
  const bool fl1 = A.flip1 != nullptr && A.flip1[lane] != 0;
  if (rank == 0)
    for (int j = threadIdx.x; j < kFusedMaxL / 32; j += blockDim.x) h1[j] = 0u;
  cl.sync();  // h1 zeroed before any DSMEM atomic reaches it; every CTA of the cluster is running

  for (int img = 0; img < A.n; ++img) {
    // ---- phase 1: conv1 + input binarization + pool -> every CTA's y1
    const uint8_t* xi = A.x + (int64_t)img * A.H * A.W * C;
    for (int u = gw; u < H1 * W1; u += nw) {
      const int py = u / W1, px = u - py * W1;
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
        any |= (S1 - 2 * pc > th1) != fl1;
      }
      const uint32_t word = ballot_pack(any);
      if (lane < ncta) y1_l[u] = word;
    }
    cl.sync();
    // ---- phase 2: conv2 + pool from the local y1 -> every CTA's y2
    {
      constexpr int RR = (K2 - 1) / 2;
      const int S2 = KK2 * 32;
      for (int u = gw; u < H2 * W2; u += nw) {
        const int py = u / W2, px = u - py * W2;
        bool any = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int oy = 2 * py + (q >> 1), ox = 2 * px + (q & 1);
          int acc = 0;
#pragma unroll
          for (int ky = 0; ky < K2; ++ky)
#pragma unroll
            for (int kx = 0; kx < K2; ++kx) {
              const int gy = oy + ky - RR, gx = ox + kx - RR;
              const uint32_t v = (gy >= 0 && gy < H1 && gx >= 0 && gx < W1) ? y1[gy * W1 + gx] : 0u;
              acc += popc(v ^ w2[ky * K2 + kx]);
            }
          any |= (S2 - 2 * acc > th2) != fl2;
        }
        const uint32_t word = ballot_pack(any);
        if (lane < ncta) y2_l[u] = word;
      }
    }
    cl.sync();
    // ---- phase 3: FC1 from the local y2, one warp per output, bits into CTA 0's h1
    {
      const int64_t d1 = (int64_t)H2 * W2 * 32;
      const int dw1 = H2 * W2;
      for (int o = gw; o < A.l1; o += nw) {
        const uint32_t* wr = A.f1 + (int64_t)o * dw1;
        int s = 0;
#pragma unroll 6
        for (int j = lane; j < dw1; j += 32) s += popc(y2[j] ^ __ldg(wr + j));
        s = __reduce_add_sync(BNN_FULL_MASK, s);
        const int acc = (int)d1 - 2 * s;  // Eq. (4)
        const int tt = A.thr_f1 != nullptr ? A.thr_f1[o] : 0;
        const bool f = A.flip_f1 != nullptr && A.flip_f1[o] != 0;
        if (lane == 0 && ((acc > tt) != f)) atomicOr(h1_0 + (o >> 5), 1u << (31 - (o & 31)));
      }
    }
    cl.sync();
    // ---- phase 4 (CTA 0): FC2 -> FC3 integer logits -> argmax
    if (rank == 0) {
      for (int j = threadIdx.x; j < kFusedMaxL / 32; j += blockDim.x) h2[j] = 0u;
      __syncthreads();
      fused_dense(h1, A.l1, A.f2, A.l2, A.thr_f2, A.flip_f2, h2, nullptr);
      __syncthreads();
      fused_dense(h2, A.l2, A.f3, A.l3, nullptr, nullptr, nullptr, s_logit);
      __syncthreads();
      if (warp == 0) {
        const bool ok = lane < A.l3;
        const int v = ok ? s_logit[lane] : 0;
        if (ok && A.logits != nullptr) A.logits[(int64_t)img * A.l3 + lane] = v;
        int bv = ok ? v : INT_MIN, bi = ok ? lane : INT_MAX;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
          const int ov = __shfl_xor_sync(BNN_FULL_MASK, bv, sh);
          const int oi = __shfl_xor_sync(BNN_FULL_MASK, bi, sh);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0 && A.cls != nullptr) A.cls[img] = bi;  // first maximum wins (R19)
      }
      for (int j = threadIdx.x; j < lw1; j += blockDim.x) h1[j] = 0u;  // next image's FC1 bits
      __syncthreads();
    }
  }
  cl.sync();  // no CTA exits while another may still address its shared memory
}

}  // namespace bnn
