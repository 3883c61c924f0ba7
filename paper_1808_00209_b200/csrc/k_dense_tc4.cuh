// k_dense_tc4.cuh -- binary fully connected layer over the batch on the tensor cores
// (Section 3.2), tcgen05.mma kind::mxf4 with +/-1 as e2m1 and unit block scales.
//
// GEMM: M = 128 images per tile, N = NT >= l outputs (multiple of 16), K = d.  The packed words of
// KC words per stage are expanded to e2m1 (16 bytes per 32-bit word = one K-chunk) in shared memory:
// plane kw holds the 128 images' (or NT outputs') chunk of word kw, so a core matrix is 8
// consecutive images x 16 B, SBO = 128 B, and the second K-chunk of an MMA (K = 64 = two words) is
// the next plane (LBO = one plane).  Two stages ping-pong: the MMAs of stage s run while stage s+1 is
// expanded.  Pad bits / rows are e2m1 zero and contribute 0.  The epilogue is lane = image: all l
// sums of an image are in one thread, so threshold-pack and the argmax need no cross-lane work.
#pragma once
#include "k_conv_tc4.cuh"
#include "k_dense.cuh"

namespace bnn {

// TWO (NT <= 128, large batches): 8-word stages keep a CTA at ~89 KB of shared memory so TWO CTAs run per SM and one's
// per-stage block barrier overlaps the other's expansion / MMAs (ncu: 27% of FC1's warp samples waited at that
// barrier with one CTA per SM): FC1 0.248 -> 0.207 ms per 65536 images; with fewer tiles than 2 x SMs (config 2's
// 4096 images) the 16-word, one-CTA-per-SM form is faster (0.033 vs 0.039 ms).  The per-net weight image is laid out
// word by word ([word][NT][16 B]), so both forms read the same image.
template <int NT, bool TWO = false>
struct DenseTc4Cfg {
  static constexpr int KC = TWO ? 8 : 16;  // words per stage (KC / 2 MMAs)
  // weight-image ring: stage use u + NBR - 2 is bulk-copied while use u is expanded (its slot was read by MMA(u - 2))
  static constexpr int NBR = (TWO || NT > 128) ? 2 : 3;
  static constexpr int CPS = TWO ? 2 : 1;  // CTAs per SM the kernel is built for
  static constexpr uint32_t A_BYTES = KC * 128 * 16;    // 32 KB
  static constexpr uint32_t B_BYTES = KC * NT * 16;
  static constexpr uint32_t TMEM_COLS = (NT + 16 <= 64) ? 64 : ((NT + 16 <= 128) ? 128 : ((NT + 16 <= 256) ? 256 : 512));
  static constexpr int LUTC = 8;                        // LUT copies (lane & 7): fewer bank conflicts
  static constexpr int RING = NT > 128 ? 2 : 4;         // TMA ring of raw activation stages (TMAX variant)
  static constexpr uint32_t RAWB = 128 * KC * 4;        // one raw stage: 128 images x KC words
  static constexpr uint32_t RAW_OFF = (2 * A_BYTES + NBR * B_BYTES + NT * 4 + 256 * 4 * LUTC + 127) / 128 * 128;
  static constexpr uint32_t SMEM = 2 * A_BYTES + NBR * B_BYTES + NT * 4 + 256 * 4 * LUTC + 16;
  static constexpr uint32_t SMEM_TMAX = RAW_OFF + RING * RAWB + 16;
};

// The shared-memory image of B for output group g, stage st: [word kw][NT][16 B] (e2m1 +/-1 of the
// outputs' packed weights, pad bits / rows zero) -- what dense_tc4_kernel expands per stage when no
// image is given.  Written once per net (prep_dense_tc4_kernel), then bulk-copied per stage.
template <int NT>
__global__ void __launch_bounds__(256) prep_dense_tc4_kernel(const DenseArgs A, uint8_t* out) {
  using C = DenseTc4Cfg<NT>;
  __shared__ uint32_t lut[256];
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((threadIdx.x >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
    lut[threadIdx.x] = v;
  }
  __syncthreads();
  const int g = blockIdx.y, st = blockIdx.x;
  const int dw = (int)A.dw, dvalid_last = (int)(A.d - (int64_t)(dw - 1) * 32);
  uint8_t* dst = out + ((size_t)g * gridDim.x + st) * C::B_BYTES;
  for (int i = threadIdx.x; i < C::KC * NT; i += blockDim.x) {
    const int n = i % NT, kw = i / NT, w = st * C::KC + kw, o = g * NT + n;
    uint32_t o4[4] = {0u, 0u, 0u, 0u};
    if (o < A.l && w < dw) {
      expand_word_fp4(__ldg(A.wt + (int64_t)o * A.dw + w), lut, o4);
      if (w == dw - 1 && dvalid_last < 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t m = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) m |= (8 * q + k < dvalid_last ? 0xFu : 0u) << (4 * k);
          o4[q] &= m;
        }
      }
    }
    *reinterpret_cast<uint4*>(dst + ((size_t)kw * NT + n) * 16) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
  }
}

// TMAX: the activation stages arrive by TMA (2-D box of KC words x 128 images) in a RING-deep shared
// ring, issued RING stages ahead, instead of one-stage-ahead register prefetches (whose L2 latency
// every stage waited for).
template <int NT, bool TMAX = false, bool TWO = false>
__global__ void __launch_bounds__(256, DenseTc4Cfg<NT, TWO>::CPS)
dense_tc4_kernel(const DenseArgs A, const __grid_constant__ CUtensorMap xmap) {
  griddep_launch();
  using C = DenseTc4Cfg<NT, TWO>;
  constexpr int KC = C::KC;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sA = dsm;                                  // 2 x [kw][128][16]
  uint8_t* sB = dsm + 2 * C::A_BYTES;                 // NBR x [kw][NT][16]
  float* s_thr = reinterpret_cast<float*>(sB + C::NBR * C::B_BYTES);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_thr + NT);  // LUTC interleaved copies: entry i, copy c at LUTC i + c
  __shared__ uint64_t bar_stage[2], bar_acc, bar_b[C::NBR], bar_raw[C::RING];
  uint8_t* sRaw = dsm + C::RAW_OFF;  // TMAX: RING x [128 images][KC words]
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.y;
  {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= (((tid >> (7 - k)) & 1) ? 0x2u : 0xAu) << (4 * k);
#pragma unroll
    for (int c = 0; c < C::LUTC; ++c) s_lut[C::LUTC * tid + c] = v;
  }
  const uint32_t* my_lut = s_lut + (lane & (C::LUTC - 1));  // this lane's copy (stride LUTC)
  const bool b_img = A.bimg != nullptr;
  if (tid < NT) {
    const int o = g * NT + tid;
    const int t = (o < A.l && A.thr != nullptr) ? max(-(1 << 24), min(1 << 24, A.thr[o])) : 0;
    s_thr[tid] = (float)t;
  }
  if (warp == 0) tc::tmem_alloc<C::TMEM_COLS>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar_stage[0], 1);
    tc::mbar_init(&bar_stage[1], 1);
    tc::mbar_init(&bar_acc, 1);
#pragma unroll
    for (int i = 0; i < C::NBR; ++i) tc::mbar_init(&bar_b[i], 1);
#pragma unroll
    for (int i = 0; i < C::RING; ++i) tc::mbar_init(&bar_raw[i], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t tmem = tmem_base_s;
  const uint32_t sfa = tmem + NT, sfb = tmem + NT + 8;
  if (warp < 4) {
    tc::tmem_st8_same(sfa + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st8_same(sfb + ((uint32_t)(warp * 32) << 16), 0x7F7F7F7Fu);
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  constexpr uint32_t idesc = tc::idesc_mxf4(128, NT);
  const int dw = (int)A.dw;
  const int nstage = (dw + KC - 1) / KC;
  const int ntiles = (A.n + 127) / 128;
  const int dvalid_last = (int)(A.d - (int64_t)(dw - 1) * 32);  // valid bits of the last word
  // K split (A.ks > 1, grid.z): this CTA accumulates stages [st0, st1) and publishes fp32 partial sums
  // (exact integers) for dense_tc4_reduce_kernel; with 64 tiles per 8192-image chunk the unsplit grid
  // leaves most SMs idle
  const int z = (int)blockIdx.z;
  const int st0 = z * nstage / A.ks, st1 = (z + 1) * nstage / A.ks;

  // Stage loads are 16-byte vectors (4 words of one image / one output row; requires dw % 4 == 0)
  // prefetched into registers right after the previous stage's MMAs are issued.
  constexpr int PA = KC * 128 / 4 / 256, PB = KC * NT / 4 / 256;
  uint4 ra[PA], rb[PB];
  auto load_stage = [&](int img0, int st) {
    const int w0 = st * KC;
#pragma unroll
    for (int q = 0; q < (TMAX ? 0 : PA); ++q) {  // TMAX: the activations arrive by TMA
      const int i = tid + q * 256;
      const int r = i & 127, k4 = i >> 7, w = w0 + 4 * k4, img = img0 + r;
      ra[q] = (w < dw && img < A.n) ? __ldg(reinterpret_cast<const uint4*>(A.x + (int64_t)img * A.dw + w))
                                    : make_uint4(0, 0, 0, 0);
    }
    if (b_img) return;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int i = tid + q * 256;
      const int n = i % NT, k4 = i / NT, w = w0 + 4 * k4, o = g * NT + n;
      rb[q] = (w < dw && o < A.l) ? __ldg(reinterpret_cast<const uint4*>(A.wt + (int64_t)o * A.dw + w))
                                  : make_uint4(0, 0, 0, 0);
    }
  };
  // 4 words -> 4 planes; pad bits of the last word -> e2m1 zero; words >= dw (zero vectors) -> zero
  auto put4 = [&](uint8_t* base, int rows, int row, int w0k, uint4 v, bool valid_row) {
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int w = w0k + e;
      uint32_t o4[4] = {0u, 0u, 0u, 0u};
      if (valid_row && w < dw) {
#pragma unroll
        for (int q = 0; q < 4; ++q) o4[q] = my_lut[C::LUTC * ((wv[e] >> (24 - 8 * q)) & 0xFFu)];
        if (w == dw - 1 && dvalid_last < 32) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) m |= (8 * q + k < dvalid_last ? 0xFu : 0u) << (4 * k);
            o4[q] &= m;
          }
        }
      }
      *reinterpret_cast<uint4*>(base + ((size_t)(w - (w0k - (w0k % KC))) * rows + row) * 16) =
          make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
  };

  uint32_t stage_uses = 0;  // global stage counter (for mbarrier parity)
  uint32_t acc_uses = 0;
  const int nst = st1 - st0;
  // TMAX: stage use u of this CTA -> (tile, stage): raw box into ring slot u % RING
  auto issue_raw = [&](uint32_t u) {
    const int t = (int)blockIdx.x + (int)(u / nst) * (int)gridDim.x, st = st0 + (int)(u % nst);
    if (t >= ntiles) return;
    uint64_t* bar = &bar_raw[u % C::RING];
    tc::mbar_arrive_expect_tx(bar, C::RAWB);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            tc::smem_addr(sRaw + (u % C::RING) * C::RAWB)),
        "l"(reinterpret_cast<uint64_t>(&xmap)), "r"(st * KC), "r"(t * 128), "r"(tc::smem_addr(bar))
        : "memory");
  };
  // weight image of stage use u into ring slot u % NBR (a per-net image: independent of the predecessor layer)
  auto issue_b = [&](uint32_t u) {
    const int t = (int)blockIdx.x + (int)(u / nst) * (int)gridDim.x, st = st0 + (int)(u % nst);
    if (t >= ntiles) return;
    tc::stage_image(sB + (u % C::NBR) * C::B_BYTES, A.bimg + ((size_t)g * nstage + st) * C::B_BYTES, C::B_BYTES,
                    &bar_b[u % C::NBR]);
  };
  if (b_img && tid == 0)
    for (uint32_t u = 0; u < (uint32_t)(C::NBR - 2); ++u) issue_b(u);
  griddep_wait();  // activations of the predecessor layer
  if constexpr (TMAX) {
    if (tid == 0)
      for (uint32_t u = 0; u < (uint32_t)C::RING; ++u) issue_raw(u);
  }
  if ((int)blockIdx.x < ntiles) load_stage((int)blockIdx.x * 128, st0);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int img0 = tile * 128;
    for (int st = st0; st < st1; ++st, ++stage_uses) {
      const int s = stage_uses & 1;
      if (stage_uses >= 2) tc::mbar_wait(&bar_stage[s], ((stage_uses - 2) >> 1) & 1);
      uint8_t* a = sA + s * C::A_BYTES;
      uint8_t* b = sB + (stage_uses % C::NBR) * C::B_BYTES;
      const int w0 = st * KC;
      // the weight operand of stage use u + NBR - 2 (pre-expanded image, L2-resident); its slot was read by MMA(u - 2)
      if (b_img && tid == 0) issue_b(stage_uses + C::NBR - 2);
      if constexpr (TMAX) {
        const uint32_t slot = stage_uses % C::RING;
        tc::mbar_wait(&bar_raw[slot], (stage_uses / C::RING) & 1);
        const uint8_t* raw = sRaw + slot * C::RAWB;
#pragma unroll
        for (int q = 0; q < PA; ++q) {
          const int i = tid + q * 256;
          const int r = i & 127, k4 = i >> 7;
          ra[q] = *reinterpret_cast<const uint4*>(raw + (r * KC + 4 * k4) * 4);  // OOB rows / words: zero fill
        }
      }
#pragma unroll
      for (int q = 0; q < PA; ++q) {
        const int i = tid + q * 256;
        const int r = i & 127, k4 = i >> 7;
        put4(a, 128, r, w0 + 4 * k4, ra[q], img0 + r < A.n);
      }
      if (!b_img) {
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          const int i = tid + q * 256;
          const int n = i % NT, k4 = i / NT;
          put4(b, NT, n, w0 + 4 * k4, rb[q], g * NT + n < A.l);
        }
      }
      tc::fence_async_smem();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      if (tid == 0) {
        if constexpr (TMAX) issue_raw(stage_uses + C::RING);  // the slot was read by every thread (barrier above)
        if (b_img) tc::mbar_wait(&bar_b[stage_uses % C::NBR], (stage_uses / C::NBR) & 1);  // weight stage landed
        const uint64_t ad0 = tc::desc_kmajor(tc::smem_addr(a), 128 * 16, 128);
        const uint64_t bd0 = tc::desc_kmajor(tc::smem_addr(b), NT * 16, 128);
#pragma unroll
        for (int i = 0; i < KC / 2; ++i) {
          tc::mma_mxf4(tmem, ad0 + (uint64_t)(2 * i * 128), bd0 + (uint64_t)(2 * i * NT), idesc, sfa, sfb,
                       (st > st0 || i > 0) ? 1u : 0u);
        }
        tc::commit(&bar_stage[s]);
        if (st == st1 - 1) tc::commit(&bar_acc);
      }
      // prefetch the next stage (next tile's first stage after the last one)
      if (!TMAX || !b_img) {  // (TMAX: only the weight words, when there is no weight image)
        if (st + 1 < st1) load_stage(img0, st + 1);
        else if (tile + (int)gridDim.x < ntiles) load_stage((tile + (int)gridDim.x) * 128, st0);
      }
    }
    // epilogue: warps 0-3, thread = image
    tc::mbar_wait(&bar_acc, acc_uses & 1);
    ++acc_uses;
    tc::fence_after();
    if (A.ks > 1 && warp < 4) {  // partial sums of this K range, thread = image, 32 columns per load
      const int img = img0 + warp * 32 + lane;
      const int LP = (int)gridDim.y * NT;
      float* dst = A.part + ((int64_t)z * ntiles * 128 + img) * LP + g * NT;
#pragma unroll 1
      for (int c0 = 0; c0 < NT && g * NT + c0 < A.l; c0 += 32) {
        int v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          __stcg(reinterpret_cast<float4*>(dst + c0 + c), make_float4(__int_as_float(v[c]), __int_as_float(v[c + 1]),
                                                                       __int_as_float(v[c + 2]), __int_as_float(v[c + 3])));
      }
    } else if (A.ks == 1 && warp < 4) {
      const int img = img0 + warp * 32 + lane;
      const bool img_ok = img < A.n;
      float best = -3.0e38f;
      int besti = 0;
#pragma unroll 1
      for (int c0 = 0; c0 < NT && g * NT + c0 < A.l; c0 += 32) {
        int v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        const int nvalid = min(32, A.l - (g * NT + c0));
        uint32_t word = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) word = __funnelshift_l(__float_as_uint(s_thr[c0 + c] - __int_as_float(v[c])), word, 1);
        word &= nvalid >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nvalid);
        if (A.flip != nullptr) {
          uint32_t fm = 0;
          for (int c = 0; c < nvalid; ++c) fm |= (A.flip[g * NT + c0 + c] != 0 ? 1u : 0u) << (31 - c);
          word ^= fm;
        }
        if (img_ok) {
          if (A.y != nullptr) A.y[(int64_t)img * A.lw + ((g * NT + c0) >> 5)] = word;
          if (A.acc != nullptr)
            for (int c = 0; c < nvalid; ++c) A.acc[(int64_t)img * A.l + g * NT + c0 + c] = (int32_t)__int_as_float(v[c]);
          if (A.cls != nullptr) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const float f = __int_as_float(v[c]);
              if (c < nvalid && f > best) { best = f; besti = g * NT + c0 + c; }  // first maximum wins (R19)
            }
          }
        }
      }
      if (A.cls != nullptr && img_ok) A.cls[img] = besti;
    }
    tc::fence_before();
    __syncthreads();  // TMEM accumulator drained before the next tile's first MMA
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// Reduction + epilogue of a K-split dense_tc4_kernel: one warp per image, lane = output column of a
// 32-column chunk (coalesced partial loads); sums the ks partials (exact: integers < 2^24 in fp32),
// then the fused epilogue's threshold (bit = acc > thr, as a ballot: lane c -> bit 31 - c, MSB-first),
// flips, acc output and first-maximum argmax (R19) over all l outputs.
__global__ void __launch_bounds__(256) dense_tc4_reduce_kernel(const DenseArgs A, int LP, int npad) {
  griddep_launch();
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int img = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (img >= A.n) return;
  float best = -3.0e38f;
  int besti = INT_MAX;
  for (int c0 = 0; c0 < A.l; c0 += 32) {
    const int o = c0 + lane;
    const bool ok = o < A.l;
    float f = 0.f;
    if (ok)
      for (int z = 0; z < A.ks; ++z) f += __ldcg(A.part + ((int64_t)z * npad + img) * LP + o);
    const int t = (ok && A.thr != nullptr) ? max(-(1 << 24), min(1 << 24, A.thr[o])) : 0;
    bool bit = ok && f > (float)t;
    if (ok && A.flip != nullptr && A.flip[o] != 0) bit = !bit;
    const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, bit));
    if (A.y != nullptr && lane == 0) A.y[(int64_t)img * A.lw + (c0 >> 5)] = word;
    if (ok) {
      if (A.acc != nullptr) A.acc[(int64_t)img * A.l + o] = (int32_t)f;
      if (f > best) { best = f; besti = o; }
    }
  }
  if (A.cls != nullptr) {
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {  // first maximum wins (R19): larger value, then lower index
      const float ov = __shfl_xor_sync(0xFFFFFFFFu, best, sh);
      const int oi = __shfl_xor_sync(0xFFFFFFFFu, besti, sh);
      if (ov > best || (ov == best && oi < besti)) { best = ov; besti = oi; }
    }
    if (lane == 0) A.cls[img] = besti;
  }
}

}  // namespace bnn
