// bnn_api.cu -- the C ABI of libbnn.so (include/bnn.h): validation, kernel dispatch and the
// whole-network orchestration (bnn_net / bnn_forward / bnn_forward_host).
// Every entry validates before launching, never throws, and reports through bnn_status +
// the thread-local bnn_last_error().
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <utility>
#include <string>
#include <vector>

#include "bnn.h"
#include "k_conv.cuh"
#include "k_conv_tc.cuh"
#include "k_conv_first_tc.cuh"
#include "k_conv_first_tma.cuh"
#include "k_conv1_fp4.cuh"
#include "k_conv_tc4.cuh"
#include "k_conv_tc4_pool.cuh"
#include "k_conv_tc4_pool3.cuh"
#include "k_dense_tc4.cuh"
#include "k_conv_tc4_big.cuh"
#include "k_dense.cuh"
#include "k_fused_small.cuh"
#include "k_fused_cluster.cuh"
#include "k_alg1.cuh"
#include "k_pack.cuh"

using namespace bnn;

namespace {

thread_local std::string g_err;

bnn_status fail(bnn_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

bnn_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BNN_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return BNN_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

#define BNN_REQUIRE_ALIGNED(p, name) \
  do { if ((p) != nullptr && !aligned16(p)) return fail(BNN_E_ALIGN, "%s: pointer not 16-byte aligned", name); } while (0)

// Per-device launch setup.  The dynamic shared-memory opt-in (cudaFuncSetAttribute) and the SM count
// belong to the CURRENT device, so they are cached per (kernel, device), behind a mutex (the entry
// points are reentrant and may be called from several threads / for several devices).
std::mutex g_dev_mu;
std::map<std::pair<const void*, int>, int> g_dev_cache;  // (kernel or tag, device) -> value

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// value of `key` on the current device, computing it once with f() (outside the lock: f may call CUDA)
template <typename F>
int dev_cached(const void* key, F&& f) {
  const std::pair<const void*, int> k(key, current_device());
  {
    std::lock_guard<std::mutex> g(g_dev_mu);
    auto it = g_dev_cache.find(k);
    if (it != g_dev_cache.end()) return it->second;
  }
  const int v = f();
  std::lock_guard<std::mutex> g(g_dev_mu);
  g_dev_cache[k] = v;
  return v;
}

int g_num_sms_tag = 0;
int num_sms() {
  return dev_cached(&g_num_sms_tag, [] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
    (void)cudaGetLastError();
    return n > 0 ? n : 148;
  });
}

// dynamic shared-memory opt-in of kfn on the current device (once per device)
template <typename F>
void ensure_smem(F kfn, uint32_t dyn_smem) {
  if (dyn_smem <= 48 * 1024) return;
  dev_cached(reinterpret_cast<const void*>(kfn), [&] {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    (void)cudaGetLastError();
    return 1;
  });
}

// tuning / test knobs (bnn_set_option)
// Stream-ordered scratch (cudaMallocAsync on the launch stream, freed with cudaFreeAsync after the
// consumer) from the device's default pool, which keeps freed blocks (release threshold = max) so a
// steady-state allocation is a pool hit, not a new mapping.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static int tag = 0;
  dev_cached(&tag, [] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    (void)cudaGetLastError();
    return 1;
  });
  return cudaMallocAsync(p, bytes, s);
}

int g_opt_conv_algo = 0;      // 0 auto, 1 force the generic one-word-per-tap conv
int g_opt_tiles_per_cta = 0;  // 0 auto, else a fixed number of tiles per CTA
int g_opt_gemv_max_n = 255;   // dense layers with n <= this use the GEMV kernel (every n below the tensor path's 256: dense_kernel's 64-image CTAs leave the SMs idle there, FC1 ~0.2 ms at 17-255 images vs 0.005-0.03 ms)
int g_opt_conv_tc = 1;        // 1: binary convs with c_in >= 32 run on tcgen05 (kind::i8) where supported
int g_opt_first_pool_tc = 1;  // 1: pooled first layers use the pool-window-ordered tensor-core kernel
int g_opt_conv_tc_fp4 = 1;    // 1: tensor-core binary convs use packed e2m1 (kind::mxf4), 0: int8 (kind::i8)
int g_opt_conv_pair = 1;      // 1: conv1_fp4 / conv_tc4_pool run as CTA pairs (cta_group::2, M = 256, half of B per SM)
int g_opt_conv_pool3 = 1;     // 1: conv_tc4_pool runs as conv_tc4_pool3_kernel (1 CTA/SM, 3 accumulator sets); 0: 2 CTAs/SM x 1 set
int g_opt_conv_pool_tc = 1;   // 1: pooled 32-channel binary convs fold the pool window into the MMA N (conv_tc4_pool)
int g_opt_first_fp4 = 1;     // 1: the binarized TMA first layer is conv1_fp4_pool_kernel (kind::mxf4, {0,1} operands, 1 CTA/SM); 0: the int8 kernel
int g_opt_first_db = 1;      // 1: the int8 TMA first layer double-buffers its TMEM accumulators (2 CTAs/SM; measured +6% whole step with the 8-deep raw ring)
int g_opt_first_exp = 0;     // timing experiments on the TMA first layer (diagnostics build only; see exp_bits)
int g_opt_first_tma = 1;     // 1: pooled u8 RGB / SIGN first layers use the TMA-fed kernel (thresholds folded into the MMA)
int g_opt_luma_band = 1;     // 1: the GRAY / LBP pre-pass of the TMA first layer is luma_band_kernel; 0: luma_u8img4_kernel
int g_opt_luma_fused = 1;    // 1: THRESH_GRAY nets compute the luma inside conv1_fp4 (no 0/1 image in HBM); 2: LBP too
int g_opt_first_real_tma = 1;  // 1: real u8 first layers (mode NONE) use the TMA kernel (u8 x +/-1 kind::i8)
unsigned long long* g_trace = nullptr;  // bnn_set_trace (diagnostics build)
int g_trace_cap = 0;
int g_trace_layer = 0;  // diagnostics build: 0 traces conv1_fp4 / the int8 TMA first layer, 1 conv_tc4_pool, 2 the fused cluster kernel
int g_opt_dense_ksplit = 1;   // 1: dense_tc4 splits K over grid.z when its tile grid leaves SMs idle
int g_opt_dense_tc = 1;       // 1: dense layers with n >= 256 and d >= 1024 run on tcgen05 (kind::mxf4)
int g_opt_dense_tma = 1;      // 1: dense_tc4 activation stages arrive by TMA into a 4-deep ring

int g_opt_fused_tc = 1;       // 1: the cluster kernel runs conv2 on the tensor cores (pool-in-N mxf4, one tile per CTA)
int g_opt_fused_cs = 0;       // cluster size of fused_cluster_kernel: 0 = 16 where the device runs it and the chunk's images fit in one wave of 16-CTA clusters, else 8; 8 = always 8
int g_opt_fused_multi = 1;    // 1: fused_cluster_kernel runs one cluster per image of a small batch; 0: one cluster
int g_opt_fused_cluster = 1;  // 1: the fused small-batch path is the thread-block-cluster kernel (DSMEM, cluster barriers); 0: cooperative
int g_opt_fused_max_n = 12;  // forward over n <= this images runs as one whole-network kernel where the topology allows (default 12: one cluster per image -- 16-CTA clusters for up to 7 images (what a B200 holds at once; 11.3-11.7 us on the device vs 13.0-15.7 us for the PDL layers), 8-CTA clusters beyond (12.5-12.7 us for 8-12 images vs 16.0-16.3 us; 16 images: 20.4 vs 16.8 us), larger n run the batched layers)
int g_opt_pdl = 1;   // 1: forward-path kernels are launched with programmatic dependent launch
int g_opt_alg1 = 0;  // 1: bnn_forward runs the paper's own design (Alg. 1 im2col + GEMM + pool + FC), for comparison
int g_opt_csa = 1;      // 1: the XOR-popcount conv compresses each kernel row's K words with carry-save adders
int g_opt_big_img = 1;  // 1: the streamed wide-channel conv stages a per-call pre-expanded weight image
int g_opt_streams = 2;  // bnn_forward over several chunks alternates chunks over 1 or 2 streams

// Launch with the programmatic-stream-serialization attribute: the kernel may be scheduled while its
// stream predecessor is still running; it runs its prologue (barriers, TMEM, weight images) and then
// blocks in griddep_wait() before touching activations (see common.cuh).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kfn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_opt_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kfn, std::forward<Args>(args)...);
}

// The same with a (cx, 1, 1) thread-block cluster (CTA pairs of the cta_group::2 kernels)
template <typename... KArgs, typename... Args>
void launch_pdl_cluster(void (*kfn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cx, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_opt_pdl ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = (unsigned)cx;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kfn, std::forward<Args>(args)...);
}

int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

int choose_tpc(int64_t total_tiles, bool restage_per_tile) {
  if (g_opt_tiles_per_cta > 0) return g_opt_tiles_per_cta;
  if (restage_per_tile) return 1;
  int64_t target = (int64_t)num_sms() * 8;
  int64_t tpc = (total_tiles + target - 1) / target;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tpc, 32));
}

// ---------------------------------------------------------------------------- pack
bnn_status launch_pack(const void* x, bnn_dtype dt, int n, int h, int w, int c, int mode, const float* T,
                       uint32_t* y, cudaStream_t s) {
  const int64_t npix = (int64_t)n * h * w;
  if (npix == 0) return BNN_OK;
  if (mode == BNN_THRESH_GRAY || mode == BNN_LBP) {
    pack_luma_kernel<<<grid_for(npix, 256), 256, 0, s>>>((const uint8_t*)x, n, h, w, mode, T, y);
    return check_launch("pack_luma_kernel");
  }
  if (dt == BNN_U8 && c == 3) {
    pack_u8c3_kernel<<<grid_for(npix / 4 + 1, 256), 256, 0, s>>>((const uint8_t*)x, npix, mode, T, y);
    return check_launch("pack_u8c3_kernel");
  }
  const int cw = (c + 31) / 32;
  const int grid = grid_for(npix * cw, 256);
  switch (dt) {
    case BNN_U8: pack_generic_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)x, npix, c, cw, mode, T, y); break;
    case BNN_I8: pack_generic_kernel<int8_t><<<grid, 256, 0, s>>>((const int8_t*)x, npix, c, cw, mode, T, y); break;
    case BNN_F32: pack_generic_kernel<float><<<grid, 256, 0, s>>>((const float*)x, npix, c, cw, mode, T, y); break;
    case BNN_I32: pack_generic_kernel<int32_t><<<grid, 256, 0, s>>>((const int32_t*)x, npix, c, cw, mode, T, y); break;
    default: return fail(BNN_E_ARG, "bnn_pack: bad dtype");
  }
  return check_launch("pack_generic_kernel");
}

// ---------------------------------------------------------------------------- conv
template <int K, int WY, int WX>
bnn_status launch_conv_bin_t(ConvArgs A, cudaStream_t s) {
  constexpr int PR = 2, PC = 8;
  constexpr int CWC = (K >= 7) ? 4 : 8;
  constexpr int TH = WY * PR, TW = WX * PC;
  A.tiles_y = (A.H + TH - 1) / TH;
  A.tiles_x = (A.W + TW - 1) / TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = choose_tpc(A.total_tiles, A.cw > CWC);
  const int64_t gx = (A.total_tiles + A.tiles_per_cta - 1) / A.tiles_per_cta;
  if (gx > 0x7fffffff) return fail(BNN_E_UNSUPPORTED, "bnn_conv2d: too many tiles");
  dim3 grid((unsigned)gx, (unsigned)((A.c_out + 31) / 32));
  if (g_opt_csa) conv_bin_kernel<K, PR, PC, WY, WX, CWC, true><<<grid, WY * WX * 32, 0, s>>>(A);
  else conv_bin_kernel<K, PR, PC, WY, WX, CWC, false><<<grid, WY * WX * 32, 0, s>>>(A);
  return check_launch("conv_bin_kernel");
}

template <int K, int WY, int WX>
bnn_status launch_conv_patch_t(ConvArgs A, cudaStream_t s) {
  constexpr int PR = 2, PC = 8;
  constexpr int TH = WY * PR, TW = WX * PC;
  A.tiles_y = (A.H + TH - 1) / TH;
  A.tiles_x = (A.W + TW - 1) / TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = choose_tpc(A.total_tiles, false);
  const int64_t gx = (A.total_tiles + A.tiles_per_cta - 1) / A.tiles_per_cta;
  dim3 grid((unsigned)gx, (unsigned)((A.c_out + 31) / 32));
  conv_patch_kernel<K, PR, PC, WY, WX><<<grid, WY * WX * 32, 0, s>>>(A);
  return check_launch("conv_patch_kernel");
}

template <int K, int WY, int WX, bool SRC_U8>
bnn_status launch_conv_strip_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  constexpr int PR = 2, PC = 8;
  constexpr int TH = WY * PR, TW = WX * PC;
  A.tiles_y = (A.H + TH - 1) / TH;
  A.tiles_x = (A.W + TW - 1) / TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = choose_tpc(A.total_tiles, false);
  const int64_t gx = (A.total_tiles + A.tiles_per_cta - 1) / A.tiles_per_cta;
  dim3 grid((unsigned)gx, (unsigned)((A.c_out + 31) / 32));
  conv_strip_kernel<K, PR, PC, WY, WX, SRC_U8><<<grid, WY * WX * 32, 0, s>>>(A, xu8, T);
  return check_launch("conv_strip_kernel");
}

template <int WY, int WX, bool SRC_U8>
bnn_status dispatch_conv_strip(int k, const ConvArgs& A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  switch (k) {
    case 3: return launch_conv_strip_t<3, WY, WX, SRC_U8>(A, xu8, T, s);
    case 5: return launch_conv_strip_t<5, WY, WX, SRC_U8>(A, xu8, T, s);
    case 7: return launch_conv_strip_t<7, WY, WX, SRC_U8>(A, xu8, T, s);
  }
  return fail(BNN_E_UNSUPPORTED, "conv_strip: k=%d", k);
}

template <int K, int NW, bool SRC_U8>
bnn_status launch_conv_first_lp_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  constexpr int TH = 16, TW = 32;
  A.tiles_y = (A.H + TH - 1) / TH;
  A.tiles_x = (A.W + TW - 1) / TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = choose_tpc(A.total_tiles, false);
  const int64_t gx = (A.total_tiles + A.tiles_per_cta - 1) / A.tiles_per_cta;
  dim3 grid((unsigned)gx, (unsigned)((A.c_out + 31) / 32));
  conv_first_lp_kernel<K, NW, SRC_U8><<<grid, 256, 0, s>>>(A, xu8, T);
  return check_launch("conv_first_lp_kernel");
}

// (k, words-per-patch) combinations of the strip layout that the lane = pixel kernel covers
template <bool SRC_U8>
bnn_status dispatch_conv_first_lp(int k, int nw, const ConvArgs& A, const uint8_t* xu8, const float* T,
                                  cudaStream_t s) {
#define BNN_LP(KK, NN) if (k == KK && nw == NN) return launch_conv_first_lp_t<KK, NN, SRC_U8>(A, xu8, T, s)
  BNN_LP(3, 1); BNN_LP(3, 2); BNN_LP(3, 3);
  BNN_LP(5, 1); BNN_LP(5, 2); BNN_LP(5, 3); BNN_LP(5, 5);
  BNN_LP(7, 2); BNN_LP(7, 4); BNN_LP(7, 7);
#undef BNN_LP
  return fail(BNN_E_UNSUPPORTED, "conv_first_lp: k=%d nw=%d", k, nw);
}

// ---- tensor-core (tcgen05 kind::i8) binary conv
// Resident CTAs per SM of a 256-thread tcgen05 kernel: registers, shared memory (227 KB usable,
// ~1 KB reserved per CTA) and TMEM columns (512 per SM).
template <typename F>
int tc_occupancy_calc(F kfn, uint32_t dyn_smem, uint32_t tmem_cols, int threads) {
  cudaFuncAttributes fa;
  int regs = 128, static_smem = 2048;
  if (cudaFuncGetAttributes(&fa, kfn) == cudaSuccess) { regs = fa.numRegs; static_smem = (int)fa.sharedSizeBytes; }
  (void)cudaGetLastError();
  const int by_regs = 65536 / (((regs + 7) & ~7) * threads);
  const int by_smem = (227 * 1024) / ((int)dyn_smem + static_smem + 1024);
  const int by_tmem = 512 / (int)tmem_cols;
  return std::max(1, std::min(std::min(by_regs, by_smem), std::min(by_tmem, 8)));
}

// ... per (kernel, current device), with the kernel's shared-memory opt-in done on that device
template <typename F>
int tc_occupancy(F kfn, uint32_t dyn_smem, uint32_t tmem_cols, int threads = 256) {
  ensure_smem(kfn, dyn_smem);
  // key: kernel pointer + 1 byte (distinct from ensure_smem's key for the same kernel)
  return dev_cached(reinterpret_cast<const char*>(kfn) + 1,
                    [&] { return tc_occupancy_calc(kfn, dyn_smem, tmem_cols, threads); });
}

template <int K, int NT, int CIN, int SRC>
bnn_status launch_conv_first_tc_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  auto kfn = conv_first_tc_kernel<K, NT, CIN, SRC>;
  using C = FirstTcCfg<K, NT, CIN, SRC>;
  const int occ = tc_occupancy(kfn, 0, C::TMEM_COLS);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + NT - 1) / NT));
  kfn<<<grid, 256, 0, s>>>(A, xu8, T);
  return check_launch("conv_first_tc_kernel");
}

// First layer on the tensor cores: strips of K * c_in <= 16 int8.  Instantiated (k, c_in) pairs:
// packed input (kSrcBits) k=3: c_in 1..5, k=5: 1..3, k=7: 1..2; u8 thresholded in the kernel
// (kSrcThresh) and real u8 (kSrcReal): c_in in {1, 3}, k in {3, 5}.  conv_algo 0 (auto) or 5 (forced).
bool use_first_tc(int c_in, int k, int src) {
  if (g_opt_conv_tc == 0 || (g_opt_conv_algo != 0 && g_opt_conv_algo != 5)) return false;
  if (src != kSrcBits) return (c_in == 3 || c_in == 1) && (k == 3 || k == 5);
  return (k == 3 && c_in >= 1 && c_in <= 5) || (k == 5 && c_in >= 1 && c_in <= 3) || (k == 7 && c_in >= 1 && c_in <= 2);
}

template <int K, int NT, int CIN, int SRC>
bnn_status launch_conv_first_tc_pool_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  auto kfn = conv_first_tc_pool_kernel<K, NT, CIN, SRC>;
  using C = FirstTcPoolCfg<K, NT, CIN, SRC>;
  const int occ = tc_occupancy(kfn, 0, C::TMEM_COLS);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + NT - 1) / NT));
  kfn<<<grid, 256, 0, s>>>(A, xu8, T);
  return check_launch("conv_first_tc_pool_kernel");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    (void)cudaGetLastError();
  });
  return fn;
}

// TMA-fed pooled first layer: u8 [n, H, W, 3] viewed as a 3-D tensor (W*3 bytes, H rows, n images);
// the row pitch must be a multiple of 16 bytes and the base 16-byte aligned.
bool use_first_tma(const ConvArgs& A, int k, const uint8_t* xu8) {
  return g_opt_first_tma && g_opt_first_pool_tc && A.pool == 2 && A.c_in == 3 && (k == 3 || k == 5) && ((A.W * 3) % 16) == 0 &&
         aligned16(xu8) && tma_encoder() != nullptr;
}

template <int K, bool FP4, bool DB = false, bool REAL = false>
bnn_status launch_conv_first_tma_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  using C = FirstTmaCfg<K, FP4, DB>;
  auto kfn = conv_first_tma_pool_kernel<K, FP4, DB, REAL>;
  constexpr uint32_t smem = C::NRAW * C::RAW_STRIDE + 2 * C::A_BYTES + C::B_BYTES + 1024;
  const int occ = tc_occupancy(kfn, smem, C::TMEM_COLS, kFirstTmaThreads);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  A.exp = g_opt_first_exp;
  A.trace = g_trace_layer == 0 ? g_trace : nullptr;
  A.trace_cap = g_trace_cap;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)A.W * 3, (cuuint64_t)A.H, (cuuint64_t)A.n};
  const cuuint64_t strides[2] = {(cuuint64_t)A.W * 3, (cuuint64_t)A.H * A.W * 3};
  const cuuint32_t box[3] = {(cuuint32_t)C::RAW_W, (cuuint32_t)C::IR, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tma_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(xu8), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BNN_E_CUDA, "conv_first_tma: cuTensorMapEncodeTiled failed (%d)", (int)r);
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + C::NT - 1) / C::NT));
  launch_pdl(kfn, grid, dim3(kFirstTmaThreads), smem, s, A, map, T);
  return check_launch("conv_first_tma_pool_kernel");
}

// The mxf4 pooled first layer (k_conv1_fp4.cuh): one CTA per SM, {0, 1} activations, TMA-fed.
template <int K, bool SPIN = false, int BIN = kBinRgb>
bnn_status launch_conv1_fp4_t(ConvArgs A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  using C = Conv1Fp4Cfg<K>;
  auto kfn = conv1_fp4_pool_kernel<K, SPIN, BIN>;
  const int occ = tc_occupancy(kfn, C::SMEM, C::TMEM_COLS, C::THREADS);
  A.exp = g_opt_first_exp;
  A.trace = g_trace_layer == 0 ? g_trace : nullptr;
  A.trace_cap = g_trace_cap;
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)A.W * 3, (cuuint64_t)A.H, (cuuint64_t)A.n};
  const cuuint64_t strides[2] = {(cuuint64_t)A.W * 3, (cuuint64_t)A.H * A.W * 3};
  const cuuint32_t box[3] = {(cuuint32_t)C::RAW_W, (cuuint32_t)(C::IR + (BIN == kBinLbp ? 2 : 0)), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tma_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(xu8), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BNN_E_CUDA, "conv1_fp4: cuTensorMapEncodeTiled failed (%d)", (int)r);
  if (g_opt_conv_pair && A.bimg != nullptr && !SPIN) {  // CTA pairs (cta_group::2): each SM reads half of B per MMA
    auto kp = conv1_fp4_pool_kernel<K, SPIN, BIN, true>;
    const int occp = tc_occupancy(kp, C::SMEM, C::TMEM_COLS, C::THREADS);
    const int64_t pairs = std::min<int64_t>((A.total_tiles + 1) / 2, (int64_t)num_sms() * occp / 2);
    dim3 grid((unsigned)(2 * std::max<int64_t>(pairs, 1)), (unsigned)((A.c_out + C::NT - 1) / C::NT));
    launch_pdl_cluster(kp, grid, dim3(C::THREADS), C::SMEM, s, 2, A, map, T);
    return check_launch("conv1_fp4_pool_kernel<pair>");
  }
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + C::NT - 1) / C::NT));
  launch_pdl(kfn, grid, dim3(C::THREADS), C::SMEM, s, A, map, T);
  return check_launch("conv1_fp4_pool_kernel");
}

// The TMA-fed pooled first layer on a u8 [n, H, W, 3] image (k in {3, 5}): the mxf4 kernel (first_fp4 = 1,
// default) or the int8 one (first_fp4 = 0; TMEM double buffering per first_db).  A.c_in may be 1
// (THRESH_GRAY via luma_u8img4_kernel: channels 1-2 get zero weights).
bnn_status dispatch_first_tma(int k, const ConvArgs& A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  if (g_opt_first_fp4 == 2) return k == 5 ? launch_conv1_fp4_t<5, true>(A, xu8, T, s) : launch_conv1_fp4_t<3, true>(A, xu8, T, s);
  if (g_opt_first_fp4) return k == 5 ? launch_conv1_fp4_t<5>(A, xu8, T, s) : launch_conv1_fp4_t<3>(A, xu8, T, s);
  if (g_opt_first_db) return k == 5 ? launch_conv_first_tma_t<5, false, true>(A, xu8, T, s) : launch_conv_first_tma_t<3, false, true>(A, xu8, T, s);
  return k == 5 ? launch_conv_first_tma_t<5, false>(A, xu8, T, s) : launch_conv_first_tma_t<3, false>(A, xu8, T, s);
}

template <int SRC>
bnn_status dispatch_conv_first_tc(int k, const ConvArgs& A, const uint8_t* xu8, const float* T, cudaStream_t s) {
  const bool wide = A.c_out > 32;
  const int c = A.c_in;
  if constexpr (SRC == kSrcThresh) {
    if (A.n > 0 && use_first_tma(A, k, xu8)) return dispatch_first_tma(k, A, xu8, T, s);
  }
  if constexpr (SRC == kSrcReal) {  // real u8 pixels (mode NONE): the TMA kernel with an unsigned A operand
    if (A.n > 0 && g_opt_first_real_tma && use_first_tma(A, k, xu8)) {
      if (g_opt_first_db) return k == 5 ? launch_conv_first_tma_t<5, false, true, true>(A, xu8, nullptr, s)
                                        : launch_conv_first_tma_t<3, false, true, true>(A, xu8, nullptr, s);
      return k == 5 ? launch_conv_first_tma_t<5, false, false, true>(A, xu8, nullptr, s)
                    : launch_conv_first_tma_t<3, false, false, true>(A, xu8, nullptr, s);
    }
  }
  if (A.pool == 2 && g_opt_first_pool_tc) {
#define BNN_FTCP(KK, CC)                                                                          \
  if (k == KK && c == CC)                                                                          \
    return wide ? launch_conv_first_tc_pool_t<KK, 64, CC, SRC>(A, xu8, T, s)                      \
                : launch_conv_first_tc_pool_t<KK, 32, CC, SRC>(A, xu8, T, s)
    if constexpr (SRC != kSrcBits) {
      BNN_FTCP(3, 1); BNN_FTCP(3, 3); BNN_FTCP(5, 1); BNN_FTCP(5, 3);
    } else {
      BNN_FTCP(3, 1); BNN_FTCP(3, 2); BNN_FTCP(3, 3); BNN_FTCP(3, 4); BNN_FTCP(3, 5);
      BNN_FTCP(5, 1); BNN_FTCP(5, 2); BNN_FTCP(5, 3);
      BNN_FTCP(7, 1); BNN_FTCP(7, 2);
    }
#undef BNN_FTCP
  }
#define BNN_FTC(KK, CC)                                                                           \
  if (k == KK && c == CC)                                                                          \
    return wide ? launch_conv_first_tc_t<KK, 128, CC, SRC>(A, xu8, T, s)                          \
                : launch_conv_first_tc_t<KK, 32, CC, SRC>(A, xu8, T, s)
  if constexpr (SRC != kSrcBits) {
    BNN_FTC(3, 1); BNN_FTC(3, 3); BNN_FTC(5, 1); BNN_FTC(5, 3);
  } else {
    BNN_FTC(3, 1); BNN_FTC(3, 2); BNN_FTC(3, 3); BNN_FTC(3, 4); BNN_FTC(3, 5);
    BNN_FTC(5, 1); BNN_FTC(5, 2); BNN_FTC(5, 3);
    BNN_FTC(7, 1); BNN_FTC(7, 2);
  }
#undef BNN_FTC
  return fail(BNN_E_UNSUPPORTED, "conv_first_tc: k=%d c_in=%d", k, c);
}

template <int K, int CW, int NT>
bnn_status launch_conv_tc_t(ConvArgs A, cudaStream_t s) {
  using C = ConvTcCfg<K, CW, NT>;
  auto kfn = conv_tc_kernel<K, CW, NT>;
  const int occ = tc_occupancy(kfn, C::SMEM, C::TMEM_COLS);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + NT - 1) / NT));
  kfn<<<grid, 256, C::SMEM, s>>>(A);
  return check_launch("conv_tc_kernel");
}

// (k, words per pixel) -> tensor-core instantiation; returns false if none applies
bool tc_supported(int k, int cw) {
  if (g_opt_conv_tc == 0) return false;
  if (g_opt_conv_tc_fp4 && (k == 3 || k == 5 || k == 7)) return true;  // small + streamed (big) kernels
  return (k == 5 && (cw == 1 || cw == 2)) || (k == 3 && (cw == 1 || cw == 2 || cw == 4)) || (k == 7 && cw == 1);
}

template <int K, int CG, int NT, int P = 1>
bnn_status launch_conv_tc4_big_t(ConvArgs A, cudaStream_t s) {
  using C = ConvTc4BigCfg<K, CG, NT, P>;
  auto kfn = conv_tc4_big_kernel<K, CG, NT, P>;
  ensure_smem(kfn, C::SMEM);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)((A.n + P - 1) / P) * A.tiles_x * A.tiles_y;  // P images per tile
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int groups = (A.c_out + NT - 1) / NT;
  // one CTA per SM in total (TMEM 512 columns, ~200 KB smem): split the SMs over the channel groups
  const int64_t per_group = std::max<int64_t>(1, num_sms() / groups);
  const int64_t gx = std::min<int64_t>(A.total_tiles, per_group);
  dim3 grid((unsigned)gx, (unsigned)groups);
  // the weight operand, expanded once for this call (stream-ordered scratch), then one bulk copy per
  // stage in the kernel instead of an expansion per stage and tile
  uint8_t* img = nullptr;
  const int nstage = (A.cw + CG - 1) / CG;
  if (g_opt_big_img && A.bimg == nullptr && A.total_tiles > (int64_t)gx) {
    if (scratch_alloc(reinterpret_cast<void**>(&img), (size_t)groups * nstage * C::B_BYTES, s) == cudaSuccess) {
      prep_tc4_big_kernel<K, CG, NT><<<dim3((unsigned)nstage, (unsigned)groups), 256, 0, s>>>(A, img);
      A.bimg = img;
    } else {
      (void)cudaGetLastError();
      img = nullptr;
    }
  }
  kfn<<<grid, 256, C::SMEM, s>>>(A);
  bnn_status st = check_launch("conv_tc4_big_kernel");
  if (img != nullptr) cudaFreeAsync(img, s);
  return st;
}

template <int K, int CW, int NT>
bnn_status launch_conv_tc4_t(ConvArgs A, cudaStream_t s) {
  using C = ConvTc4Cfg<K, CW, NT>;
  auto kfn = conv_tc4_kernel<K, CW, NT>;
  const int occ = tc_occupancy(kfn, C::SMEM, C::TMEM_COLS);
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + NT - 1) / NT));
  kfn<<<grid, 256, C::SMEM, s>>>(A);
  return check_launch("conv_tc4_kernel");
}

template <int K, bool PAIR>
bnn_status launch_conv_tc4_pool3_t(ConvArgs A, cudaStream_t s) {
  using CF = ConvTc4Pool3Cfg<K, PAIR>;
  auto kfn = conv_tc4_pool3_kernel<K, PAIR>;
  const int occ = tc_occupancy(kfn, CF::SMEM, CF::TMEM_COLS, CF::THREADS);
  A.trace = g_trace_layer == 1 ? g_trace : nullptr;
  A.trace_cap = g_trace_cap;
  A.tiles_y = (A.H + CF::P::TH - 1) / CF::P::TH;
  A.tiles_x = (A.W + CF::P::TW - 1) / CF::P::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31) - 1) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const unsigned gy = (unsigned)((A.c_out + CF::P::NT - 1) / CF::P::NT);
  if (PAIR) {
    const int64_t pairs = std::min<int64_t>((A.total_tiles + 1) / 2, (int64_t)num_sms() * occ / 2);
    launch_pdl_cluster(kfn, dim3((unsigned)(2 * std::max<int64_t>(pairs, 1)), gy), dim3(CF::THREADS), CF::SMEM, s, 2, A);
  } else {
    const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
    launch_pdl(kfn, dim3((unsigned)std::max<int64_t>(gx, 1), gy), dim3(CF::THREADS), CF::SMEM, s, A);
  }
  return check_launch(PAIR ? "conv_tc4_pool3_kernel<pair>" : "conv_tc4_pool3_kernel");
}

template <int K>
bnn_status launch_conv_tc4_pool_t(ConvArgs A, cudaStream_t s) {
  using C = ConvTc4PoolCfg<K>;
  auto kfn = conv_tc4_pool_kernel<K>;
  if (g_opt_conv_pool3) {
    if (g_opt_conv_pair && A.bimg != nullptr) return launch_conv_tc4_pool3_t<K, true>(A, s);
    return launch_conv_tc4_pool3_t<K, false>(A, s);
  }
  if (g_opt_conv_pair == 2 && A.bimg != nullptr) {  // CTA pairs (cta_group::2): each SM reads half of B per MMA
    using CP = ConvTc4PoolCfg<K, true>;
    auto kp = conv_tc4_pool_kernel<K, true>;
    const int occ = tc_occupancy(kp, CP::SMEM, CP::TMEM_COLS, kTc4PoolThreads);
    A.tiles_y = (A.H + CP::TH - 1) / CP::TH;
    A.tiles_x = (A.W + CP::TW - 1) / CP::TW;
    A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
    if (A.total_tiles >= (1ll << 31) - 1) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
    A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
    A.fd_tx = FastDiv((uint32_t)A.tiles_x);
    A.tiles_per_cta = 0;
    A.trace = g_trace_layer == 1 ? g_trace : nullptr;
    A.trace_cap = g_trace_cap;
    const int64_t pairs = std::min<int64_t>((A.total_tiles + 1) / 2, (int64_t)num_sms() * occ / 2);
    dim3 grid((unsigned)(2 * std::max<int64_t>(pairs, 1)), (unsigned)((A.c_out + CP::NT - 1) / CP::NT));
    launch_pdl_cluster(kp, grid, dim3(kTc4PoolThreads), CP::SMEM, s, 2, A);
    return check_launch("conv_tc4_pool_kernel<pair>");
  }
  const int occ = tc_occupancy(kfn, C::SMEM, C::TMEM_COLS, kTc4PoolThreads);
  A.trace = g_trace_layer == 1 ? g_trace : nullptr;
  A.trace_cap = g_trace_cap;
  A.tiles_y = (A.H + C::TH - 1) / C::TH;
  A.tiles_x = (A.W + C::TW - 1) / C::TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = 0;
  const int64_t gx = std::min<int64_t>(A.total_tiles, (int64_t)num_sms() * occ);
  dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)((A.c_out + C::NT - 1) / C::NT));
  launch_pdl(kfn, grid, dim3(kTc4PoolThreads), C::SMEM, s, A);
  return check_launch("conv_tc4_pool_kernel");
}

bool use_conv_pool_tc(int k, int cw, int pool) {
  return g_opt_conv_tc_fp4 && g_opt_conv_pool_tc && pool == 2 && cw == 1 && (k == 3 || k == 5);
}

bnn_status dispatch_conv_tc(int k, int cw, const ConvArgs& A, cudaStream_t s) {
  if (use_conv_pool_tc(k, cw, A.pool)) return k == 5 ? launch_conv_tc4_pool_t<5>(A, s) : launch_conv_tc4_pool_t<3>(A, s);
  if (g_opt_conv_tc_fp4) {
    if (k == 5 && cw == 1) return launch_conv_tc4_t<5, 1, 32>(A, s);
    if (k == 5 && cw == 2) return launch_conv_tc4_t<5, 2, 64>(A, s);
    if (k == 3 && cw == 1) return launch_conv_tc4_t<3, 1, 32>(A, s);
    if (k == 3 && cw == 2) return launch_conv_tc4_t<3, 2, 64>(A, s);
    if (k == 3 && cw == 4) return launch_conv_tc4_t<3, 4, 128>(A, s);
    if (k == 7 && cw == 1) return launch_conv_tc4_t<7, 1, 32>(A, s);
    if (k == 3) return A.W == 8 ? launch_conv_tc4_big_t<3, 4, 128, 2>(A, s) : launch_conv_tc4_big_t<3, 4, 128>(A, s);
    if (k == 5) return launch_conv_tc4_big_t<5, 2, 128>(A, s);
    if (k == 7) return launch_conv_tc4_big_t<7, 1, 128>(A, s);
  }
  if (k == 5 && cw == 1) return launch_conv_tc_t<5, 1, 32>(A, s);
  if (k == 5 && cw == 2) return launch_conv_tc_t<5, 2, 64>(A, s);
  if (k == 3 && cw == 1) return launch_conv_tc_t<3, 1, 32>(A, s);
  if (k == 3 && cw == 2) return launch_conv_tc_t<3, 2, 64>(A, s);
  if (k == 3 && cw == 4) return launch_conv_tc_t<3, 4, 128>(A, s);
  if (k == 7 && cw == 1) return launch_conv_tc_t<7, 1, 32>(A, s);
  return fail(BNN_E_UNSUPPORTED, "conv_tc: k=%d cw=%d", k, cw);
}

template <int K, int WY, int WX>
bnn_status launch_conv_real_u8_t(RealConvArgs A, cudaStream_t s) {
  constexpr int PR = 2, PC = 8;
  constexpr int TH = WY * PR, TW = WX * PC;
  constexpr int IR = TH + K - 1, IC = TW + K - 1;
  A.tiles_y = (A.H + TH - 1) / TH;
  A.tiles_x = (A.W + TW - 1) / TW;
  A.total_tiles = (int64_t)A.n * A.tiles_x * A.tiles_y;
  if (A.total_tiles >= (1ll << 31)) return fail(BNN_E_UNSUPPORTED, "conv: too many tiles (%lld) for one launch", (long long)A.total_tiles);
  A.fd_img = FastDiv((uint32_t)(A.tiles_x * A.tiles_y));
  A.fd_tx = FastDiv((uint32_t)A.tiles_x);
  A.tiles_per_cta = choose_tpc(A.total_tiles, false);
  const int nb = K * K * A.c_in, nw = (nb + 3) / 4;
  const size_t in_bytes = (size_t)((IR * IC * A.c_in + 15) & ~15);
  const size_t smem = in_bytes + (size_t)nw * TH * TW * 4 + (size_t)nw * 32 * 4;
  if (smem > 200 * 1024) return fail(BNN_E_UNSUPPORTED, "bnn_conv2d: real first layer k=%d c_in=%d too large", K, A.c_in);
  auto kfn = conv_real_u8_kernel<K, PR, PC, WY, WX>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t gx = (A.total_tiles + A.tiles_per_cta - 1) / A.tiles_per_cta;
  dim3 grid((unsigned)gx, (unsigned)((A.c_out + 31) / 32));
  kfn<<<grid, WY * WX * 32, smem, s>>>(A);
  return check_launch("conv_real_u8_kernel");
}

template <int WY, int WX>
bnn_status dispatch_conv_bin(int k, const ConvArgs& A, bool patch, cudaStream_t s) {
  if (patch) {
    switch (k) {
      case 1: return launch_conv_patch_t<1, WY, WX>(A, s);
      case 3: return launch_conv_patch_t<3, WY, WX>(A, s);
      case 5: return launch_conv_patch_t<5, WY, WX>(A, s);
      case 7: return launch_conv_patch_t<7, WY, WX>(A, s);
    }
  } else {
    switch (k) {
      case 1: return launch_conv_bin_t<1, WY, WX>(A, s);
      case 3: return launch_conv_bin_t<3, WY, WX>(A, s);
      case 5: return launch_conv_bin_t<5, WY, WX>(A, s);
      case 7: return launch_conv_bin_t<7, WY, WX>(A, s);
    }
  }
  return fail(BNN_E_UNSUPPORTED, "bnn_conv2d: k=%d not supported (1, 3, 5, 7)", k);
}

template <int WY, int WX>
bnn_status dispatch_conv_real_u8(int k, const RealConvArgs& A, cudaStream_t s) {
  switch (k) {
    case 1: return launch_conv_real_u8_t<1, WY, WX>(A, s);
    case 3: return launch_conv_real_u8_t<3, WY, WX>(A, s);
    case 5: return launch_conv_real_u8_t<5, WY, WX>(A, s);
    case 7: return launch_conv_real_u8_t<7, WY, WX>(A, s);
  }
  return fail(BNN_E_UNSUPPORTED, "bnn_conv2d: k=%d not supported (1, 3, 5, 7)", k);
}

// First-layer kernels for few input channels (one word per pixel):
//   strip  : K-tap row strips stacked rpw = 32/(K c_in) rows per word (conv_strip_kernel)
//   patch  : the K*K*c_in bits packed densely (conv_patch_kernel)
// conv_algo: 0 auto, 1 generic one-word-per-tap, 2 dense patch, 3 strip.
int strip_words(int c_in, int k) {
  const int S = k * c_in;
  if (k < 3 || S > 32) return 1 << 30;
  const int rpw = 32 / S;
  return (k + rpw - 1) / rpw;
}
int dense_words(int c_in, int k) { return (k * k * c_in + 31) / 32; }

bool use_strip(int c_in, int k) {
  if (c_in >= 32 || strip_words(c_in, k) > 7) return false;
  if (g_opt_conv_algo == 3) return true;
  return g_opt_conv_algo == 0 && strip_words(c_in, k) <= dense_words(c_in, k);
}

// lane = pixel first-layer kernel (conv_algo 0 = auto or 4 = forced)
bool use_first_lp(int c_in, int k) {
  if (g_opt_conv_algo != 0 && g_opt_conv_algo != 4) return false;
  const int nw = strip_words(c_in, k);
  if (c_in >= 32 || nw > 7) return false;
  const bool have = (k == 3 && nw <= 3) || (k == 5 && (nw <= 3 || nw == 5)) || (k == 7 && (nw == 2 || nw == 4 || nw == 7));
  if (!have) return false;
  return g_opt_conv_algo == 4 || nw <= dense_words(c_in, k);
}

bool use_patch(int c_in, int k) {
  return (g_opt_conv_algo == 0 || g_opt_conv_algo == 2) && c_in < 32 && k > 1 && k * k * c_in <= 256;
}

bnn_status launch_conv(const void* x, bnn_dtype x_dt, int n, int h, int w, int c_in, const uint32_t* wt, int c_out,
                       int k, const int32_t* thr, const uint8_t* flip, int pool, uint32_t* y, void* acc,
                       cudaStream_t s, const uint8_t* bimg = nullptr) {
  if ((int64_t)n * h * w == 0) return BNN_OK;
  const bool small = (w <= 8 || h <= 8);
  if (x_dt == BNN_BITS) {
    ConvArgs A{};
    A.x = (const uint32_t*)x; A.wt = wt; A.thr = thr; A.flip = flip; A.y = y; A.acc = (int32_t*)acc;
    A.n = n; A.H = h; A.W = w; A.cw = (c_in + 31) / 32; A.c_in = c_in; A.c_out = c_out;
    A.cwo = (c_out + 31) / 32; A.pool = pool; A.bimg = bimg;
    if (use_first_tc(c_in, k, kSrcBits)) return dispatch_conv_first_tc<kSrcBits>(k, A, nullptr, nullptr, s);
    if (use_first_lp(c_in, k)) return dispatch_conv_first_lp<false>(k, strip_words(c_in, k), A, nullptr, nullptr, s);
    if (c_in >= 32 && tc_supported(k, A.cw)) return dispatch_conv_tc(k, A.cw, A, s);
    if (use_strip(c_in, k))
      return small ? dispatch_conv_strip<4, 1, false>(k, A, nullptr, nullptr, s)
                   : dispatch_conv_strip<4, 2, false>(k, A, nullptr, nullptr, s);
    const bool patch = use_patch(c_in, k);
    return small ? dispatch_conv_bin<4, 1>(k, A, patch, s) : dispatch_conv_bin<4, 2>(k, A, patch, s);
  }
  RealConvArgs A{};
  A.x = x; A.wt = wt; A.thr = thr; A.flip = flip; A.y = y; A.acc = acc;
  A.n = n; A.H = h; A.W = w; A.c_in = c_in; A.c_out = c_out; A.cwo = (c_out + 31) / 32; A.pool = pool;
  if (x_dt == BNN_U8 && use_first_tc(c_in, k, kSrcReal)) {
    ConvArgs B{};
    B.x = nullptr; B.wt = wt; B.thr = thr; B.flip = flip; B.y = y; B.acc = (int32_t*)acc;
    B.n = n; B.H = h; B.W = w; B.cw = 1; B.c_in = c_in; B.c_out = c_out; B.cwo = (c_out + 31) / 32; B.pool = pool;
    return dispatch_conv_first_tc<kSrcReal>(k, B, (const uint8_t*)x, nullptr, s);
  }
  if (x_dt == BNN_U8) return small ? dispatch_conv_real_u8<4, 1>(k, A, s) : dispatch_conv_real_u8<4, 2>(k, A, s);
  // f32
  const int64_t work = (int64_t)n * (h / pool) * (w / pool) * A.cwo * 32;
  conv_real_f32_kernel<<<grid_for(work, 256), 256, 0, s>>>(A, k);
  return check_launch("conv_real_f32_kernel");
}

// The kernel family launch_conv / the fused first layer pick (kept in step with the dispatch above).
const char* conv_kernel_name(bnn_dtype x_dt, int c_in, int k, int pool) {
  if (x_dt == BNN_U8) {
    if (!use_first_tc(c_in, k, kSrcReal)) return "conv_real_u8_kernel";
    const bool tma = g_opt_first_real_tma && g_opt_first_tma && g_opt_first_pool_tc && pool == 2 && c_in == 3 &&
                     (k == 3 || k == 5) && tma_encoder() != nullptr;  // (+ 16-byte row pitch, checked at launch)
    return tma ? "conv_first_tma_pool_kernel" : "conv_first_tc_kernel";
  }
  if (x_dt == BNN_F32) return "conv_real_f32_kernel";
  if (use_first_tc(c_in, k, kSrcBits)) return "conv_first_tc_kernel";
  if (use_first_lp(c_in, k)) return "conv_first_lp_kernel";
  if (c_in >= 32 && tc_supported(k, (c_in + 31) / 32)) {
    const int cw = (c_in + 31) / 32;
    if (!g_opt_conv_tc_fp4) return "conv_tc_kernel";
    if (use_conv_pool_tc(k, cw, pool)) return g_opt_conv_pool3 ? "conv_tc4_pool3_kernel" : "conv_tc4_pool_kernel";
    const bool small = (k == 5 && cw <= 2) || (k == 3 && (cw <= 2 || cw == 4)) || (k == 7 && cw == 1);
    return small ? "conv_tc4_kernel" : "conv_tc4_big_kernel";
  }
  if (use_strip(c_in, k)) return "conv_strip_kernel";
  if (use_patch(c_in, k)) return "conv_patch_kernel";
  return "conv_bin_kernel";
}

// ---------------------------------------------------------------------------- dense
// Dense layers with a real batch and a long reduction run on the tensor cores (kind::mxf4).
// fp32 accumulation (TMEM, K-split partial sums) is exact only for |acc| <= d <= 2^24: wider layers stay
// on the integer pipe (dense_kernel), whatever the option says
constexpr int64_t kDenseTcMaxWords = (int64_t{1} << 24) / 32;
bool use_dense_tc(int n, int64_t dw) {
  return g_opt_dense_tc && n >= 256 && dw >= 32 && (dw % 4) == 0 && dw <= kDenseTcMaxWords;
}

// K-split factor of dense_tc4_kernel (grid.z): split when the tile grid leaves SMs idle (FC1 at 8192
// images: 64 tiles -> 2); each split then needs at least 4 stages of 16 words
int dense_ks(int n, int l, int64_t dw) {
  if (!use_dense_tc(n, dw) || !g_opt_dense_ksplit) return 1;
  const int nt = l > 128 ? 256 : 128, groups = (l + nt - 1) / nt;
  const int ctas = std::min((n + 127) / 128, num_sms()) * groups, nstage = (int)((dw + 15) / 16);
  if (2 * ctas > num_sms() || nstage < 8) return 1;
  return std::max(1, std::min(std::min(num_sms() / ctas, nstage / 4), 4));
}

bnn_status launch_dense(const uint32_t* x, int n, int64_t d, const uint32_t* wt, int l, const int32_t* thr,
                        const uint8_t* flip, uint32_t* y, int32_t* acc, int32_t* cls, cudaStream_t s,
                        const uint8_t* bimg = nullptr) {
  if (n == 0) return BNN_OK;
  DenseArgs A{};
  A.x = x; A.wt = wt; A.thr = thr; A.flip = flip; A.y = y; A.acc = acc; A.bimg = bimg;
  A.cls = (l <= 32) ? cls : nullptr;
  A.n = n; A.l = l; A.lw = (l + 31) / 32; A.d = d; A.dw = (d + 31) / 32;
  constexpr int PI = 8, NWARP = 8, DC = 64;
  bnn_status st;
  if (use_dense_tc(n, A.dw)) {
    // tensor cores: NT = 128 (l <= 128) or 256 output columns per CTA group
    const bool wide = l > 128;
    A.cls = (l <= (wide ? 256 : 128)) ? cls : nullptr;
    const int ntiles = (n + 127) / 128;
    const int nt = wide ? 256 : 128, groups = (l + nt - 1) / nt;
    A.ks = dense_ks(n, l, A.dw);
    float* part = nullptr;
    if (A.ks > 1) {
      const size_t bytes = (size_t)A.ks * ntiles * 128 * groups * nt * sizeof(float);
      if (scratch_alloc(reinterpret_cast<void**>(&part), bytes, s) != cudaSuccess) {
        cudaGetLastError();
        A.ks = 1;
        part = nullptr;
      }
      A.part = part;
    }
    if (A.ks > 1) A.cls = cls;  // the reduction kernel takes the argmax over all l
    // activation stages by TMA (2-D map over the packed [n, dw] words; dw % 4 == 0 keeps rows 16-byte aligned)
    CUtensorMap xmap;
    std::memset(&xmap, 0, sizeof(xmap));
    bool tmax = g_opt_dense_tma && aligned16(x) && tma_encoder() != nullptr;
    const bool two = !wide && ntiles >= 2 * num_sms();  // two CTAs per SM (DenseTc4Cfg<128, true>) for large batches
    if (tmax) {
      const cuuint64_t dims[2] = {(cuuint64_t)A.dw, (cuuint64_t)n};
      const cuuint64_t strides[1] = {(cuuint64_t)A.dw * 4};
      const cuuint32_t box[2] = {(cuuint32_t)(wide ? DenseTc4Cfg<256>::KC : (two ? DenseTc4Cfg<128, true>::KC : DenseTc4Cfg<128>::KC)), 128};
      const cuuint32_t estr[2] = {1, 1};
      tmax = tma_encoder()(&xmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(x), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    auto launch = [&](auto kfn, uint32_t smem) {
      ensure_smem(kfn, smem);
      const int cps = (!wide && two) ? DenseTc4Cfg<128, true>::CPS : 1;
      dim3 grid((unsigned)std::min(ntiles, num_sms() * cps), (unsigned)groups, (unsigned)A.ks);
      launch_pdl(kfn, grid, dim3(256), smem, s, A, xmap);
    };
    if (wide) {
      if (tmax) launch(dense_tc4_kernel<256, true>, DenseTc4Cfg<256>::SMEM_TMAX);
      else launch(dense_tc4_kernel<256>, DenseTc4Cfg<256>::SMEM);
    } else {
      if (two) {
        if (tmax) launch(dense_tc4_kernel<128, true, true>, DenseTc4Cfg<128, true>::SMEM_TMAX);
        else launch(dense_tc4_kernel<128, false, true>, DenseTc4Cfg<128, true>::SMEM);
      } else {
        if (tmax) launch(dense_tc4_kernel<128, true>, DenseTc4Cfg<128>::SMEM_TMAX);
        else launch(dense_tc4_kernel<128>, DenseTc4Cfg<128>::SMEM);
      }
    }
    st = check_launch("dense_tc4_kernel");
    if (st == BNN_OK && A.ks > 1) {
      launch_pdl(dense_tc4_reduce_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, s, A, groups * nt, ntiles * 128);
      st = check_launch("dense_tc4_reduce_kernel");
    }
    if (part != nullptr) cudaFreeAsync(part, s);
    if (st != BNN_OK) return st;
    if (cls != nullptr && A.cls == nullptr) {
      launch_pdl(argmax_kernel, dim3(grid_for((int64_t)n * 32, 256)), dim3(256), 0, s, (const int32_t*)acc, n, l, cls);
      return check_launch("argmax_kernel");
    }
    return BNN_OK;
  }
  if (n <= g_opt_gemv_max_n) {
    const int warps = std::min(32, l);
    launch_pdl(dense_gemv_kernel, dim3((unsigned)n, (unsigned)A.lw), dim3(warps * 32), 0, s, A);
    st = check_launch("dense_gemv_kernel");
  } else {
    dim3 grid((unsigned)((n + PI * NWARP - 1) / (PI * NWARP)), (unsigned)A.lw);
    launch_pdl(dense_kernel<PI, NWARP, DC>, grid, dim3(NWARP * 32), 0, s, A);
    st = check_launch("dense_kernel");
  }
  if (st != BNN_OK) return st;
  if (cls != nullptr && l > 32) {
    launch_pdl(argmax_kernel, dim3(grid_for((int64_t)n * 32, 256)), dim3(256), 0, s, (const int32_t*)acc, n, l, cls);
    return check_launch("argmax_kernel");
  }
  return BNN_OK;
}

}  // namespace

// =============================================================================== public ABI
extern "C" {

const char* bnn_last_error(void) { return g_err.c_str(); }

int bnn_version(void) { return 101; }

bnn_status bnn_set_trace(unsigned long long* buf, int cap) {
  if (cap < 0 || (buf == nullptr) != (cap == 0)) return fail(BNN_E_ARG, "bnn_set_trace: bad buffer / capacity");
#ifndef BNN_TRACE
  if (buf != nullptr) return fail(BNN_E_UNSUPPORTED, "bnn_set_trace: this build records no trace (build with --trace)");
#endif
  g_trace = buf;
  g_trace_cap = cap;
  return BNN_OK;
}

int bnn_set_option(const char* key, int value) {
  if (key == nullptr) return (int)fail(BNN_E_ARG, "bnn_set_option: null key");
  if (strcmp(key, "conv_algo") == 0) { g_opt_conv_algo = value; return BNN_OK; }
  if (strcmp(key, "tiles_per_cta") == 0) { g_opt_tiles_per_cta = value; return BNN_OK; }
  if (strcmp(key, "gemv_max_n") == 0) { g_opt_gemv_max_n = value; return BNN_OK; }
  if (strcmp(key, "conv_tc") == 0) { g_opt_conv_tc = value; return BNN_OK; }
  if (strcmp(key, "conv_pair") == 0) { g_opt_conv_pair = value; return BNN_OK; }
  if (strcmp(key, "conv_pool3") == 0) { g_opt_conv_pool3 = value; return BNN_OK; }
  if (strcmp(key, "first_pool_tc") == 0) { g_opt_first_pool_tc = value; return BNN_OK; }
  if (strcmp(key, "first_tma") == 0) { g_opt_first_tma = value; return BNN_OK; }
  if (strcmp(key, "first_fp4") == 0) { g_opt_first_fp4 = value; return BNN_OK; }
  if (strcmp(key, "first_db") == 0) { g_opt_first_db = value; return BNN_OK; }
#ifdef BNN_TRACE
  if (strcmp(key, "first_exp") == 0) { g_opt_first_exp = value; return BNN_OK; }  // diagnostics build only
  if (strcmp(key, "trace_layer") == 0) { g_trace_layer = value; return BNN_OK; }  // diagnostics build only
#endif
  if (strcmp(key, "dense_ksplit") == 0) { g_opt_dense_ksplit = value; return BNN_OK; }
  if (strcmp(key, "first_real_tma") == 0) { g_opt_first_real_tma = value; return BNN_OK; }
  if (strcmp(key, "luma_band") == 0) { g_opt_luma_band = value; return BNN_OK; }
  if (strcmp(key, "fused_max_n") == 0) { g_opt_fused_max_n = value; return BNN_OK; }
  if (strcmp(key, "fused_tc") == 0) { g_opt_fused_tc = value; return BNN_OK; }
  if (strcmp(key, "alg1") == 0) { g_opt_alg1 = value; return BNN_OK; }
  if (strcmp(key, "csa") == 0) { g_opt_csa = value; return BNN_OK; }
  if (strcmp(key, "big_img") == 0) { g_opt_big_img = value; return BNN_OK; }
  if (strcmp(key, "streams") == 0) { g_opt_streams = value; return BNN_OK; }
  if (strcmp(key, "pdl") == 0) { g_opt_pdl = value; return BNN_OK; }
  if (strcmp(key, "conv_pool_tc") == 0) { g_opt_conv_pool_tc = value; return BNN_OK; }
  if (strcmp(key, "conv_tc_fp4") == 0) { g_opt_conv_tc_fp4 = value; return BNN_OK; }
  if (strcmp(key, "dense_tc") == 0) { g_opt_dense_tc = value; return BNN_OK; }
  if (strcmp(key, "dense_tma") == 0) { g_opt_dense_tma = value; return BNN_OK; }
  if (strcmp(key, "luma_fused") == 0) { g_opt_luma_fused = value; return BNN_OK; }
  if (strcmp(key, "fused_cluster") == 0) { g_opt_fused_cluster = value; return BNN_OK; }
  if (strcmp(key, "fused_cs") == 0) { g_opt_fused_cs = value; return BNN_OK; }
  if (strcmp(key, "fused_multi") == 0) { g_opt_fused_multi = value ? 1 : 0; return BNN_OK; }
  return (int)fail(BNN_E_ARG, "bnn_set_option: unknown key '%s'", key);
}

bnn_status bnn_pack(const void* x, bnn_dtype dt, int n, int h, int w, int c, int mode, const float* T, uint32_t* y,
                    bnn_stream_t stream) {
  if (n < 0 || h < 0 || w < 0 || c < 1) return fail(BNN_E_ARG, "bnn_pack: bad sizes n=%d h=%d w=%d c=%d", n, h, w, c);
  if ((int64_t)n * h * w > 0 && (x == nullptr || y == nullptr)) return fail(BNN_E_ARG, "bnn_pack: null pointer");
  if (dt != BNN_U8 && dt != BNN_I8 && dt != BNN_F32 && dt != BNN_I32) return fail(BNN_E_ARG, "bnn_pack: bad dtype %d", (int)dt);
  if (mode < BNN_SIGN || mode > BNN_LBP) return fail(BNN_E_ARG, "bnn_pack: bad mode %d", mode);
  if ((mode == BNN_THRESH_RGB || mode == BNN_THRESH_GRAY) && T == nullptr)
    return fail(BNN_E_ARG, "bnn_pack: threshold mode needs T");
  if ((mode == BNN_THRESH_GRAY || mode == BNN_LBP) && (c != 3 || dt != BNN_U8))
    return fail(BNN_E_CONFIG, "bnn_pack: GRAY/LBP need u8 input with c == 3");
  BNN_REQUIRE_ALIGNED(x, "bnn_pack x");
  BNN_REQUIRE_ALIGNED(y, "bnn_pack y");
  return launch_pack(x, dt, n, h, w, c, mode, T, y, (cudaStream_t)stream);
}

bnn_status bnn_conv2d(const void* x, bnn_dtype x_dt, int n, int h, int w, int c_in, const uint32_t* wt, int c_out,
                      int k, const int32_t* thr, const uint8_t* flip, int pool, uint32_t* y, void* acc,
                      bnn_stream_t stream) {
  if (n < 0 || h < 0 || w < 0 || c_in < 1 || c_out < 1) return fail(BNN_E_ARG, "bnn_conv2d: bad sizes");
  if (k != 1 && k != 3 && k != 5 && k != 7) return fail(BNN_E_UNSUPPORTED, "bnn_conv2d: k=%d not in {1,3,5,7}", k);
  if (pool != 1 && pool != 2) return fail(BNN_E_ARG, "bnn_conv2d: pool must be 1 or 2");
  if (pool == 2 && ((h & 1) || (w & 1))) return fail(BNN_E_SHAPE, "bnn_conv2d: pool 2 needs even h, w (got %d x %d)", h, w);
  if (x_dt != BNN_BITS && x_dt != BNN_U8 && x_dt != BNN_F32) return fail(BNN_E_CONFIG, "bnn_conv2d: x dtype must be BITS, U8 or F32");
  if (x_dt != BNN_BITS && c_in > 32) return fail(BNN_E_CONFIG, "bnn_conv2d: real first layer needs c_in <= 32");
  if ((int64_t)n * h * w > 0 && y == nullptr && acc == nullptr) return fail(BNN_E_ARG, "bnn_conv2d: y and acc both null");
  if ((int64_t)n * h * w > 0 && (x == nullptr || wt == nullptr)) return fail(BNN_E_ARG, "bnn_conv2d: null pointer");
  BNN_REQUIRE_ALIGNED(x, "bnn_conv2d x");
  BNN_REQUIRE_ALIGNED(wt, "bnn_conv2d wt");
  BNN_REQUIRE_ALIGNED(y, "bnn_conv2d y");
  BNN_REQUIRE_ALIGNED(acc, "bnn_conv2d acc");
  return launch_conv(x, x_dt, n, h, w, c_in, wt, c_out, k, thr, flip, pool, y, acc, (cudaStream_t)stream);
}

bnn_status bnn_maxpool(const uint32_t* x, int n, int h, int w, int c, uint32_t* y, bnn_stream_t stream) {
  if (n < 0 || h < 0 || w < 0 || c < 1) return fail(BNN_E_ARG, "bnn_maxpool: bad sizes");
  if ((h & 1) || (w & 1)) return fail(BNN_E_SHAPE, "bnn_maxpool: h, w must be even (got %d x %d)", h, w);
  if ((int64_t)n * h * w > 0 && (x == nullptr || y == nullptr)) return fail(BNN_E_ARG, "bnn_maxpool: null pointer");
  BNN_REQUIRE_ALIGNED(x, "bnn_maxpool x");
  BNN_REQUIRE_ALIGNED(y, "bnn_maxpool y");
  const int cw = (c + 31) / 32;
  const int64_t total = (int64_t)n * (h / 2) * (w / 2) * cw;
  if (total == 0) return BNN_OK;
  maxpool_or_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(x, n, h, w, cw, y);
  return check_launch("maxpool_or_kernel");
}

bnn_status bnn_dense(const uint32_t* x, int n, int64_t d, const uint32_t* wt, int l, const int32_t* thr,
                     const uint8_t* flip, uint32_t* y, int32_t* acc, int32_t* cls, bnn_stream_t stream) {
  if (n < 0 || d < 1 || l < 1) return fail(BNN_E_ARG, "bnn_dense: bad sizes");
  if (n > 0 && (x == nullptr || wt == nullptr)) return fail(BNN_E_ARG, "bnn_dense: null pointer");
  if (n > 0 && y == nullptr && acc == nullptr && cls == nullptr) return fail(BNN_E_ARG, "bnn_dense: no output");
  if (cls != nullptr && l > 32 && acc == nullptr) return fail(BNN_E_ARG, "bnn_dense: cls with l > 32 needs acc");
  if ((d + 31) / 32 > 0x7fffffffLL) return fail(BNN_E_ARG, "bnn_dense: d too large");
  BNN_REQUIRE_ALIGNED(x, "bnn_dense x");
  BNN_REQUIRE_ALIGNED(wt, "bnn_dense wt");
  BNN_REQUIRE_ALIGNED(y, "bnn_dense y");
  BNN_REQUIRE_ALIGNED(acc, "bnn_dense acc");
  BNN_REQUIRE_ALIGNED(cls, "bnn_dense cls");
  return launch_dense(x, n, d, wt, l, thr, flip, y, acc, cls, (cudaStream_t)stream);
}

bnn_status bnn_affine(const int32_t* acc, int n, int l, const float* scale, const float* bias, float* score,
                      int32_t* cls, bnn_stream_t stream) {
  if (n < 0 || l < 1 || l > 1024) return fail(BNN_E_ARG, "bnn_affine: bad sizes (need 1 <= l <= 1024)");
  if (n > 0 && (acc == nullptr || scale == nullptr || bias == nullptr)) return fail(BNN_E_ARG, "bnn_affine: null pointer");
  if (n > 0 && score == nullptr && cls == nullptr) return fail(BNN_E_ARG, "bnn_affine: no output");
  BNN_REQUIRE_ALIGNED(acc, "bnn_affine acc");
  BNN_REQUIRE_ALIGNED(scale, "bnn_affine scale");
  BNN_REQUIRE_ALIGNED(bias, "bnn_affine bias");
  BNN_REQUIRE_ALIGNED(score, "bnn_affine score");
  BNN_REQUIRE_ALIGNED(cls, "bnn_affine cls");
  if (n == 0) return BNN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  launch_pdl(affine_argmax_kernel, dim3(grid_for((int64_t)n * 32, 256)), dim3(256), 0, s, acc, n, l, scale, bias, score, cls);
  return check_launch("affine_argmax_kernel");
}

}  // extern "C"

// =============================================================================== network
struct LayerPlan {
  int kind, k, c_in, c_out, pool, l;
  int H, W;          // input spatial dims (conv)
  int64_t d;         // dense input length
  bnn_dtype x_dt;    // conv input dtype (BITS, or U8/F32 for a real first layer)
  const uint32_t* wt;
  const int32_t* thr;
  const uint8_t* flip;
  int64_t out_words_per_img;  // packed output words per image (hidden layers)
  uint8_t* bimg = nullptr;    // pre-expanded weight operand image (pool-in-N tensor-core kernels) or null
  int bimg_fp4 = -1;          // first layer: which operand type the image was built for (1 e2m1, 0 int8)
};

struct bnn_net {
  int h, w, c;
  bnn_dtype in_dt;
  int mode;
  const float* T;
  int c0;  // channels after input binarization
  std::vector<LayerPlan> L;
  int chunk;
  int64_t img_bytes;
  int64_t packed_in_words;  // per image
  int64_t buf_words;        // per image, max over hidden layers
  uint32_t* packed_in = nullptr;
  uint32_t* buf[2] = {nullptr, nullptr};
  int32_t* logits_tmp = nullptr;
  unsigned* fused_ctr = nullptr;  // grid-barrier counter of fused_small_kernel
  uint32_t* fused_w1 = nullptr;   // [32, 3] densely packed conv1 weights for fused_small_kernel
  // the paper's design (bnn_set_option("alg1", 1)), allocated on first use
  int alg1_chunk = 0;
  uint32_t* alg1_patch = nullptr;             // [chunk, H, W, C] Alg. 1 packed patches
  int32_t* alg1_f = nullptr;                  // [chunk, H, W, C_out] GEMM-conv output
  int32_t* alg1_g[2] = {nullptr, nullptr};    // pooled maps (ping-pong)
  uint32_t* alg1_bits[2] = {nullptr, nullptr};  // packed dense inputs / outputs
  std::vector<uint32_t*> alg1_w;              // per conv layer: Wp [c_out, C]
  // host-pipeline resources (lazy)
  int hchunk = 0;
  void* d_in[2] = {nullptr, nullptr};
  int32_t* d_logits[2] = {nullptr, nullptr};
  int32_t* d_cls[2] = {nullptr, nullptr};
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  // per-stage profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> pending_stage;  // stage of event pair i (events 2i, 2i+1 of the pool)
  std::vector<double> stage_ms;
  std::vector<int64_t> stage_launches;
  // graph-replayed staging path (bnn_forward_staged)
  int max_staged = 0;
  void* st_in = nullptr;
  int32_t* st_logits = nullptr;
  int32_t* st_cls = nullptr;
  cudaStream_t cap_stream = nullptr;
  // second chunk stream of bnn_forward (chunks alternate streams so one chunk's low-occupancy dense
  // layers and kernel tails overlap the next chunk's convolutions); its own workspace, lazily created
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint32_t* packed_in2 = nullptr;
  uint32_t* buf2[2] = {nullptr, nullptr};
  int32_t* logits_tmp2 = nullptr;
  std::vector<cudaGraphExec_t> graphs;  // index n
};

namespace {

void net_free(bnn_net* net) {
  if (!net) return;
  for (LayerPlan& P : net->L) cudaFree(P.bimg);
  cudaFree(net->packed_in);
  cudaFree(net->buf[0]);
  cudaFree(net->buf[1]);
  cudaFree(net->logits_tmp);
  cudaFree(net->fused_ctr);
  cudaFree(net->fused_w1);
  cudaFree(net->alg1_patch);
  cudaFree(net->alg1_f);
  for (int i = 0; i < 2; ++i) { cudaFree(net->alg1_g[i]); cudaFree(net->alg1_bits[i]); }
  for (uint32_t* w : net->alg1_w) cudaFree(w);
  for (int i = 0; i < 2; ++i) {
    cudaFree(net->d_in[i]);
    cudaFree(net->d_logits[i]);
    cudaFree(net->d_cls[i]);
    if (net->ev_h2d[i]) cudaEventDestroy(net->ev_h2d[i]);
    if (net->ev_comp[i]) cudaEventDestroy(net->ev_comp[i]);
    if (net->ev_d2h[i]) cudaEventDestroy(net->ev_d2h[i]);
  }
  for (cudaEvent_t e : net->ev_pool) cudaEventDestroy(e);
  for (cudaGraphExec_t g : net->graphs)
    if (g) cudaGraphExecDestroy(g);
  cudaFree(net->st_in);
  cudaFree(net->st_logits);
  cudaFree(net->st_cls);
  if (net->cap_stream) cudaStreamDestroy(net->cap_stream);
  if (net->h2d) cudaStreamDestroy(net->h2d);
  if (net->s2) cudaStreamDestroy(net->s2);
  if (net->ev_fork) cudaEventDestroy(net->ev_fork);
  if (net->ev_join) cudaEventDestroy(net->ev_join);
  cudaFree(net->packed_in2);
  cudaFree(net->buf2[0]);
  cudaFree(net->buf2[1]);
  cudaFree(net->logits_tmp2);
  if (net->d2h) cudaStreamDestroy(net->d2h);
  delete net;
}

bnn_status check_pad_bits(const uint32_t* dev, int64_t rows, int64_t words_per_row, int valid_bits_last,
                          const char* what, int layer) {
  if (valid_bits_last == 32) return BNN_OK;
  std::vector<uint32_t> h((size_t)(rows * words_per_row));
  cudaError_t e = cudaMemcpy(h.data(), dev, h.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_net_create: reading %s of layer %d: %s", what, layer, cudaGetErrorString(e));
  const uint32_t mask = (valid_bits_last == 0) ? 0u : (0xffffffffu >> valid_bits_last);
  for (int64_t r = 0; r < rows; ++r)
    if (h[(size_t)(r * words_per_row + words_per_row - 1)] & mask)
      return fail(BNN_E_PADBITS, "bnn_net_create: layer %d %s row %lld has nonzero pad bits", layer, what, (long long)r);
  return BNN_OK;
}

// Returns the start event of a new (start, end) pair for `stage`, recorded on s; or null.
struct ProfScope {
  bnn_net* net;
  cudaStream_t s;
  cudaEvent_t end = nullptr;
  ProfScope(bnn_net* n, int stage, cudaStream_t st) : net(n), s(st) {
    if (!net->prof) return;
    if (net->ev_used + 2 > net->ev_pool.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { net->prof = false; return; }
        net->ev_pool.push_back(e);
      }
    }
    cudaEvent_t b = net->ev_pool[net->ev_used];
    end = net->ev_pool[net->ev_used + 1];
    net->ev_used += 2;
    net->pending_stage.push_back(stage);
    cudaEventRecord(b, s);
  }
  ~ProfScope() {
    if (end) cudaEventRecord(end, s);
  }
};

// Layer 0 fuses the input threshold (SIGN / THRESH_RGB on u8 pixels) into the strip conv kernel.
bool fused_input(const bnn_net* net) {
  if (net->mode != BNN_SIGN && net->mode != BNN_THRESH_RGB) return false;
  if (net->in_dt != BNN_U8 || net->c > 4 || net->L[0].kind != 1) return false;
  return use_first_tc(net->c, net->L[0].k, kSrcThresh) || use_first_lp(net->c, net->L[0].k) || use_strip(net->c, net->L[0].k);
}

// THRESH_GRAY / LBP nets whose first layer fits the TMA-fed pooled kernel: luma_u8img4_kernel writes a
// 0/1 u8 image into the packed-input workspace and the TMA kernel reads it with threshold x > 0.
bool use_luma_tma(const bnn_net* net) {
  if (net->mode != BNN_THRESH_GRAY && net->mode != BNN_LBP) return false;
  if (net->in_dt != BNN_U8 || net->c != 3 || net->L[0].kind != 1) return false;
  const LayerPlan& P = net->L[0];
  return g_opt_first_tma && g_opt_first_pool_tc && g_opt_conv_algo == 0 && P.pool == 2 && (P.k == 3 || P.k == 5) &&
         (P.c_in == 1 || P.c_in == 3) && (P.W * 3) % 16 == 0 && (net->w % 4) == 0 && tma_encoder() != nullptr &&
         net->packed_in_words * 4 >= (int64_t)P.H * P.W * 3;
}

// THRESH_GRAY (luma_fused >= 1) / LBP (luma_fused == 2) with the luma computed inside conv1_fp4_pool_kernel
// (no luma pre-pass).  LBP's in-kernel neighbour pass is byte-granular and measured slower than the
// pre-pass (config 2: 5.6 vs 9.4 M images/s), so LBP keeps luma_u8img4_kernel by default.
bool luma_fused(const bnn_net* net) {
  const bool mode_ok = net->mode == BNN_THRESH_GRAY ? g_opt_luma_fused >= 1 : (net->mode == BNN_LBP && g_opt_luma_fused == 2);
  return mode_ok && g_opt_first_fp4 && use_luma_tma(net);
}

// Small batches of a vehicle-shaped net run as one cooperative kernel (k_fused_small.cuh).
bool use_fused_small(const bnn_net* net, int nb) {
  if (nb < 1 || nb > g_opt_fused_max_n || net->fused_ctr == nullptr || net->fused_w1 == nullptr) return false;
  if (net->in_dt != BNN_U8 || (net->mode != BNN_SIGN && net->mode != BNN_THRESH_RGB) || net->c > 4) return false;
  if (net->L.size() != 5 || (net->h % 4) != 0 || (net->w % 4) != 0) return false;
  const LayerPlan &a = net->L[0], &b = net->L[1], &d1 = net->L[2], &d2 = net->L[3], &d3 = net->L[4];
  if (a.kind != 1 || a.c_out != 32 || a.pool != 2 || a.k * a.k * net->c > 96) return false;
  if (b.kind != 1 || b.c_in != 32 || b.c_out != 32 || b.pool != 2 || (b.k != 1 && b.k != 3 && b.k != 5)) return false;
  if (d1.kind != 2 || d2.kind != 2 || d3.kind != 2) return false;
  if (net->buf_words < (int64_t)(net->h / 4) * (net->w / 4) + (d1.l + 31) / 32) return false;  // y2 + h1 in buf[1]
  if (d1.l > kFusedMaxL || d2.l > kFusedMaxL || d3.l > 32) return false;
  return true;
}

bnn_status launch_fused_small(bnn_net* net, const void* images, int nb, int32_t* logits, int32_t* cls, cudaStream_t s) {
  const LayerPlan &a = net->L[0], &b = net->L[1], &d1 = net->L[2], &d2 = net->L[3], &d3 = net->L[4];
  FusedSmallArgs A{};
  A.x = (const uint8_t*)images; A.T = (net->mode == BNN_THRESH_RGB) ? net->T : nullptr;
  A.n = nb; A.H = net->h; A.W = net->w; A.C = net->c; A.K1 = a.k; A.K2 = b.k;
  A.w1 = a.wt; A.w1p = net->fused_w1; A.thr1 = a.thr; A.flip1 = a.flip; A.w2 = b.wt; A.thr2 = b.thr; A.flip2 = b.flip;
  A.f1 = d1.wt; A.f2 = d2.wt; A.f3 = d3.wt; A.thr_f1 = d1.thr; A.thr_f2 = d2.thr; A.flip_f1 = d1.flip; A.flip_f2 = d2.flip;
  A.l1 = d1.l; A.l2 = d2.l; A.l3 = d3.l;
  A.y1 = net->buf[0]; A.y2 = net->buf[1]; A.h1 = net->buf[1] + (int64_t)nb * (net->h / 4) * (net->w / 4); A.logits = logits; A.cls = cls; A.barrier = net->fused_ctr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)num_sms());
  cfg.blockDim = dim3(kFusedWarps * 32);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency of the whole grid (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (b.k == 5) cudaLaunchKernelEx(&cfg, fused_small_kernel<5>, A);
  else if (b.k == 3) cudaLaunchKernelEx(&cfg, fused_small_kernel<3>, A);
  else cudaLaunchKernelEx(&cfg, fused_small_kernel<1>, A);
  return check_launch("fused_small_kernel");
}

// Cluster size of fused_cluster_kernel on the current device: 16 (non-portable) if the device runs a
// 16-CTA cluster of it, else 8; 0 if neither (then the cooperative kernel serves).  Returned as
// size + 256 x (clusters of that size the device holds at once)
template <typename F>
int fused_cluster_size(F kfn, size_t smem, int only = 0) {
  return dev_cached(reinterpret_cast<const char*>(kfn) + 2 + (only == 8), [&] {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int cs : {kClusterMax, 8}) {
      if (only != 0 && cs != only) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)cs);
      cfg.blockDim = dim3(kFusedWarps * 32);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kfn, &cfg) == cudaSuccess && nclusters >= 1) {
        (void)cudaGetLastError();
        return cs + 256 * nclusters;
      }
      (void)cudaGetLastError();
    }
    return 0;
  });
}

bnn_status launch_fused_cluster(bnn_net* net, const void* images, int nb, int32_t* logits, int32_t* cls, cudaStream_t s,
                                bool* launched) {
  *launched = false;
  const LayerPlan &a = net->L[0], &b = net->L[1], &d1 = net->L[2], &d2 = net->L[3], &d3 = net->L[4];
  FusedSmallArgs A{};
  A.x = (const uint8_t*)images; A.T = (net->mode == BNN_THRESH_RGB) ? net->T : nullptr;
  A.n = nb; A.H = net->h; A.W = net->w; A.C = net->c; A.K1 = a.k; A.K2 = b.k;
  A.w1 = a.wt; A.w1p = net->fused_w1; A.thr1 = a.thr; A.flip1 = a.flip; A.w2 = b.wt; A.thr2 = b.thr; A.flip2 = b.flip;
  A.f1 = d1.wt; A.f2 = d2.wt; A.f3 = d3.wt; A.thr_f1 = d1.thr; A.thr_f2 = d2.thr; A.flip_f1 = d1.flip; A.flip_f2 = d2.flip;
  A.l1 = d1.l; A.l2 = d2.l; A.l3 = d3.l;
  A.logits = logits; A.cls = cls;
  A.trace = g_trace_layer == 2 ? g_trace : nullptr;
  // bulk copies need 16-byte rows: raw image rows (W C bytes) and FC1 weight rows (H/4 W/4 words)
  if ((net->w * net->c) % 16 != 0 || ((net->h / 4) * (net->w / 4)) % 4 != 0) return BNN_OK;
  const size_t smem = (size_t)FusedClusterLayout(net->h, net->w, net->c, a.k, 8, d1.l, d2.l, d3.l).total * 4;
  if (smem > 200 * 1024) return BNN_OK;
  auto go = [&](auto kfn) -> bnn_status {
    int cv = fused_cluster_size(kfn, smem, g_opt_fused_cs == 8 ? 8 : 0);
    // more images than 16-CTA clusters fit at once: 8-CTA clusters (twice as many fit; ~1 us slower per image)
    if (g_opt_fused_cs == 0 && g_opt_fused_multi && (cv & 255) == 16 && nb > (cv >> 8)) {
      const int cv8 = fused_cluster_size(kfn, smem, 8);
      if ((cv8 & 255) == 8) cv = cv8;
    }
    const int cs = cv & 255;
    if (cs == 0) return BNN_OK;
    // one cluster per image up to what the device holds at once (images are independent; a cluster
    // serves images cid, cid + ncl, ... when the batch is larger)
    const int ncl = std::max(1, std::min(nb, (cv >> 8) * g_opt_fused_multi + (1 - g_opt_fused_multi)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cs * ncl));
    cfg.blockDim = dim3(kFusedWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kfn, A);
    *launched = true;
    return check_launch("fused_cluster_kernel");
  };
  // conv2 on the tensor cores inside the cluster when its pool-in-N weight image exists (k = 5, 32 -> 32 channels)
  const bool tc2 = g_opt_fused_tc && b.k == 5 && b.bimg != nullptr && b.c_in == 32 && b.c_out == 32 && b.pool == 2 &&
                   net->w % 32 == 0;  // (conv2 tiles' 8-word pooled rows stay inside the W/4-word map rows)
  A.w2img = tc2 ? b.bimg : nullptr;
  // conv1 on the tensor cores (conv1_fp4's strips and weight image) for the vehicle geometry
  const bool tc1 = tc2 && a.k == 5 && net->c == 3 && a.c_out == 32 && a.pool == 2 && a.bimg != nullptr && a.bimg_fp4 == 1;
  A.w1img = tc1 ? a.bimg : nullptr;
  if (b.k == 5) return tc1 ? go(fused_cluster_kernel<5, true, true>) : (tc2 ? go(fused_cluster_kernel<5, true>) : go(fused_cluster_kernel<5>));
  if (b.k == 3) return go(fused_cluster_kernel<3>);
  return go(fused_cluster_kernel<1>);
}

bnn_status forward_chunk(bnn_net* net, const void* images, int nb, int32_t* logits, int32_t* cls, cudaStream_t s) {
  if (use_fused_small(net, nb)) {
    ProfScope ps(net, 1, s);
    if (g_opt_fused_cluster) {
      bool launched = false;
      const bnn_status st = launch_fused_cluster(net, images, nb, logits, cls, s, &launched);
      if (st != BNN_OK || launched) return st;
    }
    return launch_fused_small(net, images, nb, logits, cls, s);
  }
  const void* cur = images;
  bnn_dtype cur_dt = net->in_dt;
  const int nl = (int)net->L.size();
  int first = 0;
  if (fused_input(net)) {
    // layer 0 reads the u8 image and thresholds it itself (no packed round trip through HBM)
    const LayerPlan& P = net->L[0];
    ProfScope ps(net, 1, s);
    ConvArgs A{};
    A.x = nullptr; A.wt = P.wt; A.thr = P.thr; A.flip = P.flip; A.y = net->buf[0]; A.acc = nullptr;
    A.n = nb; A.H = P.H; A.W = P.W; A.cw = 1; A.c_in = P.c_in; A.c_out = P.c_out;
    A.cwo = (P.c_out + 31) / 32; A.pool = P.pool;
    A.bimg = (P.bimg_fp4 == (g_opt_first_fp4 ? 1 : 0)) ? P.bimg : nullptr;  // image built for this operand type
    const float* T = (net->mode == BNN_THRESH_RGB) ? net->T : nullptr;
    const bool small = (P.W <= 8 || P.H <= 8);
    bnn_status st;
    if (use_first_tc(P.c_in, P.k, kSrcThresh))
      st = dispatch_conv_first_tc<kSrcThresh>(P.k, A, (const uint8_t*)images, T, s);
    else if (use_first_lp(P.c_in, P.k))
      st = dispatch_conv_first_lp<true>(P.k, strip_words(P.c_in, P.k), A, (const uint8_t*)images, T, s);
    else
      st = small ? dispatch_conv_strip<4, 1, true>(P.k, A, (const uint8_t*)images, T, s)
                 : dispatch_conv_strip<4, 2, true>(P.k, A, (const uint8_t*)images, T, s);
    if (st != BNN_OK) return st;
    cur = net->buf[0];
    cur_dt = BNN_BITS;
    first = 1;
  } else if (luma_fused(net)) {
    // THRESH_GRAY / LBP fused into the first layer: the builders compute the integer luma from the raw RGB box
    const LayerPlan& P = net->L[0];
    ProfScope ps(net, 1, s);
    ConvArgs A{};
    A.wt = P.wt; A.thr = P.thr; A.flip = P.flip; A.y = net->buf[0];
    A.n = nb; A.H = P.H; A.W = P.W; A.cw = 1; A.c_in = P.c_in; A.c_out = P.c_out;
    A.cwo = (P.c_out + 31) / 32; A.pool = P.pool;
    A.bimg = (P.bimg_fp4 == 1) ? P.bimg : nullptr;
    bnn_status st;
    if (net->mode == BNN_LBP)
      st = P.k == 5 ? launch_conv1_fp4_t<5, false, kBinLbp>(A, (const uint8_t*)images, nullptr, s)
                    : launch_conv1_fp4_t<3, false, kBinLbp>(A, (const uint8_t*)images, nullptr, s);
    else
      st = P.k == 5 ? launch_conv1_fp4_t<5, false, kBinGray>(A, (const uint8_t*)images, net->T, s)
                    : launch_conv1_fp4_t<3, false, kBinGray>(A, (const uint8_t*)images, net->T, s);
    if (st != BNN_OK) return st;
    cur = net->buf[0];
    cur_dt = BNN_BITS;
    first = 1;
  } else if (use_luma_tma(net)) {
    {
      ProfScope ps(net, 0, s);
      const int64_t npix = (int64_t)nb * net->h * net->w;
      const size_t lsm = luma_band_smem(net->w);
      bnn_status st = BNN_OK;
      const int64_t nblk = (int64_t)nb * ((net->h + kLumaBand - 1) / kLumaBand);
      if (g_opt_luma_band && lsm <= 48 * 1024 && nblk < (1ll << 31)) {  // one CTA per band of rows (luma computed once)
        luma_band_kernel<<<(unsigned)nblk, 256, lsm, s>>>((const uint8_t*)images, nb, net->h, net->w, net->mode, net->T,
                                                         reinterpret_cast<uint8_t*>(net->packed_in));
        st = check_launch("luma_band_kernel");
      } else {
        luma_u8img4_kernel<<<grid_for(npix / 4, 256), 256, 0, s>>>((const uint8_t*)images, nb, net->h, net->w, net->mode,
                                                                   net->T, reinterpret_cast<uint8_t*>(net->packed_in));
        st = check_launch("luma_u8img4_kernel");
      }
      if (st != BNN_OK) return st;
    }
    const LayerPlan& P = net->L[0];
    ProfScope ps(net, 1, s);
    ConvArgs A{};
    A.wt = P.wt; A.thr = P.thr; A.flip = P.flip; A.y = net->buf[0];
    A.n = nb; A.H = P.H; A.W = P.W; A.cw = 1; A.c_in = P.c_in; A.c_out = P.c_out;
    A.cwo = (P.c_out + 31) / 32; A.pool = P.pool;
    A.bimg = (P.bimg_fp4 == (g_opt_first_fp4 ? 1 : 0)) ? P.bimg : nullptr;
    bnn_status st = dispatch_first_tma(P.k, A, reinterpret_cast<const uint8_t*>(net->packed_in), nullptr, s);
    if (st != BNN_OK) return st;
    cur = net->buf[0];
    cur_dt = BNN_BITS;
    first = 1;
  } else if (net->mode != BNN_MODE_NONE) {
    ProfScope ps(net, 0, s);
    bnn_status st = launch_pack(images, net->in_dt, nb, net->h, net->w, net->c, net->mode, net->T, net->packed_in, s);
    if (st != BNN_OK) return st;
    cur = net->packed_in;
    cur_dt = BNN_BITS;
  }
  for (int i = first; i < nl; ++i) {
    const LayerPlan& P = net->L[i];
    const bool last = (i == nl - 1);
    bnn_status st;
    ProfScope ps(net, i + 1, s);
    if (P.kind == 1) {
      uint32_t* out = net->buf[i & 1];
      st = launch_conv(cur, cur_dt, nb, P.H, P.W, P.c_in, P.wt, P.c_out, P.k, P.thr, P.flip, P.pool, out, nullptr, s,
                       cur_dt == BNN_BITS && P.c_in == 32 ? P.bimg : nullptr);
      cur = out;
      cur_dt = BNN_BITS;
    } else if (!last) {
      uint32_t* out = net->buf[i & 1];
      st = launch_dense((const uint32_t*)cur, nb, P.d, P.wt, P.l, P.thr, P.flip, out, nullptr, nullptr, s, P.bimg);
      cur = out;
    } else {
      int32_t* lg = logits ? logits : net->logits_tmp;
      st = launch_dense((const uint32_t*)cur, nb, P.d, P.wt, P.l, nullptr, nullptr, nullptr, lg,
                        P.l <= 32 ? cls : nullptr, s, P.bimg);
      if (st == BNN_OK && cls != nullptr && P.l > 32) {
        ProfScope pa(net, nl + 1, s);
        argmax_kernel<<<grid_for((int64_t)nb * 32, 256), 256, 0, s>>>(lg, nb, P.l, cls);
        st = check_launch("argmax_kernel");
      }
    }
    if (st != BNN_OK) return st;
  }
  return BNN_OK;
}

int launches_per_chunk(const bnn_net* net, bool want_cls, int nb) {
  if (use_fused_small(net, nb)) return 1;
  int n = (net->mode != BNN_MODE_NONE && !fused_input(net) && !luma_fused(net) ? 1 : 0) + (int)net->L.size();
  if (want_cls && net->L.back().l > 32) n += 1;
  for (const LayerPlan& P : net->L)  // K-split dense layers add their reduction kernel
    if (P.kind == 2 && dense_ks(nb, P.l, (P.d + 31) / 32) > 1) n += 1;
  return n;
}

}  // namespace

extern "C" {

bnn_status bnn_net_create(int h, int w, int c, bnn_dtype in_dt, int mode, const float* T, const bnn_layer* layers,
                          int n_layers, int max_batch, bnn_net** out) {
  if (out == nullptr) return fail(BNN_E_ARG, "bnn_net_create: out is null");
  *out = nullptr;
  if (h < 1 || w < 1 || c < 1 || n_layers < 1 || layers == nullptr) return fail(BNN_E_ARG, "bnn_net_create: bad sizes");
  if (max_batch < 1 || max_batch > 65536) return fail(BNN_E_ARG, "bnn_net_create: max_batch must be in [1, 65536]");
  if (in_dt != BNN_U8 && in_dt != BNN_F32) return fail(BNN_E_CONFIG, "bnn_net_create: input dtype must be U8 or F32");
  if (mode < BNN_MODE_NONE || mode > BNN_LBP) return fail(BNN_E_ARG, "bnn_net_create: bad mode %d", mode);
  if ((mode == BNN_THRESH_RGB || mode == BNN_THRESH_GRAY) && T == nullptr) return fail(BNN_E_ARG, "bnn_net_create: mode needs T");
  if ((mode == BNN_THRESH_GRAY || mode == BNN_LBP) && (c != 3 || in_dt != BNN_U8))
    return fail(BNN_E_CONFIG, "bnn_net_create: GRAY/LBP need u8 input with 3 channels");
  if (layers[n_layers - 1].kind != 2) return fail(BNN_E_CONFIG, "bnn_net_create: the last layer must be dense");

  bnn_net* net = new (std::nothrow) bnn_net();
  if (!net) return fail(BNN_E_NOMEM, "bnn_net_create: out of host memory");
  net->h = h; net->w = w; net->c = c; net->in_dt = in_dt; net->mode = mode; net->T = T;
  net->img_bytes = (int64_t)h * w * c * (in_dt == BNN_U8 ? 1 : 4);
  net->c0 = (mode == BNN_THRESH_GRAY) ? 1 : (mode == BNN_LBP ? 3 : c);
  net->packed_in_words = (mode == BNN_MODE_NONE) ? 0 : (int64_t)h * w * ((net->c0 + 31) / 32);
  int H = h, W = w, C = net->c0;
  int64_t D = -1;  // >= 0 once in the dense part
  net->buf_words = 1;
  for (int i = 0; i < n_layers; ++i) {
    const bnn_layer& Ls = layers[i];
    LayerPlan P{};
    P.kind = Ls.kind; P.k = Ls.k; P.c_out = Ls.c_out; P.pool = Ls.pool; P.l = Ls.l;
    P.wt = Ls.wt; P.thr = Ls.thr; P.flip = Ls.flip;
    if (Ls.wt == nullptr) { net_free(net); return fail(BNN_E_ARG, "bnn_net_create: layer %d has no weights", i); }
    if (!aligned16(Ls.wt)) { net_free(net); return fail(BNN_E_ALIGN, "bnn_net_create: layer %d weights not 16-byte aligned", i); }
    if (Ls.kind == 1) {
      if (D >= 0) { net_free(net); return fail(BNN_E_SHAPE, "bnn_net_create: conv layer %d after a dense layer", i); }
      if (Ls.k != 1 && Ls.k != 3 && Ls.k != 5 && Ls.k != 7) { net_free(net); return fail(BNN_E_UNSUPPORTED, "bnn_net_create: layer %d k=%d", i, Ls.k); }
      if (Ls.c_out < 1 || (Ls.pool != 1 && Ls.pool != 2)) { net_free(net); return fail(BNN_E_ARG, "bnn_net_create: layer %d bad c_out/pool", i); }
      if (Ls.pool == 2 && ((H & 1) || (W & 1))) { net_free(net); return fail(BNN_E_SHAPE, "bnn_net_create: layer %d pools an odd map %dx%d", i, H, W); }
      P.c_in = C; P.H = H; P.W = W;
      P.x_dt = (i == 0 && mode == BNN_MODE_NONE) ? in_dt : BNN_BITS;
      if (P.x_dt != BNN_BITS && C > 32) { net_free(net); return fail(BNN_E_CONFIG, "bnn_net_create: real first layer needs c <= 32"); }
      const int cw = (C + 31) / 32;
      bnn_status st = check_pad_bits(Ls.wt, (int64_t)Ls.c_out * Ls.k * Ls.k, cw, C % 32 == 0 ? 32 : C % 32, "weights", i);
      if (st != BNN_OK) { net_free(net); return st; }
      H /= Ls.pool; W /= Ls.pool; C = Ls.c_out;
      P.out_words_per_img = (int64_t)H * W * ((C + 31) / 32);
      net->buf_words = std::max(net->buf_words, P.out_words_per_img);
    } else if (Ls.kind == 2) {
      if (i == 0 && mode == BNN_MODE_NONE) { net_free(net); return fail(BNN_E_CONFIG, "bnn_net_create: mode NONE needs a conv first layer"); }
      if (Ls.l < 1) { net_free(net); return fail(BNN_E_ARG, "bnn_net_create: layer %d l < 1", i); }
      if (D < 0) {
        if (C % 32 != 0 && (int64_t)H * W != 1) {
          net_free(net);
          return fail(BNN_E_UNSUPPORTED, "bnn_net_create: conv->dense at layer %d needs channels %% 32 == 0 (got %d)", i, C);
        }
        D = (int64_t)H * W * C;
      }
      P.d = D;
      const int64_t dw = (D + 31) / 32;
      bnn_status st = check_pad_bits(Ls.wt, Ls.l, dw, D % 32 == 0 ? 32 : (int)(D % 32), "weights", i);
      if (st != BNN_OK) { net_free(net); return st; }
      D = Ls.l;
      P.out_words_per_img = (Ls.l + 31) / 32;
      if (i != n_layers - 1) net->buf_words = std::max(net->buf_words, P.out_words_per_img);
    } else {
      net_free(net);
      return fail(BNN_E_ARG, "bnn_net_create: layer %d has unknown kind %d", i, Ls.kind);
    }
    net->L.push_back(P);
  }
  net->chunk = max_batch;
  cudaError_t e = cudaSuccess;
  if (net->packed_in_words) e = cudaMalloc(&net->packed_in, (size_t)(net->packed_in_words * max_batch * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->buf[0], (size_t)(net->buf_words * max_batch * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->buf[1], (size_t)(net->buf_words * max_batch * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->logits_tmp, (size_t)net->L.back().l * max_batch * 4);
  if (e == cudaSuccess) e = cudaMalloc(&net->fused_ctr, 2 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(net->fused_ctr, 0, 2 * sizeof(unsigned));
  if (e == cudaSuccess && net->L[0].kind == 1 && net->L[0].c_out == 32 && net->L[0].k * net->L[0].k * net->c <= 96 &&
      net->c <= 4) {
    e = cudaMalloc(&net->fused_w1, 32 * 3 * sizeof(uint32_t));
    if (e == cudaSuccess) prep_fused_w1_kernel<<<1, 32>>>(net->L[0].wt, net->L[0].k, net->c, net->fused_w1);
  }
  if (e != cudaSuccess) {
    net_free(net);
    return fail(BNN_E_CUDA, "bnn_net_create: workspace allocation: %s", cudaGetErrorString(e));
  }
  // Weight operands of the pool-in-N tensor-core kernels and of the tensor-core dense layers, expanded
  // once here (the kernels then stage them with bulk copies instead of re-expanding the packed weights
  // in every CTA).
  for (size_t i = 0; i < net->L.size() && e == cudaSuccess; ++i) {
    LayerPlan& P = net->L[i];
    if (P.kind == 2) {
      // dense layers on the tensor cores at the chunk size: the e2m1 weight image, one bulk copy per stage
      const int64_t dw = (P.d + 31) / 32;
      if (!use_dense_tc(std::min(net->chunk, 256), dw)) continue;
      DenseArgs D{};
      D.wt = P.wt; D.l = P.l; D.d = P.d; D.dw = dw;
      const bool wide = P.l > 128;
      const int nt = wide ? 256 : 128, groups = (P.l + nt - 1) / nt;
      const int kc = wide ? DenseTc4Cfg<256>::KC : DenseTc4Cfg<128>::KC;
      const int nstage = (int)((dw + kc - 1) / kc);
      const size_t bb = wide ? DenseTc4Cfg<256>::B_BYTES : DenseTc4Cfg<128>::B_BYTES;
      if ((e = cudaMalloc(&P.bimg, (size_t)groups * nstage * bb)) != cudaSuccess) break;
      if (wide) prep_dense_tc4_kernel<256><<<dim3((unsigned)nstage, (unsigned)groups), 256>>>(D, P.bimg);
      else prep_dense_tc4_kernel<128><<<dim3((unsigned)nstage, (unsigned)groups), 256>>>(D, P.bimg);
      e = cudaGetLastError();
      continue;
    }
    if (P.kind != 1 || P.pool != 2 || (P.k != 3 && P.k != 5)) continue;
    ConvArgs A{};
    A.wt = P.wt; A.thr = P.thr; A.flip = P.flip; A.c_in = P.c_in; A.c_out = P.c_out;
    const int groups = (P.c_out + 31) / 32;
    const bool first_u8 = i == 0 && net->in_dt == BNN_U8 && net->c == 3 &&
                          (net->mode == BNN_SIGN || net->mode == BNN_THRESH_RGB || use_luma_tma(net));
    if (first_u8) {
      const bool fp4 = g_opt_first_fp4 != 0;
      const size_t bb = P.k == 5 ? (fp4 ? Conv1Fp4Cfg<5>::B_BYTES : FirstTmaCfg<5, false>::B_BYTES)
                                 : (fp4 ? Conv1Fp4Cfg<3>::B_BYTES : FirstTmaCfg<3, false>::B_BYTES);
      if ((e = cudaMalloc(&P.bimg, (size_t)groups * bb)) != cudaSuccess) break;
      P.bimg_fp4 = fp4 ? 1 : 0;
      if (P.k == 5) {
        if (fp4) prep_conv1_fp4_kernel<5><<<groups, 256>>>(A, P.bimg);
        else prep_first_tma_kernel<5, false><<<groups, 256>>>(A, P.bimg);
      } else {
        if (fp4) prep_conv1_fp4_kernel<3><<<groups, 256>>>(A, P.bimg);
        else prep_first_tma_kernel<3, false><<<groups, 256>>>(A, P.bimg);
      }
    } else if (P.x_dt == BNN_BITS && P.c_in == 32) {
      const size_t bytes = (size_t)groups * (P.k == 5 ? ConvTc4PoolCfg<5>::B_BYTES : ConvTc4PoolCfg<3>::B_BYTES);
      if ((e = cudaMalloc(&P.bimg, bytes)) != cudaSuccess) break;
      if (P.k == 5) prep_tc4_pool_kernel<5><<<groups, 256>>>(A, P.bimg);
      else prep_tc4_pool_kernel<3><<<groups, 256>>>(A, P.bimg);
    }
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    net_free(net);
    return fail(BNN_E_CUDA, "bnn_net_create: weight image preparation: %s", cudaGetErrorString(e));
  }
  *out = net;
  return BNN_OK;
}

}  // extern "C" (reopened below)

namespace {

// ---- the paper's design as a comparison pipeline (k_alg1.cuh): supported for u8 SIGN / THRESH_RGB
// nets whose conv layers have k <= 5 (B = k*k <= 32 bits per channel word) and no thresholds/flips
bnn_status second_stream_prepare(bnn_net* net) {
  if (net->s2 != nullptr) return BNN_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&net->s2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->ev_join, cudaEventDisableTiming);
  const size_t mb = (size_t)net->chunk;
  if (e == cudaSuccess && net->packed_in_words) e = cudaMalloc(&net->packed_in2, (size_t)(net->packed_in_words * mb * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->buf2[0], (size_t)(net->buf_words * mb * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->buf2[1], (size_t)(net->buf_words * mb * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->logits_tmp2, (size_t)net->L.back().l * mb * 4);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(BNN_E_CUDA, "bnn_forward: second stream workspace: %s", cudaGetErrorString(e));
  }
  return BNN_OK;
}

// forward_chunk on the second workspace (the kernels read the workspace pointers from the net)
bnn_status forward_chunk_ws2(bnn_net* net, const void* x, int nb, int32_t* logits, int32_t* cls, cudaStream_t s) {
  std::swap(net->packed_in, net->packed_in2);
  std::swap(net->buf[0], net->buf2[0]);
  std::swap(net->buf[1], net->buf2[1]);
  std::swap(net->logits_tmp, net->logits_tmp2);
  bnn_status st = forward_chunk(net, x, nb, logits, cls, s);
  std::swap(net->packed_in, net->packed_in2);
  std::swap(net->buf[0], net->buf2[0]);
  std::swap(net->buf[1], net->buf2[1]);
  std::swap(net->logits_tmp, net->logits_tmp2);
  return st;
}

bool alg1_supported(const bnn_net* net) {
  if (net->in_dt != BNN_U8 || (net->mode != BNN_SIGN && net->mode != BNN_THRESH_RGB) || net->w > 512) return false;
  for (size_t i = 0; i < net->L.size(); ++i) {
    const LayerPlan& P = net->L[i];
    if (P.kind == 1 && (P.k > 5 || P.thr != nullptr || P.flip != nullptr)) return false;
    if (P.kind == 2 && i + 1 < net->L.size() && (P.thr != nullptr || P.flip != nullptr)) return false;
  }
  return true;
}

bnn_status alg1_prepare(bnn_net* net) {
  if (net->alg1_chunk > 0) return BNN_OK;
  const int chunk = std::min(net->chunk, 256);
  int64_t patch = 0, f = 0, g = 0, bits = 0;
  for (const LayerPlan& P : net->L) {
    if (P.kind == 1) {
      patch = std::max<int64_t>(patch, (int64_t)P.H * P.W * P.c_in);
      f = std::max<int64_t>(f, (int64_t)P.H * P.W * P.c_out);
      g = std::max<int64_t>(g, (int64_t)(P.H / P.pool) * (P.W / P.pool) * P.c_out);
    } else {
      bits = std::max<int64_t>(bits, std::max<int64_t>((P.d + 31) / 32, (P.l + 31) / 32));
    }
  }
  cudaError_t e = cudaMalloc(&net->alg1_patch, (size_t)(patch * chunk * 4));
  if (e == cudaSuccess) e = cudaMalloc(&net->alg1_f, (size_t)(f * chunk * 4));
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&net->alg1_g[i], (size_t)(g * chunk * 4));
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&net->alg1_bits[i], (size_t)(bits * chunk * 4));
  for (const LayerPlan& P : net->L) {
    if (P.kind != 1 || e != cudaSuccess) continue;
    uint32_t* wp = nullptr;
    e = cudaMalloc(&wp, (size_t)P.c_out * P.c_in * 4);
    if (e == cudaSuccess) {
      net->alg1_w.push_back(wp);
      alg1_prep_weights_kernel<<<grid_for((int64_t)P.c_out * P.c_in, 256), 256>>>(P.wt, P.c_out, P.k, P.c_in, wp);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(BNN_E_CUDA, "alg1: workspace: %s", cudaGetErrorString(e));
  net->alg1_chunk = chunk;
  return BNN_OK;
}

bnn_status alg1_forward_chunk(bnn_net* net, const void* images, int nb, int32_t* logits, int32_t* cls, cudaStream_t s) {
  const void* cur = images;
  bool cur_u8 = true;
  int g = 0, conv_i = 0;
  const uint32_t* xbits = nullptr;
  int64_t xd = 0;
  for (size_t i = 0; i < net->L.size(); ++i) {
    const LayerPlan& P = net->L[i];
    ProfScope ps(net, (int)i + 1, s);
    if (P.kind == 1) {
      const int R = (P.k - 1) / 2;
      const size_t smem = (size_t)(kAlg1S + 2 * R) * (P.W + 2 * R) * sizeof(int);
      dim3 grid((unsigned)((P.H + kAlg1S - 1) / kAlg1S), (unsigned)nb), block((unsigned)P.W, kAlg1S);
      if (cur_u8)
        alg1_im2col_pack_kernel<true><<<grid, block, smem, s>>>(cur, net->mode == BNN_THRESH_RGB ? net->T : nullptr,
                                                                P.H, P.W, P.c_in, P.k, net->alg1_patch);
      else
        alg1_im2col_pack_kernel<false><<<grid, block, smem, s>>>(cur, nullptr, P.H, P.W, P.c_in, P.k, net->alg1_patch);
      bnn_status st = check_launch("alg1_im2col_pack_kernel");
      if (st != BNN_OK) return st;
      const int64_t M = (int64_t)nb * P.H * P.W;
      dim3 gg((unsigned)((M + kAlg1Tile - 1) / kAlg1Tile), (unsigned)((P.c_out + kAlg1Tile - 1) / kAlg1Tile));
      alg1_gemm_conv_kernel<<<gg, dim3(kAlg1Tile, kAlg1Tile), 0, s>>>(net->alg1_patch, net->alg1_w[conv_i], M, P.c_in,
                                                                      P.c_out, P.k * P.k, net->alg1_f);
      if ((st = check_launch("alg1_gemm_conv_kernel")) != BNN_OK) return st;
      if (P.pool == 2) {
        alg1_maxpool_kernel<<<grid_for((int64_t)nb * (P.H / 2) * (P.W / 2) * P.c_out, 256), 256, 0, s>>>(
            net->alg1_f, nb, P.H, P.W, P.c_out, net->alg1_g[g]);
        if ((st = check_launch("alg1_maxpool_kernel")) != BNN_OK) return st;
        cur = net->alg1_g[g];
        g ^= 1;
      } else {
        // unpooled: the GEMM output is the next layer's map; copy so alg1_f can be rewritten
        cudaMemcpyAsync(net->alg1_g[g], net->alg1_f, (size_t)M * P.c_out * 4, cudaMemcpyDeviceToDevice, s);
        cur = net->alg1_g[g];
        g ^= 1;
      }
      cur_u8 = false;
      ++conv_i;
      continue;
    }
    // dense: pack the previous map first (Table 2 "including packing")
    if (xbits == nullptr) {
      alg1_pack_kernel<<<grid_for((int64_t)nb * ((P.d + 31) / 32), 256), 256, 0, s>>>((const int32_t*)cur, nb, P.d,
                                                                                       net->alg1_bits[0]);
      bnn_status st = check_launch("alg1_pack_kernel");
      if (st != BNN_OK) return st;
      xbits = net->alg1_bits[0];
    }
    xd = P.d;
    const bool last = i + 1 == net->L.size();
    uint32_t* ybits = net->alg1_bits[xbits == net->alg1_bits[0] ? 1 : 0];
    int32_t* lg = logits != nullptr ? logits : net->logits_tmp;
    if (!last) cudaMemsetAsync(ybits, 0, (size_t)nb * ((P.l + 31) / 32) * 4, s);
    alg1_fc_kernel<<<dim3((unsigned)P.l, (unsigned)nb), 64, 0, s>>>(xbits, xd, P.wt, P.l, last ? nullptr : ybits,
                                                                    last ? lg : nullptr);
    bnn_status st = check_launch("alg1_fc_kernel");
    if (st != BNN_OK) return st;
    if (last && cls != nullptr) {
      argmax_kernel<<<grid_for((int64_t)nb * 32, 256), 256, 0, s>>>(lg, nb, P.l, cls);
      if ((st = check_launch("argmax_kernel")) != BNN_OK) return st;
    }
    xbits = ybits;
  }
  return BNN_OK;
}

}  // namespace

extern "C" {

bnn_status bnn_forward(bnn_net* net, const void* images, int n, int32_t* logits, int32_t* cls, bnn_stream_t stream) {
  if (net == nullptr) return fail(BNN_E_ARG, "bnn_forward: null net");
  if (n < 0) return fail(BNN_E_ARG, "bnn_forward: n < 0");
  if (n > 0 && images == nullptr) return fail(BNN_E_ARG, "bnn_forward: null images");
  BNN_REQUIRE_ALIGNED(images, "bnn_forward images");
  BNN_REQUIRE_ALIGNED(logits, "bnn_forward logits");
  BNN_REQUIRE_ALIGNED(cls, "bnn_forward cls");
  const int L = net->L.back().l;
  if (g_opt_alg1) {
    if (!alg1_supported(net)) return fail(BNN_E_UNSUPPORTED, "bnn_forward (alg1): net not supported by the paper pipeline");
    bnn_status st = alg1_prepare(net);
    if (st != BNN_OK) return st;
    for (int s0 = 0; s0 < n; s0 += net->alg1_chunk) {
      const int nb = std::min(net->alg1_chunk, n - s0);
      const void* x = (const uint8_t*)images + (int64_t)s0 * net->img_bytes;
      st = alg1_forward_chunk(net, x, nb, logits ? logits + (int64_t)s0 * L : nullptr, cls ? cls + s0 : nullptr,
                              (cudaStream_t)stream);
      if (st != BNN_OK) return st;
    }
    return BNN_OK;
  }
  const int chunks = (n + net->chunk - 1) / net->chunk;
  cudaStream_t s = (cudaStream_t)stream;
  const int last_nb = n - (chunks - 1) * net->chunk;
  const bool fused_any = g_opt_fused_max_n > 0 && (net->chunk <= g_opt_fused_max_n || last_nb <= g_opt_fused_max_n);
  const bool two = chunks >= 2 && g_opt_streams >= 2 && !fused_any;  // (cooperative chunks stay on one stream)
  if (two) {
    bnn_status st = second_stream_prepare(net);
    if (st != BNN_OK) return st;
    cudaEventRecord(net->ev_fork, s);
    cudaStreamWaitEvent(net->s2, net->ev_fork, 0);
  }
  for (int c = 0; c < chunks; ++c) {
    const int s0 = c * net->chunk, nb = std::min(net->chunk, n - s0);
    const void* x = (const uint8_t*)images + (int64_t)s0 * net->img_bytes;
    int32_t* lg = logits ? logits + (int64_t)s0 * L : nullptr;
    int32_t* cl = cls ? cls + s0 : nullptr;
    const bnn_status st = (two && (c & 1)) ? forward_chunk_ws2(net, x, nb, lg, cl, net->s2) : forward_chunk(net, x, nb, lg, cl, s);
    if (st != BNN_OK) return st;
  }
  if (two) {
    cudaEventRecord(net->ev_join, net->s2);
    cudaStreamWaitEvent(s, net->ev_join, 0);
  }
  return BNN_OK;
}

bnn_status bnn_forward_scores(bnn_net* net, const void* images, int n, const float* scale, const float* bias,
                              int32_t* logits, float* scores, int32_t* cls, bnn_stream_t stream) {
  if (net == nullptr) return fail(BNN_E_ARG, "bnn_forward_scores: null net");
  if (n > 0 && logits == nullptr) return fail(BNN_E_ARG, "bnn_forward_scores: logits buffer required");
  const int L = net->L.back().l;
  if (L > 1024) return fail(BNN_E_UNSUPPORTED, "bnn_forward_scores: more than 1024 classes");
  if (n > 0 && (scale == nullptr || bias == nullptr)) return fail(BNN_E_ARG, "bnn_forward_scores: null scale / bias");
  if (n > 0 && scores == nullptr && cls == nullptr) return fail(BNN_E_ARG, "bnn_forward_scores: no output");
  bnn_status st = bnn_forward(net, images, n, logits, nullptr, stream);
  if (st != BNN_OK || n == 0) return st;
  return bnn_affine(logits, n, L, scale, bias, scores, cls, stream);
}

bnn_status bnn_net_staging(bnn_net* net, int max_staged, void** in, int32_t** logits, int32_t** cls) {
  if (net == nullptr) return fail(BNN_E_ARG, "bnn_net_staging: null net");
  if (max_staged < 1 || max_staged > 256 || max_staged > net->chunk)
    return fail(BNN_E_ARG, "bnn_net_staging: max_staged must be in [1, min(256, max_batch)]");
  if (net->max_staged < max_staged) {
    for (cudaGraphExec_t g : net->graphs)
      if (g) cudaGraphExecDestroy(g);
    net->graphs.clear();
    cudaFree(net->st_in);
    cudaFree(net->st_logits);
    cudaFree(net->st_cls);
    net->st_in = nullptr; net->st_logits = nullptr; net->st_cls = nullptr; net->max_staged = 0;
    cudaError_t e = cudaMalloc(&net->st_in, (size_t)(net->img_bytes * max_staged));
    if (e == cudaSuccess) e = cudaMalloc(&net->st_logits, (size_t)net->L.back().l * max_staged * 4);
    if (e == cudaSuccess) e = cudaMalloc(&net->st_cls, (size_t)max_staged * 4);
    if (e == cudaSuccess && net->cap_stream == nullptr) e = cudaStreamCreateWithFlags(&net->cap_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_net_staging: %s", cudaGetErrorString(e));
    net->max_staged = max_staged;
    net->graphs.assign(max_staged + 1, nullptr);
  }
  if (in) *in = net->st_in;
  if (logits) *logits = net->st_logits;
  if (cls) *cls = net->st_cls;
  return BNN_OK;
}

bnn_status bnn_forward_staged(bnn_net* net, int n, bnn_stream_t stream) {
  if (net == nullptr) return fail(BNN_E_ARG, "bnn_forward_staged: null net");
  if (net->max_staged == 0) return fail(BNN_E_ARG, "bnn_forward_staged: call bnn_net_staging first");
  if (n < 1 || n > net->max_staged) return fail(BNN_E_ARG, "bnn_forward_staged: n=%d not in [1, %d]", n, net->max_staged);
  cudaStream_t s = (cudaStream_t)stream;
  if (net->graphs[n] == nullptr) {
    const bool prof = net->prof;
    net->prof = false;
    cudaError_t e = cudaStreamBeginCapture(net->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { net->prof = prof; return fail(BNN_E_CUDA, "bnn_forward_staged: begin capture: %s", cudaGetErrorString(e)); }
    bnn_status st = forward_chunk(net, net->st_in, n, net->st_logits, net->st_cls, net->cap_stream);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(net->cap_stream, &graph);
    net->prof = prof;
    if (st != BNN_OK) { if (graph) cudaGraphDestroy(graph); return st; }
    if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_staged: end capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_staged: instantiate: %s", cudaGetErrorString(e));
    net->graphs[n] = exec;
  }
  cudaError_t e = cudaGraphLaunch(net->graphs[n], s);
  if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_staged: launch: %s", cudaGetErrorString(e));
  return BNN_OK;
}

const char* bnn_net_layer_kernel(const bnn_net* net, int layer, int n) {
  if (net == nullptr || layer < 0 || layer >= (int)net->L.size()) return "";
  const LayerPlan& P = net->L[layer];
  if (P.kind == 2) {
    const int nn = std::min(n, net->chunk);
    if (use_dense_tc(nn, (P.d + 31) / 32)) return "dense_tc4_kernel";
    return nn <= g_opt_gemv_max_n ? "dense_gemv_kernel" : "dense_kernel";
  }
  const char* tma_name = g_opt_first_fp4 ? "conv1_fp4_pool_kernel" : "conv_first_tma_pool_kernel";
  if (layer == 0 && use_luma_tma(net)) return tma_name;
  if (layer == 0 && fused_input(net)) {
    if (use_first_tc(P.c_in, P.k, kSrcThresh)) {
      if (P.pool != 2 || !g_opt_first_pool_tc) return "conv_first_tc_kernel";
      const bool tma = g_opt_first_tma && P.c_in == 3 && (P.k == 3 || P.k == 5) && (P.W * 3) % 16 == 0 && tma_encoder();
      return tma ? tma_name : "conv_first_tc_pool_kernel";
    }
    return use_first_lp(P.c_in, P.k) ? "conv_first_lp_kernel" : "conv_strip_kernel";
  }
  return conv_kernel_name(P.x_dt, P.c_in, P.k, P.pool);
}

int bnn_forward_launches(const bnn_net* net, int n) {
  if (!net || n <= 0) return 0;
  const int chunks = (n + net->chunk - 1) / net->chunk;
  int total = 0;
  for (int c = 0; c < chunks; ++c) total += launches_per_chunk(net, true, std::min(net->chunk, n - c * net->chunk));
  return total;
}

bnn_status bnn_forward_host(bnn_net* net, const void* h_images, int n, int32_t* h_logits, int32_t* h_cls,
                            bnn_stream_t stream) {
  if (net == nullptr) return fail(BNN_E_ARG, "bnn_forward_host: null net");
  if (n < 0) return fail(BNN_E_ARG, "bnn_forward_host: n < 0");
  if (n > 0 && h_images == nullptr) return fail(BNN_E_ARG, "bnn_forward_host: null images");
  cudaStream_t s = (cudaStream_t)stream;
  const int L = net->L.back().l;
  cudaError_t e = cudaSuccess;
  if (net->hchunk == 0) {
    const int hc = std::min(net->chunk, 4096);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaMalloc(&net->d_in[i], (size_t)(net->img_bytes * hc));
      if (e == cudaSuccess) e = cudaMalloc(&net->d_logits[i], (size_t)L * hc * 4);
      if (e == cudaSuccess) e = cudaMalloc(&net->d_cls[i], (size_t)hc * 4);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->ev_h2d[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->ev_comp[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->ev_d2h[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&net->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&net->d2h, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_host: staging allocation: %s", cudaGetErrorString(e));
    net->hchunk = hc;
  }
  const int hc = net->hchunk;
  // order the copy streams after everything already queued on the compute stream
  cudaEventRecord(net->ev_comp[0], s);
  cudaEventRecord(net->ev_comp[1], s);
  cudaEventRecord(net->ev_d2h[0], s);
  cudaEventRecord(net->ev_d2h[1], s);
  int chunk_idx = 0;
  for (int s0 = 0; s0 < n; s0 += hc, ++chunk_idx) {
    const int b = chunk_idx & 1;
    const int nb = std::min(hc, n - s0);
    cudaStreamWaitEvent(net->h2d, net->ev_comp[b], 0);
    e = cudaMemcpyAsync(net->d_in[b], (const uint8_t*)h_images + (int64_t)s0 * net->img_bytes,
                        (size_t)(nb * net->img_bytes), cudaMemcpyHostToDevice, net->h2d);
    if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_host: H2D: %s", cudaGetErrorString(e));
    cudaEventRecord(net->ev_h2d[b], net->h2d);
    cudaStreamWaitEvent(s, net->ev_h2d[b], 0);
    cudaStreamWaitEvent(s, net->ev_d2h[b], 0);
    bnn_status st = forward_chunk(net, net->d_in[b], nb, net->d_logits[b], net->d_cls[b], s);
    if (st != BNN_OK) return st;
    cudaEventRecord(net->ev_comp[b], s);
    cudaStreamWaitEvent(net->d2h, net->ev_comp[b], 0);
    if (h_logits) {
      e = cudaMemcpyAsync(h_logits + (int64_t)s0 * L, net->d_logits[b], (size_t)nb * L * 4, cudaMemcpyDeviceToHost, net->d2h);
      if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_host: D2H: %s", cudaGetErrorString(e));
    }
    if (h_cls) {
      e = cudaMemcpyAsync(h_cls + s0, net->d_cls[b], (size_t)nb * 4, cudaMemcpyDeviceToHost, net->d2h);
      if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_host: D2H: %s", cudaGetErrorString(e));
    }
    cudaEventRecord(net->ev_d2h[b], net->d2h);
  }
  e = cudaStreamSynchronize(net->d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(BNN_E_CUDA, "bnn_forward_host: %s", cudaGetErrorString(e));
  return BNN_OK;
}

int bnn_net_profile(bnn_net* net, int enable) {
  if (net == nullptr) return -(int)fail(BNN_E_ARG, "bnn_net_profile: null net");
  const int ns = (int)net->L.size() + 2;
  if (enable) {
    cudaDeviceSynchronize();
    net->ev_used = 0;
    net->pending_stage.clear();
    net->stage_ms.assign(ns, 0.0);
    net->stage_launches.assign(ns, 0);
  }
  net->prof = enable != 0;
  return ns;
}

int bnn_net_profile_read(bnn_net* net, double* ms, int64_t* launches, int cap) {
  if (net == nullptr) return -(int)fail(BNN_E_ARG, "bnn_net_profile_read: null net");
  const int ns = (int)net->L.size() + 2;
  if ((int)net->stage_ms.size() != ns) { net->stage_ms.assign(ns, 0.0); net->stage_launches.assign(ns, 0); }
  for (size_t i = 0; i < net->pending_stage.size(); ++i) {
    cudaEvent_t b = net->ev_pool[2 * i], e = net->ev_pool[2 * i + 1];
    cudaError_t err = cudaEventSynchronize(e);
    float t = 0.f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&t, b, e);
    if (err != cudaSuccess) return -(int)fail(BNN_E_CUDA, "bnn_net_profile_read: %s", cudaGetErrorString(err));
    net->stage_ms[net->pending_stage[i]] += t;
    net->stage_launches[net->pending_stage[i]] += 1;
  }
  net->pending_stage.clear();
  net->ev_used = 0;
  for (int i = 0; i < ns && i < cap; ++i) {
    if (ms) ms[i] = net->stage_ms[i];
    if (launches) launches[i] = net->stage_launches[i];
  }
  return ns;
}

void bnn_net_destroy(bnn_net* net) { net_free(net); }

}  // extern "C"
