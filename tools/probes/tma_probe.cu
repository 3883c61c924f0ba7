// tma_probe.cu -- checks a 3-D u8 TMA box load (cp.async.bulk.tensor) the way the fused first-layer
// kernel issues it: tensor map as a __grid_constant__ parameter vs in global memory, box 80 vs 64.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, uint8_t* out, int bytes, int use_global,
                  int x, int y, int z, int form) {
  __shared__ alignas(128) uint8_t buf[4096];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t mp = use_global ? reinterpret_cast<uint64_t>(gm) : reinterpret_cast<uint64_t>(&m);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    if (form == 0)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              sa(buf)),
          "l"(mp), "r"(x), "r"(y), "r"(z), "r"(sa(&bar))
          : "memory");
    else if (form == 1)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              sa(buf)),
          "l"(mp), "r"(x), "r"(y), "r"(z), "r"(sa(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(buf)),
          "l"(mp), "r"(x), "r"(y), "r"(sa(&bar))
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(
          sa(&bar)));
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int boxw_arg = argc > 1 ? atoi(argv[1]) : 80, use_global = argc > 2 ? atoi(argv[2]) : 0;
  const int form = argc > 3 ? atoi(argv[3]) : 0, direct = argc > 4 ? atoi(argv[4]) : 0;
  const int prom = argc > 5 ? atoi(argv[5]) : 1;
  const int N = 2, H = 96, W = 96, C = 3;
  std::vector<uint8_t> h((size_t)N * H * W * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7 + 3);
  uint8_t *d, *o;
  cudaMalloc(&d, h.size());
  cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = direct ? &cuTensorMapEncodeTiled : reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  printf("entry point %p (q=%d) direct %p\n", fn, (int)q, (void*)&cuTensorMapEncodeTiled);
  {
    const int boxw = boxw_arg;
    {
      CUtensorMap map;
      const bool two = form == 2;
      const cuuint64_t dims[3] = {(cuuint64_t)W * C, two ? (cuuint64_t)H * N : (cuuint64_t)H, (cuuint64_t)N};
      const cuuint64_t strides[2] = {(cuuint64_t)W * C, (cuuint64_t)H * W * C};
      const cuuint32_t box[3] = {(cuuint32_t)boxw, 36, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, two ? 2 : 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      CUtensorMap* gm;
      cudaMalloc(&gm, sizeof(CUtensorMap));
      cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
      cudaMemset(o, 0xEE, 4096);
      const int bytes = boxw * 36, x = argc > 6 ? atoi(argv[6]) : 16 * 3 - 6, y = two ? 96 - 2 : -2, z = 1;
      k<<<1, 128>>>(map, gm, o, bytes, use_global, x, y, z, form);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint8_t> got(bytes);
      cudaMemcpy(got.data(), o, bytes, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r2 = 0; r2 < 36; ++r2)
        for (int c = 0; c < boxw; ++c) {
          const int gy = (two ? y - 96 : y) + r2, gx = x + c;
          const uint8_t want = (gy < 0 || gy >= H || gx < 0 || gx >= W * C) ? (two && gy < 0 ? h[((size_t)(96 + gy)) * W * C + gx] : 0) : h[((size_t)z * H + gy) * W * C + gx];
          bad += got[r2 * boxw + c] != want;
        }
      printf("box %d global %d form %d direct %d prom %d: encode %d, launch %s, mismatches %d\n", boxw, use_global, form, direct, prom, (int)r, cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
