// tma_probe2.cu -- narrows down TMA failures: 1-D bulk copy, 2-D f32 tile, launch with/without a
// cluster attribute.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait0(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D_%=;\n\tbra W_%=;\n\tD_%=:\n\t}\n" ::"r"(
          sa(bar)));
}

__global__ void k_bulk(const float* src, float* out, int n) {
  __shared__ alignas(128) float buf[1024];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                 "l"(src), "r"(n * 4), "r"(sa(&bar))
                 : "memory");
  }
  wait0(&bar);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

__global__ void k_tile(const __grid_constant__ CUtensorMap m, float* out, int n) {
  __shared__ alignas(1024) float buf[32 * 8];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(32 * 8 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                     sa(buf)),
                 "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(0), "r"(sa(&bar))
                 : "memory");
  }
  wait0(&bar);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0, cluster = argc > 2 ? atoi(argv[2]) : 0;
  std::vector<float> h(64 * 64);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 4096 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaError_t e;
  int bad = 0, n = 0;
  if (which == 0) {
    n = 1024;
    k_bulk<<<1, 128>>>(d, o, n);
    e = cudaDeviceSynchronize();
  } else {
    CUtensorMap map;
    const cuuint64_t dims[2] = {64, 64};
    const cuuint64_t strides[1] = {64 * 4};
    const cuuint32_t box[2] = {32, 8};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    n = 256;
    if (cluster) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(128);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_tile, map, o, n);
    } else {
      k_tile<<<1, 128>>>(map, o, n);
    }
    e = cudaDeviceSynchronize();
  }
  std::vector<float> got(n);
  cudaMemcpy(got.data(), o, n * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) {
    const float want = which == 0 ? h[i] : h[(i / 32) * 64 + i % 32];
    bad += got[i] != want;
  }
  printf("which %d cluster %d: %s, mismatches %d\n", which, cluster, cudaGetErrorString(e), bad);
  return 0;
}
