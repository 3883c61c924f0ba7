// Integer-pipe throughput probe for sm_100a (B200).
//
// Measures, per SM per SM-clock, the warp-lane throughput of the instructions the
// binary conv inner loop is made of (SURVEY.md §7 "hard parts" 1: the POPC rate on
// sm_100 is unverified; it is the roofline denominator of the packed conv).
//   POPC   : r = popc(r)                      (8 independent chains / thread)
//   LOP3   : r = lop3(r, a, b, 0x96)
//   IADD3  : r = r + a + b
//   XPA    : acc += popc(x ^ w)  (the real inner-loop mix: LOP3 + POPC + IADD3)
//   IDP4A  : acc = dp4a(acc, a, b)
// Each kernel reports cycles from clock64() per CTA; rate = lanes*ops / (cycles * CTAs per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_popc(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t r[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) r[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("popc.b32 %0, %0;" : "+r"(r[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lop3(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t r[CH];
  uint32_t a = seed ^ threadIdx.x, b = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) r[i] = seed * (threadIdx.x + 1) + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(a), "r"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_iadd3(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t r[CH];
  uint32_t a = seed ^ threadIdx.x, b = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) r[i] = seed * (threadIdx.x + 1) + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(r[i]) : "r"(a), "r"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The real inner-loop mix: acc_i += popc(x_i ^ w); x_i then rotated by the next word.
__global__ void k_xpa(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t x[CH], acc[CH];
  uint32_t w0 = seed ^ (threadIdx.x * 77u), w1 = seed * 3u + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) { x[i] = seed * (threadIdx.x + 1) + i; acc[i] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    uint32_t w = (it & 1) ? w1 : w0;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      uint32_t t;
      asm volatile("xor.b32 %0, %1, %2;" : "=r"(t) : "r"(x[i]), "r"(w));
      asm volatile("popc.b32 %0, %0;" : "+r"(t));
      acc[i] += t;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dp4a(uint32_t* out, long long* cyc, uint32_t seed) {
  int r[CH];
  int a = seed ^ threadIdx.x, b = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i) r[i] = seed * (threadIdx.x + 1) + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("dp4a.s32.s32 %0, %1, %2, %0;" : "+r"(r[i]) : "r"(a), "r"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(uint32_t*, long long*, uint32_t);

static void run(const char* name, kfn f, int ops_per_chain_iter, int sms) {
  const int threads = 256, per_sm = 4;
  const int blocks = sms * per_sm;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sizeof(uint32_t) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  f<<<blocks, threads>>>(out, cyc, 1u);  // warm-up
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, cyc, 12345u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mean = 0; long long mx = 0;
  for (int i = 0; i < blocks; ++i) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= blocks;
  double lane_ops_per_block = (double)threads * ITERS * CH * ops_per_chain_iter;
  // all per_sm blocks run concurrently on one SM (256 thr * 4 = 1024 thr/SM)
  double per_sm_per_clk = lane_ops_per_block * per_sm / mean;
  double total = lane_ops_per_block * blocks;
  printf("%-6s lanes/clk/SM=%7.2f  (max-cyc based %7.2f)  chip=%.3e/s  time=%.3f ms  implied_clk=%.0f MHz\n",
         name, per_sm_per_clk, lane_ops_per_block * per_sm / mx, total / (ms * 1e-3), ms,
         mx / (ms * 1e-3) / 1e6);
  delete[] h;
  cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s  SMs=%d  cc=%d.%d  clock(kHz)=%d\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    run("POPC", k_popc, 1, sms);
    run("LOP3", k_lop3, 1, sms);
    run("IADD", k_iadd3, 2, sms);
    run("XPA", k_xpa, 1, sms);  // per popc (1 xor + 1 popc + 1 add)
    run("DP4A", k_dp4a, 1, sms);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
