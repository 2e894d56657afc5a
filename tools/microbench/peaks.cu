// Microbenchmarks that fix the denominators used in DESIGN.md: FP32 FFMA issue
// peak, shared-memory atomic throughput (u32 native vs fp32 CAS loop), and the
// SM clock seen while they run.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 peaks.cu -o peaks
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void ffma_peak(float* out, float a, float b, int iters) {
  float v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = fmaf(v[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i];
  if (s == 12345.f) out[0] = s;
}

// each lane hits a distinct word (spread), no intra-warp conflicts
__global__ void atoms_u32(unsigned* out, int iters, unsigned stride) {
  __shared__ unsigned s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * stride) & 8191;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[idx], (unsigned)it);
    idx = (idx + 33) & 8191;
  }
  __syncthreads();
  if (s[threadIdx.x] == 0xdeadbeef) out[0] = 1;
}
__global__ void atoms_f32(float* out, int iters, unsigned stride) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * stride) & 8191;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[idx], 1.0f);
    idx = (idx + 33) & 8191;
  }
  __syncthreads();
  if (s[threadIdx.x] == -1.f) out[0] = 1;
}
__global__ void sts_u32(unsigned* out, int iters, unsigned stride) {
  __shared__ unsigned s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * stride) & 8191;
  for (int it = 0; it < iters; ++it) {
    s[idx] += (unsigned)it;   // plain read-modify-write (racy by design, throughput only)
    idx = (idx + 33) & 8191;
  }
  __syncthreads();
  if (s[threadIdx.x] == 0xdeadbeef) out[0] = 1;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"clock_khz_attr\":%d}\n", p.name, p.multiProcessorCount, clk_khz);
  float* d; CK(cudaMalloc(&d, 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // FFMA: 8 independent chains per thread, 1024 thr/block, 2 blocks/SM
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 16, threads = 512, blocks = sms * 4;
    ffma_peak<8><<<blocks, threads>>>(d, 0.999f, 1e-4f, 64);
    cudaEventRecord(e0);
    ffma_peak<8><<<blocks, threads>>>(d, 0.999f, 1e-4f, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"ffma_tflops\":%.2f,\"ms\":%.3f,\"implied_ghz_at_128lanes\":%.3f}\n", flops / ms / 1e9,
           ms, flops / ms / 1e6 / (sms * 128.0 * 2));
  }
  // smem atomics: lanes per SM per cycle estimate from time and clock
  for (int kind = 0; kind < 3; ++kind) {
    for (unsigned stride : {1u, 33u}) {
      int iters = 1 << 14, threads = 512, blocks = sms * 2;
      cudaEventRecord(e0);
      if (kind == 0) atoms_u32<<<blocks, threads>>>((unsigned*)d, iters, stride);
      else if (kind == 1) atoms_f32<<<blocks, threads>>>(d, iters, stride);
      else sts_u32<<<blocks, threads>>>((unsigned*)d, iters, stride);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lane_ops = (double)iters * threads * blocks;
      printf("{\"kind\":\"%s\",\"stride\":%u,\"ms\":%.3f,\"lane_ops_per_sm_per_ns\":%.3f}\n",
             kind == 0 ? "atoms_u32" : kind == 1 ? "atoms_f32_cas" : "lds_sts_rmw", stride, ms,
             lane_ops / sms / (ms * 1e6));
    }
  }
  CK(cudaGetLastError());
  return 0;
}
