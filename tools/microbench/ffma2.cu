// Packed FP32 (FFMA2, PTX fma.rn.f32x2, sm_100a) throughput vs scalar FFMA.
// If FFMA2 retires 2 FMAs per lane per issue slot at the FMA-pipe rate, an
// issue-bound FP32 loop can halve its FP32 issue slots.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }

template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
  const float t = threadIdx.x * 1e-9f;
  u64 v[8], x[8];
  float s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = pk(t + i, t - i); x[i] = pk(1.0f + t + i * 1e-3f, 0.999f - t); s[i] = 0.5f + t * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = ffma2(pk(a, a), v[i], pk(b, b));          // uniform scalars
      else if (MODE == 1) v[i] = ffma2(pk(s[i], s[i]), x[i], v[i]);    // scalar reg x packed reg + packed
      else v[i] = ffma2(x[i], x[(i + 3) & 7], v[i]);                   // three packed regs
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += lo(v[i]);
  if (r == 12345.f) out[0] = r;
}

int main() {
  float* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocks = 148 * 4, iters = 1 << 14;
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(d, 0.999f, 1e-4f, 64);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, 0.999f, 1e-4f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma_lane_ops = 2.0 * 8 * iters * (double)threads * blocks;   // 2 FMAs per FFMA2 lane
    printf("{\"mode\":\"%s\",\"fp32_tflops\":%.2f,\"ffma2_warp_inst_per_clk_per_sm_at_1965MHz\":%.3f}\n",
           name, 2.0 * fma_lane_ops / ms / 1e9, fma_lane_ops / 2 / 32 / (ms * 1e-3) / 148 / 1.965e9);
  };
  run(k<0>, "ffma2_uniform");
  run(k<1>, "ffma2_scalar_reg_bcast");
  run(k<2>, "ffma2_three_packed_regs");
  return 0;
}
