// Ceiling of the packed-fp32 pair-test loop in isolation: the exact
// batch body of spin_persistent (8 centres x 2 packed point pairs per thread, centre
// constants from shared memory), with and without the predicate chain + mask OR.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float a, float b) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ f2 bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ unsigned pbit(unsigned mask, float s, float c, float abe, float h, float qn, float nqt, unsigned bit) {
  asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\tsetp.le.and.f32 p, %3, %4, p;\n\tsetp.ge.and.f32 p, %5, %6, p;\n\t@p or.b32 %0, %0, %7;\n\t}"
      : "+r"(mask) : "f"(s), "f"(c), "f"(abe), "f"(h), "f"(qn), "f"(nqt), "r"(bit));
  return mask;
}

template <int TEST, int NTH, int NP>
__global__ void __launch_bounds__(NTH, 1) k(unsigned* out, float ct, float ht, int iters) {
  __shared__ float4 sA[64], sB[64];
  if (threadIdx.x < 64) {
    sA[threadIdx.x] = make_float4(0.3f + threadIdx.x * 1e-3f, 0.4f, 0.5f, -0.1f);
    sB[threadIdx.x] = make_float4(0.2f, 0.1f, 0.3f + threadIdx.x * 1e-3f, -0.05f);
  }
  __syncthreads();
  const float t = threadIdx.x * 1e-4f;
  f2 X[NP], Y[NP], Z[NP], NXX[NP], NX[NP], NY[NP], NZ[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    X[i] = pk2(t + i, t + 1e-3f); Y[i] = pk2(0.1f + t, t * i); Z[i] = pk2(0.3f * i, t); NXX[i] = pk2(-t, -0.1f * i);
    NX[i] = pk2(0.1f, 0.2f + t * i); NY[i] = pk2(0.5f + i, t); NZ[i] = pk2(t, 0.7f - i * 0.1f);
  }
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    constexpr int CBn = 16 / NP;   // centres per 32-bit mask (2*NP points per thread)
#pragma unroll 1
    for (int cb = 0; cb < 64; cb += CBn) {
      unsigned mask = 0;
#pragma unroll
      for (int c = 0; c < CBn; ++c) {
        const float4 A4 = sA[cb + c], B4 = sB[cb + c];
#pragma unroll
        for (int k2 = 0; k2 < NP; ++k2) {
          const f2 s2 = fma2(bc2(A4.x), NX[k2], fma2(bc2(A4.y), NY[k2], mul2(bc2(A4.z), NZ[k2])));
          const f2 be2 = fma2(bc2(A4.x), X[k2], fma2(bc2(A4.y), Y[k2], fma2(bc2(A4.z), Z[k2], bc2(A4.w))));
          const f2 tn2 = fma2(bc2(B4.x), X[k2], fma2(bc2(B4.y), Y[k2], fma2(bc2(B4.z), Z[k2], NXX[k2])));
          const f2 qn2 = fma2(be2, be2, tn2);
          float s0, s1, b0, b1, q0, q1;
          up2(s2, s0, s1); up2(be2, b0, b1); up2(qn2, q0, q1);
          const int bit = c * 2 * NP + 2 * k2;
          if (TEST) {
            mask = pbit(mask, s0, ct, fabsf(b0), ht, q0, B4.w, 1u << bit);
            mask = pbit(mask, s1, ct, fabsf(b1), ht, q1, B4.w, 1u << (bit + 1));
          } else {
            mask += __float_as_uint(s0 + b0 + q0) ^ __float_as_uint(s1 + b1 + q1);
          }
        }
      }
      acc += mask;
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  unsigned* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int nth, const char* name) {
    const int iters = 2000, blocks = 148;
    kern<<<blocks, nth>>>(d, 0.5f, 0.2f, 10);
    cudaEventRecord(e0);
    kern<<<blocks, nth>>>(d, 0.5f, 0.2f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)iters * 64 * (name[11] == '2' ? 2 : name[11] == '4' ? 4 : name[11] == '8' ? 8 : 16) * nth * blocks;
    printf("{\"variant\":\"%s\",\"threads\":%d,\"pairs_per_s\":%.3e,\"fp32_frac_20flop\":%.3f}\n", name, nth,
           pairs / (ms * 1e-3), pairs * 20 / (ms * 1e-3) / 74.45e12);
  };
  run(k<1, 768, 2>, 768, "full_test_K4");
  run(k<1, 512, 4>, 512, "full_test_K8");
  run(k<1, 384, 4>, 384, "full_test_K8_384");
  run(k<1, 1024, 1>, 1024, "full_test_K2");
  run(k<1, 256, 8>, 256, "full_test_K16");
  return 0;
}
