// The BRUTE sphere filter as a tensor-core contraction (legacy mma.sync, tf32), in
// isolation, against the packed-fp32 loop of the kernel (hotloop2.cu V3).
//   The margin m(x, c) = B_c.x - |x|^2 + K_c is a bilinear form of the point vector
//   (x, y, z, -|x|^2) and the centre vector (Bx, By, Bz, 1) plus a per-centre constant:
//   one mma.sync.m16n8k4 (tf32 in, fp32 accumulate, C = K) gives 16 points x 8 centres.
//   Sign bytes of the four fp32 outputs per thread are gathered with PRMT as in V3.
//   V3  : packed fp32 (3 FFMA2 + FADD2 per two pairs), the kernel's loop
//   V9  : mma.sync m16n8k4 tf32 (A fragments from the staged tile, B/K in registers)
//   V10 : V9 without the sign gather (tensor pipe ceiling of this pattern)
// check(): one warp, random inputs: |m_mma - m_fp64| against the tf32 bound.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float a, float b) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ f2 bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ void up2u(f2 v, unsigned& lo, unsigned& hi) { asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v)); }
__device__ __forceinline__ unsigned gather4(unsigned mask, unsigned v0, unsigned v1, unsigned v2, unsigned v3, unsigned K) {
  unsigned a, b, c, d;
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(a) : "r"(v0), "r"(v1));
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(b) : "r"(v2), "r"(v3));
  asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(c) : "r"(a), "r"(b));
  asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(d) : "r"(c), "r"(K), "r"(mask));
  return d;
}
__device__ __forceinline__ unsigned tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma4(float& d0, float& d1, float& d2, float& d3, unsigned a0, unsigned a1,
                                     unsigned b0, float c0, float c1) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
               : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3)
               : "r"(a0), "r"(a1), "r"(b0), "f"(c0), "f"(c1), "f"(c0), "f"(c1));
}

// staged tile per warp: 128 points as float4 {x, y, z, -|x|^2}, point t at sP[t]
template <int V, int NTH, int UNR = 1>
__global__ void __launch_bounds__(NTH, 1) k(unsigned* out, int iters) {
  __shared__ float4 sP[2 * 128];   // two tiles shared by the warps (same bank pattern)
  __shared__ float4 sB[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * 128; i += NTH) {
    const float x = 0.3f + i * 1e-4f, y = 0.1f - i * 2e-5f, z = -0.2f + i * 1e-6f;
    sP[i] = make_float4(x, y, z, -(x * x + y * y + z * z));
  }
  if (threadIdx.x < 64) sB[threadIdx.x] = make_float4(0.2f, 0.1f, 0.3f + threadIdx.x * 1e-3f, -0.05f);
  __syncthreads();
  const float4* tile = sP + (warp & 1) * 128;
  unsigned acc = 0;
  if (V == 3) {
    for (int it = 0; it < iters; ++it) {
      f2 X[2], Y[2], Z[2], W[2];
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const float4 p0 = tile[(2 * pr) * 32 + lane], p1 = tile[(2 * pr + 1) * 32 + lane];
        X[pr] = pk2(p0.x, p1.x); Y[pr] = pk2(p0.y, p1.y); Z[pr] = pk2(p0.z, p1.z); W[pr] = pk2(p0.w, p1.w);
      }
#pragma unroll UNR
      for (int cb = 0; cb < 64; cb += 8) {
        unsigned rej = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 B4 = sB[cb + c];
          unsigned v[4];
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            const f2 m2 = add2(fma2(bc2(B4.x), X[k2], fma2(bc2(B4.y), Y[k2], fma2(bc2(B4.z), Z[k2], bc2(B4.w)))), W[k2]);
            up2u(m2, v[2 * k2], v[2 * k2 + 1]);
          }
          rej = gather4(rej, v[0], v[1], v[2], v[3], 0x01010101u << c);
        }
        acc += rej;
      }
    }
  } else {
    const int gid = lane >> 2, tig = lane & 3;
    // centre fragments for the group, held for every tile: b = component tig of centre
    // cb*8 + gid, K of centres cb*8 + 2 tig (+1)
    unsigned bf[8];
    float k0[8], k1[8];
#pragma unroll
    for (int cb = 0; cb < 8; ++cb) {
      const float* bc = reinterpret_cast<const float*>(&sB[cb * 8 + gid]);
      bf[cb] = tig == 3 ? __float_as_uint(1.0f) : tf32(bc[tig]);
      k0[cb] = sB[cb * 8 + 2 * tig].w;
      k1[cb] = sB[cb * 8 + 2 * tig + 1].w;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll UNR
      for (int rb = 0; rb < 8; ++rb) {
        const float* pa = reinterpret_cast<const float*>(tile + rb * 16 + gid);
        const unsigned a0 = tf32(pa[tig]), a1 = tf32(pa[8 * 4 + tig]);
        unsigned word = 0;
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) {
          float d0, d1, d2, d3;
          mma4(d0, d1, d2, d3, a0, a1, bf[cb], k0[cb], k1[cb]);
          if (V == 9) word = gather4(word, __float_as_uint(d0), __float_as_uint(d1), __float_as_uint(d2),
                                     __float_as_uint(d3), 0x01010101u << cb);
          else word += __float_as_uint(d0) ^ __float_as_uint(d3);
        }
        acc += word;
      }
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

// throughput of other legacy mma shapes (operands are dummies; 128 outputs per instruction)
//   S=0 m16n8k8 tf32 -> f32, S=1 m16n8k8 f16 -> f32, S=2 m16n8k16 f16 -> f32,
//   S=3 m16n8k8 f16 -> f16, S=4 m16n8k16 bf16 -> f32
template <int S, int NTH>
__global__ void __launch_bounds__(NTH, 1) kshape(unsigned* out, int iters) {
  const int lane = threadIdx.x & 31;
  unsigned a[4] = {0x3c003c00u + lane, 0x3c003c01u, 0x3c003c02u, 0x3c003c03u};
  unsigned b[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) { b[c][0] = 0x3c00u * c + lane; b[c][1] = 0x3c01u + c; }
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) {
      a[0] += rb;
      unsigned word = 0;
#pragma unroll
      for (int cb = 0; cb < 8; ++cb) {
        float d0, d1, d2, d3;
        const float c0 = 0.5f, c1 = 0.25f;
        if (S == 0) {
          asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%10,%11};"
                       : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[cb][0]), "r"(b[cb][1]), "f"(c0), "f"(c1));
        } else if (S == 1) {
          asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%7,%8};"
                       : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3) : "r"(a[0]), "r"(a[1]), "r"(b[cb][0]), "f"(c0), "f"(c1));
        } else if (S == 2) {
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%10,%11};"
                       : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[cb][0]), "r"(b[cb][1]), "f"(c0), "f"(c1));
        } else if (S == 3) {
          unsigned h0, h1;
          asm volatile("mma.sync.aligned.m16n8k8.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3}, {%4}, {%5,%6};"
                       : "=r"(h0), "=r"(h1) : "r"(a[0]), "r"(a[1]), "r"(b[cb][0]), "r"(0x3c003c00u), "r"(0x3c003c00u));
          d0 = __uint_as_float(h0); d1 = __uint_as_float(h1); d2 = d0; d3 = d1;
        } else {
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%10,%11};"
                       : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[cb][0]), "r"(b[cb][1]), "f"(c0), "f"(c1));
        }
        word = gather4(word, __float_as_uint(d0), __float_as_uint(d1), __float_as_uint(d2), __float_as_uint(d3), 0x01010101u << cb);
      }
      acc += word;
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

// one warp: 16 points x 8 centres through the mma, against fp64
__global__ void check(const float4* pts, const float4* cen, double* err, float* mm) {
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  const float* pa = reinterpret_cast<const float*>(pts + gid);
  const unsigned a0 = tf32(pa[tig]), a1 = tf32(pa[8 * 4 + tig]);
  const float* bc = reinterpret_cast<const float*>(cen + gid);
  const unsigned b = tig == 3 ? __float_as_uint(1.0f) : tf32(bc[tig]);
  float d[4];
  mma4(d[0], d[1], d[2], d[3], a0, a1, b, cen[2 * tig].w, cen[2 * tig + 1].w);
  for (int j = 0; j < 4; ++j) {
    const int p = gid + 8 * (j >> 1), c = 2 * tig + (j & 1);
    const float4 P = pts[p], C = cen[c];
    const double ex = (double)C.x * P.x + (double)C.y * P.y + (double)C.z * P.z + (double)P.w + (double)C.w;
    err[p * 8 + c] = (double)d[j] - ex;
    mm[p * 8 + c] = d[j];
  }
}

int main() {
  unsigned* d; cudaMalloc(&d, 64);
  // ---- layout / precision check
  {
    float4 hp[16], hc[8];
    unsigned s = 12345u;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) * (1.0f / 16777216.0f) * 2.f - 1.f; };
    for (int i = 0; i < 16; ++i) { float x = rnd() * 1.4f, y = rnd() * 1.4f, z = rnd() * 1.4f; hp[i] = make_float4(x, y, z, -(x * x + y * y + z * z)); }
    for (int i = 0; i < 8; ++i) hc[i] = make_float4(rnd() * 2.7f, rnd() * 2.7f, rnd() * 2.7f, rnd());
    float4 *dp, *dc; double* de; float* dm;
    cudaMalloc(&dp, sizeof hp); cudaMalloc(&dc, sizeof hc); cudaMalloc(&de, 128 * 8); cudaMalloc(&dm, 128 * 4);
    cudaMemcpy(dp, hp, sizeof hp, cudaMemcpyHostToDevice); cudaMemcpy(dc, hc, sizeof hc, cudaMemcpyHostToDevice);
    check<<<1, 32>>>(dp, dc, de, dm);
    double he[128]; cudaMemcpy(he, de, sizeof he, cudaMemcpyDeviceToHost);
    double mx = 0, mxrel = 0;
    for (int p = 0; p < 16; ++p)
      for (int c = 0; c < 8; ++c) {
        const double scale = fabs(hc[c].x * hp[p].x) + fabs(hc[c].y * hp[p].y) + fabs(hc[c].z * hp[p].z) + fabs(hp[p].w);
        mx = fmax(mx, fabs(he[p * 8 + c]));
        mxrel = fmax(mxrel, fabs(he[p * 8 + c]) / scale);
      }
    printf("{\"check\":\"mma m16n8k4 tf32 vs fp64\",\"max_abs_err\":%.3e,\"max_err_over_sum_abs_terms\":%.3e,\"tf32_unit\":%.3e,\"err\":\"%s\"}\n",
           mx, mxrel, ldexp(1.0, -11), cudaGetErrorString(cudaGetLastError()));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int nth, const char* name) {
    const int iters = 4000, blocks = 148;
    kern<<<blocks, nth>>>(d, 10);
    cudaEventRecord(e0);
    kern<<<blocks, nth>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)iters * 64 * 128 * (nth / 32) * blocks;
    printf("{\"variant\":\"%s\",\"threads\":%d,\"pairs_per_s\":%.3e,\"fp32_frac_20flop\":%.3f,\"err\":\"%s\"}\n", name, nth,
           pairs / (ms * 1e-3), pairs * 20 / (ms * 1e-3) / 74.45e12, cudaGetErrorString(cudaGetLastError()));
  };
  for (int r = 0; r < 2; ++r) {
    run(k<3, 768, 2>, 768, "V3_sphonly_ffma2_unroll2");
    run(k<9, 768, 1>, 768, "V9_mma_tf32");
    run(k<9, 768, 2>, 768, "V9_mma_tf32_unroll2");
    run(k<9, 512, 2>, 512, "V9_mma_tf32_512");
    run(k<9, 1024, 2>, 1024, "V9_mma_tf32_1024");
    run(k<10, 768, 2>, 768, "V10_mma_only");
    run(kshape<0, 768>, 768, "S0_m16n8k8_tf32_f32");
    run(kshape<1, 768>, 768, "S1_m16n8k8_f16_f32");
    run(kshape<2, 768>, 768, "S2_m16n8k16_f16_f32");
    run(kshape<3, 768>, 768, "S3_m16n8k8_f16_f16acc");
    run(kshape<4, 768>, 768, "S4_m16n8k16_bf16_f32");
  }
  return 0;
}
