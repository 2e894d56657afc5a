// spin_kernels.cu — launch dispatch of the persistent spin kernel (spin_persistent.cuh)
// and the HBM-bound helper kernels: cloud re-layout/validation (a1), exclusive scan,
// CELLS grid build (a4) and centre ordering (a5).
#include "spin_persistent.cuh"
#include <cub/device/device_radix_sort.cuh>

namespace spin {

// ------------------------------------------------------------------ dispatch
// kernel_ptr_M_S_D: MODE M, support placement S, dealer D (0 chunk table, 1 WF / AWF
// compare-and-swap; a separate instantiation, so the table dealer's code is unchanged)
#define SPIN_DECL(m, s, d) const void* kernel_ptr_##m##_##s##_##d(int prune, int G, int nt, int cl);
SPIN_DECL(0, 0, 0) SPIN_DECL(0, 1, 0) SPIN_DECL(0, 2, 0) SPIN_DECL(1, 0, 0) SPIN_DECL(1, 1, 0) SPIN_DECL(1, 2, 0)
SPIN_DECL(0, 0, 1) SPIN_DECL(0, 1, 1) SPIN_DECL(0, 2, 1) SPIN_DECL(1, 0, 1) SPIN_DECL(1, 1, 1) SPIN_DECL(1, 2, 1)
#undef SPIN_DECL
static const void* kernel_for(int mode, int prune, int G, int sup, int nt, int deal, int cl) {
  if (prune == 1 && sup == 2) sup = 1;   // adaptive placement is BRUTE-only
  typedef const void* (*Fn)(int, int, int, int);
  static const Fn tab[2][2][3] = {
      {{kernel_ptr_0_0_0, kernel_ptr_0_1_0, kernel_ptr_0_2_0}, {kernel_ptr_1_0_0, kernel_ptr_1_1_0, kernel_ptr_1_2_0}},
      {{kernel_ptr_0_0_1, kernel_ptr_0_1_1, kernel_ptr_0_2_1}, {kernel_ptr_1_0_1, kernel_ptr_1_1_1, kernel_ptr_1_2_1}}};
  return tab[deal ? 1 : 0][mode ? 1 : 0][sup](prune, G, nt, cl);
}

LaunchCfg choose_launch(int W, int mode, int prune, bool allow_cluster) {
  // One CTA per SM.  Images live in shared memory (NEAREST 4 B/bin, BILINEAR 6 B/bin);
  // CELLS take the largest G <= 32 whose 768-thread layout fits; BRUTE the first entry
  // of the measured preference list below that fits.
  constexpr int LIMIT = 220 * 1024;
  LaunchCfg lc;
  lc.threads = NT_DEFAULT;
  lc.cl = 1;
#ifdef SPIN_MEASURE
  const char* dg = std::getenv("SPIN_DEBUG_G");   // measurement builds only (unvalidated)
  const char* dn = std::getenv("SPIN_DEBUG_NT");
#else
  const char* dg = nullptr;
  const char* dn = nullptr;
#endif
  if (dg) {
    lc.G = std::atoi(dg);
    if (dn) lc.threads = std::atoi(dn);
  } else if (prune == 1) {
    // CELLS: larger groups grow the visited box (measured: 32 best)
    int G = 32;
    while (G > 4 && make_layout(G, W, mode, prune, NT_DEFAULT).total > LIMIT) G >>= 1;
    lc.G = G;
  } else {
    // BRUTE, in order of preference (measured on C2 / C4): 768 threads with G = 64 or
    // 32; 512 threads with G = 32 where 32 images no longer fit beside 24 staged warp tiles
    // (W = 28 .. 32: with the dense lane-per-centre tiles one lane per centre fills the warp;
    // C4 BILINEAR 372 ms with 768 threads / G = 24 -> 306 ms, NEAREST 332 ms on two-CTA
    // clusters -> 279 ms); then 768 threads with smaller G.  Two-CTA clusters
    // sharing G = 48 (24 images per CTA, DSMEM adds; the cluster layout may use the whole
    // 227 KB opt-in) only on request (SPIN_F_CLUSTER_PAIR, BRUTE NEAREST).
    static const int pref[][3] = {{768, 48, 2}, {768, 64, 1}, {768, 32, 1}, {512, 32, 1},
                                  {768, 24, 1}, {768, 16, 1}, {768, 8, 1}, {768, 4, 1}};
    for (const auto& c : pref) {
      if (c[2] > 1 && !allow_cluster) continue;
      lc.threads = c[0];
      lc.G = c[1];
      lc.cl = c[2];
      const size_t lim = c[2] > 1 ? 227 * 1024 - 1024 : LIMIT;   // (static smem < 1 KB)
      if (make_layout(lc.G, W, mode, prune, lc.threads, lc.cl).total <= lim) break;
    }
  }
  lc.smem = make_layout(lc.G, W, mode, prune, lc.threads, lc.cl).total;
  return lc;
}

// cloud padding: a multiple of every CTA tile (768 x 4 and 512 x 4 points)
int tile_points() { return 6144; }

// resident workers of a persistent launch: CTAs (cl = 1) or two-CTA clusters (cl = 2)
int resident_workers(const LaunchCfg& lc, int W, int mode, int prune, int sms) {
  const void* f = kernel_for(mode, prune, lc.G, 1, lc.threads, 0, lc.cl);
  if (!f) return 0;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
  (void)W;
  if (lc.cl == 1) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, lc.threads, lc.smem) != cudaSuccess)
      return 0;
    return nb * sms;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)lc.cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(lc.cl * sms));
  cfg.blockDim = dim3((unsigned)lc.threads);
  cfg.dynamicSmemBytes = lc.smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, f, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nc;
}

cudaError_t launch_spin(const LaunchCfg& lc, int mode, int prune, int grid, const KParams& p,
                        cudaStream_t s) {
  const void* f = kernel_for(mode, prune, lc.G, p.support_in_hot, lc.threads, p.wf ? 1 : 0, lc.cl);
  if (!f) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&p};
  if (lc.cl == 1) return cudaLaunchKernel(f, dim3(grid), dim3(lc.threads), args, lc.smem, s);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)lc.cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)lc.threads);
  cfg.dynamicSmemBytes = lc.smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, f, args);
}

// ------------------------------------------------------------------ a1: relayout + validation
__device__ __forceinline__ int float_flip(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

__global__ void k_relayout(const float* __restrict__ pts, const float* __restrict__ nrm, int64_t N,
                           int64_t Npad, float4* __restrict__ pos, float4* __restrict__ nrm4,
                           int32_t* bad, int* absmax_bits, int* aabb_bits) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Npad) return;
  if (j >= N) {
    // sentinel: |x|^2 = 2^100 (finite, so the tf32 hi/lo split of the tensor-core filter
    // stays NaN-free) makes every margin hugely negative: it never passes
    pos[j] = make_float4(0.f, 0.f, 0.f, SENTINEL_R2);
    nrm4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float x = pts[3 * j], y = pts[3 * j + 1], z = pts[3 * j + 2];
  const float a = nrm[3 * j], b = nrm[3 * j + 1], c = nrm[3 * j + 2];
  const double n2 = (double)a * a + (double)b * b + (double)c * c;
  // |coordinate| <= 2^40 keeps |x|^2 and every filter product far from fp32 overflow
  const bool ok = fabsf(x) <= COORD_MAX && fabsf(y) <= COORD_MAX && fabsf(z) <= COORD_MAX &&
                  isfinite(a) && isfinite(b) &&
                  isfinite(c) && n2 >= 0.999 * 0.999 && n2 <= 1.001 * 1.001;
  if (!ok) atomicMin(bad, (int32_t)min(j, (int64_t)0x7fffffff));
  const double xx = (double)x * x + (double)y * y + (double)z * z;
  pos[j] = make_float4(x, y, z, __double2float_rn(xx));
  nrm4[j] = make_float4(a, b, c, 0.f);
  const float r = __double2float_ru(sqrt(xx));
  atomicMax(absmax_bits, __float_as_int(ok ? r : 0.f));
  if (ok) {
    atomicMin(&aabb_bits[0], float_flip(x));
    atomicMin(&aabb_bits[1], float_flip(y));
    atomicMin(&aabb_bits[2], float_flip(z));
    atomicMax(&aabb_bits[3], float_flip(x));
    atomicMax(&aabb_bits[4], float_flip(y));
    atomicMax(&aabb_bits[5], float_flip(z));
  }
}

// BRUTE tiles in the shared-memory staging layout, so a warp's 128 points are ONE 4 KB
// bulk copy: chunk c holds points 128c .. 128c+127; point 128c + 32k + l (lane l, point
// k of that lane) sits in records r = 0..3 of pair k/2, half k&1:
//   r0 {x, x', y, y'}  r1 {z, z', -|x|^2, -|x'|^2}  r2 {nx, nx', ny, ny'}  r3 {nz, nz', 0, 0}
__global__ void k_pair_layout(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                              int64_t Npad, float* __restrict__ tpos) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Npad) return;
  const int64_t c = j >> 7;
  const int within = (int)(j & 127), k = within >> 5, l = within & 31, pr = k >> 1, hf = k & 1;
  const float4 a = pos[j], n = nrm[j];
  float* base = tpos + c * 1024;    // 256 float4 per chunk
  auto rec = [&](int r) { return base + ((r * 2 + pr) * 32 + l) * 4; };
  rec(0)[hf] = a.x;
  rec(0)[2 + hf] = a.y;
  rec(1)[hf] = a.z;
  rec(1)[2 + hf] = -a.w;
  rec(2)[hf] = n.x;
  rec(2)[2 + hf] = n.y;
  rec(3)[hf] = n.z;
  rec(3)[2 + hf] = 0.f;
}
cudaError_t launch_pair_layout(const float4* pos, const float4* nrm, int64_t Npad, float4* tpos,
                               cudaStream_t s) {
  k_pair_layout<<<(unsigned)((Npad + 255) / 256), 256, 0, s>>>(pos, nrm, Npad, (float*)tpos);
  return cudaGetLastError();
}

// The mma.sync A fragments (BRUTE tensor-core filter, spin_persistent FRAG): per 128-point
// chunk c, row block rb and lane L = (gid, tig) of the m16n8k8 tf32 fragment, the uint4
// (hi(v0), hi(v1), lo(v0), lo(v1)) with v0, v1 = component tig (x, y, z, -|x|^2) of the
// chunk's points 32 k0 + sl and 32 (k0 + 1) + sl, k0 = 2 (rb >> 2), sl = (rb & 3) * 8 +
// ((gid + rb) & 7) -- the rows gid and gid + 8 of row block rb in the staged pair layout;
// hi = round to nearest tf32, lo = (v - hi) truncated to tf32 (1.0 in the w column: the
// constant-1 column that carries K).  The split the kernel used to do per tile and group.
__global__ void k_mma_frags(const float4* __restrict__ pos, int64_t n, uint4* __restrict__ frag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;   // n = chunks * 256
  const int64_t c = i >> 8;
  const int rb = (int)(i >> 5) & 7, L = (int)(i & 31), gid = L >> 2, tig = L & 3;
  const int sl = (rb & 3) * 8 + ((gid + rb) & 7), k0 = 2 * (rb >> 2);
  auto comp = [&](int64_t j) {
    const float4 a = pos[j];
    return tig == 0 ? a.x : tig == 1 ? a.y : tig == 2 ? a.z : -a.w;
  };
  const float v0 = comp(c * 128 + 32 * k0 + sl), v1 = comp(c * 128 + 32 * (k0 + 1) + sl);
  auto hi = [](float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; };
  const unsigned h0 = hi(v0), h1 = hi(v1);
  const unsigned l0 = tig == 3 ? 0x3f800000u : __float_as_uint(v0 - __uint_as_float(h0)) & 0xffffe000u;
  const unsigned l1 = tig == 3 ? 0x3f800000u : __float_as_uint(v1 - __uint_as_float(h1)) & 0xffffe000u;
  frag[i] = make_uint4(h0, h1, l0, l1);
}
cudaError_t launch_mma_frags(const float4* pos, int64_t Npad, float4* mfrag, cudaStream_t s) {
  const int64_t n = (Npad / 128) * 256;
  k_mma_frags<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pos, n, reinterpret_cast<uint4*>(mfrag));
  return cudaGetLastError();
}

// The tcgen05 A operand (BRUTE, spin_persistent TC): per 128-point chunk c, 4 KB with row
// r = point 128 c + r as (x_hi, y_hi, z_hi, w_hi | x_lo, y_lo, z_lo, 1), w = -|x|^2, hi =
// x rounded to tf32, lo = x - hi truncated to tf32 (the mma.sync filter's operands, split
// once at load time instead of per group); canonical no-swizzle K-major layout: the 16-byte
// half kc of row r at (r & 7) * 16 + (r >> 3) * 256 + kc * 128
__global__ void k_tf32_operand(const float4* __restrict__ pos, int64_t Npad, float* __restrict__ tfa) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Npad) return;
  const float4 a = pos[j];
  const float v[3] = {a.x, a.y, a.z};
  float* row = tfa + (j >> 7) * 1024 + ((int)(j & 7) * 16 + (int)((j & 127) >> 3) * 256) / 4;
  auto hi = [](float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u); };
  for (int c = 0; c < 3; ++c) {
    const float h = hi(v[c]);
    row[c] = h;
    row[32 + c] = __uint_as_float(__float_as_uint(v[c] - h) & 0xffffe000u);
  }
  row[3] = hi(-a.w);
  row[35] = 1.0f;
}
cudaError_t launch_tf32_operand(const float4* pos, int64_t Npad, float4* tfa, cudaStream_t s) {
  k_tf32_operand<<<(unsigned)((Npad + 255) / 256), 256, 0, s>>>(pos, Npad, (float*)tfa);
  return cudaGetLastError();
}

cudaError_t launch_relayout(const float* pts, const float* nrm, int64_t N, int64_t Npad,
                            float4* pos, float4* nrm4, int32_t* bad, float* absmax, float* aabb,
                            cudaStream_t s) {
  const int tb = 256;
  const int64_t nb = (Npad + tb - 1) / tb;
  k_relayout<<<(unsigned)nb, tb, 0, s>>>(pts, nrm, N, Npad, pos, nrm4, bad, (int*)absmax,
                                         (int*)aabb);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ exclusive scan (3 phases)
constexpr int SCAN_TB = 1024, SCAN_IPT = 4, SCAN_TILE = SCAN_TB * SCAN_IPT;

__device__ int block_excl_scan(int v, int* s_w, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += n;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += n;
    }
    s_w[lane] = w;
  }
  __syncthreads();
  total = s_w[(blockDim.x >> 5) - 1];
  const int r = x - v + (warp > 0 ? s_w[warp - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void k_scan_tiles(const int32_t* in, int32_t* out, int64_t n, int32_t* tile_sums) {
  __shared__ int s_w[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  int v[SCAN_IPT], sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    sum += v[i];
  }
  int total;
  int run = block_excl_scan(sum, s_w, total);
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}
__global__ void k_scan_sums(int32_t* sums, int nt, int32_t* out_total) {
  __shared__ int s_w[32];
  int carry = 0;
  for (int b0 = 0; b0 < nt; b0 += SCAN_TB) {
    const int i = b0 + threadIdx.x;
    const int v = i < nt ? sums[i] : 0;
    int total;
    const int r = block_excl_scan(v, s_w, total);
    if (i < nt) sums[i] = r + carry;
    carry += total;
  }
  if (threadIdx.x == 0) *out_total = carry;
}
__global__ void k_scan_add(int32_t* out, int64_t n, const int32_t* sums) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  const int add = sums[blockIdx.x];
  for (int i = threadIdx.x; i < SCAN_TILE; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

size_t scan_tmp_elems(int64_t n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }

// out[0..n] = exclusive scan of in[0..n), out[n] = total
cudaError_t launch_exclusive_scan(const int32_t* in, int32_t* out, int64_t n, int32_t* tmp,
                                  cudaStream_t s) {
  const int nt = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  if (nt == 0) return cudaMemsetAsync(out, 0, sizeof(int32_t), s);
  k_scan_tiles<<<nt, SCAN_TB, 0, s>>>(in, out, n, tmp);
  k_scan_sums<<<1, SCAN_TB, 0, s>>>(tmp, nt, out + n);
  k_scan_add<<<nt, SCAN_TB, 0, s>>>(out, n, tmp);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a4: CELLS grid build
__global__ void k_cell_keys(const float4* __restrict__ pos, int32_t N, float ox, float oy, float oz,
                            float inv_h, int dx, int dy, int dz, int32_t* keys, int32_t* counts) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const float4 a = pos[j];
  const int cx = cell_coord(a.x, ox, inv_h, dx);
  const int cy = cell_coord(a.y, oy, inv_h, dy);
  const int cz = cell_coord(a.z, oz, inv_h, dz);
  const int key = (cz * dy + cy) * dx + cx;
  keys[j] = key;
  atomicAdd(&counts[key], 1);
}
__global__ void k_cell_scatter(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                               int32_t N, int32_t Npad, const int32_t* keys,
                               const int32_t* cell_start, int32_t* cursor, float4* spos,
                               float4* snrm) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Npad) return;
  if (j >= N) {
    spos[j] = make_float4(0.f, 0.f, 0.f, SENTINEL_R2);
    snrm[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int key = keys[j];
  const int dst = cell_start[key] + atomicAdd(&cursor[key], 1);
  spos[dst] = pos[j];
  snrm[dst] = nrm[j];
}

cudaError_t launch_cell_build(const float4* pos, const float4* nrm, int32_t N, int32_t Npad,
                              float ox, float oy, float oz, float inv_h, int dx, int dy, int dz,
                              int32_t* keys, int32_t* counts, int32_t* cell_start, int32_t* cursor,
                              int32_t* scan_tmp, float4* spos, float4* snrm, cudaStream_t s) {
  const int64_t ncells = (int64_t)dx * dy * dz;
  cudaError_t e;
  if ((e = cudaMemsetAsync(counts, 0, ncells * sizeof(int32_t), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cursor, 0, ncells * sizeof(int32_t), s)) != cudaSuccess) return e;
  const int tb = 256;
  k_cell_keys<<<(N + tb - 1) / tb, tb, 0, s>>>(pos, N, ox, oy, oz, inv_h, dx, dy, dz, keys, counts);
  if ((e = launch_exclusive_scan(counts, cell_start, ncells, scan_tmp, s)) != cudaSuccess) return e;
  k_cell_scatter<<<(Npad + tb - 1) / tb, tb, 0, s>>>(pos, nrm, N, Npad, keys, cell_start, cursor,
                                                     spos, snrm);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a5: centre ordering
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__global__ void k_centre_keys(const int32_t* centre_idx, int64_t M, const float4* cpos, int32_t N,
                              float ox, float oy, float oz, float inv_h, int dx, int dy, int dz,
                              int shift, int32_t* keys, int32_t* counts) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int c = centre_idx[m];
  int key = 0;
  if (c >= 0 && c < N) {
    const float4 a = cpos[c];
    const uint32_t cx = (uint32_t)cell_coord(a.x, ox, inv_h, dx) >> shift;
    const uint32_t cy = (uint32_t)cell_coord(a.y, oy, inv_h, dy) >> shift;
    const uint32_t cz = (uint32_t)cell_coord(a.z, oz, inv_h, dz) >> shift;
    key = (int)(spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2));
  }
  keys[m] = key;
  atomicAdd(&counts[key], 1);
}
__global__ void k_centre_scatter(int64_t M, const int32_t* keys, const int32_t* starts,
                                 int32_t* cursor, int32_t* order) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int key = keys[m];
  order[starts[key] + atomicAdd(&cursor[key], 1)] = (int32_t)m;
}

cudaError_t launch_centre_order(const int32_t* centre_idx, int64_t M, const float4* cpos, int32_t N,
                                float ox, float oy, float oz, float inv_h, int dx, int dy, int dz,
                                int shift, int bits, int32_t* keys, int32_t* counts,
                                int32_t* starts, int32_t* cursor, int32_t* scan_tmp,
                                int32_t* order, cudaStream_t s) {
  const int64_t nb = (int64_t)1 << (3 * bits);
  cudaError_t e;
  if ((e = cudaMemsetAsync(counts, 0, nb * sizeof(int32_t), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cursor, 0, nb * sizeof(int32_t), s)) != cudaSuccess) return e;
  const int tb = 256;
  const unsigned g = (unsigned)((M + tb - 1) / tb);
  k_centre_keys<<<g, tb, 0, s>>>(centre_idx, M, cpos, N, ox, oy, oz, inv_h, dx, dy, dz, shift,
                                 keys, counts);
  if ((e = launch_exclusive_scan(counts, starts, nb, scan_tmp, s)) != cudaSuccess) return e;
  k_centre_scatter<<<g, tb, 0, s>>>(M, keys, starts, cursor, order);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a1/a5 BRUTE: Morton order
// BRUTE streams the cloud in a spatially sorted copy (Morton order of a 2^10-per-axis grid
// over the cubic hull of the AABB) and takes its centres in the same order, so that the
// candidates of a group of G neighbouring centres concentrate in few warp tiles (DESIGN.md
// 7.1 "dense tiles").  The images are a permutation-invariant function of the cloud (integer
// counts / fixed-point sums), so this is a layout choice only.  The sort is CUB's stable
// radix sort on (key, index): deterministic, so every device of a shared dealer derives the
// same chunk -> image map.
__device__ __forceinline__ uint32_t morton_key(float4 a, MortonGrid mg) {
  auto q = [&](float x, float o) {
    const float t = fminf(fmaxf(__fmul_rn(__fsub_rn(x, o), mg.inv), 0.0f), 1023.0f);
    return (uint32_t)t;
  };
  return spread3(q(a.x, mg.ox)) | (spread3(q(a.y, mg.oy)) << 1) | (spread3(q(a.z, mg.oz)) << 2);
}
__global__ void k_morton_keys(const int32_t* __restrict__ idx, int64_t n, const float4* __restrict__ pos,
                              int32_t N, MortonGrid mg, uint32_t* keys, int32_t* vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = idx ? idx[i] : (int)i;
  keys[i] = (c >= 0 && c < N) ? morton_key(pos[c], mg) : 0u;
  vals[i] = (int32_t)i;
}
__global__ void k_gather_cloud(const int32_t* __restrict__ perm, int32_t N, int64_t Npad,
                               const float4* __restrict__ pos, const float4* __restrict__ nrm,
                               float4* bpos, float4* bnrm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Npad) return;
  const int64_t j = i < N ? perm[i] : i;   // the sentinel padding stays at the end
  bpos[i] = pos[j];
  bnrm[i] = nrm[j];
}

size_t morton_sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0, 30);
  return bytes;
}

// order[0..n) = the positions 0..n-1 sorted by the Morton key of pos[idx[i]] (idx null:
// of pos[i]); scratch: k0, k1 (keys), v0 (values) of n elements, temp of
// morton_sort_temp_bytes(n)
cudaError_t launch_morton_order(const int32_t* idx, int64_t n, const float4* pos, int32_t N,
                                MortonGrid mg, uint32_t* k0, uint32_t* k1, int32_t* v0,
                                int32_t* order, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int tb = 256;
  k_morton_keys<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(idx, n, pos, N, mg, k0, v0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k0, k1, v0, order, (int)n, 0, 30, s);
}

cudaError_t launch_gather_cloud(const int32_t* perm, int32_t N, int64_t Npad, const float4* pos,
                                const float4* nrm, float4* bpos, float4* bnrm, cudaStream_t s) {
  const int tb = 256;
  k_gather_cloud<<<(unsigned)((Npad + tb - 1) / tb), tb, 0, s>>>(perm, N, Npad, pos, nrm, bpos, bnrm);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ diagnostic: per-pair decisions
// The accept path's own decision (decide -> resolve, the device functions the persistent
// kernel runs on every candidate) for EVERY (centre, point) pair of a few centres, so the
// tests can compare each pair's bin with the oracle's: NEAREST bins must be identical,
// BILINEAR region decisions identical and (i0, j0) may differ only at interior bin edges
// ("flips", counted).  codes[m][j] = -1 (no contribution) or k*W + l / i0*W + j0.
template <int MODE>
__global__ void k_pair_codes(const __grid_constant__ KParams p, const int32_t* __restrict__ centre_idx,
                             int32_t* __restrict__ codes) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p.N) return;
  const int64_t m = blockIdx.y;
  const int c = centre_idx[m];
  int32_t code = -1;
  if (c >= 0 && c < p.N) {
    const float4 P4 = p.cpos[c];
    float4 N4 = p.cnrm[c];
    N4.w = (float)((double)N4.x * N4.x + (double)N4.y * N4.y + (double)N4.z * N4.z - 1.0);
    const float4 A = p.pos[j], B = p.nrm[j];
    const float4 X4 = make_float4(A.x, A.y, A.z, 0.f), NX4 = make_float4(B.x, B.y, B.z, 0.f);
    Ctr ct{0, 0, 0, 0, 0};
    Dec d = decide<MODE>(p, P4, N4, X4, NX4);
    if (d.status == 2) resolve<MODE>(p, d, P4, N4, X4, NX4, ct);
    if (d.status) code = d.bin;
  }
  codes[m * (int64_t)p.N + j] = code;
}

cudaError_t launch_pair_codes(const KParams& p, int mode, const int32_t* centre_idx, int64_t M,
                              int32_t* codes, cudaStream_t s) {
  for (int64_t m0 = 0; m0 < M; m0 += 65535) {
    const dim3 grid((unsigned)((p.N + 255) / 256), (unsigned)std::min<int64_t>(65535, M - m0));
    if (mode == 0)
      k_pair_codes<0><<<grid, 256, 0, s>>>(p, centre_idx + m0, codes + m0 * (int64_t)p.N);
    else
      k_pair_codes<1><<<grid, 256, 0, s>>>(p, centre_idx + m0, codes + m0 * (int64_t)p.N);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ diagnostic: in-sphere pairs
// SURVEY §8(d)'s implementation-independent CELLS count: pairs with |x - p| <= R, one warp
// per centre over the grid rows of p's R-box, the test in double with numpy's operation
// order (no contraction), so the oracle's float64 count is matched exactly.
__global__ void k_count_in_sphere(const int32_t* __restrict__ centre_idx, int64_t M,
                                  const float4* __restrict__ cpos, int32_t N,
                                  const float4* __restrict__ spos, const int32_t* __restrict__ cell_start,
                                  float ox, float oy, float oz, float inv_h, int dx, int dy, int dz,
                                  double R, float R_up, unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double R2 = R * R;
  unsigned long long local = 0;
  for (int64_t m = wid; m < M; m += nw) {
    const int c = centre_idx[m];
    if (c < 0 || c >= N) continue;
    const float4 P4 = cpos[c];
    const int x0 = cell_coord(__fsub_rd(P4.x, R_up), ox, inv_h, dx), x1 = cell_coord(__fadd_ru(P4.x, R_up), ox, inv_h, dx);
    const int y0 = cell_coord(__fsub_rd(P4.y, R_up), oy, inv_h, dy), y1 = cell_coord(__fadd_ru(P4.y, R_up), oy, inv_h, dy);
    const int z0 = cell_coord(__fsub_rd(P4.z, R_up), oz, inv_h, dz), z1 = cell_coord(__fadd_ru(P4.z, R_up), oz, inv_h, dz);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const int base = (z * dy + y) * dx;
        const int a = cell_start[base + x0], e = cell_start[base + x1 + 1];
        for (int j = a + lane; j < e; j += 32) {
          const float4 X = spos[j];
          const double ddx = __dsub_rn((double)X.x, (double)P4.x);
          const double ddy = __dsub_rn((double)X.y, (double)P4.y);
          const double ddz = __dsub_rn((double)X.z, (double)P4.z);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)), __dmul_rn(ddz, ddz));
          local += d2 <= R2;
        }
      }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0 && local) atomicAdd(count, local);
}

cudaError_t launch_count_in_sphere(const int32_t* centre_idx, int64_t M, const float4* cpos, int32_t N,
                                   const float4* spos, const int32_t* cell_start, float ox, float oy,
                                   float oz, float inv_h, int dx, int dy, int dz, double R, float R_up,
                                   unsigned long long* count, int sms, cudaStream_t s) {
  k_count_in_sphere<<<sms * 8, 256, 0, s>>>(centre_idx, M, cpos, N, spos, cell_start, ox, oy, oz,
                                            inv_h, dx, dy, dz, R, R_up, count);
  return cudaGetLastError();
}

}  // namespace spin
