// spin_internal.h — structures shared by the host planner (spin_api.cpp) and the
// sm_100a kernels (spin_kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spin {

// Per-launch parameters of the persistent spin kernel (passed __grid_constant__).
struct KParams {
  // ---- cloud (a1).  BRUTE: original order; CELLS: cell-sorted copy.  Both have
  // N real points followed by sentinel padding (|x|^2 = +inf never passes).
  const float4* __restrict__ pos;   // {x, y, z, |x|^2}
  const float4* __restrict__ nrm;   // {nx, ny, nz, 0}
  const float4* __restrict__ tpos;  // BRUTE: the cloud in 128-point warp-tile pair layout
                                    // (4 KB per chunk, the smem staging layout; TMA source)
  const float4* __restrict__ mfrag; // BRUTE: per 128-point chunk the mma.sync A fragments (4 KB:
                                    // uint4 (x_hi, x'_hi, x_lo, x'_lo) per row block and lane)
  const float4* __restrict__ tfa;   // BRUTE: per 128-point chunk the tcgen05 A operand (4 KB:
                                    // tf32 (x,y,z,-|x|^2) hi and (x,y,z) lo + 1, canonical layout)
  const float4* __restrict__ cpos;  // original-order copies, indexed by centre index
  const float4* __restrict__ cnrm;
  int32_t N;
  int32_t n_tiles;                  // BRUTE: padded length / (NT*K)

  // ---- centres and output (a5, a12)
  const int32_t* __restrict__ centre_idx;  // [M]
  const int32_t* __restrict__ order;       // [M] processing position -> m, or nullptr
  int64_t M;
  int32_t W;
  float* __restrict__ out;                 // [M][W][W]

  // ---- dealing (a3, a6)
  const int32_t* __restrict__ bounds;      // chunk boundaries in units, [n_chunks + 1]
  int32_t n_chunks;
  int32_t unit_images;                     // images per unit
  int32_t is_static;                       // chunk = blockIdx.x, no atomics
  unsigned int* counter;                   // the "master": one u32 in global memory
  // WF / AWF (weighted factoring, dealt by CAS; wf = 1 WF, 2 AWF, 0 table dealer)
  int32_t wf;
  unsigned long long* wf_state;            // (next unit : 24 | batch R : 24 | count : 16)
  float* awf_rate;                         // [grid] measured units per microsecond (AWF)
  int32_t n_units, fac_div, P;
  uint32_t wq_slow, wq_fast;               // WF integer weights (mean 1024)

  // ---- region constants (a2).  Doubles are exact host values; floats are the
  // conservative fp32 thresholds of the hot loop.
  double b, cos_As;          // cos_As = -inf disables the support test
  double A;                  // W/2
  double mid, Qmax;          // beta window centre, alpha^2 bound: region is |beta-mid|<=h, q<=Qmax
  double rho2;               // hot loop: squared radius of the sphere about the (rounded)
                             // window centre that contains the region
  double E_sph;              // hot-loop bound on the error of the sphere margin
  int32_t mma;               // BRUTE: sphere filter on the tensor cores (tf32 B and K)
  double Eq_hot;             // CELLS hot loop: bound on |q''_fp32 - q''| (added to Qmax - C)
  float c_test, h_test;      // hot loop: s >= c_test (support), CELLS |beta''| <= h_test
  int32_t has_support;
  int32_t cta_offset;        // global worker index of CTA 0 (STATIC block assignment)
  int32_t slow_ctas;         // heterogeneity emulation: CTAs below this index are slow
  float slowdown;            // their per-group time multiplier (>= 1)
  int32_t slow_first;        // fast CTAs wait for the slow CTAs' first requests
  int32_t support_in_hot;    // 1: hot loop tests the support; 0: accept path only; 2: adaptive (BRUTE)
  // accept path, fp32 stage
  float c_f;                 // (float)cos_As, its rounding is inside Es_a
  float inv_b, inv_b2, Af;
  float Wf;                  // (float)W
  float Au;                  // u = fma(-beta, inv_b, Au): W/2 (scaled) or fl32(W/(2b)) (literal)
  float floor_f;             // 1.0 for SPIN_F_FLOOR_BINS, else 0.0
  float Wff, bin_magic;      // W + floor_f; 2^23 - floor_f (W + 1) (NEAREST bin index, decide)
  float self_kf;             // (float)self_k
  float Es_a, Eu_a, Ew_a, D2g;
  int32_t literal, floor_bins, no_fast_cert;
  int32_t dense_min;         // BRUTE tensor-core tiles: lane-per-centre accept when candidates >=
                             // dense_min x live points (0: always compact)
  int32_t debug_skip;        // measurement only (env SPIN_DEBUG_SKIP): 1 skip accept, 2 skip compaction too
  int32_t self_fast;         // d == 0 pairs can be decided exactly without arithmetic
  int32_t self_k, self_l;    // their (k, l) (NEAREST) or (i0, -) ; self_k = -1: no contribution
  float self_a;              // BILINEAR: a for the self pair

  // ---- CELLS (a4)
  const int32_t* __restrict__ cell_start;  // [ncells + 1]
  int32_t dimx, dimy, dimz;
  float ox, oy, oz, inv_h;                 // cell = floor((x - o) * inv_h)
  float R_up;                              // region radius rounded up
  float h_cell;                            // cell edge (1 / inv_h, as the host chose it)
  int32_t row_cap;

  // ---- instrumentation (a13) and errors
  unsigned long long* stats;               // [8] global counters
  unsigned long long* cta_t0;              // [P]
  unsigned long long* cta_t1;              // [P]
  int32_t* cta_units;                      // [P]
  int32_t* err_flags;                      // [0]: bad centre index seen; [1]: overflow
  uint32_t* hi_scratch;                    // BILINEAR carry words, [P][G][(W*W+1)/2], zero
  unsigned int* seg_done;                  // e2e pipelining: images finished per output segment
  int32_t seg_images;                      // images per segment (seg_done != nullptr)
};

enum StatSlot {
  ST_VISITED = 0, ST_CAND = 1, ST_ACC = 2, ST_F64 = 3, ST_EXACT = 4, ST_SUPHOT = 5, ST_DENSE = 6, ST_DROWS = 7, ST_NSLOTS = 8
};

// Launch configuration chosen by the planner.
struct LaunchCfg {
  int G;           // images per group (4 .. 64; 48 over a two-CTA cluster)
  int threads;     // threads per CTA (768, or 512 for G = 32 at W > 24)
  int cl;          // CTAs per cluster: 1, or 2 (BRUTE: one worker = a CTA pair, DSMEM images)
  size_t smem;     // dynamic shared memory bytes
};

// ---- launchers implemented in spin_kernels.cu
LaunchCfg choose_launch(int W, int mode, int prune, bool allow_cluster);
int tile_points();   // cloud padding: a multiple of every CTA tile (threads x KP points)
// padding sentinel |x|^2 (finite: the tensor-core filter splits it into tf32 hi/lo parts)
constexpr float SENTINEL_R2 = 0x1p100f;
// largest accepted |coordinate| (SPIN_E_INPUT above): |x|^2 and the filter products stay finite
constexpr float COORD_MAX = 0x1p40f;
constexpr int KP_POINTS = 4;   // points per thread (register blocking; SPIN_KP)
int resident_workers(const LaunchCfg& lc, int W, int mode, int prune, int sms);
cudaError_t launch_spin(const LaunchCfg& lc, int mode, int prune, int grid, const KParams& p,
                        cudaStream_t s);

// cloud relayout + validation (a1)
cudaError_t launch_pair_layout(const float4* pos, const float4* nrm, int64_t Npad, float4* tpos,
                               cudaStream_t s);
// the mma.sync A fragments of every 128-point chunk (BRUTE; from the Morton-ordered cloud)
cudaError_t launch_mma_frags(const float4* pos, int64_t Npad, float4* mfrag, cudaStream_t s);
// the tcgen05 A operand of every 128-point chunk (BRUTE; from the Morton-ordered cloud)
cudaError_t launch_tf32_operand(const float4* pos, int64_t Npad, float4* tfa, cudaStream_t s);
cudaError_t launch_relayout(const float* pts, const float* nrm, int64_t N, int64_t Npad,
                            float4* pos, float4* nrm4, int32_t* bad, float* absmax,
                            float* aabb, cudaStream_t s);

// CELLS grid build (a4): keys + histogram, exclusive scan, scatter
cudaError_t launch_cell_build(const float4* pos, const float4* nrm, int32_t N, int32_t Npad,
                              float ox, float oy, float oz, float inv_h, int dx, int dy, int dz,
                              int32_t* keys, int32_t* counts, int32_t* cell_start,
                              int32_t* cursor, int32_t* scan_tmp, float4* spos, float4* snrm,
                              cudaStream_t s);
// centre ordering (a5): coarse Morton bucket counting sort
cudaError_t launch_count_in_sphere(const int32_t* centre_idx, int64_t M, const float4* cpos, int32_t N,
                                   const float4* spos, const int32_t* cell_start, float ox, float oy,
                                   float oz, float inv_h, int dx, int dy, int dz, double R, float R_up,
                                   unsigned long long* count, int sms, cudaStream_t s);
cudaError_t launch_centre_order(const int32_t* centre_idx, int64_t M, const float4* cpos,
                                int32_t N, float ox, float oy, float oz, float inv_h, int dx,
                                int dy, int dz, int shift, int bits, int32_t* keys,
                                int32_t* counts, int32_t* starts, int32_t* cursor,
                                int32_t* scan_tmp, int32_t* order, cudaStream_t s);
// BRUTE Morton order (a1 cloud copy, a5 centre order): 10 bits per axis over the cubic
// hull of the AABB, q = min(1023, floor((x - o) * inv))
struct MortonGrid {
  float ox, oy, oz, inv;
};
size_t morton_sort_temp_bytes(int64_t n);
cudaError_t launch_morton_order(const int32_t* idx, int64_t n, const float4* pos, int32_t N,
                                MortonGrid mg, uint32_t* k0, uint32_t* k1, int32_t* v0,
                                int32_t* order, void* temp, size_t temp_bytes, cudaStream_t s);
cudaError_t launch_gather_cloud(const int32_t* perm, int32_t N, int64_t Npad, const float4* pos,
                                const float4* nrm, float4* bpos, float4* bnrm, cudaStream_t s);
// diagnostic: the accept path's per-pair decision for every (centre, point) pair
cudaError_t launch_pair_codes(const KParams& p, int mode, const int32_t* centre_idx, int64_t M,
                              int32_t* codes, cudaStream_t s);
cudaError_t launch_exclusive_scan(const int32_t* in, int32_t* out, int64_t n, int32_t* tmp,
                                  cudaStream_t s);
size_t scan_tmp_elems(int64_t n);

}  // namespace spin
