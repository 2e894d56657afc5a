// spin_persistent.cuh — the persistent spin kernel of the hot path (sm_100a).
// Instantiated in spin_inst.cu (one translation unit per (mode, support, dealer) triple
// so the 112 variants compile in parallel); dispatched from spin_kernels.cu.
//
// Persistent spin kernel: P resident CTAs; each CTA
// asks the device "master" (one u32 in global memory) for the next chunk of the
// schedule (the five-step protocol of PAPER.md:262-267 collapsed to one atomicAdd;
// STATIC takes chunk blockIdx.x), and for every group of G images in the chunk:
//   a7  loads the G centres (p, n) and folds them into per-centre fp32 constants,
//       zeroes G images in shared memory (tempSpinImage + init),
//   a8  streams the cloud through registers (BRUTE: all N points, Alg. 1's inner
//       loop P:161; CELLS: the grid rows around the group), each thread holding K
//       points that are reused against all G centres (n-body blocking),
//   a9  runs the conservative pair test — BRUTE: the region's bounding sphere as a tf32
//       tensor-core GEMM (mma.sync, points split hi/lo), or on packed fp32 with the
//       support n.nx >= cos_As; CELLS: beta window and alpha^2 bound
//        plus support on packed fp32 — packing pass bits into a mask,
//   a10 compacts candidates into a per-warp shared-memory queue and processes them
//       32 at a time: exact-certified bin decision, shared-memory u32 atomics
//       (NEAREST ++) or 2^-23 fixed point (BILINEAR),
//   a11 re-takes any decision fp32 cannot certify in fp64 and then exactly
//       (spin_exact.cuh),
//   a12 writes the G images to out[m] in the caller's order (add(spinImages)),
//   a13 records %globaltimer start/finish and units per CTA (fig:loadim).
// Tensor cores only for the BRUTE sphere margin, a genuine bilinear form.
#pragma once
#include <cstdint>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "spin_internal.h"

#ifndef SPIN_NT
#define SPIN_NT 768
#endif
#ifndef SPIN_KP
#define SPIN_KP 4
#endif
#ifndef SPIN_APL_BRUTE
#define SPIN_APL_BRUTE 1      // BRUTE candidates per lane per accept pass
#endif
#ifndef SPIN_BRUTE_TMA
#define SPIN_BRUTE_TMA 1      // BRUTE: stage each warp tile with one 4 KB bulk copy (TMA)
#endif
#ifndef SPIN_TMA_WAIT_ALL
#define SPIN_TMA_WAIT_ALL 1   // every lane polls the tile mbarrier (0: lane 0 polls, warp barrier)
#endif
#ifndef SPIN_APL_CELLS
#define SPIN_APL_CELLS 2      // CELLS candidates per lane per accept pass
#endif
#ifndef SPIN_APL_CELLS_NEAREST
#define SPIN_APL_CELLS_NEAREST 1  // CELLS NEAREST candidates per lane per accept pass
#endif
#ifndef SPIN_HOT_UNROLL
#define SPIN_HOT_UNROLL 2     // unroll of the sphere-only centre-batch loop
#endif
#ifndef SPIN_BRUTE_MMA
#define SPIN_BRUTE_MMA 1      // BRUTE sphere filter on the tensor cores (0: packed fp32 FFMA2)
#endif
#ifndef SPIN_IMG_PAD
#define SPIN_IMG_PAD 1        // 1: odd image stride in shared memory for CELLS BILINEAR (0: W^2)
#endif
#ifndef SPIN_IMG_RES
#define SPIN_IMG_RES 1        // BRUTE image stride in shared memory = SPIN_IMG_RES (mod 32)
#endif
#ifndef SPIN_DEFER_STAGE
#define SPIN_DEFER_STAGE 1    // tensor-core tiles: A fragments prefetched from tpos into registers,
                              // bulk copy into shared memory only for tiles with candidates
#endif
#ifndef SPIN_TC
#define SPIN_TC 0             // BRUTE 512-thread G = 32: the sphere filter on tcgen05 (5th-gen tensor
                              // cores).  Correct (parity tests pass) but measured slower: C4
                              // BILINEAR 481 vs 275 ms -- the 4 KB A tile per 128-point chunk has
                              // to stream from L2 for every group, and three buffers per
                              // warpgroup do not cover its latency (warps wait on the MMA
                              // barrier 37% of samples; tensor pipe 3% busy).
#endif
#ifndef SPIN_FRAG_TILE
#define SPIN_FRAG_TILE 1      // BRUTE tensor-core tiles stage precomputed A fragments (p.mfrag)
#endif
#ifndef SPIN_PASS1
#define SPIN_PASS1 1          // BRUTE tensor-core tiles: pre-pass phase with prefetched fragment tiles
#endif
#ifndef SPIN_DENSE_QUEUE
#define SPIN_DENSE_QUEUE 1    // BRUTE: dense tiles queued per group and drained by all warps
#endif
#ifndef SPIN_DENSE_ROWS
#define SPIN_DENSE_ROWS 1     // dense tiles: live rows per step (2 measured slower: C4 275 -> 281 ms)
#endif
#ifndef SPIN_FILTER_PREPASS
#define SPIN_FILTER_PREPASS 1 // tensor-core filter: AND the margins' sign bits first, gather only
                              // tiles holding a candidate
#endif
#ifndef SPIN_CELLS_LAYOUT2
#define SPIN_CELLS_LAYOUT2 1  // CELLS: component-major staged tile and entries that decode with two shifts
#endif
#ifndef SPIN_CELLS_CULL
#define SPIN_CELLS_CULL 0     // CELLS: warp tiles of 128 consecutive points; centre batches whose regions
                              // cannot reach the tile's bounding box skip the pair test.  Parity-clean and
                              // the cull fires (26% of the batches on C5, 6% on C3: SPIN_CULL_DIAG), but
                              // the consecutive tiles cost what it saves (their candidates collide in
                              // the image adds): C5 132.5 -> 133.1 ms, C3 40.1 -> 41.6 ms: off
#endif
#ifndef SPIN_CULL_DIAG
#define SPIN_CULL_DIAG 0      // diagnostic builds: culled / tested centre batches in tiles_dense / dense_rows
#endif
#ifndef SPIN_CAND_PER_TILE
#define SPIN_CAND_PER_TILE 0  // 1: candidates counted once per compacted tile (measured equal to slightly slower: C2 2.92 -> 3.00 ms)
#endif
#ifndef SPIN_CELLS_PIN
#define SPIN_CELLS_PIN 1      // CELLS accept passes: shared-window addresses pinned in registers
#endif
#ifndef SPIN_SELF_RESOLVE
#define SPIN_SELF_RESOLVE 1   // NEAREST: the self pair is recognised in resolve(), not in every decision
#endif
#ifndef SPIN_FRAG_REG
#define SPIN_FRAG_REG 0       // 512-thread BRUTE tensor-core tiles: A fragments straight from L2 into
                              // registers (half a tile at a time, the next half's loads in flight during
                              // the HMMAs) instead of a bulk copy the warp waits for.  Parity-clean,
                              // measured slower (C4 filter 106 -> 130 ms, BILINEAR 245 -> 269 ms: the
                              // per-lane loads go through L1 / LSU, the bulk copy does not): off
#endif
#ifndef SPIN_EXP_ABL
#define SPIN_EXP_ABL 0        // measurement only (wrong images): pre-pass ablations, bit 0: no HMMAs, bit 1: no
                              // fragment copy, bit 2: no AND chain, bit 3: no tile ever holds a candidate,
                              // bit 5: candidate tiles do not stage their points, bit 6: nor compute masks
#endif
#ifndef SPIN_EXP_FRAG_BYTES
#define SPIN_EXP_FRAG_BYTES 4096u   // measurement only: bytes of the fragment tile actually copied
#endif
#ifndef SPIN_PIN_IMG
#define SPIN_PIN_IMG 1        // dense walks: the lane's image address pinned in a register
#endif
#ifndef SPIN_CELLS_HALVES
#define SPIN_CELLS_HALVES 1   // CELLS: a tile that overflows the ring is compacted in two halves
                              // (1: NEAREST only -- C5 152.3 -> 150.0 ms, W = 24 556 -> 545 ms; BILINEAR,
                              // two candidates per lane per pass, measured slower: C3 41.8 -> 43.3 ms)
#endif
#ifndef SPIN_QCAP_CELLS
#define SPIN_QCAP_CELLS 1024  // CELLS per-warp candidate ring (entries)
#endif
#ifndef SPIN_APL_CL
#define SPIN_APL_CL 1         // two-CTA cluster variant: candidates per lane per accept pass
#endif
#ifndef SPIN_MMA_BATCH
#define SPIN_MMA_BATCH 3      // tensor-core filter: column blocks in flight before their sign gather
#endif
#ifndef SPIN_APL_BRUTE512
#define SPIN_APL_BRUTE512 1   // the same for the 512-thread (W = 32) variant
#endif
#include "spin_exact.cuh"

namespace spin {

constexpr int HOT_UNROLL = SPIN_HOT_UNROLL;   // sphere-only batch loop unroll
constexpr int NT_DEFAULT = SPIN_NT;   // threads per CTA (one CTA per SM); 512 for G = 32 at W > 24
constexpr int KP = SPIN_KP;       // points per thread (register blocking)
constexpr int LOGKP = KP == 4 ? 2 : 1;
constexpr int CB_MAX = 32 / KP;   // centres per mask batch: CB * KP <= 32 bits
__host__ __device__ constexpr int cb_of(int G) { return G < CB_MAX ? G : CB_MAX; }
// per-warp candidate ring of u16 entries (power of two): BRUTE tiles hold few candidates
// (~2% of pairs), CELLS tiles in dense clusters many
// (G <= 32 BRUTE groups hold ~100 candidates per warp tile: a 256-entry ring frees the
// shared memory that lets W = 32 run 768-thread CTAs with G = 24)
__host__ __device__ constexpr int qcap_of(int prune, int G = 64) {
  return prune ? SPIN_QCAP_CELLS : (G <= 48 ? 256 : 512);
}

static_assert(CB_MAX * KP == 32 && KP == 4 && KP == KP_POINTS, "mask is one u32: bit (k << 3) | c");

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned msb(unsigned m) {   // m != 0
  unsigned b;
  asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(m));
  return b;
}
// ---- 1-D bulk copy (TMA engine) global -> shared with an mbarrier transaction count
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
               :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(b), "r"(phase) : "memory");
  } while (!done);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- thread-block clusters (BRUTE, two CTAs sharing one group of centres; DSMEM)
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {   // every thread of every CTA
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the shared::cluster address of a local shared-memory object in CTA `rank`'s copy
__device__ __forceinline__ unsigned mapa_rank(const void* local, unsigned rank) {
  unsigned r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ void red_cluster_add(unsigned addr, unsigned v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(unsigned addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}

// The ONE cell-coordinate function used for binning points and for bounding the
// visited rows: monotone non-decreasing in x (IEEE sub/mul by a positive constant
// and floor are monotone), clamped to [0, dim).
__device__ __forceinline__ int cell_coord(float x, float o, float inv_h, int dim) {
  float t = __fmul_rn(__fsub_rn(x, o), inv_h);
  t = fminf(fmaxf(t, 0.0f), (float)(dim - 1));
  return (int)floorf(t);
}

// Packed fp32 (sm_100a FFMA2 / FMUL2): two points per instruction, a scalar centre
// constant broadcast to both halves.  Halves one FP32 issue slot per pair.
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2 bc2(float a) { return pk2(a, a); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// ---- tensor-core sphere filter (BRUTE): tf32 operands, legacy mma.sync (HMMA)
// round to the nearest tf32 (10-bit mantissa, ties away), low 13 bits zero
__device__ __forceinline__ unsigned tf32u(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float tf32f(float x) { return __uint_as_float(tf32u(x)); }
// D[16x8] = A[16x8] B[8x8] + C, tf32 in, fp32 accumulate (one HMMA.1688.F32.TF32)
__device__ __forceinline__ void mma_tf32(float& d0, float& d1, float& d2, float& d3, unsigned a0,
                                         unsigned a1, unsigned a2, unsigned a3, unsigned b0,
                                         unsigned b1, float c0, float c1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%10,%11};"
               : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3)
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void up2u(f2 v, unsigned& lo, unsigned& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
// ---- 5th-generation tensor cores (tcgen05, sm_100a): the BRUTE sphere filter of the
// 512-thread G = 32 launch as ONE tcgen05.mma per 128-point chunk (M = 128 points, N = 32
// centres, K = 8 tf32), operands in shared memory (no swizzle, K-major canonical layout:
// 8-row x 16-byte core matrices, LBO = 128 B between the two K halves, SBO = 256 B between
// 8-row groups), the fp32 margins in tensor memory, read back lane = point
// tcgen05 pipeline depth per warpgroup: A buffers in shared memory, accumulator tiles in
// tensor memory (4 warpgroups x 4 x 32 columns = all 512); the shared-memory carve-out of
// the staged-tile and mask regions: A buffers, then the B operand, then 32 points per warp
constexpr int TC_NA = 3, TC_NB = 4, TC_NBAR = TC_NA + 2 * TC_NB;
constexpr int TC_OFF_B = 4 * TC_NA * 4096, TC_OFF_PTS = TC_OFF_B + 1024;
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned phase) {
  unsigned done;
  asm volatile("{\n\t.reg .pred p;\n\t"
               "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase) : "memory");
  return done != 0;
}
__device__ __forceinline__ uint64_t umma_desc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) |
         ((uint64_t)(256u >> 4) << 32) | ((uint64_t)1 << 46);   // version 1, SWIZZLE_NONE
}
// instruction descriptor: D f32 (bits 4-5 = 1), A and B tf32 (bits 7-9, 10-12 = 2), both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(unsigned d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
// 32 consecutive tensor-memory columns of this warp's lane quarter: v[c] = column base + c
// of lane (32 (warp % 4) + lane)
__device__ __forceinline__ void tmem_ld32(unsigned taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
               "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
               "%30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                 "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                 "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                 "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// CELLS (cylinder test): pass = (s >= c) && (|beta''| <= h) && (-q'' >= -Qt)
__device__ __forceinline__ unsigned pair_bit_n(unsigned mask, float s, float c, float abe, float h,
                                               float qn, float nqt, unsigned bit) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.f32 p, %1, %2;\n\t"
      "setp.le.and.f32 p, %3, %4, p;\n\t"
      "setp.ge.and.f32 p, %5, %6, p;\n\t"
      "@p or.b32 %0, %0, %7;\n\t}"
      : "+r"(mask)
      : "f"(s), "f"(c), "f"(abe), "f"(h), "f"(qn), "f"(nqt), "r"(bit));
  return mask;
}
// CELLS, support decided later: (|beta''| <= h) && (-q'' >= -Qt)
__device__ __forceinline__ unsigned pair_bit_r(unsigned mask, float abe, float h, float qn,
                                               float nqt, unsigned bit) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.le.f32 p, %1, %2;\n\t"
      "setp.ge.and.f32 p, %3, %4, p;\n\t"
      "@p or.b32 %0, %0, %5;\n\t}"
      : "+r"(mask)
      : "f"(abe), "f"(h), "f"(qn), "f"(nqt), "r"(bit));
  return mask;
}
// BRUTE, support and sphere: pass = (s >= c) && (m >= 0), one predicate chain + one OR
__device__ __forceinline__ unsigned pair_bit_sm(unsigned mask, float s, float c, float m,
                                                unsigned bit) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.f32 p, %1, %2;\n\t"
      "setp.ge.and.f32 p, %3, 0f00000000, p;\n\t"
      "@p or.b32 %0, %0, %4;\n\t}"
      : "+r"(mask)
      : "f"(s), "f"(c), "f"(m), "r"(bit));
  return mask;
}
// sphere only: the sign bytes of the four margins m0..m3 of one centre (sign-replicating
// PRMT: 0xff where negative), ANDed with the centre's bit in every byte, ORed into the
// mask as "rejected" bits (three PRMT + one LOP3 for four pairs; callers invert)
__device__ __forceinline__ unsigned reject_bits4(unsigned rej, unsigned m0, unsigned m1,
                                                 unsigned m2, unsigned m3, unsigned K) {
  unsigned a, b, c, d;
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(a) : "r"(m0), "r"(m1));
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(b) : "r"(m2), "r"(m3));
  asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(c) : "r"(a), "r"(b));
  asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(d) : "r"(c), "r"(K), "r"(rej));
  return d;
}

// the same gather for "accepted" bits: acc | (K & ~sign bytes) in the final LOP3
__device__ __forceinline__ unsigned accept_bits4(unsigned acc, unsigned m0, unsigned m1,
                                                 unsigned m2, unsigned m3, unsigned K) {
  unsigned a, b, c, d;
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(a) : "r"(m0), "r"(m1));
  asm("prmt.b32 %0, %1, %2, 0xfbfb;" : "=r"(b) : "r"(m2), "r"(m3));
  asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(c) : "r"(a), "r"(b));
  asm("lop3.b32 %0, %1, %2, %3, 0xae;" : "=r"(d) : "r"(c), "r"(K), "r"(acc));
  return d;
}

// ------------------------------------------------------------------ smem layout
// Shared-memory image stride in words.  BILINEAR: odd (W^2 or W^2 + 1), so the same bin
// of neighbouring images falls in different banks (measured: C3 43.8 -> 41.8 ms, C4 401 ->
// 398 ms; for NEAREST the padding measured 1-3% slower)
// BRUTE (both modes): W^2 padded to IS = SPIN_IMG_RES (mod 32), so that the dense
// lane-per-centre adds (lane g -> word g * IS + bin) of neighbouring centres, whose bins for
// one point differ by a few columns, spread over the banks as (SPIN_IMG_RES * g + bin) mod 32
__host__ __device__ constexpr int img_stride(int W, int mode, int prune) {
  return prune == 0 ? W * W + ((SPIN_IMG_RES - W * W) & 31)
         : (mode == 1 && SPIN_IMG_PAD) ? ((W * W) | 1) : W * W;
}
struct Layout {
  size_t oA, oB, oP, oN, oM, oImg, oHi, oQ, oTP, oTN, oMask, oRowS, oRowO, total;
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
// G: the group's centres (constants, mask words, entries); the CTA holds G / cl of their
// images (cl = 2: a two-CTA cluster shares one group, each CTA owning half the images)
__host__ __device__ inline Layout make_layout(int G, int W, int mode, int prune, int nt, int cl = 1) {
  const int NWARP = nt / 32, ROWCAP = nt;   // CELLS: grid rows staged per batch = threads
  Layout L;
  size_t o = 0;
  L.oA = o; o += 16 * (size_t)G;
  L.oB = o; o += 16 * (size_t)G;
  L.oP = o; o += 16 * (size_t)G;
  L.oN = o; o += 16 * (size_t)G;
  L.oM = o; o = align16(o + 4 * (size_t)G);
  // everything but the images has a compile-time offset (G, NT, mode, prune are template
  // constants); the images, whose size depends on the runtime W, go last
  L.oQ = o; o += 2 * (size_t)qcap_of(prune, G) * NWARP;
  o = align16(o);
  L.oTP = o; o += 32 * (size_t)32 * KP * NWARP;    // per-warp staged tile, pair layout (32 B/point)
  L.oTN = o;
  L.oMask = o; o += 4 * (size_t)32 * (G / cb_of(G)) * NWARP;   // per-warp pass masks of the tile
  L.oRowS = o;
  L.oRowO = o;
  if (prune == 1) {
    o += 4 * ROWCAP;
    L.oRowO = o;
    o += 4 * (ROWCAP + 1);
    o = align16(o);
  }
  L.oImg = o; o = align16(o + 4 * (size_t)img_stride(W, mode, prune) * (G / cl));
  L.oHi = o;
  L.total = o;
  return L;
}

// ------------------------------------------------------------------ counters
struct Ctr {
  unsigned cand, acc, f64, exact, srej;   // srej: candidates the support test rejected
};

// BILINEAR accumulator: 2^-23 fixed point.  The 32-bit low words live in shared
// memory; the rare carries (one per 512 units of weight in a bin) go to 16-bit carry
// words (two bins per u32) in a per-CTA global scratch that is zero between groups,
// and raise a shared flag so that only groups with carries read or clear it.
// round(w * 2^23) for w in [0,1] is the mantissa of 1 + w.
__device__ __forceinline__ uint32_t fixed23(float w) {
  return __float_as_uint(w + 1.0f) - 0x3f800000u;
}
static __device__ __noinline__ void carry_fixed(uint32_t* hi, int bin, int32_t* err, int* carry_flag) {
  const uint32_t sh = (uint32_t)(bin & 1) * 16u;
  const uint32_t prev = atomicAdd(&hi[bin >> 1], 1u << sh);
  if (((prev >> sh) & 0xffffu) == 0xffffu) atomicOr(&err[1], 1);
  *carry_flag = 1;
}

// ------------------------------------------------------------------ accept path
// round-to-nearest-even for |x| < 2^22 on the FMA pipe (no F2I/FRND on the XU pipe)
__device__ __forceinline__ float rint_magic(float x) {
  return __fsub_rn(__fadd_rn(x, 12582912.0f), 12582912.0f);
}

// k*W + l for integral floats k, l in [0, W) (< 2^12) on the FMA pipe: the float sum is
// exact, +2^23 puts the integer in the low mantissa bits (no F2I on the XU pipe).  Used
// only for certified verdicts; other lanes may carry garbage, masked in range.
__device__ __forceinline__ int bin_index(float k, float l, float Wf) {
  return (int)(__float_as_uint(__fadd_rn(__fmaf_rn(k, Wf, l), 8388608.0f)) & 0x7fffffu);
}

// The slow stages, out of line; operands by value so the fast path keeps no stack.
static __device__ __noinline__ SlowOut slow_pair(float4 P4, float4 N4, float4 X4, float4 NX4, int W,
                                          double A, double b, double cos_As, int has_support,
                                          int literal, int floor_bins, int mode) {
  PairD D;
  D.p[0] = P4.x; D.p[1] = P4.y; D.p[2] = P4.z;
  D.n[0] = N4.x; D.n[1] = N4.y; D.n[2] = N4.z;
  D.x[0] = X4.x; D.x[1] = X4.y; D.x[2] = X4.z;
  D.nx[0] = NX4.x; D.nx[1] = NX4.y; D.nx[2] = NX4.z;
  return slow_decide(D, W, A, b, cos_As, has_support, literal, floor_bins, mode);
}

// One candidate (centre slot g, point X): the certified fp32 decision, branch-free.
//   status 0: certainly no contribution; 1: contributes (bin / weights below);
//   2: some decision is not certified in fp32 -> slow_pair (fp64, then exact).
struct Dec {
  int status;
  int far;      // |d|^2 certainly beyond the certified domain: certainly outside the region
  int sup_out;  // certainly rejected by the support test
  int bin;      // NEAREST: k*W + l; BILINEAR: i0*W + j0
  float a, c;   // BILINEAR fractional offsets along k and l
};

template <int MODE>
__device__ __forceinline__ Dec decide(const KParams& p, const float4 P4, const float4 N4,
                                      const float4 X4, const float4 NX4) {
  const float Wf = p.Wf, Wm1 = Wf - 1.0f;
  const float d0 = __fsub_rn(X4.x, P4.x), d1 = __fsub_rn(X4.y, P4.y), d2 = __fsub_rn(X4.z, P4.z);
  // support test, inclusive, cosine form (#5); c_f = -inf disables it (ds = +inf)
  const float s = fmaf(N4.x, NX4.x, fmaf(N4.y, NX4.y, N4.z * NX4.z));
  const float ds = s - p.c_f;
  const bool sup_out = ds < -p.Es_a;                                 // certainly rejected
  const float be = fmaf(N4.x, d0, fmaf(N4.y, d1, N4.z * d2));       // np_i.(X-P)
  const float dd = fmaf(d0, d0, fmaf(d1, d1, d2 * d2));              // ||X-P||^2
  const float q = fmaf(-be, be, dd);                                 // alpha^2
  // u = W/2 - beta/b (scaled, #2) or (W/2 - beta)/b (literal: Au = fl(W/(2b)), in Eu)
  const float uval = fmaf(-be, p.inv_b, p.Au);
  const float wval = q * p.inv_b2;                                   // (alpha/b)^2
  // fp32 verdicts need the certified domain (|d| <= D) and |u| < 2^21 (magic rounding)
  // (SPIN_F_NO_FAST_CERT arrives as D2g = -1: every candidate is uncertain)
  // (NEAREST: dd == 0 -- the self pair, a duplicate point, or an underflow -- goes to resolve(),
  // which knows the self pair's bin without arithmetic; keeps ~7 instructions out of every decision)
  const bool unc0 = !(ds > p.Es_a) | !(dd <= p.D2g) | (SPIN_SELF_RESOLVE && MODE == 0 && !(dd > 0.0f)) |
                    !(fabsf(uval) < 2097152.0f);
  Dec r;
  r.a = 0.f;
  r.c = 0.f;
  r.sup_out = sup_out;
  // fl(dd) carries a relative error below 6u, and D2g exceeds the region's largest |d|^2
  // by more than 0.2% (spin_api.cpp plan_thresholds), so dd > D2g certainly leaves the
  // region (D2g < 0: SPIN_F_NO_FAST_CERT, every decision goes to the slow stages)
  r.far = (dd > p.D2g) & (p.D2g >= 0.0f);
  if (MODE == 0) {
    // the self pair (d == 0): beta = q = 0 exactly, k = ceil(W/2) (or floor), l = 0 (#8)
    const bool self = !SPIN_SELF_RESOLVE && (fabsf(d0) + fabsf(d1) + fabsf(d2) == 0.f) & (p.self_fast != 0);
    // row k = ceil(u) (or floor): certified when u is farther than Eu from an integer;
    // |u| < 2^22 inside the certified domain (dd <= D2g), garbage is ignored outside it
    const float rr = rint_magic(uval);
    const float du = uval - rr;                                      // exact
    bool ku = !(fabsf(du) > p.Eu_a);
    // (kf and lf carry the floor-reading shift floor_f, taken out once in the bin index: k and
    // l are small integers, every sum below is exact)
    const float ff = p.floor_f, Wff = p.Wff;
    float kf = rr + (du > 0.f ? 1.0f : 0.0f);
    // column l = ceil(sqrt(w)) (or floor): certified when w is farther than Ew from
    // every perfect square (fl^2 is exact); sqrt only proposes fl, the squares decide
    // (w below 1e-30, negative included, proposes fl = 0 like the exact zero)
    const float wc = fmaxf(wval, 1e-30f);
    float rs;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(wc));
    const float fl = rint_magic(fmaf(wc, rs, -0.5f));
    const float dlo = fmaf(-fl, fl, wval), dhi = fmaf(fl + 1.0f, fl + 1.0f, -wval);
    const bool wneg = wval < -p.Ew_a;
    bool lu = !(wneg | ((dlo > p.Ew_a) & (dhi > p.Ew_a)));
    float lf = wneg ? ff : fl + 1.0f;
    if (self) { kf = p.self_kf + ff; lf = ff; ku = false; lu = false; }
    const bool out = (!ku & ((kf < ff) | (kf >= Wff))) | (!lu & (lf >= Wff));
    r.status = (sup_out | (!unc0 & out)) ? 0 : ((unc0 | ku | lu) ? 2 : 1);
    // (k - ff) W + (l - ff) + 2^23
    r.bin = (int)(__float_as_uint(__fadd_rn(__fmaf_rn(kf, Wf, lf), p.bin_magic)) & 0x7fffffu);
  } else {
    // BILINEAR region 0 <= u < W-1, w < (W-1)^2  (#12); the self pair (u = W/2, w = 0)
    // is interior for W >= 3 and needs no special case
    const bool uu = !((fabsf(uval) > p.Eu_a) & (fabsf(uval - Wm1) > p.Eu_a));
    const float lim = Wm1 * Wm1;
    const bool wu = !(fabsf(wval - lim) > p.Ew_a);
    const bool out = (!uu & !((uval > 0.f) & (uval < Wm1))) | (!wu & !(wval < lim));
    r.status = (sup_out | (!unc0 & out)) ? 0 : ((unc0 | uu | wu) ? 2 : 1);
    // v only places the splat (continuous in v across bin edges); the region edge was
    // decided on w above.  alpha^2 = |d|^2 - beta^2 cancels when X - P is nearly parallel
    // to n (its error ~3u|d|^2 becomes 3u|d|^2 / (2 b alpha) in v), so within 1/8 rad of
    // the normal axis (alpha^2 < |d|^2 / 64) the splat takes alpha^2 from Lagrange's
    // identity, |d x n|^2 - (|n|^2 - 1)|d|^2, whose fp32 error is O(u |d| alpha); outside
    // it the direct form's v error is below 12u|d|/b.  The approximate square root (MUFU,
    // ~2 ulp) is within the tolerance.
    float qs = q;
    if (q < dd * 0.015625f) {   // (a warp-vote variant measured 1-2% slower)
      const float cx = fmaf(d1, N4.z, -(d2 * N4.y));
      const float cy = fmaf(d2, N4.x, -(d0 * N4.z));
      const float cz = fmaf(d0, N4.y, -(d1 * N4.x));
      qs = fmaf(cx, cx, fmaf(cy, cy, fmaf(cz, cz, -N4.w * dd)));
    }
    float v;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(v) : "f"(fmaxf(qs * p.inv_b2, 0.0f)));
    const float fi = fminf(fmaxf(rint_magic(uval - 0.5f), 0.0f), Wm1 - 1.0f);
    const float fj = fminf(fmaxf(rint_magic(v - 0.5f), 0.0f), Wm1 - 1.0f);
    r.a = fminf(fmaxf(uval - fi, 0.0f), 1.0f);
    r.c = fminf(fmaxf(v - fj, 0.0f), 1.0f);
    r.bin = bin_index(fi, fj, Wf);
  }
  return r;
}

// Resolve an uncertain decision in fp64 / exactly (out of line, rare).
template <int MODE>
__device__ __forceinline__ void resolve(const KParams& p, Dec& d, const float4 P4, const float4 N4,
                                        const float4 X4, const float4 NX4, Ctr& ct) {
  if (SPIN_SELF_RESOLVE && MODE == 0 && p.self_fast &&
      fabsf(X4.x - P4.x) + fabsf(X4.y - P4.y) + fabsf(X4.z - P4.z) == 0.f) {
    // the self pair (d == 0 exactly): beta = q = 0, k = ceil(W/2) (or floor), l = 0 (#8); only
    // its support test (|n|^2 against cos A_s) needs a certain verdict
    const float s = fmaf(N4.x, NX4.x, fmaf(N4.y, NX4.y, N4.z * NX4.z));
    if (s - p.c_f > p.Es_a) {
      d.status = p.self_k >= 0;
      d.bin = p.self_k * p.W + p.self_l;
      return;
    }
  }
  ++ct.f64;
  const SlowOut r = slow_pair(P4, N4, X4, NX4, p.W, p.A, p.b, p.cos_As, p.has_support, p.literal,
                              p.floor_bins, MODE);
  ct.exact += r.n_exact;
  d.status = r.accept;
  if (MODE == 0) d.bin = r.k * p.W + r.l;
}

// Splat an accepted pair into its image (tempSpinImage[k,l]++).
// CL = 2 (NEAREST): the image of group slot g lives in CTA g / (G/2) of the cluster; the
// count goes through a shared::cluster address (a fire-and-forget DSMEM reduction when the
// owner is the partner CTA).  (BILINEAR stays on one-CTA workers: its fixed-point carries
// need the old value back, and four returning DSMEM atomics per splat measured slower.)
template <int MODE, int G, int CL>
__device__ __forceinline__ void apply_cl(const Dec& d, uint32_t* sImg, int IS, int g) {
  static_assert(MODE == 0, "clusters: NEAREST only");
  constexpr int GL = G / CL;
  const unsigned owner = (unsigned)(g / GL);
  const int ls = g - (int)owner * GL;
  red_cluster_add(mapa_rank(sImg + ls * IS, owner) + 4u * (unsigned)d.bin, 1u);
}

__device__ __forceinline__ uint32_t atoms_add(unsigned addr, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(addr), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void reds_add(unsigned addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
// apply() with the image as a 32-bit shared-window address (no generic-address
// conversion per pair)
template <int MODE, int G>
__device__ __forceinline__ void apply_s(const KParams& p, const Dec& d, unsigned img, int slot,
                                        int* carry_flag) {
  if (MODE == 0) {
    reds_add(img + 4u * (unsigned)d.bin, 1u);
  } else {
    const int W = p.W;
    const unsigned a0 = img + 4u * (unsigned)d.bin, a1 = a0 + 4u * (unsigned)W;
    const uint32_t v0 = fixed23((1.0f - d.a) * (1.0f - d.c)), v1 = fixed23(d.a * (1.0f - d.c));
    const uint32_t v2 = fixed23((1.0f - d.a) * d.c), v3 = fixed23(d.a * d.c);
    const uint32_t o0 = atoms_add(a0, v0), o1 = atoms_add(a1, v1);
    const uint32_t o2 = atoms_add(a0 + 4u, v2), o3 = atoms_add(a1 + 4u, v3);
    if (max(max(o0, o1), max(o2, o3)) >= 0xff800000u) {
      const int hiWords = (W * W + 1) / 2;
      uint32_t* hi = p.hi_scratch + ((size_t)blockIdx.x * G + slot) * hiWords;
      if (o0 + v0 < o0) carry_fixed(hi, d.bin, p.err_flags, carry_flag);
      if (o1 + v1 < o1) carry_fixed(hi, d.bin + W, p.err_flags, carry_flag);
      if (o2 + v2 < o2) carry_fixed(hi, d.bin + 1, p.err_flags, carry_flag);
      if (o3 + v3 < o3) carry_fixed(hi, d.bin + W + 1, p.err_flags, carry_flag);
    }
  }
}

template <int MODE, int G>
__device__ __forceinline__ void apply(const KParams& p, const Dec& d, uint32_t* img, int slot,
                                      int* carry_flag) {
  if (MODE == 0) {
    atomicAdd(&img[d.bin], 1u);
  } else {
    const int W = p.W;
    // four u32 adds; a wrapped low word (at most one per 512 units of weight in a bin) is
    // carried into its 16-bit high word on one shared, rarely taken branch
    const int b0 = d.bin, b1 = d.bin + W, b2 = d.bin + 1, b3 = d.bin + W + 1;
    const uint32_t v0 = fixed23((1.0f - d.a) * (1.0f - d.c)), v1 = fixed23(d.a * (1.0f - d.c));
    const uint32_t v2 = fixed23((1.0f - d.a) * d.c), v3 = fixed23(d.a * d.c);
    const uint32_t o0 = atomicAdd(&img[b0], v0), o1 = atomicAdd(&img[b1], v1);
    const uint32_t o2 = atomicAdd(&img[b2], v2), o3 = atomicAdd(&img[b3], v3);
    // v <= 2^23, so a wrap needs old >= 2^32 - 2^23: one screen for all four, the exact
    // test on the rare branch
    if (max(max(o0, o1), max(o2, o3)) >= 0xff800000u) {
      const int hiWords = (W * W + 1) / 2;
      uint32_t* hi = p.hi_scratch + ((size_t)blockIdx.x * G + slot) * hiWords;
      if (o0 + v0 < o0) carry_fixed(hi, b0, p.err_flags, carry_flag);
      if (o1 + v1 < o1) carry_fixed(hi, b1, p.err_flags, carry_flag);
      if (o2 + v2 < o2) carry_fixed(hi, b2, p.err_flags, carry_flag);
      if (o3 + v3 < o3) carry_fixed(hi, b3, p.err_flags, carry_flag);
    }
  }
}

// ------------------------------------------------------------------ WF / AWF dealer
// Weighted factoring (beyond the paper, its future work P:238; spin.h SPIN_WF / SPIN_AWF),
// called by warp 0: this worker's integer weight (mean 1024) — a priori (WF) or from the
// measured rates (AWF: mine over the mean of the workers that have reported; a one-unit
// probing chunk before my first measurement) — then lane 0 claims [wu[0], wu[1]) by
// compare-and-swap on the packed state (next : 24 | batch R : 24 | count : 16): a batch
// of P claims shares R = the units
// left at its first claim (FAC2 batches), the same integer rule as the host
// trace (spin_api.cpp wf_chunk).  Out of line: one call per chunk.
static __device__ __noinline__ void wf_claim(const KParams& p, int lane, int* wu,
                                             unsigned long long& t_claim) {
  unsigned wq = (int)blockIdx.x < p.slow_ctas ? p.wq_slow : p.wq_fast;
  if (p.wf == 2) {
    const volatile float* rates = p.awf_rate;
    float sum = 0.f;
    int cnt = 0;
    for (int i = lane; i < (int)gridDim.x; i += 32) {
      const float r = rates[i];
      if (r > 0.f) { sum += r; ++cnt; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    const float mine = rates[blockIdx.x];
    // before its first measurement a worker probes with a one-unit chunk (weight 0 -> the
    // minimum chunk), so the weights are known before the large early chunks
    wq = 0u;
    if (mine > 0.f && cnt > 0)
      wq = (unsigned)fminf(fmaxf(rintf(1024.f * mine * (float)cnt / sum), 16.f), 65536.f);
  }
  if (lane == 0) {
    const unsigned U = (unsigned)p.n_units;
    const unsigned long long den = (unsigned long long)p.fac_div * (unsigned)p.P * 1024ull;
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(p.wf_state);
    for (;;) {
      const unsigned next = (unsigned)(old & 0xffffffull);
      if (next >= U) { wu[0] = wu[1] = (int)U; break; }
      const unsigned cnt = (unsigned)(old >> 48);
      const unsigned Rb = cnt == 0 ? U - next : (unsigned)((old >> 24) & 0xffffffull);
      unsigned long long c = ((unsigned long long)Rb * wq + den - 1ull) / den;
      c = min(max(c, 1ull), (unsigned long long)(U - next));
      const unsigned nn = next + (unsigned)c;
      const unsigned nc = cnt + 1u >= (unsigned)p.P ? 0u : cnt + 1u;
      const unsigned long long nw = (unsigned long long)nn | ((unsigned long long)Rb << 24) |
                                    ((unsigned long long)nc << 48);
      const unsigned long long prev = atomicCAS(p.wf_state, old, nw);
      if (prev == old) { wu[0] = (int)next; wu[1] = (int)nn; break; }
      old = prev;
    }
    atomicAdd(p.counter, 1u);   // requests (stats n_chunks; the slow-first wait)
    t_claim = gtimer();
  }
}

// ------------------------------------------------------------------ the kernel
// SUP = 1: the hot loop evaluates the support test for every pair (the paper's order,
// P:166 before P:169-171); SUP = 0: the hot loop tests the region only and the support
// test is decided in the accept path (SPIN_F_SUPPORT_LAST, or no support test at all).
// CL = 2 (BRUTE NEAREST, table dealer): a two-CTA thread-block cluster is ONE worker: both CTAs take
// the same chunk (dealt by rank 0, passed through DSMEM) and the same groups of G centres;
// each owns G/2 of the images and streams every other point tile, so the per-tile work
// (bulk copy, tf32 split, compaction) is shared by G centres while each SM holds only
// G/2 images.
template <int MODE, int PRUNE, int G, int SUP, int NT, int DEAL, int CL>
__global__ void __launch_bounds__(NT, 1) spin_persistent(const __grid_constant__ KParams p) {
  static_assert(CL == 1 || (CL == 2 && MODE == 0 && PRUNE == 0 && DEAL == 0 && G % 2 == 0),
                "clusters: BRUTE NEAREST, table dealer");
  constexpr int GL = G / CL;        // images this CTA owns
  constexpr int NWARP = NT / 32;
  constexpr int ROWCAP = NT;        // CELLS: grid rows staged per batch
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_chunk;
  __shared__ int s_total, s_live;
  __shared__ int s_rng[6];
  __shared__ unsigned long long s_ctr[8];

  const int W = p.W;
  const int WW = W * W;
  const int IS = img_stride(W, MODE, PRUNE);   // shared-memory image stride (words)
  const Layout L = make_layout(G, W, MODE, PRUNE, NT, CL);
  const unsigned crank = CL > 1 ? cluster_rank() : 0u;
  float4* sA = reinterpret_cast<float4*>(smem + L.oA);
  float4* sB = reinterpret_cast<float4*>(smem + L.oB);
  float4* sP = reinterpret_cast<float4*>(smem + L.oP);
  float4* sN = reinterpret_cast<float4*>(smem + L.oN);
  int* sM = reinterpret_cast<int*>(smem + L.oM);
  uint32_t* sImg = reinterpret_cast<uint32_t*>(smem + L.oImg);
  __shared__ int s_carry;
  int* sRowS = reinterpret_cast<int*>(smem + L.oRowS);
  int* sRowO = reinterpret_cast<int*>(smem + L.oRowO);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool skip_accept = p.debug_skip != 0;   // measurement knob (SPIN_DEBUG_SKIP)
  // BRUTE BILINEAR stages tiles with one bulk copy (measured: C4 455 -> 435 ms, C2 3.68 ->
  // 3.66 ms); BRUTE NEAREST keeps per-lane loads (measured faster there: C2 3.39 vs 3.48,
  // P6 26.9 vs 27.5 ms with the bulk copy)
  constexpr bool TMA_TILE = PRUNE == 0 && SPIN_BRUTE_TMA;
  __shared__ __align__(8) uint64_t s_tile_bar[NWARP];   // BRUTE: tile bulk-copy barrier per warp
  unsigned tile_phase = 0;
  if (TMA_TILE) {
    if (lane == 0) mbar_init(&s_tile_bar[warp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  // tcgen05 filter (BRUTE, one-CTA 512-thread workers with G = 32; the planner's tf32 bound
  // applies to it unchanged): four warpgroups, each streaming every fourth 128-point chunk
  // through ONE tensor-core MMA into a double-buffered tensor-memory tile
  constexpr bool TC = SPIN_TC && PRUNE == 0 && CL == 1 && NT == 512 && G == 32 && SUP != 1 &&
                      SPIN_BRUTE_MMA && SPIN_BRUTE_TMA;
  static_assert(!TC || TC_OFF_PTS + NWARP * 1024 <= 4096 * NWARP + 4 * 32 * (G / cb_of(G)) * NWARP,
                "tcgen05 buffers must fit the staged-tile and mask regions");
  __shared__ __align__(8) uint64_t s_tcbar[TC ? 4 * TC_NBAR : 1];   // per warpgroup: A full, D full, D empty
  __shared__ unsigned s_tmem;
  const bool tc_on = TC && p.mma && p.tfa != nullptr;
  if (tc_on) {
    if (tid < 4 * TC_NBAR) mbar_init(&s_tcbar[tid], (tid % TC_NBAR) >= TC_NA + TC_NB ? 4u : 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                   :: "r"((unsigned)__cvta_generic_to_shared(&s_tmem)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  unsigned tc_it = 0;   // chunks this warp's warpgroup has streamed (all groups): buffer / phase
  constexpr int QCAP = qcap_of(PRUNE, G);
  uint16_t* sQ = reinterpret_cast<uint16_t*>(smem + L.oQ) + warp * QCAP;
  // staged tile of this warp in pair layout: record r (0..3) of point pair pr (0..KP/2-1)
  // of lane l at sT[(r * (KP/2) + pr) * 32 + l]; r0 {x,x',y,y'}, r1 {z,z',-|x|^2,-|x'|^2},
  // r2 {nx,nx',ny,ny'}, r3 {nz,nz',0,0}
  float4* sT = reinterpret_cast<float4*>(smem + L.oTP) + warp * 32 * KP * 2;
  constexpr int CB = cb_of(G);
  // BRUTE sphere filter on the tensor cores (mma.sync tf32, hi/lo split of the points):
  // NCB column blocks of 8 centres, 8 row blocks of 16 points per warp tile
  constexpr bool MMA_FILTER = PRUNE == 0 && SPIN_BRUTE_MMA;
  constexpr int NCB = (G + 7) / 8;
  static_assert(!MMA_FILTER || (NCB == G / CB && KP == 4), "mma mask layout: NCB words per lane");
  unsigned* sMask = reinterpret_cast<unsigned*>(smem + L.oMask) + warp * 32 * (G / CB);
  const int hiWords = (WW + 1) / 2;
  uint32_t* gHi = p.hi_scratch + (size_t)blockIdx.x * GL * hiWords;   // zero outside groups
  if (tid == 0) s_carry = 0;
  if (CL > 1) cluster_sync_all();   // every CTA of the cluster has started (DSMEM rule)

  if (tid < 8) s_ctr[tid] = 0ull;
  const unsigned long long t0 = gtimer();
  Ctr ct{0, 0, 0, 0, 0};
  // SUP = 2 (BRUTE, adaptive support placement, per warp): a warp starts with the support
  // test in the accept path and moves it into its hot loop when, in one tile, the
  // candidates the test rejects exceed 1/SUP_RATIO of the tile's pairs; it re-probes
  // after SUP_PROBE tiles.  Images are identical either way.
  constexpr unsigned SUP_RATIO = 64;
  constexpr int SUP_PROBE = 16;
  bool sup_on = false;
  int sup_count = 0;
  unsigned sup_tiles = 0;
  unsigned dense_tiles = 0, dense_rows = 0;   // lane 0 of each warp (stats)
  int units_done = 0;
  unsigned long long visited = 0;
  bool first = true;

  // BRUTE dense-tile queue of a group (chunk indices), drained by every warp in phase 2
  // (BILINEAR: C4 275 -> 267 ms, C2 equal; NEAREST, whose re-staging and mask recomputation
  // cost more than the balance gains: C4 243 -> 258 ms, P6 21.9 -> 22.4 ms, so not used)
  // PASS1 (with the precomputed fragments): phase 1 only runs the pre-pass, streaming the
  // fragment tiles through ONE buffer per warp with the next tile's copy in flight, and
  // queues every tile that holds a candidate; phase 2 re-stages and decides the queued tiles
  // (measured: 768-thread CTAs C2 BILINEAR 3.18 -> 3.06 ms, NEAREST 2.90 -> 2.83 ms, P6
  // 20.31 -> 20.43 ms; 512-thread CTAs slower, C4 BILINEAR 251.7 -> 257.4 ms, NEAREST 229.5
  // -> 232.8 ms: 768-thread CTAs only, SPIN_PASS1 = 2 forces it everywhere)
  constexpr bool PASS1 = PRUNE == 0 && CL == 1 && SPIN_BRUTE_MMA && SPIN_BRUTE_TMA && SPIN_FRAG_TILE &&
                         (SPIN_PASS1 == 2 || (SPIN_PASS1 == 1 && NT > 512));
  constexpr bool DQ = PASS1 || (PRUNE == 0 && CL == 1 && MODE == 1 && SPIN_BRUTE_MMA && SPIN_BRUTE_TMA &&
                                SPIN_DENSE_QUEUE);
  constexpr int DQ_CAP = DQ ? 512 : 1;
  __shared__ int s_dq[DQ_CAP];
  __shared__ int s_dq_n, s_dq_head;
  if (DQ && tid == 0) s_dq_n = s_dq_head = 0;
  __shared__ int s_wu[2];              // WF/AWF: the claimed unit range
  // AWF bookkeeping of tid 0 (in shared memory: no registers live across the loop):
  // [0] claim time, [1] chunk time so far, [2] units so far
  __shared__ unsigned long long s_awf[3];
  if (DEAL && tid == 0) s_awf[0] = s_awf[1] = s_awf[2] = 0ull;
  for (;;) {
    // ---- a6: request a chunk (PAPER.md:336-342 / 372-377)
    if (DEAL ? warp == 0 : tid == 0) {
      if (lane == 0 && first && p.slow_first && (int)blockIdx.x >= p.slow_ctas) {
        // heterogeneity emulation: the slow workers request first
        while (*reinterpret_cast<volatile unsigned*>(p.counter) < (unsigned)p.slow_ctas) __nanosleep(256);
      }
      if (DEAL) {
        __syncwarp();
        wf_claim(p, lane, s_wu, s_awf[0]);   // warp 0 (AWF reads the rates), lane 0 claims
      } else if (CL == 1 || crank == 0) {
        // (a cluster is one worker: rank 0 asks and hands the chunk to its partner)
        const int ch = p.is_static ? (first ? p.cta_offset + (int)(blockIdx.x / CL) : p.n_chunks)
                                   : (int)atomicAdd(p.counter, 1u);
        s_chunk = ch;
        if (CL > 1) st_cluster_s32(mapa_rank(&s_chunk, 1u), ch);
      }
    }
    if (CL > 1) cluster_sync_all();
    else __syncthreads();
    first = false;
    int u0, u1;
    if (DEAL) {
      u0 = s_wu[0];
      u1 = s_wu[1];
      if (u0 >= u1) break;
    } else {
      const int u = s_chunk;
      if (u >= p.n_chunks) break;
      u0 = p.bounds[u];
      u1 = p.bounds[u + 1];
    }
    const long long i0 = (long long)u0 * p.unit_images;
    const long long i1 = min((long long)u1 * p.unit_images, (long long)p.M);

    for (long long g0 = i0; g0 < i1; g0 += G) {
      const int gcount = (int)min((long long)G, i1 - g0);
      const unsigned long long tg0 = gtimer();
      // ---- a7: group setup (tempSpinImage, init, P = OP[i])
      if (tid < G) {
        const int slot = tid;
        float4 A4 = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 B4 = make_float4(0.f, 0.f, 0.f, PRUNE == 0 ? -INFINITY : INFINITY);
        float4 P4 = make_float4(0.f, 0.f, 0.f, 0.f), N4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int mm = -1;
        if (slot < gcount) {
          const long long ip = g0 + slot;
          const int m = p.order ? p.order[ip] : (int)ip;
          const int c = p.centre_idx[m];
          if (c >= 0 && c < p.N) {
            P4 = __ldg(&p.cpos[c]);
            N4 = __ldg(&p.cnrm[c]);
            // |n|^2 - 1 for the BILINEAR splat position (Lagrange's identity, decide)
            N4.w = (float)((double)N4.x * N4.x + (double)N4.y * N4.y + (double)N4.z * N4.z - 1.0);
            const double mid = p.mid;
            if (PRUNE == 0) {
              // BRUTE: sphere of radius rho about c~ = B/2, B = fl(2(p + mid n)) (DESIGN.md
              // 7.1): K = rho^2 - |c~|^2 + 2E rounded up, so the fp32 margin
              // B.x - |x|^2 + K is positive for every pair of the region
              // with the tensor-core filter B is rounded to tf32 (an exact operand;
              // |B - 2c'| <= 2^-11 |2c'|, the planner's rho covers the shift of c~)
              float Bx = __double2float_rn(2.0 * ((double)P4.x + mid * N4.x));
              float By = __double2float_rn(2.0 * ((double)P4.y + mid * N4.y));
              float Bz = __double2float_rn(2.0 * ((double)P4.z + mid * N4.z));
              if (MMA_FILTER && p.mma) { Bx = tf32f(Bx); By = tf32f(By); Bz = tf32f(Bz); }
              const double cx = 0.5 * Bx, cy = 0.5 * By, cz = 0.5 * Bz;
              const double K = p.rho2 - (cx * cx + cy * cy + cz * cz) + 2.0 * p.E_sph;
              float Kf = __double2float_ru(K);
              if (MMA_FILTER && p.mma) Kf = tf32f(Kf);   // a tensor-core operand too (in E)
              A4 = make_float4(N4.x, N4.y, N4.z, 0.f);
              B4 = make_float4(Bx, By, Bz, Kf);
            } else {
              // CELLS: the region cylinder itself, beta'' = n.x - n.p - mid and
              // -q'' = beta''^2 + 2(p + mid n).x - |x|^2 - C >= -Qt
              const double px = P4.x, py = P4.y, pz = P4.z, nx = N4.x, ny = N4.y, nz = N4.z;
              const double np = nx * px + ny * py + nz * pz;
              const double C = (px * px + py * py + pz * pz) + 2.0 * mid * np + mid * mid;
              const double Qt = p.Qmax - C + p.Eq_hot + 1e-12 * (fabs(C) + p.Qmax);
              A4 = make_float4(N4.x, N4.y, N4.z, __double2float_rn(-np - mid));
              B4 = make_float4(__double2float_rn(2.0 * (px + mid * nx)),
                               __double2float_rn(2.0 * (py + mid * ny)),
                               __double2float_rn(2.0 * (pz + mid * nz)), __double2float_rd(-Qt));
            }
            mm = m;
          } else {
            atomicOr(&p.err_flags[0], 1);
            mm = -(m + 2);  // image written as zeros
          }
        }
        sA[slot] = A4;
        sB[slot] = B4;
        sP[slot] = P4;
        sN[slot] = N4;
        sM[slot] = mm;
      }
      for (int i = tid; i < GL * IS; i += NT) sImg[i] = 0u;
      int nrows = 0;
      if (PRUNE == 1) {
        __syncthreads();
        // bounding box of the live centres, grown by R (rounded outward)
        if (warp == 0) {
          float lo[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
          bool live = false;
          for (int sl = lane; sl < G; sl += 32) {
            if (sM[sl] >= 0) {
              const float4 P4 = sP[sl];
              live = true;
              lo[0] = fminf(lo[0], P4.x); lo[1] = fminf(lo[1], P4.y); lo[2] = fminf(lo[2], P4.z);
              hi3[0] = fmaxf(hi3[0], P4.x); hi3[1] = fmaxf(hi3[1], P4.y); hi3[2] = fmaxf(hi3[2], P4.z);
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
              hi3[a] = fmaxf(hi3[a], __shfl_xor_sync(0xffffffffu, hi3[a], o));
            }
          }
          const int anyl = __any_sync(0xffffffffu, live);
          if (lane == 0) {
            s_live = anyl;
            if (anyl) {
              s_rng[0] = cell_coord(__fsub_rd(lo[0], p.R_up), p.ox, p.inv_h, p.dimx);
              s_rng[1] = cell_coord(__fadd_ru(hi3[0], p.R_up), p.ox, p.inv_h, p.dimx);
              s_rng[2] = cell_coord(__fsub_rd(lo[1], p.R_up), p.oy, p.inv_h, p.dimy);
              s_rng[3] = cell_coord(__fadd_ru(hi3[1], p.R_up), p.oy, p.inv_h, p.dimy);
              s_rng[4] = cell_coord(__fsub_rd(lo[2], p.R_up), p.oz, p.inv_h, p.dimz);
              s_rng[5] = cell_coord(__fadd_ru(hi3[2], p.R_up), p.oz, p.inv_h, p.dimz);
            }
          }
        }
        __syncthreads();
        if (s_live) nrows = (s_rng[3] - s_rng[2] + 1) * (s_rng[5] - s_rng[4] + 1);
      }
      if (CL > 1) cluster_sync_all();   // both CTAs zeroed their images before any remote add
      else __syncthreads();

      // ---- a8-a10: stream points, pair test, compact, accept
      // Each thread holds KP points in registers for all G centres.  Per batch of CB
      // centres the pass bits go to one u32 mask (bit = k*8 + c) stored in smem; once
      // per tile the warp compacts all its bits into 16-bit entries (mask word, source
      // lane, mask bit) and processes them 32 at a time, reading the point from the
      // warp's staged copy of the tile (no global re-load).
      unsigned qhead = 0, qtail = 0;
      float2 pf[8];            // DEFER: A-fragment pairs of this warp's next tile (prefetched)
      bool have_pf = false;
      uint4 pfr[4];            // FRAGREG: row blocks 0-3 of the next tile's fragments (prefetched)
      bool have_pfr = false;
      constexpr int NWD = G / CB;                      // mask words per lane per tile
      // candidate operands: centre slot gs, point (source lane, k) from the staged tile
      // entry = (mask word w << 10) | (source lane << 5) | mask bit (k << 3 | c)
      // Tiles filtered on the tensor cores (BRUTE, support test not in the hot loop) use
      // the mma layout: mask word w = column block cb of lane L holds bit (j << 3) | rb for
      // output j of the HMMA of row block rb: centre slot (2(L&3) + (j&1)) * NCB + cb
      // and row r = (L>>2) + 8(j>>1) of row block rb, staged at lane (rb&3)*8 + ((r+rb)&7),
      // point (rb>>2)*2 + (r>>3).  (Slots and rows are spread so that one lane's
      // candidates read different shared-memory banks in the accept passes.)
      bool tile_mma = false;
      // CELLS (CL2: component-major staged tile, entries with the centre slot in bits 0-4 and
      // the point lane * 4 + k in bits 5-11): see stage() and enc_entry below
      // (groups of 8, 16 or 32 centres: a 5-bit centre slot, 8 centres per mask word)
      constexpr bool CL2 = PRUNE == 1 && SPIN_CELLS_LAYOUT2 && G <= 32 && CB == 8;
      // CL2: shared-window addresses of the centre constants, the warp's staged tile, its ring
      // and the images, opaque to the compiler (which otherwise rematerialises the window base
      // -- an S2R and its dependants -- and the warp offset in every accept pass)
      unsigned pin_c = 0u, pin_t = 0u, pin_q = 0u;
      if (CL2 && SPIN_CELLS_PIN) {
        pin_c = (unsigned)__cvta_generic_to_shared(sP);
        pin_t = (unsigned)__cvta_generic_to_shared(sT);
        pin_q = (unsigned)__cvta_generic_to_shared(sQ);
        asm volatile("mov.u32 %0, %0;" : "+r"(pin_c));
        asm volatile("mov.u32 %0, %0;" : "+r"(pin_t));
        asm volatile("mov.u32 %0, %0;" : "+r"(pin_q));
      }
      auto lds_f4 = [](unsigned a) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
        return v;
      };
      auto lds_f = [](unsigned a) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
        return v;
      };
      auto load_q = [&](unsigned i) -> unsigned {   // ring / queue entry i of this warp
        if (CL2 && SPIN_CELLS_PIN) {
          unsigned short v;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(pin_q + 2u * i));
          return (unsigned)v;
        }
        return (unsigned)sQ[i];
      };
      auto decode_entry = [&](unsigned e, int& gs, int& sl, int& kk) {
        if (CL2) {
          gs = (int)(e & 31u);
          sl = (int)(e >> 7);
          kk = (int)(e >> 5) & 3;
        } else if (MMA_FILTER && tile_mma) {
          const int bit = (int)(e & 31u), ln = (int)(e >> 5) & 31;
          const int cbk = (int)(e >> 10), rb = bit & 7, jv = bit >> 3;
          gs = (2 * (ln & 3) + (jv & 1)) * NCB + cbk;
          const int r = (ln >> 2) + 8 * (jv >> 1);
          sl = (rb & 3) * 8 + ((r + rb) & 7);
          kk = (rb >> 2) * 2 + (r >> 3);
        } else {
          gs = (int)(e >> 10) * CB + (int)(e & 7u);
          sl = (int)(e >> 5) & 31;    // source lane
          kk = (int)(e >> 3) & 3;     // point k of that lane
        }
      };
      auto load_entry = [&](unsigned e, int& gs, float4& P4, float4& N4, float4& X4, float4& NX4) {
        if (CL2) {
          // component c of point (lane sl, k) at float c * 128 + sl * 4 + k = c * 128 + (e >> 5)
          gs = (int)(e & 31u);
          if (SPIN_CELLS_PIN) {
            const unsigned ca = pin_c + 16u * (e & 31u), ra = pin_t + ((e >> 3) & 0x1ffcu);
            P4 = lds_f4(ca);
            N4 = lds_f4(ca + (unsigned)(L.oN - L.oP));
            X4 = make_float4(lds_f(ra), lds_f(ra + 512u), lds_f(ra + 1024u), 0.f);
            NX4 = make_float4(lds_f(ra + 2048u), lds_f(ra + 2560u), lds_f(ra + 3072u), 0.f);
            return;
          }
          P4 = sP[gs];
          N4 = sN[gs];
          const float* rec = reinterpret_cast<const float*>(sT) + (e >> 5);
          X4 = make_float4(rec[0], rec[128], rec[256], 0.f);
          NX4 = make_float4(rec[512], rec[640], rec[768], 0.f);
          return;
        }
        int sl, kk;
        decode_entry(e, gs, sl, kk);
        P4 = sP[gs];
        N4 = sN[gs];
        const float* rec = reinterpret_cast<const float*>(sT + (kk >> 1) * 32 + sl) + (kk & 1);
        constexpr int RS = (KP / 2) * 32 * 4;                       // floats between records
        X4 = make_float4(rec[0], rec[2], rec[RS], 0.f);
        NX4 = make_float4(rec[2 * RS], rec[2 * RS + 2], rec[3 * RS], 0.f);
      };
      // CELLS (dense, latency-bound) takes two candidates per lane per pass so that the
      // two independent decisions interleave; BRUTE keeps one (fewer live registers).
      // (CELLS: two per lane for BILINEAR, one for NEAREST, as measured: C3 47.3 vs 48.0 ms,
      // C5 188 vs 191 ms)
      constexpr int APL = PRUNE == 1 ? (MODE == 1 ? SPIN_APL_CELLS : SPIN_APL_CELLS_NEAREST)
                                     : CL > 1 ? SPIN_APL_CL
                                     : (NT == 512 ? SPIN_APL_BRUTE512 : SPIN_APL_BRUTE);
      auto process_pair = [&](unsigned e0, bool v0, unsigned e1, bool v1) {
        float4 P0, N0, X0, NX0, P1, N1, X1, NX1;
        int g0, g1 = 0;
        load_entry(e0, g0, P0, N0, X0, NX0);
        Dec d0 = decide<MODE>(p, P0, N0, X0, NX0);
        Dec d1;
        d1.status = 0;
        if (APL == 2) {
          load_entry(e1, g1, P1, N1, X1, NX1);
          d1 = decide<MODE>(p, P1, N1, X1, NX1);
          if (!v1) d1.status = 0;
        }
        if (!v0) d0.status = 0;
        if (!SPIN_CAND_PER_TILE) ct.cand += (unsigned)v0 + (APL == 2 ? (unsigned)v1 : 0u);
        if (SUP == 2) ct.srej += (unsigned)(v0 & (d0.sup_out != 0));
        if (d0.status == 2) resolve<MODE>(p, d0, P0, N0, X0, NX0, ct);
        if (APL == 2 && d1.status == 2) resolve<MODE>(p, d1, P1, N1, X1, NX1, ct);
        if (d0.status) {
          ++ct.acc;
          if constexpr (CL > 1) apply_cl<MODE, G, CL>(d0, sImg, IS, g0);
          else if (CL2 && SPIN_CELLS_PIN)
            apply_s<MODE, G>(p, d0, pin_c + (unsigned)(L.oImg - L.oP) + 4u * (unsigned)(g0 * IS), g0, &s_carry);
          else apply<MODE, G>(p, d0, sImg + g0 * IS, g0, &s_carry);
        }
        if (APL == 2 && d1.status) {
          ++ct.acc;
          if constexpr (CL > 1) apply_cl<MODE, G, CL>(d1, sImg, IS, g1);
          else if (CL2 && SPIN_CELLS_PIN)
            apply_s<MODE, G>(p, d1, pin_c + (unsigned)(L.oImg - L.oP) + 4u * (unsigned)(g1 * IS), g1, &s_carry);
          else apply<MODE, G>(p, d1, sImg + g1 * IS, g1, &s_carry);
        }
      };
      // Dense tensor-core tiles (BRUTE, one-CTA workers; DESIGN.md 7.1 "dense tiles"): with
      // the cloud and the centres in Morton order a group's candidates fill few warp tiles,
      // and those densely.  There lane l takes centre slot l (+ 32 s) and the warp walks the
      // tile's live points (those with any candidate), reading each point once by broadcast:
      // no entries to write or decode, one image per lane (no same-address atomics), and
      // each lane tests its own pair's bit in the mma-layout mask.  Used when the tile holds
      // at least dense_min candidates per live point, else the compaction path.
      constexpr bool DENSE = PRUNE == 0 && CL == 1 && MMA_FILTER;
      auto run_dense = [&](unsigned mor, int mcnt, int chunk, bool phase2) -> bool {
        const int total = __reduce_add_sync(0xffffffffu, mcnt);
        if (total == 0) return false;
        // live rows: OR over this lane's column blocks, then over the 4 lanes of a row group
        // (tig), then over the centre parity j & 1: bit half * 8 + rb = row gid + 8 half of
        // row block rb
        unsigned v = mor | __shfl_xor_sync(0xffffffffu, mor, 1);
        v |= __shfl_xor_sync(0xffffffffu, v, 2);
        v |= v >> 8;
        const unsigned v16 = (v & 0xffu) | ((v >> 8) & 0xff00u);
        unsigned lw[4];
        int live = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {   // word i: row groups 2i (low half) and 2i + 1
          lw[i] = __shfl_sync(0xffffffffu, v16, 8 * i) | (__shfl_sync(0xffffffffu, v16, 8 * i + 4) << 16);
          live += __popc(lw[i]);
        }
        // (a step costs one decision per centre slot of the lane: the threshold scales with
        // GS; measured C2 (G = 64): 8 per slot 3.29 ms, 16: 3.24 ms)
        if ((PASS1 || !phase2) && total < live * p.dense_min * ((G + 31) / 32)) return false;
        if (DQ && !PASS1 && !phase2) {
          // the group's dense tiles are few and land on few warps (the cloud is Morton
          // ordered): queue the tile for the CTA-wide second phase, where every warp takes
          // queued tiles until none are left (inline when the queue is full)
          int slot = 0;
          if (lane == 0) slot = atomicAdd(&s_dq_n, 1);
          slot = __shfl_sync(0xffffffffu, slot, 0);
          if (slot < DQ_CAP) {
            if (lane == 0) s_dq[slot] = chunk;
            return true;
          }
        }
        if (lane == 0) {
          ++dense_tiles;
          dense_rows += (unsigned)live;
          ct.cand += (unsigned)total;   // the tile's filter candidates (mask bits)
        }
        if (skip_accept) return true;
        // no per-pair mask bit: decide() is exact on its own, and a pair the filter rejected
        // is either certainly far (status 0) or decided like any candidate
        constexpr int GS = (G + 31) / 32;
        constexpr int RS = (KP / 2) * 32 * 4;   // floats between staged records
        const float* sTf = reinterpret_cast<const float*>(sT);
        float4 cP[GS], cN[GS];
        unsigned glive = 0u;   // bit s: slot lane + 32 s holds a live centre
#pragma unroll
        for (int s = 0; s < GS; ++s) {
          const int g = min(lane + 32 * s, G - 1);
          cP[s] = sP[g];
          cN[s] = sN[g];
          glive |= (unsigned)(lane + 32 * s < G && sM[g] >= 0) << s;
        }
        unsigned img0 = (unsigned)__cvta_generic_to_shared(sImg);
        // (opaque to the compiler, which otherwise rematerialises the shared-window base --
        // an S2R and four dependent instructions -- inside the row loop)
        if (SPIN_PIN_IMG) asm volatile("mov.u32 %0, %0;" : "+r"(img0));
        // live rows by bit scan, two per step where the word holds two (two independent
        // decisions in flight; 768-thread CTAs, with 80 registers, one).  (A row list in the
        // entry ring measured slower: C4 NEAREST 243 -> 276 ms)
        // (NEAREST on the 512-thread launch takes two: C4 NEAREST 213.2 -> 209.8 ms; BILINEAR, with its
        // longer splat, 245.2 -> 246.3 ms and keeps one)
        constexpr int DR = NT <= 512 ? (SPIN_DENSE_ROWS == 1 && MODE == 0 ? 2 : SPIN_DENSE_ROWS) : 1;
        unsigned w0 = lw[0], w1 = lw[1], w2 = lw[2], w3 = lw[3];
        auto row_point = [&](int i, int bq, float4& X4, float4& NX4) {
          const int gid = 2 * i + (bq >> 4), half = (bq >> 3) & 1, rb = bq & 7;
          const int r = gid + 8 * half;
          const int sl = (rb & 3) * 8 + ((r + rb) & 7);
          const float* rec = sTf + ((rb >> 2) * 32 + sl) * 4 + half;
          X4 = make_float4(rec[0], rec[2], rec[RS], 0.f);
          NX4 = make_float4(rec[2 * RS], rec[2 * RS + 2], rec[3 * RS], 0.f);
        };
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          unsigned wv = w0;
          w0 = w1;
          w1 = w2;
          w2 = w3;
          while (wv) {
            const int ba = __ffs(wv) - 1;
            wv &= wv - 1u;
            const bool two = DR == 2 && wv != 0u;
            const int bb = two ? __ffs(wv) - 1 : ba;
            if (two) wv &= wv - 1u;
            float4 Xa, NXa, Xb, NXb;
            row_point(i, ba, Xa, NXa);
            if (DR == 2) row_point(i, bb, Xb, NXb);
#pragma unroll
            for (int s = 0; s < GS; ++s) {
              const int g = lane + 32 * s;
              const bool gl = (glive >> s) & 1u;
              Dec da = decide<MODE>(p, cP[s], cN[s], Xa, NXa);
              Dec db;
              if (DR == 2) db = decide<MODE>(p, cP[s], cN[s], Xb, NXb);
              else db.status = 0, db.far = 1, db.sup_out = 0;
              if (!gl || da.far) da.status = 0;
              if (!gl || db.far || !two) db.status = 0;
              if (SUP == 2) ct.srej += (unsigned)(da.sup_out & (da.far == 0) & (int)gl) +
                                       (unsigned)(db.sup_out & (db.far == 0) & (int)gl & (int)two);
              if (da.status == 2) resolve<MODE>(p, da, cP[s], cN[s], Xa, NXa, ct);
              if (DR == 2 && db.status == 2) resolve<MODE>(p, db, cP[s], cN[s], Xb, NXb, ct);
              const unsigned ia = img0 + 4u * (unsigned)(g * IS);
              if (da.status) {
                ++ct.acc;
                apply_s<MODE, G>(p, da, ia, g, &s_carry);
              }
              if (DR == 2 && db.status) {
                ++ct.acc;
                apply_s<MODE, G>(p, db, ia, g, &s_carry);
              }
            }
          }
        }
        return true;
      };
      // entry of mask bit `raw` (= k * 8 + c) of this lane's mask word w.  CL2: centre slot
      // w * 8 + c | (lane * 4 + k) << 5 = base + raw + 24 k; else (w, lane, raw) fields
      auto enc_base = [&](unsigned w) -> unsigned {
        return CL2 ? (w << 3) | ((unsigned)lane << 7) : (w << 10) | ((unsigned)lane << 5);
      };
      auto enc_entry = [&](unsigned eb, unsigned raw) -> unsigned {
        return CL2 ? eb + raw + 3u * (raw & 0x18u) : eb | raw;
      };
      // entries of mask words [w0, w1) of the tile: cnt = this lane's bits in them, x = the
      // inclusive lane prefix of cnt, total = the warp's
      auto compact_range = [&](const int w0, const int w1, const int cnt, const int x, const int total) {
        unsigned wm = 0u;   // this lane's nonzero mask words (BRUTE flat loop)
        if (PRUNE == 0) {
#pragma unroll
          for (int w = 0; w < NWD; ++w) wm |= (unsigned)(sMask[w * 32 + lane] != 0u) << w;
        }
        if (total == 0) return;
        if (SPIN_CAND_PER_TILE) ct.cand += (unsigned)cnt;   // (this lane's share of the tile's candidates)
        qhead = qtail = 0u;   // the ring is empty between tiles
        // common case: the whole tile fits the ring and one scan places every entry;
        // dense tiles go CHB bits of a mask word (<= 32 * CHB entries) at a time, each
        // appended after the ring was drained to < 64 pending entries.
        constexpr int CHB = QCAP >= 64 + 512 ? 16 : QCAP >= 64 + 256 ? 8 : 4;
        static_assert(QCAP >= 64 + 32 * CHB, "ring too small for the dense path");
        const bool dense = total > QCAP - 64;
        const int nchunks = dense ? (32 / CHB) * w1 : (32 / CHB) * w0 + 1;
        for (int ci = (32 / CHB) * w0;;) {
          if (ci < nchunks) {
            if (!dense) {
              // no wrap: total <= QCAP - 64 entries from slot 0
              uint16_t* q = sQ + (x - cnt);
              if (PRUNE == 0) {
                // sparse (BRUTE, ~0.7 bits per lane word): one flat loop over this lane's
                // set bits, so the warp trip count is the largest per-lane count, not the
                // sum over words of per-word maxima
                unsigned m = 0u, eb = 0u;
                for (int left = cnt; left > 0; --left) {
                  if (m == 0u) {                  // next nonzero word of this lane
                    const unsigned w = msb(wm);
                    wm ^= 1u << w;
                    m = sMask[w * 32 + lane];
                    eb = (w << 10) | ((unsigned)lane << 5);
                  }
                  const unsigned bit = msb(m);    // highest set bit (one FLO)
                  m ^= 1u << bit;
                  *q++ = (uint16_t)(eb | bit);
                }
              } else {
                // dense (CELLS): word by word
#pragma unroll 1
                for (int w = w0; w < w1; ++w) {
                  unsigned m = sMask[w * 32 + lane];
                  const unsigned eb = enc_base((unsigned)w);
                  while (m) {
                    const unsigned bit = msb(m);
                    m ^= 1u << bit;
                    *q++ = (uint16_t)enc_entry(eb, bit);
                  }
                }
              }
              qtail = (unsigned)total;
              // every entry of the tile sits at slots 0 .. total-1: plain passes of 32 x APL
              {
                __syncwarp();
                if (skip_accept) return;
                constexpr int PASS = 32 * APL;
                for (int base = 0; base < total; base += PASS) {
                  const int i0 = base + lane;
                  const bool v0 = i0 < total, v1 = APL == 2 && i0 + 32 < total;
                  const unsigned e0 = v0 ? load_q((unsigned)i0) : 0u;
                  const unsigned e1 = v1 ? load_q((unsigned)i0 + 32u) : 0u;
                  if (v0) process_pair(e0, v0, e1, v1);
                }
                return;
              }
            } else {
              constexpr int CPW = 32 / CHB;               // chunks per mask word
              const int sub = ci % CPW;
              if (PRUNE == 1 && CPW > 1 && sub == 0) {
                // a whole mask word that fits the ring goes in one scan
                unsigned mw = sMask[(ci / CPW) * 32 + lane];
                const int cw = __popc(mw);
                int xw = cw;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const int y = __shfl_up_sync(0xffffffffu, xw, o);
                  if (lane >= o) xw += y;
                }
                const int tw = __shfl_sync(0xffffffffu, xw, 31);
                if (tw <= QCAP - 64) {
                  unsigned pos = qtail + (unsigned)(xw - cw);
                  const unsigned eb = enc_base((unsigned)(ci / CPW));
                  while (mw) {
                    const unsigned bit = msb(mw);
                    mw ^= 1u << bit;
                    sQ[pos & (QCAP - 1)] = (uint16_t)enc_entry(eb, bit);
                    ++pos;
                  }
                  qtail += (unsigned)tw;
                  ci += CPW;
                  goto appended;
                }
              }
              {
              unsigned m = (sMask[(ci / CPW) * 32 + lane] >> (CHB * sub)) & ((1u << CHB) - 1u);
              const int c2 = __popc(m);
              int x2 = c2;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x2, o);
                if (lane >= o) x2 += y;
              }
              const int t2 = __shfl_sync(0xffffffffu, x2, 31);
              unsigned pos = qtail + (unsigned)(x2 - c2);
              // entry = (word, lane, raw mask bit CHB * sub + b)
              const unsigned eb = enc_base((unsigned)(ci / CPW));
              while (m) {
                const unsigned bit = msb(m);
                m ^= 1u << bit;
                sQ[pos & (QCAP - 1)] = (uint16_t)enc_entry(eb, (unsigned)(CHB * sub) + bit);
                ++pos;
              }
              qtail += (unsigned)t2;
              }
              ++ci;
            }
          appended:;
          }
          const bool more = ci < nchunks;
          __syncwarp();
          for (;;) {
            const unsigned avail = qtail - qhead;
            constexpr unsigned PASS = 32u * APL;
            if (avail == 0u || (avail < PASS && more)) break;
            const unsigned n = min(PASS, avail);
            const bool v0 = (unsigned)lane < n, v1 = APL == 2 && (unsigned)lane + 32u < n;
            const unsigned e0 = load_q((qhead + lane) & (QCAP - 1));
            const unsigned e1 = APL == 2 ? load_q((qhead + 32u + lane) & (QCAP - 1)) : 0u;
            __syncwarp();
            qhead += n;
            if (v0 && !skip_accept) process_pair(v0 ? e0 : 0u, v0, v1 ? e1 : 0u, v1);
          }
          if (!more) break;
        }
      };
      // CELLS tiles (20% of the pairs are candidates; a tile of 4096 pairs often exceeds the
      // ring): a tile whose entries do not fit the ring is compacted and accepted in two
      // halves of its mask words, each placed by ONE scan from slot 0 (the two halves' counts
      // share the scan, 16 bits each), instead of the chunked ring path per mask word
      constexpr bool HALVES = PRUNE == 1 && (SPIN_CELLS_HALVES == 2 || (SPIN_CELLS_HALVES == 1 && MODE == 0)) && NWD >= 2 && NWD % 2 == 0;
      auto compact_and_accept = [&]() {
        unsigned cnt = 0u;
#pragma unroll
        for (int w = 0; w < NWD; ++w)
          cnt += (unsigned)__popc(sMask[w * 32 + lane]) << (HALVES && w >= NWD / 2 ? 16 : 0);
        unsigned x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, x, 31);
        if (tot == 0u) return;
        const int total = HALVES ? (int)(tot & 0xffffu) + (int)(tot >> 16) : (int)tot;
        const bool split = HALVES && total > QCAP - 64;
        // (one call site: the accept passes are inlined once)
#pragma unroll 1
        for (int hh = 0; hh < (split ? 2 : 1); ++hh) {
          const int sh = 16 * hh;
          const int w0 = split ? hh * (NWD / 2) : 0, w1 = split ? w0 + NWD / 2 : NWD;
          const int c = split ? (int)((cnt >> sh) & 0xffffu)
                              : HALVES ? (int)(cnt & 0xffffu) + (int)(cnt >> 16) : (int)cnt;
          const int xx = split ? (int)((x >> sh) & 0xffffu)
                               : HALVES ? (int)(x & 0xffffu) + (int)(x >> 16) : (int)x;
          const int tt = split ? (int)((tot >> sh) & 0xffffu) : total;
          if (hh) __syncwarp();   // the first half's entries were read before they are overwritten
          compact_range(w0, w1, c, xx, tt);
        }
      };
      // the 8-byte A-fragment pair of row block rb of thread (gid, tig) within a 128-point
      // chunk in pair layout (the same offset in the staged tile and in tpos)
      auto frag_off = [&](int rb) {
        const int gid = lane >> 2, tig = lane & 3;
        const int sl = (rb & 3) * 8 + ((gid + rb) & 7);
        return (((tig >> 1) * (KP / 2) + (rb >> 2)) * 32 + sl) * 4 + 2 * (tig & 1);
      };
      auto load_frags = [&](float2 (&dst)[8], int chunk) {
        const float* src = reinterpret_cast<const float*>(p.tpos) + (size_t)chunk * 1024;
#pragma unroll
        for (int rb = 0; rb < 8; ++rb) {
          float2 v;
          asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
                       : "=f"(v.x), "=f"(v.y) : "l"(src + frag_off(rb)));
          dst[rb] = v;
        }
      };
      auto run_tile = [&](const int (&j)[KP], int next_chunk, bool phase2) {
        // stage the tile in pair layout (the accept path's copy and the packed-fp32 filter's
        // operands), read back so each f32x2 operand arrives as an aligned register pair
        f2 X2[KP / 2], Y2[KP / 2], Z2[KP / 2], NXX2[KP / 2], NX2[KP / 2], NY2[KP / 2], NZ2[KP / 2];
        // CELLS cull: centre slots whose region can reach this warp tile's bounding box
        constexpr bool CULL = CL2 && SPIN_CELLS_CULL;
        unsigned act = 0xffffffffu;
        // the tile's precomputed tf32 A fragments (FRAG): 4 KB, one uint4 per (row block, lane)
        auto stage_frag = [&]() {
          if (SPIN_EXP_ABL & 2) return;
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(sT, p.mfrag + (size_t)(j[0] >> 7) * 256, SPIN_EXP_FRAG_BYTES, &s_tile_bar[warp]);
          }
          mbar_wait(&s_tile_bar[warp], tile_phase);
          tile_phase ^= 1u;
        };
        auto stage = [&]() {
          if (TMA_TILE) {
            // the warp's 128 points, already in staging layout in HBM (tpos): one bulk copy
            // into the warp's staged tile; prior generic reads of the buffer are ordered
            // before the async-proxy write by the proxy fence
            if (lane == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              bulk_load(sT, p.tpos + (size_t)(j[0] >> 7) * 256, 4096u, &s_tile_bar[warp]);
            }
            if (SPIN_TMA_WAIT_ALL || lane == 0) mbar_wait(&s_tile_bar[warp], tile_phase);
            if (!SPIN_TMA_WAIT_ALL) __syncwarp();   // lane 0 acquired the phase; the warp barrier orders the rest
            tile_phase ^= 1u;
          }
          if (CL2) {
            // component-major: float4 c of lane l = component c of the lane's four points
            // (x, y, z, -|x|^2, nx, ny, nz): the packed-fp32 operands of point pairs (0,1) and
            // (2,3) are its two halves, and an accept-path operand sits at c * 128 + l * 4 + k
            float4 a[KP], b[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              a[k] = __ldg(&p.pos[j[k]]);
              b[k] = __ldg(&p.nrm[j[k]]);
            }
            sT[0 * 32 + lane] = make_float4(a[0].x, a[1].x, a[2].x, a[3].x);
            sT[1 * 32 + lane] = make_float4(a[0].y, a[1].y, a[2].y, a[3].y);
            sT[2 * 32 + lane] = make_float4(a[0].z, a[1].z, a[2].z, a[3].z);
            sT[3 * 32 + lane] = make_float4(-a[0].w, -a[1].w, -a[2].w, -a[3].w);
            sT[4 * 32 + lane] = make_float4(b[0].x, b[1].x, b[2].x, b[3].x);
            sT[5 * 32 + lane] = make_float4(b[0].y, b[1].y, b[2].y, b[3].y);
            sT[6 * 32 + lane] = make_float4(b[0].z, b[1].z, b[2].z, b[3].z);
            if (CULL) {
              // bounding box of the tile's points (sentinels excluded), reduced over the warp in
              // the order-preserving integer image of the floats (one REDUX per bound)
              float lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
              for (int k = 0; k < KP; ++k) {
                if (j[k] < p.N) {
                  lo3[0] = fminf(lo3[0], a[k].x); hi3[0] = fmaxf(hi3[0], a[k].x);
                  lo3[1] = fminf(lo3[1], a[k].y); hi3[1] = fmaxf(hi3[1], a[k].y);
                  lo3[2] = fminf(lo3[2], a[k].z); hi3[2] = fmaxf(hi3[2], a[k].z);
                }
              }
              auto ford = [](float x) { const int i = __float_as_int(x); return i ^ ((i >> 31) & 0x7fffffff); };
              auto finv = [](int i) { return __int_as_float(i ^ ((i >> 31) & 0x7fffffff)); };
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                lo3[c] = finv(__reduce_min_sync(0xffffffffu, ford(lo3[c])));
                hi3[c] = finv(__reduce_max_sync(0xffffffffu, ford(hi3[c])));
              }
              // lane = centre slot: every point X of the box has a_i <= X_i - P_i <= b_i, so
              // |X - P|^2 >= sum max(0, a_i, -b_i)^2 and n.(X - P) lies in [bmin, bmax]; the region
              // needs |X - P| <= R and |n.(X - P) - mid| <= h (h_test also covers the hot filter's
              // rounding; sl the rounding here: <= 4u of the summed magnitudes)
              bool may = false;
              if (lane < G) {
                const float4 P4 = sP[lane], N4 = sN[lane];
                const float ax = lo3[0] - P4.x, bx = hi3[0] - P4.x, ay = lo3[1] - P4.y, by = hi3[1] - P4.y;
                const float az = lo3[2] - P4.z, bz = hi3[2] - P4.z;
                const float dx = fmaxf(0.f, fmaxf(ax, -bx)), dy = fmaxf(0.f, fmaxf(ay, -by));
                const float dz = fmaxf(0.f, fmaxf(az, -bz));
                const float dist2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const float bmin = fminf(N4.x * ax, N4.x * bx) + fminf(N4.y * ay, N4.y * by) + fminf(N4.z * az, N4.z * bz);
                const float bmax = fmaxf(N4.x * ax, N4.x * bx) + fmaxf(N4.y * ay, N4.y * by) + fmaxf(N4.z * az, N4.z * bz);
                const float sl = 2e-6f * (fabsf(ax) + fabsf(bx) + fabsf(ay) + fabsf(by) + fabsf(az) + fabsf(bz)) +
                                 1e-5f * p.h_test + 1e-30f;
                const float midf = (float)p.mid, hs = p.h_test + sl;
                may = sM[lane] >= 0 && dist2 * 0.99999f <= p.R_up * p.R_up * 1.00001f &&
                      bmin - midf <= hs && bmax - midf >= -hs;
              }
              act = __ballot_sync(0xffffffffu, may);
            }
          }
#pragma unroll
          for (int k = 0; !TMA_TILE && !CL2 && k < KP; k += 2) {
            const float4 a0 = __ldg(&p.pos[j[k]]), a1 = __ldg(&p.pos[j[k + 1]]);
            const float4 b0 = __ldg(&p.nrm[j[k]]), b1 = __ldg(&p.nrm[j[k + 1]]);
            const int pr = k / 2;
            sT[(0 * (KP / 2) + pr) * 32 + lane] = make_float4(a0.x, a1.x, a0.y, a1.y);
            sT[(1 * (KP / 2) + pr) * 32 + lane] = make_float4(a0.z, a1.z, -a0.w, -a1.w);
            sT[(2 * (KP / 2) + pr) * 32 + lane] = make_float4(b0.x, b1.x, b0.y, b1.y);
            sT[(3 * (KP / 2) + pr) * 32 + lane] = make_float4(b0.z, b1.z, 0.f, 0.f);
          }
          __syncwarp();
        };
        const bool sup_hot = SUP == 1 || (SUP == 2 && sup_on);
        tile_mma = MMA_FILTER && p.mma && (!sup_hot || phase2);   // (queued tiles were mma tiles)
        // tensor-core tiles read their A fragments from registers loaded straight from tpos
        // one tile ahead (software pipeline), and stage the tile in shared memory only when
        // the pre-pass finds a candidate (most tiles of a group hold none); other tiles
        // stage first
        // (512-thread CTAs, whose 128 registers per thread hold the prefetch; 768-thread CTAs
        // stage every tile: SPIN_DEFER_STAGE = 2 defers there too, loading A from tpos
        // without the prefetch, which spills)
        // (measured, C4: NEAREST 246.7 -> 242.8 ms deferred, BILINEAR 275.0 -> 279.4 ms: NEAREST only)
        // FRAG: tensor-core tiles stage their precomputed A fragments (split hi/lo once at
        // load time: 8 LDS.128 per tile instead of 8 LDS.64 and ~70 ALU / FMA operations) and
        // the points only once the pre-pass found a candidate
        constexpr bool FRAG = PRUNE == 0 && MMA_FILTER && TMA_TILE && SPIN_FRAG_TILE;
        constexpr bool DEFER = !FRAG && PRUNE == 0 && MMA_FILTER && TMA_TILE &&
                               (SPIN_DEFER_STAGE == 2 || (SPIN_DEFER_STAGE == 1 && NT <= 512 && MODE == 0));
        constexpr bool PREFETCH = DEFER && NT <= 512;
        // FRAGREG: the fragments go from L2 to registers, row blocks 0-3 prefetched during the
        // previous tile and 4-7 during this tile's first HMMAs; the warp never waits for a whole
        // 4 KB copy, and shared memory is touched only by tiles with a candidate (their points)
        constexpr bool FRAGREG = FRAG && SPIN_FRAG_REG && NT <= 512 && !PASS1 && SPIN_EXP_FRAG_BYTES == 4096u;
        static_assert(!FRAGREG || SPIN_FILTER_PREPASS, "FRAGREG loads its fragments in the pre-pass");
        const bool fragreg = FRAGREG && tile_mma && !phase2;
        uint4 fa[4], fb[4];
        auto ldfrag4 = [&](uint4 (&dst)[4], int chunk, int half) {
          const uint4* src = reinterpret_cast<const uint4*>(p.mfrag) + (size_t)chunk * 256 + half * 128 + lane;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(dst[i].x), "=r"(dst[i].y), "=r"(dst[i].z), "=r"(dst[i].w) : "l"(src + i * 32));
        };
        if (fragreg) {
        } else if (FRAG && tile_mma) stage_frag();
        else if (!(DEFER && tile_mma) || phase2) stage();
        if (PREFETCH && !tile_mma) have_pf = false;   // (a packed-fp32 tile consumes no prefetch)
        if (FRAGREG && !fragreg) have_pfr = false;
        unsigned dense_or = 0u;   // mma tiles: OR and popcount of this lane's mask words
        int dense_cnt = 0;
        bool tile_empty = false;  // mma tiles: the pre-pass found no candidate (masks not written)
        if (tile_mma) {
          // sphere margins m = B.x - |x|^2 + K of 16 points x 8 centres per HMMA:
          // A = the points as (x, y, z, -|x|^2) split into tf32 hi and lo parts (columns
          // 0-3 and 4-7; x = hi + lo + O(2^-22 |x|)), B = (Bx, By, Bz, 1) twice (B is tf32
          // exactly), and K.  The planner's E bounds the tf32 / accumulation error, so
          // every pair of the region still has m > 0.
          const int gid = lane >> 2, tig = lane & 3;
          // A = 16 points x 8: (x_hi, y_hi, z_hi, w_hi, x_lo, y_lo, z_lo, 1), w = -|x|^2;
          // B = 8 centres x 8: (Bx, By, Bz, 1, Bx, By, Bz, K) (B and K tf32 exactly), so
          // D = B.(x_hi + x_lo) + w_hi + K with no accumulator input.  Thread (gid, tig)
          // supplies component tig of rows gid and gid + 8 (records r0 {x,x',y,y'},
          // r1 {z,z',-|x|^2,-|x'|^2} of the staged pair layout; see decode_entry).
          // hi = round to nearest tf32 (half an ulp of the 10-bit mantissa added, low 13
          // bits cleared; every |value| here is below 2^101), lo = x - hi (exact) cut to
          // tf32: |x - hi - lo| <= 2^-21 |x|, |w - w_hi| <= 2^-11 |w| (planner's E_mma).
          // (w split hi/lo with K through the accumulator input -- a 2^-21 |w| bound, 3%
          // fewer candidates -- measured slower: the {K, K', K, K'} accumulator quads cost
          // registers and moves per HMMA, C4 275 -> 299 ms, NEAREST 243 -> 289 ms)
          const float* sTf = reinterpret_cast<const float*>(sT);
          // B fragments of the group's centres (column gid = centre slot gid*NCB + cb,
          // rows tig and tig + 4)
          unsigned bu0[NCB], bu1[NCB];
          const float* sBf = reinterpret_cast<const float*>(sB);
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) {
            const int sb = gid * NCB + cb;
            float b1 = sBf[(G >= 8 || sb < G ? sb : 0) * 4 + tig];
            float b0 = tig == 3 ? 1.0f : b1;
            if (G < 8 && sb >= G) {   // no such centre: margin -inf
              b0 = 0.0f;
              b1 = tig == 3 ? -INFINITY : 0.0f;
            }
            bu0[cb] = __float_as_uint(b0);
            bu1[cb] = __float_as_uint(b1);
          }
          // A fragment of row block rb: rows gid and gid + 8 at staged lane
          // (rb&3)*8 + ((gid+rb)&7), points (rb>>2)*2 + 0 / 1 = the two halves of one pair
          // record (adjacent floats) -- from the staged tile, or (DEFER) from registers
          // holding the same 8 bytes of tpos
          float2 cur[8];
          if (FRAG) {
          } else if (phase2) {
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) cur[rb] = *reinterpret_cast<const float2*>(sTf + frag_off(rb));
          } else if (DEFER && PREFETCH) {
            if (!have_pf) load_frags(pf, j[0] >> 7);
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) cur[rb] = pf[rb];
            have_pf = next_chunk >= 0;
            if (have_pf) load_frags(pf, next_chunk);
          } else if (DEFER) {
            load_frags(cur, j[0] >> 7);
          } else {
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) cur[rb] = *reinterpret_cast<const float2*>(sTf + frag_off(rb));
          }
          auto afrag = [&](int rb, unsigned& h0, unsigned& h1, unsigned& l0, unsigned& l1) {
            if (FRAGREG && fragreg) {
              const uint4 fr = rb < 4 ? fa[rb & 3] : fb[rb & 3];
              h0 = fr.x;
              h1 = fr.y;
              l0 = fr.z;
              l1 = fr.w;
              return;
            }
            if (FRAG) {
              const uint4 fr = reinterpret_cast<const uint4*>(sT)[(SPIN_EXP_FRAG_BYTES < 4096u ? (rb & 3) : rb) * 32 + lane];
              h0 = fr.x;
              h1 = fr.y;
              l0 = fr.z;
              l1 = fr.w;
              return;
            }
            const float v0 = cur[rb].x, v1 = cur[rb].y;
            h0 = (__float_as_uint(v0) + 0x1000u) & 0xffffe000u;
            h1 = (__float_as_uint(v1) + 0x1000u) & 0xffffe000u;
            l0 = tig == 3 ? 0x3f800000u : __float_as_uint(v0 - __uint_as_float(h0)) & 0xffffe000u;
            l1 = tig == 3 ? 0x3f800000u : __float_as_uint(v1 - __uint_as_float(h1)) & 0xffffe000u;
          };
          // pre-pass: every margin of the tile, reduced to "any sign bit clear" by 3-input
          // ANDs (two LOP3 per HMMA instead of the four-instruction sign gather); with the
          // Morton-ordered cloud most tiles hold no candidate for a group and stop here
          bool tile_any = true;
          if (SPIN_FILTER_PREPASS && !phase2) {
            // (one accumulator per column block, for shorter LOP3 chains, measured slower:
            // C4 filter 127 -> 146 ms)
            unsigned andv = 0xffffffffu;
            if (FRAGREG && fragreg) {
              if (!have_pfr) ldfrag4(pfr, j[0] >> 7, 0);
#pragma unroll
              for (int i = 0; i < 4; ++i) fa[i] = pfr[i];
              ldfrag4(fb, j[0] >> 7, 1);
            }
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) {
              if (FRAGREG && fragreg && rb == 4) {   // row blocks 0-3 of the next tile
                have_pfr = next_chunk >= 0;
                if (have_pfr) ldfrag4(pfr, next_chunk, 0);
              }
              unsigned h0, h1, l0, l1;
              afrag(rb, h0, h1, l0, l1);
#pragma unroll
              for (int cb = 0; cb < NCB; ++cb) {
                float d0, d1, d2, d3;
                if (SPIN_EXP_ABL & 1) {
                  d0 = __uint_as_float(h0 ^ bu0[cb]); d1 = __uint_as_float(h1 ^ bu1[cb]);
                  d2 = __uint_as_float(l0 ^ bu0[cb]); d3 = __uint_as_float(l1 ^ bu1[cb]);
                } else {
                  mma_tf32(d0, d1, d2, d3, h0, h1, l0, l1, bu0[cb], bu1[cb], 0.0f, 0.0f);
                }
                if (SPIN_EXP_ABL & 4) {
                  if (rb == 7 && cb == NCB - 1) andv = __float_as_uint(d0) & __float_as_uint(d1) & __float_as_uint(d2) & __float_as_uint(d3);
                } else {
                  andv &= __float_as_uint(d0) & __float_as_uint(d1);
                  andv &= __float_as_uint(d2) & __float_as_uint(d3);
                }
              }
            }
            tile_any = __any_sync(0xffffffffu, (int)andv >= 0);
            if (SPIN_EXP_ABL & 8) tile_any = false;
          }
          tile_empty = !tile_any;
          if (tile_any) {
          if (DEFER && !phase2) stage();   // the candidates' points for the accept path
          if (FRAGREG && fragreg) {
            // (rare: row blocks 0-3 again, an L2 hit; the prefetch is dropped so that its
            // registers are free during the tile's accept path)
            ldfrag4(fa, j[0] >> 7, 0);
            have_pfr = false;
          }
          unsigned accm[NCB];
#pragma unroll
          for (int w = 0; w < NCB; ++w) accm[w] = 0u;
#pragma unroll
          for (int rb = 0; rb < ((SPIN_EXP_ABL & 64) ? 0 : 8); ++rb) {
            unsigned h0, h1, l0, l1;
            afrag(rb, h0, h1, l0, l1);
            // up to MB products of the row block in flight before their sign gather (all of
            // them for NCB <= 3; NCB = 6 (the cluster's 48 centres) in two batches of three,
            // which keeps the register count within the 768-thread budget)
            constexpr int MB = (CL == 1 || NCB < SPIN_MMA_BATCH) ? NCB : SPIN_MMA_BATCH;
#pragma unroll
            for (int c0 = 0; c0 < NCB; c0 += MB) {
              float d[MB][4];
#pragma unroll
              for (int i = 0; i < MB; ++i)
                if (c0 + i < NCB)
                  mma_tf32(d[i][0], d[i][1], d[i][2], d[i][3], h0, h1, l0, l1, bu0[c0 + i], bu1[c0 + i], 0.0f, 0.0f);
#pragma unroll
              for (int i = 0; i < MB; ++i)
                if (c0 + i < NCB)
                  accm[c0 + i] = accept_bits4(accm[c0 + i], __float_as_uint(d[i][0]), __float_as_uint(d[i][1]),
                                              __float_as_uint(d[i][2]), __float_as_uint(d[i][3]),
                                              0x01010101u << rb);
            }
          }
#pragma unroll
          for (int w = 0; w < NCB; ++w) {
            sMask[w * 32 + lane] = accm[w];
            dense_or |= accm[w];
            dense_cnt += __popc(accm[w]);
          }
          if (FRAG && !(SPIN_EXP_ABL & 32)) {   // the candidates' points for the accept path replace the fragments
            __syncwarp();
            stage();
          }
          }
        } else {
        if (CL2) {
          f2 r[14];
#pragma unroll
          for (int c = 0; c < 7; ++c)
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r[2 * c]), "=l"(r[2 * c + 1])
                         : "r"((unsigned)__cvta_generic_to_shared(sT + c * 32 + lane)));
#pragma unroll
          for (int pr = 0; pr < 2; ++pr) {
            X2[pr] = r[0 + pr]; Y2[pr] = r[2 + pr]; Z2[pr] = r[4 + pr]; NXX2[pr] = r[6 + pr];
            NX2[pr] = r[8 + pr]; NY2[pr] = r[10 + pr]; NZ2[pr] = r[12 + pr];
          }
        }
#pragma unroll
        for (int pr = 0; !CL2 && pr < KP / 2; ++pr) {
          f2 r[8];
          const float4* base = sT + pr * 32 + lane;
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r[0]), "=l"(r[1]) : "r"((unsigned)__cvta_generic_to_shared(base)));
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r[2]), "=l"(r[3]) : "r"((unsigned)__cvta_generic_to_shared(base + (KP / 2) * 32)));
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r[4]), "=l"(r[5]) : "r"((unsigned)__cvta_generic_to_shared(base + 2 * (KP / 2) * 32)));
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r[6]), "=l"(r[7]) : "r"((unsigned)__cvta_generic_to_shared(base + 3 * (KP / 2) * 32)));
          X2[pr] = r[0]; Y2[pr] = r[1]; Z2[pr] = r[2]; NXX2[pr] = r[3];
          NX2[pr] = r[4]; NY2[pr] = r[5]; NZ2[pr] = r[6];
        }
        const float c_test = p.c_test, h_test = p.h_test;
        // a partial group skips its empty batches (their mask words are zero)
        const int cb_end = ((gcount + CB - 1) / CB) * CB;
        for (int cb = cb_end; cb < G; cb += CB) sMask[(cb / CB) * 32 + lane] = 0u;
        // mask bit (k << 3) | c: point k of this lane, centre cb + c; one loop per variant
        // so the variant branch is taken once per tile, not once per batch
        if (PRUNE == 0 && !sup_hot) {
#pragma unroll HOT_UNROLL
          for (int cb = 0; cb < cb_end; cb += CB) {
            unsigned rej = 0u;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
              const float4 B4 = sB[cb + c];
              unsigned mb[KP];
#pragma unroll
              for (int k2 = 0; k2 < KP / 2; ++k2) {
                // sphere margin m = 2c~.x - |x|^2 + K >= 0 for every pair of the region
                // (bounded)
                const f2 m2 = add2(fma2(bc2(B4.x), X2[k2], fma2(bc2(B4.y), Y2[k2],
                                   fma2(bc2(B4.z), Z2[k2], bc2(B4.w)))), NXX2[k2]);
                up2u(m2, mb[2 * k2], mb[2 * k2 + 1]);
              }
              rej = reject_bits4(rej, mb[0], mb[1], mb[2], mb[3], 0x01010101u << c);
            }
            sMask[(cb / CB) * 32 + lane] = ~rej & (0x01010101u * ((1u << CB) - 1u));
          }
        } else if (PRUNE == 0) {
#pragma unroll 1
          for (int cb = 0; cb < cb_end; cb += CB) {
            unsigned mask = 0u;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
              const float4 A4 = sA[cb + c];
              const float4 B4 = sB[cb + c];
#pragma unroll
              for (int k2 = 0; k2 < KP / 2; ++k2) {
                // support n.nx >= c and the sphere margin
                const f2 s2 = fma2(bc2(A4.x), NX2[k2], fma2(bc2(A4.y), NY2[k2], mul2(bc2(A4.z), NZ2[k2])));
                const f2 m2 = add2(fma2(bc2(B4.x), X2[k2], fma2(bc2(B4.y), Y2[k2],
                                   fma2(bc2(B4.z), Z2[k2], bc2(B4.w)))), NXX2[k2]);
                float s0, s1, q0, q1;
                up2(s2, s0, s1);
                up2(m2, q0, q1);
                mask = pair_bit_sm(mask, s0, c_test, q0, 1u << ((2 * k2) * 8 + c));
                mask = pair_bit_sm(mask, s1, c_test, q1, 1u << ((2 * k2 + 1) * 8 + c));
              }
            }
            sMask[(cb / CB) * 32 + lane] = mask;
          }
        } else {
#pragma unroll 1
          for (int cb = 0; cb < cb_end; cb += CB) {
            if (SPIN_CULL_DIAG && lane == 0) ++dense_rows;
            if (CULL && ((act >> cb) & ((1u << CB) - 1u)) == 0u) {   // no centre of the batch reaches the tile
              if (SPIN_CULL_DIAG && lane == 0) ++dense_tiles;
              sMask[(cb / CB) * 32 + lane] = 0u;
              continue;
            }
            unsigned mask = 0u;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
              const float4 A4 = sA[cb + c];
              const float4 B4 = sB[cb + c];
#pragma unroll
              for (int k2 = 0; k2 < KP / 2; ++k2) {
                // support n.nx; beta'' = n.x - n.p - mid;
                // -q'' = beta''^2 + 2(p + mid n).x - |x|^2 = C - q
                f2 s2 = 0ull;
                if (SUP) s2 = fma2(bc2(A4.x), NX2[k2], fma2(bc2(A4.y), NY2[k2], mul2(bc2(A4.z), NZ2[k2])));
                const f2 be2 = fma2(bc2(A4.x), X2[k2], fma2(bc2(A4.y), Y2[k2], fma2(bc2(A4.z), Z2[k2], bc2(A4.w))));
                const f2 tn2 = fma2(bc2(B4.x), X2[k2], fma2(bc2(B4.y), Y2[k2], fma2(bc2(B4.z), Z2[k2], NXX2[k2])));
                const f2 qn2 = fma2(be2, be2, tn2);
                float s0, s1, b0, b1, q0, q1;
                up2(s2, s0, s1);
                up2(be2, b0, b1);
                up2(qn2, q0, q1);
                const unsigned bit0 = 1u << ((2 * k2) * 8 + c), bit1 = 1u << ((2 * k2 + 1) * 8 + c);
                if (SUP) {
                  mask = pair_bit_n(mask, s0, c_test, fabsf(b0), h_test, q0, B4.w, bit0);
                  mask = pair_bit_n(mask, s1, c_test, fabsf(b1), h_test, q1, B4.w, bit1);
                } else {
                  mask = pair_bit_r(mask, fabsf(b0), h_test, q0, B4.w, bit0);
                  mask = pair_bit_r(mask, fabsf(b1), h_test, q1, B4.w, bit1);
                }
              }
            }
            sMask[(cb / CB) * 32 + lane] = mask;
          }
        }
        }
        __syncwarp();
        bool done = tile_empty;
        if constexpr (DENSE) {
          if (!done && tile_mma && p.dense_min > 0 && p.debug_skip < 2)
            done = run_dense(dense_or, dense_cnt, j[0] >> 7, phase2);
        }
        if (!done && p.debug_skip < 2) compact_and_accept();
        if (SUP == 2) {
          if (!sup_on) {
            const unsigned r = __reduce_add_sync(0xffffffffu, ct.srej);
            if (r * SUP_RATIO > (unsigned)(32 * KP * gcount)) {
              sup_on = true;
              sup_count = SUP_PROBE;
            }
          } else {
            ++sup_tiles;
            if (--sup_count == 0) sup_on = false;
          }
          ct.srej = 0u;
        }
        __syncwarp();
      };

      if (TC && tc_on) {
        // ---- B operand of the group: 32 centres x (Bx, By, Bz, 1, Bx, By, Bz, K), canonical
        // K-major layout (core matrix = 8 centres x 4 values)
        unsigned char* tcbase = smem + L.oTP;
        {
          float* sBt = reinterpret_cast<float*>(tcbase + TC_OFF_B);
          for (int t = tid; t < G * 8; t += NT) {
            const int n = t >> 3, k = t & 7, c = k & 3;
            const float4 b4 = sB[n];
            const float v = c == 0 ? b4.x : c == 1 ? b4.y : c == 2 ? b4.z : (k < 4 ? 1.0f : b4.w);
            sBt[((n & 7) * 16 + (n >> 3) * 256 + (k >> 2) * 128) / 4 + c] = v;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
        }
        const int q = warp >> 2, wq = warp & 3;       // warpgroup, tensor-memory lane quarter
        const int nch = (p.N + 127) >> 7;             // 128-point chunks holding real points
        const int nq = nch > q ? (nch - q + 3) >> 2 : 0;   // this warpgroup's: q, q + 4, ...
        // per warpgroup: TC_NA A buffers (4 KB each) and TC_NB tensor-memory tiles (32 columns)
        uint64_t* bar = s_tcbar + q * TC_NBAR;        // A full [0, NA), D full [NA, NA+NB), D empty
        const unsigned sA0 = (unsigned)__cvta_generic_to_shared(tcbase + q * (TC_NA * 4096));
        const uint64_t bdesc = umma_desc((unsigned)__cvta_generic_to_shared(tcbase + TC_OFF_B));
        const unsigned tmem = s_tmem + (unsigned)(q * (TC_NB * 32));
        constexpr uint32_t IDESC = umma_idesc_tf32(128, G);
        float4* sPW = reinterpret_cast<float4*>(tcbase + TC_OFF_PTS) + warp * 64;   // the warp's 32 points
        float4* sNW = sPW + 32;
        const bool issuer = wq == 0 && lane == 0;
        // the issuer (lane 0 of the warpgroup's first warp, itself a consumer) keeps the A
        // ring full and issues every MMA whose A has landed and whose tensor-memory tile has
        // been drained, without blocking except for the chunk its own warp needs next
        int ld_n = 0, mma_n = 0;
        auto poll = [&](int i, bool block) {
          while (ld_n < nq && ld_n < i + TC_NA) {   // A slot of chunk ld_n - NA: its MMA completed
            const unsigned it = tc_it + (unsigned)ld_n;
            bulk_load(tcbase + q * (TC_NA * 4096) + (it % TC_NA) * 4096,
                      reinterpret_cast<const unsigned char*>(p.tfa) + (size_t)(q + 4 * ld_n) * 4096, 4096u,
                      &bar[it % TC_NA]);
            ++ld_n;
          }
          while (mma_n < ld_n && mma_n < i + TC_NB) {
            const unsigned it = tc_it + (unsigned)mma_n, a = it % TC_NA, d = it % TC_NB, ud = it / TC_NB;
            const bool must = block && mma_n <= i;
            if (must) {
              mbar_wait(&bar[a], (it / TC_NA) & 1u);
              if (ud > 0) mbar_wait(&bar[TC_NA + TC_NB + d], (ud - 1u) & 1u);
            } else if (!mbar_test(&bar[a], (it / TC_NA) & 1u) ||
                       (ud > 0 && !mbar_test(&bar[TC_NA + TC_NB + d], (ud - 1u) & 1u))) {
              break;
            }
            tc_fence_after();
            umma_tf32(tmem + d * 32u, umma_desc(sA0 + a * 4096u), bdesc, IDESC);
            umma_commit(&bar[TC_NA + d]);
            ++mma_n;
          }
        };
        for (int i = 0; i < nq; ++i) {
          const unsigned it = tc_it + (unsigned)i, d = it % TC_NB;
          if (issuer) poll(i, true);
          __syncwarp();
          mbar_wait(&bar[TC_NA + d], (it / TC_NB) & 1u);
          tc_fence_after();
          uint32_t v[32];
          tmem_ld32(tmem + d * 32u + ((unsigned)(32 * wq) << 16), v);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar[TC_NA + TC_NB + d]);
          if (issuer) poll(i + 1, false);   // (chunk i's MMA completed: its A slot is free)
          __syncwarp();
          // every margin of this lane's point against the 32 centres, reduced to "any sign
          // bit clear" (a margin >= +0: a candidate)
          unsigned andv = 0xffffffffu;
#pragma unroll
          for (int g = 0; g < 32; g += 2) andv &= v[g] & v[g + 1];
          if (!__any_sync(0xffffffffu, (int)andv >= 0)) continue;
          // candidate mask of this lane's point: bit g <-> centre slot g
          unsigned m = 0u;
#pragma unroll
          for (int c = 0; c < 8; ++c) m = accept_bits4(m, v[c], v[8 + c], v[16 + c], v[24 + c], 0x01010101u << c);
          const int cnt = __popc(m);
          const int total = __reduce_add_sync(0xffffffffu, cnt);
          const unsigned liveb = __ballot_sync(0xffffffffu, m != 0u);
          const int live = __popc(liveb);
          ct.cand += (unsigned)cnt;
          // this warp's 32 points (chunk point 32 wq + lane = TMEM lane) into shared memory
          {
            const int jp = (q + 4 * i) * 128 + 32 * wq + lane;
            sPW[lane] = __ldg(&p.pos[jp]);
            sNW[lane] = __ldg(&p.nrm[jp]);
          }
          __syncwarp();
          if (skip_accept) continue;
          if (p.dense_min > 0 && total >= live * p.dense_min) {
            // dense: lane = centre slot, walk the live points (broadcast reads)
            if (lane == 0) {
              ++dense_tiles;
              dense_rows += (unsigned)live;
            }
            const float4 cP = sP[lane], cN = sN[lane];
            const bool gl = sM[lane] >= 0;
            const unsigned ia = (unsigned)__cvta_generic_to_shared(sImg) + 4u * (unsigned)(lane * IS);
            unsigned lv = liveb;
            while (lv) {
              const int pt = __ffs(lv) - 1;
              lv &= lv - 1u;
              const unsigned mp = __shfl_sync(0xffffffffu, m, pt);
              const float4 X4 = sPW[pt], NX4 = sNW[pt];
              Dec d = decide<MODE>(p, cP, cN, X4, NX4);
              const bool v0 = gl && ((mp >> lane) & 1u);
              if (!v0) d.status = 0;
              if (SUP == 2) ct.srej += (unsigned)(v0 & (d.sup_out != 0));
              if (d.status == 2) resolve<MODE>(p, d, cP, cN, X4, NX4, ct);
              if (d.status) {
                ++ct.acc;
                apply_s<MODE, G>(p, d, ia, lane, &s_carry);
              }
            }
          } else {
            // sparse: entries (point lane << 5 | centre slot) in the ring, eight centre slots
            // (<= 256 entries) at a time, passes of 32
            static_assert(QCAP >= 256, "ring: 32 lanes x 8 slots");
#pragma unroll 1
            for (int c8 = 0; c8 < 32; c8 += 8) {
              const unsigned mb = (m >> c8) & 0xffu;
              const int cb8 = __popc(mb);
              int x = cb8;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
              }
              const int tot8 = __shfl_sync(0xffffffffu, x, 31);
              if (tot8 == 0) continue;
              uint16_t* qd = sQ + (x - cb8);
              for (unsigned mm = mb; mm; mm &= mm - 1u) *qd++ = (uint16_t)((lane << 5) | (c8 + __ffs(mm) - 1));
              __syncwarp();
              for (int base = 0; base < tot8; base += 32) {
                if (base + lane < tot8) {
                  const unsigned e = sQ[base + lane];
                  const int pt = (int)(e >> 5), gs = (int)(e & 31u);
                  const float4 P4 = sP[gs], N4 = sN[gs], X4 = sPW[pt], NX4 = sNW[pt];
                  Dec d = decide<MODE>(p, P4, N4, X4, NX4);
                  if (SUP == 2) ct.srej += (unsigned)(d.sup_out != 0);
                  if (d.status == 2) resolve<MODE>(p, d, P4, N4, X4, NX4, ct);
                  if (d.status) {
                    ++ct.acc;
                    apply<MODE, G>(p, d, sImg + gs * IS, gs, &s_carry);
                  }
                }
              }
              __syncwarp();
            }
          }
        }
        tc_it += (unsigned)nq;
      } else if (PRUNE == 0) {
        // PASS1 state: the next tile's fragment copy is in flight into the warp's buffer
        bool pf_inflight = false;
        unsigned pb0[PASS1 ? NCB : 1], pb1[PASS1 ? NCB : 1];   // B fragments of the group
        if (PASS1) {
          const int gid = lane >> 2, tig = lane & 3;
          const float* sBf = reinterpret_cast<const float*>(sB);
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) {
            const int sb = gid * NCB + cb;
            float b1 = sBf[(G >= 8 || sb < G ? sb : 0) * 4 + tig];
            float b0 = tig == 3 ? 1.0f : b1;
            if (G < 8 && sb >= G) {
              b0 = 0.0f;
              b1 = tig == 3 ? -INFINITY : 0.0f;
            }
            pb0[cb] = __float_as_uint(b0);
            pb1[cb] = __float_as_uint(b1);
          }
        }
        auto frag_copy = [&](int chunk) {
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(sT, p.mfrag + (size_t)chunk * 256, 4096u, &s_tile_bar[warp]);
          }
        };
        for (int t = (int)crank; t < p.n_tiles; t += CL) {   // (a cluster splits the tiles)
          const int base = t * (NT * KP) + tid;
          int j[KP];
#pragma unroll
          for (int k = 0; k < KP; ++k) j[k] = base + k * NT;
          if (TMA_TILE) j[0] = t * (NT * KP) + warp * 128;   // the warp's 128-point chunk
          const int next = t + CL < p.n_tiles ? (t + CL) * NWARP + warp : -1;
          const bool sup_hot1 = SUP == 1 || (SUP == 2 && sup_on);
          if (PASS1 && p.mma && !sup_hot1) {
            // ---- phase 1: the pre-pass of the tile from its staged fragments
            const int chunk = j[0] >> 7;
            if (!pf_inflight) frag_copy(chunk);
            mbar_wait(&s_tile_bar[warp], tile_phase);
            tile_phase ^= 1u;
            pf_inflight = false;
            uint4 fr[8];
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) fr[rb] = reinterpret_cast<const uint4*>(sT)[rb * 32 + lane];
            __syncwarp();
            // prefetch the next tile's fragments into the (now free) buffer while the HMMAs
            // run, unless the queue is nearly full (a tile with a candidate then has to be
            // decided inline, in this buffer)
            int room = 0;
            if (lane == 0) room = *reinterpret_cast<volatile int*>(&s_dq_n) < DQ_CAP - NWARP;
            room = __shfl_sync(0xffffffffu, room, 0);
            if (next >= 0 && room) {
              frag_copy(next);
              pf_inflight = true;
            }
            unsigned andv = 0xffffffffu;
#pragma unroll
            for (int rb = 0; rb < 8; ++rb) {
#pragma unroll
              for (int cb = 0; cb < NCB; ++cb) {
                float d0, d1, d2, d3;
                mma_tf32(d0, d1, d2, d3, fr[rb].x, fr[rb].y, fr[rb].z, fr[rb].w, pb0[cb], pb1[cb], 0.0f, 0.0f);
                andv &= __float_as_uint(d0) & __float_as_uint(d1);
                andv &= __float_as_uint(d2) & __float_as_uint(d3);
              }
            }
            if (__any_sync(0xffffffffu, (int)andv >= 0)) {
              if (pf_inflight) {
                if (lane == 0) s_dq[atomicAdd(&s_dq_n, 1)] = chunk;   // room was reserved
              } else {
                run_tile(j, -1, true);   // queue nearly full: re-stage and decide inline
              }
            }
          } else {
            if (PASS1 && pf_inflight) {   // (a packed-fp32 tile: drain the prefetch first)
              mbar_wait(&s_tile_bar[warp], tile_phase);
              tile_phase ^= 1u;
              pf_inflight = false;
            }
            run_tile(j, next, false);
          }
        }
        if (DQ) {
          // phase 2: the group's queued tiles, dealt to the warps one at a time
          __syncthreads();
          const int nq = min(s_dq_n, DQ_CAP);
          for (;;) {
            int k = 0;
            if (lane == 0) k = atomicAdd(&s_dq_head, 1);
            k = __shfl_sync(0xffffffffu, k, 0);
            if (k >= nq) break;
            int j[KP];
            j[0] = s_dq[k] * 128;
#pragma unroll
            for (int kk = 1; kk < KP; ++kk) j[kk] = j[0];
            run_tile(j, -1, true);
          }
          __syncthreads();
          if (tid == 0) s_dq_n = s_dq_head = 0;
        }
      } else {
        // rows of the visited box, batched ROWCAP at a time
        const int cx0 = s_rng[0], cx1 = s_rng[1], cy0 = s_rng[2], cy1 = s_rng[3], cz0 = s_rng[4];
        const int ny = cy1 - cy0 + 1;
        for (int rb = 0; rb < nrows; rb += ROWCAP) {
          const int nb = min(ROWCAP, nrows - rb);
          int len = 0, start = 0;
          if (tid < nb) {
            const int row = rb + tid;
            const int cz = cz0 + row / ny, cy = cy0 + row % ny;
            const int base = (cz * p.dimy + cy) * p.dimx;
            // x-cells of this row that some live centre's R-sphere can reach: the hull
            // of the chords over the group (every region point lies in its centre's
            // sphere), bounds widened by s against the rounding of the cell mapping
            const float hc = p.h_cell;
            const float ylo = cy == 0 ? -INFINITY : fmaf((float)cy, hc, p.oy);
            const float yhi = cy == p.dimy - 1 ? INFINITY : fmaf((float)(cy + 1), hc, p.oy);
            const float zlo = cz == 0 ? -INFINITY : fmaf((float)cz, hc, p.oz);
            const float zhi = cz == p.dimz - 1 ? INFINITY : fmaf((float)(cz + 1), hc, p.oz);
            const float R2 = p.R_up * p.R_up * 1.000001f;
            int xl = cx1 + 1, xh = cx0 - 1;
            for (int g = 0; g < G; ++g) {
              if (sM[g] < 0) continue;
              const float4 P4 = sP[g];
              const float s = 4e-6f * (fabsf(P4.y) + fabsf(P4.z) + fabsf(p.oy) + fabsf(p.oz) + 2.f * hc) + 1e-30f;
              const float dy = fmaxf(0.f, fmaxf(ylo - P4.y, P4.y - yhi) - s);
              const float dz = fmaxf(0.f, fmaxf(zlo - P4.z, P4.z - zhi) - s);
              const float d2 = fmaf(dy, dy, dz * dz) * 0.999999f;
              if (!(d2 <= R2)) continue;
              const float hx = sqrtf(R2 - d2) * 1.000001f + s;
              xl = min(xl, cell_coord(__fsub_rd(P4.x, hx), p.ox, p.inv_h, p.dimx));
              xh = max(xh, cell_coord(__fadd_ru(P4.x, hx), p.ox, p.inv_h, p.dimx));
            }
            xl = max(xl, cx0);
            xh = min(xh, cx1);
            if (xl <= xh) {
              start = p.cell_start[base + xl];
              len = p.cell_start[base + xh + 1] - start;
            }
          }
          // block exclusive scan of len over NT threads
          int v = len;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
          }
          __shared__ int s_wsum[NWARP];
          if (lane == 31) s_wsum[warp] = v;
          __syncthreads();
          if (warp == 0) {
            int ws = lane < NWARP ? s_wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < NWARP; o <<= 1) {
              const int n = __shfl_up_sync(0xffffffffu, ws, o);
              if (lane >= o) ws += n;
            }
            if (lane < NWARP) s_wsum[lane] = ws;
            if (lane == NWARP - 1) s_total = ws;
          }
          __syncthreads();
          const int excl = v - len + (warp > 0 ? s_wsum[warp - 1] : 0);
          if (tid < nb) {
            sRowS[tid] = start;
            sRowO[tid] = excl;
          }
          if (tid == 0) sRowO[nb] = s_total;
          __syncthreads();
          const int T = s_total;
          if (tid == 0) {
            int live = 0;
            for (int g = 0; g < G; ++g) live += sM[g] >= 0;
            visited += (unsigned long long)T * live;
          }
          int lo = 0;   // row of this thread's previous point (its f is smaller)
          for (int f0 = 0; f0 < T; f0 += NT * KP) {
            int j[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              // (CULL: a warp's 128 points are consecutive in the gathered order, a compact box)
              const int f = CL2 && SPIN_CELLS_CULL ? f0 + warp * (32 * KP) + k * 32 + lane : f0 + tid + k * NT;
              if (f < T) {
                // largest r with sRowO[r] <= f: gallop from the previous point's row, then
                // bisect
                int step = 1;
                while (lo + step < nb && sRowO[lo + step] <= f) {
                  lo += step;
                  step <<= 1;
                }
                int hi = min(lo + step, nb) - 1;
                while (lo < hi) {
                  const int mid = (lo + hi + 1) >> 1;
                  if (sRowO[mid] <= f) lo = mid; else hi = mid - 1;
                }
                j[k] = sRowS[lo] + (f - sRowO[lo]);
              } else {
                j[k] = p.N;  // sentinel
              }
            }
            run_tile(j, -1, false);
          }
          __syncthreads();
        }
      }
      if (CL > 1) cluster_sync_all();   // every (remote) add into this CTA's images is done
      else __syncthreads();
      // ---- a12: write the images back in the caller's order
      for (int i = tid; i < GL * WW; i += NT) {
        const int ls = i / WW;            // local image; group slot crank * GL + ls
        const int slot = (int)crank * GL + ls;
        const int e = i - ls * WW;
        int mm = sM[slot];
        if (mm == -1) continue;
        float val = 0.0f;
        if (mm < -1) {
          mm = -(mm + 2);
        } else if (MODE == 0) {
          const uint32_t cnt = sImg[ls * IS + e];
          if (cnt >= (1u << 24)) atomicOr(&p.err_flags[1], 1);
          val = (float)cnt;
        } else {
          const uint32_t h =
              s_carry ? (gHi[ls * hiWords + (e >> 1)] >> ((e & 1) * 16)) & 0xffffu : 0u;
          const double fx = (double)h * 4294967296.0 + (double)sImg[ls * IS + e];
          val = (float)(fx * (1.0 / 8388608.0));
        }
        __stcs(&p.out[(long long)mm * WW + e], val);
      }
      if (p.seg_done != nullptr) {
        // e2e pipelining (spin_generate_host): publish finished images per output segment
        // so the copy stream can start their D2H while the kernel still runs
        __threadfence_system();
        __syncthreads();
        if (tid == 0) {
          // (this CTA's images: group slots crank * GL .. crank * GL + GL - 1)
          long long a = g0 + (long long)crank * GL;
          const long long bnd = g0 + min((long long)gcount, (long long)(crank + 1) * GL);
          while (a < bnd) {
            const long long sg = a / p.seg_images;
            const long long e = min(bnd, (sg + 1) * (long long)p.seg_images);
            atomicAdd(&p.seg_done[sg], (unsigned)(e - a));
            a = e;
          }
        }
      }
      if (MODE == 1) {
        __syncthreads();
        if (s_carry) {                       // leave the carry scratch zero for the next group
          for (int i = tid; i < GL * hiWords; i += NT) gHi[i] = 0u;
          __syncthreads();
          if (tid == 0) s_carry = 0;
        }
      }
      if ((int)blockIdx.x < p.slow_ctas && tid == 0) {
        // heterogeneity emulation: a slow worker takes `slowdown` x the group's time
        const unsigned long long tg1 = gtimer();
        const unsigned long long until = tg1 + (unsigned long long)((double)(p.slowdown - 1.0f) * (double)(tg1 - tg0));
        while (gtimer() < until) __nanosleep(512);
      }
      __syncthreads();
    }
    if (crank == 0) units_done += u1 - u0;   // (a cluster's units are counted once)
    if (DEAL && p.wf == 2 && tid == 0) {
      // AWF: my rate so far, units per microsecond of chunk time (incl. any emulated idling)
      s_awf[2] += (unsigned long long)(u1 - u0);
      s_awf[1] += gtimer() - s_awf[0];
      reinterpret_cast<volatile float*>(p.awf_rate)[blockIdx.x] =
          (float)((double)s_awf[2] * 1e3 / (double)max(s_awf[1], 1ull));
    }
  }

  if (tc_on) {
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(s_tmem) : "memory");
  }
  // ---- a13: instrumentation
  const unsigned long long t1 = gtimer();
  atomicAdd(&s_ctr[0], (unsigned long long)ct.cand);
  atomicAdd(&s_ctr[1], (unsigned long long)ct.acc);
  atomicAdd(&s_ctr[2], (unsigned long long)ct.f64);
  atomicAdd(&s_ctr[3], (unsigned long long)ct.exact);
  if (tid == 0) atomicAdd(&s_ctr[4], visited);
  if (lane == 0 && sup_tiles) atomicAdd(&s_ctr[5], (unsigned long long)sup_tiles);
  if (lane == 0 && dense_tiles) {
    atomicAdd(&s_ctr[6], (unsigned long long)dense_tiles);
    atomicAdd(&s_ctr[7], (unsigned long long)dense_rows);
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&p.stats[ST_CAND], s_ctr[0]);
    atomicAdd(&p.stats[ST_ACC], s_ctr[1]);
    atomicAdd(&p.stats[ST_F64], s_ctr[2]);
    atomicAdd(&p.stats[ST_EXACT], s_ctr[3]);
    atomicAdd(&p.stats[ST_VISITED], s_ctr[4]);
    if (s_ctr[5]) atomicAdd(&p.stats[ST_SUPHOT], s_ctr[5]);
    if (s_ctr[6]) {
      atomicAdd(&p.stats[ST_DENSE], s_ctr[6]);
      atomicAdd(&p.stats[ST_DROWS], s_ctr[7]);
    }
    p.cta_t0[blockIdx.x] = t0;
    p.cta_t1[blockIdx.x] = t1;
    p.cta_units[blockIdx.x] = units_done;
  }
}

}  // namespace spin
