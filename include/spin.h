/*
 * spin.h — C ABI of libspin, the B200 (sm_100a) spin-image engine.
 *
 * The hot path is the DOALL spin-image loop of the paper (Eleliemy, Mohammed,
 * Ciorba, "Efficient Generation of Parallel Spin-images Using Dynamic Loop
 * Scheduling", arXiv 1811.00901): Algorithm 1 `calculateSpinImages(W, B, S, OP, N)`
 * (`algo:spin`) and its per-chunk form Algorithm 2
 * `adCalculateSpinImages(..., spinImages, start, end)` (PAPER.md:286-319,
 * `algo:adaptedcalc`), with its iterations dealt by the paper's STATIC / SS / GSS /
 * FAC loop schedules (§2.2; `getChunk`).
 *
 * Naming follows BASELINE.json: N = number of oriented points (the paper's M,
 * PAPER.md:109), M = number of spin images (the paper's N),
 * b = bin size (the paper's B), A_s = support angle (the paper's S).
 *
 * Conventions for every entry point
 *   - d_* arguments are CUDA DEVICE pointers, h_* arguments are HOST pointers.
 *     spin_create / spin_load_cloud accept either (the copy uses cudaMemcpyDefault).
 *   - Arrays are dense, row-major, little-endian, 4-byte aligned.
 *   - No C++ exception crosses this boundary.  Every call returns a spin_status;
 *     spin_last_error() then holds a thread-local message naming the offending
 *     argument or index.
 *   - `stream` is a cudaStream_t (NULL = the legacy default stream).  Calls are
 *     asynchronous with respect to the host unless stated otherwise.
 */
#ifndef SPIN_H_
#define SPIN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPIN_ABI_VERSION 6

typedef struct spin_ctx* spin_handle;
typedef struct CUstream_st* spin_stream; /* identical to cudaStream_t */

typedef enum {
  SPIN_OK = 0,
  SPIN_E_INVAL = 1,    /* a synchronous argument check failed                        */
  SPIN_E_RANGE = 2,    /* a centre index outside [0, N) (detected on the device)     */
  SPIN_E_INPUT = 3,    /* non-finite coordinate, |coordinate| > 2^40, or |normal| outside [0.999, 1.001] */
  SPIN_E_NOMEM = 4,    /* device or host allocation failed                           */
  SPIN_E_CUDA = 5,     /* a CUDA runtime error (message carries cudaGetErrorString) */
  SPIN_E_OVERFLOW = 6  /* an accumulator could not hold a bin (see spin_generate)   */
} spin_status;

/* Loop schedules of PAPER.md §2.2.  STATIC = PSIA's fixed blocks
 * (P:476-477); SS = one unit per request; GSS = ceil(R/P) per request
 * (P:224-228); FAC = batches of P equal chunks, size ceil(R_batch/(2P))
 * (the FAC2 reading).
 * Beyond the paper (its "more complex DLS techniques" future work; SURVEY §8(f)
 * NEXT-4): WF = weighted factoring — FAC2 batches of P chunks, but the chunk a worker
 * receives is weighted by its relative speed w_i (mean 1):
 * ceil(R_batch * wq_i / (fac_divisor * P * 1024)) with wq_i = round(1024 w_i); the
 * speeds are known a priori — here those of the heterogeneous-worker emulation below
 * (slow CTAs 1/slowdown, the rest 1, normalised to mean 1).  AWF = adaptive weighted
 * factoring — the same rule with w_i = the worker's measured rate (units per busy time
 * over its chunks so far) over the mean rate of the workers that have reported; a worker
 * without a measurement yet probes with a one-unit chunk.  WF/AWF chunks depend on who requests, so they are claimed on
 * the device by a compare-and-swap on the packed batch state; they need n_units < 2^24,
 * P < 2^16 and no shared multi-device dealer. */
typedef enum { SPIN_STATIC = 0, SPIN_SS = 1, SPIN_GSS = 2, SPIN_FAC = 3, SPIN_WF = 4,
               SPIN_AWF = 5 } spin_schedule;

/* NEAREST: the paper's integer count tempSpinImage[k,l]++ (P:173-174).
 * BILINEAR: weight 1 split over the 4 bins around (u, v) (north star; not in the
 * paper — SURVEY.md §8(c) #12). */
typedef enum { SPIN_NEAREST = 0, SPIN_BILINEAR = 1 } spin_mode;

/* BRUTE: every (centre, point) pair, as Alg. 1's inner loop.
 * CELLS: exact uniform-grid pruning — only points in cells that intersect the
 * bounding box of a centre group grown by the region radius are visited. */
typedef enum { SPIN_BRUTE = 0, SPIN_CELLS = 1 } spin_prune;

/* flags */
#define SPIN_F_LITERAL_HALF_WIDTH 0x1u /* u = (W/2 - beta)/b exactly as printed; default u = W/2 - beta/b (#2) */
#define SPIN_F_FLOOR_BINS         0x2u /* NEAREST: k = floor(u), l = floor(v) (Johnson) instead of ceil */
#define SPIN_F_NO_SORT            0x4u /* CELLS: keep the caller's centre order (control run)    */
#define SPIN_F_NO_FAST_CERT       0x8u /* testing: send every candidate through the fp64 / exact decision stages   */
#define SPIN_F_SUPPORT_LAST       0x10u /* evaluate the support test only for the pair-test candidates: same
                                           images, fewer flops per pair (the geometric test runs first)         */
#define SPIN_F_SUPPORT_FIRST      0x20u /* evaluate the support test for every pair, as P:166 orders it.  With
                                           neither flag, CELLS does so and BRUTE places it adaptively per warp
                                           (accept path while it rejects few candidates)         */
#define SPIN_F_CLUSTER_PAIR       0x40u /* BRUTE NEAREST, table dealer, one device: run each worker as a two-CTA
                                           thread-block cluster sharing a group of 48 centres (24 images per
                                           CTA, partner counts as DSMEM reductions) where that layout fits
                                           (W <= 32).  Same images; by default one-CTA workers (faster since
                                           the dense lane-per-centre tiles)                   */
#define SPIN_F_NO_DENSE           0x80u /* BRUTE: always compact candidates, never the dense lane-per-centre
                                           tiles (control run; same images)                               */

/* Scheduling parameters.  All-zero = defaults. */
typedef struct {
  int32_t P;             /* "processing elements" (P:230, P:338 workersCount) = resident CTAs
                            of the persistent launch; 0 -> occupancy x SM count           */
  int32_t unit;          /* images per scheduling iteration; 0 -> the kernel group size G;
                            1 = the paper's one-image iteration            */
  int32_t gss_min_chunk; /* GSS minimum chunk in units; 0 -> 1 (#16)                      */
  int32_t fac_divisor;   /* FAC: chunk = ceil(R_batch / (fac_divisor * P)); 0 -> 2 (#15)   */
  uint32_t flags;        /* SPIN_F_* */
  /* Heterogeneous-worker emulation (the paper's Type1/Type2 runs; SURVEY
   * §8(f) NEXT-1).  Timing only: images are identical for every setting. */
  int32_t slow_ctas;     /* CTAs 0 .. slow_ctas-1 are slow workers; 0 -> none              */
  float slowdown;        /* their time multiplier (>= 1; 0 -> 1): after each group a slow
                            CTA idles (slowdown - 1) x the group's measured compute time  */
  int32_t slow_first;    /* dynamic schedules: the fast CTAs wait until every slow CTA has
                            issued its first request (the machine-file order) */
  /* One schedule across several devices (the paper's master-worker
   * over many nodes): every device runs spin_generate on the SAME centres with
   * the same P (the total worker count) and one shared dealer counter.  Each device
   * writes only the images of the chunks its CTAs took; the rest of its d_out is left
   * untouched (zero it and sum, or gather, across devices). */
  int32_t grid;          /* CTAs launched on this device; 0 -> P                          */
  int32_t cta_offset;    /* global worker index of this device's CTA 0 (STATIC: CTA c takes
                            block c); cta_offset + grid <= P                              */
  uint32_t* d_counter;   /* shared dealer: a u32 in device, peer or IPC-mapped memory that
                            the caller zeroes before the call on every device; NULL -> the
                            handle's own counter (reset by every call)                     */
} spin_chunk_params;

/* Optional per-call statistics.  Passing non-NULL makes spin_generate synchronise
 * `stream` before it returns (the counters are read back). */
typedef struct {
  double elapsed_ms;        /* device time of the persistent kernel (CUDA events)          */
  double grid_build_ms;     /* CELLS: device time of a grid (re)build in this call, else 0 */
  int64_t pairs_visited;    /* (centre, point) pairs evaluated by the pair test            */
  int64_t pairs_candidate;  /* pairs that passed the fp32 conservative region test         */
  int64_t pairs_accepted;   /* pairs that contributed (NEAREST: sum of all counts)         */
  int64_t fp64_fallbacks;   /* decisions the fp32 stage could not certify                  */
  int64_t exact_fallbacks;  /* decisions the fp64 stage could not certify (exact stage)    */
  int32_t P;                /* CTAs launched on this device (the grid)                      */
  int32_t G;                /* images per group (a two-CTA cluster shares one group)       */
  int32_t n_units;          /* scheduling units                                            */
  int32_t n_chunks;         /* chunks in the schedule                                      */
  uint64_t* h_cta_start_ns; /* caller array [P] or NULL: %globaltimer at CTA start         */
  uint64_t* h_cta_end_ns;   /* caller array [P] or NULL: %globaltimer at CTA finish        */
  int32_t* h_cta_units;     /* caller array [P] or NULL: units processed per CTA           */
  int32_t cta_capacity;     /* length of the three arrays above                            */
  int64_t tiles_support_hot; /* BRUTE: warp tiles (32 x 4 points x G centres) whose hot
                                 loop ran the support test (adaptive placement)             */
  int32_t filter_mma;       /* BRUTE: 1 if the sphere filter ran on the tensor cores (tf32
                               mma.sync), 0 if on packed fp32 (far-from-origin clouds,
                               SPIN_NO_MMA, or CELLS)                                         */
  int32_t cta_per_worker;   /* 1, or 2 when a worker of the schedule is a two-CTA cluster
                               (BRUTE at large W: the pair shares one group of G images, each
                               CTA holding G/2 in shared memory, DSMEM adds); workers =
                               P / cta_per_worker; units are counted on the first CTA      */
  int64_t tiles_dense;      /* BRUTE: warp tiles whose candidates took the lane-per-centre
                               path (dense tiles of the Morton-ordered cloud)              */
  int64_t dense_rows;       /* BRUTE: live points those tiles walked (one warp step each)   */
} spin_stats;

/*
 * spin_create — make a handle that owns a device copy of the oriented point cloud.
 *   points, normals: fp32 [N][3] (x,y,z) — the set OP of PAPER.md:115 with normals
 *                    np_i.  Host or device pointers (cudaMemcpyDefault).
 *   N: number of oriented points, 1 <= N < 2^31 - 12288 (room for the tile padding).
 * Copies and re-lays the cloud out as SoA float4 {x,y,z,|x|^2} + {nx,ny,nz,0} in
 * HBM (the input "replicated to every worker", P:256 / P:333, is resident once).
 * Validates: every coordinate finite with |coordinate| <= 2^40, every |normal| in [0.999, 1.001]
 * (SPIN_E_INPUT names the first bad index).  Normals are NOT renormalised (#7).
 * Synchronises `stream`.  The caller may free its arrays when it returns.
 */
spin_status spin_create(const float* points, const float* normals, int64_t N,
                        spin_stream stream, spin_handle* out);

/*
 * spin_load_cloud — replace the handle's cloud (same rules as spin_create).
 * Reuses the device buffers when N fits the current capacity; cached cell grids
 * are invalidated.  Synchronises `stream`.  If it fails after the argument checks
 * (SPIN_E_INPUT, SPIN_E_NOMEM, SPIN_E_CUDA) the handle holds NO cloud: every later
 * spin_generate / spin_count_in_sphere / spin_pair_codes returns SPIN_E_INVAL until a
 * load succeeds (never a mix of the old and the new cloud).
 */
spin_status spin_load_cloud(spin_handle h, const float* points, const float* normals,
                            int64_t N, spin_stream stream);

/*
 * spin_generate — the hot path: M spin images, one per centre (Alg. 1 / Alg. 2).
 *   d_centre_idx: int32 [M] device; image m spins around point d_centre_idx[m]
 *                 (duplicates allowed; the paper's case is iota(0, paper-N)).
 *   M: number of images, M >= 0 (M = 0 is a no-op).
 *   W: image width in bins, 1 <= W <= 64 (BILINEAR: W >= 2).
 *   b: bin size in cloud length units, finite, 1e-30 <= b <= 1e30.
 *   cos_As: cosine of the support angle: a point contributes only if
 *           n . n_x >= cos_As (inclusive, #5).  -INFINITY disables the test (the
 *           paper's S = 2 pi).  Otherwise must lie in [-1, 1].
 *   sched, cp: loop schedule and its parameters (cp may be NULL = defaults).
 *   mode, prune: see the enums.
 *   d_out: fp32 [M][W][W] device, fully overwritten; out[m][k][l], row k = beta bin,
 *          column l = alpha bin, as tempSpinImage[k,l].  NEAREST counts are
 *          exact integers in fp32 (counts <= N < 2^24 required, else SPIN_E_INVAL).
 *   stats: optional (see spin_stats).
 * Results equal the EXACT-arithmetic evaluation of Alg. 1 on the fp32 inputs
 * (b and cos_As as exact doubles): NEAREST bit-exact; BILINEAR to fp32 weight
 * rounding (2^-24 per corner).  Every decision the fp32 stage cannot certify is
 * re-taken in fp64 and, if still uncertain, exactly.
 * Schedule, P and unit never change the result (NEAREST and BILINEAR both
 * bit-reproducible).  Asynchronous on `stream` (unless stats != NULL).
 * A centre index outside [0, N) zeroes that image and latches SPIN_E_RANGE, which
 * this call returns if stats != NULL, else the next call on the handle returns.
 * d_centre_idx and d_out must not alias each other or handle memory.  A handle is
 * not safe for concurrent spin_generate calls (shared scratch): serialise per handle.
 * CUDA graphs: a call may be captured (stream capture) once an uncaptured call with
 * the same (W, mode, prune, sched, cp, M) has set up the handle's tables and grid; a
 * captured call records only memsets and kernels, skips the deferred error report
 * and refuses stats (SPIN_E_INVAL).  Replays reuse the captured pointers and sizes.
 */
spin_status spin_generate(spin_handle h, const int32_t* d_centre_idx, int64_t M, int32_t W,
                          double b, double cos_As, spin_schedule sched,
                          const spin_chunk_params* cp, spin_mode mode, spin_prune prune,
                          float* d_out, spin_stats* stats, spin_stream stream);

/*
 * spin_generate_host — spin_generate with HOST buffers: copies h_centre_idx [M]
 * to the device, runs, delivers the images to h_out [M][W][W] and synchronises
 * `stream`.  If all of h_out is page-locked and mapped (cudaHostAlloc /
 * cudaHostRegister / torch pin_memory under unified addressing) the kernel writes
 * each finished group of images straight into it over the host link, overlapped with
 * the groups still being computed, whatever the processing order.  Otherwise the
 * images go to handle-owned device scratch and are copied afterwards; for BRUTE runs of
 * >= 8 MB in the caller's centre order (SPIN_F_NO_SORT) that D2H copy is pipelined:
 * the kernel counts finished images per output segment (~2 MB each, 16 .. 256
 * segments) and a handle-owned copy stream waits on each counter
 * (cuStreamWaitValue32, resolved through cudaGetDriverEntryPoint) before copying that
 * segment.  A shared dealer (cp->d_counter) is rejected with SPIN_E_INVAL: multi-device
 * runs use spin_generate.
 */
spin_status spin_generate_host(spin_handle h, const int32_t* h_centre_idx, int64_t M,
                               int32_t W, double b, double cos_As, spin_schedule sched,
                               const spin_chunk_params* cp, spin_mode mode, spin_prune prune,
                               float* h_out, spin_stats* stats, spin_stream stream);

/*
 * spin_chunk_sequence — host-only trace of a schedule (SPEC getChunk traces):
 * writes the chunk boundaries b_0 = 0 < b_1 < ... < b_n = n_units into h_bounds
 * (capacity `cap` entries, n_chunks + 1 needed) and the chunk count into *n_chunks.
 * SPIN_E_RANGE if cap is too small (*n_chunks still set).  P >= 1, n_units >= 0.
 * SPIN_WF: the sequence for requests in round-robin worker order 0, 1, ..., P-1, 0, ...
 * with the weights cp implies; SPIN_AWF (measured weights) has no static trace:
 * SPIN_E_INVAL.
 */
spin_status spin_chunk_sequence(spin_schedule sched, int64_t n_units, int32_t P,
                                const spin_chunk_params* cp, int64_t* h_bounds, int64_t cap,
                                int64_t* n_chunks);

/* spin_region_radius — upper bound on |X - P| of any contributing pair for (W, b,
 * mode, flags): sqrt(alpha_max^2 + |beta|_max^2).  Host-only. */
double spin_region_radius(int32_t W, double b, spin_mode mode, uint32_t flags);

/* spin_count_in_sphere — the implementation-independent work measure of SURVEY §8(d)
 * for CELLS: sum over the M centres of #{points x : |x - p| <= R} (R = e.g.
 * spin_region_radius), counted exactly (double, numpy's operation order) on the
 * handle's cell grid (built for R if needed).  Diagnostic, not part of spin_generate;
 * synchronises `stream`. */
spin_status spin_count_in_sphere(spin_handle h, const int32_t* d_centre_idx, int64_t M, double R,
                                 int64_t* count, spin_stream stream);

/* spin_pair_codes — DIAGNOSTIC (tests only; not part of spin_generate).  For each of the
 * M centres d_centre_idx[m] and EVERY cloud point j (handle order), the accept path's
 * certified per-pair decision (the same device functions spin_generate runs on every
 * candidate: fp32 with certified bounds, then fp64, then exact) under the same region
 * constants (Alg. 1 lines P:166-174; readings of DESIGN.md §3):
 *   d_codes[m * N + j] = -1 if the pair does not contribute, else
 *                        NEAREST  k * W + l   (its bin),
 *                        BILINEAR i0 * W + j0 (the splat's base corner, reading #12).
 * d_codes is int32 [M][N] device memory owned by the caller.  NEAREST codes equal the
 * exact definition's; BILINEAR region decisions do too, while (i0, j0) may differ from an
 * exact evaluation only for pairs within fp32 rounding of an INTERIOR bin edge, where the
 * splat is continuous (the "flips" the parity tests count and report).  Asynchronous on
 * `stream`.  SPIN_E_INVAL as spin_generate (bad W, b, cos_As, mode, flags, null pointers)
 * or when the handle holds no valid cloud. */
spin_status spin_pair_codes(spin_handle h, const int32_t* d_centre_idx, int64_t M, int32_t W,
                            double b, double cos_As, spin_mode mode, uint32_t flags,
                            int32_t* d_codes, spin_stream stream);

/* spin_cos_from_degrees — cos of an angle in degrees, exact at 0, 60, 90, 120, 180
 * (1, 0.5, 0, -0.5, -1); >= 180 degrees returns -INFINITY (test disabled). */
double spin_cos_from_degrees(double deg);

/* spin_default_P — the resident-CTA count the persistent launch would use for
 * (W, mode, prune) on the current device (occupancy x SMs); <= 0 on error. */
int32_t spin_default_P(int32_t W, spin_mode mode, spin_prune prune);

void spin_destroy(spin_handle h);
const char* spin_last_error(void);
int32_t spin_abi_version(void);

/* ---- Shared dealer across devices / processes: the paper's
 * master as one u32 counter that every device's CTAs increment with
 * atomicAdd, over NVLink peer memory or CUDA IPC.  The counter is a plain cudaMalloc
 * of its own (so its IPC handle maps exactly this allocation). */
spin_status spin_dealer_alloc(uint32_t** d_counter);          /* on the current device, zeroed */
/* the 64-byte CUDA IPC handle of a counter from spin_dealer_alloc, for another process */
spin_status spin_dealer_ipc_handle(const uint32_t* d_counter, unsigned char handle[64]);
/* map another process's counter into this one (peer access enabled lazily) */
spin_status spin_dealer_ipc_open(const unsigned char handle[64], uint32_t** d_counter);
/* zero the counter on `stream` (before every schedule; order it before every device's
 * spin_generate, e.g. with a barrier after a synchronize) */
spin_status spin_dealer_reset(uint32_t* d_counter, spin_stream stream);
/* release: opened != 0 unmaps an IPC mapping, else frees the allocation */
spin_status spin_dealer_free(uint32_t* d_counter, int32_t opened);

/* ---- Host-side ingestion: the paper's OP = read3DPoints(OF)
 * (Alg. 3).  Pure host code, no device and no handle needed; errors set
 * spin_last_error with the file and line. */

/* spin_read_xyzn — an xyzn text file: one oriented point per line, six reals
 * "x y z nx ny nz", blank lines and '#' comments skipped, file order kept (indices are
 * the paper's i of OP[i]).  Normals are normalised in double, then rounded to fp32.
 *   points, normals: caller fp32 [cap][3], or both NULL to count only; *n_out = points.
 *   SPIN_E_INPUT: malformed line, non-finite value, zero normal (names the line), empty
 *   cloud; SPIN_E_RANGE: more than cap points; SPIN_E_INVAL: null path / unreadable. */
spin_status spin_read_xyzn(const char* path, float* points, float* normals, int64_t cap,
                           int64_t* n_out);

/* spin_read_off — an ASCII OFF triangle mesh ("OFF", "nv nf ne", nv vertex lines, nf
 * lines "3 i j k").  vertices: fp32 [vcap][3], faces: int32 [fcap][3]; pass NULL for
 * either to read only the counts *nv_out, *nf_out.  SPIN_E_INPUT on a malformed or
 * non-triangle face or an index outside [0, nv). */
spin_status spin_read_off(const char* path, float* vertices, int64_t vcap, int32_t* faces,
                          int64_t fcap, int64_t* nv_out, int64_t* nf_out);

/* spin_vertex_normals — per-vertex unit normals of a triangle mesh: the normalised sum
 * of the incident faces' un-normalised normals (e1 x e2, so area-weighted), accumulated
 * in double.  normals: caller fp32 [nv][3].  SPIN_E_INPUT if a vertex has no incident
 * face or only zero-area ones, or a face index is out of range. */
spin_status spin_vertex_normals(const float* vertices, int64_t nv, const int32_t* faces,
                                int64_t nf, float* normals);

#ifdef __cplusplus
}
#endif
#endif /* SPIN_H_ */
