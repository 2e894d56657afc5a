// spin_api.cpp — the C ABI of include/spin.h and the host planner.
//
// Planner duties per spin_generate call: validate (§8(b)),
// region constants and certified fp32 thresholds (a2), the chunk-boundary table of
// the schedule (a3, §2.2), the CELLS grid (a4, cached per cell size) and
// the centre ordering (a5), then one launch of the persistent kernel (a6-a13).
#include "../../include/spin.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "spin_internal.h"

using namespace spin;

namespace {

thread_local std::string g_err;

spin_status fail(spin_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
}  // namespace

// shared with spin_io.cpp (host-side ingestion): same thread-local last-error text
namespace spin {
spin_status io_fail(spin_status st, const char* fmt, ...);
}
spin_status spin::io_fail(spin_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

namespace {
spin_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SPIN_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(call, what)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);   \
  } while (0)

constexpr double U32 = 5.9604644775390625e-08;  // 2^-24

template <typename T>
spin_status ensure(T*& ptr, int64_t& cap, int64_t need, const char* what) {
  if (need <= cap && ptr) return SPIN_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  int64_t n = std::max<int64_t>(need, 1);
  if (cudaMalloc((void**)&ptr, (size_t)n * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return fail(SPIN_E_NOMEM, "cudaMalloc failed for %s (%lld elements)", what, (long long)n);
  }
  cap = n;
  return SPIN_OK;
}

float f32_up(double x) {
  float f = (float)x;
  if ((double)f < x) f = std::nextafter(f, INFINITY);
  return f;
}
float f32_down(double x) {
  float f = (float)x;
  if ((double)f > x) f = std::nextafter(f, -INFINITY);
  return f;
}

// The set of (u, v) that contributes, per mode and flags:
//   NEAREST ceil : k = ceil(u) in [0,W)  <=> u in (-1, W-1];  l = ceil(v) <= W-1  <=> v <= W-1
//   NEAREST floor: k = floor(u) in [0,W) <=> u in [0, W);     v < W
//   BILINEAR     : floor(u) in [0,W-2]   <=> u in [0, W-1);   v < W-1
// and beta = (W/2 - u) b (scaled) or W/2 - u b (literal).
struct Region {
  double ulo, uhi, vmax;
  double beta_lo, beta_hi, Qmax, mid, h, R;
};
Region region_of(int W, double b, int mode, uint32_t flags) {
  Region r;
  if (mode == SPIN_NEAREST && !(flags & SPIN_F_FLOOR_BINS)) {
    r.ulo = -1.0; r.uhi = W - 1.0; r.vmax = W - 1.0;
  } else if (mode == SPIN_NEAREST) {
    r.ulo = 0.0; r.uhi = (double)W; r.vmax = (double)W;
  } else {
    r.ulo = 0.0; r.uhi = W - 1.0; r.vmax = W - 1.0;
  }
  const double A = 0.5 * W;
  auto beta_of = [&](double u) { return (flags & SPIN_F_LITERAL_HALF_WIDTH) ? A - u * b : (A - u) * b; };
  const double b1 = beta_of(r.uhi), b2 = beta_of(r.ulo);
  r.beta_lo = std::min(b1, b2);
  r.beta_hi = std::max(b1, b2);
  r.Qmax = (r.vmax * b) * (r.vmax * b);
  r.mid = 0.5 * (r.beta_lo + r.beta_hi);
  r.h = 0.5 * (r.beta_hi - r.beta_lo);
  const double bm = std::max(std::fabs(r.beta_lo), std::fabs(r.beta_hi));
  r.R = std::sqrt(r.Qmax + bm * bm);
  return r;
}

// WF integer weights (mean 1024): slow workers 1/slowdown, the rest 1, normalised to mean 1
void wf_weights(int32_t P, int32_t slow, float slowdown, uint32_t* wq_slow, uint32_t* wq_fast) {
  const int S = std::min(std::max(slow, 0), P);
  const double ws = slowdown > 1.0f ? 1.0 / slowdown : 1.0;
  const double mean = (S * ws + (P - S)) / P;
  *wq_slow = (uint32_t)std::max(1.0, std::floor(1024.0 * ws / mean + 0.5));
  *wq_fast = (uint32_t)std::max(1.0, std::floor(1024.0 / mean + 0.5));
}

// one WF claim: the chunk of a worker with integer weight wq given the batch state
// (next unit, batch remaining Rb, chunks dealt in this batch cnt); the device dealer
// (spin_persistent) applies the same integer rule
inline int64_t wf_chunk(int64_t n, int64_t next, int64_t Rb, uint32_t wq, int32_t fac_div, int32_t P) {
  const int64_t den = (int64_t)fac_div * P * 1024;
  const int64_t c = (Rb * (int64_t)wq + den - 1) / den;
  return std::min(std::max<int64_t>(c, 1), n - next);
}

void build_bounds(spin_schedule sched, int64_t n, int32_t P, int32_t gss_min, int32_t fac_div,
                  std::vector<int64_t>& out, int32_t slow = 0, float slowdown = 1.0f) {
  out.clear();
  out.push_back(0);
  if (n <= 0) return;
  int64_t R = n;
  switch (sched) {
    case SPIN_STATIC: {  // P near-equal blocks, the first n mod P one larger (#17)
      const int64_t q = n / P, r = n % P;
      const int64_t nb = std::min<int64_t>(P, n);
      for (int64_t i = 0; i < nb; ++i) out.push_back(out.back() + q + (i < r ? 1 : 0));
      break;
    }
    case SPIN_SS:        // one iteration per request
      for (int64_t i = 1; i <= n; ++i) out.push_back(i);
      break;
    case SPIN_GSS:       // ceil(remaining / P), at least gss_min (#16)
      while (R > 0) {
        int64_t c = std::min(R, std::max<int64_t>(gss_min, (R + P - 1) / P));
        out.push_back(out.back() + c);
        R -= c;
      }
      break;
    case SPIN_FAC:       // batches of P equal chunks ceil(R / (fac_div P)) (#15)
      while (R > 0) {
        const int64_t c = std::max<int64_t>(1, (R + (int64_t)fac_div * P - 1) / ((int64_t)fac_div * P));
        for (int i = 0; i < P && R > 0; ++i) {
          const int64_t t = std::min(c, R);
          out.push_back(out.back() + t);
          R -= t;
        }
      }
      break;
    case SPIN_WF: {      // weighted factoring, requests in round-robin worker order
      uint32_t wqs, wqf;
      wf_weights(P, slow, slowdown, &wqs, &wqf);
      int64_t next = 0, Rb = 0;
      int32_t cnt = 0, who = 0;
      while (next < n) {
        if (cnt == 0) Rb = n - next;
        const int64_t c = wf_chunk(n, next, Rb, who < slow ? wqs : wqf, fac_div, P);
        next += c;
        out.push_back(next);
        cnt = cnt + 1 == P ? 0 : cnt + 1;
        who = who + 1 == P ? 0 : who + 1;
      }
      break;
    }
    default:
      break;
  }
}

}  // namespace

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct spin_ctx {
  int dev = 0, sms = 0;
  int64_t N = 0, Npad = 0, cap = 0;
  float4* pos = nullptr;
  float4* nrm = nullptr;
  float4* tpos = nullptr;   // BRUTE warp-tile pair layout (2 float4 per point), Morton order
  float4* bpos = nullptr;   // BRUTE: the cloud in Morton order (bpos[i] = pos[perm[i]])
  float4* bnrm = nullptr;
  float4* tfa = nullptr;    // BRUTE tcgen05 A operand (2 float4 per point)
  float4* mfrag = nullptr;  // BRUTE mma.sync A fragments (2 float4 per point)
  MortonGrid mgrid{0.f, 0.f, 0.f, 0.f};
  // Morton sort scratch (cloud at load time, centres per BRUTE call)
  uint32_t* mk0 = nullptr; int64_t mk0_cap = 0;
  uint32_t* mk1 = nullptr; int64_t mk1_cap = 0;
  int32_t* mv0 = nullptr; int64_t mv0_cap = 0;
  int32_t* mperm = nullptr; int64_t mperm_cap = 0;
  unsigned char* mtemp = nullptr; int64_t mtemp_cap = 0;
  float absmax = 0.f;
  float aabb[6] = {0, 0, 0, 0, 0, 0};
  uint64_t cloud_version = 0;
  // CELLS grid cache
  bool grid_valid = false;
  uint64_t grid_version = 0;
  float grid_h = 0.f;
  int dx = 0, dy = 0, dz = 0;
  float ox = 0, oy = 0, oz = 0, inv_h = 0, h_cell = 0;
  int32_t* cell_start = nullptr; int64_t cell_start_cap = 0;
  float4* spos = nullptr; int64_t spos_cap = 0;
  float4* snrm = nullptr; int64_t snrm_cap = 0;
  int32_t* keys = nullptr; int64_t keys_cap = 0;
  int32_t* counts = nullptr; int64_t counts_cap = 0;
  int32_t* cursor = nullptr; int64_t cursor_cap = 0;
  int32_t* scan_tmp = nullptr; int64_t scan_tmp_cap = 0;
  // centre ordering scratch
  int32_t* ckeys = nullptr; int64_t ckeys_cap = 0;
  int32_t* cstarts = nullptr; int64_t cstarts_cap = 0;
  int32_t* order = nullptr; int64_t order_cap = 0;
  // dealing
  int32_t* bounds = nullptr; int64_t bounds_cap = 0;
  std::vector<int64_t> bounds_h;
  long long bounds_key[6] = {-1, -1, -1, -1, -1, -1};
  unsigned* counter = nullptr;
  unsigned long long* stats = nullptr;
  int32_t* err = nullptr;
  int32_t* h_err = nullptr;  // pinned copy of the previous call's flags
  cudaEvent_t ev_err = nullptr, ev0 = nullptr, ev1 = nullptr, evg0 = nullptr, evg1 = nullptr;
  bool err_pending = false;
  unsigned long long* cta_t0 = nullptr; unsigned long long* cta_t1 = nullptr;
  int32_t* cta_units = nullptr; int64_t cta_cap = 0;
  uint32_t* hi_scratch = nullptr; int64_t hi_cap = 0;   // kept zero between launches
  // e2e pipelining of spin_generate_host: per-segment completion counters + copy stream
  unsigned* seg_done = nullptr; int64_t seg_cap = 0;
  // WF/AWF dealer: [0] packed batch state, [1] unused, [2..] per-CTA measured rates (float)
  unsigned long long* wf_state = nullptr; int64_t wf_cap = 0;
  int32_t pipe_seg_images = 0;                         // armed for the next launch only
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_seg0 = nullptr;
  int stream_wait_ok = -1;                             // -1 unknown, 0 no, 1 yes
  WaitValue32Fn wait_value32 = nullptr;
  // cloud staging (AoS input) and reductions
  float* stage_p = nullptr; int64_t stage_p_cap = 0;
  float* stage_n = nullptr; int64_t stage_n_cap = 0;
  int32_t* red = nullptr;     // [0] bad index, [1] absmax bits, [2..7] aabb bits
  int32_t* h_red = nullptr;   // pinned
  // host-buffer path scratch
  int32_t* cidx = nullptr; int64_t cidx_cap = 0;
  float* outbuf = nullptr; int64_t outbuf_cap = 0;
};

namespace {

spin_status ensure_morton_scratch(spin_ctx* h, int64_t n) {
  spin_status st;
  if ((st = ensure(h->mk0, h->mk0_cap, n, "sort keys")) != SPIN_OK) return st;
  if ((st = ensure(h->mk1, h->mk1_cap, n, "sort keys")) != SPIN_OK) return st;
  if ((st = ensure(h->mv0, h->mv0_cap, n, "sort values")) != SPIN_OK) return st;
  if ((st = ensure(h->mperm, h->mperm_cap, n, "sort order")) != SPIN_OK) return st;
  return ensure(h->mtemp, h->mtemp_cap, (int64_t)morton_sort_temp_bytes(n), "sort scratch");
}

spin_status load_cloud(spin_ctx* h, const float* points, const float* normals, int64_t N,
                       cudaStream_t s) {
  if (!points || !normals) return fail(SPIN_E_INVAL, "points/normals must be non-null");
  const int64_t TILE_POINTS = tile_points();
  if (N < 1 || N >= ((int64_t)1 << 31) - 2 * TILE_POINTS)
    return fail(SPIN_E_INVAL, "N=%lld outside [1, 2^31 - 12288)", (long long)N);
  const int64_t Npad = ((N + 1 + TILE_POINTS - 1) / TILE_POINTS) * TILE_POINTS;  // >= 1 sentinel
  // from here on the device copy is being replaced: until it is validated the handle holds
  // NO cloud (spin_generate refuses with SPIN_E_INVAL), never a mix of old and new state
  h->N = 0;
  h->Npad = 0;
  h->grid_valid = false;
  h->cloud_version++;
  if (Npad > h->cap) {
    if (h->pos) cudaFree(h->pos);
    if (h->nrm) cudaFree(h->nrm);
    if (h->tpos) cudaFree(h->tpos);
    if (h->bpos) cudaFree(h->bpos);
    if (h->bnrm) cudaFree(h->bnrm);
    if (h->tfa) cudaFree(h->tfa);
    if (h->mfrag) cudaFree(h->mfrag);
    h->pos = h->nrm = h->tpos = h->bpos = h->bnrm = h->tfa = h->mfrag = nullptr;
    h->cap = 0;
    if (cudaMalloc((void**)&h->pos, Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->nrm, Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->bpos, Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->bnrm, Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->tpos, 2 * Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->tfa, 2 * Npad * sizeof(float4)) != cudaSuccess ||
        cudaMalloc((void**)&h->mfrag, 2 * Npad * sizeof(float4)) != cudaSuccess) {
      cudaGetLastError();
      return fail(SPIN_E_NOMEM, "cudaMalloc of the cloud (%lld points) failed", (long long)N);
    }
    h->cap = Npad;
  }
  // stage AoS input on the device (host or device source: cudaMemcpyDefault)
  spin_status st;
  if ((st = ensure(h->stage_p, h->stage_p_cap, N * 3, "staging")) != SPIN_OK) return st;
  if ((st = ensure(h->stage_n, h->stage_n_cap, N * 3, "staging")) != SPIN_OK) return st;
  CK(cudaMemcpyAsync(h->stage_p, points, N * 3 * sizeof(float), cudaMemcpyDefault, s), "copy points");
  CK(cudaMemcpyAsync(h->stage_n, normals, N * 3 * sizeof(float), cudaMemcpyDefault, s), "copy normals");
  const int32_t big = 0x7fffffff;
  // [0] first bad index; [1] absmax bits 0; aabb min as flipped +max, max as flipped -max
  const int32_t init[8] = {big, 0, 0x7fffffff, 0x7fffffff, 0x7fffffff, (int32_t)0x80000000,
                           (int32_t)0x80000000, (int32_t)0x80000000};
  std::memcpy(h->h_red, init, sizeof init);
  CK(cudaMemcpyAsync(h->red, h->h_red, sizeof init, cudaMemcpyHostToDevice, s), "init");
  CK(launch_relayout(h->stage_p, h->stage_n, N, Npad, h->pos, h->nrm, h->red,
                     reinterpret_cast<float*>(h->red + 1), reinterpret_cast<float*>(h->red + 2), s),
     "relayout");
  CK(cudaMemcpyAsync(h->h_red, h->red, sizeof init, cudaMemcpyDeviceToHost, s), "readback");
  CK(cudaStreamSynchronize(s), "spin_create sync");
  int32_t red[8];
  std::memcpy(red, h->h_red, sizeof red);
  const int32_t bad = red[0];
  if (bad != big)
    return fail(SPIN_E_INPUT, "point %d: non-finite coordinate, |coordinate| > 2^40, or |normal| outside [0.999, 1.001]", bad);
  auto unflip = [](int32_t i) { int32_t v = i >= 0 ? i : i ^ 0x7fffffff; float f; std::memcpy(&f, &v, 4); return f; };
  std::memcpy(&h->absmax, &red[1], 4);
  for (int a = 0; a < 6; ++a) h->aabb[a] = unflip(red[2 + a]);
  // BRUTE layout: the cloud in Morton order (bpos, bnrm) and its warp-tile pair layout
  // (tpos); a layout choice only, the images are invariant under point order
  {
    const float ext = std::max(std::max(h->aabb[3] - h->aabb[0], h->aabb[4] - h->aabb[1]),
                               std::max(h->aabb[5] - h->aabb[2], 1e-30f));
    h->mgrid = MortonGrid{h->aabb[0], h->aabb[1], h->aabb[2], (float)(1024.0 / ((double)ext * (1.0 + 1e-6)))};
    if ((st = ensure_morton_scratch(h, N)) != SPIN_OK) return st;
    CK(launch_morton_order(nullptr, N, h->pos, (int32_t)N, h->mgrid, h->mk0, h->mk1, h->mv0, h->mperm,
                           h->mtemp, (size_t)h->mtemp_cap, s),
       "cloud Morton order");
    CK(launch_gather_cloud(h->mperm, (int32_t)N, Npad, h->pos, h->nrm, h->bpos, h->bnrm, s), "gather");
    CK(launch_pair_layout(h->bpos, h->bnrm, Npad, h->tpos, s), "pair layout");
    CK(launch_tf32_operand(h->bpos, Npad, h->tfa, s), "tcgen05 operand");
    CK(launch_mma_frags(h->bpos, Npad, h->mfrag, s), "mma fragments");
    CK(cudaStreamSynchronize(s), "spin_create sync");
  }
  h->N = N;
  h->Npad = Npad;
  h->cloud_version++;
  return SPIN_OK;
}

// a2: region constants and the certified fp32 thresholds of the hot loop and the accept
// path, shared by spin_generate and the spin_pair_codes diagnostic
void plan_thresholds(const spin_ctx* h, int32_t W, double b, double cos_As, bool has_support,
                     spin_mode mode, spin_prune prune, uint32_t flags, const Region& rg,
                     KParams& p) {
  const double X = std::max((double)h->absmax, 1e-30) * (1.0 + 1e-6);
  const double u = U32;
  const double amid = std::fabs(rg.mid);
  // hot loop (fp32): candidates are the pairs inside the sphere about the rounded window
  // centre c~ = fl(2(p + mid n))/2 that contains the region cylinder (|beta - mid| <= h,
  // alpha^2 <= Qmax), margin m = B.x - |x|^2 + K with B = 2c~, K = rho^2 - |c~|^2 + 2E
  // (DESIGN.md 7.1).  |c~ - c'| <= u (X + |mid|) widens the radius.
  // Two BRUTE filters share the margin: packed fp32 (FFMA2) and the tensor cores (tf32
  // mma.sync), whose operands B and K are rounded to tf32: |c~ - c'| <= 2^-11 |c'|.
  // fp32 error: 5u per term magnitude.  Tensor cores (x, y, z split into tf32 hi + lo,
  // w = -|x|^2 and K rounded to tf32, exact products, fp32 accumulation): 2^-21 |B||x| +
  // 2^-11 (|x|^2 + |K|) (round to nearest at 11 significant bits) plus an accumulation
  // allowance of 2^-19 of the summed magnitudes
  // (and 2^-100 absolute for flushed subnormals).  E bounds the filter in use, so every
  // region pair keeps m > 0.  The tensor cores are used unless their
  // looser bound grows the candidate sphere by more than 25% (clouds far from the origin
  // relative to the region size; the packed-fp32 filter has neither the pre-pass nor the
  // dense tiles, so the tensor cores win well beyond the 6% of round 1)
  auto sphere = [&](bool mma, double& rho_o, double& E_o) {
    const double shift = 1.01 * (mma ? std::ldexp(1.0, -11) : u) * (X + amid);
    rho_o = std::sqrt(rg.h * rg.h + rg.Qmax) + shift;
    const double Ms = rho_o * rho_o + (2.0 * X + amid) * (2.0 * X + amid) * 1.01;
    E_o = 6.0 * u * Ms * 1.05;
    if (mma) {
      const double Kmax = 1.05 * (rho_o * rho_o + (X + amid) * (X + amid)) + 4.0 * E_o;
      const double BX = 2.02 * (X + amid) * X;
      E_o += 1.01 * (std::ldexp(1.0, -21) * BX + std::ldexp(1.0, -11) * (X * X + Kmax) +
                     std::ldexp(1.0, -19) * (BX + X * X + Kmax)) + std::ldexp(1.0, -100);
    }
  };
  double rho, E_sph, rho_f, E_f;
  sphere(true, rho, E_sph);
  sphere(false, rho_f, E_f);
  const bool use_mma = prune == SPIN_BRUTE && std::getenv("SPIN_NO_MMA") == nullptr &&
                       rho * rho + 3.0 * E_sph <= 1.25 * (rho_f * rho_f + 3.0 * E_f);
  if (!use_mma) {
    rho = rho_f;
    E_sph = E_f;
  }
  const double shift = 1.01 * (use_mma ? std::ldexp(1.0, -11) : u) * (X + amid);
  const double Es_h = 4.0 * u * 1.01;
  // CELLS hot loop: the region cylinder in expanded forms (bounds hold inside the region)
  const double Eb_h = 8.0 * u * (X + amid) * 1.01;
  const double Et_h = 16.0 * u * (X + amid) * (X + amid) * 1.01;
  const double Eq_h = Et_h + Eb_h * (2.0 * rg.h + Eb_h) + 2.0 * u * (rg.Qmax + 2.0 * (X + amid) * (X + amid));
  p.b = b;
  p.cos_As = has_support ? cos_As : -INFINITY;
  p.A = 0.5 * W;
  p.mid = rg.mid;
  p.Qmax = rg.Qmax;
  p.rho2 = rho * rho;
  p.E_sph = E_sph;
  p.mma = use_mma ? 1 : 0;
  p.Eq_hot = Eq_h;
  p.h_test = f32_up(rg.h + Eb_h);
  p.c_test = has_support ? f32_down(cos_As - Es_h) : -INFINITY;
  p.has_support = has_support ? 1 : 0;
  // where the support test runs (same images either way): not at all without one; in the
  // accept path only (SPIN_F_SUPPORT_LAST); on every pair (SPIN_F_SUPPORT_FIRST, and CELLS
  // by default); BRUTE by default adaptively per warp (2)
  p.support_in_hot = !has_support ? 0
                     : (flags & SPIN_F_SUPPORT_LAST) ? 0
                     : (flags & SPIN_F_SUPPORT_FIRST) ? 1
                     : (prune == SPIN_BRUTE ? 2 : 1);
  // candidates satisfy |d| <= D.  BRUTE: |x - c~|^2 <= rho^2 + 4E, so
  // |d| <= |c~ - p| + sqrt(rho^2 + 4E).  CELLS: q <= Qmax + 2Eq, |beta| <= |mid| + h_test + Eb.
  const double Dh = (amid + shift + std::sqrt(rho * rho + 4.0 * E_sph)) * 1.001;
  const double Cmax = (X + amid) * (X + amid) * 1.01;
  const double bmax = amid + (double)p.h_test + Eb_h;
  const double D2c = (rg.Qmax + 2.0 * Eq_h + 4.0 * u * (rg.Qmax + Cmax) + bmax * bmax) * 1.001;
  const double D2 = (prune == SPIN_BRUTE ? Dh * Dh : D2c) + 1e-30;
  const double D = std::sqrt(D2);
  // accept path, fp32 direct forms, valid while |d| <= D
  const double Es_a = 5.5 * u * 1.01;
  const double Eb_a = 4.2 * u * D * 1.002;
  const double Edd_a = 5.2 * u * D2;
  const double Eq_a = Edd_a + Eb_a * (2.0 * D + Eb_a) + 1.01 * u * D2;
  double Eu_a;
  if (!(flags & SPIN_F_LITERAL_HALF_WIDTH))
    Eu_a = ((Eb_a + 1.01 * u * D) / b + u * (p.A + D / b)) * 1.01;
  else  // u = fma(-beta, fl(1/b), fl(W/(2b))): rounding of both constants and the fma
    Eu_a = (Eb_a + 4.01 * u * (p.A + D)) / b * 1.05;
  const double Ew_a = (Eq_a + 2.01 * u * D2) / (b * b) * 1.01;
  p.c_f = has_support ? (float)cos_As : -INFINITY;
  p.inv_b = (float)(1.0 / b);
  p.inv_b2 = (float)(1.0 / (b * b));
  p.Af = (float)p.A;
  p.Wf = (float)W;
  p.Au = (flags & SPIN_F_LITERAL_HALF_WIDTH) ? (float)(p.A / b) : (float)p.A;
  p.floor_f = (flags & SPIN_F_FLOOR_BINS) ? 1.0f : 0.0f;
  p.Wff = (float)W + p.floor_f;
  p.bin_magic = 8388608.0f - p.floor_f * ((float)W + 1.0f);
  p.Es_a = f32_up(Es_a);
  p.Eu_a = f32_up(Eu_a);
  p.Ew_a = f32_up(Ew_a);
  p.D2g = f32_down(D2);
  p.literal = (flags & SPIN_F_LITERAL_HALF_WIDTH) ? 1 : 0;
  p.floor_bins = (flags & SPIN_F_FLOOR_BINS) ? 1 : 0;
  p.no_fast_cert = (flags & SPIN_F_NO_FAST_CERT) ? 1 : 0;
  // BRUTE tensor-core tiles go lane-per-centre when they hold >= dense_min candidates per
  // live point (measured)
  p.dense_min = (flags & SPIN_F_NO_DENSE) ? 0 : 8;
#ifdef SPIN_MEASURE
  if (const char* dbg = std::getenv("SPIN_DEBUG_SKIP")) p.debug_skip = std::atoi(dbg);   // measurement builds only
  if (const char* dm = std::getenv("SPIN_DENSE_MIN")) p.dense_min = std::atoi(dm);
#endif
  // self pair (d = 0): beta = q = 0 exactly, u = W/2 (scaled reading only)
  p.self_fast = p.literal ? 0 : 1;
  if (mode == SPIN_NEAREST) {
    const int k = p.floor_bins ? (int)std::floor(p.A) : (int)std::ceil(p.A);
    p.self_k = (k >= 0 && k < W) ? k : -1;
    p.self_kf = (float)p.self_k;
    p.self_l = 0;
    p.self_a = 0.f;
  } else {
    const double i0 = std::floor(p.A);
    const bool in = p.A >= 0.0 && p.A < W - 1.0;
    p.self_k = in ? (int)i0 : -1;
    p.self_l = 0;
    p.self_a = (float)(p.A - i0);
  }
  if (!(Eu_a < 0.25 && Ew_a < 0.25)) p.no_fast_cert = 1;  // fp32 cannot resolve bins: skip it
  if (p.no_fast_cert) p.D2g = -1.0f;   // the fp32 stage certifies nothing (decide: dd <= D2g fails)

}

spin_status ensure_grid(spin_ctx* h, float R, cudaStream_t s, double* build_ms) {
  // cell edge R/8 (with the per-row chord hulls and the fine centre order,
  // measured against R/3 .. R/16: C3 41.9, C5 152.4, C5 W=24 561.7 ms at R/8, 42.4 /
  // 159.0 / 570.2 at R/4); grow it if the grid would exceed 2^24 cells
  double hh = 0.125 * R;
#ifdef SPIN_MEASURE
  if (const char* c = std::getenv("SPIN_DEBUG_CELLS_PER_R")) hh = R / std::atof(c);   // measurement builds only
#endif
  const double ex = std::max(1e-30, (double)h->aabb[3] - h->aabb[0]);
  const double ey = std::max(1e-30, (double)h->aabb[4] - h->aabb[1]);
  const double ez = std::max(1e-30, (double)h->aabb[5] - h->aabb[2]);
  while ((ex / hh + 2) * (ey / hh + 2) * (ez / hh + 2) > (double)(1 << 24)) hh *= 1.25;
  const float hf = (float)hh;
  if (h->grid_valid && h->grid_version == h->cloud_version && h->grid_h == hf) {
    *build_ms = 0.0;
    return SPIN_OK;
  }
  h->ox = h->aabb[0];
  h->oy = h->aabb[1];
  h->oz = h->aabb[2];
  h->inv_h = (float)(1.0 / hh);
  h->h_cell = (float)hh;
  auto dim = [&](float lo, float hi) {
    const float t = (hi - lo) * h->inv_h;  // same rounding as the device cell_coord
    return (int)std::floor(t) + 1;
  };
  h->dx = dim(h->aabb[0], h->aabb[3]);
  h->dy = dim(h->aabb[1], h->aabb[4]);
  h->dz = dim(h->aabb[2], h->aabb[5]);
  const int64_t ncells = (int64_t)h->dx * h->dy * h->dz;
  spin_status st;
  if ((st = ensure(h->cell_start, h->cell_start_cap, ncells + 1, "cell_start")) != SPIN_OK) return st;
  if ((st = ensure(h->counts, h->counts_cap, std::max<int64_t>(ncells, 1 << 18), "counts")) != SPIN_OK) return st;
  if ((st = ensure(h->cursor, h->cursor_cap, std::max<int64_t>(ncells, 1 << 18), "cursor")) != SPIN_OK) return st;
  if ((st = ensure(h->scan_tmp, h->scan_tmp_cap, (int64_t)scan_tmp_elems(std::max<int64_t>(ncells, 1 << 18)) + 1, "scan_tmp")) != SPIN_OK) return st;
  if ((st = ensure(h->keys, h->keys_cap, h->N, "keys")) != SPIN_OK) return st;
  if ((st = ensure(h->spos, h->spos_cap, h->Npad, "spos")) != SPIN_OK) return st;
  if ((st = ensure(h->snrm, h->snrm_cap, h->Npad, "snrm")) != SPIN_OK) return st;
  CK(cudaEventRecord(h->evg0, s), "event");
  CK(launch_cell_build(h->pos, h->nrm, (int32_t)h->N, (int32_t)h->Npad, h->ox, h->oy, h->oz,
                       h->inv_h, h->dx, h->dy, h->dz, h->keys, h->counts, h->cell_start,
                       h->cursor, h->scan_tmp, h->spos, h->snrm, s),
     "cell build");
  CK(cudaEventRecord(h->evg1, s), "event");
  *build_ms = -1.0;  // measured later if stats are requested
  h->grid_valid = true;
  h->grid_version = h->cloud_version;
  h->grid_h = hf;
  return SPIN_OK;
}

}  // namespace

extern "C" {

int32_t spin_abi_version(void) { return SPIN_ABI_VERSION; }
const char* spin_last_error(void) { return g_err.c_str(); }

double spin_cos_from_degrees(double deg) {
  if (deg >= 180.0) return -INFINITY;
  if (deg == 0.0) return 1.0;
  if (deg == 60.0) return 0.5;
  if (deg == 90.0) return 0.0;
  if (deg == 120.0) return -0.5;
  return std::cos(deg * (M_PI / 180.0));
}

spin_status spin_count_in_sphere(spin_handle h, const int32_t* d_centre_idx, int64_t M, double R,
                                 int64_t* count, spin_stream stream) {
  if (!h || !count) return fail(SPIN_E_INVAL, "null handle or count");
  if (h->N <= 0) return fail(SPIN_E_INVAL, "no valid cloud loaded (the last spin_load_cloud failed)");
  if (M < 0 || M >= ((int64_t)1 << 31)) return fail(SPIN_E_INVAL, "M=%lld out of range", (long long)M);
  if (!std::isfinite(R) || R <= 0.0 || R > 1e30) return fail(SPIN_E_INVAL, "R=%g must be positive and finite", R);
  *count = 0;
  if (M == 0) return SPIN_OK;
  if (!d_centre_idx) return fail(SPIN_E_INVAL, "null d_centre_idx");
  cudaStream_t s = (cudaStream_t)stream;
  const float R_up = (float)(R * (1.0 + 1e-6));
  double gms = 0.0;
  spin_status st = ensure_grid(h, R_up, s, &gms);
  if (st != SPIN_OK) return st;
  unsigned long long* d_cnt = (unsigned long long*)h->stats;   // scratch slot, zeroed below
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s), "memset");
  CK(launch_count_in_sphere(d_centre_idx, M, h->pos, (int32_t)h->N, h->spos, h->cell_start, h->ox,
                            h->oy, h->oz, h->inv_h, h->dx, h->dy, h->dz, R, R_up, d_cnt, h->sms, s),
     "count kernel");
  unsigned long long c = 0;
  CK(cudaMemcpyAsync(&c, d_cnt, sizeof c, cudaMemcpyDeviceToHost, s), "count readback");
  CK(cudaStreamSynchronize(s), "count sync");
  *count = (int64_t)c;
  return SPIN_OK;
}

spin_status spin_pair_codes(spin_handle h, const int32_t* d_centre_idx, int64_t M, int32_t W,
                            double b, double cos_As, spin_mode mode, uint32_t flags,
                            int32_t* d_codes, spin_stream stream) {
  if (!h) return fail(SPIN_E_INVAL, "null handle");
  if (h->N <= 0) return fail(SPIN_E_INVAL, "no valid cloud loaded (the last spin_load_cloud failed)");
  if (M < 0 || M >= ((int64_t)1 << 31)) return fail(SPIN_E_INVAL, "M=%lld out of range", (long long)M);
  if (W < 1 || W > 64) return fail(SPIN_E_INVAL, "W=%d outside [1, 64]", W);
  if (mode != SPIN_NEAREST && mode != SPIN_BILINEAR) return fail(SPIN_E_INVAL, "bad mode %d", (int)mode);
  if (mode == SPIN_BILINEAR && W < 2) return fail(SPIN_E_INVAL, "BILINEAR needs W >= 2");
  if (!std::isfinite(b) || b < 1e-30 || b > 1e30) return fail(SPIN_E_INVAL, "b=%g must be finite in [1e-30, 1e30]", b);
  const bool has_support = !(std::isinf(cos_As) && cos_As < 0);
  if (has_support && !(cos_As >= -1.0 && cos_As <= 1.0))
    return fail(SPIN_E_INVAL, "cos_As=%g must be in [-1, 1] or -inf", cos_As);
  if (flags & ~0xffu) return fail(SPIN_E_INVAL, "unknown flag bits 0x%x", flags);
  if (M == 0) return SPIN_OK;
  if (!d_centre_idx || !d_codes) return fail(SPIN_E_INVAL, "null d_centre_idx or d_codes");
  const Region rg = region_of(W, b, (int)mode, flags);
  KParams p{};
  plan_thresholds(h, W, b, cos_As, has_support, mode, SPIN_BRUTE, flags, rg, p);
  p.cpos = h->pos;
  p.cnrm = h->nrm;
  p.pos = h->pos;
  p.nrm = h->nrm;
  p.N = (int32_t)h->N;
  p.W = W;
  p.err_flags = h->err;
  CK(launch_pair_codes(p, (int)mode, d_centre_idx, M, d_codes, (cudaStream_t)stream), "pair codes");
  return SPIN_OK;
}

double spin_region_radius(int32_t W, double b, spin_mode mode, uint32_t flags) {
  return region_of(W, b, (int)mode, flags).R;
}

spin_status spin_chunk_sequence(spin_schedule sched, int64_t n_units, int32_t P,
                                const spin_chunk_params* cp, int64_t* h_bounds, int64_t cap,
                                int64_t* n_chunks) {
  if (P < 1) return fail(SPIN_E_INVAL, "P=%d must be >= 1", P);
  if (n_units < 0) return fail(SPIN_E_INVAL, "n_units must be >= 0");
  if (sched < SPIN_STATIC || sched > SPIN_WF)
    return fail(SPIN_E_INVAL, sched == SPIN_AWF ? "AWF weights are measured at run time: no static trace"
                                                : "bad schedule %d", (int)sched);
  spin_chunk_params d{};
  if (cp) d = *cp;
  if (d.gss_min_chunk < 0 || d.fac_divisor < 0) return fail(SPIN_E_INVAL, "negative chunk parameter");
  std::vector<int64_t> b;
  build_bounds(sched, n_units, P, d.gss_min_chunk ? d.gss_min_chunk : 1,
               d.fac_divisor ? d.fac_divisor : 2, b, d.slow_ctas, d.slowdown);
  if (n_chunks) *n_chunks = (int64_t)b.size() - 1;
  if ((int64_t)b.size() > cap || !h_bounds)
    return fail(SPIN_E_RANGE, "need %lld bound entries, cap is %lld", (long long)b.size(), (long long)cap);
  std::memcpy(h_bounds, b.data(), b.size() * sizeof(int64_t));
  return SPIN_OK;
}

int32_t spin_default_P(int32_t W, spin_mode mode, spin_prune prune) {
  if (W < 1 || W > 64) return -1;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const LaunchCfg lc = choose_launch(W, (int)mode, (int)prune, false);
  return resident_workers(lc, W, (int)mode, (int)prune, sms);
}

spin_status spin_create(const float* points, const float* normals, int64_t N, spin_stream stream,
                        spin_handle* out) {
  if (!out) return fail(SPIN_E_INVAL, "out handle pointer is null");
  *out = nullptr;
  spin_ctx* h = new (std::nothrow) spin_ctx();
  if (!h) return fail(SPIN_E_NOMEM, "host allocation failed");
  cudaStream_t s = (cudaStream_t)stream;
  auto bail = [&](spin_status st) { spin_destroy(h); return st; };
  if (cudaGetDevice(&h->dev) != cudaSuccess) return bail(fail(SPIN_E_CUDA, "no CUDA device"));
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev);
  if (cudaMalloc((void**)&h->counter, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc((void**)&h->stats, ST_NSLOTS * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc((void**)&h->err, 4 * sizeof(int32_t)) != cudaSuccess ||
      cudaMallocHost((void**)&h->h_err, 4 * sizeof(int32_t)) != cudaSuccess ||
      cudaMalloc((void**)&h->red, 8 * sizeof(int32_t)) != cudaSuccess ||
      cudaMallocHost((void**)&h->h_red, 8 * sizeof(int32_t)) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(SPIN_E_NOMEM, "handle allocation failed"));
  }
  if (cudaMemset(h->err, 0, 4 * sizeof(int32_t)) != cudaSuccess)
    return bail(fail(SPIN_E_CUDA, "memset failed"));
  std::memset(h->h_err, 0, 4 * sizeof(int32_t));
  cudaEventCreateWithFlags(&h->ev_err, cudaEventDisableTiming);
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);
  cudaEventCreate(&h->evg0);
  cudaEventCreate(&h->evg1);
  spin_status st = load_cloud(h, points, normals, N, s);
  if (st != SPIN_OK) return bail(st);
  *out = h;
  return SPIN_OK;
}

spin_status spin_load_cloud(spin_handle h, const float* points, const float* normals, int64_t N,
                            spin_stream stream) {
  if (!h) return fail(SPIN_E_INVAL, "null handle");
  return load_cloud(h, points, normals, N, (cudaStream_t)stream);
}

void spin_destroy(spin_handle h) {
  if (!h) return;
  void* ptrs[] = {h->pos, h->nrm, h->tpos, h->bpos, h->bnrm, h->tfa, h->mfrag, h->mk0, h->mk1, h->mv0, h->mperm, h->mtemp, h->cell_start, h->spos, h->snrm, h->keys, h->counts,
                  h->cursor, h->scan_tmp, h->ckeys, h->cstarts, h->order, h->bounds,
                  h->counter, h->stats, h->err, h->cta_t0, h->cta_t1, h->cta_units, h->cidx,
                  h->outbuf, h->stage_p, h->stage_n, h->red, h->hi_scratch, h->seg_done,
                  h->wf_state};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->h_err) cudaFreeHost(h->h_err);
  if (h->h_red) cudaFreeHost(h->h_red);
  cudaEvent_t evs[] = {h->ev_err, h->ev0, h->ev1, h->evg0, h->evg1, h->ev_seg0};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  delete h;
}

spin_status spin_generate(spin_handle h, const int32_t* d_centre_idx, int64_t M, int32_t W,
                          double b, double cos_As, spin_schedule sched,
                          const spin_chunk_params* cp, spin_mode mode, spin_prune prune,
                          float* d_out, spin_stats* stats, spin_stream stream) {
  if (!h) return fail(SPIN_E_INVAL, "null handle");
  if (h->N <= 0) return fail(SPIN_E_INVAL, "no valid cloud loaded (the last spin_load_cloud failed)");
  cudaStream_t s = (cudaStream_t)stream;
  // inside a stream capture (CUDA graphs) nothing may synchronise or query events: the
  // deferred error report is skipped and stats are refused
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) cap = cudaStreamCaptureStatusNone;
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (capturing && stats) return fail(SPIN_E_INVAL, "stats synchronise the stream: not inside a stream capture");
  // ---- a deferred SPIN_E_RANGE / overflow from an earlier asynchronous call
  // (the device word is sticky: every call's readback carries the flags of all calls since
  // the last report, so a flag whose own readback was never inspected is not lost)
  if (!capturing && h->err_pending && cudaEventQuery(h->ev_err) == cudaSuccess) {
    h->err_pending = false;
    if (h->h_err[0] || h->h_err[1]) {
      const bool range = h->h_err[0] != 0;
      h->h_err[0] = h->h_err[1] = 0;
      CK(cudaMemsetAsync(h->err, 0, 2 * sizeof(int32_t), s), "memset");
      return range ? fail(SPIN_E_RANGE, "an earlier call saw a centre index outside [0, N)")
                   : fail(SPIN_E_OVERFLOW, "an earlier call overflowed a bin accumulator");
    }
  }
  // ---- synchronous argument checks (§8(b) SPIN_E_INVAL)
  if (M < 0) return fail(SPIN_E_INVAL, "M=%lld must be >= 0", (long long)M);
  if (M >= ((int64_t)1 << 31)) return fail(SPIN_E_INVAL, "M=%lld must be < 2^31", (long long)M);
  if (W < 1 || W > 64) return fail(SPIN_E_INVAL, "W=%d outside [1, 64]", W);
  if (mode != SPIN_NEAREST && mode != SPIN_BILINEAR) return fail(SPIN_E_INVAL, "bad mode %d", (int)mode);
  if (mode == SPIN_BILINEAR && W < 2) return fail(SPIN_E_INVAL, "BILINEAR needs W >= 2");
  if (prune != SPIN_BRUTE && prune != SPIN_CELLS) return fail(SPIN_E_INVAL, "bad prune %d", (int)prune);
  if (sched < SPIN_STATIC || sched > SPIN_AWF) return fail(SPIN_E_INVAL, "bad schedule %d", (int)sched);
  if (!std::isfinite(b) || b < 1e-30 || b > 1e30) return fail(SPIN_E_INVAL, "b=%g must be finite in [1e-30, 1e30]", b);
  const bool has_support = !(std::isinf(cos_As) && cos_As < 0);
  if (has_support && !(cos_As >= -1.0 && cos_As <= 1.0))
    return fail(SPIN_E_INVAL, "cos_As=%g must be in [-1, 1] or -inf", cos_As);
  spin_chunk_params cpar{};
  if (cp) cpar = *cp;
  if (cpar.P < 0 || cpar.unit < 0 || cpar.gss_min_chunk < 0 || cpar.fac_divisor < 0 ||
      cpar.grid < 0 || cpar.cta_offset < 0)
    return fail(SPIN_E_INVAL, "negative chunk parameter");
  if (cpar.flags & ~0xffu) return fail(SPIN_E_INVAL, "unknown flag bits 0x%x", cpar.flags);
  if (cpar.slow_ctas < 0 || !(cpar.slowdown == 0.0f || (cpar.slowdown >= 1.0f && cpar.slowdown <= 1e6f)))
    return fail(SPIN_E_INVAL, "slow_ctas must be >= 0 and slowdown 0 or in [1, 1e6]");
  if ((cpar.flags & SPIN_F_SUPPORT_LAST) && (cpar.flags & SPIN_F_SUPPORT_FIRST))
    return fail(SPIN_E_INVAL, "SPIN_F_SUPPORT_LAST and SPIN_F_SUPPORT_FIRST are exclusive");
  if (M > 0 && (!d_centre_idx || !d_out)) return fail(SPIN_E_INVAL, "null d_centre_idx or d_out with M > 0");
  if (stats) {
    stats->elapsed_ms = stats->grid_build_ms = 0.0;
    stats->pairs_visited = stats->pairs_candidate = stats->pairs_accepted = 0;
    stats->fp64_fallbacks = stats->exact_fallbacks = 0;
    stats->P = stats->G = stats->n_units = stats->n_chunks = 0;
    stats->cta_per_worker = 1;
  }
  if (M == 0) return SPIN_OK;

  // ---- launch shape, P, units, chunk table (a3)
  const bool wf = sched == SPIN_WF || sched == SPIN_AWF;   // dealt on the device by CAS
  // a worker is one CTA, or on request (SPIN_F_CLUSTER_PAIR; BRUTE, table dealer, one
  // device, no slow-worker emulation) a two-CTA cluster sharing a group of centres
  //
  // (NEAREST only: its partner adds are fire-and-forget DSMEM reductions, C4 NEAREST 376 ->
  // 343 ms; BILINEAR's fixed-point carries need the old value back, and four returning DSMEM
  // atomics per splat made C4 BILINEAR slower, 405 -> 529 ms)
  const bool allow_cluster = (cpar.flags & SPIN_F_CLUSTER_PAIR) && prune == SPIN_BRUTE &&
                             mode == SPIN_NEAREST && !wf && !cpar.d_counter &&
                             cpar.grid == 0 && cpar.cta_offset == 0 &&
                             !(cpar.slowdown > 1.0f && cpar.slow_ctas > 0);
  const LaunchCfg lc = choose_launch(W, (int)mode, (int)prune, allow_cluster);
  const int workers = resident_workers(lc, W, (int)mode, (int)prune, h->sms);
  if (workers <= 0) return fail(SPIN_E_CUDA, "kernel does not fit on the device (smem %zu)", lc.smem);
  const int P = cpar.P > 0 ? cpar.P : workers;          // workers of the schedule
  if (P > 1 << 20) return fail(SPIN_E_INVAL, "P=%d too large", P);
  const int grid = cpar.grid > 0 ? cpar.grid : P * lc.cl;   // CTAs on this device
  if ((int64_t)cpar.cta_offset + grid / lc.cl > P)
    return fail(SPIN_E_INVAL, "cta_offset %d + grid %d exceeds P %d", cpar.cta_offset, grid, P);
  const int unit = cpar.unit > 0 ? cpar.unit : lc.G;
  const int64_t n_units = (M + unit - 1) / unit;
  const int gmin = cpar.gss_min_chunk ? cpar.gss_min_chunk : 1;
  const int fdiv = cpar.fac_divisor ? cpar.fac_divisor : 2;
  if (wf && (n_units >= (1 << 24) || P >= (1 << 16) || cpar.d_counter))
    return fail(SPIN_E_INVAL, "WF/AWF need n_units < 2^24 (have %lld), P < 2^16 (have %d) and no shared dealer",
                (long long)n_units, P);
  const long long key[6] = {(long long)sched, (long long)n_units, P, gmin, fdiv, 1};
  if (!wf && !std::equal(key, key + 6, h->bounds_key)) {
    build_bounds(sched, n_units, P, gmin, fdiv, h->bounds_h);
    std::vector<int32_t> b32(h->bounds_h.begin(), h->bounds_h.end());
    spin_status st = ensure(h->bounds, h->bounds_cap, (int64_t)b32.size(), "chunk table");
    if (st != SPIN_OK) return st;
    CK(cudaMemcpyAsync(h->bounds, b32.data(), b32.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s), "chunk table");
    CK(cudaStreamSynchronize(s), "chunk table");  // b32 is a temporary
    std::copy(key, key + 6, h->bounds_key);
  }
  const int n_chunks = wf ? 0 : (int)h->bounds_h.size() - 1;
  if (wf) {   // packed batch state (u64) + per-CTA measured rates (AWF)
    spin_status st = ensure(h->wf_state, h->wf_cap, 2 + grid, "WF dealer state");
    if (st != SPIN_OK) return st;
    CK(cudaMemsetAsync(h->wf_state, 0, (2 + grid) * sizeof(unsigned long long), s), "memset");
  }
  if (h->cta_cap < grid) {
    if (h->cta_t0) cudaFree(h->cta_t0);
    if (h->cta_t1) cudaFree(h->cta_t1);
    if (h->cta_units) cudaFree(h->cta_units);
    h->cta_t0 = h->cta_t1 = nullptr;
    h->cta_units = nullptr;
    h->cta_cap = 0;
    if (cudaMalloc((void**)&h->cta_t0, grid * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void**)&h->cta_t1, grid * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc((void**)&h->cta_units, grid * sizeof(int32_t)) != cudaSuccess) {
      cudaGetLastError();
      return fail(SPIN_E_NOMEM, "per-CTA instrumentation allocation failed");
    }
    h->cta_cap = grid;
  }

  // ---- a2: region constants and certified thresholds
  const uint32_t flags = cpar.flags;
  const Region rg = region_of(W, b, (int)mode, flags);
  KParams p{};
  plan_thresholds(h, W, b, cos_As, has_support, mode, prune, flags, rg, p);

  // ---- cloud, centres, dealing, outputs
  p.cpos = h->pos;
  p.cnrm = h->nrm;
  p.N = (int32_t)h->N;
  p.centre_idx = d_centre_idx;
  p.order = nullptr;
  p.M = M;
  p.W = W;
  p.out = d_out;
  p.bounds = h->bounds;
  p.n_chunks = n_chunks;
  p.unit_images = unit;
  p.is_static = sched == SPIN_STATIC ? 1 : 0;
  p.wf = sched == SPIN_WF ? 1 : sched == SPIN_AWF ? 2 : 0;
  if (wf) {
    p.wf_state = h->wf_state;
    p.awf_rate = reinterpret_cast<float*>(h->wf_state + 2);
    p.n_units = (int32_t)n_units;
    p.fac_div = fdiv;
    p.P = P;
    wf_weights(P, cpar.slowdown > 1.0f ? cpar.slow_ctas : 0, cpar.slowdown, &p.wq_slow, &p.wq_fast);
  }
  p.cta_offset = cpar.cta_offset;
  p.slow_ctas = cpar.slowdown > 1.0f ? std::min(cpar.slow_ctas, grid) : 0;
  p.slowdown = cpar.slowdown > 1.0f ? cpar.slowdown : 1.0f;
  // (the wait needs every slow CTA resident: only for a persistent launch)
  p.slow_first = (cpar.slow_first && !p.is_static && grid / lc.cl <= workers && !cpar.d_counter) ? 1 : 0;
  p.counter = cpar.d_counter ? cpar.d_counter : h->counter;
  p.stats = h->stats;
  p.cta_t0 = h->cta_t0;
  p.cta_t1 = h->cta_t1;
  p.cta_units = h->cta_units;
  p.err_flags = h->err;
  if (mode == SPIN_BILINEAR) {
    const int64_t need = (int64_t)grid * lc.G * ((W * W + 1) / 2);
    if (need > h->hi_cap) {
      spin_status st = ensure(h->hi_scratch, h->hi_cap, need, "carry scratch");
      if (st != SPIN_OK) return st;
      CK(cudaMemsetAsync(h->hi_scratch, 0, need * sizeof(uint32_t), s), "memset");
    }
    p.hi_scratch = h->hi_scratch;
  }
  p.row_cap = 256;
  double grid_ms = 0.0;
  if (prune == SPIN_BRUTE) {
    p.pos = h->bpos;
    p.nrm = h->bnrm;
    p.tpos = h->tpos;
    p.tfa = h->tfa;
    p.mfrag = h->mfrag;
    p.n_tiles = (int32_t)((h->N + lc.threads * KP_POINTS - 1) / (lc.threads * KP_POINTS));
    if (!(flags & SPIN_F_NO_SORT)) {
      // a5: centres in the cloud's Morton order, so that a group's G centres are neighbours
      // and their candidates fill few warp tiles (stable sort: the same order on every device)
      spin_status st = ensure_morton_scratch(h, M);
      if (st == SPIN_OK) st = ensure(h->order, h->order_cap, M, "centre order");
      if (st != SPIN_OK) return st;
      CK(launch_morton_order(d_centre_idx, M, h->pos, (int32_t)h->N, h->mgrid, h->mk0, h->mk1, h->mv0,
                             h->order, h->mtemp, (size_t)h->mtemp_cap, s),
         "centre Morton order");
      p.order = h->order;
    }
  } else {
    const float R = f32_up(rg.R * (1.0 + 1e-6) + 1e-30);
    spin_status st = ensure_grid(h, R, s, &grid_ms);
    if (st != SPIN_OK) return st;
    p.pos = h->spos;
    p.nrm = h->snrm;
    p.cell_start = h->cell_start;
    p.dimx = h->dx; p.dimy = h->dy; p.dimz = h->dz;
    p.ox = h->ox; p.oy = h->oy; p.oz = h->oz;
    p.inv_h = h->inv_h;
    p.h_cell = h->h_cell;
    p.R_up = R;
    if (!(flags & SPIN_F_NO_SORT)) {
      // centre keys: Morton codes of a grid of up to 2^ob cells per axis — coarser than
      // the cell grid (shift) or finer (sub-cell refinement sub), so that G consecutive
      // centres of a dense region form a compact group (C5: 2^8 per axis cuts the visited
      // pairs by 16% and the time by 6% against 2^6); ob grows with M so the 2^(3 ob)
      // counting-sort buckets stay within 64 M
      int ob = 6;
      while (ob < 8 && ((int64_t)1 << (3 * (ob + 1))) <= 64 * M) ++ob;
#ifdef SPIN_MEASURE
      if (const char* e = std::getenv("SPIN_ORDER_BITS")) ob = std::min(std::max(std::atoi(e), 1), 8);
#endif
      int shift = 0, sub = 0;
      const int dmax = std::max(h->dx, std::max(h->dy, h->dz));
      while ((dmax >> shift) > (1 << ob)) ++shift;
      while (shift == 0 && (dmax << (sub + 1)) <= (1 << ob)) ++sub;
      int bits = 0;
      while ((1 << bits) < (((dmax << sub) - 1) >> shift) + 1) ++bits;
      bits = std::max(bits, 1);
      const int64_t nb = (int64_t)1 << (3 * bits);
      if ((st = ensure(h->ckeys, h->ckeys_cap, M, "centre keys")) != SPIN_OK) return st;
      if ((st = ensure(h->order, h->order_cap, M, "centre order")) != SPIN_OK) return st;
      if ((st = ensure(h->cstarts, h->cstarts_cap, nb + 1, "centre buckets")) != SPIN_OK) return st;
      if ((st = ensure(h->counts, h->counts_cap, nb, "counts")) != SPIN_OK) return st;
      if ((st = ensure(h->cursor, h->cursor_cap, nb, "cursor")) != SPIN_OK) return st;
      if ((st = ensure(h->scan_tmp, h->scan_tmp_cap, (int64_t)scan_tmp_elems(nb) + 1, "scan_tmp")) != SPIN_OK) return st;
      CK(launch_centre_order(d_centre_idx, M, h->pos, (int32_t)h->N, h->ox, h->oy, h->oz,
                             h->inv_h * (float)(1 << sub), h->dx << sub, h->dy << sub, h->dz << sub,
                             shift, bits, h->ckeys, h->counts,
                             h->cstarts, h->cursor, h->scan_tmp, h->order, s),
         "centre order");
      if (cpar.d_counter) {
        // a shared dealer needs the SAME chunk -> images map on every device; the device
        // scatter orders centres within a bucket by atomic arrival, so re-derive the
        // order as a stable counting sort of the same keys on the host (M ints each way)
        std::vector<int32_t> keys((size_t)M), ord((size_t)M), cnt((size_t)nb + 1, 0);
        CK(cudaMemcpyAsync(keys.data(), h->ckeys, M * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "keys");
        CK(cudaStreamSynchronize(s), "keys");
        for (int64_t m = 0; m < M; ++m) ++cnt[(size_t)keys[m] + 1];
        for (int64_t k = 0; k < nb; ++k) cnt[(size_t)k + 1] += cnt[(size_t)k];
        for (int64_t m = 0; m < M; ++m) ord[(size_t)cnt[(size_t)keys[m]]++] = (int32_t)m;
        CK(cudaMemcpyAsync(h->order, ord.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, s), "order");
        CK(cudaStreamSynchronize(s), "order");   // ord is a temporary
      }
      p.order = h->order;
    }
  }

  // ---- e2e pipelining armed by spin_generate_host (BRUTE: images leave in caller order)
  if (h->pipe_seg_images > 0 && p.order == nullptr) {
    const int64_t nseg = (M + h->pipe_seg_images - 1) / h->pipe_seg_images;
    spin_status st = ensure(h->seg_done, h->seg_cap, nseg, "segment counters");
    if (st != SPIN_OK) return st;
    CK(cudaMemsetAsync(h->seg_done, 0, nseg * sizeof(unsigned), s), "memset");
    CK(cudaEventRecord(h->ev_seg0, s), "event");
    p.seg_done = h->seg_done;
    p.seg_images = h->pipe_seg_images;
  } else {
    h->pipe_seg_images = 0;
  }

  // ---- a6-a13: the persistent launch
  if (!cpar.d_counter) CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned), s), "memset");
  CK(cudaMemsetAsync(h->stats, 0, ST_NSLOTS * sizeof(unsigned long long), s), "memset");
  if (!capturing) CK(cudaEventRecord(h->ev0, s), "event");
  CK(launch_spin(lc, (int)mode, (int)prune, grid, p, s), "spin kernel launch");
  if (!capturing) {
    CK(cudaEventRecord(h->ev1, s), "event");
    CK(cudaMemcpyAsync(h->h_err, h->err, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "err readback");
    CK(cudaEventRecord(h->ev_err, s), "event");
    h->err_pending = true;
  }

  if (stats) {
    CK(cudaStreamSynchronize(s), "stats sync");
    unsigned long long sv[ST_NSLOTS];
    CK(cudaMemcpy(sv, h->stats, sizeof sv, cudaMemcpyDeviceToHost), "stats");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    stats->elapsed_ms = ms;
    if (grid_ms < 0.0) {
      float gm = 0.f;
      cudaEventElapsedTime(&gm, h->evg0, h->evg1);
      stats->grid_build_ms = gm;
    }
    stats->pairs_visited = prune == SPIN_BRUTE ? M * h->N : (int64_t)sv[ST_VISITED];
    stats->pairs_candidate = (int64_t)sv[ST_CAND];
    stats->pairs_accepted = (int64_t)sv[ST_ACC];
    stats->fp64_fallbacks = (int64_t)sv[ST_F64];
    stats->exact_fallbacks = (int64_t)sv[ST_EXACT];
    stats->tiles_support_hot = (int64_t)sv[ST_SUPHOT];
    stats->tiles_dense = (int64_t)sv[ST_DENSE];
    stats->dense_rows = (int64_t)sv[ST_DROWS];
    stats->filter_mma = p.mma;
    stats->P = grid;
    stats->cta_per_worker = lc.cl;
    stats->G = lc.G;
    stats->n_units = (int32_t)n_units;
    stats->n_chunks = n_chunks;
    if (wf) {   // requests counted on the device; every CTA's last request finds no work
      unsigned requests = 0;
      CK(cudaMemcpy(&requests, h->counter, sizeof requests, cudaMemcpyDeviceToHost), "requests");
      stats->n_chunks = (int32_t)requests - grid;
    }
    const int nc = std::min(grid, stats->cta_capacity);
    if (nc > 0) {
      if (stats->h_cta_start_ns) CK(cudaMemcpy(stats->h_cta_start_ns, h->cta_t0, nc * 8, cudaMemcpyDeviceToHost), "cta");
      if (stats->h_cta_end_ns) CK(cudaMemcpy(stats->h_cta_end_ns, h->cta_t1, nc * 8, cudaMemcpyDeviceToHost), "cta");
      if (stats->h_cta_units) CK(cudaMemcpy(stats->h_cta_units, h->cta_units, nc * 4, cudaMemcpyDeviceToHost), "cta");
    }
    h->err_pending = false;
    if (h->h_err[0] || h->h_err[1]) {
      const bool range = h->h_err[0] != 0;
      h->h_err[0] = h->h_err[1] = 0;
      CK(cudaMemsetAsync(h->err, 0, 2 * sizeof(int32_t), s), "memset");
      return range ? fail(SPIN_E_RANGE, "a centre index is outside [0, N); its image is zero")
                   : fail(SPIN_E_OVERFLOW, "a bin accumulator overflowed");
    }
  }
  return SPIN_OK;
}

spin_status spin_dealer_alloc(uint32_t** d_counter) {
  if (!d_counter) return fail(SPIN_E_INVAL, "null d_counter");
  *d_counter = nullptr;
  CK(cudaMalloc((void**)d_counter, 256), "dealer alloc");
  CK(cudaMemset(*d_counter, 0, 256), "dealer zero");
  return SPIN_OK;
}

spin_status spin_dealer_ipc_handle(const uint32_t* d_counter, unsigned char handle[64]) {
  if (!d_counter || !handle) return fail(SPIN_E_INVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
  cudaIpcMemHandle_t hd;
  CK(cudaIpcGetMemHandle(&hd, (void*)d_counter), "dealer ipc handle");
  std::memcpy(handle, &hd, 64);
  return SPIN_OK;
}

spin_status spin_dealer_ipc_open(const unsigned char handle[64], uint32_t** d_counter) {
  if (!d_counter || !handle) return fail(SPIN_E_INVAL, "null argument");
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, 64);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess), "dealer ipc open");
  *d_counter = (uint32_t*)p;
  return SPIN_OK;
}

spin_status spin_dealer_reset(uint32_t* d_counter, spin_stream stream) {
  if (!d_counter) return fail(SPIN_E_INVAL, "null d_counter");
  CK(cudaMemsetAsync(d_counter, 0, sizeof(uint32_t), (cudaStream_t)stream), "dealer reset");
  return SPIN_OK;
}

spin_status spin_dealer_free(uint32_t* d_counter, int32_t opened) {
  if (!d_counter) return SPIN_OK;
  if (opened) CK(cudaIpcCloseMemHandle(d_counter), "dealer ipc close");
  else CK(cudaFree(d_counter), "dealer free");
  return SPIN_OK;
}

spin_status spin_generate_host(spin_handle h, const int32_t* h_centre_idx, int64_t M, int32_t W,
                               double b, double cos_As, spin_schedule sched,
                               const spin_chunk_params* cp, spin_mode mode, spin_prune prune,
                               float* h_out, spin_stats* stats, spin_stream stream) {
  if (!h) return fail(SPIN_E_INVAL, "null handle");
  if (M < 0) return fail(SPIN_E_INVAL, "M must be >= 0");
  if (M == 0) return spin_generate(h, nullptr, 0, W, b, cos_As, sched, cp, mode, prune, nullptr, stats, stream);
  if (!h_centre_idx || !h_out) return fail(SPIN_E_INVAL, "null host buffer");
  if (W < 1 || W > 64) return fail(SPIN_E_INVAL, "W=%d outside [1, 64]", W);
  if (cp && cp->d_counter)
    return fail(SPIN_E_INVAL, "a shared dealer (d_counter) needs device buffers: use spin_generate");
  cudaStream_t s = (cudaStream_t)stream;
  spin_status st;
  if ((st = ensure(h->cidx, h->cidx_cap, M, "centre scratch")) != SPIN_OK) return st;
  CK(cudaMemcpyAsync(h->cidx, h_centre_idx, M * sizeof(int32_t), cudaMemcpyHostToDevice, s), "H2D centres");
  // Page-locked (mapped) output: the kernel's write-back stores go straight to host memory
  // over the host link, overlapped with the groups still being computed, in any processing
  // order (BRUTE's Morton order, CELLS' cell order) -- no device copy, no D2H afterwards.
  {
    const size_t bytes = (size_t)M * W * W * sizeof(float);
    cudaPointerAttributes a0{}, a1{};
    const bool ok0 = cudaPointerGetAttributes(&a0, h_out) == cudaSuccess;
    const bool ok1 = cudaPointerGetAttributes(&a1, reinterpret_cast<const char*>(h_out) + bytes - 1) == cudaSuccess;
    cudaGetLastError();
    if (ok0 && ok1 && a0.type == cudaMemoryTypeHost && a1.type == cudaMemoryTypeHost && a0.devicePointer &&
        a1.devicePointer &&
        reinterpret_cast<const char*>(a1.devicePointer) - reinterpret_cast<const char*>(a0.devicePointer) ==
            (ptrdiff_t)(bytes - 1)) {
      st = spin_generate(h, h->cidx, M, W, b, cos_As, sched, cp, mode, prune,
                         reinterpret_cast<float*>(a0.devicePointer), stats, stream);
      if (st != SPIN_OK) return st;
      CK(cudaStreamSynchronize(s), "sync");
      return SPIN_OK;
    }
  }
  if ((st = ensure(h->outbuf, h->outbuf_cap, M * W * W, "image scratch")) != SPIN_OK) return st;
  // Pipeline the D2H of the images with the kernel: the kernel counts finished images
  // per output segment; a copy stream waits on each counter (cuStreamWaitValue32) and
  // copies that segment while later groups are still being computed.
  const size_t img_bytes = (size_t)W * W * sizeof(float);
  const bool pipe = prune == SPIN_BRUTE && (size_t)M * img_bytes >= ((size_t)8 << 20);
  if (pipe && h->stream_wait_ok != 0) {
    if (!h->copy_stream) {
      CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking), "copy stream");
      CK(cudaEventCreateWithFlags(&h->ev_seg0, cudaEventDisableTiming), "event");
    }
    if (h->stream_wait_ok < 0) {
      // the driver entry point through the runtime (libspin does not link libcuda)
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      h->stream_wait_ok = (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) ==
                               cudaSuccess && q == cudaDriverEntryPointSuccess && fn)
                              ? 1 : 0;
      h->wait_value32 = reinterpret_cast<WaitValue32Fn>(fn);
    }
  }
  const bool piped = pipe && h->stream_wait_ok == 1;
  // ~2 MB segments (16 .. 256): the last one is copied after the kernel ends
  const int32_t nseg_target = (int32_t)std::min<int64_t>(
      256, std::max<int64_t>(16, (int64_t)((size_t)M * img_bytes >> 21)));
  const int32_t seg_images = (int32_t)std::max<int64_t>(1, (M + nseg_target - 1) / nseg_target);
  h->pipe_seg_images = piped ? seg_images : 0;
  st = spin_generate(h, h->cidx, M, W, b, cos_As, sched, cp, mode, prune, h->outbuf, stats, stream);
  const bool armed = h->pipe_seg_images > 0;
  h->pipe_seg_images = 0;
  if (st != SPIN_OK) return st;
  if (armed) {
    CK(cudaStreamWaitEvent(h->copy_stream, h->ev_seg0, 0), "wait");
    for (int64_t a = 0, sg = 0; a < M; a += seg_images, ++sg) {
      const int64_t n = std::min<int64_t>(seg_images, M - a);
      if (h->wait_value32((CUstream)h->copy_stream, (CUdeviceptr)(h->seg_done + sg), (cuuint32_t)n,
                          CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
        // could not enqueue the wait: finish the remaining copy after the kernel instead
        CK(cudaStreamSynchronize(s), "sync");
        CK(cudaMemcpyAsync(h_out + a * W * W, h->outbuf + a * W * W, (size_t)(M - a) * img_bytes,
                           cudaMemcpyDeviceToHost, h->copy_stream), "D2H images");
        break;
      }
      CK(cudaMemcpyAsync(h_out + a * W * W, h->outbuf + a * W * W, (size_t)n * img_bytes,
                         cudaMemcpyDeviceToHost, h->copy_stream), "D2H images");
    }
    CK(cudaStreamSynchronize(h->copy_stream), "sync copy");
    CK(cudaStreamSynchronize(s), "sync");
    return SPIN_OK;
  }
  CK(cudaMemcpyAsync(h_out, h->outbuf, (size_t)M * W * W * sizeof(float), cudaMemcpyDeviceToHost, s), "D2H images");
  CK(cudaStreamSynchronize(s), "sync");
  return SPIN_OK;
}

}  // extern "C"
