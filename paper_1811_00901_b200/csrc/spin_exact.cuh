// spin_exact.cuh — the two slow decision stages of the accept path (fp64, then exact).
//
// Reading #14: every integer decision of
// Alg. 1 (support test P:166, row k P:169, column l P:171, bounds P:173) is the one
// EXACT real arithmetic takes on the fp32 inputs (b, cos_As exact doubles).  The
// fp32 stage in spin_kernels.cu certifies most decisions; what it cannot certify is
// re-taken here in fp64 with per-pair forward error bounds, and what fp64 cannot
// certify is decided by an exact sign computation over floating-point expansions
// (TwoSum / TwoProduct with fma, Grow-Expansion with zero elimination).  For fp32
// inputs every product below is exact or has an exact TwoProduct split, and no
// intermediate can overflow or underflow double, so the exact stage is exact for
// every finite input — there are no residual ties.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace spin {

constexpr double U64 = 1.1102230246251565e-16;  // 2^-53

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = fma(a, b, -p);
}

// Grow-Expansion (Shewchuk 1997, Thm. 10) with zero elimination: e[0..n) is a
// nonoverlapping expansion in increasing magnitude; returns the new length.
__device__ __forceinline__ int grow(double* e, int n, double b) {
  double Q = b;
  int m = 0;
  for (int i = 0; i < n; ++i) {
    double s, err;
    two_sum(Q, e[i], s, err);
    if (err != 0.0) e[m++] = err;
    Q = s;
  }
  if (Q != 0.0 || m == 0) e[m++] = Q;
  return m;
}
__device__ __forceinline__ int exp_sign(const double* e, int n) {
  double top = e[n - 1];
  return top > 0.0 ? 1 : (top < 0.0 ? -1 : 0);
}
__device__ __forceinline__ int grow_prod(double* e, int n, double a, double b) {
  double p, r;
  two_prod(a, b, p, r);
  n = grow(e, n, r);
  return grow(e, n, p);
}

struct PairD {
  double p[3], n[3], x[3], nx[3];
};

// sign(n . nx - c), exactly (products of two fp32 values are exact in double)
static __device__ __noinline__ int exact_sign_support(const PairD& P, double c) {
  double e[8];
  int m = 0;
  for (int i = 0; i < 3; ++i) m = grow(e, m, P.n[i] * P.nx[i]);
  m = grow(e, m, -c);
  return exp_sign(e, m);
}

// T(k) = (A - k) b (scaled reading #2) or A - k b (literal, P:169 as printed).
// Returns sign(beta - T(k)), beta = n.(x - p) = sum n_i x_i - sum n_i p_i.
// u <= k  <=>  sign >= 0 for both readings.
static __device__ __noinline__ int exact_sign_beta_minus_T(const PairD& P, double A, double b, int k,
                                                    int literal) {
  double e[16];
  int m = 0;
  for (int i = 0; i < 3; ++i) {
    m = grow(e, m, P.n[i] * P.x[i]);      // exact (24 x 24 bits)
    m = grow(e, m, -(P.n[i] * P.p[i]));   // exact
  }
  double th, tl;
  if (!literal) {
    two_prod(A - (double)k, b, th, tl);  // A - k is a small half-integer: exact
    m = grow(e, m, -tl);
    m = grow(e, m, -th);
  } else {
    two_prod((double)k, b, th, tl);
    m = grow(e, m, tl);
    m = grow(e, m, th);
    m = grow(e, m, -A);
  }
  return exp_sign(e, m);
}

// sign(q - mm * b^2) with q = |x - p|^2 - beta^2, mm = m^2 a small integer.
static __device__ __noinline__ int exact_sign_q_minus(const PairD& P, double b, double mm) {
  double e[80];
  int m = 0;
  // |d|^2 with d_i = dh_i + dl_i exactly
  for (int i = 0; i < 3; ++i) {
    double dh, dl;
    two_sum(P.x[i], -P.p[i], dh, dl);
    m = grow_prod(e, m, dh, dh);
    m = grow_prod(e, m, 2.0 * dh, dl);
    m = grow_prod(e, m, dl, dl);
  }
  // - beta^2, beta = sum_j t_j with the 6 exact products t_j
  double t[6];
  for (int i = 0; i < 3; ++i) {
    t[2 * i] = P.n[i] * P.x[i];
    t[2 * i + 1] = -(P.n[i] * P.p[i]);
  }
  for (int a = 0; a < 6; ++a) {
    m = grow_prod(e, m, -t[a], t[a]);
    for (int c = a + 1; c < 6; ++c) m = grow_prod(e, m, -2.0 * t[a], t[c]);
  }
  // - mm * b^2
  double bh, bl;
  two_prod(b, b, bh, bl);
  m = grow_prod(e, m, -mm, bl);
  m = grow_prod(e, m, -mm, bh);
  return exp_sign(e, m);
}

// Result of the slow decision for one pair.
struct SlowOut {
  int accept;   // 0 / 1
  int k, l;     // NEAREST bins (valid when accept)
  int n_exact;  // decisions taken by the exact stage
};

// fp64 stage with per-pair certified bounds, escalating each uncertain decision to
// the exact stage.  `mode` 0 NEAREST / 1 BILINEAR (BILINEAR returns region only).
static __device__ __noinline__ SlowOut slow_decide(const PairD& P, int W, double A, double b,
                                            double cos_As, int has_support, int literal,
                                            int floor_bins, int mode) {
  SlowOut r{0, 0, 0, 0};
  int& n_exact = r.n_exact;
  const double u = U64;
  // --- support
  if (has_support) {
    double t0 = P.n[0] * P.nx[0], t1 = P.n[1] * P.nx[1], t2 = P.n[2] * P.nx[2];  // exact
    double s = __dadd_rn(__dadd_rn(t0, t1), t2);
    double es = 3.0 * u * (fabs(t0) + fabs(t1) + fabs(t2));
    int sg;
    if (s - cos_As > es) sg = 1;
    else if (s - cos_As < -es) sg = -1;
    else { ++n_exact; sg = exact_sign_support(P, cos_As); }
    if (sg < 0) return r;
  }
  // --- projection in plain double ops
  double d[3], sb = 0.0;
  for (int i = 0; i < 3; ++i) d[i] = __dsub_rn(P.x[i], P.p[i]);
  double b0 = __dmul_rn(P.n[0], d[0]), b1 = __dmul_rn(P.n[1], d[1]), b2 = __dmul_rn(P.n[2], d[2]);
  double beta = __dadd_rn(__dadd_rn(b0, b1), b2);
  sb = fabs(b0) + fabs(b1) + fabs(b2);
  double eb = 6.0 * u * sb;
  double dd = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
  double edd = 6.0 * u * dd;
  double bb = __dmul_rn(beta, beta);
  double q = __dsub_rn(dd, bb);
  double eq = edd + (2.0 * fabs(beta) + eb) * eb + 2.0 * u * (bb + fabs(q));
  double uu, eu;
  if (!literal) {
    double t = __ddiv_rn(beta, b);
    uu = __dsub_rn(A, t);
    eu = eb / b * (1.0 + 4.0 * u) + 2.0 * u * (fabs(t) + fabs(uu));
  } else {
    double t = __dsub_rn(A, beta);
    uu = __ddiv_rn(t, b);
    eu = (eb + u * fabs(t)) / b * (1.0 + 4.0 * u) + 2.0 * u * fabs(uu);
  }
  double b2d = __dmul_rn(b, b);
  double w = __ddiv_rn(q, b2d);
  double ew = eq / b2d * (1.0 + 6.0 * u) + 4.0 * u * fabs(w);
  eu = eu * 1.01 + 1e-300;
  ew = ew * 1.01 + 1e-300;

  const double Wm1 = (double)(W - 1);
  if (mode == 0) {
    // ---------------- row k.  ceil: contributes iff u in (-1, W-1]; floor: u in [0, W)
    if (uu + eu < -1.5 || uu - eu > (double)W + 0.5) return r;   // certainly outside
    int k;
    double uc = uu;
    double rr = rint(uc);
    if (fabs(uc - rr) > eu) {
      k = floor_bins ? (int)floor(uc) : (int)ceil(uc);
    } else {
      ++n_exact;
      // ceil: k = smallest integer with u <= k  (u <= k <=> sign(beta - T(k)) >= 0)
      // floor: k = largest integer with u >= k  (u >= k <=> sign(beta - T(k)) <= 0)
      // (start clamped to [-1, W] and every step bounded: a k outside [0, W) is rejected
      // anyway, so a huge eu cannot make the search walk 2^31 rows)
      k = (int)fmin(fmax(rr, -1.0), (double)W);
      if (!floor_bins) {
        while (k >= 0 && exact_sign_beta_minus_T(P, A, b, k - 1, literal) >= 0) --k;
        while (k < W && exact_sign_beta_minus_T(P, A, b, k, literal) < 0) ++k;
      } else {
        while (k >= 0 && exact_sign_beta_minus_T(P, A, b, k, literal) > 0) --k;
        while (k < W && exact_sign_beta_minus_T(P, A, b, k + 1, literal) <= 0) ++k;
      }
    }
    if (k < 0 || k >= W) return r;
    // ---------------- column l
    int l;
    double v = sqrt(fmax(w, 0.0));
    double fl = floor(v);
    double dlo = w - fl * fl, dhi = (fl + 1.0) * (fl + 1.0) - w;
    if (w < -ew) {
      l = 0;
    } else if (dlo > ew && dhi > ew) {
      l = floor_bins ? (int)fl : (int)fl + 1;
    } else {
      ++n_exact;
      int mm = (int)fmin(fl, (double)W + 2.0);
      if (!floor_bins) {  // smallest m >= 0 with q <= m^2 b^2
        while (mm > 0 && exact_sign_q_minus(P, b, (double)(mm - 1) * (mm - 1)) <= 0) --mm;
        while (mm <= W && exact_sign_q_minus(P, b, (double)mm * mm) > 0) ++mm;
      } else {            // largest m >= 0 with m^2 b^2 <= q (q < 0 clamps to 0)
        while (mm > 0 && exact_sign_q_minus(P, b, (double)mm * mm) < 0) --mm;
        while (mm <= W && exact_sign_q_minus(P, b, (double)(mm + 1) * (mm + 1)) >= 0) ++mm;
      }
      l = mm;
    }
    if (l < 0 || l >= W) return r;
    r.accept = 1;
    r.k = k;
    r.l = l;
    return r;
  }
  // ---------------- BILINEAR region: 0 <= u < W-1 and w < (W-1)^2  (#12)
  bool in_u;
  if (fabs(uu) > eu && fabs(uu - Wm1) > eu) {
    in_u = (uu > 0.0) && (uu < Wm1);
  } else {
    ++n_exact;
    // u >= 0 <=> sign(beta - T(0)) <= 0 ;  u < W-1 <=> sign(beta - T(W-1)) > 0
    in_u = exact_sign_beta_minus_T(P, A, b, 0, literal) <= 0 &&
           exact_sign_beta_minus_T(P, A, b, W - 1, literal) > 0;
  }
  if (!in_u) return r;
  bool in_w;
  double lim = Wm1 * Wm1;
  if (fabs(w - lim) > ew) {
    in_w = w < lim;
  } else {
    ++n_exact;
    in_w = exact_sign_q_minus(P, b, lim) < 0;
  }
  r.accept = in_w ? 1 : 0;
  return r;
}

}  // namespace spin
