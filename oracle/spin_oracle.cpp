// ORACLE for the spin-image hot path (C++ edition) — TEST INFRASTRUCTURE ONLY.
//
// Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl
// reference` legs may load this library (through oracle/spin_oracle_cpp.py).  It shares
// no code, header, table or constant with the product path (paper_1811_00901_b200/,
// libspin.so) and includes nothing from it.  `__graft_entry__.build()` compiles it
// (building the checker is not using it).
//
// What it computes is the plain definition of the paper's Algorithm 1
// (`calculateSpinImages`, `algo:spin`), one image per centre, every
// cloud point visited (the inner loop `for j = 0 -> M`), under the readings of
// SURVEY.md §8(c) listed in DESIGN.md §3:
//
//   support   acos(np_i . np_j) <= S            read as  n . nx >= cos_As  (#5/#6)
//   beta  = n . (X - P)
//   alpha = sqrt(|X - P|^2 - beta^2)   (clamped at 0)
//   u = W/2 - beta/b  (scaled reading #2; flag LITERAL: (W/2 - beta)/b),  v = alpha/b
//   NEAREST : k = ceil(u), l = ceil(v)  (flag FLOOR: floor);  0 <= k,l < W -> image[k][l] += 1
//             (#4)
//   BILINEAR: i0 = floor(u), j0 = floor(v); 0 <= i0, j0 <= W-2 -> weight 1 split over the
//             four corners by a = u - i0, c = v - j0 (#12 — NOT in the paper: parity of the
//             splat rule is pinned only by X1 and its invariants)
//
// Precision reading #14: the result is defined in EXACT real arithmetic on the fp32 inputs,
// with b and cos_As exact doubles.  Every integer decision is therefore taken so that it
// equals the exact one:
//   stage 1  plain double with a-priori forward error bounds (the throughput path; the
//            bounds are derived in DESIGN.md §4);
//   stage 2  the same decisions in THRESHOLD form (no division, no sqrt:
//            k = ceil(u)  <=>  (W/2 - k) b <= beta < (W/2 - k + 1) b,
//            l = ceil(v)  <=>  ((l-1) b)^2 < q <= (l b)^2,  l = 0 <=> q <= 0)
//            in double "interval" arithmetic whose per-operation rounding error is
//            measured exactly by error-free transformations (TwoSum / TwoProduct), so
//            exact ties (margin exactly 0 with every operation exact) are decided too;
//   stage 3  the threshold form again in __float128 (113-bit significand);
//   stage 4  anything still undecided is returned to the caller, which decides it with
//            the Python oracle's exact rational arithmetic (oracle/spin_oracle.py
//            exact_pair, fractions.Fraction).
// BILINEAR weights are evaluated in double from u and v (continuous inside the region).
//
// Oracle-CELLS: an independent uniform grid (edge 1.0001 R, R = the region radius), the
// 27 cells around the centre's cell, the same per-pair decision -> equals oracle-BRUTE
// (NEAREST bit for bit; BILINEAR up to the order of the double sums, ~1e-16).
//
// Pins (tests/test_oracle_cpp.py, -m "not gpu"): the hand-worked goldens X1-X4, the
// config-1 closed form, total weight = in-region count, signed-permutation / dyadic
// translation / 2^k scale invariance, CELLS == BRUTE, equality with the (independently
// pinned) Python oracle on seeded clouds including dyadic clouds full of exact ties.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace {

constexpr int NEAREST = 0, BILINEAR = 1;
constexpr int F_LITERAL = 1, F_FLOOR = 2;
// test-only switches (tests/test_oracle_cpp.py): send EVERY pair to stage 2 / 3 / 4, so the
// threshold-form stages are checked against stage 1 and the exact rational decisions
constexpr int F_FORCE2 = 1 << 8, F_FORCE3 = 1 << 9, F_FORCE4 = 1 << 10;
constexpr int F_FORCE = F_FORCE2 | F_FORCE3 | F_FORCE4;

typedef __float128 q128;

// ------------------------------------------------------------------ unit roundoffs
template <class F> F unit_roundoff();
template <> double unit_roundoff<double>() { return 0x1p-53; }
q128 make_u128() {
  q128 u = 1;
  for (int i = 0; i < 113; ++i) u /= 2;   // 2^-113, exact
  return u;
}
const q128 U128 = make_u128();
template <> q128 unit_roundoff<q128>() { return U128; }
template <class F> F fabs_(F x) { return x < 0 ? -x : x; }

// ------------------------------------------------------------------ error-free transformations
// TwoSum (Knuth): s + e == a + b exactly, s = fl(a + b)   (round to nearest, no overflow)
template <class F> void two_sum(F a, F b, F& s, F& e) {
  s = a + b;
  const F bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// TwoProduct: p + e == a * b exactly, p = fl(a * b).  double: one fma; __float128:
// Dekker's product with Veltkamp splitting (split constant 2^57 + 1)
void two_prod(double a, double b, double& p, double& e) {
  p = a * b;
  e = std::fma(a, b, -p);
}
q128 make_split() {
  q128 c = 1;
  for (int i = 0; i < 57; ++i) c *= 2;
  return c + 1;                            // 2^57 + 1
}
const q128 SPLIT128 = make_split();
void split128(q128 a, q128& hi, q128& lo) {
  const q128 t = SPLIT128 * a;
  hi = t - (t - a);
  lo = a - hi;
}
void two_prod(q128 a, q128 b, q128& p, q128& e) {
  p = a * b;
  q128 ah, al, bh, bl;
  split128(a, ah, al);
  split128(b, bh, bl);
  e = ((ah * bh - p) + ah * bl + al * bh) + al * bl;
}

// A value with a rigorous bound on its distance to the exact real result: |v - exact| <= e.
// e == 0 means the value is exact (every rounding so far was measured to be zero).
template <class F> struct Iv {
  F v, e;
};
template <class F> Iv<F> exact(F v) { return {v, F(0)}; }
template <class F> F up(F x) {   // x * (1 + 8u): covers the roundings of the bound's own sums
  return x * (F(1) + 8 * unit_roundoff<F>());
}
template <class F> Iv<F> add(Iv<F> a, Iv<F> b) {
  F s, t;
  two_sum(a.v, b.v, s, t);
  return {s, up(a.e + b.e + fabs_(t))};
}
template <class F> Iv<F> neg(Iv<F> a) { return {-a.v, a.e}; }
template <class F> Iv<F> sub(Iv<F> a, Iv<F> b) { return add(a, neg(b)); }
template <class F> Iv<F> mul(Iv<F> a, Iv<F> b) {
  F p, t;
  two_prod(a.v, b.v, p, t);
  return {p, up(fabs_(a.v) * b.e + fabs_(b.v) * a.e + a.e * b.e + fabs_(t))};
}
// certified comparison: +1 (x > y), 0 (x == y), -1 (x < y), 2 (cannot tell)
template <class F> int cmp(Iv<F> x, Iv<F> y) {
  const F d = x.v - y.v;
  const F e = x.e + y.e;
  if (e == F(0)) return d > 0 ? 1 : (d < 0 ? -1 : 0);
  const F lim = e * (F(1) + 8 * unit_roundoff<F>());
  if (d > lim) return 1;
  if (-d > lim) return -1;
  return 2;
}

struct Job {
  const float* X;     // [N][3]
  const float* Nr;    // [N][3]
  int64_t N;
  int W;
  double b, cos_As;
  int mode, flags;
  bool has_support;
};

// One pair's outcome.  state: 0 no contribution, 1 contributes, 2 undecided (stage 4)
struct Outcome {
  int state;
  int k, l;       // NEAREST bin / BILINEAR (i0, j0)
  double a, c;    // BILINEAR fractional offsets
};

// ------------------------------------------------------------------ stages 2 / 3: threshold form
// beta value where u == j:  scaled u = W/2 - beta/b -> (W/2 - j) b;  literal u = (W/2 - beta)/b
// -> W/2 - j b.  u is decreasing in beta.
template <class F> Iv<F> beta_at(const Job& J, int j) {
  const Iv<F> b = exact<F>(F(J.b));
  const Iv<F> half = exact<F>(F(J.W) / F(2));   // W <= 64: exact
  if (J.flags & F_LITERAL) return sub(half, mul(exact<F>(F(j)), b));
  return mul(sub(half, exact<F>(F(j))), b);
}
template <class F> Iv<F> sq_edge(const Job& J, int m) {   // (m b)^2
  const Iv<F> mb = mul(exact<F>(F(m)), exact<F>(F(J.b)));
  return mul(mb, mb);
}

// Decide one pair exactly in threshold form with precision F; state 2 = still undecided.
// k0 / l0: the approximate row / column (from stage 1) where the searches start.
template <class F>
Outcome decide_threshold(const Job& J, const float* p, const float* n, const float* x,
                         const float* nx, int k0, int l0) {
  Outcome o{2, 0, 0, 0.0, 0.0};
  if (J.has_support) {
    Iv<F> s = mul(exact<F>(F(n[0])), exact<F>(F(nx[0])));
    s = add(s, mul(exact<F>(F(n[1])), exact<F>(F(nx[1]))));
    s = add(s, mul(exact<F>(F(n[2])), exact<F>(F(nx[2]))));
    const int r = cmp(s, exact<F>(F(J.cos_As)));
    if (r == 2) return o;
    if (r < 0) { o.state = 0; return o; }                  // acos(.) > S
  }
  Iv<F> d[3];
  for (int i = 0; i < 3; ++i) d[i] = sub(exact<F>(F(x[i])), exact<F>(F(p[i])));
  Iv<F> beta = mul(exact<F>(F(n[0])), d[0]);
  beta = add(beta, mul(exact<F>(F(n[1])), d[1]));
  beta = add(beta, mul(exact<F>(F(n[2])), d[2]));
  Iv<F> dd = mul(d[0], d[0]);
  dd = add(dd, mul(d[1], d[1]));
  dd = add(dd, mul(d[2], d[2]));
  const Iv<F> q = sub(dd, mul(beta, beta));                  // alpha^2 (unclamped)
  const int W = J.W;
  const bool floor_bins = J.mode == NEAREST && (J.flags & F_FLOOR);
  // ---- row: NEAREST ceil: k <=> beta in [beta_at(k), beta_at(k-1));
  //           NEAREST floor: k <=> beta in (beta_at(k+1), beta_at(k)];
  //           BILINEAR i0 = floor(u) in [0, W-2] <=> beta in (beta_at(W-1), beta_at(0)]
  int k = 0;
  if (J.mode == BILINEAR) {
    const int lo = cmp(beta, beta_at<F>(J, W - 1));          // need beta > beta_at(W-1)
    const int hi = cmp(beta, beta_at<F>(J, 0));              // need beta <= beta_at(0)
    if (lo == 2 || hi == 2) {
      // an undecided edge only matters if the other one admits the pair
      if ((lo != 2 && lo <= 0) || (hi != 2 && hi > 0)) { o.state = 0; return o; }
      return o;
    }
    if (lo <= 0 || hi > 0) { o.state = 0; return o; }
  } else {
    k = std::min(std::max(k0, -2), W + 1);
    bool found = false;
    for (int it = 0; it < 2 * W + 16 && !found; ++it) {
      // does beta lie below / inside / above row k's window?
      int below, above;   // below: beta under the window (u too large -> k+1); above: k-1
      if (!floor_bins) {
        const int c1 = cmp(beta, beta_at<F>(J, k));          // need >= 0
        const int c2 = cmp(beta, beta_at<F>(J, k - 1));      // need < 0
        if (c1 == 2 || c2 == 2) return o;
        below = c1 < 0;
        above = c2 >= 0;
      } else {
        const int c1 = cmp(beta, beta_at<F>(J, k + 1));      // need > 0
        const int c2 = cmp(beta, beta_at<F>(J, k));          // need <= 0
        if (c1 == 2 || c2 == 2) return o;
        below = c1 <= 0;
        above = c2 > 0;
      }
      if (!below && !above) { found = true; break; }
      if (below) {
        if (k >= W) { o.state = 0; return o; }               // k only grows: out of range
        ++k;
      } else {
        if (k < 0) { o.state = 0; return o; }
        --k;
      }
    }
    if (!found) return o;
    if (k < 0 || k >= W) { o.state = 0; return o; }
  }
  // ---- column: ceil: l = 0 <=> q <= 0; l = m >= 1 <=> ((m-1)b)^2 < q <= (m b)^2
  //              floor: l = m <=> (m b)^2 <= max(q, 0) < ((m+1) b)^2
  //              BILINEAR: j0 = floor(v) <= W-2 <=> q < ((W-1) b)^2
  int l = 0;
  if (J.mode == BILINEAR) {
    const int r = cmp(q, sq_edge<F>(J, W - 1));
    if (r == 2) return o;
    if (r >= 0) { o.state = 0; return o; }
  } else {
    l = std::min(std::max(l0, 0), W + 1);
    bool found = false;
    for (int it = 0; it < 2 * W + 16; ++it) {
      int grow, shrink;
      if (!floor_bins) {
        const int c1 = cmp(q, sq_edge<F>(J, l));              // need <= 0
        if (c1 == 2) return o;
        grow = c1 > 0;
        shrink = 0;
        if (!grow && l > 0) {
          const int c2 = cmp(q, sq_edge<F>(J, l - 1));        // need > 0
          if (c2 == 2) return o;
          shrink = c2 <= 0;
        }
      } else {
        const int c1 = cmp(q, sq_edge<F>(J, l + 1));          // need < 0
        if (c1 == 2) return o;
        grow = c1 >= 0;
        shrink = 0;
        if (!grow && l > 0) {
          const int c2 = cmp(q, sq_edge<F>(J, l));            // need >= 0
          if (c2 == 2) return o;
          shrink = c2 < 0;
        }
      }
      if (!grow && !shrink) { found = true; break; }
      if (grow) {
        if (l >= W) { o.state = 0; return o; }
        ++l;
      } else {
        --l;
      }
    }
    if (!found) return o;
    if (l >= W) { o.state = 0; return o; }
  }
  o.state = 1;
  o.k = k;
  o.l = l;
  return o;
}

// ------------------------------------------------------------------ stage 1: plain double
inline double dist_to_int(double x) { return std::fabs(x - std::nearbyint(x)); }
inline double dist_to_square(double w) {   // to the nearest m^2, m >= 0 (w may be < 0)
  const double r = std::floor(std::sqrt(std::max(w, 0.0)));
  double best = std::fabs(w);
  for (double dm = -1.0; dm <= 2.0; dm += 1.0) {
    const double m = std::max(r + dm, 0.0);
    best = std::min(best, std::fabs(w - m * m));
  }
  return best;
}

// BILINEAR weights from double u and v (stage-independent: the region is decided exactly
// elsewhere; inside it the splat is continuous in u and v, reading #12)
inline void bilinear_offsets(int W, double u, double w, Outcome& o) {
  const double v = std::sqrt(std::max(w, 0.0));
  const double fi = std::min(std::max(std::floor(u), 0.0), double(W - 2));
  const double fj = std::min(std::max(std::floor(v), 0.0), double(W - 2));
  o.k = (int)fi;
  o.l = (int)fj;
  o.a = std::min(std::max(u - fi, 0.0), 1.0);
  o.c = std::min(std::max(v - fj, 0.0), 1.0);
}

struct PairStats {
  int64_t stage2 = 0, stage3 = 0, stage4 = 0;
};

Outcome escalate(const Job& J, const float* p, const float* n, const float* x, const float* nx,
                 int k0, int l0, double u, double w, PairStats& ps);

inline Outcome decide_pair(const Job& J, const float* p, const float* n, const float* x,
                           const float* nx, PairStats& ps) {
  const double U = 0x1p-53;
  const int W = J.W;
  const bool force = (J.flags & F_FORCE) != 0;
  bool unsure = force;
  // ---- support: three exact products, two roundings
  if (J.has_support) {
    const double t0 = (double)n[0] * nx[0], t1 = (double)n[1] * nx[1], t2 = (double)n[2] * nx[2];
    const double s = (t0 + t1) + t2;
    const double es = 4 * U * (std::fabs(t0) + std::fabs(t1) + std::fabs(t2));
    if (!force && s - J.cos_As < -es) return Outcome{0, 0, 0, 0, 0};
    if (!(s - J.cos_As > es)) unsure = true;
  }
  // ---- projection
  const double d0 = (double)x[0] - p[0], d1 = (double)x[1] - p[1], d2 = (double)x[2] - p[2];
  const double b0 = (double)n[0] * d0, b1 = (double)n[1] * d1, b2 = (double)n[2] * d2;
  const double beta = (b0 + b1) + b2;
  const double eb = 6 * U * (std::fabs(b0) + std::fabs(b1) + std::fabs(b2));
  // ---- u (the row coordinate)
  const double half = W / 2.0;
  double u, eu;
  if (J.flags & F_LITERAL) {
    const double t = half - beta;
    u = t / J.b;
    eu = (eb + U * std::fabs(t)) / J.b * (1 + 4 * U) + 2 * U * std::fabs(u);
  } else {
    const double t = beta / J.b;
    u = half - t;
    eu = eb / J.b * (1 + 4 * U) + 2 * U * (std::fabs(t) + std::fabs(u));
  }
  eu += 1e-300;
  // the rows that contribute: NEAREST ceil k in [0, W) <=> u in (-1, W-1]; floor u in [0, W);
  // BILINEAR i0 in [0, W-2] <=> u in [0, W-1).  Certainly outside -> no contribution.
  const bool floor_bins = J.mode == NEAREST && (J.flags & F_FLOOR);
  double u_lo, u_hi, w_hi;   // u range and the bound on w = v^2 (ceil: w <= w_hi; else w < w_hi)
  if (J.mode == NEAREST && !floor_bins) { u_lo = -1; u_hi = W - 1; w_hi = double(W - 1) * (W - 1); }
  else if (J.mode == NEAREST) { u_lo = 0; u_hi = W; w_hi = double(W) * W; }
  else { u_lo = 0; u_hi = W - 1; w_hi = double(W - 1) * (W - 1); }
  if (!force && (u + eu < u_lo || u - eu > u_hi)) return Outcome{0, 0, 0, 0, 0};
  // ---- alpha^2 = |X-P|^2 - beta^2 and w = v^2 = alpha^2 / b^2
  const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
  const double edd = 6 * U * dd;
  const double bb = beta * beta;
  const double q = dd - bb;
  const double eq = edd + (2 * std::fabs(beta) + eb) * eb + 2 * U * (bb + std::fabs(q));
  const double b2q = J.b * J.b;
  const double w = q / b2q;
  const double ew = eq / b2q * (1 + 6 * U) + 4 * U * std::fabs(w) + 1e-300;
  if (!force && w - ew > w_hi) return Outcome{0, 0, 0, 0, 0};
  Outcome o{0, 0, 0, 0.0, 0.0};
  int k0 = 0, l0 = 0;
  if (J.mode == NEAREST) {
    if (dist_to_int(u) <= eu) unsure = true;
    if (dist_to_square(w) <= ew) unsure = true;
    const double wc = std::max(w, 0.0);
    double k = floor_bins ? std::floor(u) : std::ceil(u);
    // l from the squares (independent of sqrt's rounding): smallest m with m^2 >= w (ceil),
    // largest m with m^2 <= w (floor)
    double l = floor_bins ? std::floor(std::sqrt(wc)) : std::ceil(std::sqrt(wc));
    if (!floor_bins) {
      if (l > 0 && (l - 1) * (l - 1) >= w) l -= 1;
      if (l * l < w) l += 1;
    } else {
      if (l * l > wc) l -= 1;
      if ((l + 1) * (l + 1) <= wc) l += 1;
    }
    k0 = (int)std::min(std::max(k, -4.0), W + 4.0);
    l0 = (int)std::min(std::max(l, 0.0), W + 4.0);
    if (!unsure) {
      if (k >= 0 && k < W && l >= 0 && l < W) {
        o.state = 1;
        o.k = (int)k;
        o.l = (int)l;
      }
      return o;
    }
  } else {
    // BILINEAR region: 0 <= u < W-1 and w < (W-1)^2
    const double lim = double(W - 1) * (W - 1);
    if (std::fabs(u) <= eu || std::fabs(u - (W - 1)) <= eu || std::fabs(w - lim) <= ew) unsure = true;
    if (!unsure) {
      if (u >= 0 && u < W - 1 && w < lim) {
        o.state = 1;
        bilinear_offsets(W, u, w, o);
      }
      return o;
    }
  }
  return escalate(J, p, n, x, nx, k0, l0, u, w, ps);
}

// ---- stages 2 and 3: threshold form, measured rounding errors (out of line: rare)
__attribute__((noinline)) Outcome escalate(const Job& J, const float* p, const float* n,
                                           const float* x, const float* nx, int k0, int l0,
                                           double u, double w, PairStats& ps) {
  Outcome r{2, 0, 0, 0.0, 0.0};
  if (!(J.flags & (F_FORCE3 | F_FORCE4))) {
    ++ps.stage2;
    r = decide_threshold<double>(J, p, n, x, nx, k0, l0);
  }
  if (r.state == 2 && !(J.flags & F_FORCE4)) {
    ++ps.stage3;
    r = decide_threshold<q128>(J, p, n, x, nx, k0, l0);
  }
  if (r.state == 2) {
    ++ps.stage4;
    return r;
  }
  if (r.state == 1 && J.mode == BILINEAR) bilinear_offsets(J.W, u, w, r);
  return r;
}

// ------------------------------------------------------------------ images
struct ImageOut {
  double* img;        // [W][W]
  int32_t* contrib;   // [W][W] or null (BILINEAR contributors: pairs with weight > 0 on the bin)
  int64_t in_region;
};

inline void splat(const Job& J, const Outcome& o, ImageOut& io) {
  const int W = J.W;
  ++io.in_region;
  if (J.mode == NEAREST) {
    io.img[o.k * W + o.l] += 1.0;
    return;
  }
  const double a = o.a, c = o.c;
  const double wt[4] = {(1 - a) * (1 - c), a * (1 - c), (1 - a) * c, a * c};
  const int bins[4] = {o.k * W + o.l, (o.k + 1) * W + o.l, o.k * W + o.l + 1, (o.k + 1) * W + o.l + 1};
  for (int t = 0; t < 4; ++t) {
    io.img[bins[t]] += wt[t];
    if (io.contrib && wt[t] > 0) io.contrib[bins[t]] += 1;
  }
}

struct Unsure {
  int64_t m, j;
};

// the image of centre ci over the points Xs[a..b) (Xs/Ns: the cloud itself, or the
// grid's cell-sorted copy, whose original indices idx[] name the undecided pairs)
void image_of(const Job& J, int64_t m, int64_t ci, const float* Xs, const float* Ns,
              const int64_t* idx, int64_t a, int64_t b, ImageOut& io, PairStats& ps,
              std::vector<Unsure>& uns) {
  const float* p = J.X + 3 * ci;
  const float* n = J.Nr + 3 * ci;
  for (int64_t t = a; t < b; ++t) {
    const Outcome o = decide_pair(J, p, n, Xs + 3 * t, Ns + 3 * t, ps);
    if (o.state == 1) splat(J, o, io);
    else if (o.state == 2) uns.push_back({m, idx ? idx[t] : t});
  }
}

// region radius: an upper bound on |X - P| for any contributing pair:
// |X-P|^2 = alpha^2 + beta^2 with the u- and v-ranges that contribute
double region_radius(int W, double b, int mode, int flags) {
  double u_lo, u_hi, v_max;
  if (mode == NEAREST && !(flags & F_FLOOR)) { u_lo = -1; u_hi = W - 1; v_max = W - 1; }
  else if (mode == NEAREST) { u_lo = 0; u_hi = W; v_max = W; }
  else { u_lo = 0; u_hi = W - 1; v_max = W - 1; }
  double b1, b2;
  if (flags & F_LITERAL) { b1 = W / 2.0 - u_lo * b; b2 = W / 2.0 - u_hi * b; }
  else { b1 = (W / 2.0 - u_lo) * b; b2 = (W / 2.0 - u_hi) * b; }
  const double bm = std::max(std::fabs(b1), std::fabs(b2));
  return std::sqrt((v_max * b) * (v_max * b) + bm * bm) * (1.0 + 1e-9) + 1e-300;
}

// Oracle-CELLS grid: edge h = 1.0001 R; a point within R of a centre lies in the 27 cells
// around the centre's cell
struct Grid {
  double h, o[3];
  int64_t dim[3];
  std::vector<int64_t> key_sorted, idx_sorted;
  std::vector<float> Xs, Ns;   // the cloud in cell order (contiguous reads per cell)
  int64_t cell(const double* x, int64_t c3[3]) const {
    for (int a = 0; a < 3; ++a) c3[a] = (int64_t)std::floor((x[a] - o[a]) / h);
    return (c3[2] * dim[1] + c3[1]) * dim[0] + c3[0];
  }
  void build(const float* X, const float* Nr, int64_t N, double R) {
    h = 1.0001 * R;
    for (int a = 0; a < 3; ++a) {
      o[a] = INFINITY;
      for (int64_t i = 0; i < N; ++i) o[a] = std::min(o[a], (double)X[3 * i + a]);
    }
    std::vector<std::pair<int64_t, int64_t>> kv((size_t)N);
    int64_t mx[3] = {0, 0, 0};
    std::vector<int64_t> c3s((size_t)N * 3);
    for (int64_t i = 0; i < N; ++i) {
      for (int a = 0; a < 3; ++a) {
        c3s[3 * i + a] = (int64_t)std::floor(((double)X[3 * i + a] - o[a]) / h);
        mx[a] = std::max(mx[a], c3s[3 * i + a]);
      }
    }
    for (int a = 0; a < 3; ++a) dim[a] = mx[a] + 1;
    for (int64_t i = 0; i < N; ++i)
      kv[i] = {(c3s[3 * i + 2] * dim[1] + c3s[3 * i + 1]) * dim[0] + c3s[3 * i], i};
    std::sort(kv.begin(), kv.end());
    key_sorted.resize((size_t)N);
    idx_sorted.resize((size_t)N);
    Xs.resize((size_t)N * 3);
    Ns.resize((size_t)N * 3);
    for (int64_t i = 0; i < N; ++i) {
      key_sorted[i] = kv[i].first;
      idx_sorted[i] = kv[i].second;
      for (int a = 0; a < 3; ++a) {
        Xs[3 * i + a] = X[3 * kv[i].second + a];
        Ns[3 * i + a] = Nr[3 * kv[i].second + a];
      }
    }
  }
  // the [lo, hi) ranges (in cell order) of the 27 cells around p's cell
  void neighbours(const float* p, std::vector<std::pair<int64_t, int64_t>>& out) const {
    out.clear();
    const double x[3] = {p[0], p[1], p[2]};
    int64_t c[3];
    cell(x, c);
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t k3[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
          bool ok = true;
          for (int a = 0; a < 3; ++a) ok &= k3[a] >= 0 && k3[a] < dim[a];
          if (!ok) continue;
          const int64_t key = (k3[2] * dim[1] + k3[1]) * dim[0] + k3[0];
          auto lo = std::lower_bound(key_sorted.begin(), key_sorted.end(), key);
          auto hi = std::upper_bound(lo, key_sorted.end(), key);
          if (hi > lo) out.push_back({lo - key_sorted.begin(), hi - key_sorted.begin()});
        }
  }
};

int n_threads(int req) {
  if (req > 0) return req;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

}  // namespace

extern "C" {

// Images of centres cen[0..M) (oracle-BRUTE if cells == 0, oracle-CELLS otherwise).
//   out       double [M][W][W]   (zeroed here)
//   contrib   int32  [M][W][W] or null (BILINEAR: pairs with nonzero weight per bin)
//   in_region int64  [M] or null (pairs that contribute, per image)
//   unsure    int64  [cap][2] (m, j) pairs left undecided by stages 1-3, *n_unsure their
//             count (if it exceeds cap the call returns 1 and the caller must retry)
//   stats     int64  [4]: stage-2 pairs, stage-3 pairs, stage-4 pairs, visited pairs
// Returns 0 on success, 1 if the unsure buffer was too small, 2 on bad arguments.
int so_generate(const float* X, const float* Nr, int64_t N, const int32_t* cen, int64_t M, int W,
                double b, double cos_As, int mode, int flags, int cells, int threads, double* out,
                int32_t* contrib, int64_t* in_region, int64_t* unsure, int64_t cap,
                int64_t* n_unsure, int64_t* stats) {
  if (N < 1 || M < 0 || W < 1 || !(b > 0) || (mode != NEAREST && mode != BILINEAR)) return 2;
  Job J{X, Nr, N, W, b, cos_As, mode, flags, !(std::isinf(cos_As) && cos_As < 0)};
  const int64_t WW = (int64_t)W * W;
  std::memset(out, 0, sizeof(double) * (size_t)(M * WW));
  if (contrib) std::memset(contrib, 0, sizeof(int32_t) * (size_t)(M * WW));
  Grid grid;
  if (cells) grid.build(X, Nr, N, region_radius(W, b, mode, flags));
  std::atomic<int64_t> next(0);
  std::mutex mu;
  std::vector<Unsure> all_uns;
  int64_t tot[4] = {0, 0, 0, 0};
  auto worker = [&]() {
    PairStats ps;
    std::vector<Unsure> uns;
    std::vector<std::pair<int64_t, int64_t>> ranges;
    int64_t visited = 0;
    for (;;) {
      const int64_t m = next.fetch_add(1);
      if (m >= M) break;
      const int64_t ci = cen[m];
      ImageOut io{out + m * WW, contrib ? contrib + m * WW : nullptr, 0};
      if (ci < 0 || ci >= N) continue;   // the caller validates; an invalid centre is empty
      if (cells) {
        grid.neighbours(X + 3 * ci, ranges);
        for (const auto& r : ranges) {
          image_of(J, m, ci, grid.Xs.data(), grid.Ns.data(), grid.idx_sorted.data(), r.first,
                   r.second, io, ps, uns);
          visited += r.second - r.first;
        }
      } else {
        image_of(J, m, ci, X, Nr, nullptr, 0, N, io, ps, uns);
        visited += N;
      }
      if (in_region) in_region[m] = io.in_region;
    }
    std::lock_guard<std::mutex> g(mu);
    all_uns.insert(all_uns.end(), uns.begin(), uns.end());
    tot[0] += ps.stage2;
    tot[1] += ps.stage3;
    tot[2] += ps.stage4;
    tot[3] += visited;
  };
  const int T = (int)std::min<int64_t>(n_threads(threads), std::max<int64_t>(M, 1));
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  std::sort(all_uns.begin(), all_uns.end(),
            [](const Unsure& a, const Unsure& b2) { return a.m != b2.m ? a.m < b2.m : a.j < b2.j; });
  *n_unsure = (int64_t)all_uns.size();
  if (stats) for (int i = 0; i < 4; ++i) stats[i] = tot[i];
  if ((int64_t)all_uns.size() > cap) return 1;
  for (size_t i = 0; i < all_uns.size(); ++i) {
    unsure[2 * i] = all_uns[i].m;
    unsure[2 * i + 1] = all_uns[i].j;
  }
  return 0;
}

// Per-pair decisions of ONE centre against every cloud point (for the BILINEAR flip count:
// pairs whose GPU (i0, j0) differs from the oracle's).  state[j]: 0 / 1 / 2 (undecided,
// the caller decides exactly); kk[j], ll[j]: NEAREST (k, l) or BILINEAR (i0, j0); uu[j], vv[j]:
// the double u and v = sqrt(max(w, 0)) of the pair.
int so_pair_bins(const float* X, const float* Nr, int64_t N, int64_t ci, int W, double b,
                 double cos_As, int mode, int flags, int threads, int32_t* state, int32_t* kk,
                 int32_t* ll, double* uu, double* vv) {
  if (N < 1 || ci < 0 || ci >= N || W < 1 || !(b > 0)) return 2;
  Job J{X, Nr, N, W, b, cos_As, mode, flags, !(std::isinf(cos_As) && cos_As < 0)};
  const float* p = X + 3 * ci;
  const float* n = Nr + 3 * ci;
  const int T = n_threads(threads);
  auto work = [&](int t) {
    PairStats ps;
    for (int64_t j = t; j < N; j += T) {
      const float* x = X + 3 * j;
      const Outcome o = decide_pair(J, p, n, x, Nr + 3 * j, ps);
      state[j] = o.state;
      kk[j] = o.k;
      ll[j] = o.l;
      const double d0 = (double)x[0] - p[0], d1 = (double)x[1] - p[1], d2 = (double)x[2] - p[2];
      const double beta = ((double)n[0] * d0 + (double)n[1] * d1) + (double)n[2] * d2;
      const double q = (d0 * d0 + d1 * d1) + d2 * d2 - beta * beta;
      uu[j] = (flags & F_LITERAL) ? (W / 2.0 - beta) / b : W / 2.0 - beta / b;
      vv[j] = std::sqrt(std::max(q, 0.0)) / b;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return 0;
}

double so_region_radius(int W, double b, int mode, int flags) {
  return region_radius(W, b, mode, flags);
}

}  // extern "C"
