// objectives.cuh -- interval extensions of the ten benchmark objectives of
// PAPER.md Appendix A (lines 264-348) plus the §2.1 worked example (line 75),
// and of their first-order partial derivatives (§3.1).
//
// Every objective is written as an outer function of K "accumulators", each a
// sum or a product over the n variables of a per-variable term:
//     f(x) = outer(A_0, ..., A_{K-1}),   A_k = (+ or *)_i term_k(x_i, i).
// This is exactly the natural interval extension of the Appendix A formula
// (reading R3); the grouping lets the branch kernel reuse the
// per-variable terms of a parent for all of its m^d children.  Levy (A11) is
// a chain sum (term i couples y_i and y_{i+1}) and is handled separately
// (CHAIN = true).
//
// Derivative interface: separable objectives (SEP = true) have d f / d x_i =
// dsep(x_i); the others are dfin(ctx(A), g(x_i), x_i, excl) where g are per
// variable ingredients and excl[k] is the product accumulator A_k without
// variable i.
#pragma once
#include "ival.cuh"

namespace ib {

enum { SUM = 0, PROD = 1 };

// x * p for an interval p with p.lo >= 0: exactly the two products Eq. (5)
// selects (bit-identical to the general operator*, 2 DMUL instead of 8)
__device__ __forceinline__ Iv mulpos(Iv x, Iv p) {
  return Iv{x.lo >= 0.0 ? __dmul_rd(x.lo, p.lo) : __dmul_rd(x.lo, p.hi),
            x.hi >= 0.0 ? __dmul_ru(x.hi, p.hi) : __dmul_ru(x.hi, p.lo)};
}

// outward reciprocal [1/r.hi, 1/r.lo] of an interval with r.lo > 0
__device__ __forceinline__ Iv recip_pos(Iv r) { return Iv{__drcp_rd(r.hi), __drcp_ru(r.lo)}; }

// x_i / r over a box, with |x_i / r| <= s known a priori (R5);
// rinv = recip_pos(r) when r.lo > 0 (x * [1/r] encloses x / r)
__device__ __forceinline__ Iv ratio_q(Iv x, Iv r, Iv rinv, double s) {
  if (r.lo > 0.0) {
    Iv q = mulpos(x, rinv);
    return Iv{fmax(q.lo, -s), fmin(q.hi, s)};
  }
  return Iv{x.lo >= 0.0 ? 0.0 : -s, x.hi <= 0.0 ? 0.0 : s};
}

__device__ __forceinline__ Iv two_x(Iv x) { return scale(2.0, x); }
__device__ __forceinline__ Iv c_pi_s(double c) { return scale(c, c_pi()); }

struct NoCtx {};

// ---------------------------------------------------------------- fid 0
// §2.1 line 75: f = sum_i (x_i - x_i * x_i)
struct ObjExample {
  static constexpr int K = 1, KG = 0;
  static constexpr bool SEP = true, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) { t[0] = x - x * x; }
  __device__ static Iv outer(const Iv* A, int) { return A[0]; }
  __device__ static Iv dsep(Iv x, int, int) { return iv(1.0) - two_x(x); }
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv, int, int, Iv*) {}
  __device__ static Iv dfin(const Ctx&, const Iv*, Iv x, int i, int n, const Iv*) { return dsep(x, i, n); }
};

// ---------------------------------------------------------------- fid 1
// (A1) -20 exp(-0.02 sqrt(A0/n)) - exp(A1/n) + 20 + e, A0 = sum x^2, A1 = sum cos(2 pi x)
struct ObjAckley {
  static constexpr int K = 2, KG = 2;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) {
    t[0] = sqr(x);
    t[1] = icospi(two_x(x));
  }
  __device__ static Iv outer(const Iv* A, int n) {
    Iv r = isqrt(divc(A[0], (double)n));
    Iv t1 = scale(-20.0, iexp(-c_002() * r));
    Iv t2 = -iexp(divc(A[1], (double)n));
    return ((t1 + t2) + iv(20.0)) + c_e();
  }
  // lower / upper endpoint of outer() alone: the same operations as outer()
  // restricted to the endpoint they feed (bit-identical to outer().lo/.hi)
  __device__ static double outer_lo(const Iv* A, int n) {
    double rlo = __dsqrt_rd(fmax(__ddiv_rd(A[0].lo, (double)n), 0.0));
    double e1 = widen_up<ULPS_EXP>(exp(__dmul_ru(-K::C0_02_LO, rlo)));
    double t1 = __dmul_rd(-20.0, e1);
    double t2 = -widen_up<ULPS_EXP>(exp(__ddiv_ru(A[1].hi, (double)n)));
    return __dadd_rd(__dadd_rd(__dadd_rd(t1, t2), 20.0), K::E_LO);
  }
  __device__ static double outer_hi(const Iv* A, int n) {
    double rhi = __dsqrt_ru(fmax(__ddiv_ru(A[0].hi, (double)n), 0.0));
    double e1 = fmax(widen_dn<ULPS_EXP>(exp(__dmul_rd(-K::C0_02_HI, rhi))), 0.0);
    double t1 = __dmul_ru(-20.0, e1);
    double t2 = -fmax(widen_dn<ULPS_EXP>(exp(__ddiv_rd(A[1].lo, (double)n))), 0.0);
    return __dadd_ru(__dadd_ru(__dadd_ru(t1, t2), 20.0), K::E_HI);
  }
  // d f/d x_i = (0.4/n) e^{-0.02 r} x_i/r + (2 pi/n) e^{A1/n} sin(2 pi x_i)
  struct Ctx {
    Iv r, rinv, a, b;
    double s;
  };
  __device__ static Ctx ctx(const Iv* A, int n) {
    Ctx c;
    c.r = isqrt(divc(A[0], (double)n));
    c.rinv = c.r.lo > 0.0 ? recip_pos(c.r) : Iv{0.0, 0.0};
    c.a = mulpos(iexp(-c_002() * c.r), divc(scale(4.0, c_01()), (double)n));  // both factors >= 0
    c.b = mulpos(iexp(divc(A[1], (double)n)), divc(c_pi_s(2.0), (double)n));
    c.s = __dsqrt_ru((double)n);
    return c;
  }
  __device__ static void ding(Iv x, int, int, Iv* g) {
    g[0] = x;
    g[1] = isinpi(two_x(x));
  }
  __device__ static Iv dfin(const Ctx& c, const Iv* g, Iv, int, int, const Iv*) {
    return mulpos(ratio_q(g[0], c.r, c.rinv, c.s), c.a) + mulpos(g[1], c.b);
  }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// ---------------------------------------------------------------- fid 2
// (A3) 0.1 A0 - cos(5 sqrt(A0)), A0 = sum (x-5)^2
struct ObjBelegundu {
  static constexpr int K = 1, KG = 1;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) { t[0] = sqr(x - iv(5.0)); }
  __device__ static Iv outer(const Iv* A, int) {
    Iv r = isqrt(A[0]);
    return c_01() * A[0] - icos(scale(5.0, r));
  }
  // (x_i - 5)(0.2 + 5 H), H = sin(5 r)/r in [-5, 5]
  struct Ctx {
    Iv G;
  };
  __device__ static Ctx ctx(const Iv* A, int) {
    Iv r = isqrt(A[0]);
    Iv h{-5.0, 5.0};
    if (r.lo > 0.0) {
      Iv q = isin(scale(5.0, r)) / r;
      h = Iv{fmax(q.lo, -5.0), fmin(q.hi, 5.0)};
    }
    return Ctx{scale(2.0, c_01()) + scale(5.0, h)};
  }
  __device__ static void ding(Iv x, int, int, Iv* g) { g[0] = x - iv(5.0); }
  __device__ static Iv dfin(const Ctx& c, const Iv* g, Iv, int, int, const Iv*) { return g[0] * c.G; }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// ---------------------------------------------------------------- fid 3
// (A5) -0.1 A0 + A1, A0 = sum cos(5 pi x), A1 = sum x^2
struct ObjBreiman {
  static constexpr int K = 2, KG = 0;
  static constexpr bool SEP = true, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) {
    t[0] = icospi(scale(5.0, x));
    t[1] = sqr(x);
  }
  __device__ static Iv outer(const Iv* A, int) { return (-c_01()) * A[0] + A[1]; }
  // 0.5 pi sin(5 pi x) + 2 x
  __device__ static Iv dsep(Iv x, int, int) { return c_pi_s(0.5) * isinpi(scale(5.0, x)) + two_x(x); }
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv, int, int, Iv*) {}
  __device__ static Iv dfin(const Ctx&, const Iv*, Iv x, int i, int n, const Iv*) { return dsep(x, i, n); }
};

// ---------------------------------------------------------------- fid 4
// (A7) 1 + sum [8 sin^2(7 g^2) + 6 sin^2(14 g^2) + g^2], g = x - 0.9
struct ObjFu {
  static constexpr int K = 1, KG = 0;
  static constexpr bool SEP = true, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) {
    Iv g = x - c_09();
    Iv q = sqr(g);
    Iv a = sqr(isin(scale(7.0, q)));
    Iv b = sqr(isin(scale(14.0, q)));
    t[0] = (scale(8.0, a) + scale(6.0, b)) + q;
  }
  __device__ static Iv outer(const Iv* A, int) { return iv(1.0) + A[0]; }
  // g (112 sin(14 q) + 168 sin(28 q) + 2)
  __device__ static Iv dsep(Iv x, int, int) {
    Iv g = x - c_09();
    Iv q = sqr(g);
    Iv t = (scale(112.0, isin(scale(14.0, q))) + scale(168.0, isin(scale(28.0, q)))) + iv(2.0);
    return g * t;
  }
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv, int, int, Iv*) {}
  __device__ static Iv dfin(const Ctx&, const Iv*, Iv x, int i, int n, const Iv*) { return dsep(x, i, n); }
};

// ---------------------------------------------------------------- fid 5
// (A9) 1 + A0/4000 - A1, A0 = sum x^2, A1 = prod cos(x_i / sqrt(i))
__device__ __forceinline__ Iv griewank_kappa(int i0) {
  double k = (double)(i0 + 1);
  return Iv{__ddiv_rd(1.0, __dsqrt_ru(k)), __ddiv_ru(1.0, __dsqrt_rd(k))};
}
struct ObjGriewank {
  static constexpr int K = 2, KG = 2;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = true;
  __device__ static int kind(int k) { return k == 0 ? SUM : PROD; }
  __device__ static void terms(Iv x, int i, int, Iv* t) {
    t[0] = sqr(x);
    t[1] = icos(mulpos(x, griewank_kappa(i)));
  }
  __device__ static Iv outer(const Iv* A, int) { return (iv(1.0) + divc(A[0], 4000.0)) - A[1]; }
  // x_i/2000 + k_i sin(k_i x_i) prod_{j != i} cos(k_j x_j)
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv x, int i, int, Iv* g) {
    Iv k = griewank_kappa(i);
    g[0] = divc(x, 2000.0);
    g[1] = mulpos(isin(mulpos(x, k)), k);
  }
  __device__ static Iv dfin(const Ctx&, const Iv* g, Iv, int, int, const Iv* excl) { return g[0] + g[1] * excl[1]; }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// ---------------------------------------------------------------- fid 6
// (A11)-(A12) Levy, chain form.  Per-variable quantities:
//   y = 1 + 0.25 (x - 1), u = (y - 1)^2, v = 1 + 10 sin^2(pi y),
//   s0 = 10 sin^2(pi y) (first term, variable 1 only),
//   du = (y - 1)/2 = du/dx, sg = 2.5 pi sin(2 pi y) = dv/dx.
// f = pi/n { s0(y_1) + sum_{i<n} u_i v_{i+1} + u_n }.
struct LevyVals {
  Iv u, v, s0, du, sg;
};
struct ObjLevy {
  static constexpr int K = 1, KG = 0;
  static constexpr bool SEP = false, CHAIN = true;
  static constexpr bool HASPROD = false;
  __device__ static LevyVals vals(Iv x) {
    Iv y = iv(1.0) + scale(0.25, x - iv(1.0));
    Iv ym1 = y - iv(1.0);
    Iv sp = sqr(isinpi(y));
    LevyVals r;
    r.u = sqr(ym1);
    r.s0 = scale(10.0, sp);
    r.v = iv(1.0) + r.s0;
    r.du = scale(0.5, ym1);
    r.sg = c_pi_s(2.5) * isinpi(two_x(y));
    return r;
  }
  __device__ static Iv outer(Iv acc, int n) { return mulpos(acc, divc(c_pi(), (double)n)); }
  // d f / d x_i (0-based i); uprev = u_{i-1}, vnext = v_{i+1}
  __device__ static Iv deriv(const LevyVals& me, Iv uprev, Iv vnext, int i, int n) {
    Iv acc = iv(0.0);
    if (i == 0) acc = acc + me.sg;
    if (i < n - 1) acc = acc + mulpos(me.du, vnext);  // v >= 1
    if (i > 0) acc = acc + mulpos(me.sg, uprev);      // u >= 0
    if (i == n - 1) acc = acc + me.du;
    return mulpos(acc, divc(c_pi(), (double)n));
  }
};

// ---------------------------------------------------------------- fid 7
// (A14) 10 n + sum [x^2 - 10 cos(2 pi x)]
struct ObjRastrigin {
  static constexpr int K = 1, KG = 0;
  static constexpr bool SEP = true, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) { t[0] = sqr(x) - scale(10.0, icospi(two_x(x))); }
  __device__ static Iv outer(const Iv* A, int n) { return iv(10.0 * (double)n) + A[0]; }
  // 2 x + 20 pi sin(2 pi x)
  __device__ static Iv dsep(Iv x, int, int) { return two_x(x) + c_pi_s(20.0) * isinpi(two_x(x)); }
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv, int, int, Iv*) {}
  __device__ static Iv dfin(const Ctx&, const Iv*, Iv x, int i, int n, const Iv*) { return dsep(x, i, n); }
};

// ---------------------------------------------------------------- fid 8
// (A16) 1 - cos(2 pi r) + 0.1 r, r = sqrt(sum x^2)
struct ObjSalomon {
  static constexpr int K = 1, KG = 1;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = false;
  __device__ static int kind(int) { return SUM; }
  __device__ static void terms(Iv x, int, int, Iv* t) { t[0] = sqr(x); }
  __device__ static Iv outer(const Iv* A, int) {
    Iv r = isqrt(A[0]);
    return (iv(1.0) - icospi(two_x(r))) + c_01() * r;
  }
  // (2 pi sin(2 pi r) + 0.1) x_i / r, |x_i/r| <= 1
  struct Ctx {
    Iv r, rinv, t;
  };
  __device__ static Ctx ctx(const Iv* A, int) {
    Ctx c;
    c.r = isqrt(A[0]);
    c.rinv = c.r.lo > 0.0 ? recip_pos(c.r) : Iv{0.0, 0.0};
    c.t = mulpos(isinpi(two_x(c.r)), c_pi_s(2.0)) + c_01();
    return c;
  }
  __device__ static void ding(Iv x, int, int, Iv* g) { g[0] = x; }
  __device__ static Iv dfin(const Ctx& c, const Iv* g, Iv, int, int, const Iv*) {
    return c.t * ratio_q(g[0], c.r, c.rinv, 1.0);
  }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// ---------------------------------------------------------------- fid 9
// (A18) A0/(2n) - 4n A1, A0 = sum x^2, A1 = prod cos x
struct ObjStyblinski {
  static constexpr int K = 2, KG = 2;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = true;
  __device__ static int kind(int k) { return k == 0 ? SUM : PROD; }
  __device__ static void terms(Iv x, int, int, Iv* t) {
    t[0] = sqr(x);
    t[1] = icos(x);
  }
  __device__ static Iv outer(const Iv* A, int n) {
    return divc(A[0], 2.0 * (double)n) - mulpos(A[1], iv(4.0 * (double)n));
  }
  // x_i / n + 4 n sin(x_i) prod_{j != i} cos(x_j)
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv x, int, int n, Iv* g) {
    g[0] = divc(x, (double)n);
    g[1] = mulpos(isin(x), iv(4.0 * (double)n));
  }
  __device__ static Iv dfin(const Ctx&, const Iv* g, Iv, int, int, const Iv* excl) { return g[0] + g[1] * excl[1]; }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// ---------------------------------------------------------------- fid 10
// (A20) -2.5 A0 - A1, A0 = prod sin(x - pi/6), A1 = prod sin(5 (x - pi/6))
struct ObjZabinsky {
  static constexpr int K = 2, KG = 2;
  static constexpr bool SEP = false, CHAIN = false;
  static constexpr bool HASPROD = true;
  __device__ static int kind(int) { return PROD; }
  __device__ static Iv g_of(Iv x) { return x - divc(c_pi(), 6.0); }
  __device__ static void terms(Iv x, int, int, Iv* t) {
    Iv g = g_of(x);
    t[0] = isin(g);
    t[1] = isin(scale(5.0, g));
  }
  __device__ static Iv outer(const Iv* A, int) { return scale(-2.5, A[0]) - A[1]; }
  // -2.5 cos(g_i) prod_{j!=i} sin(g_j) - 5 cos(5 g_i) prod_{j!=i} sin(5 g_j)
  using Ctx = NoCtx;
  __device__ static Ctx ctx(const Iv*, int) { return {}; }
  __device__ static void ding(Iv x, int, int, Iv* g) {
    Iv gg = g_of(x);
    g[0] = scale(-2.5, icos(gg));
    g[1] = scale(-5.0, icos(scale(5.0, gg)));
  }
  __device__ static Iv dfin(const Ctx&, const Iv* g, Iv, int, int, const Iv* excl) {
    return g[0] * excl[0] + g[1] * excl[1];
  }
  __device__ static Iv dsep(Iv, int, int) { return Iv{-CUDART_INF, CUDART_INF}; }
};

// endpoint-only evaluation of outer(): F::outer_lo / F::outer_hi when the
// objective provides them (cheaper), else the full interval's endpoint
template <class F, class = void>
struct HasOuterLo {
  static constexpr bool value = false;
};
template <class F>
struct HasOuterLo<F, decltype((void)F::outer_lo)> {
  static constexpr bool value = true;
};
template <class F>
__device__ __forceinline__ double outer_lo(const Iv* A, int n) {
  if constexpr (HasOuterLo<F>::value) return F::outer_lo(A, n);
  else return F::outer(A, n).lo;
}
template <class F>
__device__ __forceinline__ double outer_hi(const Iv* A, int n) {
  if constexpr (HasOuterLo<F>::value) return F::outer_hi(A, n);
  else return F::outer(A, n).hi;
}

template <class F>
__device__ __forceinline__ Iv acc_ident(int k) {
  return F::kind(k) == PROD ? iv(1.0) : iv(0.0);
}
template <class F>
__device__ __forceinline__ Iv acc_comb(int k, Iv a, Iv b) {
  return F::kind(k) == PROD ? a * b : a + b;
}

// fid -> type dispatch
#define IB_DISPATCH_FID(fid, ...)                                  \
  switch (fid) {                                                   \
    case 0: { using F = ObjExample; __VA_ARGS__; } break;          \
    case 1: { using F = ObjAckley; __VA_ARGS__; } break;           \
    case 2: { using F = ObjBelegundu; __VA_ARGS__; } break;        \
    case 3: { using F = ObjBreiman; __VA_ARGS__; } break;          \
    case 4: { using F = ObjFu; __VA_ARGS__; } break;               \
    case 5: { using F = ObjGriewank; __VA_ARGS__; } break;         \
    case 6: { using F = ObjLevy; __VA_ARGS__; } break;             \
    case 7: { using F = ObjRastrigin; __VA_ARGS__; } break;        \
    case 8: { using F = ObjSalomon; __VA_ARGS__; } break;          \
    case 9: { using F = ObjStyblinski; __VA_ARGS__; } break;       \
    case 10: { using F = ObjZabinsky; __VA_ARGS__; } break;        \
    default: break;                                                \
  }

}  // namespace ib
