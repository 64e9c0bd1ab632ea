// ival.cuh -- rigorous FP64 interval arithmetic on sm_100a.
//
// PAPER.md §2.1 Eq. (3)-(6) (lines 63-69) define the interval operations and
// line 71 requires outward rounding.  Here every endpoint is produced by the
// hardware directed-rounding instructions (__dadd_rd/__dadd_ru, __dmul_rd/ru,
// __ddiv_rd/ru, __dsqrt_rd/ru -> DADD/DMUL with .RM/.RP), which are never
// contracted into FMAs.  Transcendentals come from CUDA's libdevice (exp: 1
// ulp, sinpi/cospi: 2 ulp documented maximum error) and are widened outward by
// one more ulp step than documented; the widening step x -> __dsub_rd(x,
// 2^-1074) is exactly nextafter(x, -inf) because directed rounding of x minus
// the smallest subnormal always lands on the neighbouring double.
//
// Periodic functions are evaluated in units of pi (sinpi/cospi), so the
// extremum test "does U contain an integer" is exact in floating point; a
// general argument t is first mapped to u = t * [1/pi] with outward rounding.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace ib {

struct Iv {
  double lo, hi;
};

// tight enclosures of constants, checked by tests/test_capi_symbols.py
// against 50-digit rationals
namespace K {
constexpr double PI_LO = 0x1.921fb54442d18p+1, PI_HI = 0x1.921fb54442d19p+1;
constexpr double INV_PI_LO = 0x1.45f306dc9c882p-2, INV_PI_HI = 0x1.45f306dc9c883p-2;
constexpr double E_LO = 0x1.5bf0a8b145769p+1, E_HI = 0x1.5bf0a8b14576ap+1;
constexpr double C0_02_LO = 0x1.47ae147ae147ap-6, C0_02_HI = 0x1.47ae147ae147bp-6;
constexpr double C0_1_LO = 0x1.9999999999999p-4, C0_1_HI = 0x1.999999999999ap-4;
constexpr double C0_9_LO = 0x1.cccccccccccccp-1, C0_9_HI = 0x1.ccccccccccccdp-1;
constexpr double TINY = 0x1p-1074;
}  // namespace K

constexpr int ULPS_TRIG = 3;  // documented 2 ulp (sinpi, cospi) + 1
constexpr int ULPS_EXP = 2;   // documented 1 ulp (exp) + 1

__device__ __forceinline__ Iv iv(double a) { return Iv{a, a}; }
__device__ __forceinline__ Iv iv(double a, double b) { return Iv{a, b}; }

__device__ __forceinline__ double next_dn(double x) { return __dsub_rd(x, K::TINY); }
__device__ __forceinline__ double next_up(double x) { return __dadd_ru(x, K::TINY); }
template <int S>
__device__ __forceinline__ double widen_dn(double x) {
#pragma unroll
  for (int i = 0; i < S; ++i) x = next_dn(x);
  return x;
}
template <int S>
__device__ __forceinline__ double widen_up(double x) {
#pragma unroll
  for (int i = 0; i < S; ++i) x = next_up(x);
  return x;
}

__device__ __forceinline__ Iv operator+(Iv a, Iv b) { return Iv{__dadd_rd(a.lo, b.lo), __dadd_ru(a.hi, b.hi)}; }
__device__ __forceinline__ Iv operator-(Iv a, Iv b) { return Iv{__dsub_rd(a.lo, b.hi), __dsub_ru(a.hi, b.lo)}; }
__device__ __forceinline__ Iv operator-(Iv a) { return Iv{-a.hi, -a.lo}; }

// Eq. (5): min / max of the four endpoint products
__device__ __forceinline__ Iv operator*(Iv a, Iv b) {
  double p0 = __dmul_rd(a.lo, b.lo), p1 = __dmul_rd(a.lo, b.hi);
  double p2 = __dmul_rd(a.hi, b.lo), p3 = __dmul_rd(a.hi, b.hi);
  double q0 = __dmul_ru(a.lo, b.lo), q1 = __dmul_ru(a.lo, b.hi);
  double q2 = __dmul_ru(a.hi, b.lo), q3 = __dmul_ru(a.hi, b.hi);
  return Iv{fmin(fmin(p0, p1), fmin(p2, p3)), fmax(fmax(q0, q1), fmax(q2, q3))};
}

// product by a point constant c (exact c)
__device__ __forceinline__ Iv scale(double c, Iv a) {
  return c >= 0.0 ? Iv{__dmul_rd(c, a.lo), __dmul_ru(c, a.hi)}
                  : Iv{__dmul_rd(c, a.hi), __dmul_ru(c, a.lo)};
}

// Eq. (6) for a divisor interval b with 0 not in b
__device__ __forceinline__ Iv operator/(Iv a, Iv b) {
  if (b.lo <= 0.0 && b.hi >= 0.0) return Iv{-CUDART_INF, CUDART_INF};
  double p0 = __ddiv_rd(a.lo, b.lo), p1 = __ddiv_rd(a.lo, b.hi);
  double p2 = __ddiv_rd(a.hi, b.lo), p3 = __ddiv_rd(a.hi, b.hi);
  double q0 = __ddiv_ru(a.lo, b.lo), q1 = __ddiv_ru(a.lo, b.hi);
  double q2 = __ddiv_ru(a.hi, b.lo), q3 = __ddiv_ru(a.hi, b.hi);
  return Iv{fmin(fmin(p0, p1), fmin(p2, p3)), fmax(fmax(q0, q1), fmax(q2, q3))};
}

// division by a positive point constant c
__device__ __forceinline__ Iv divc(Iv a, double c) { return Iv{__ddiv_rd(a.lo, c), __ddiv_ru(a.hi, c)}; }

__device__ __forceinline__ Iv sqr(Iv a) {
  if (a.lo >= 0.0) return Iv{__dmul_rd(a.lo, a.lo), __dmul_ru(a.hi, a.hi)};
  if (a.hi <= 0.0) return Iv{__dmul_rd(a.hi, a.hi), __dmul_ru(a.lo, a.lo)};
  double m = fmax(-a.lo, a.hi);
  return Iv{0.0, __dmul_ru(m, m)};
}

__device__ __forceinline__ Iv isqrt(Iv a) {
  return Iv{__dsqrt_rd(fmax(a.lo, 0.0)), __dsqrt_ru(fmax(a.hi, 0.0))};
}

// the transcendental enclosures are out-of-line: one copy of their code per
// kernel keeps the instruction footprint of the large kernels (k_fused,
// k_search) small enough to stay in the instruction caches
static __device__ __noinline__ Iv iexp(Iv a) {
  return Iv{fmax(widen_dn<ULPS_EXP>(exp(a.lo)), 0.0), widen_up<ULPS_EXP>(exp(a.hi))};
}

// cos(pi u) over U: maxima at even integers, minima at odd integers.
static __device__ __noinline__ Iv icospi(Iv u) {
  if (!(u.lo <= u.hi) || !(__dsub_ru(u.hi, u.lo) < 2.0) || fabs(u.lo) > 0x1p50 || fabs(u.hi) > 0x1p50)
    return Iv{-1.0, 1.0};
  double c0 = cospi(u.lo), c1 = cospi(u.hi);
  Iv r{widen_dn<ULPS_TRIG>(fmin(c0, c1)), widen_up<ULPS_TRIG>(fmax(c0, c1))};
  double k = ceil(u.lo);  // width < 2: at most k and k + 1 lie in U
  if (k <= u.hi) {
    if (fmod(k, 2.0) == 0.0) r.hi = 1.0; else r.lo = -1.0;
  }
  if (k + 1.0 <= u.hi) {
    if (fmod(k + 1.0, 2.0) == 0.0) r.hi = 1.0; else r.lo = -1.0;
  }
  return Iv{fmax(r.lo, -1.0), fmin(r.hi, 1.0)};
}

// sin(pi u) over U: maxima at u = k + 1/2 with k even, minima with k odd.
static __device__ __noinline__ Iv isinpi(Iv u) {
  if (!(u.lo <= u.hi) || !(__dsub_ru(u.hi, u.lo) < 2.0) || fabs(u.lo) > 0x1p50 || fabs(u.hi) > 0x1p50)
    return Iv{-1.0, 1.0};
  double s0 = sinpi(u.lo), s1 = sinpi(u.hi);
  Iv r{widen_dn<ULPS_TRIG>(fmin(s0, s1)), widen_up<ULPS_TRIG>(fmax(s0, s1))};
  double vlo = __dsub_rd(u.lo, 0.5), vhi = __dsub_ru(u.hi, 0.5);
  double k = ceil(vlo);
  for (int t = 0; t < 3; ++t, k += 1.0) {
    if (k <= vhi) {
      if (fmod(k, 2.0) == 0.0) r.hi = 1.0; else r.lo = -1.0;
    }
  }
  return Iv{fmax(r.lo, -1.0), fmin(r.hi, 1.0)};
}

// t -> t / pi, outward
__device__ __forceinline__ Iv over_pi(Iv t) {
  return Iv{t.lo >= 0.0 ? __dmul_rd(t.lo, K::INV_PI_LO) : __dmul_rd(t.lo, K::INV_PI_HI),
            t.hi >= 0.0 ? __dmul_ru(t.hi, K::INV_PI_HI) : __dmul_ru(t.hi, K::INV_PI_LO)};
}
__device__ __forceinline__ Iv icos(Iv t) { return icospi(over_pi(t)); }
__device__ __forceinline__ Iv isin(Iv t) { return isinpi(over_pi(t)); }

__device__ __forceinline__ Iv c_pi() { return Iv{K::PI_LO, K::PI_HI}; }
__device__ __forceinline__ Iv c_e() { return Iv{K::E_LO, K::E_HI}; }
__device__ __forceinline__ Iv c_002() { return Iv{K::C0_02_LO, K::C0_02_HI}; }
__device__ __forceinline__ Iv c_01() { return Iv{K::C0_1_LO, K::C0_1_HI}; }
__device__ __forceinline__ Iv c_09() { return Iv{K::C0_9_LO, K::C0_9_HI}; }

// ordered 64-bit key of a double: unsigned order == double order
__device__ __forceinline__ uint64_t okey(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// canonical lower bound: NaN -> -inf, -0 -> +0 (reading R7)
__device__ __forceinline__ double canon_lb(double x) {
  if (x != x) return -CUDART_INF;
  return x == 0.0 ? 0.0 : x;
}

}  // namespace ib
