/*
 * oracle/ia.c -- interval arithmetic for the CPU oracle (TEST INFRASTRUCTURE).
 * See ia.h for the paper passages followed.  Compiled with
 *   -frounding-math -ffp-contract=off
 * so that GCC neither folds nor contracts across rounding-mode changes.
 */
#include "ia.h"

#include <fenv.h>
#include <math.h>
#include <stdlib.h>

/* GCC ignores FENV_ACCESS; -frounding-math (Makefile) is what makes this safe. */

ia_consts_t IA_C;

/* ---- directed scalar operations: set mode, compute, restore ----------- */
#define DIRECTED2(NAME, MODE, OP)                     \
    double NAME(double a, double b) {                 \
        volatile double va = a, vb = b, r;            \
        fesetround(MODE);                             \
        r = va OP vb;                                 \
        fesetround(FE_TONEAREST);                     \
        return r;                                     \
    }
DIRECTED2(ia_add_dn, FE_DOWNWARD, +)
DIRECTED2(ia_add_up, FE_UPWARD, +)
DIRECTED2(ia_sub_dn, FE_DOWNWARD, -)
DIRECTED2(ia_sub_up, FE_UPWARD, -)
DIRECTED2(ia_mul_dn, FE_DOWNWARD, *)
DIRECTED2(ia_mul_up, FE_UPWARD, *)
DIRECTED2(ia_div_dn, FE_DOWNWARD, /)
DIRECTED2(ia_div_up, FE_UPWARD, /)

double ia_sqrt_dn(double a) {
    volatile double va = a, r;
    fesetround(FE_DOWNWARD);
    r = sqrt(va);
    fesetround(FE_TONEAREST);
    return r;
}
double ia_sqrt_up(double a) {
    volatile double va = a, r;
    fesetround(FE_UPWARD);
    r = sqrt(va);
    fesetround(FE_TONEAREST);
    return r;
}

double ia_widen_dn(double x, int k) {
    for (int i = 0; i < k; ++i) x = nextafter(x, -INFINITY);
    return x;
}
double ia_widen_up(double x, int k) {
    for (int i = 0; i < k; ++i) x = nextafter(x, INFINITY);
    return x;
}

ia_t ia_from_decimal(const char* s) {
    ia_t r;
    fesetround(FE_DOWNWARD);
    r.lo = strtod(s, NULL);
    fesetround(FE_UPWARD);
    r.hi = strtod(s, NULL);
    fesetround(FE_TONEAREST);
    return r;
}

double ia_max(double a, double b) { return a > b ? a : b; }
double ia_min(double a, double b) { return a < b ? a : b; }

ia_t ia_pt(double x) {
    ia_t r = {x, x};
    return r;
}
ia_t ia_make(double lo, double hi) {
    ia_t r = {lo, hi};
    return r;
}
ia_t ia_neg(ia_t a) { return ia_make(-a.hi, -a.lo); }

/* Eq. (3): [x1,x2] + [y1,y2] = [x1 + y1, x2 + y2] */
ia_t ia_add(ia_t a, ia_t b) { return ia_make(ia_add_dn(a.lo, b.lo), ia_add_up(a.hi, b.hi)); }

/* Eq. (4): [x1,x2] - [y1,y2] = [x1 - y2, x2 - y1] */
ia_t ia_sub(ia_t a, ia_t b) { return ia_make(ia_sub_dn(a.lo, b.hi), ia_sub_up(a.hi, b.lo)); }

/* Eq. (5): min / max of the four endpoint products */
ia_t ia_mul(ia_t a, ia_t b) {
    double p[4] = {ia_mul_dn(a.lo, b.lo), ia_mul_dn(a.lo, b.hi), ia_mul_dn(a.hi, b.lo),
                   ia_mul_dn(a.hi, b.hi)};
    double q[4] = {ia_mul_up(a.lo, b.lo), ia_mul_up(a.lo, b.hi), ia_mul_up(a.hi, b.lo),
                   ia_mul_up(a.hi, b.hi)};
    ia_t r = {p[0], q[0]};
    for (int i = 1; i < 4; ++i) {
        r.lo = ia_min(r.lo, p[i]);
        r.hi = ia_max(r.hi, q[i]);
    }
    return r;
}

/* Eq. (6): a / b = a * (1/b); here written directly as min/max of the four
 * endpoint quotients, valid because every caller passes b with 0 not in b. */
ia_t ia_div(ia_t a, ia_t b) {
    if (b.lo <= 0.0 && b.hi >= 0.0) return ia_make(-INFINITY, INFINITY);
    double p[4] = {ia_div_dn(a.lo, b.lo), ia_div_dn(a.lo, b.hi), ia_div_dn(a.hi, b.lo),
                   ia_div_dn(a.hi, b.hi)};
    double q[4] = {ia_div_up(a.lo, b.lo), ia_div_up(a.lo, b.hi), ia_div_up(a.hi, b.lo),
                   ia_div_up(a.hi, b.hi)};
    ia_t r = {p[0], q[0]};
    for (int i = 1; i < 4; ++i) {
        r.lo = ia_min(r.lo, p[i]);
        r.hi = ia_max(r.hi, q[i]);
    }
    return r;
}

/* x^2 over a: the exact range of the square (one occurrence of x, so no
 * dependence problem, §2.1 line 75). */
ia_t ia_sqr(ia_t a) {
    if (a.lo >= 0.0) return ia_make(ia_mul_dn(a.lo, a.lo), ia_mul_up(a.hi, a.hi));
    if (a.hi <= 0.0) return ia_make(ia_mul_dn(a.hi, a.hi), ia_mul_up(a.lo, a.lo));
    double m = ia_max(-a.lo, a.hi);
    return ia_make(0.0, ia_mul_up(m, m));
}

ia_t ia_sqrt(ia_t a) {
    double lo = a.lo > 0.0 ? a.lo : 0.0;
    double hi = a.hi > 0.0 ? a.hi : 0.0;
    return ia_make(ia_sqrt_dn(lo), ia_sqrt_up(hi));
}

ia_t ia_exp(ia_t a) {
    double lo = ia_widen_dn(exp(a.lo), IA_LIBM_ULPS);
    double hi = ia_widen_up(exp(a.hi), IA_LIBM_ULPS);
    if (lo < 0.0) lo = 0.0;
    return ia_make(lo, hi);
}

/* Range of cos over T=[t0,t1].  cos is monotone between consecutive multiples
 * of pi; its maxima are at 2k*pi and minima at (2k+1)*pi.  For every integer j
 * whose enclosure j*[pi_lo,pi_hi] meets T we include the extremum (this is
 * conservative when the meeting is only due to the width of the pi
 * enclosure).  Endpoint values come from libm, widened outward. */
static ia_t range_periodic(ia_t t, int is_sin) {
    if (!(t.lo <= t.hi)) return ia_make(-1.0, 1.0);
    ia_t two_pi = ia_make(2.0 * IA_C.pi.lo, 2.0 * IA_C.pi.hi);
    if (ia_sub_up(t.hi, t.lo) >= two_pi.lo) return ia_make(-1.0, 1.0);
    double c0 = is_sin ? sin(t.lo) : cos(t.lo);
    double c1 = is_sin ? sin(t.hi) : cos(t.hi);
    ia_t r = ia_make(ia_widen_dn(ia_min(c0, c1), IA_LIBM_ULPS),
                     ia_widen_up(ia_max(c0, c1), IA_LIBM_ULPS));
    /* candidate extremum indices: extremum j sits at (j + off) * pi,
     * off = 0 for cos, 1/2 for sin */
    double off = is_sin ? 0.5 : 0.0;
    double jlo = floor(t.lo / IA_C.pi.hi - off) - 2.0;
    double jhi = ceil(t.hi / IA_C.pi.lo - off) + 2.0;
    /* also consider the other rounding of the quotient (negative t) */
    jlo = ia_min(jlo, floor(t.lo / IA_C.pi.lo - off) - 2.0);
    jhi = ia_max(jhi, ceil(t.hi / IA_C.pi.hi - off) + 2.0);
    for (double j = jlo; j <= jhi; j += 1.0) {
        ia_t pos = ia_mul(ia_pt(j + off), IA_C.pi); /* j+off exact: |j| < 2^51 */
        if (pos.hi >= t.lo && pos.lo <= t.hi) {
            /* cos: j even -> +1, odd -> -1.  sin: (j+1/2)pi, j even -> +1. */
            double jm = fmod(fabs(j), 2.0);
            if (jm == 0.0)
                r.hi = 1.0;
            else
                r.lo = -1.0;
        }
    }
    if (r.lo < -1.0) r.lo = -1.0;
    if (r.hi > 1.0) r.hi = 1.0;
    return r;
}

ia_t ia_cos(ia_t a) { return range_periodic(a, 0); }
ia_t ia_sin(ia_t a) { return range_periodic(a, 1); }

ia_t ia_hull(ia_t a, ia_t b) { return ia_make(ia_min(a.lo, b.lo), ia_max(a.hi, b.hi)); }
ia_t ia_intersect(ia_t a, ia_t b) { return ia_make(ia_max(a.lo, b.lo), ia_min(a.hi, b.hi)); }

/* Decimal expansions (40+ significant digits) of the constants the paper's
 * benchmark functions use (Appendix A).  strtod under directed rounding gives
 * the tightest enclosing doubles. */
void ia_init(void) {
    IA_C.pi = ia_from_decimal("3.14159265358979323846264338327950288419716939937510");
    IA_C.e = ia_from_decimal("2.71828182845904523536028747135266249775724709369995");
    IA_C.c0_02 = ia_from_decimal("0.02");
    IA_C.c0_1 = ia_from_decimal("0.1");
    IA_C.c0_9 = ia_from_decimal("0.9");
}
