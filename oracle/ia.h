/*
 * oracle/ia.h -- plain, slow, obviously-correct interval arithmetic for the
 * CPU oracle.  TEST INFRASTRUCTURE ONLY: nothing on the product path may
 * include, link or call this (see oracle/README.md).  It shares no code with
 * paper_2507_01770_b200/csrc.
 *
 * Paper reference (§2.1, lines 61-71): interval operations
 * Eq. (3) addition, Eq. (4) subtraction, Eq. (5) multiplication,
 * Eq. (6) division, with "optimal outward rounding" (line 71): the lower
 * endpoint is rounded towards -inf and the upper endpoint towards +inf.
 *
 * How rounding is done here: every endpoint operation of + - * / sqrt is
 * executed after fesetround(FE_DOWNWARD) or fesetround(FE_UPWARD) and the
 * mode is restored afterwards.  Transcendentals (exp, sin, cos) are called
 * from glibc libm in the default round-to-nearest mode and the result is then
 * widened outward by IA_LIBM_ULPS steps of nextafter(): glibc documents
 * <= 1 ulp error for double exp/sin/cos on x86_64; we add one more step for
 * the case where the true value lies in the neighbouring binade.
 */
#ifndef ORACLE_IA_H
#define ORACLE_IA_H

#define IA_LIBM_ULPS 2

typedef struct {
    double lo, hi;
} ia_t;

/* directed scalar operations (fesetround based) */
double ia_add_dn(double a, double b);
double ia_add_up(double a, double b);
double ia_sub_dn(double a, double b);
double ia_sub_up(double a, double b);
double ia_mul_dn(double a, double b);
double ia_mul_up(double a, double b);
double ia_div_dn(double a, double b);
double ia_div_up(double a, double b);
double ia_sqrt_dn(double a);
double ia_sqrt_up(double a);
double ia_widen_dn(double x, int k);
double ia_widen_up(double x, int k);
/* strtod of a decimal string under FE_DOWNWARD / FE_UPWARD */
ia_t ia_from_decimal(const char* s);

ia_t ia_pt(double x);                 /* degenerate interval [x, x] */
ia_t ia_make(double lo, double hi);
ia_t ia_neg(ia_t a);
ia_t ia_add(ia_t a, ia_t b);          /* Eq. (3) */
ia_t ia_sub(ia_t a, ia_t b);          /* Eq. (4) */
ia_t ia_mul(ia_t a, ia_t b);          /* Eq. (5) */
ia_t ia_div(ia_t a, ia_t b);          /* Eq. (6), only for 0 not in b */
ia_t ia_sqr(ia_t a);                  /* {x^2 : x in a} (single occurrence) */
ia_t ia_sqrt(ia_t a);                 /* {sqrt(x) : x in a, x >= 0} */
ia_t ia_exp(ia_t a);
ia_t ia_cos(ia_t a);                  /* {cos(t) : t in a} */
ia_t ia_sin(ia_t a);                  /* {sin(t) : t in a} */
ia_t ia_hull(ia_t a, ia_t b);
ia_t ia_intersect(ia_t a, ia_t b);
double ia_max(double a, double b);
double ia_min(double a, double b);

/* tight constants, filled by ia_init() from decimal strings */
typedef struct {
    ia_t pi, e, c0_02, c0_1, c0_9;
} ia_consts_t;
extern ia_consts_t IA_C;
void ia_init(void);

#endif
