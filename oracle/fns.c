/*
 * oracle/fns.c -- natural interval extensions of the paper's objective
 * functions and of their first-order partial derivatives.
 * TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Each function is the formula of PAPER.md Appendix A written out term by
 * term, evaluated left to right over i = 1..n with the interval operations
 * of ia.c (natural interval extension, §2.1 lines 73-75).  The
 * derivatives are the analytic partial derivatives of those formulas, used by
 * the first-order (monotonicity) test of PAPER.md §3.1 lines 142-144.  The
 * exact algebraic form of every extension is fixed in DESIGN.md
 * ("Readings R3-R6"); the CUDA path evaluates the same forms.
 *
 * fid  function (PAPER.md line)
 *  0   x - x*x  worked example of §2.1 (line 75), summed over i
 *  1   Ackley      (A1) line 270
 *  2   Belegundu   (A3) line 278
 *  3   Breiman     (A5) line 286
 *  4   Fu          (A7) line 294
 *  5   Griewank    (A9) line 302
 *  6   Levy        (A11)-(A12) lines 310-312
 *  7   Rastrigin   (A14) line 320
 *  8   Salomon     (A16) line 328
 *  9   Styblinski  (A18) line 336
 * 10   Zabinsky    (A20) line 344
 */
#include <math.h>
#include <stdlib.h>

#include "ia.h"
#include "oracle.h"

static ia_t K(double c) { return ia_pt(c); }

static ia_t two_pi(void) { return ia_make(2.0 * IA_C.pi.lo, 2.0 * IA_C.pi.hi); }

/* kappa_i = 1/sqrt(i) (Griewank, i is 1-based) */
static ia_t griewank_kappa(int i1) {
    ia_t s = ia_make(ia_sqrt_dn((double)i1), ia_sqrt_up((double)i1));
    return ia_div(K(1.0), s);
}

/* Levy (A12): y_i = 1 + 0.25 (x_i - 1) */
static ia_t levy_y(ia_t x) { return ia_add(K(1.0), ia_mul(K(0.25), ia_sub(x, K(1.0)))); }
/* u_i = (y_i - 1)^2 */
static ia_t levy_u(ia_t y) { return ia_sqr(ia_sub(y, K(1.0))); }
/* v_i = 1 + 10 sin^2(pi y_i) */
static ia_t levy_v(ia_t y) {
    return ia_add(K(1.0), ia_mul(K(10.0), ia_sqr(ia_sin(ia_mul(IA_C.pi, y)))));
}

/* ---------------------------------------------------------------------- */
/* f over a box X[0..n-1]                                                  */
ia_t or_F(int fid, int n, const ia_t* X) {
    ia_t nn = K((double)n);
    switch (fid) {
        case 0: { /* sum_i (x_i - x_i * x_i) */
            ia_t s = K(0.0);
            for (int i = 0; i < n; ++i) s = ia_add(s, ia_sub(X[i], ia_mul(X[i], X[i])));
            return s;
        }
        case 1: { /* (A1) -20 exp(-0.02 sqrt(1/n sum x^2)) - exp(1/n sum cos 2 pi x) + 20 + e */
            ia_t s1 = K(0.0), s2 = K(0.0);
            for (int i = 0; i < n; ++i) {
                s1 = ia_add(s1, ia_sqr(X[i]));
                s2 = ia_add(s2, ia_cos(ia_mul(two_pi(), X[i])));
            }
            ia_t r = ia_sqrt(ia_div(s1, nn));
            ia_t t1 = ia_mul(K(-20.0), ia_exp(ia_mul(ia_neg(IA_C.c0_02), r)));
            ia_t t2 = ia_neg(ia_exp(ia_div(s2, nn)));
            return ia_add(ia_add(ia_add(t1, t2), K(20.0)), IA_C.e);
        }
        case 2: { /* (A3) 0.1 sum (x-5)^2 - cos(5 sqrt(sum (x-5)^2)) */
            ia_t s = K(0.0);
            for (int i = 0; i < n; ++i) s = ia_add(s, ia_sqr(ia_sub(X[i], K(5.0))));
            ia_t r = ia_sqrt(s);
            return ia_sub(ia_mul(IA_C.c0_1, s), ia_cos(ia_mul(K(5.0), r)));
        }
        case 3: { /* (A5) -0.1 sum cos(5 pi x) + sum x^2 */
            ia_t five_pi = ia_mul(K(5.0), IA_C.pi);
            ia_t s1 = K(0.0), s2 = K(0.0);
            for (int i = 0; i < n; ++i) {
                s1 = ia_add(s1, ia_cos(ia_mul(five_pi, X[i])));
                s2 = ia_add(s2, ia_sqr(X[i]));
            }
            return ia_add(ia_mul(ia_neg(IA_C.c0_1), s1), s2);
        }
        case 4: { /* (A7) 1 + sum [8 sin^2(7 g^2) + 6 sin^2(14 g^2) + g^2], g = x - 0.9 */
            ia_t s = K(0.0);
            for (int i = 0; i < n; ++i) {
                ia_t g = ia_sub(X[i], IA_C.c0_9);
                ia_t q = ia_sqr(g);
                ia_t a = ia_sqr(ia_sin(ia_mul(K(7.0), q)));
                ia_t b = ia_sqr(ia_sin(ia_mul(K(14.0), q)));
                s = ia_add(s, ia_add(ia_add(ia_mul(K(8.0), a), ia_mul(K(6.0), b)), q));
            }
            return ia_add(K(1.0), s);
        }
        case 5: { /* (A9) 1 + sum x^2 / 4000 - prod cos(x_i / sqrt(i)) */
            ia_t s = K(0.0), p = K(1.0);
            for (int i = 0; i < n; ++i) {
                s = ia_add(s, ia_sqr(X[i]));
                p = ia_mul(p, ia_cos(ia_mul(griewank_kappa(i + 1), X[i])));
            }
            return ia_sub(ia_add(K(1.0), ia_div(s, K(4000.0))), p);
        }
        case 6: { /* (A11) pi/n {10 sin^2(pi y1) + sum_{i<n} u_i v_{i+1} + u_n} */
            ia_t y0 = levy_y(X[0]);
            ia_t acc = ia_mul(K(10.0), ia_sqr(ia_sin(ia_mul(IA_C.pi, y0))));
            for (int i = 0; i + 1 < n; ++i)
                acc = ia_add(acc, ia_mul(levy_u(levy_y(X[i])), levy_v(levy_y(X[i + 1]))));
            acc = ia_add(acc, levy_u(levy_y(X[n - 1])));
            return ia_mul(ia_div(IA_C.pi, nn), acc);
        }
        case 7: { /* (A14) 10 n + sum [x^2 - 10 cos(2 pi x)] */
            ia_t s = K(0.0);
            for (int i = 0; i < n; ++i)
                s = ia_add(s, ia_sub(ia_sqr(X[i]),
                                     ia_mul(K(10.0), ia_cos(ia_mul(two_pi(), X[i])))));
            return ia_add(ia_mul(K(10.0), nn), s);
        }
        case 8: { /* (A16) 1 - cos(2 pi sqrt(sum x^2)) + 0.1 sqrt(sum x^2) */
            ia_t s = K(0.0);
            for (int i = 0; i < n; ++i) s = ia_add(s, ia_sqr(X[i]));
            ia_t r = ia_sqrt(s);
            return ia_add(ia_sub(K(1.0), ia_cos(ia_mul(two_pi(), r))), ia_mul(IA_C.c0_1, r));
        }
        case 9: { /* (A18) 1/(2n) sum x^2 - 4n prod cos(x) */
            ia_t s = K(0.0), p = K(1.0);
            for (int i = 0; i < n; ++i) {
                s = ia_add(s, ia_sqr(X[i]));
                p = ia_mul(p, ia_cos(X[i]));
            }
            return ia_sub(ia_div(s, ia_mul(K(2.0), nn)), ia_mul(ia_mul(K(4.0), nn), p));
        }
        case 10: { /* (A20) -2.5 prod sin(x - pi/6) - prod sin(5 (x - pi/6)) */
            ia_t pi6 = ia_div(IA_C.pi, K(6.0));
            ia_t p1 = K(1.0), p2 = K(1.0);
            for (int i = 0; i < n; ++i) {
                ia_t g = ia_sub(X[i], pi6);
                p1 = ia_mul(p1, ia_sin(g));
                p2 = ia_mul(p2, ia_sin(ia_mul(K(5.0), g)));
            }
            return ia_sub(ia_mul(K(-2.5), p1), p2);
        }
    }
    return ia_make(-INFINITY, INFINITY);
}

/* x_i / r over the box, intersected with the a-priori bound |x_i / r| <= s
 * (Ackley: s = sqrt(n); Salomon: s = 1).  When r can be 0 only the sign of
 * x_i is known.  DESIGN.md reading R5. */
static ia_t ratio_q(ia_t x, ia_t r, double s) {
    if (r.lo > 0.0) {
        ia_t q = ia_div(x, r);
        return ia_make(ia_max(q.lo, -s), ia_min(q.hi, s));
    }
    return ia_make(x.lo >= 0.0 ? 0.0 : -s, x.hi <= 0.0 ? 0.0 : s);
}

/* ---------------------------------------------------------------------- */
/* d f / d x_i over a box X (i is 0-based)                                 */
ia_t or_dF(int fid, int n, const ia_t* X, int i) {
    ia_t nn = K((double)n);
    ia_t x = X[i];
    switch (fid) {
        case 0: /* 1 - 2 x */
            return ia_sub(K(1.0), ia_mul(K(2.0), x));
        case 1: { /* (0.4/n) e^{-0.02 r} x_i/r + (2 pi/n) e^{S2/n} sin(2 pi x_i) */
            ia_t s1 = K(0.0), s2 = K(0.0);
            for (int j = 0; j < n; ++j) {
                s1 = ia_add(s1, ia_sqr(X[j]));
                s2 = ia_add(s2, ia_cos(ia_mul(two_pi(), X[j])));
            }
            ia_t r = ia_sqrt(ia_div(s1, nn));
            ia_t c04 = ia_mul(K(4.0), IA_C.c0_1);
            ia_t a = ia_mul(ia_div(c04, nn), ia_exp(ia_mul(ia_neg(IA_C.c0_02), r)));
            ia_t b = ia_mul(ia_div(two_pi(), nn), ia_exp(ia_div(s2, nn)));
            ia_t q = ratio_q(x, r, ia_sqrt_up((double)n));
            return ia_add(ia_mul(a, q), ia_mul(b, ia_sin(ia_mul(two_pi(), x))));
        }
        case 2: { /* (x_i - 5) (0.2 + 5 H), H = sin(5r)/r in [-5, 5] */
            ia_t s = K(0.0);
            for (int j = 0; j < n; ++j) s = ia_add(s, ia_sqr(ia_sub(X[j], K(5.0))));
            ia_t r = ia_sqrt(s);
            ia_t h = ia_make(-5.0, 5.0);
            if (r.lo > 0.0) {
                ia_t q = ia_div(ia_sin(ia_mul(K(5.0), r)), r);
                h = ia_make(ia_max(q.lo, -5.0), ia_min(q.hi, 5.0));
            }
            ia_t c02 = ia_mul(K(2.0), IA_C.c0_1);
            return ia_mul(ia_sub(x, K(5.0)), ia_add(c02, ia_mul(K(5.0), h)));
        }
        case 3: { /* 0.5 pi sin(5 pi x) + 2 x */
            ia_t half_pi = ia_mul(K(0.5), IA_C.pi);
            ia_t five_pi = ia_mul(K(5.0), IA_C.pi);
            return ia_add(ia_mul(half_pi, ia_sin(ia_mul(five_pi, x))), ia_mul(K(2.0), x));
        }
        case 4: { /* g (112 sin(14 q) + 168 sin(28 q) + 2), g = x - 0.9, q = g^2 */
            ia_t g = ia_sub(x, IA_C.c0_9);
            ia_t q = ia_sqr(g);
            ia_t t = ia_add(ia_add(ia_mul(K(112.0), ia_sin(ia_mul(K(14.0), q))),
                                   ia_mul(K(168.0), ia_sin(ia_mul(K(28.0), q)))),
                            K(2.0));
            return ia_mul(g, t);
        }
        case 5: { /* x_i/2000 + k_i sin(k_i x_i) prod_{j != i} cos(k_j x_j) */
            ia_t p = K(1.0);
            for (int j = 0; j < n; ++j)
                if (j != i) p = ia_mul(p, ia_cos(ia_mul(griewank_kappa(j + 1), X[j])));
            ia_t k = griewank_kappa(i + 1);
            return ia_add(ia_div(x, K(2000.0)), ia_mul(ia_mul(k, ia_sin(ia_mul(k, x))), p));
        }
        case 6: { /* pi/n ([i=0] s_0 + [i<n-1] (y_i-1)/2 v_{i+1} + [i>0] u_{i-1} s_i
                     + [i=n-1] (y_i-1)/2),  s_i = 2.5 pi sin(2 pi y_i) */
            ia_t c25pi = ia_mul(K(2.5), IA_C.pi);
            ia_t y = levy_y(x);
            ia_t s_i = ia_mul(c25pi, ia_sin(ia_mul(two_pi(), y)));
            ia_t du = ia_mul(K(0.5), ia_sub(y, K(1.0)));
            ia_t acc = K(0.0);
            if (i == 0) acc = ia_add(acc, s_i);
            if (i < n - 1) acc = ia_add(acc, ia_mul(du, levy_v(levy_y(X[i + 1]))));
            if (i > 0) acc = ia_add(acc, ia_mul(levy_u(levy_y(X[i - 1])), s_i));
            if (i == n - 1) acc = ia_add(acc, du);
            return ia_mul(ia_div(IA_C.pi, nn), acc);
        }
        case 7: { /* 2 x + 20 pi sin(2 pi x) */
            ia_t c20pi = ia_mul(K(20.0), IA_C.pi);
            return ia_add(ia_mul(K(2.0), x), ia_mul(c20pi, ia_sin(ia_mul(two_pi(), x))));
        }
        case 8: { /* (2 pi sin(2 pi r) + 0.1) x_i / r, |x_i/r| <= 1 */
            ia_t s = K(0.0);
            for (int j = 0; j < n; ++j) s = ia_add(s, ia_sqr(X[j]));
            ia_t r = ia_sqrt(s);
            ia_t t = ia_add(ia_mul(two_pi(), ia_sin(ia_mul(two_pi(), r))), IA_C.c0_1);
            return ia_mul(t, ratio_q(x, r, 1.0));
        }
        case 9: { /* x_i / n + 4 n sin(x_i) prod_{j != i} cos(x_j) */
            ia_t p = K(1.0);
            for (int j = 0; j < n; ++j)
                if (j != i) p = ia_mul(p, ia_cos(X[j]));
            return ia_add(ia_div(x, nn), ia_mul(ia_mul(ia_mul(K(4.0), nn), ia_sin(x)), p));
        }
        case 10: { /* -2.5 cos(g_i) prod_{j!=i} sin(g_j) - 5 cos(5 g_i) prod_{j!=i} sin(5 g_j) */
            ia_t pi6 = ia_div(IA_C.pi, K(6.0));
            ia_t p1 = K(1.0), p2 = K(1.0);
            for (int j = 0; j < n; ++j) {
                if (j == i) continue;
                ia_t g = ia_sub(X[j], pi6);
                p1 = ia_mul(p1, ia_sin(g));
                p2 = ia_mul(p2, ia_sin(ia_mul(K(5.0), g)));
            }
            ia_t g = ia_sub(x, pi6);
            ia_t a = ia_mul(ia_mul(K(-2.5), ia_cos(g)), p1);
            ia_t b = ia_mul(ia_mul(K(-5.0), ia_cos(ia_mul(K(5.0), g))), p2);
            return ia_add(a, b);
        }
    }
    return ia_make(-INFINITY, INFINITY);
}

/* ---------------------------------------------------------------------- */
/* C entry points used by tests through ctypes                             */
static ia_t* to_box(int n, const double* lo, const double* hi) {
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) X[i] = ia_make(lo[i], hi[i]);
    return X;
}

int or_eval_box(int fid, int n, const double* lo, const double* hi, double* out) {
    if (fid < 0 || fid >= OR_NUM_FUNCS || n < 1) return -1;
    ia_t* X = to_box(n, lo, hi);
    ia_t r = or_F(fid, n, X);
    free(X);
    out[0] = r.lo;
    out[1] = r.hi;
    return 0;
}

int or_eval_point(int fid, int n, const double* x, double* out) {
    return or_eval_box(fid, n, x, x, out);
}

int or_grad_box(int fid, int n, const double* lo, const double* hi, int i, double* out) {
    if (fid < 0 || fid >= OR_NUM_FUNCS || n < 1 || i < 0 || i >= n) return -1;
    ia_t* X = to_box(n, lo, hi);
    ia_t r = or_dF(fid, n, X, i);
    free(X);
    out[0] = r.lo;
    out[1] = r.hi;
    return 0;
}
