/*
 * oracle/search.c -- the coordinate pattern search that supplies the initial
 * incumbent GUB (reading R9), written plainly: every value it
 * compares is the upper end of the natural interval extension of f at a
 * point (or_F on degenerate intervals), so every value is a rigorous upper
 * bound of f at a feasible point, which is all PAPER.md §3.1
 * ask of a sample ("any sampling strategy is acceptable"; GUB = the smallest
 * upper bound over the sampled points).
 * TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Algorithm (R9).  First a line search along the diagonal of [l, u] (the
 * paper's own sample points lie on diagonals, line 219):
 *   x(t) = clamp(l + t (u - l)), t_k = k / 2^14 (k = 0..2^14, t = 1/2 is the
 *   midpoint), t* = the t_k with the smallest upper(F(x(t_k))) (first k on
 *   ties); then at most 16 rounds of t* +- 2^-j (j = 11..58, minus before
 *   plus), moving to the best candidate while it is strictly better.
 * Then, from x = x(t*):
 *   repeat for at most rmax rounds:
 *     fcur = upper(F(x))
 *     proposal: for every variable i, over the candidate values c = 0..127
 *       (c < 32: grid point l_i + ((u_i - l_i) / 31) * c, c = 31 -> u_i;
 *        c >= 32: x_i + s * (u_i - l_i) * 2^-j, j = (c - 32) / 2 + 1,
 *        s = -1 for even c, +1 for odd c; skipped when outside [l_i, u_i]),
 *       v_c = upper(F(x with x_i replaced by the candidate)); the smallest
 *       v_c (first c on ties) is the proposal xs_i with value fb_i if
 *       v_c < fcur, else xs_i = x_i, fb_i = fcur;
 *     moves: y_a = clamp(x + 2^-a (xs - x)) for a = 0..7 with value
 *       upper(F(y_a)), and the single move of the variable with the smallest
 *       fb_i (first i on ties) with value fb_i;
 *     the move with the smallest value (order: a = 0..7, then the single
 *     move; first on ties) is taken if its value < fcur, else stop.
 *   The result is the final x and fcur = upper(F(x)) there.
 * Round to nearest, no FMA (-ffp-contract=off).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "ia.h"
#include "oracle.h"

#define SR_GRID 32
#define SR_SCALES 48
#define SR_CANDS (SR_GRID + 2 * SR_SCALES)
#define SR_ALPHAS 8
#define SR_DIAG_LOG2 14
#define SR_DIAG_ROUNDS 16
#define SR_DIAG_J0 11
#define SR_DIAG_J1 58

/* x(t) = clamp(l + t (u - l)) */
static void diag_point(int n, const double* l, const double* u, double t, double* x) {
    for (int i = 0; i < n; ++i) {
        double v = l[i] + t * (u[i] - l[i]);
        x[i] = v < l[i] ? l[i] : (v > u[i] ? u[i] : v);
    }
}

static double upper_at(int fid, int n, const double* x, ia_t* X) {
    for (int i = 0; i < n; ++i) X[i] = ia_pt(x[i]);
    return or_F(fid, n, X).hi;
}

/* candidate c of variable i (R9); returns 0 when it lies outside [l_i, u_i] */
int or_search_candidate(double xi, double li, double ui, int c, double* p) {
    double span = ui - li;
    if (c < SR_GRID) {
        if (c == SR_GRID - 1) {
            *p = ui;
            return 1;
        }
        double w = span / (double)(SR_GRID - 1);
        double q = li + w * (double)c;
        *p = q < ui ? q : ui;
        return 1;
    }
    int j = (c - SR_GRID) / 2 + 1;
    double h = ldexp(span, -j);
    double q = (c & 1) ? xi + h : xi - h;
    if (q < li || q > ui) return 0;
    *p = q;
    return 1;
}

int or_search_propose(int fid, int n, const double* x, const double* l, const double* u,
                      double fcur, double* xs, double* fb) {
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)n);
    memcpy(y, x, sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        double best = INFINITY, bp = x[i];
        for (int c = 0; c < SR_CANDS; ++c) {
            double p;
            if (!or_search_candidate(x[i], l[i], u[i], c, &p)) continue;
            y[i] = p;
            double v = upper_at(fid, n, y, X);
            if (v < best) {
                best = v;
                bp = p;
            }
        }
        y[i] = x[i];
        if (best < fcur) {
            xs[i] = bp;
            fb[i] = best;
        } else {
            xs[i] = x[i];
            fb[i] = fcur;
        }
    }
    free(X);
    free(y);
    return 0;
}

int or_search_diag(int fid, int n, const double* l, const double* u, double* t_out, double* f_out) {
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)n);
    const long nd = (1L << SR_DIAG_LOG2) + 1;
    double ts = 0.0, fs = INFINITY;
    for (long k = 0; k < nd; ++k) {
        double t = ldexp((double)k, -SR_DIAG_LOG2);
        diag_point(n, l, u, t, x);
        double v = upper_at(fid, n, x, X);
        if (v < fs) {
            fs = v;
            ts = t;
        }
    }
    for (int r = 0; r < SR_DIAG_ROUNDS; ++r) {
        double bv = fs, bt = ts;
        for (int j = SR_DIAG_J0; j <= SR_DIAG_J1; ++j)
            for (int s = -1; s <= 1; s += 2) {
                double t = ts + (double)s * ldexp(1.0, -j);
                if (t < 0.0 || t > 1.0) continue;
                diag_point(n, l, u, t, x);
                double v = upper_at(fid, n, x, X);
                if (v < bv) {
                    bv = v;
                    bt = t;
                }
            }
        if (!(bv < fs)) break;
        fs = bv;
        ts = bt;
    }
    *t_out = ts;
    *f_out = fs;
    free(X);
    free(x);
    return 0;
}

int or_search(int fid, int n, const double* l, const double* u, int rmax, double* x_out,
              double* f_out, int* rounds_out) {
    double* x = x_out;
    double* xs = (double*)malloc(sizeof(double) * (size_t)n);
    double* fb = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    double* ybest = (double*)malloc(sizeof(double) * (size_t)n);
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)n);
    double t0, f0;
    or_search_diag(fid, n, l, u, &t0, &f0);
    diag_point(n, l, u, t0, x);
    double fcur = upper_at(fid, n, x, X);
    int r = 0;
    while (r < rmax) {
        or_search_propose(fid, n, x, l, u, fcur, xs, fb);
        double vbest = INFINITY;
        int have = 0;
        for (int a = 0; a < SR_ALPHAS; ++a) {
            double al = ldexp(1.0, -a);
            for (int i = 0; i < n; ++i) {
                double v = x[i] + al * (xs[i] - x[i]);
                y[i] = v < l[i] ? l[i] : (v > u[i] ? u[i] : v);
            }
            double v = upper_at(fid, n, y, X);
            if (v < vbest) {
                vbest = v;
                memcpy(ybest, y, sizeof(double) * (size_t)n);
                have = 1;
            }
        }
        int istar = 0;
        for (int i = 1; i < n; ++i)
            if (fb[i] < fb[istar]) istar = i;
        if (fb[istar] < vbest) {
            vbest = fb[istar];
            memcpy(ybest, x, sizeof(double) * (size_t)n);
            ybest[istar] = xs[istar];
            have = 1;
        }
        if (!have || !(vbest < fcur)) break;
        memcpy(x, ybest, sizeof(double) * (size_t)n);
        ++r;
        fcur = upper_at(fid, n, x, X);
    }
    *f_out = fcur;
    if (rounds_out) *rounds_out = r;
    free(X);
    free(ybest);
    free(y);
    free(fb);
    free(xs);
    return 0;
}
