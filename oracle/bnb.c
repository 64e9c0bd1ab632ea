/*
 * oracle/bnb.c -- the batched best-first interval branch-and-bound of
 * PAPER.md §3.1 (flowchart, lines 126-152) and §3.2 (partition and variable
 * cycling, lines 158-184), written step by step, slow and plain.
 * TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * One iteration (paper order, Fig. 2):
 *   1. select the regions with the smallest lower bound from the list L
 *      (line 130; batched: the B smallest, ties broken by list position,
 *      processed in list order, reading R1);
 *   2. partition each selected region into m^d subregions along the d
 *      variables given by its cycling index (lines 140, 176-184, Eq. 8-11);
 *   3. sample: evaluate f in interval arithmetic at the midpoint of every
 *      subregion and update GUB with the smallest upper bound (line 134;
 *      midpoint sampling is reading R2);
 *   4. rule out subregions whose lower bound exceeds GUB (line 140) or that
 *      fail the first-order test (lines 142-144);
 *   5. insert the remaining subregions into L (line 146), with cycling index
 *      advanced by d (line 184);
 *   6. regions of L whose lower bound exceeds GUB are removed (line 136);
 *   7. stop when every region of L is narrower than eps_x in all dimensions
 *      (line 148, 219) and GUB - GLB <= eps_f (line 150).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "ia.h"
#include "oracle.h"

int or_init(void) {
    ia_init();
    return 0;
}

/* Eq. (10)-(11) generalised to m subintervals: the k-th partition point of
 * [a, b] is a + ((b - a) / m) * k, with the end points kept exact. Round to
 * nearest, no fused multiply-add (build flag -ffp-contract=off). */
static double part_point(double a, double b, int m, int k) {
    if (k <= 0) return a;
    if (k >= m) return b;
    double w = (b - a) / (double)m;
    double t = w * (double)k;
    double p = a + t;
    return p < b ? p : b;
}

/* Child `code` of box (plo, phi): digit j of code in base m (least
 * significant first, Eq. 8-9) selects the subinterval of variable
 * (cyc + j) mod n.  code == OR_CODE_WHOLE returns the box itself. */
int or_child_box(int n, const double* plo, const double* phi, int cyc, int d, int m, long code,
                 double* clo, double* chi) {
    memcpy(clo, plo, sizeof(double) * (size_t)n);
    memcpy(chi, phi, sizeof(double) * (size_t)n);
    if (code == OR_CODE_WHOLE) return 0;
    for (int j = 0; j < d; ++j) {
        int dim = (cyc + j) % n;
        int p = (int)(code % m);
        code /= m;
        clo[dim] = part_point(plo[dim], phi[dim], m, p);
        chi[dim] = part_point(plo[dim], phi[dim], m, p + 1);
    }
    return 0;
}

static double midpoint(double a, double b) {
    double t = b - a;
    double mid = a + t * 0.5;
    if (mid < a) mid = a;
    if (mid > b) mid = b;
    return mid;
}

static double canon_lb(double lb) {
    if (isnan(lb)) return -INFINITY;
    if (lb == 0.0) return 0.0; /* -0.0 -> +0.0 */
    return lb;
}

/* Upper bound of f at the midpoint of the box (line 134, "interval
 * evaluation ... at each of these sample points"). */
static double box_ub(int fid, int n, const double* lo, const double* hi, ia_t* X) {
    for (int i = 0; i < n; ++i) X[i] = ia_pt(midpoint(lo[i], hi[i]));
    return or_F(fid, n, X).hi;
}

static double box_width(int n, const double* lo, const double* hi) {
    double w = 0.0;
    for (int i = 0; i < n; ++i) {
        double t = hi[i] - lo[i];
        if (t > w) w = t;
    }
    return w;
}

/* first-order test: "for any i in {1, 2, ..., n}, if
 * DLB_i > 0 and X_i.lo != l_i ... if DUB_i < 0 and X_i.hi != u_i".
 * mono == 2: every variable, as printed; mono == 1: the d split variables
 * only (reading R4; identical for separable objectives). */
static int monotone_pruned(int fid, int n, const ia_t* X, int cyc, int d, int mono,
                           const double* l, const double* u) {
    int nv = mono == 2 ? n : d;
    for (int j = 0; j < nv; ++j) {
        int i = (cyc + j) % n;
        ia_t D = or_dF(fid, n, X, i);
        if (D.lo > 0.0 && X[i].lo != l[i]) return 1;
        if (D.hi < 0.0 && X[i].hi != u[i]) return 1;
    }
    return 0;
}

static long ipow(int m, int d) {
    long r = 1;
    for (int j = 0; j < d; ++j) r *= m;
    return r;
}

int or_branch(int fid, int n, int nb, const double* plo, const double* phi, const int* pcyc,
              int d, int m, const double* l, const double* u, int mono, double gub_in,
              double* gub_out, long cap, int* out_parent, long* out_code, double* out_lb,
              double* out_w, long* out_count) {
    if (d < 1 || d > n || m < 2) return -1;
    long kids = ipow(m, d);
    double* clo = (double*)malloc(sizeof(double) * (size_t)n);
    double* chi = (double*)malloc(sizeof(double) * (size_t)n);
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)n);
    /* step 3: sample every subregion, update GUB */
    double gub = gub_in;
    for (int b = 0; b < nb; ++b)
        for (long c = 0; c < kids; ++c) {
            or_child_box(n, plo + (size_t)b * n, phi + (size_t)b * n, pcyc[b], d, m, c, clo, chi);
            double ub = box_ub(fid, n, clo, chi, X);
            if (ub < gub) gub = ub;
        }
    /* step 4-5: bound, rule out, keep survivors in (parent, code) order */
    long cnt = 0;
    int rc = 0;
    for (int b = 0; b < nb; ++b)
        for (long c = 0; c < kids; ++c) {
            or_child_box(n, plo + (size_t)b * n, phi + (size_t)b * n, pcyc[b], d, m, c, clo, chi);
            for (int i = 0; i < n; ++i) X[i] = ia_make(clo[i], chi[i]);
            double lb = canon_lb(or_F(fid, n, X).lo);
            if (!(lb <= gub)) continue;
            if (mono && monotone_pruned(fid, n, X, pcyc[b], d, mono, l, u)) continue;
            if (cnt < cap) {
                out_parent[cnt] = b;
                out_code[cnt] = c;
                out_lb[cnt] = lb;
                out_w[cnt] = box_width(n, clo, chi);
            } else {
                rc = 1; /* capacity exceeded: count is still exact */
            }
            ++cnt;
        }
    *gub_out = gub;
    *out_count = cnt;
    free(clo);
    free(chi);
    free(X);
    return rc;
}

/* ---------------------------------------------------------------------- */
typedef struct {
    double lb, w;
    int cyc;
    long pos; /* insertion sequence, only used for stable ordering */
    double* box; /* lo[0..n-1], hi[0..n-1] */
} rec_t;

/* Optional trace of or_solve for the selection / incumbent pins
 * (tests/test_oracle_bnb.py).  Per iteration, appended as doubles:
 *   pn, lb[0..pn-1] (the list L in list order after step 6),
 *   nb, idx[0..nb-1] (positions in that list of the selected regions, in the
 *   order they are processed), gub before and after steps 2-5.
 * Recording stops (silently) when the buffer is full. */
static double* g_trace = NULL;
static long g_trace_cap = 0, g_trace_len = 0;

void or_set_trace(double* buf, long cap) {
    g_trace = buf;
    g_trace_cap = cap;
    g_trace_len = 0;
}
long or_trace_len(void) { return g_trace_len; }

static void trace_put(double v) {
    if (g_trace && g_trace_len < g_trace_cap) g_trace[g_trace_len] = v;
    if (g_trace) ++g_trace_len;
}

static int rec_cmp(const void* a, const void* b) {
    const rec_t* x = *(const rec_t* const*)a;
    const rec_t* y = *(const rec_t* const*)b;
    if (x->lb < y->lb) return -1;
    if (x->lb > y->lb) return 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos ? 1 : 0);
}

int or_solve(int fid, int n, const double* l, const double* u, double eps_f, double eps_x, int d,
             int m, long bmax, int mono, long max_iter, long cap, int search, double* surv_lo,
             double* surv_hi, double* surv_lb, or_result_t* res) {
    if (d > n) d = n;
    if (d < 1 || m < 2 || bmax < 1) return -1;
    long kids = ipow(m, d);
    ia_t* X = (ia_t*)malloc(sizeof(ia_t) * (size_t)n);
    /* list L as an array of records, in insertion order */
    long pcap = 1024, pn = 0, seq = 0;
    rec_t* pool = (rec_t*)malloc(sizeof(rec_t) * (size_t)pcap);
    /* initialisation (line 128): one region covering the whole domain */
    pool[0].box = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    memcpy(pool[0].box, l, sizeof(double) * (size_t)n);
    memcpy(pool[0].box + n, u, sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) X[i] = ia_make(l[i], u[i]);
    pool[0].lb = canon_lb(or_F(fid, n, X).lo);
    pool[0].w = box_width(n, l, u);
    pool[0].cyc = 0;
    pool[0].pos = seq++;
    pn = 1;

    double gub = INFINITY;
    /* initial incumbent from the coordinate pattern search (reading R9,
     * oracle/search.c); search = its round limit, 0 = no search */
    if (search > 0) {
        double* xs0 = (double*)malloc(sizeof(double) * (size_t)n);
        double fs = INFINITY;
        or_search(fid, n, l, u, search, xs0, &fs, NULL);
        if (fs < gub) gub = fs;
        free(xs0);
    }
    long iter = 0, evals = 0;
    int status = 1;
    double* clo = (double*)malloc(sizeof(double) * (size_t)n);
    double* chi = (double*)malloc(sizeof(double) * (size_t)n);
    rec_t** order = NULL;
    for (;;) {
        /* step 6: drop regions of L whose lower bound exceeds GUB */
        long live = 0;
        for (long k = 0; k < pn; ++k) {
            if (pool[k].lb <= gub)
                pool[live++] = pool[k];
            else
                free(pool[k].box);
        }
        pn = live;
        if (pn == 0) {
            status = 2;
            break;
        }
        /* step 7: stopping criteria */
        double glb = INFINITY, maxw = 0.0;
        for (long k = 0; k < pn; ++k) {
            if (pool[k].lb < glb) glb = pool[k].lb;
            if (pool[k].w > maxw) maxw = pool[k].w;
        }
        if (maxw <= eps_x && ia_sub_up(gub, glb) <= eps_f) {
            status = 0;
            break;
        }
        if (iter >= max_iter) {
            status = 1;
            break;
        }
        /* step 1: select the B regions with smallest (lb, position) */
        order = (rec_t**)realloc(order, sizeof(rec_t*) * (size_t)pn);
        for (long k = 0; k < pn; ++k) order[k] = &pool[k];
        qsort(order, (size_t)pn, sizeof(rec_t*), rec_cmp);
        long nb = pn < bmax ? pn : bmax;
        double* plo = (double*)malloc(sizeof(double) * (size_t)nb * n);
        double* phi = (double*)malloc(sizeof(double) * (size_t)nb * n);
        int* pcyc = (int*)malloc(sizeof(int) * (size_t)nb);
        char* taken = (char*)calloc((size_t)pn, 1);
        for (long b = 0; b < nb; ++b) taken[order[b] - pool] = 1;
        /* the selected regions are processed in list order (R1) */
        if (g_trace) {
            trace_put((double)pn);
            for (long k = 0; k < pn; ++k) trace_put(pool[k].lb);
            trace_put((double)nb);
            for (long k = 0; k < pn; ++k)
                if (taken[k]) trace_put((double)k);
        }
        long bb = 0;
        for (long k = 0; k < pn; ++k) {
            if (!taken[k]) continue;
            memcpy(plo + bb * n, pool[k].box, sizeof(double) * (size_t)n);
            memcpy(phi + bb * n, pool[k].box + n, sizeof(double) * (size_t)n);
            pcyc[bb] = pool[k].cyc;
            ++bb;
        }
        /* remove the selected regions from L, keeping the order of the rest */
        long keep = 0;
        for (long k = 0; k < pn; ++k) {
            if (taken[k])
                free(pool[k].box);
            else
                pool[keep++] = pool[k];
        }
        pn = keep;
        free(taken);
        /* steps 2-5 */
        long ocap = nb * kids;
        int* opar = (int*)malloc(sizeof(int) * (size_t)ocap);
        long* ocode = (long*)malloc(sizeof(long) * (size_t)ocap);
        double* olb = (double*)malloc(sizeof(double) * (size_t)ocap);
        double* ow = (double*)malloc(sizeof(double) * (size_t)ocap);
        long ocnt = 0;
        if (g_trace) trace_put(gub);
        or_branch(fid, n, (int)nb, plo, phi, pcyc, d, m, l, u, mono, gub, &gub, ocap, opar, ocode,
                  olb, ow, &ocnt);
        if (g_trace) trace_put(gub);
        evals += nb * kids;
        if (pn + ocnt > pcap) {
            while (pn + ocnt > pcap) pcap *= 2;
            pool = (rec_t*)realloc(pool, sizeof(rec_t) * (size_t)pcap);
        }
        for (long k = 0; k < ocnt; ++k) {
            rec_t* r = &pool[pn++];
            int b = opar[k];
            r->box = (double*)malloc(sizeof(double) * 2 * (size_t)n);
            or_child_box(n, plo + (size_t)b * n, phi + (size_t)b * n, pcyc[b], d, m, ocode[k],
                         r->box, r->box + n);
            r->lb = olb[k];
            r->w = ow[k];
            r->cyc = (pcyc[b] + d) % n; /* line 184: cycling index advances by d */
            r->pos = seq++;
        }
        free(opar);
        free(ocode);
        free(olb);
        free(ow);
        free(plo);
        free(phi);
        free(pcyc);
        ++iter;
    }
    /* output (line 150): GLB, GUB and the regions of L */
    double glb = INFINITY;
    for (long k = 0; k < pn; ++k)
        if (pool[k].lb < glb) glb = pool[k].lb;
    res->glb = glb;
    res->gub = gub;
    res->iters = iter;
    res->evals = evals;
    res->n_surv = pn;
    res->status = status;
    for (long k = 0; k < pn; ++k) {
        if (k < cap) {
            memcpy(surv_lo + k * n, pool[k].box, sizeof(double) * (size_t)n);
            memcpy(surv_hi + k * n, pool[k].box + n, sizeof(double) * (size_t)n);
            surv_lb[k] = pool[k].lb;
        }
        free(pool[k].box);
    }
    free(pool);
    free(order);
    free(clo);
    free(chi);
    free(X);
    return 0;
}
