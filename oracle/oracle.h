/*
 * oracle/oracle.h -- C entry points of the CPU oracle.
 * TEST INFRASTRUCTURE ONLY: callable from tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs, never from the
 * product path (paper_2507_01770_b200/).
 */
#ifndef ORACLE_H
#define ORACLE_H

#include "ia.h"

#define OR_NUM_FUNCS 11
#define OR_CODE_WHOLE (-1L)

ia_t or_F(int fid, int n, const ia_t* X);
ia_t or_dF(int fid, int n, const ia_t* X, int i);

int or_init(void);
int or_eval_box(int fid, int n, const double* lo, const double* hi, double* out);
int or_eval_point(int fid, int n, const double* x, double* out);
int or_grad_box(int fid, int n, const double* lo, const double* hi, int i, double* out);

int or_child_box(int n, const double* plo, const double* phi, int cyc, int d, int m, long code,
                 double* clo, double* chi);

int or_branch(int fid, int n, int nb, const double* plo, const double* phi, const int* pcyc,
              int d, int m, const double* l, const double* u, int mono, double gub_in,
              double* gub_out, long cap, int* out_parent, long* out_code, double* out_lb,
              double* out_w, long* out_count);

typedef struct {
    double glb, gub;
    long iters, evals, n_surv;
    int status; /* 0 converged, 1 max_iter, 2 pool empty, <0 error */
} or_result_t;

int or_search_candidate(double xi, double li, double ui, int c, double* p);
int or_search_propose(int fid, int n, const double* x, const double* l, const double* u,
                      double fcur, double* xs, double* fb);
int or_search_diag(int fid, int n, const double* l, const double* u, double* t_out, double* f_out);
int or_search(int fid, int n, const double* l, const double* u, int rmax, double* x_out,
              double* f_out, int* rounds_out);

void or_set_trace(double* buf, long cap);
long or_trace_len(void);

int or_solve(int fid, int n, const double* l, const double* u, double eps_f, double eps_x, int d,
             int m, long bmax, int mono, long max_iter, long cap, int search, double* surv_lo,
             double* surv_hi, double* surv_lb, or_result_t* res);

#endif
