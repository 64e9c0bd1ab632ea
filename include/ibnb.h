/*
 * ibnb.h -- C ABI of the B200 interval branch-and-bound hot path
 * (libibnb.so, built from paper_2507_01770_b200/csrc).
 *
 * Problem (§1 Eq. (1)-(2), lines 25-31): minimise f(x) subject to
 * l <= x <= u, f one of the objectives of Appendix A selected by `fid`:
 *   0 example x - x^2 (§2.1 line 75, summed over variables)
 *   1 Ackley (A1)   2 Belegundu (A3)   3 Breiman (A5)   4 Fu (A7)
 *   5 Griewank (A9) 6 Levy (A11)       7 Rastrigin (A14) 8 Salomon (A16)
 *   9 Styblinski (A18)                 10 Zabinsky (A20)
 * The method returns an enclosure [f_lo, f_hi] of the global minimum (GLB,
 * GUB of §3.1 "Output result", lines 150-152) and the regions of the list L
 * that may contain the minimiser.
 *
 * Conventions for every call:
 *  - plain pointers and sizes only; "device" pointers are CUDA device memory
 *    of the current device, "host" pointers are host memory;
 *  - all floating point is IEEE binary64;
 *  - boxes are stored box-major: box k, variable i at lo[k*ld + i], with
 *    separate lo and hi planes (structure of arrays over the two endpoints);
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *    device-pointer calls are asynchronous on that stream unless stated;
 *  - workspace memory is owned by the caller (e.g. a torch uint8 tensor) and
 *    must stay alive and unused by others until the call's work completes;
 *  - return value: 0 on success, a negative IB_E* code on invalid arguments
 *    or capacity overflow, a positive cudaError_t value on a CUDA failure.
 *    ib_last_error() returns a thread-local message for the last failure.
 * There is no CPU fallback: every compute step runs in CUDA kernels.
 */
#ifndef IBNB_H
#define IBNB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IB_OK 0
#define IB_EINVAL (-1)       /* bad fid / n / d / m / pointer / size */
#define IB_ENOSPACE (-2)     /* workspace, list L or archive capacity exceeded */
#define IB_EEMPTY (-3)       /* list L became empty (cannot happen for a correct f) */
#define IB_ENODEV (-4)       /* no CUDA device */

#define IB_STATUS_CONVERGED 0 /* both tolerances met */
#define IB_STATUS_MAX_ITER 1  /* iteration limit reached first */
#define IB_STATUS_EMPTY 2     /* (multi-GPU) this rank's list L was emptied by the shared GUB */
#define IB_NPROF 8

/* Version string of the library. */
const char* ib_version(void);
/* Message of the last failure in this thread ("" if none). */
const char* ib_last_error(void);
/* Number of objectives (fid range is 0 .. ib_num_functions()-1). */
int ib_num_functions(void);

/* Options of the branch-and-bound (§3.1-3.2).  Zero fields take the
 * defaults given in brackets. */
typedef struct {
    int d;            /* variables partitioned per iteration, the variable-cycling
                         chunk (§3.2) [min(n, 16)], 1 <= d <= 20
                         (bench.py: d = 18 at n = 10,000, m^d close to 148 SMs x
                         2048 threads, the occupancy rule of §3.2) */
    int m;            /* pieces per partitioned variable, uniform partition
                         Eq. (10)-(11) generalised [2 = bisection], 2 <= m <= 8,
                         m^d <= 2^24, d*m <= 64 */
    int mono;         /* first-order (monotonicity) test of §3.1:
                         1 on [default], -1 off */
    int profile;      /* 1: time every kernel launch with CUDA events on the
                         solve stream (ib_result.t_ms / launches / units) */
    int search;       /* rounds of the coordinate pattern search that supplies
                         the initial incumbent GUB before the first iteration
                         (sampling, §3.1; reading R9;
                         see ib_search) [32]; -1 = no search */
    int reserved;     /* must be 0 */
    int64_t bmax;     /* regions selected per iteration (smallest lower bounds,
                         line 130, batched) [max(1, min(2^22 / m^d, 2^17 / n))] */
    int64_t max_iter; /* iteration limit [1,000,000] */
    int64_t pool_cap; /* capacity of the list L in records [derived from workspace] */
    int64_t arch_cap; /* capacity of the archive of selected regions [derived] */
    void* gub_shared; /* multi-GPU (north_star: the incumbent shared "each
                         iteration" over NVLink): device address of ONE 64-bit
                         word, the same word on every rank (one rank's memory,
                         mapped into the others with ib_ipc_open), holding the
                         incumbent GUB as an ordered integer (initialise to
                         ~0).  Every iteration of the deep-dive kernel
                         atomically lowers it to the rank's GUB and takes the
                         minimum back (one NVLink atomic, overlapped with the
                         children); the batch paths do the same before every
                         chunk of <= 64 iterations; NULL [default]: not
                         shared.  The value is
                         only ever a rigorous upper bound of f at a feasible
                         point of the whole domain, so sharing never affects
                         rigour, only how early regions are ruled out. */
} ib_options;

typedef struct {
    double f_lo;      /* GLB: rigorous lower bound of the global minimum */
    double f_hi;      /* GUB: rigorous upper bound of the global minimum */
    int64_t iters;    /* iterations executed */
    int64_t evals;    /* child boxes whose lower bound was evaluated (B * m^d per
                         iteration); the midpoint upper bound is only evaluated
                         for children with lower bound <= the incumbent at the
                         iteration start (any other cannot lower GUB) */
    int64_t n_surv;   /* regions left in L (all of them enclose no better point) */
    int64_t peak_pool;/* largest size of L seen */
    double max_width; /* widest remaining region (max over variables) */
    int status;       /* IB_STATUS_* */
    int n_kernels;    /* CUDA kernels this call launched */
    /* per kernel, filled when opt.profile = 1 (else zero):
     * 0 k_prep (units: parents), 1 k_child_eval (children), 2 k_cand
     * (children), 3 k_list: statistics + radix select + selection on the
     * hot index, refills (units: algorithmic bytes read), 4 k_mono
     * (candidates), 5 k_emit
     * (candidates), 6 k_fused: whole iterations in one persistent kernel
     * (units: iterations), 7 k_chain: the deep-dive chain, one region per
     * iteration, one grid barrier per iteration (units: iterations) */
    double t_ms[IB_NPROF];
    int64_t launches[IB_NPROF];
    int64_t units[IB_NPROF];
    int64_t radix_records; /* records scanned by radix passes 2..8 */
    double f_search;       /* GUB supplied by the initial search (+inf: none) */
    int64_t search_rounds; /* accepted moves of that search */
    int64_t rebalanced;    /* ib_solve_dev_mg: regions received (> 0) or sent (< 0) */
    int64_t transfers;     /* ib_solve_dev_mg: rebalancing transfers this rank took part in */
} ib_result;

/* Multi-GPU incumbent exchange (GUB is the best sample
 * found anywhere).  When fn != NULL, after every chunk of iterations (the
 * runtime's unit of host synchronisation: 1, 2, 4, ... doubling up to 64
 * iterations) the runtime
 * writes xchg[0] = local GUB and xchg[1] = (local search finished ? 0 : -1)
 * to the DEVICE buffer xchg and calls fn(user) on the host thread; fn must
 * replace xchg by its element-wise minimum over all ranks, enqueued on the
 * caller's `stream` (e.g. an NCCL all-reduce(MIN)); the runtime orders it
 * between its own kernels with events.  The run ends when every rank has
 * finished; a rank whose list L empties (all its regions ruled out by the
 * shared GUB) is finished, not failed.  A stale GUB between exchanges only
 * delays pruning (any upper bound of the minimum is valid). */
typedef void (*ib_exchange_fn)(void* user);

/* Bytes of caller-owned device workspace needed by ib_solve*() for a problem
 * of dimension n with options *opt (NULL = defaults) and a list L of at most
 * pool_cap records (0 = derive pool_cap from the other options). */
size_t ib_solve_workspace_size(int fid, int n, const ib_options* opt, int64_t pool_cap);

/* Full solve, HOST buffers (the end-to-end call).
 *   l, u        host, n doubles each, l[i] < u[i] finite (Eq. (2))
 *   eps_f       stop when GUB - GLB <= eps_f (enclosure width, line 150)
 *   eps_x       ... and every region of L has width <= eps_x in all
 *               variables (region size tolerance, lines 148 and 219)
 *   ws, ws_bytes  device workspace (>= ib_solve_workspace_size)
 *   res         host, receives the enclosure and counters
 *   surv_lo/hi  host, optional (may be NULL): the first surv_cap surviving
 *               regions, box-major with ld = n; surv_lb their lower bounds
 * Synchronous: returns after the results are in host memory. */
int ib_solve(int fid, int n, const double* l, const double* u, double eps_f, double eps_x,
             const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
             double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream);

/* Same as ib_solve with l, u in DEVICE memory and optional DEVICE outputs
 * surv_lo/surv_hi/surv_lb.  res is host.  Synchronous. */
int ib_solve_dev(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                 const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                 double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream);

/* ib_solve_dev with a per-iteration incumbent exchange (see ib_exchange_fn);
 * xchg: device, 2 doubles. */
int ib_solve_dev_ex(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                    const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                    double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream, ib_exchange_fn fn,
                    void* user, double* xchg);

/* Multi-GPU box rebalancing (north_star: "periodic NVLink box rebalancing
 * when survivor counts skew").  tfn(user, src, dst, buf, bytes) is called on
 * EVERY rank with the same arguments; the caller must copy `bytes` bytes from
 * rank src's buf to rank dst's buf (e.g. NCCL send / recv on the caller's
 * stream, ordered with the solve by events); other ranks do nothing. */
typedef void (*ib_transfer_fn)(void* user, int src, int dst, void* buf, size_t bytes);

/* ib_solve_dev_ex with box rebalancing.  xchg: device, 4 doubles (GUB,
 * finished flag, -(live * 1024 + rank), live * 1024 + rank -- fn reduces all
 * four with MIN).  fn is called twice per chunk: for the incumbent, then for
 * the list sizes under the shared incumbent.  After that, when the largest list of live
 * regions (rank a) holds more than twice the smallest (rank b) plus two
 * batches, rank a sends its last K = (largest - smallest) / 2 live regions
 * (capped by the transfer buffer: 8 (2n + 3) bytes per region) to rank b
 * through tfn; the received regions join rank b's list L.  Any region of the
 * domain stays in exactly one list, so the union of the enclosures is the
 * enclosure of the global minimum.  rank: 0 <= rank < 1024 (this process);
 * tbuf: device buffer of tbuf_bytes bytes (same size on every rank). */
int ib_solve_dev_mg(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                    const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                    double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream, ib_exchange_fn fn,
                    ib_transfer_fn tfn, void* user, double* xchg, int rank, double* tbuf, size_t tbuf_bytes);

/* Natural interval extension of f over nbox explicit boxes (device):
 * out[2k], out[2k+1] = lower / upper bound of f over box k.  For points pass
 * lo == hi.  Asynchronous. */
int ib_eval_boxes(int fid, int n, int64_t nbox, const double* lo, const double* hi, int64_t ld,
                  double* out, void* stream);

/* Enclosures of partial derivatives d f / d x_dim over box req_box[k]
 * (device arrays of nreq entries) -> out[2k], out[2k+1].  Asynchronous. */
int ib_eval_grad(int fid, int n, int64_t nreq, const double* lo, const double* hi, int64_t ld,
                 const int64_t* req_box, const int32_t* req_dim, double* out, void* stream);

/* Bytes of device workspace for ib_branch with nb parents. */
size_t ib_branch_workspace_size(int fid, int n, int d, int m, int64_t nb);

/* One branch-and-bound iteration on an explicit batch of nb parent boxes
 * (device, box-major, ld): every parent is partitioned into m^d children
 * along variables (pcyc[b] + j) mod n, j < d (variable cycling); the
 * midpoint upper bound of every child is min-reduced into *gub (device, in:
 * incumbent, out: updated); children with lower bound > GUB or failing the
 * first-order test (mono = 1) are discarded and the survivors written, in
 * (parent, child code) order, to out_parent / out_code / out_lb / out_w
 * (device, capacity nb * m^d).  *out_count (device) receives their number.
 * l, u: device bounds (edge rule of the first-order test).  Asynchronous. */
int ib_branch(int fid, int n, int d, int m, int mono, int64_t nb, const double* plo, const double* phi,
              int64_t ld, const int32_t* pcyc, const double* l, const double* u, double* gub,
              void* ws, size_t ws_bytes, int32_t* out_parent, uint32_t* out_code, double* out_lb,
              double* out_w, int64_t* out_count, void* stream);

/* Coordinate pattern search of DESIGN.md reading R9 (the sampling step
 * that supplies the initial incumbent, §3.1): a line
 * search along the diagonal x(t) = l + t (u - l) of [l, u] (t = k / 2^14,
 * k = 0..2^14, then up to 16 rounds of t +- 2^-j, j = 11..58; the paper's own
 * samples lie on diagonals, line 219), then from x(t*) at most `rounds`
 * improving coordinate moves, each the best of
 *   - the 8 joint moves x + 2^-a (xs - x), a = 0..7, where xs_i is the best
 *     of 128 candidates for variable i with the others fixed (32 grid points
 *     of [l_i, u_i], x_i +- (u_i - l_i) 2^-j for j = 1..48), and
 *   - the single best coordinate move;
 * every compared value is the upper end of an interval enclosure of f at a
 * point of [l, u], so *f_out is a rigorous upper bound of the global minimum.
 *   l, u        device, n doubles, l < u
 *   x_out       device, n doubles (may be NULL): the final point
 *   f_out       device, 1 double (may be NULL): upper bound of f(x_out)
 *   rounds_out  device, 1 int32 (may be NULL): accepted moves
 *   ws          device workspace >= ib_search_workspace_size(n)
 * One cooperative kernel launch; asynchronous on `stream`. */
size_t ib_search_workspace_size(int n);
int ib_search(int fid, int n, const double* l, const double* u, int rounds, double* x_out, double* f_out,
              int32_t* rounds_out, void* ws, size_t ws_bytes, void* stream);

/* Stable compaction: indices i < n with keys[i] <= thr, in increasing order
 * (device out_idx, capacity n; *out_count device).  ws: >= 8 * (n/1024 + 2)
 * bytes.  Asynchronous. */
int ib_compact_le(const double* keys, int64_t n, double thr, int64_t* out_idx, int64_t* out_count,
                  void* ws, size_t ws_bytes, void* stream);

/* Selection step of the list L (line 130, batched): among records with
 * lb[i] <= gub, the (up to) bmax smallest by (lb, index) are selected
 * (sel_idx, increasing index order); the other live records are kept
 * (keep_idx, increasing order).  Device arrays of capacity n; counts are
 * written to host *n_sel, *n_keep.  Synchronous. */
int ib_select(const double* lb, int64_t n, double gub, int64_t bmax, int64_t* sel_idx, int64_t* keep_idx,
              int64_t* n_sel, int64_t* n_keep, void* ws, size_t ws_bytes, void* stream);
size_t ib_select_workspace_size(int64_t n);

/* Inter-process handle of a device allocation (cudaIpcGetMemHandle): 64
 * bytes into handle.  ib_ipc_open maps a handle of another process (same or
 * peer GPU, NVLink) and returns the device address; ib_ipc_close unmaps it.
 * For ib_options.gub_shared across processes (tested with two processes on
 * one GPU; bench.py --mode partition exchanges the incumbent with NCCL per
 * chunk instead).  Return 0 or a CUDA error code. */
int ib_ipc_get_handle(const void* dptr, void* handle);
int ib_ipc_open(const void* handle, void** dptr);
int ib_ipc_close(void* dptr);

#ifdef __cplusplus
}
#endif
#endif
