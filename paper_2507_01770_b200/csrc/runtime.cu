// runtime.cu -- host side of the B200 branch-and-bound: workspace arena,
// the iteration driver of PAPER.md §3.1 (Fig. 2) and the extern "C" entry
// points declared in include/ibnb.h.  The host never touches a box: it only
// reads a 40-byte statistics block per iteration (and the 256-bin histogram
// when the list L is larger than the batch) to decide the next launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ibnb.h"
#include "kernels.cuh"

namespace ib {
int launch_prep(const Problem&, int, const int32_t*, const uint32_t*, const int32_t*, const double*,
                const double*, const int32_t*, double*, double*, int32_t*, double*, int, cudaStream_t);
int launch_child_eval(const Problem&, const double*, int, long, unsigned long long*, double*, cudaStream_t);
int launch_child_prune(const Problem&, const double*, int, long, const unsigned long long*, const double*,
                       const int32_t*, Pool, const uint64_t*, uint64_t*, uint32_t*, uint64_t*, cudaStream_t);

// children per child-eval thread: G = m^h <= 8 (h <= d)
static Problem make_problem(int fid, int n, int d, int m, long kids, int ld, int mono, const double* l,
                            const double* u) {
  int h = 0, G = 1;
  while (h < d && G * m <= 8) {
    G *= m;
    ++h;
  }
  int mbits = (m & (m - 1)) == 0 ? __builtin_ctz((unsigned)m) : 0;
  return Problem{fid, n, d, m, (int)kids, h, G, mbits, mbits * d, ld, mono, l, u};
}
int launch_pool_stats(Pool, const uint64_t*, long, const unsigned long long*, Stats*, cudaStream_t);
int launch_radix_hist(Pool, long, const unsigned long long*, int, unsigned long long, unsigned int*,
                      cudaStream_t);
int launch_partition(Pool, long, const unsigned long long*, int, unsigned long long, unsigned long long,
                     int32_t*, uint32_t*, double*, Pool, uint64_t*, uint32_t*, cudaStream_t);
int launch_gc(const int32_t*, long, const int32_t*, long, uint8_t*, long, int32_t*, uint64_t*, uint32_t*,
              uint64_t*, cudaStream_t);
int launch_alloc(const int32_t*, long, int, int32_t*, cudaStream_t);
int launch_compact_le(const double*, long, double, int64_t*, uint64_t*, uint32_t*, uint64_t*, cudaStream_t);
int launch_extract(const Problem&, Pool, long, const double*, const double*, const int32_t*, double*, double*,
                   double*, cudaStream_t);
int launch_eval_boxes(int, int, long, const double*, const double*, long, double*, cudaStream_t);
int launch_eval_grad(int, int, long, const double*, const double*, long, const int64_t*, const int32_t*,
                     double*, cudaStream_t);

// ------------------------------------------------------------ small kernels
__global__ void k_iota32(int32_t* a, long n, int32_t base) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    a[i] = base + (int32_t)i;
}
__global__ void k_fill_u32(uint32_t* a, long n, uint32_t v) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) a[i] = v;
}
__global__ void k_fill_f64(double* a, long n, double v) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) a[i] = v;
}
__global__ void k_i32_to_i64(const int32_t* a, long n, int64_t* b) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__device__ __forceinline__ unsigned long long okey_d(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv_d(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__global__ void k_gub_to_key(const double* g, unsigned long long* k) { *k = okey_d(*g); }
__global__ void k_key_to_gub(const unsigned long long* k, double* g) { *g = okey_inv_d(*k); }
__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }

static unsigned blocks_for(long n) {
  long g = (n + 255) / 256;
  return (unsigned)std::max(1L, std::min(g, 148L * 16));
}

static uint64_t okey_h(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
static double okey_inv_h(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  std::memcpy(&x, &b, 8);
  return x;
}
// a - b rounded upward, via TwoSum (host runs in round-to-nearest)
static double sub_up(double a, double b) {
  if (std::isinf(a) || std::isinf(b)) return a - b;
  volatile double s = a - b;
  volatile double bb = s - a;
  volatile double err = (a - (s - bb)) + (-b - bb);
  return err > 0.0 ? std::nextafter((double)s, INFINITY) : (double)s;
}

// ------------------------------------------------------------ errors
static thread_local std::string g_err;
static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) return fail((int)e_, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
#define CKL(x)                                                                      \
  do {                                                                              \
    int e_ = (x);                                                                   \
    if (e_ != 0) return fail(e_, "%s: %s", #x, cudaGetErrorString((cudaError_t)e_)); \
  } while (0)

// ------------------------------------------------------------ arena
struct Arena {
  char* base;
  size_t off, cap;
  bool dry;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += sizeof(T) * count;
    return p;
  }
};

struct Opts {
  int d, m, mono;
  long kids, bmax, max_iter, pool_cap, arch_cap;
  int ld, tab_stride;
};

static int resolve_opts(int fid, int n, const ib_options* o, int64_t pool_cap_arg, Opts& r) {
  if (fid < 0 || fid > 10) return fail(IB_EINVAL, "fid %d out of range", fid);
  if (n < 1 || n > (1 << 24)) return fail(IB_EINVAL, "n %d out of range", n);
  ib_options z;
  std::memset(&z, 0, sizeof z);
  if (!o) o = &z;
  r.d = o->d > 0 ? o->d : std::min(n, 10);
  if (r.d > n) r.d = n;
  r.m = o->m > 0 ? o->m : 2;
  r.mono = o->mono < 0 ? 0 : 1;
  if (r.d > D_MAX || r.m < 2 || r.m > M_MAX || r.d * r.m > DM_MAX)
    return fail(IB_EINVAL, "unsupported d=%d m=%d", r.d, r.m);
  double kids = std::pow((double)r.m, (double)r.d);
  if (kids > (double)(1 << 24)) return fail(IB_EINVAL, "m^d too large");
  r.kids = (long)kids;
  // default batch: ~4M children per iteration, fewer parents for large n
  // (every unpruned child stays in L)
  r.bmax = o->bmax > 0 ? o->bmax : std::max(1L, std::min((1L << 22) / r.kids, (1L << 17) / n));
  r.max_iter = o->max_iter > 0 ? o->max_iter : 1000000;
  long pc = o->pool_cap > 0 ? o->pool_cap : pool_cap_arg;
  if (pc <= 0) pc = std::max(1L << 26, 4 * r.bmax * r.kids);
  r.pool_cap = pc;
  r.ld = (n + 1) & ~1;  // even row stride -> 16-byte aligned rows
  long ac = o->arch_cap;
  if (ac <= 0) {
    long by_bytes = (16L << 30) / (16L * r.ld);  // 16 GiB archive budget
    ac = std::min(std::max(r.pool_cap / 4, 4 * r.bmax + 2), by_bytes);
    ac = std::max(ac, 2 * r.bmax + 2);
  }
  r.arch_cap = ac;
  r.tab_stride = HDR + r.d * r.m * ENT;
  return 0;
}

struct SolveWs {
  Pool pa, pb;
  int32_t *sel_slot, *new_slot, *sc, *free_list;
  uint32_t* sel_code;
  double *sel_lb, *alo, *ahi, *tab, *l, *u, *root_out, *clb;
  uint64_t *desc, *cnt;  // cnt[0] out_count, cnt[1] out_base, cnt[2] gc count
  uint32_t* tile_ctr;
  unsigned long long* gub_key;
  Stats* stats;
  unsigned int* hist;
  uint8_t* mark;
};

static size_t layout(const Opts& o, int n, Arena& A, SolveWs& w) {
  auto pool = [&](Pool& p) {
    p.lb = A.take<double>(o.pool_cap);
    p.w = A.take<double>(o.pool_cap);
    p.slot = A.take<int32_t>(o.pool_cap);
    p.code = A.take<uint32_t>(o.pool_cap);
  };
  pool(w.pa);
  pool(w.pb);
  w.sel_slot = A.take<int32_t>(o.bmax);
  w.sel_code = A.take<uint32_t>(o.bmax);
  w.sel_lb = A.take<double>(o.bmax);
  w.new_slot = A.take<int32_t>(o.bmax);
  w.alo = A.take<double>((size_t)o.arch_cap * o.ld);
  w.ahi = A.take<double>((size_t)o.arch_cap * o.ld);
  w.sc = A.take<int32_t>(o.arch_cap);
  w.free_list = A.take<int32_t>(o.arch_cap);
  w.mark = A.take<uint8_t>(o.arch_cap);
  w.tab = A.take<double>((size_t)o.bmax * o.tab_stride);
  w.clb = A.take<double>((size_t)o.bmax * o.kids);
  long tiles = std::max({o.pool_cap, o.bmax * o.kids, o.arch_cap}) / TILE + 2;
  w.desc = A.take<uint64_t>((size_t)tiles * 3);
  w.cnt = A.take<uint64_t>(4);
  w.tile_ctr = A.take<uint32_t>(4);
  w.gub_key = A.take<unsigned long long>(1);
  w.stats = A.take<Stats>(1);
  w.hist = A.take<unsigned int>(256);
  w.l = A.take<double>(n);
  w.u = A.take<double>(n);
  w.root_out = A.take<double>(2);
  return A.off + 256;
}

// per-launch CUDA-event timing of the kernel classes (opt.profile)
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Rec {
    int cls;
    long units;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  size_t next = 0;
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[next++];
  }
  cudaEvent_t cur_a = nullptr;
  void begin(cudaStream_t st) {
    if (!on || recs.size() > 20000) return;
    cur_a = ev();
    cudaEventRecord(cur_a, st);
  }
  void end(int cls, long units, cudaStream_t st) {
    if (!on || !cur_a) return;
    cudaEvent_t b = ev();
    cudaEventRecord(b, st);
    recs.push_back(Rec{cls, units, cur_a, b});
    cur_a = nullptr;
  }
  void collect(ib_result* res) {
    for (int c = 0; c < IB_NPROF; ++c) {
      res->t_ms[c] = 0.0;
      res->launches[c] = 0;
      res->units[c] = 0;
    }
    for (auto& q : recs) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, q.a, q.b);
      res->t_ms[q.cls] += ms;
      res->launches[q.cls] += 1;
      res->units[q.cls] += q.units;
    }
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

__global__ void k_xchg_put(const unsigned long long* gub_key, double* xchg, double done) {
  xchg[0] = okey_inv_d(*gub_key);
  xchg[1] = done;
}
__global__ void k_xchg_take(unsigned long long* gub_key, const double* xchg) {
  unsigned long long k = okey_d(xchg[0]);
  if (k < *gub_key) *gub_key = k;
}

static int solve_impl(int fid, int n, const double* l_dev, const double* u_dev, const double* l_host,
                      const double* u_host, double eps_f, double eps_x, const ib_options* opt, void* ws,
                      size_t ws_bytes, ib_result* res, double* so_lo, double* so_hi, double* so_lb,
                      int64_t surv_cap, bool host_out, cudaStream_t st, ib_exchange_fn xfn, void* xuser,
                      double* xchg) {
  Opts o;
  int rc = resolve_opts(fid, n, opt, 0, o);
  if (rc) return rc;
  if (!res) return fail(IB_EINVAL, "res is NULL");
  if (xfn && !xchg) return fail(IB_EINVAL, "exchange buffer is NULL");
  std::memset(res, 0, sizeof(*res));
  Arena A{(char*)ws, 0, ws_bytes, false};
  SolveWs w;
  size_t need = layout(o, n, A, w);
  if (!ws || ws_bytes < need) return fail(IB_ENOSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  Problem P = make_problem(fid, n, o.d, o.m, o.kids, o.ld, o.mono, w.l, w.u);
  Prof prof;
  prof.on = opt && opt->profile == 1;
  long nk = 0;  // kernels launched by this call

  // bounds and the root region (line 128): archive slot 0, list L = {root}
  std::vector<double> lh(n), uh(n);
  if (l_host) {
    std::memcpy(lh.data(), l_host, sizeof(double) * n);
    std::memcpy(uh.data(), u_host, sizeof(double) * n);
    CK(cudaMemcpyAsync(w.l, l_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.u, u_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  } else {
    CK(cudaMemcpyAsync(w.l, l_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(w.u, u_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(lh.data(), l_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(uh.data(), u_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  double w0 = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!(lh[i] < uh[i]) || !std::isfinite(lh[i]) || !std::isfinite(uh[i]))
      return fail(IB_EINVAL, "bounds must be finite with l < u (variable %d)", i);
    w0 = std::max(w0, uh[i] - lh[i]);
  }
  CK(cudaMemcpyAsync(w.alo, w.l, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(w.ahi, w.u, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(w.sc, 0, sizeof(int32_t), st));
  CKL(launch_eval_boxes(fid, n, 1, w.alo, w.ahi, o.ld, w.root_out, st));
  nk += 2;  // root bound + free-list iota
  // free list: slots 1 .. arch_cap-1
  k_iota32<<<blocks_for(o.arch_cap - 1), 256, 0, st>>>(w.free_list, o.arch_cap - 1, 1);
  long free_top = o.arch_cap - 1;
  double root[2];
  CK(cudaMemcpyAsync(root, w.root_out, sizeof root, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double lb0 = root[0] != root[0] ? -INFINITY : (root[0] == 0.0 ? 0.0 : root[0]);
  uint32_t whole = CODE_WHOLE;
  int32_t zero = 0;
  unsigned long long inf_key = okey_h(INFINITY);
  uint64_t one = 1;
  CK(cudaMemcpyAsync(w.pa.lb, &lb0, 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.pa.w, &w0, 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.pa.slot, &zero, 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.pa.code, &whole, 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.gub_key, &inf_key, 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(w.cnt, &one, 8, cudaMemcpyHostToDevice, st));

  struct Rb {
    Stats s;
    unsigned long long gub_key;
    uint64_t count;
    double gdone;
  } rb;
  rb.gdone = -1.0;
  long iter = 0, evals = 0, peak = 1, nx = 0;
  int status = IB_STATUS_MAX_ITER;
  double glb = INFINITY, gub = INFINITY, maxw = 0.0;
  long pbound = 1, pcount = 1, live = 0;
  for (;;) {
    // steps 6-7: statistics of the live part of L (lb <= GUB): one sync
    prof.begin(st);
    CKL(launch_pool_stats(w.pa, w.cnt, pbound, w.gub_key, w.stats, st));
    nk += 2;
    prof.end(3, pbound, st);
    CK(cudaMemcpyAsync(&rb.s, w.stats, sizeof(Stats), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&rb.gub_key, w.gub_key, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&rb.count, w.cnt, 8, cudaMemcpyDeviceToHost, st));
    if (xfn) CK(cudaMemcpyAsync(&rb.gdone, xchg + 1, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    pcount = (long)rb.count;
    peak = std::max(peak, pcount);
    live = (long)rb.s.live;
    gub = okey_inv_h(rb.gub_key);
    glb = live ? okey_inv_h(rb.s.min_lb_key) : INFINITY;
    std::memcpy(&maxw, &rb.s.max_w_bits, 8);
    bool done = false;
    if (live == 0) {
      status = xfn ? IB_STATUS_EMPTY : IB_EEMPTY;
      done = true;
    } else if (maxw <= eps_x && sub_up(gub, glb) <= eps_f) {
      status = IB_STATUS_CONVERGED;
      done = true;
    } else if (iter >= o.max_iter) {
      status = IB_STATUS_MAX_ITER;
      done = true;
    }
    if (!xfn && done) break;
    if (xfn && nx > 0 && rb.gdone == 0.0) break;  // every rank finished
    long B = 0, K = 0;
    if (!done) {
      // step 1: select the B smallest (lb, position) live records
      B = std::min(live, o.bmax);
      int known = 0;
      unsigned long long prefix = 0, r_need = 0;
      if (live > o.bmax) {
        unsigned long long need = (unsigned long long)B;
        unsigned int h[256];
        while (known < 64) {
          prof.begin(st);
          CKL(launch_radix_hist(w.pa, pcount, w.gub_key, known, prefix, w.hist, st));
          nk += 1;
          prof.end(4, pcount, st);
          CK(cudaMemcpyAsync(h, w.hist, sizeof h, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          unsigned long long cum = 0;
          int dig = 0;
          for (; dig < 256; ++dig) {
            if (cum + h[dig] >= need) break;
            cum += h[dig];
          }
          if (dig == 256) return fail(IB_EINVAL, "radix select inconsistent");
          need -= cum;
          prefix = (prefix << 8) | (unsigned long long)dig;
          known += 8;
          if (h[dig] == need) break;
        }
        r_need = need;
      }
      K = live - B;
      prof.begin(st);
      CKL(launch_partition(w.pa, pcount, w.gub_key, known, prefix, r_need, w.sel_slot, w.sel_code, w.sel_lb,
                           w.pb, w.desc, w.tile_ctr, st));
      nk += 1;
      prof.end(5, pcount, st);
      // archive slots for the B new parents (mark-and-collect when short)
      if (free_top < B) {
        CKL(launch_gc(w.pb.slot, K, w.sel_slot, B, w.mark, o.arch_cap, w.free_list, w.desc, w.tile_ctr,
                      w.cnt + 2, st));
        nk += 3;
        uint64_t fc;
        CK(cudaMemcpyAsync(&fc, w.cnt + 2, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        free_top = (long)fc;
        if (free_top < B) return fail(IB_ENOSPACE, "archive full (%ld slots)", o.arch_cap);
      }
      CKL(launch_alloc(w.free_list, free_top, (int)B, w.new_slot, st));
      nk += 3;  // alloc + prep + child_eval
      free_top -= B;
      if (K + B * o.kids > o.pool_cap)
        return fail(IB_ENOSPACE, "list L capacity %ld exceeded (%ld kept + %ld children)", o.pool_cap, K,
                    B * o.kids);
      // steps 2-3: partition (SPSD) and midpoint sampling -> GUB
      prof.begin(st);
      CKL(launch_prep(P, (int)B, w.sel_slot, w.sel_code, w.new_slot, w.alo, w.ahi, w.sc, w.alo, w.ahi, w.sc,
                      w.tab, o.tab_stride, st));
      prof.end(0, B, st);
      prof.begin(st);
      CKL(launch_child_eval(P, w.tab, o.tab_stride, B * o.kids, w.gub_key, w.clb, st));
      prof.end(1, B * o.kids, st);
    }
    if (xfn) {
      // multi-GPU: GUB <- min over ranks (line 134 across the partition)
      k_xchg_put<<<1, 1, 0, st>>>(w.gub_key, xchg, done ? 0.0 : -1.0);
      nk += 2;
      xfn(xuser);
      ++nx;
      k_xchg_take<<<1, 1, 0, st>>>(w.gub_key, xchg);
      CK(cudaGetLastError());
    }
    if (!done) {
      // steps 4-5: bound, rule out, insert survivors after the kept records
      k_set_u64<<<1, 1, 0, st>>>(w.cnt + 1, (uint64_t)K);
      nk += 2;  // set + child_prune
      prof.begin(st);
      CKL(launch_child_prune(P, w.tab, o.tab_stride, B * o.kids, w.gub_key, w.clb, w.new_slot, w.pb, w.cnt + 1,
                             w.desc, w.tile_ctr, w.cnt, st));
      prof.end(2, B * o.kids, st);
      std::swap(w.pa, w.pb);
      ++iter;
      evals += B * o.kids;
      pbound = K + B * o.kids;
    }
  }
  if (status == IB_EEMPTY) return fail(IB_EEMPTY, "list L became empty after %ld iterations", iter);
  // output (line 150): GLB, GUB and the live regions of L, in list order
  CKL(launch_partition(w.pa, pcount, w.gub_key, 64, 0ull, 0ull, w.sel_slot, w.sel_code, w.sel_lb, w.pb, w.desc,
                       w.tile_ctr, st));
  nk += 1;
  long ncopy = std::min((long)surv_cap, live);
  if (so_lo && so_hi && ncopy > 0) {
    if (host_out) {
      // stage through the (now unused) tables buffer, in chunks
      long per = std::max(1L, (long)(((size_t)o.bmax * o.tab_stride) / (size_t)(2 * n + 1)));
      double* tlo = w.tab;
      for (long s = 0; s < ncopy; s += per) {
        long k = std::min(per, ncopy - s);
        double* thi = tlo + (size_t)k * n;
        double* tlb = thi + (size_t)k * n;
        Pool sub{w.pb.lb + s, w.pb.w + s, w.pb.slot + s, w.pb.code + s};
        CKL(launch_extract(P, sub, k, w.alo, w.ahi, w.sc, tlo, thi, tlb, st));
        nk += 1;
        CK(cudaMemcpyAsync(so_lo + (size_t)s * n, tlo, sizeof(double) * k * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(so_hi + (size_t)s * n, thi, sizeof(double) * k * n, cudaMemcpyDeviceToHost, st));
        if (so_lb) CK(cudaMemcpyAsync(so_lb + s, tlb, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
    } else {
      CKL(launch_extract(P, w.pb, ncopy, w.alo, w.ahi, w.sc, so_lo, so_hi, so_lb, st));
      nk += 1;
    }
  }
  CK(cudaStreamSynchronize(st));
  prof.collect(res);
  res->f_lo = glb;
  res->f_hi = gub;
  res->iters = iter;
  res->evals = evals;
  res->n_surv = live;
  res->peak_pool = peak;
  res->max_width = maxw;
  res->status = status;
  res->n_kernels = (int)std::min(nk, (long)INT32_MAX);
  return 0;
}

}  // namespace ib

using namespace ib;

extern "C" {

const char* ib_version(void) { return "ibnb 0.1.0 (sm_100a, fp64 directed rounding)"; }
const char* ib_last_error(void) { return g_err.c_str(); }
int ib_num_functions(void) { return 11; }

size_t ib_solve_workspace_size(int fid, int n, const ib_options* opt, int64_t pool_cap) {
  Opts o;
  if (resolve_opts(fid, n, opt, pool_cap, o)) return 0;
  Arena A{nullptr, 0, 0, true};
  SolveWs w;
  return layout(o, n, A, w);
}

int ib_solve(int fid, int n, const double* l, const double* u, double eps_f, double eps_x,
             const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
             double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream) {
  if (!l || !u) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, nullptr, nullptr, l, u, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo, surv_hi,
                    surv_lb, surv_cap, true, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

int ib_solve_dev(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                 const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                 double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream) {
  if (!l_dev || !u_dev) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, l_dev, u_dev, nullptr, nullptr, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo,
                    surv_hi, surv_lb, surv_cap, false, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

int ib_solve_dev_ex(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                    const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                    double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream, ib_exchange_fn fn,
                    void* user, double* xchg) {
  if (!l_dev || !u_dev) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, l_dev, u_dev, nullptr, nullptr, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo,
                    surv_hi, surv_lb, surv_cap, false, (cudaStream_t)stream, fn, user, xchg);
}

int ib_eval_boxes(int fid, int n, int64_t nbox, const double* lo, const double* hi, int64_t ld, double* out,
                  void* stream) {
  if (fid < 0 || fid > 10 || n < 1 || nbox < 0 || ld < n || (!lo && nbox) || (!hi && nbox) || (!out && nbox))
    return fail(IB_EINVAL, "ib_eval_boxes: bad arguments");
  CKL(launch_eval_boxes(fid, n, (long)nbox, lo, hi, (long)ld, out, (cudaStream_t)stream));
  return 0;
}

int ib_eval_grad(int fid, int n, int64_t nreq, const double* lo, const double* hi, int64_t ld,
                 const int64_t* req_box, const int32_t* req_dim, double* out, void* stream) {
  if (fid < 0 || fid > 10 || n < 1 || nreq < 0 || ld < n) return fail(IB_EINVAL, "ib_eval_grad: bad arguments");
  CKL(launch_eval_grad(fid, n, (long)nreq, lo, hi, (long)ld, req_box, req_dim, out, (cudaStream_t)stream));
  return 0;
}

struct BranchWs {
  int32_t *iota, *dst_sc;
  uint32_t* whole;
  double *dlo, *dhi, *tab, *clb;
  uint64_t *desc, *cnt;
  uint32_t* tile_ctr;
  unsigned long long* gub_key;
};
static size_t branch_layout(int n, int d, int m, long nb, Arena& A, BranchWs& w) {
  long kids = (long)std::pow((double)m, (double)d);
  int ld = (n + 1) & ~1;
  int stride = HDR + d * m * ENT;
  w.iota = A.take<int32_t>(nb);
  w.dst_sc = A.take<int32_t>(nb);
  w.whole = A.take<uint32_t>(nb);
  w.dlo = A.take<double>((size_t)nb * ld);
  w.dhi = A.take<double>((size_t)nb * ld);
  w.tab = A.take<double>((size_t)nb * stride);
  w.clb = A.take<double>((size_t)nb * kids);
  w.desc = A.take<uint64_t>((size_t)(nb * kids / TILE + 2));
  w.cnt = A.take<uint64_t>(2);
  w.tile_ctr = A.take<uint32_t>(1);
  w.gub_key = A.take<unsigned long long>(1);
  return A.off + 256;
}

size_t ib_branch_workspace_size(int fid, int n, int d, int m, int64_t nb) {
  (void)fid;
  if (n < 1 || d < 1 || d > n || d > D_MAX || m < 2 || m > M_MAX || d * m > DM_MAX || nb < 0) return 0;
  Arena A{nullptr, 0, 0, true};
  BranchWs w;
  return branch_layout(n, d, m, (long)nb, A, w);
}

int ib_branch(int fid, int n, int d, int m, int mono, int64_t nb, const double* plo, const double* phi,
              int64_t ld, const int32_t* pcyc, const double* l, const double* u, double* gub, void* ws,
              size_t ws_bytes, int32_t* out_parent, uint32_t* out_code, double* out_lb, double* out_w,
              int64_t* out_count, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (fid < 0 || fid > 10 || n < 1 || d < 1 || d > n || d > D_MAX || m < 2 || m > M_MAX || d * m > DM_MAX ||
      nb < 1 || ld < n)
    return fail(IB_EINVAL, "ib_branch: bad arguments");
  double kids_d = std::pow((double)m, (double)d);
  if (kids_d > (double)(1 << 24) || nb * kids_d > 4.0e9) return fail(IB_EINVAL, "ib_branch: too many children");
  long kids = (long)kids_d;
  Arena A{(char*)ws, 0, ws_bytes, false};
  BranchWs w;
  size_t need = branch_layout(n, d, m, (long)nb, A, w);
  if (!ws || ws_bytes < need) return fail(IB_ENOSPACE, "ib_branch workspace %zu < %zu", ws_bytes, need);
  int ldi = (n + 1) & ~1;
  Problem P = make_problem(fid, n, d, m, kids, ldi, mono ? 1 : 0, l, u);
  k_iota32<<<blocks_for(nb), 256, 0, st>>>(w.iota, nb, 0);
  k_fill_u32<<<blocks_for(nb), 256, 0, st>>>(w.whole, nb, CODE_WHOLE);
  k_gub_to_key<<<1, 1, 0, st>>>(gub, w.gub_key);
  k_set_u64<<<1, 1, 0, st>>>(w.cnt + 1, 0ull);
  if ((int)ld != ldi) {
    // copy the parents into our stride first (plain strided copy)
    CK(cudaMemcpy2DAsync(w.dlo, sizeof(double) * ldi, plo, sizeof(double) * ld, sizeof(double) * n, nb,
                         cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpy2DAsync(w.dhi, sizeof(double) * ldi, phi, sizeof(double) * ld, sizeof(double) * n, nb,
                         cudaMemcpyDeviceToDevice, st));
    plo = w.dlo;
    phi = w.dhi;
  }
  CKL(launch_prep(P, (int)nb, w.iota, w.whole, w.iota, plo, phi, pcyc, w.dlo, w.dhi, w.dst_sc, w.tab,
                  HDR + d * m * ENT, st));
  CKL(launch_child_eval(P, w.tab, HDR + d * m * ENT, nb * kids, w.gub_key, w.clb, st));
  Pool out{out_lb, out_w, out_parent, out_code};
  CKL(launch_child_prune(P, w.tab, HDR + d * m * ENT, nb * kids, w.gub_key, w.clb, w.iota, out, w.cnt + 1,
                         w.desc, w.tile_ctr, (uint64_t*)out_count, st));
  k_key_to_gub<<<1, 1, 0, st>>>(w.gub_key, gub);
  CK(cudaGetLastError());
  return 0;
}

int ib_compact_le(const double* keys, int64_t n, double thr, int64_t* out_idx, int64_t* out_count, void* ws,
                  size_t ws_bytes, void* stream) {
  size_t need = 8 * (size_t)(n / TILE + 2) + 256 + 64;
  if (n < 0 || !out_count || !ws || ws_bytes < need) return fail(IB_EINVAL, "ib_compact_le: bad arguments");
  uint32_t* tile_ctr = (uint32_t*)ws;
  uint64_t* desc = (uint64_t*)((char*)ws + 256);
  CKL(launch_compact_le(keys, (long)n, thr, out_idx, desc, tile_ctr, (uint64_t*)out_count, (cudaStream_t)stream));
  return 0;
}

size_t ib_select_workspace_size(int64_t n) {
  if (n < 0) return 0;
  Arena A{nullptr, 0, 0, true};
  A.take<double>(n);     // w
  A.take<int32_t>(n);    // slot (iota)
  A.take<uint32_t>(n);   // code
  A.take<double>(n);     // keep lb
  A.take<double>(n);     // keep w
  A.take<int32_t>(n);    // keep slot
  A.take<uint32_t>(n);   // keep code
  A.take<int32_t>(n);    // sel slot
  A.take<uint32_t>(n);   // sel code
  A.take<double>(n);     // sel lb
  A.take<uint64_t>((size_t)(n / TILE + 2) * 3);
  A.take<uint32_t>(4);
  A.take<unsigned long long>(1);
  A.take<Stats>(1);
  A.take<unsigned int>(256);
  return A.off + 256;
}

int ib_select(const double* lb, int64_t n, double gub, int64_t bmax, int64_t* sel_idx, int64_t* keep_idx,
              int64_t* n_sel, int64_t* n_keep, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || bmax < 1 || !n_sel || !n_keep) return fail(IB_EINVAL, "ib_select: bad arguments");
  if (!ws || ws_bytes < ib_select_workspace_size(n)) return fail(IB_ENOSPACE, "ib_select: workspace too small");
  Arena A{(char*)ws, 0, ws_bytes, false};
  Pool in{const_cast<double*>(lb), A.take<double>(n), A.take<int32_t>(n), A.take<uint32_t>(n)};
  Pool keep{A.take<double>(n), A.take<double>(n), A.take<int32_t>(n), A.take<uint32_t>(n)};
  int32_t* sel_slot = A.take<int32_t>(n);
  uint32_t* sel_code = A.take<uint32_t>(n);
  double* sel_lb = A.take<double>(n);
  uint64_t* desc = A.take<uint64_t>((size_t)(n / TILE + 2) * 3);
  uint32_t* tile_ctr = A.take<uint32_t>(4);
  unsigned long long* gkey = A.take<unsigned long long>(1);
  Stats* stats = A.take<Stats>(1);
  unsigned int* hist = A.take<unsigned int>(256);
  if (n == 0) {
    *n_sel = *n_keep = 0;
    return 0;
  }
  k_fill_f64<<<blocks_for(n), 256, 0, st>>>(in.w, n, 0.0);
  k_iota32<<<blocks_for(n), 256, 0, st>>>(in.slot, n, 0);
  k_fill_u32<<<blocks_for(n), 256, 0, st>>>(in.code, n, 0u);
  unsigned long long gk = okey_h(gub);
  uint64_t nn = (uint64_t)n;
  CK(cudaMemcpyAsync(gkey, &gk, 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(tile_ctr + 2, &nn, 8, cudaMemcpyHostToDevice, st));
  CKL(launch_pool_stats(in, (const uint64_t*)(tile_ctr + 2), (long)n, gkey, stats, st));
  Stats s;
  CK(cudaMemcpyAsync(&s, stats, sizeof s, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  long live = (long)s.live;
  long B = std::min(live, (long)bmax);
  int known = 0;
  unsigned long long prefix = 0, r_need = 0;
  if (live > bmax) {
    unsigned long long need = (unsigned long long)B;
    unsigned int h[256];
    while (known < 64) {
      CKL(launch_radix_hist(in, (long)n, gkey, known, prefix, hist, st));
      CK(cudaMemcpyAsync(h, hist, sizeof h, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long cum = 0;
      int dig = 0;
      for (; dig < 256; ++dig) {
        if (cum + h[dig] >= need) break;
        cum += h[dig];
      }
      need -= cum;
      prefix = (prefix << 8) | (unsigned long long)dig;
      known += 8;
      if (h[dig] == need) break;
    }
    r_need = need;
  }
  CKL(launch_partition(in, (long)n, gkey, known, prefix, r_need, sel_slot, sel_code, sel_lb, keep, desc, tile_ctr,
                       st));
  if (B > 0) k_i32_to_i64<<<blocks_for(B), 256, 0, st>>>(sel_slot, B, sel_idx);
  if (live - B > 0) k_i32_to_i64<<<blocks_for(live - B), 256, 0, st>>>(keep.slot, live - B, keep_idx);
  CK(cudaStreamSynchronize(st));
  *n_sel = B;
  *n_keep = live - B;
  return 0;
}

}  // extern "C"
