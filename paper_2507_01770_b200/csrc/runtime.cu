// runtime.cu -- host side of the B200 branch-and-bound: workspace arena, the
// iteration driver of PAPER.md §3.1 (Fig. 2) and the extern "C" entry points
// of include/ibnb.h.
//
// The host never touches a box and takes no per-iteration decision: every
// iteration's stop test, batch size and radix-select digits are computed on
// the GPU (Ctl, kernels.cuh), and iterations after the stop are no-ops.  The
// host enqueues chunks of iterations (replaying one captured CUDA graph per
// iteration when possible) and synchronises once per chunk to read the
// control block, compact L and collect archive slots when needed.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ibnb.h"
#include "kernels.cuh"

namespace ib {
int launch_iteration(const Problem&, const IterBufs&, long, long, cudaStream_t, IterHook*, long);
int launch_branch(const Problem&, const IterBufs&, long, cudaStream_t);
int launch_fused(const Problem&, const IterBufs&, int, long, cudaStream_t);
int launch_chain(const Problem&, const IterBufs&, const ChainBufs&, int, cudaStream_t);
int launch_chainc(const Problem&, const IterBufs&, const ChainBufs&, int, int, cudaStream_t);
int launch_select_only(Pool, Ctl*, unsigned int*, long, cudaStream_t);
int launch_xchg_put(const Ctl*, double*, cudaStream_t);
int launch_apply_pending(Ctl*, long, cudaStream_t);
int launch_final_width(Pool, Ctl*, long, cudaStream_t);
int launch_xchg_take(Ctl*, const double*, cudaStream_t);
int launch_partition(Pool, long, const unsigned long long*, int, unsigned long long, unsigned long long, int32_t*,
                     uint32_t*, double*, Pool, uint64_t*, uint32_t*, uint64_t*, cudaStream_t);
int launch_gc(Pool, Ctl*, long, uint8_t*, long, int32_t*, uint64_t*, uint32_t*, cudaStream_t);
int launch_compact_le(const double*, long, double, int64_t*, uint64_t*, uint32_t*, uint64_t*, cudaStream_t);
int launch_extract(const Problem&, Pool, long, const double*, const double*, const int32_t*, double*, double*,
                   double*, cudaStream_t);
int launch_eval_boxes(int, int, long, const double*, const double*, long, double*, cudaStream_t);
int launch_eval_grad(int, int, long, const double*, const double*, long, const int64_t*, const int32_t*,
                     double*, cudaStream_t);
size_t search_ws_bytes(int n, int grid);
int search_grid_max();
int launch_search(int fid, int n, const double* l, const double* u, int rounds, void* ws, size_t ws_bytes,
                  unsigned long long* gub_key, double* x_out, double* f_out, int32_t* rounds_out, cudaStream_t st);

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
// root record of L (line 128) from the root bound computed by ib_eval
__global__ void k_root(const double* root_out, double w0, Pool p, Ctl* ctl) {
  double lb = root_out[0];
  lb = lb != lb ? -CUDART_INF : (lb == 0.0 ? 0.0 : lb);
  p.lb[0] = lb;
  p.w[0] = w0;
  p.slot[0] = 0;
  p.code[0] = CODE_WHOLE;
  ctl->pcount = 1;
}
// after a compaction of L: new record count, positions changed -> rebuild the hot index
// multi-GPU incumbent word (ib_options.gub_shared): lower it to this rank's
// GUB and take the other ranks' value back -- before every chunk, so the
// batch paths (k_fused, the iteration graph) prune with it too; k_chain also
// does this every iteration
__global__ void k_gub_shared(Ctl* ctl, unsigned long long* word) {
  const unsigned long long old = atomicMin(word, ctl->gub_key);
  if (old < ctl->gub_key) ctl->gub_key = old;
}
__global__ void k_set_pcount(Ctl* ctl, const uint64_t* c) {
  ctl->pcount = *c;
  ctl->hot_valid = 0;
  ctl->list_fast = 0;
  ctl->nhot = 0;
  ctl->compact_hint = 0;
}
// ---- multi-GPU rebalancing (ib_solve_dev_mg)
// live records of L (lb <= GUB) -> xchg[2], xchg[3] = -(live * 1024 + rank),
// live * 1024 + rank: after an element-wise MIN over ranks they hold the
// largest and the smallest list (ties: highest / lowest rank)
__global__ void k_count_live(Pool p, const Ctl* ctl, unsigned long long* acc) {
  const double gub = okey_inv_d(ctl->gub_key);
  const long cnt = (long)ctl->pcount;
  unsigned long long c = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long)gridDim.x * blockDim.x)
    c += p.lb[i] <= gub;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(acc, c);
}
__global__ void k_live_key(const unsigned long long* acc, int rank, double* xchg) {
  const double key = (double)(*acc) * 1024.0 + (double)rank;
  xchg[2] = -key;
  xchg[3] = key;
}
// exported regions [first, first + k) of a compacted list: width and the
// cycling index the region will be split on next (k_prep's rule, line 184)
__global__ void k_export_meta(Pool p, long first, long k, const int32_t* sc, int d, int n, double* out_w,
                              double* out_cyc) {
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (long)gridDim.x * blockDim.x) {
    const long q = first + r;
    const int psc = sc[p.slot[q]];
    out_w[r] = p.w[q];
    out_cyc[r] = (double)(p.code[q] == CODE_WHOLE ? psc : (psc + d) % n);
  }
}
// received regions: archive slots from the free list, records appended to L
__global__ void k_import(Pool p, const Ctl* ctl, const double* in_lo, const double* in_hi, const double* in_lb,
                         const double* in_w, const double* in_cyc, long k, int n, int ld, double* alo, double* ahi,
                         int32_t* sc, const int32_t* free_list) {
  const unsigned long long top = ctl->free_top, base = ctl->pcount;
  for (long r = blockIdx.x; r < k; r += gridDim.x) {
    const int slot = free_list[top - 1 - r];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      alo[(size_t)slot * ld + i] = in_lo[(size_t)r * n + i];
      ahi[(size_t)slot * ld + i] = in_hi[(size_t)r * n + i];
    }
    if (threadIdx.x == 0) {
      sc[slot] = (int32_t)in_cyc[r];
      p.lb[base + r] = in_lb[r];
      p.w[base + r] = in_w[r];
      p.slot[base + r] = slot;
      p.code[base + r] = CODE_WHOLE;
    }
  }
}
// list changed outside an iteration: new record count, hot index rebuilt
__global__ void k_list_changed(Ctl* ctl, long pcount, long taken_slots) {
  // a rank that had converged or run out of regions works again on what it
  // received (an error or the iteration limit stays final)
  if (taken_slots > 0 && (ctl->done == 1 || ctl->done == 3)) ctl->done = 0;
  ctl->pcount = (unsigned long long)pcount;
  ctl->free_top -= (unsigned long long)taken_slots;
  ctl->hot_valid = 0;
  ctl->list_fast = 0;
  ctl->nhot = 0;
  ctl->compact_hint = 0;
}

__global__ void k_branch_ctl(Ctl* ctl, const double* gub, long nb, long cap) {
  unsigned long long* z = reinterpret_cast<unsigned long long*>(ctl);
  for (size_t i = 0; i < sizeof(Ctl) / 8; ++i) z[i] = 0ull;
  ctl->gub_key = okey_d(*gub);
  ctl->B = (unsigned long long)nb;
  ctl->pool_cap = (unsigned long long)cap;
}
__global__ void k_branch_out(const Ctl* ctl, double* gub, int64_t* count) {
  *gub = okey_inv_d(ctl->gub_key);
  *count = (int64_t)ctl->nsurv;
}

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
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail((int)e_, "%s: %s", #x, cudaGetErrorString(e_));     \
  } while (0)
#define CKL(x)                                                                             \
  do {                                                                                     \
    int e_ = (x);                                                                          \
    if (e_ != 0) return fail(e_, "%s: %s", #x, cudaGetErrorString((cudaError_t)e_));       \
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
  int d, m, mono, search;
  long kids, bmax, max_iter, pool_cap, arch_cap;
  int ld, tab_stride;
};

static int resolve_opts(int fid, int n, const ib_options* o, int64_t pool_cap_arg, Opts& r) {
  if (fid < 0 || fid > 10) return fail(IB_EINVAL, "fid %d out of range", fid);
  if (n < 1 || n > (1 << 24)) return fail(IB_EINVAL, "n %d out of range", n);
  ib_options z;
  std::memset(&z, 0, sizeof z);
  if (!o) o = &z;
  r.d = o->d > 0 ? o->d : std::min(n, 16);
  if (r.d > n) r.d = n;
  r.m = o->m > 0 ? o->m : 2;
  r.mono = o->mono < 0 ? 0 : 1;
  r.search = o->search < 0 ? 0 : (o->search > 0 ? o->search : 32);
  if (r.d > D_MAX || r.m < 2 || r.m > M_MAX || r.d * r.m > DM_MAX)
    return fail(IB_EINVAL, "unsupported d=%d m=%d", r.d, r.m);
  double kids = std::pow((double)r.m, (double)r.d);
  if (kids > (double)(1 << 24)) return fail(IB_EINVAL, "m^d too large");
  r.kids = (long)kids;
  // default batch: ~4M children per iteration, fewer parents for large n
  // (every unpruned child stays in L; reading R1)
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

// children per child-eval thread: G = m^h <= 8 (h <= d)
// k_prep blocks per parent: one unless n is large and the batch too small
// to fill the SMs, then slices of >= 256 variables
static int prep_slices(int n, long bmax) {
  if (n < 512 || bmax >= 296) return 1;
  long s = std::min((long)(n + 127) / 128, std::max(1L, 1184 / bmax));  // 128 variables: one per half-block thread
  return (int)std::max(1L, s);
}

static Problem make_problem(int fid, int n, int d, int m, long kids, int ld, int mono, const double* l,
                            const double* u, long bmax) {
  // a child-eval thread owns G = m^h children when they share work (the
  // combination of the d - h higher pieces of K-accumulator objectives); the
  // Levy chain (fid 6) recomputes its chain terms per child, so a thread per
  // child spreads them over more threads
  int h = 0, G = 1;
  while (fid != 6 && h < d && G * m <= 8) {
    G *= m;
    ++h;
  }
  int mbits = (m & (m - 1)) == 0 ? __builtin_ctz((unsigned)m) : 0;
  const int ps = prep_slices(n, bmax);
  // the child phase combines the slice partials when every block of it sees
  // at most two parents and their tables fit its shared memory (bisection)
  const int prest = ps > 1 && m == 2 && d <= D_MAX && kids / G >= TPB;
  int mitm = d > 16;  // the pair tree of chain_children covers d - 1 <= 16 terms
  if (const char* e = std::getenv("IBNB_CHAIN_MITM")) mitm = mitm || std::atoi(e) != 0;
  return Problem{fid, n, d, m, (int)kids, h, G, mbits, mbits * d, ld, mono, ps, prest, mitm, l, u};
}

static long tiles_of(long n) { return std::max(1L, (n + TILE - 1) / TILE); }

struct SolveWs {
  Pool pa, pb;
  int32_t *sel_slot, *new_slot, *sc, *free_list;
  uint32_t *sel_code, *cand, *hot0, *hot1;
  uint8_t *ok, *mark;
  double *alo, *ahi, *tab, *clb, *l, *u, *root_out, *f_search;
  int32_t* search_rounds;
  char* search_ws;
  size_t search_bytes;
  uint64_t *desc, *desc2, *cnt;
  uint32_t* tile_ctr;
  Ctl* ctl;
  unsigned int* hist;
  double* ppart;
  unsigned int* pticket;
  uint32_t* pot;
  uint64_t* pbits;
  ChainBufs chain;
};

// blocks of the chain kernel (one per SM) and its slice of the variables
static int chain_grid() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char* e = std::getenv("IBNB_CHAIN_GRID")) sms = std::max(16, std::min(sms, std::atoi(e)));
  return sms;
}
static int chain_per(int n) { return (n + chain_grid() - 1) / chain_grid(); }
// the cluster form of the chain (chainc.cuh): CS CTAs with DSMEM exchange;
// IBNB_CHAIN=2 selects it (the grid form is the default), IBNB_CHAIN_CS=8 a
// cluster of 8
static int chain_cs() {
  if (const char* e = std::getenv("IBNB_CHAIN_CS")) return std::atoi(e) == 8 ? 8 : 16;
  return 16;
}
static bool chainc_applies(const Problem& P) {
  const char* e = std::getenv("IBNB_CHAIN");
  if (!e || std::atoi(e) != 2 || P.fid == 6) return false;  // opt-in (IBNB_CHAIN=2); not the Levy chain sum
  const int cs = chain_cs();
  const int per = (P.n + cs - 1) / cs;
  return chainc_smem(per) <= 185u * 1024u;
}
// the chain kernel applies (chain.cuh): bisection, the next chunk disjoint
// from the current one, a non-chain objective, the slices in shared memory
static bool chain_applies(const Problem& P) {
  if (const char* e = std::getenv("IBNB_CHAIN"))
    if (std::atoi(e) == 0) return false;
  // Levy (fid 6, a chain sum, R11): n >= 3d + 2 keeps the chunk's neighbours
  // out of the next and the previous chunk
  const long nmin = P.fid == 6 ? 3L * P.d + 2 : 2L * P.d;
  return P.m == 2 && P.n >= nmin && P.d >= 2 && 16L * chain_per(P.n) <= 110L * 1024;
}

static size_t layout(const Opts& o, int n, Arena& A, SolveWs& w) {
  // Order matters for the latency-bound small-batch regime: the control
  // block and every small per-iteration array come first and share a few
  // 2 MB pages (TLB reach), then the per-iteration child arrays, then the
  // hot index, the list L and the archive (the large, sparsely touched
  // regions) and the search workspace.
  const long kids_tot = o.bmax * o.kids;
  w.ctl = A.take<Ctl>(1);
  w.cnt = A.take<uint64_t>(4);
  w.tile_ctr = A.take<uint32_t>(4);
  w.hist = A.take<unsigned int>(16 * 256);
  w.sel_slot = A.take<int32_t>(o.bmax);
  w.sel_code = A.take<uint32_t>(o.bmax);
  w.new_slot = A.take<int32_t>(o.bmax);
  w.ppart = A.take<double>((size_t)o.bmax * prep_slices(n, o.bmax) * 10);
  w.pticket = A.take<unsigned int>(o.bmax);
  w.pot = A.take<uint32_t>(PCAP);
  w.pbits = A.take<uint64_t>((size_t)(kids_tot + 63) / 64 + 8);
  w.chain.cnt = A.take<unsigned long long>(3);
  w.chain.gacc = A.take<unsigned long long>(3);
  w.chain.pcode = A.take<uint32_t>(3 * PCAP);
  w.chain.plb = A.take<double>(3 * PCAP);
  w.chain.pw = A.take<double>(3 * PCAP);
  w.chain.part = A.take<double>((size_t)2 * chain_grid() * CH_PART);
  w.chain.tabn = A.take<double>((size_t)2 * DM_MAX * ENT);
  w.chain.exits = A.take<unsigned long long>(8);
  w.chain.per = chain_per(n);
  w.chain.grid = chain_grid();
  w.root_out = A.take<double>(2);
  w.f_search = A.take<double>(1);
  w.search_rounds = A.take<int32_t>(1);
  w.l = A.take<double>(n);
  w.u = A.take<double>(n);
  w.tab = A.take<double>((size_t)o.bmax * o.tab_stride);
  long tiles = tiles_of(std::max({o.pool_cap, kids_tot, o.arch_cap})) + 2;
  w.desc = A.take<uint64_t>((size_t)tiles * 3);
  w.desc2 = A.take<uint64_t>((size_t)tiles * 3);
  w.clb = A.take<double>((size_t)kids_tot);
  w.cand = A.take<uint32_t>((size_t)kids_tot);
  w.ok = A.take<uint8_t>((size_t)kids_tot);
  w.hot0 = A.take<uint32_t>(o.pool_cap);
  w.hot1 = A.take<uint32_t>(o.pool_cap);
  auto pool = [&](Pool& p) {
    p.lb = A.take<double>(o.pool_cap);
    p.w = A.take<double>(o.pool_cap);
    p.slot = A.take<int32_t>(o.pool_cap);
    p.code = A.take<uint32_t>(o.pool_cap);
  };
  pool(w.pa);
  pool(w.pb);
  w.sc = A.take<int32_t>(o.arch_cap);
  w.free_list = A.take<int32_t>(o.arch_cap);
  w.mark = A.take<uint8_t>(o.arch_cap);
  w.alo = A.take<double>((size_t)o.arch_cap * o.ld);
  w.ahi = A.take<double>((size_t)o.arch_cap * o.ld);
  w.search_bytes = search_ws_bytes(n, search_grid_max());
  w.search_ws = A.take<char>(w.search_bytes);
  return A.off + 256;
}

// per-class CUDA-event timing (opt.profile)
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  cudaEvent_t cur[IB_NPROF] = {};
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[next++];
  }
  void begin(int cls, cudaStream_t st) {
    if (!on || recs.size() > 60000) return;
    cur[cls] = ev();
    cudaEventRecord(cur[cls], st);
  }
  void end(int cls, cudaStream_t st) {
    if (!on || !cur[cls]) return;
    cudaEvent_t b = ev();
    cudaEventRecord(b, st);
    recs.push_back(Rec{cls, cur[cls], b});
    cur[cls] = nullptr;
  }
  void collect(ib_result* res) {
    for (auto& q : recs) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, q.a, q.b);
      res->t_ms[q.cls] += ms;
      res->launches[q.cls] += 1;
    }
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct Hook : IterHook {
  Prof* prof = nullptr;
  ib_exchange_fn xfn = nullptr;
  void* xuser = nullptr;
  double* xchg = nullptr;
  Ctl* ctl = nullptr;
  void begin(int cls, long, cudaStream_t st) override { prof->begin(cls, st); }
  void end(int cls, cudaStream_t st) override { prof->end(cls, st); }
  // the incumbent exchange runs once per chunk of iterations (see below), not
  // inside an iteration
  void exchange(cudaStream_t) override {}
};

// grid bound baked into a captured iteration: generous, so that one graph
// serves the whole solve in the common case
static long graph_bound_for(long pool_bound, unsigned long long pcount, long per_it, long cap) {
  long b = std::max(pool_bound, (long)(2 * pcount) + 8 * per_it);
  long p2 = 1;
  while (p2 < b) p2 <<= 1;  // round up to a power of two: fewer distinct graphs
  return std::min(p2, cap);
}

struct GraphKey {
  Problem P;
  const double* pool;
  void* ws;
  long bound;
  long list_hint;  // k_list grid size class
  long bmax, pool_cap, arch_cap;  // workspace layout
  const void* tstamp;              // trace counters (IBNB_TRACE) baked into the kernels' arguments
};
static bool same_problem(const Problem& a, const Problem& b) { return std::memcmp(&a, &b, sizeof(Problem)) == 0; }

// per-thread reusable host resources: pinned control block, private stream,
// instantiated iteration graphs
struct ThreadCache {
  Ctl* host = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;
  struct Entry {
    GraphKey k;
    cudaGraphExec_t ge;
  };
  std::vector<Entry> graphs;
  cudaGraphExec_t find(const GraphKey& k, long need_bound) {
    for (auto& e : graphs)
      if (same_problem(e.k.P, k.P) && e.k.pool == k.pool && e.k.ws == k.ws && e.k.bmax == k.bmax &&
          e.k.list_hint == k.list_hint && e.k.tstamp == k.tstamp &&
          e.k.pool_cap == k.pool_cap && e.k.arch_cap == k.arch_cap && e.k.bound >= need_bound)
        return e.ge;
    return nullptr;
  }
  void put(const GraphKey& k, cudaGraphExec_t ge) {
    if (graphs.size() >= 8) {
      cudaGraphExecDestroy(graphs.front().ge);
      graphs.erase(graphs.begin());
    }
    graphs.push_back(Entry{k, ge});
  }
};
static ThreadCache& thread_cache() {
  static thread_local ThreadCache tc;
  return tc;
}

static int solve_impl(int fid, int n, const double* l_dev, const double* u_dev, const double* l_host,
                      const double* u_host, double eps_f, double eps_x, const ib_options* opt, void* ws,
                      size_t ws_bytes, ib_result* res, double* so_lo, double* so_hi, double* so_lb,
                      int64_t surv_cap, bool host_out, cudaStream_t user_st, ib_exchange_fn xfn, void* xuser,
                      double* xchg, ib_transfer_fn tfn = nullptr, int rank = 0, double* tbuf = nullptr,
                      size_t tbuf_bytes = 0) {
  Opts o;
  int rc = resolve_opts(fid, n, opt, 0, o);
  if (rc) return rc;
  if (!res) return fail(IB_EINVAL, "res is NULL");
  if (xfn && !xchg) return fail(IB_EINVAL, "exchange buffer is NULL");
  if (tfn && (!xfn || !tbuf || rank < 0 || rank > 1023)) return fail(IB_EINVAL, "rebalancing needs xfn, tbuf, 0 <= rank < 1024");
  std::memset(res, 0, sizeof(*res));
  Arena A{(char*)ws, 0, ws_bytes, false};
  SolveWs w;
  size_t need = layout(o, n, A, w);
  if (!ws || ws_bytes < need) return fail(IB_ENOSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  Problem P = make_problem(fid, n, o.d, o.m, o.kids, o.ld, o.mono, w.l, w.u, o.bmax);
  Prof prof;
  prof.on = opt && opt->profile == 1;
  const bool use_graph = !prof.on;
  // graph capture needs a non-legacy stream: work on a private stream (cached
  // per thread) ordered after the caller's stream (the call is synchronous)
  cudaStream_t st = user_st;
  ThreadCache& tc = thread_cache();
  if (!tc.host) CK(cudaMallocHost(&tc.host, sizeof(Ctl)));
  if (use_graph) {
    if (!tc.stream) CK(cudaStreamCreateWithFlags(&tc.stream, cudaStreamNonBlocking));
    if (!tc.ev) CK(cudaEventCreateWithFlags(&tc.ev, cudaEventDisableTiming));
    CK(cudaEventRecord(tc.ev, user_st));
    CK(cudaStreamWaitEvent(tc.stream, tc.ev, 0));
    st = tc.stream;
  }
  struct SyncOnExit {
    cudaStream_t s;
    ~SyncOnExit() { cudaStreamSynchronize(s); }
  } sync_on_exit{st};
  Ctl* hctl = tc.host;
  const bool trace = std::getenv("IBNB_TRACE") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = trace ? now() : 0.0;
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
  Ctl& hc = *hctl;
  std::memset(&hc, 0, sizeof hc);
  hc.gub_key = okey_h(INFINITY);
  hc.free_top = (unsigned long long)(o.arch_cap - 1);
  hc.eps_f = eps_f;
  hc.eps_x = eps_x;
  hc.bmax = (unsigned long long)o.bmax;
  hc.max_iter = (unsigned long long)o.max_iter;
  hc.pool_cap = (unsigned long long)o.pool_cap;
  hc.acc_min_key = hc.acc_min_key2 = hc.acc_min_key3 = ~0ull;
  hc.tau_key = ~0ull;
  hc.hot_valid = 0;  // built by the first iteration's refill
  hc.hot_target = (unsigned long long)(8 * o.bmax + 16384);
  CK(cudaMemcpyAsync(w.ctl, &hc, sizeof hc, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(w.hist, 0, 16 * 256 * sizeof(unsigned int), st));
  CK(cudaMemsetAsync(w.pticket, 0, sizeof(unsigned int) * o.bmax, st));
  CK(cudaMemcpyAsync(w.alo, w.l, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(w.ahi, w.u, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(w.sc, 0, sizeof(int32_t), st));
  CKL(launch_eval_boxes(fid, n, 1, w.alo, w.ahi, o.ld, w.root_out, st));
  k_root<<<1, 1, 0, st>>>(w.root_out, w0, w.pa, w.ctl);
  // free list: slots 1 .. arch_cap-1
  k_iota32<<<blocks_for(o.arch_cap - 1), 256, 0, st>>>(w.free_list, o.arch_cap - 1, 1);
  nk += 3;
  // sampling (line 134, reading R9): the coordinate pattern search supplies
  // the initial incumbent GUB (ordered-int atomicMin into ctl->gub_key)
  double f_search = INFINITY;
  int32_t search_rounds = 0;
  if (o.search > 0) {
    CKL(launch_search(fid, n, w.l, w.u, o.search, w.search_ws, w.search_bytes, &w.ctl->gub_key, nullptr, w.f_search,
                      w.search_rounds, st));
    CK(cudaMemcpyAsync(&f_search, w.f_search, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&search_rounds, w.search_rounds, 4, cudaMemcpyDeviceToHost, st));
    nk += 1;
  }

  IterBufs ib{};
  ib.ctl = w.ctl;
  ib.hist = w.hist;
  ib.sel_slot = w.sel_slot;
  ib.sel_code = w.sel_code;
  ib.new_slot = w.new_slot;
  ib.free_list = w.free_list;
  ib.src_lo = w.alo;
  ib.src_hi = w.ahi;
  ib.src_sc = w.sc;
  ib.dst_lo = w.alo;
  ib.dst_hi = w.ahi;
  ib.dst_sc = w.sc;
  ib.tab = w.tab;
  ib.tab_stride = o.tab_stride;
  ib.clb = w.clb;
  ib.cand = w.cand;
  ib.ok = w.ok;
  ib.desc = w.desc;
  ib.desc2 = w.desc2;
  ib.tile_ctr = w.tile_ctr;
  ib.hot0 = w.hot0;
  ib.hot1 = w.hot1;
  ib.ppart = w.ppart;
  ib.pticket = w.pticket;
  ib.pot = w.pot;
  ib.pbits = w.pbits;
  if (const char* e = std::getenv("IBNB_SPARSE"))  // 0: always the dense insertion (A/B measurements)
    if (std::atoi(e) == 0) ib.pbits = nullptr;
  unsigned long long* tstamp = nullptr;
  if (trace) {
    CK(cudaMalloc(&tstamp, 32 * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(tstamp, 0, 32 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(w.chain.exits, 0, 8 * sizeof(unsigned long long), st));
    ib.tstamp = tstamp;
  }
  struct FreeOnExit {
    unsigned long long* p;
    ~FreeOnExit() { if (p) cudaFree(p); }
  } free_tstamp{tstamp};
  Hook hook;
  hook.prof = &prof;
  hook.xfn = xfn;
  hook.xuser = xuser;
  hook.xchg = xchg;
  hook.ctl = w.ctl;
  const int kIterKernels = 4;  // kernels per iteration (launch_iteration)

  // fused-kernel thresholds (IBNB_FUSE_KIDS / IBNB_FUSE_POOL override; 0 = off)
  long fuse_kids = 1L << 20, fuse_pool = 1L << 16;
  if (const char* e = std::getenv("IBNB_FUSE_KIDS")) fuse_kids = std::atol(e);
  if (const char* e = std::getenv("IBNB_FUSE_POOL")) fuse_pool = std::atol(e);
  unsigned long long pcount = 1, free_top = hc.free_top, peak = 1;
  long fused_iters = 0, chain_iters = 0, iter_prev = 0, chain_launches = 0;
  const bool use_chain = chain_applies(P);
  w.chain.gshared = opt ? reinterpret_cast<unsigned long long*>(opt->gub_shared) : nullptr;
  const bool use_chainc = use_chain && chainc_applies(P) && !w.chain.gshared;
  ChainBufs cbc = w.chain;
  cbc.per = (n + chain_cs() - 1) / chain_cs();
  // iterations per chain launch: the host reads the control block between
  // launches (multi-GPU: the incumbent exchange runs there)
  long chain_budget = xfn ? 64 : 4096;
  if (const char* e = std::getenv("IBNB_CHAIN_ITERS")) chain_budget = std::max(1L, std::atol(e));
  long chunk = 1;
  for (;;) {
    const long per_it = o.bmax * o.kids;
    // capacity planning for the chunk: shorten it to what L can take in the
    // worst case (every child survives), compact L only when even one
    // iteration might not fit, collect archive slots when short
    chunk = std::max(1L, std::min(chunk, (o.pool_cap - (long)pcount) / std::max(1L, per_it)));
    if ((long)pcount + chunk * per_it > o.pool_cap) {
      // compact L: keep the live records (lb <= GUB), list order preserved
      CKL(launch_partition(w.pa, (long)pcount, &w.ctl->gub_key, 64, 0ull, 0ull, nullptr, nullptr, nullptr, w.pb,
                           w.desc, w.tile_ctr, w.cnt, st));
      k_set_pcount<<<1, 1, 0, st>>>(w.ctl, w.cnt);
      nk += 2;
      std::swap(w.pa, w.pb);
      CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      pcount = hc.pcount;
      if ((long)pcount + per_it > o.pool_cap)
        return fail(IB_ENOSPACE, "list L capacity %ld exceeded (%llu live + %ld children)", o.pool_cap, pcount,
                    per_it);
      chunk = std::max(1L, std::min(chunk, (o.pool_cap - (long)pcount) / per_it));
    }
    if ((long)free_top < chunk * o.bmax) {
      CKL(launch_gc(w.pa, w.ctl, (long)pcount, w.mark, o.arch_cap, w.free_list, w.desc, w.tile_ctr, st));
      nk += 2;
      CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      free_top = hc.free_top;
      if ((long)free_top < o.bmax) return fail(IB_ENOSPACE, "archive full (%ld slots)", o.arch_cap);
      chunk = std::max(1L, std::min(chunk, (long)free_top / o.bmax));
    }
    ib.pool = w.pa;
    if (w.chain.gshared) {
      k_gub_shared<<<1, 1, 0, st>>>(w.ctl, w.chain.gshared);
      nk += 1;
    }
    const long pool_bound = (long)pcount + chunk * per_it;
    // k_list grid class from the records L holds now: two classes, so that
    // the cached iteration graphs do not multiply
    const long list_hint = (long)pcount <= 65536 ? 65536 : (1L << 40);
    // small batches: whole iterations in one persistent cooperative kernel;
    // the deep dive (one live region, one survivor per iteration) as a chain
    const bool fused = o.bmax * o.kids <= fuse_kids && (long)pcount <= fuse_pool;
    const bool chain = use_chain && hc.list_fast && hc.nhot == 1 && !hc.pending_end &&
                       (long)free_top >= 2 && (long)pcount + o.kids <= o.pool_cap;
    if (chain) {
      prof.begin(7, st);
      if (use_chainc) CKL(launch_chainc(P, ib, cbc, chain_cs(), (int)chain_budget, st));
      else CKL(launch_chain(P, ib, w.chain, (int)chain_budget, st));
      prof.end(7, st);
      nk += 1 - chunk * kIterKernels;
      ++chain_launches;
    } else if (fused) {
      prof.begin(6, st);
      CKL(launch_fused(P, ib, (int)chunk, o.bmax, st));
      prof.end(6, st);
      nk += 1 - chunk * kIterKernels;  // one launch for the chunk
    } else if (use_graph) {
      // one captured iteration per (problem, buffers, grid bound), cached per
      // thread and replayed; re-captured when its grid bound is exceeded
      GraphKey key{P, ib.pool.lb, ws, graph_bound_for(pool_bound, pcount, per_it, o.pool_cap), list_hint, o.bmax,
                   o.pool_cap, o.arch_cap, ib.tstamp};
      cudaGraphExec_t ge = tc.find(key, pool_bound);
      if (!ge) {
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int lr = launch_iteration(P, ib, key.bound, o.bmax, st, nullptr, list_hint);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (lr) return fail(lr, "capture of the iteration failed");
        CK(ce);
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        tc.put(key, ge);
        if (trace) fprintf(stderr, "[ibnb] captured iteration graph, bound %ld\n", key.bound);
      }
      for (long c = 0; c < chunk; ++c) CK(cudaGraphLaunch(ge, st));
    } else {
      for (long c = 0; c < chunk; ++c) CKL(launch_iteration(P, ib, pool_bound, o.bmax, st, &hook, list_hint));
    }
    nk += chunk * kIterKernels;
    // count the survivors of the chunk's last iteration (normally done by the
    // next iteration's k_list) before the host looks at L
    CKL(launch_apply_pending(w.ctl, o.kids, st));
    nk += 1;
    if (xfn) {
      // multi-GPU incumbent exchange, once per chunk (<= 64 iterations): the
      // caller's all-reduce(MIN) runs on the caller's stream, ordered between
      // the put and the take on the solve stream by events
      CKL(launch_xchg_put(w.ctl, xchg, st));
      if (st != user_st) {
        CK(cudaEventRecord(tc.ev, st));
        CK(cudaStreamWaitEvent(user_st, tc.ev, 0));
      }
      xfn(xuser);
      if (st != user_st) {
        CK(cudaEventRecord(tc.ev, user_st));
        CK(cudaStreamWaitEvent(st, tc.ev, 0));
      }
      CKL(launch_xchg_take(w.ctl, xchg, st));
      nk += 2;
      if (tfn) {
        // list sizes under the shared incumbent, for the rebalancing
        // decision: a second MIN exchange (GUB and flag entries unchanged)
        CK(cudaMemsetAsync(w.cnt + 3, 0, 8, st));
        k_count_live<<<148 * 4, 256, 0, st>>>(w.pa, w.ctl, (unsigned long long*)(w.cnt + 3));
        k_live_key<<<1, 1, 0, st>>>((unsigned long long*)(w.cnt + 3), rank, xchg);
        nk += 2;
        if (st != user_st) {
          CK(cudaEventRecord(tc.ev, st));
          CK(cudaStreamWaitEvent(user_st, tc.ev, 0));
        }
        xfn(xuser);
        if (st != user_st) {
          CK(cudaEventRecord(tc.ev, user_st));
          CK(cudaStreamWaitEvent(st, tc.ev, 0));
        }
      }
    }
    double xh[4] = {0, 0, 0, 0};
    if (tfn) CK(cudaMemcpyAsync(xh, xchg, sizeof xh, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    pcount = hc.pcount;
    free_top = hc.free_top;
    peak = std::max(peak, pcount);
    if (tfn && !hc.gdone) {
      // box rebalancing (north_star): when the largest list is more than twice
      // the smallest (+ 2 batches), its rank sends the last K of its live
      // regions to the rank with the smallest list.  Every rank takes the same
      // decision from the reduced values.
      const double kmax = -xh[2], kmin = xh[3];
      const long lmax = (long)(kmax / 1024.0), lmin = (long)(kmin / 1024.0);
      const int donor = (int)(kmax - 1024.0 * (double)lmax), recv = (int)(kmin - 1024.0 * (double)lmin);
      const long per = 2L * n + 3;  // doubles per region in the transfer buffer
      long K = std::min((lmax - lmin) / 2, (long)(tbuf_bytes / (8 * (size_t)per)));
      K = std::min(K, std::min(o.pool_cap / 8, o.arch_cap / 8));
      if (donor != recv && lmax > 2 * lmin + 2 * o.bmax && K > 0) {
        double* t_lo = tbuf;
        double* t_hi = tbuf + (size_t)K * n;
        double* t_lb = tbuf + (size_t)2 * K * n;
        double* t_w = t_lb + K;
        double* t_cyc = t_w + K;
        if (rank == donor) {
          // compact the live records (list order kept), export the last K
          CKL(launch_partition(w.pa, (long)pcount, &w.ctl->gub_key, 64, 0ull, 0ull, nullptr, nullptr, nullptr, w.pb,
                               w.desc, w.tile_ctr, w.cnt, st));
          uint64_t live_c = 0;
          CK(cudaMemcpyAsync(&live_c, w.cnt, 8, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          std::swap(w.pa, w.pb);
          const long keep = (long)live_c - K;
          if (keep < 0) return fail(IB_EINVAL, "rebalancing: %ld live records, %ld to send", (long)live_c, K);
          Pool sub{w.pa.lb + keep, w.pa.w + keep, w.pa.slot + keep, w.pa.code + keep};
          CKL(launch_extract(P, sub, K, w.alo, w.ahi, w.sc, t_lo, t_hi, t_lb, st));
          k_export_meta<<<blocks_for(K), 256, 0, st>>>(w.pa, keep, K, w.sc, o.d, n, t_w, t_cyc);
          k_list_changed<<<1, 1, 0, st>>>(w.ctl, keep, 0);
          nk += 4;
          pcount = (unsigned long long)keep;
        }
        // the caller moves K regions from the donor's tbuf to the receiver's
        if (st != user_st) {
          CK(cudaEventRecord(tc.ev, st));
          CK(cudaStreamWaitEvent(user_st, tc.ev, 0));
        }
        tfn(xuser, donor, recv, tbuf, (size_t)(8 * per * K));
        if (st != user_st) {
          CK(cudaEventRecord(tc.ev, user_st));
          CK(cudaStreamWaitEvent(st, tc.ev, 0));
        }
        if (rank == recv) {
          if ((long)free_top < K + o.bmax) {
            CKL(launch_gc(w.pa, w.ctl, (long)pcount, w.mark, o.arch_cap, w.free_list, w.desc, w.tile_ctr, st));
            CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            free_top = hc.free_top;
            nk += 2;
          }
          if ((long)free_top < K + o.bmax || (long)pcount + K > o.pool_cap)
            return fail(IB_ENOSPACE, "rebalancing: no room for %ld received regions", K);
          k_import<<<(unsigned)std::min(K, 148L * 8), 128, 0, st>>>(w.pa, w.ctl, t_lo, t_hi, t_lb, t_w, t_cyc, K, n,
                                                                    o.ld, w.alo, w.ahi, w.sc, w.free_list);
          k_list_changed<<<1, 1, 0, st>>>(w.ctl, (long)pcount + K, K);
          nk += 2;
          pcount += (unsigned long long)K;
          free_top -= (unsigned long long)K;
        }
        CK(cudaStreamSynchronize(st));
        res->rebalanced += (rank == donor ? -K : (rank == recv ? K : 0));
        res->transfers += 1;
      }
    }
    if (chain) chain_iters += (long)hc.iter - iter_prev;
    else if (fused) fused_iters += (long)hc.iter - iter_prev;
    iter_prev = (long)hc.iter;
    if (hc.err) return fail(hc.err, "capacity exceeded on the device (L %ld, archive %ld)", o.pool_cap, o.arch_cap);
    if (trace)
      fprintf(stderr, "[ibnb] t=%.3f ms %s chunk=%ld iter=%llu |L|=%llu live_hot=%llu nhot=%llu B=%llu refills=%llu "
              "width_passes=%llu done=%d\n", now() - t_start, chain ? "chain" : (fused ? "fused" : "graph"), chunk,
              hc.iter, hc.pcount, hc.live, hc.nhot, hc.B, hc.nrefill, hc.nwidth, hc.done);
    if (xfn ? hc.gdone : hc.done) break;
    chunk = std::min(chunk * 2, 64L);
    // lazy deletion leaves selected / ruled-out records in L: compact when a
    // refill of the hot index found it more than half dead
    if (hc.compact_hint && (long)pcount > (1L << 18)) {
      CKL(launch_partition(w.pa, (long)pcount, &w.ctl->gub_key, 64, 0ull, 0ull, nullptr, nullptr, nullptr, w.pb,
                           w.desc, w.tile_ctr, w.cnt, st));
      k_set_pcount<<<1, 1, 0, st>>>(w.ctl, w.cnt);
      nk += 2;
      std::swap(w.pa, w.pb);
      CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      pcount = hc.pcount;
      if (trace) fprintf(stderr, "[ibnb] compacted L -> %llu records\n", pcount);
    }
  }
  if (trace && tstamp) {
    unsigned long long tsh[32];
    CK(cudaMemcpyAsync(tsh, tstamp, sizeof tsh, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const char* ph[6] = {"list", "prep", "child_eval", "cand", "mono", "emit"};
    double it = (double)std::max(1ull, tsh[6]);
    fprintf(stderr, "[ibnb] fused phases over %llu iterations (us/iter):", tsh[6]);
    for (int k = 0; k < 6; ++k) fprintf(stderr, " %s=%.2f", ph[k], tsh[k] / it / 1e3);
#ifdef IBNB_PROBE
    {
      extern int probe_read(unsigned long long*);
      unsigned long long pr[64];
      if (probe_read(pr) == 0) {
        fprintf(stderr, "\n[ibnb] probes (cycles/iter):");
        for (int k = 0; k < 64; ++k)
          if (pr[k]) fprintf(stderr, " p%d=%.0f", k, pr[k] / it);
      }
    }
#endif
    fprintf(stderr, "\n[ibnb] slowest block's own work per phase (us/iter):");
    for (int k = 0; k < 6; ++k) fprintf(stderr, " %s=%.2f", ph[k], tsh[8 + k] / it / 1e3);
    unsigned long long ex[8];
    CK(cudaMemcpyAsync(ex, w.chain.exits, sizeof ex, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const char* why[7] = {"no_survivor", "several_survivors", "over_pcap", "stop", "max_iter", "budget", "entry"};
    if (tsh[31])
      fprintf(stderr, "\n[ibnb] chain phases over %llu iterations (us/iter, block 0): children=%.2f slice=%.2f "
              "barrier=%.2f candidates=%.2f next_table=%.2f", tsh[31], tsh[26] / 1e3 / tsh[31], tsh[27] / 1e3 / tsh[31],
              tsh[28] / 1e3 / tsh[31], tsh[29] / 1e3 / tsh[31], tsh[30] / 1e3 / tsh[31]);
    fprintf(stderr, "\n[ibnb] chain launches %ld, exits:", chain_launches);
    for (int k = 0; k < 7; ++k) fprintf(stderr, " %s=%llu", why[k], ex[k]);
    if (tsh[31]) fprintf(stderr, " potential_children_per_iter=%.2f listed_per_iter=%.2f", (double)ex[7] / tsh[31],
                         (double)tsh[25] / tsh[31]);
    if (tsh[17] + tsh[19])
      fprintf(stderr, "\n[ibnb] chain phase 1 per block (us): slice/entry blocks %.2f (%llu), children blocks %.2f (%llu)",
              tsh[16] / 1e3 / std::max(1ull, tsh[17]), tsh[17], tsh[18] / 1e3 / std::max(1ull, tsh[19]), tsh[19]);
    if (tsh[22])
      fprintf(stderr, "\n[ibnb] k_insert launches %llu, sparse %llu, potential candidates per launch %.1f", tsh[22],
              tsh[23], (double)tsh[24] / (double)tsh[22]);
    fprintf(stderr, "\n");
  }
  // exact max width of the remaining regions for the result
  CKL(launch_final_width(w.pa, w.ctl, (long)pcount, st));
  nk += 2;
  CK(cudaMemcpyAsync(&hc, w.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const Ctl c = hc;
  int status;
  switch (c.done) {
    case 1: status = IB_STATUS_CONVERGED; break;
    case 2: status = IB_STATUS_MAX_ITER; break;
    default: status = (xfn || w.chain.gshared) ? IB_STATUS_EMPTY : IB_EEMPTY; break;
  }
  if (status == IB_EEMPTY) return fail(IB_EEMPTY, "list L became empty after %llu iterations", c.iter);
  // output (line 150): GLB, GUB and the live regions of L, in list order
  CKL(launch_partition(w.pa, (long)pcount, &w.ctl->gub_key, 64, 0ull, 0ull, nullptr, nullptr, nullptr, w.pb, w.desc,
                       w.tile_ctr, w.cnt, st));
  nk += 1;
  uint64_t live_all = 0;  // every live region of L (hot and cold)
  CK(cudaMemcpyAsync(&live_all, w.cnt, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const long live = (long)live_all;
  const long ncopy = std::min((long)surv_cap, live);
  if (so_lo && so_hi && ncopy > 0) {
    if (host_out) {
      // stage through the (unused) child-bound buffer, in chunks; when it
      // cannot hold one region (very large n, small batches) a staging buffer
      // is allocated for the copy
      const size_t need1 = 2 * (size_t)n + 1, cap_d = (size_t)o.bmax * o.kids;
      double* tlo = w.clb;
      size_t stage_d = cap_d;
      struct Owned {
        double* p = nullptr;
        cudaStream_t s;
        ~Owned() { if (p) cudaFreeAsync(p, s); }
      } owned{nullptr, st};
      if (cap_d < need1) {
        stage_d = need1 * (size_t)std::min(ncopy, 16L);
        CK(cudaMallocAsync((void**)&owned.p, sizeof(double) * stage_d, st));
        tlo = owned.p;
      }
      const long per = std::max(1L, (long)(stage_d / need1));
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
  res->units[0] = (int64_t)c.sum_B;      // prep: parents
  res->units[1] = (int64_t)c.evals;      // child_eval: children
  res->units[2] = (int64_t)c.evals;      // cand: children scanned
  res->units[3] = (int64_t)c.list_bytes;  // list: algorithmic bytes (hot scans, refills, width passes)
  res->units[4] = (int64_t)c.sum_cand;   // mono: candidates tested
  res->units[5] = (int64_t)c.sum_cand;   // emit: candidates scanned
  res->units[6] = (int64_t)fused_iters;  // fused: iterations run inside k_fused
  res->units[7] = (int64_t)chain_iters;  // chain: iterations run inside k_chain
  res->radix_records = (int64_t)c.sum_radix;
  res->f_lo = live ? okey_inv_h(c.min_lb_key) : INFINITY;
  res->f_hi = okey_inv_h(c.gub_key);
  res->iters = (int64_t)c.iter;
  res->evals = (int64_t)c.evals;
  res->n_surv = live;
  res->peak_pool = (int64_t)peak;
  std::memcpy(&res->max_width, &c.acc_max_w, 8);
  res->status = status;
  res->n_kernels = (int)std::min(nk, (long)INT32_MAX);
  res->f_search = f_search;
  res->search_rounds = search_rounds;
  return 0;
}

}  // namespace ib

using namespace ib;

extern "C" {

const char* ib_version(void) { return "ibnb 0.3.0 (sm_100a, fp64 directed rounding, device-driven iteration)"; }

int ib_ipc_get_handle(const void* dptr, void* handle) {
  if (!dptr || !handle) return fail(IB_EINVAL, "ib_ipc_get_handle: NULL argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dptr));
  if (e != cudaSuccess) return fail((int)e, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, sizeof h);
  return 0;
}

int ib_ipc_open(const void* handle, void** dptr) {
  if (!dptr || !handle) return fail(IB_EINVAL, "ib_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail((int)e, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return 0;
}

int ib_ipc_close(void* dptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  if (e != cudaSuccess) return fail((int)e, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return 0;
}
const char* ib_last_error(void) { return g_err.c_str(); }
int ib_num_functions(void) { return 11; }

size_t ib_solve_workspace_size(int fid, int n, const ib_options* opt, int64_t pool_cap) {
  Opts o;
  if (resolve_opts(fid, n, opt, pool_cap, o)) return 0;
  Arena A{nullptr, 0, 0, true};
  SolveWs w;
  return layout(o, n, A, w);
}

int ib_solve(int fid, int n, const double* l, const double* u, double eps_f, double eps_x, const ib_options* opt,
             void* ws, size_t ws_bytes, ib_result* res, double* surv_lo, double* surv_hi, double* surv_lb,
             int64_t surv_cap, void* stream) {
  if (!l || !u) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, nullptr, nullptr, l, u, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo, surv_hi, surv_lb,
                    surv_cap, true, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

int ib_solve_dev(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                 const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo, double* surv_hi,
                 double* surv_lb, int64_t surv_cap, void* stream) {
  if (!l_dev || !u_dev) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, l_dev, u_dev, nullptr, nullptr, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo, surv_hi,
                    surv_lb, surv_cap, false, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

int ib_solve_dev_ex(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                    const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                    double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream, ib_exchange_fn fn, void* user,
                    double* xchg) {
  if (!l_dev || !u_dev) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, l_dev, u_dev, nullptr, nullptr, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo, surv_hi,
                    surv_lb, surv_cap, false, (cudaStream_t)stream, fn, user, xchg);
}

int ib_solve_dev_mg(int fid, int n, const double* l_dev, const double* u_dev, double eps_f, double eps_x,
                    const ib_options* opt, void* ws, size_t ws_bytes, ib_result* res, double* surv_lo,
                    double* surv_hi, double* surv_lb, int64_t surv_cap, void* stream, ib_exchange_fn fn,
                    ib_transfer_fn tfn, void* user, double* xchg, int rank, double* tbuf, size_t tbuf_bytes) {
  if (!l_dev || !u_dev) return fail(IB_EINVAL, "l/u NULL");
  g_err.clear();
  return solve_impl(fid, n, l_dev, u_dev, nullptr, nullptr, eps_f, eps_x, opt, ws, ws_bytes, res, surv_lo, surv_hi,
                    surv_lb, surv_cap, false, (cudaStream_t)stream, fn, user, xchg, tfn, rank, tbuf, tbuf_bytes);
}

int ib_eval_boxes(int fid, int n, int64_t nbox, const double* lo, const double* hi, int64_t ld, double* out,
                  void* stream) {
  if (fid < 0 || fid > 10 || n < 1 || nbox < 0 || ld < n || (!lo && nbox) || (!hi && nbox) || (!out && nbox))
    return fail(IB_EINVAL, "ib_eval_boxes: bad arguments");
  CKL(launch_eval_boxes(fid, n, (long)nbox, lo, hi, (long)ld, out, (cudaStream_t)stream));
  return 0;
}

int ib_eval_grad(int fid, int n, int64_t nreq, const double* lo, const double* hi, int64_t ld, const int64_t* req_box,
                 const int32_t* req_dim, double* out, void* stream) {
  if (fid < 0 || fid > 10 || n < 1 || nreq < 0 || ld < n) return fail(IB_EINVAL, "ib_eval_grad: bad arguments");
  CKL(launch_eval_grad(fid, n, (long)nreq, lo, hi, (long)ld, req_box, req_dim, out, (cudaStream_t)stream));
  return 0;
}

struct BranchWs {
  int32_t *iota, *dst_sc;
  uint32_t *whole, *cand;
  uint8_t* ok;
  double *dlo, *dhi, *tab, *clb;
  uint64_t *desc, *desc2;
  uint32_t* tile_ctr;
  Ctl* ctl;
  double* ppart;
  unsigned int* pticket;
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
  w.cand = A.take<uint32_t>((size_t)nb * kids);
  w.ok = A.take<uint8_t>((size_t)nb * kids);
  w.desc = A.take<uint64_t>((size_t)tiles_of(nb * kids) + 2);
  w.desc2 = A.take<uint64_t>((size_t)2 * tiles_of(nb * kids) + 4);
  w.tile_ctr = A.take<uint32_t>(4);
  w.ctl = A.take<Ctl>(1);
  w.ppart = A.take<double>((size_t)nb * prep_slices(n, nb) * 10);
  w.pticket = A.take<unsigned int>(nb);
  return A.off + 256;
}

size_t ib_branch_workspace_size(int fid, int n, int d, int m, int64_t nb) {
  (void)fid;
  if (n < 1 || d < 1 || d > n || d > D_MAX || m < 2 || m > M_MAX || d * m > DM_MAX || nb < 0) return 0;
  Arena A{nullptr, 0, 0, true};
  BranchWs w;
  return branch_layout(n, d, m, (long)nb, A, w);
}

int ib_branch(int fid, int n, int d, int m, int mono, int64_t nb, const double* plo, const double* phi, int64_t ld,
              const int32_t* pcyc, const double* l, const double* u, double* gub, void* ws, size_t ws_bytes,
              int32_t* out_parent, uint32_t* out_code, double* out_lb, double* out_w, int64_t* out_count,
              void* stream) {
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
  Problem P = make_problem(fid, n, d, m, kids, ldi, mono ? 1 : 0, l, u, (long)nb);
  k_iota32<<<blocks_for(nb), 256, 0, st>>>(w.iota, nb, 0);
  k_fill_u32<<<blocks_for(nb), 256, 0, st>>>(w.whole, nb, CODE_WHOLE);
  k_branch_ctl<<<1, 1, 0, st>>>(w.ctl, gub, nb, nb * kids);
  CK(cudaMemsetAsync(w.pticket, 0, sizeof(unsigned int) * nb, st));
  if ((int)ld != ldi) {
    // bring the parents to our even row stride first
    CK(cudaMemcpy2DAsync(w.dlo, sizeof(double) * ldi, plo, sizeof(double) * ld, sizeof(double) * n, nb,
                         cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpy2DAsync(w.dhi, sizeof(double) * ldi, phi, sizeof(double) * ld, sizeof(double) * n, nb,
                         cudaMemcpyDeviceToDevice, st));
    plo = w.dlo;
    phi = w.dhi;
  }
  IterBufs ib{};
  ib.ctl = w.ctl;
  ib.pool = Pool{out_lb, out_w, out_parent, out_code};
  ib.sel_slot = w.iota;
  ib.sel_code = w.whole;
  ib.new_slot = w.iota;
  ib.src_lo = plo;
  ib.src_hi = phi;
  ib.src_sc = pcyc;
  ib.dst_lo = w.dlo;
  ib.dst_hi = w.dhi;
  ib.dst_sc = w.dst_sc;
  ib.tab = w.tab;
  ib.tab_stride = HDR + d * m * ENT;
  ib.clb = w.clb;
  ib.cand = w.cand;
  ib.ok = w.ok;
  ib.desc = w.desc;
  ib.desc2 = w.desc2;
  ib.tile_ctr = w.tile_ctr;
  ib.ppart = w.ppart;
  ib.pticket = w.pticket;
  CKL(launch_branch(P, ib, (long)nb, st));
  k_branch_out<<<1, 1, 0, st>>>(w.ctl, gub, out_count);
  CK(cudaGetLastError());
  return 0;
}

size_t ib_search_workspace_size(int n) {
  if (n < 1) return 0;
  return search_ws_bytes(n, search_grid_max());
}

int ib_search(int fid, int n, const double* l, const double* u, int rounds, double* x_out, double* f_out,
              int32_t* rounds_out, void* ws, size_t ws_bytes, void* stream) {
  if (fid < 0 || fid > 10 || n < 1 || rounds < 0 || !l || !u || !ws) return fail(IB_EINVAL, "ib_search: bad arguments");
  if (ws_bytes < ib_search_workspace_size(n)) return fail(IB_ENOSPACE, "ib_search: workspace too small");
  CKL(launch_search(fid, n, l, u, rounds, ws, ws_bytes, nullptr, x_out, f_out, rounds_out, (cudaStream_t)stream));
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
  A.take<double>(n);    // w
  A.take<int32_t>(n);   // slot (iota)
  A.take<uint32_t>(n);  // code
  A.take<double>(n);    // keep lb
  A.take<double>(n);    // keep w
  A.take<int32_t>(n);   // keep slot
  A.take<uint32_t>(n);  // keep code
  A.take<int32_t>(n);   // sel slot
  A.take<uint64_t>((size_t)(n / TILE + 2) * 3);
  A.take<uint32_t>(4);
  A.take<Ctl>(1);
  A.take<unsigned int>(256);
  A.take<uint64_t>(2);
  return A.off + 256;
}

// selection step alone, with the same device statistics / radix-select
// kernels as a solve, then a stable partition with the resulting spec
int ib_select(const double* lb, int64_t n, double gub, int64_t bmax, int64_t* sel_idx, int64_t* keep_idx,
              int64_t* n_sel, int64_t* n_keep, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || bmax < 1 || !n_sel || !n_keep) return fail(IB_EINVAL, "ib_select: bad arguments");
  if (!ws || ws_bytes < ib_select_workspace_size(n)) return fail(IB_ENOSPACE, "ib_select: workspace too small");
  if (n == 0) {
    *n_sel = *n_keep = 0;
    return 0;
  }
  Arena A{(char*)ws, 0, ws_bytes, false};
  Pool in{const_cast<double*>(lb), A.take<double>(n), A.take<int32_t>(n), A.take<uint32_t>(n)};
  Pool keep{A.take<double>(n), A.take<double>(n), A.take<int32_t>(n), A.take<uint32_t>(n)};
  int32_t* sel_slot = A.take<int32_t>(n);
  uint64_t* desc = A.take<uint64_t>((size_t)(n / TILE + 2) * 3);
  uint32_t* tile_ctr = A.take<uint32_t>(4);
  Ctl* ctl = A.take<Ctl>(1);
  unsigned int* hist = A.take<unsigned int>(256);
  uint64_t* cnt = A.take<uint64_t>(2);
  k_fill_f64<<<blocks_for(n), 256, 0, st>>>(in.w, n, 0.0);
  k_iota32<<<blocks_for(n), 256, 0, st>>>(in.slot, n, 0);
  k_fill_u32<<<blocks_for(n), 256, 0, st>>>(in.code, n, 0u);
  Ctl hc;
  std::memset(&hc, 0, sizeof hc);
  hc.pcount = (unsigned long long)n;
  hc.gub_key = okey_h(gub);
  hc.eps_f = -1.0;  // never "converged"
  hc.eps_x = -1.0;
  hc.bmax = (unsigned long long)bmax;
  hc.max_iter = ~0ull;
  hc.pool_cap = (unsigned long long)n;
  hc.acc_min_key = ~0ull;
  hc.free_top = ~0ull;  // no archive in a bare selection
  CK(cudaMemcpyAsync(ctl, &hc, sizeof hc, cudaMemcpyHostToDevice, st));
  CKL(launch_select_only(in, ctl, hist, (long)n, st));
  CK(cudaMemcpyAsync(&hc, ctl, sizeof hc, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  long live = (long)hc.live;
  long B = std::min(live, (long)bmax);
  CKL(launch_partition(in, (long)n, &ctl->gub_key, hc.known, hc.prefix, hc.known == 0 ? 0ull : hc.need, sel_slot,
                       nullptr, nullptr, keep, desc, tile_ctr, cnt, st));
  if (B > 0) k_i32_to_i64<<<blocks_for(B), 256, 0, st>>>(sel_slot, B, sel_idx);
  if (live - B > 0) k_i32_to_i64<<<blocks_for(live - B), 256, 0, st>>>(keep.slot, live - B, keep_idx);
  CK(cudaStreamSynchronize(st));
  *n_sel = B;
  *n_keep = live - B;
  return 0;
}

}  // extern "C"
