// kernels.cuh -- device data layout shared by the kernels and the host
// runtime of the branch-and-bound hot path (no torch types anywhere).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ib {

constexpr uint32_t CODE_WHOLE = 0xffffffffu;  // record = the archived box itself
constexpr int D_MAX = 20;                       // split variables per iteration
constexpr int M_MAX = 8;                        // pieces per split variable
constexpr int DM_MAX = 64;                      // d * m table entries per parent
constexpr int HDR = 56;                         // doubles of per-parent header
constexpr int ENT = 24;                         // doubles per (variable, piece) entry
constexpr int TPB = 256;                        // threads per block (all kernels)
constexpr int IPT = 4;                          // items per thread in scans
constexpr int TILE = TPB * IPT;
constexpr int LSMAX = 4;                        // hot entries per thread of the single-block list phase
constexpr int PCAP = 256;                       // k_fused: potential candidates handled by one block

// header offsets (doubles)
constexpr int H_REST = 0;    // K intervals (K <= 2): rest accumulators
constexpr int H_RESTM = 4;   // K intervals: rest accumulators at the midpoint
constexpr int H_WREST = 8;   // max width over the unsplit variables
constexpr int H_CHUNK = 9;   // first split variable c
constexpr int H_LEVY_NB = 10;  // Levy: neighbour values [L: u v um vm][R: u v um vm]
constexpr int H_LEVY_NT = 26;  // Levy: number of affected chain terms
constexpr int H_LEVY_T = 27;   // Levy: term descriptors kind*65536 + li*256 + lj (<= d + 3 = 23)
constexpr int H_LEVY_LR = 50;  // Levy: left / right neighbour variable (or -1)

// entry offsets (doubles)
constexpr int E_LO = 0, E_HI = 1, E_T = 2;  // then T[K] (2K), Tm[K] (2K), G[KG] (2KG), flag

// pool of pending boxes (the paper's list L, §3.2): one record
// = lower bound, max width, archive slot of the parent box, child code
struct Pool {
  double* lb;
  double* w;
  int32_t* slot;
  uint32_t* code;
};

// statistics of the live part of L (lb <= GUB), one atomic update per block
struct Stats {
  unsigned long long live;
  unsigned long long min_lb_key;
  unsigned long long max_w_bits;  // w >= 0: bit pattern order == value order
};

// Device-resident control block of a solve: every decision of the iteration
// (stop test, batch size, radix-select digits, counts) is taken on the GPU,
// so the host only synchronises once per chunk of iterations.  Kernels return
// immediately once `done` is set.
struct Ctl {
  unsigned long long pcount;    // records in L, live and dead (appended order)
  unsigned long long live;      // records with lb <= GUB (statistics pass)
  unsigned long long min_lb_key;
  unsigned long long max_w_bits;
  unsigned long long gub_key;   // incumbent GUB, ordered-int encoded
  unsigned long long B;         // regions selected this iteration
  unsigned long long ncand;     // children with lb <= GUB
  unsigned long long nsurv;     // children inserted into L
  unsigned long long free_top;  // archive free list
  unsigned long long iter, evals;
  unsigned long long prefix, need;  // radix select state
  int known, resolved;
  int done;   // 0 running, 1 converged, 2 iteration limit, 3 L empty, 4 error
  int err;    // IB_ENOSPACE when a capacity would be exceeded
  int gdone;  // multi-GPU: every rank finished (from the exchange)
  int xdone;  // multi-GPU: this rank stopped working (local decision)
  int need_w;  // the stop test needs the max width of L (width pass requested)
  int pad3;
  double eps_f, eps_x;
  unsigned long long bmax, max_iter, pool_cap;
  unsigned long long acc_live, acc_min_key, acc_max_w;  // per-pass accumulators (statistics)
  unsigned long long acc_live2, acc_min_key2;           // refill pass
  unsigned long long acc_live3, acc_min_key3;           // rebuilt hot index
  unsigned long long list_bytes;                        // algorithmic bytes of k_list
  unsigned int blocks_done;      // last-block election counter
  unsigned int fused_ticket;     // k_fused: last block of the insertion pass
  int list_pre;                  // k_fused: the next list phase already ran (last block)
  unsigned long long npot;       // k_fused: children with lb <= GUB at the iteration start (potential candidates)
  unsigned int pending_end;      // the survivors of the last iteration are not yet counted in pcount
  unsigned long long sum_pool;   // records scanned by the statistics pass
  unsigned long long sum_radix;  // records scanned by radix passes 2..8
  unsigned long long sum_B;      // parents prepared
  unsigned long long sum_cand;   // children that passed the lower-bound test
  // hot index of L: positions (increasing) of the records with key < tau_key
  unsigned long long tau_key;    // ~0: every record is hot
  unsigned long long nhot;       // entries of the current hot buffer
  unsigned long long nsurv_hot;  // survivors of this iteration appended to it
  unsigned long long nhot_keep;  // entries kept by the selection
  unsigned long long hot_target; // hot index size aimed at by a refill
  unsigned long long sum_refill; // records of L scanned by refills
  unsigned long long live_total; // live records of L at the last refill
  unsigned long long nrefill;    // refills so far
  unsigned long long nwidth;     // width passes so far
  int hsel;       // current hot buffer (0 / 1)
  int hot_valid;  // 0: the hot index must be rebuilt (start, after compaction)
  int compact_hint;  // a refill found L more than half dead
  int list_fast;  // k_fused: the next list phase may run on one block (set by emit)
};

struct Problem {
  int fid, n, d, m, kids;  // kids = m^d
  int h, G;                // a child-eval thread owns G = m^h children
  int mbits;               // log2(m) when m is a power of two, else 0
  int kbits;               // log2(m^d) when m is a power of two, else 0
  int ld;                  // archive row stride (doubles)
  int mono;                // apply the first-order test
  int pslices;             // k_prep blocks per parent (variable slices)
  int prest;               // 1: the rest accumulators are combined from the slice partials by the child phase
  int mitm;                // k_chain children by meet in the middle (d > 16, or IBNB_CHAIN_MITM=1)
  const double* l;         // device copies of the bounds
  const double* u;
};

// device buffers one iteration reads / writes (all sizes come from Ctl)
struct IterBufs {
  Ctl* ctl;
  unsigned int* hist;
  Pool pool;
  int32_t *sel_slot, *new_slot, *free_list;
  uint32_t* sel_code;
  const double *src_lo, *src_hi;
  const int32_t* src_sc;
  double *dst_lo, *dst_hi;
  int32_t* dst_sc;
  double* tab;
  int tab_stride;
  double* clb;
  uint32_t* cand;
  uint8_t* ok;
  uint64_t *desc, *desc2;
  uint32_t* tile_ctr;
  uint32_t *hot0, *hot1;  // hot index double buffer
  double* ppart;           // k_prep slice partials: [bmax][pslices][10]
  unsigned int* pticket;   // k_prep per-parent arrival tickets [bmax] (zero between launches)
  unsigned long long* tstamp;  // k_fused phase timer (trace only; nullptr otherwise)
  uint32_t* pot;               // k_fused: potential candidates (child indices), PCAP entries
  uint64_t* pbits;             // graph path: potential-candidate bitmap of the children (k_child_eval -> k_insert)
};

// buffers of the deep-dive chain kernel (chain.cuh)
constexpr int CH_PART = 10;  // doubles per slice partial (as k_prep's)
struct ChainBufs {
  unsigned long long* cnt;   // [3] potential candidates appended per iteration slot
  unsigned long long* gacc;  // [3] midpoint minima (ordered keys) per slot
  uint32_t* pcode;           // [3][PCAP] potential candidates (child codes)
  double* plb;               // [3][PCAP] their lower bounds
  double* pw;                // [3][PCAP] their max widths
  double* part;              // [2][grid][CH_PART] slice partials
  double* tabn;              // [2][DM_MAX * ENT] entries of the next chunk
  unsigned long long* exits;  // [8] why launches left the chain (trace statistics): 0 no survivor,
                              // 1 several survivors, 2 > PCAP potential candidates, 3 stop test,
                              // 4 iteration limit, 5 launch budget, 6 nothing to chain at entry
  unsigned long long* gshared;  // multi-GPU: the incumbent word shared by every rank (or nullptr)
  int per;                   // variables per block slice
  int tcache;                // k_chain keeps the slice's term cache in shared memory (set by the launcher)
  int grid;                  // k_chain blocks (one per SM, IBNB_CHAIN_GRID caps it)
};

// host callbacks around the kernel classes of an iteration: profiling
// events (class 0 prep, 1 child_eval, 2 prune, 3 statistics, 4 radix,
// 5 select) and the multi-GPU incumbent exchange
struct IterHook {
  virtual void begin(int cls, long units, cudaStream_t st) = 0;
  virtual void end(int cls, cudaStream_t st) = 0;
  virtual void exchange(cudaStream_t st) = 0;
  virtual ~IterHook() {}
};

// dynamic shared memory of k_chainc (chainc.cuh): the slice (2 per doubles)
// and the exchange buffers (chunk entries, potential-candidate lists, both
// parities)
size_t chainc_smem(int per);

// launchers of the kernels templated on one objective, instantiated in that
// objective's translation unit (bnb_kernels.cu, -DIBNB_OBJ_TU -DIBNB_FID=f)
struct ObjLaunch {
  void (*prep)(const Problem&, const IterBufs&, long, const int32_t*, cudaStream_t);
  void (*eval)(const Problem&, const IterBufs&, long, cudaStream_t, bool);
  void (*mono)(const Problem&, const IterBufs&, long, cudaStream_t);
  int (*insert)(const Problem&, const IterBufs&, long, cudaStream_t);
  int (*fused)(const Problem&, const IterBufs&, int, long, unsigned, cudaStream_t);
  int (*chain)(const Problem&, const IterBufs&, const ChainBufs&, int, unsigned, cudaStream_t);
  int (*chainc)(const Problem&, const IterBufs&, const ChainBufs&, int, int, cudaStream_t);
  void (*eval_boxes)(int, long, const double*, const double*, long, double*, unsigned, cudaStream_t);
  void (*eval_grad)(int, long, const double*, const double*, long, const int64_t*, const int32_t*, double*, unsigned,
                    cudaStream_t);
};

}  // namespace ib
