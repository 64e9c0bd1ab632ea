// bnb_kernels.cu -- the CUDA kernels of one branch-and-bound iteration
// (§3.1 flowchart, §3.2 partition / variable cycling) and of the
// explicit-batch evaluators.  Host launchers at the bottom are called by
// runtime.cu; nothing here knows about torch.  Every phase is a device
// function so that the multi-kernel path and the persistent k_fused run the
// same code:
//   k_list / list_dev   : iteration end, statistics of the hot index of L,
//                         stop test (lines 148-150), batch size, radix select
//                         and selection of the B smallest lower bounds
//                         (line 130; lazy deletion, lines 136); list_small_dev
//                         is the one-block variant
//   k_prep / prep_item  : materialise the selected regions (Eq. 8-11), reduce
//                         the terms of the unsplit variables over slices of
//                         the variables (two threads per variable), tabulate
//                         the pieces of the d split variables
//   k_child_eval        : lower bound and midpoint upper bound of every child
//                         (line 134: warp min -> ordered-int atomicMin on GUB)
//   k_cand, k_mono,     : candidates (lb <= GUB, line 140), first-order test
//   k_emit                (lines 142-144), stable decoupled-look-back
//                         insertion of the survivors into L (line 146)
//   k_fused             : whole iterations in one cooperative launch (small
//                         batches), with the one-block insertion + selection
//   k_partition, k_gc_* : compaction of L, archive slot collection
//   k_eval_boxes/_grad  : explicit-batch evaluators (parity tests)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "objectives.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

// every definition of this file (and of chain.cuh / chainc.cuh) lives in a
// namespace of its own per objective translation unit, so that the units'
// copies of the non-template device functions do not collide at link time
#ifdef IBNB_OBJ_TU
#define IBNB_CAT2(a, b) a##b
#define IBNB_CAT(a, b) IBNB_CAT2(a, b)
#define IB_NS_BEGIN namespace ib { inline namespace IBNB_CAT(obj, IBNB_FID) {
#define IB_NS_END } }
#else
#define IB_NS_BEGIN namespace ib {
#define IB_NS_END }
#endif

IB_NS_BEGIN

// ------------------------------------------------------------ probes
// -DIBNB_PROBE builds (diagnosis only): block 0 / thread 0 accumulates the
// clock64 cycles between probe points of a device function into g_probe
#ifdef IBNB_PROBE
#ifdef IBNB_OBJ_TU
static
#endif
__device__ unsigned long long g_probe[64];
#define PROBE_BEGIN unsigned long long _pt = clock64(), _pd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PROBE(k)                                   \
  {                                                \
    unsigned long long _t = clock64();             \
    _pd[k] += _t - _pt;                            \
    _pt = _t;                                      \
  }
#define PROBE_END(base)                                                    \
  if (blockIdx.x == 0 && threadIdx.x == 0)                                 \
    for (int _k = 0; _k < 8; ++_k) g_probe[(base) + _k] += _pd[_k];
#else
#define PROBE_BEGIN
#define PROBE(k)
#define PROBE_END(base)
#endif

// ------------------------------------------------------------ partition
// Eq. (10)-(11) with m pieces, round-to-nearest, no FMA (bit-identical to
// the oracle's part_point, reading R2).
__device__ __forceinline__ double part_point(double a, double b, int m, int k) {
  if (k <= 0) return a;
  if (k >= m) return b;
  double w = __ddiv_rn(__dsub_rn(b, a), (double)m);
  double p = __dadd_rn(a, __dmul_rn(w, (double)k));
  return p < b ? p : b;
}
__device__ __forceinline__ double midpt(double a, double b) {
  double mid = __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), 0.5));
  return fmin(fmax(mid, a), b);
}
__device__ __forceinline__ int digit(uint32_t code, int j, int m) {
  if (m == 2) return (code >> j) & 1u;
  for (int t = 0; t < j; ++t) code /= (uint32_t)m;
  return (int)(code % (uint32_t)m);
}

// ------------------------------------------------------------ reductions
template <class F>
__device__ __forceinline__ void warp_reduce_acc(Iv* a) {
#pragma unroll
  for (int k = 0; k < F::K; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Iv t{__shfl_xor_sync(0xffffffffu, a[k].lo, o), __shfl_xor_sync(0xffffffffu, a[k].hi, o)};
      a[k] = acc_comb<F>(k, a[k], t);
    }
  }
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block reduction of K interval accumulators (result valid in thread 0)
template <class F, int BS = TPB>
__device__ __forceinline__ void block_reduce_acc(Iv* a) {
  warp_reduce_acc<F>(a);
  if constexpr (BS > 32) {
    __shared__ Iv s_acc[BS / 32][2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
      for (int k = 0; k < F::K; ++k) s_acc[wid][k] = a[k];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < BS / 32; ++w)
        for (int k = 0; k < F::K; ++k) a[k] = acc_comb<F>(k, a[k], s_acc[w][k]);
    }
    __syncthreads();
  }
}
template <int BS = TPB>
__device__ __forceinline__ double block_max(double v) {
  v = warp_max(v);
  if constexpr (BS > 32) {
    __shared__ double s_m[BS / 32];
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 1; w < BS / 32; ++w) v = fmax(v, s_m[w]);
    __syncthreads();
  }
  return v;
}

__device__ __forceinline__ void put(double* p, Iv v) {
  p[0] = v.lo;
  p[1] = v.hi;
}
__device__ __forceinline__ Iv get(const double* p) { return Iv{p[0], p[1]}; }

// ------------------------------------------------------------ Levy helpers
struct LevyChunk {
  int c, d, n, L, R;
  __device__ bool inJ(int t) const { return ((t - c + n) % n) < d; }
  __device__ int local(int t) const {
    int jj = (t - c + n) % n;
    if (jj < d) return jj;
    return t == L ? d : d + 1;
  }
};
__device__ __forceinline__ LevyChunk levy_chunk(int c, int d, int n) {
  LevyChunk q{c, d, n, -1, -1};
  if (d < n) {
    int L = c - 1;  // chain neighbour left of the chunk
    if (c >= 1 && !q.inJ(L)) q.L = L;
    int R = (c + d) % n;
    if (R != 0 && !q.inJ(R)) q.R = R;
  }
  return q;
}

// warp level of block_reduce_prep (xor butterfly: every lane ends with the
// same bits, the combinations are commutative)
template <class F>
__device__ __forceinline__ void warp_reduce_prep(Iv* acc, Iv* accm, double& wmax) {
  constexpr int K = F::CHAIN ? 1 : F::K;
  auto comb = [](int k, Iv a, Iv b) -> Iv {
    if constexpr (F::CHAIN) return a + b;
    else return acc_comb<F>(k, a, b);
  };
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      Iv t{__shfl_xor_sync(0xffffffffu, acc[k].lo, o), __shfl_xor_sync(0xffffffffu, acc[k].hi, o)};
      Iv tm{__shfl_xor_sync(0xffffffffu, accm[k].lo, o), __shfl_xor_sync(0xffffffffu, accm[k].hi, o)};
      acc[k] = comb(k, acc[k], t);
      accm[k] = comb(k, accm[k], tm);
    }
    wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  }
}

// prep: one block reduction of the rest accumulators of the box (acc) and of
// its midpoint (accm) and of the max unsplit width, in a single pass
// (results valid in thread 0); Levy reduces one chain sum each
template <class F, int BS>
__device__ __forceinline__ void block_reduce_prep(Iv* acc, Iv* accm, double& wmax) {
  constexpr int K = F::CHAIN ? 1 : F::K;
  auto comb = [](int k, Iv a, Iv b) -> Iv {
    if constexpr (F::CHAIN) return a + b;
    else return acc_comb<F>(k, a, b);
  };
  warp_reduce_prep<F>(acc, accm, wmax);
  if constexpr (BS > 32) {
    __shared__ Iv s_a[BS / 32][2], s_m[BS / 32][2];
    __shared__ double s_w[BS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
      for (int k = 0; k < K; ++k) {
        s_a[wid][k] = acc[k];
        s_m[wid][k] = accm[k];
      }
      s_w[wid] = wmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < BS / 32; ++w) {
        for (int k = 0; k < K; ++k) {
          acc[k] = comb(k, acc[k], s_a[w][k]);
          accm[k] = comb(k, accm[k], s_m[w][k]);
        }
        wmax = fmax(wmax, s_w[w]);
      }
    }
    __syncthreads();
  }
}

// the S slice partials of parent b combined in a fixed tree order
// (deterministic; results valid in thread 0)
template <class F, int BS>
__device__ __forceinline__ void combine_partials(const double* __restrict__ ppart, int b, int S, Iv* acc, Iv* accm,
                                                 double& wmax) {
  const double* pp = ppart + (size_t)b * S * 10;
  Iv ra[2], rm[2];
  double rw = 0.0;
#pragma unroll
  for (int k = 0; k < 2; ++k) ra[k] = rm[k] = iv(0.0);
  if constexpr (!F::CHAIN) {
#pragma unroll
    for (int k = 0; k < F::K; ++k) ra[k] = rm[k] = acc_ident<F>(k);
  }
  for (int t = threadIdx.x; t < S; t += BS) {
    const double* pt = pp + (size_t)t * 10;
    if constexpr (F::CHAIN) {
      ra[0] = ra[0] + get(pt);
      rm[0] = rm[0] + get(pt + 4);
    } else {
#pragma unroll
      for (int k = 0; k < F::K; ++k) {
        ra[k] = acc_comb<F>(k, ra[k], get(pt + 2 * k));
        rm[k] = acc_comb<F>(k, rm[k], get(pt + 4 + 2 * k));
      }
    }
    rw = fmax(rw, pt[8]);
  }
  block_reduce_prep<F, BS>(ra, rm, rw);
  for (int k = 0; k < 2; ++k) {
    acc[k] = ra[k];
    accm[k] = rm[k];
  }
  wmax = rw;
}

// one part of the table entry of a piece [pa, pb] (midpoint xm) of split
// variable i (non-chain objectives): part 0 bounds + box terms, 1 midpoint
// terms, 2 derivative ingredients + the separable first-order flag (PAPER.md
// lines 142-144: derivative of constant sign off the domain edge)
template <class F>
__device__ __forceinline__ void piece_entry(const Problem& P, double pa, double pb, double xm, int i, int part,
                                            double* e) {
  const int n = P.n;
  if (part == 0) {
    Iv tt[2];
    F::terms(Iv{pa, pb}, i, n, tt);
    e[E_LO] = pa;
    e[E_HI] = pb;
    for (int k = 0; k < F::K; ++k) put(e + E_T + 2 * k, tt[k]);
  } else if (part == 1) {
    Iv tm[2];
    F::terms(Iv{xm, xm}, i, n, tm);
    for (int k = 0; k < F::K; ++k) put(e + E_T + 2 * F::K + 2 * k, tm[k]);
  } else {
    Iv g[2];
    if constexpr (F::KG > 0) {
      F::ding(Iv{pa, pb}, i, n, g);
      for (int k = 0; k < F::KG; ++k) put(e + E_T + 4 * F::K + 2 * k, g[k]);
    }
    double flag = 0.0;
    if constexpr (F::SEP) {
      Iv D = F::dsep(Iv{pa, pb}, i, n);
      if ((D.lo > 0.0 && pa != P.l[i]) || (D.hi < 0.0 && pb != P.u[i])) flag = 1.0;
    }
    e[E_T + 4 * F::K + 2 * F::KG] = flag;
  }
}

// ====================================================================== prep
// Parent b of the batch is handled by P.pslices blocks (one block when the
// batch is large; for large n and small batches the n variables are cut into
// slices so that the O(n) reduction spreads over the SMs).  Block (b, s):
// materialises its slice of the new parent (source row: archive slot
// sel_slot[b] of src_lo/src_hi with record code sel_code[b]; destination:
// slot new_slot[b] of dst_lo/dst_hi) and reduces the terms of its unsplit
// variables; the partial results go to ppart, and the last block of the
// parent to finish (threadfence + ticket) combines them in slice order and
// writes the header and the piece tables.  src_sc / dst_sc hold each slot's
// chunk start.
template <class F, int BS>
__device__ __forceinline__ void prep_item(const Problem& P, const Ctl* __restrict__ ctl,
                                          const int32_t* __restrict__ sel_slot, const uint32_t* __restrict__ sel_code,
                                          int32_t* __restrict__ new_slot, const int32_t* __restrict__ free_list,
                                          const double* __restrict__ src_lo, const double* __restrict__ src_hi,
                                          const int32_t* __restrict__ src_sc, double* dst_lo, double* dst_hi,
                                          int32_t* dst_sc, double* tab, int tab_stride, double* __restrict__ ppart,
                                          unsigned int* __restrict__ pticket, const int b, const int s) {
  const int S = P.pslices;
  if (ctl->done || b >= (int)ctl->B) return;
  const int n = P.n, d = P.d, m = P.m;
  const int src = sel_slot[b];
  const uint32_t code = sel_code[b];
  // archive slot of the new parent: popped from the free list (solve) or given
  const int dst = free_list ? free_list[ctl->free_top - 1 - b] : new_slot[b];
  if (free_list && s == 0 && threadIdx.x == 0) new_slot[b] = dst;
  const int psc = src_sc[src];
  const int c = (code == CODE_WHOLE) ? psc : (psc + d) % n;  // line 184
  const double* slo = src_lo + (size_t)src * P.ld;
  const double* shi = src_hi + (size_t)src * P.ld;
  double* dlo = dst_lo + (size_t)dst * P.ld;
  double* dhi = dst_hi + (size_t)dst * P.ld;
  double* T = tab + (size_t)b * tab_stride;
  // variable i of the new parent (Eq. 8-11 applied to the selected record)
  auto mat = [&](int i, double& a, double& bb) {
    a = slo[i];
    bb = shi[i];
    if (code != CODE_WHOLE) {
      int jj = (i - psc + n) % n;
      if (jj < d) {
        int p = digit(code, jj, m);
        double a2 = part_point(a, bb, m, p), b2 = part_point(a, bb, m, p + 1);
        a = a2;
        bb = b2;
      }
    }
  };
  const int per = (n + S - 1) / S;
  const int i0 = s * per, i1 = min(n, i0 + per);

  Iv acc[2], accm[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) acc[k] = accm[k] = iv(0.0);
  if constexpr (!F::CHAIN) {
#pragma unroll
    for (int k = 0; k < F::K; ++k) acc[k] = accm[k] = acc_ident<F>(k);
  }
  double wmax = 0.0;
  LevyChunk q = levy_chunk(c, d, n);
  // two threads per variable: half 0 the box (and the row, the width), half 1
  // the midpoint, so that each thread's transcendental chain is one
  // enclosure long; block_reduce_prep combines both halves
  constexpr int HB = BS / 2;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  if constexpr (!F::CHAIN) {
    for (int i = i0 + hv; i < i1; i += HB) {
      double a, bb;
      mat(i, a, bb);
      if (half == 0) {
        dlo[i] = a;
        dhi[i] = bb;
      }
      if (((i - c + n) % n) >= d) {
        Iv t[2];
        if (half == 0) {
          wmax = fmax(wmax, __dsub_rn(bb, a));
          F::terms(Iv{a, bb}, i, n, t);
        } else {
          const double xm = midpt(a, bb);
          F::terms(Iv{xm, xm}, i, n, t);
        }
#pragma unroll
        for (int k = 0; k < F::K; ++k) {
          if (half == 0) acc[k] = acc_comb<F>(k, acc[k], t[k]);
          else accm[k] = acc_comb<F>(k, accm[k], t[k]);
        }
      }
    }
  } else {
    // Levy: rest = sum of chain terms that involve no split variable; the
    // values of variable i + 1 come from the neighbouring thread of the same
    // half (shared memory), recomputed only across block boundaries
    __shared__ Iv s_v[BS];
    for (int base = i0; base < i1; base += HB) {  // block-uniform trip count
      const int i = base + hv;
      const bool in = i < i1;
      LevyVals v;
      double a = 0.0, bb = 0.0;
      if (in) {
        mat(i, a, bb);
        if (half == 0) {
          dlo[i] = a;
          dhi[i] = bb;
          if (((i - c + n) % n) >= d) wmax = fmax(wmax, __dsub_rn(bb, a));
          v = ObjLevy::vals(Iv{a, bb});
        } else {
          const double xm = midpt(a, bb);
          v = ObjLevy::vals(Iv{xm, xm});
        }
        s_v[threadIdx.x] = v.v;
      }
      __syncthreads();
      if (in) {
        Iv& r = half == 0 ? acc[0] : accm[0];
        const bool ji = q.inJ(i);
        if (i == 0 && !ji) r = r + v.s0;
        if (i <= n - 2 && !ji && !q.inJ(i + 1)) {
          Iv wv;
          if (hv + 1 < HB && i + 1 < i1) {
            wv = s_v[threadIdx.x + 1];
          } else {
            double a1, b1;
            mat(i + 1, a1, b1);
            if (half == 0) {
              wv = ObjLevy::vals(Iv{a1, b1}).v;
            } else {
              const double xm1 = midpt(a1, b1);
              wv = ObjLevy::vals(Iv{xm1, xm1}).v;
            }
          }
          r = r + mulpos(v.u, wv);
        }
        if (i == n - 1 && !ji) r = r + v.u;
      }
      __syncthreads();
    }
  }
  block_reduce_prep<F, BS>(acc, accm, wmax);
  // tables of the m pieces of the d split variables, by the block that owns
  // the variable (slices run in parallel); three threads per entry: bounds +
  // box terms, midpoint terms, derivative ingredients + separable flag
  for (int t = threadIdx.x; t < 3 * d * m; t += BS) {
    const int ent = t % (d * m), part = t / (d * m);
    int j = ent / m, p = ent % m;
    int i = (c + j) % n;
    if (i < i0 || i >= i1) continue;
    double a, bb;
    mat(i, a, bb);
    double pa = part_point(a, bb, m, p), pb = part_point(a, bb, m, p + 1);
    double xm = midpt(pa, pb);
    double* e = T + HDR + (size_t)ent * ENT;
    if constexpr (F::CHAIN) {
      if (part == 0) {
        LevyVals v = ObjLevy::vals(Iv{pa, pb});
        e[E_LO] = pa;
        e[E_HI] = pb;
        put(e + 2, v.u);
        put(e + 4, v.v);
        put(e + 6, v.s0);
        put(e + 8, v.du);
        put(e + 10, v.sg);
      } else if (part == 1) {
        LevyVals vm = ObjLevy::vals(Iv{xm, xm});
        put(e + 12, vm.u);
        put(e + 14, vm.v);
        put(e + 16, vm.s0);
      }
    } else {
      piece_entry<F>(P, pa, pb, xm, i, part, e);
    }
  }
  if (S > 1 && P.prest) {
    // publish this slice's partial; the child phase combines them (the next
    // grid barrier / kernel boundary orders it); slice 0 writes the header
    if (threadIdx.x == 0) {
      double* pp = ppart + ((size_t)b * S + s) * 10;
      for (int k = 0; k < 2; ++k) {
        put(pp + 2 * k, acc[k]);
        put(pp + 4 + 2 * k, accm[k]);
      }
      pp[8] = wmax;
    }
    if (s != 0) return;
  } else if (S > 1) {
    // publish this slice's partial; the last slice block of parent b goes on
    // (the rows and tables of this block are read only after the next grid
    // barrier or kernel boundary; only the partial must precede the ticket)
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      double* pp = ppart + ((size_t)b * S + s) * 10;
      for (int k = 0; k < 2; ++k) {
        put(pp + 2 * k, acc[k]);
        put(pp + 4 + 2 * k, accm[k]);
      }
      pp[8] = wmax;
      __threadfence();
      s_last = atomicAdd(&pticket[b], 1u) == (unsigned)(S - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    combine_partials<F, BS>(ppart, b, S, acc, accm, wmax);
    if (threadIdx.x == 0) {
      pticket[b] = 0u;  // every slice block of b has arrived: reset for the next launch
    }
  }
  if constexpr (F::CHAIN) {
    // neighbour values of the chunk (box and midpoint of the left and the
    // right neighbour variable), one thread each
    if (threadIdx.x < 4) {
      const int sd = threadIdx.x >> 1, mid = threadIdx.x & 1;
      const int nbv = sd == 0 ? q.L : q.R;
      Iv X = iv(0.0);
      if (nbv >= 0) mat(nbv, X.lo, X.hi);
      if (mid) {
        const double xm = midpt(X.lo, X.hi);
        X = Iv{xm, xm};
      }
      const LevyVals v = ObjLevy::vals(X);
      double* nb_ = T + H_LEVY_NB + 8 * sd + 4 * mid;
      put(nb_ + 0, v.u);
      put(nb_ + 2, v.v);
    }
  }
  if (threadIdx.x == 0) {
    if (!(S > 1 && P.prest)) {
      for (int k = 0; k < 2; ++k) {
        put(T + H_REST + 2 * k, acc[k]);
        put(T + H_RESTM + 2 * k, accm[k]);
      }
      T[H_WREST] = wmax;
    }
    T[H_CHUNK] = (double)c;
    dst_sc[dst] = c;
    if constexpr (F::CHAIN) {
      // the list of affected chain terms
      int nt = 0;
      double* td = T + H_LEVY_T;
      if (q.inJ(0)) td[nt++] = (double)(0 * 65536 + q.local(0) * 256);
      int ncand = d < n ? d + 1 : n;
      for (int t = 0; t < ncand; ++t) {
        int i = d < n ? (c - 1 + t + n) % n : t;
        if (i > n - 2) continue;
        if (q.inJ(i) || q.inJ(i + 1)) td[nt++] = (double)(1 * 65536 + q.local(i) * 256 + q.local(i + 1));
      }
      if (q.inJ(n - 1)) td[nt++] = (double)(2 * 65536 + q.local(n - 1) * 256);
      T[H_LEVY_NT] = (double)nt;
      T[H_LEVY_LR] = (double)q.L;
      T[H_LEVY_LR + 1] = (double)q.R;
    }
  }
}

template <class F, int BS>
__global__ void __launch_bounds__(BS) k_prep(Problem P, const Ctl* __restrict__ ctl, const int32_t* __restrict__ sel_slot,
                                             const uint32_t* __restrict__ sel_code, int32_t* __restrict__ new_slot,
                                             const int32_t* __restrict__ free_list, const double* __restrict__ src_lo,
                                             const double* __restrict__ src_hi, const int32_t* __restrict__ src_sc,
                                             double* dst_lo, double* dst_hi, int32_t* dst_sc, double* tab,
                                             int tab_stride, double* __restrict__ ppart,
                                             unsigned int* __restrict__ pticket) {
  const int b = blockIdx.x / P.pslices;
  prep_item<F, BS>(P, ctl, sel_slot, sel_code, new_slot, free_list, src_lo, src_hi, src_sc, dst_lo, dst_hi, dst_sc,
                   tab, tab_stride, ppart, pticket, b, blockIdx.x - b * P.pslices);
}

// ================================================================ children
// Child g of the batch: parent b = g / m^d, code = g % m^d; digit j of the
// code (base m) is the piece of split variable (c + j) mod n.
struct ChildIdx {
  int b;
  uint32_t code;
};
__device__ __forceinline__ ChildIdx child_of(long g, const Problem& P) {
  if (P.mbits) return ChildIdx{(int)(g >> P.kbits), (uint32_t)g & (uint32_t)(P.kids - 1)};
  return ChildIdx{(int)(g / P.kids), (uint32_t)(g % P.kids)};
}
// piece of split variable j in child `code`
__device__ __forceinline__ int piece(uint32_t code, int j, const Problem& P) {
  if (P.mbits) return (int)((code >> (j * P.mbits)) & (uint32_t)(P.m - 1));
  for (int t = 0; t < j; ++t) code /= (uint32_t)P.m;
  return (int)(code % (uint32_t)P.m);
}

// Levy accessors over (split pieces | neighbours)
struct LevyView {
  const double* T;
  const int* e;  // entry index per split variable
  int d;
  __device__ Iv u(int li, bool mid) const {
    if (li < d) return get(T + HDR + (size_t)e[li] * ENT + (mid ? 12 : 2));
    return get(T + H_LEVY_NB + 8 * (li - d) + (mid ? 4 : 0));
  }
  __device__ Iv v(int li, bool mid) const {
    if (li < d) return get(T + HDR + (size_t)e[li] * ENT + (mid ? 14 : 4));
    return get(T + H_LEVY_NB + 8 * (li - d) + (mid ? 6 : 2));
  }
  __device__ Iv s0(int li, bool mid) const { return get(T + HDR + (size_t)e[li] * ENT + (mid ? 16 : 6)); }
  __device__ Iv acc(bool mid) const {
    Iv a = get(T + (mid ? H_RESTM : H_REST));
    int nt = (int)T[H_LEVY_NT];
    for (int t = 0; t < nt; ++t) {
      int dsc = (int)T[H_LEVY_T + t];
      int kind = dsc >> 16, li = (dsc >> 8) & 255, lj = dsc & 255;
      if (kind == 0)
        a = a + s0(li, mid);
      else if (kind == 1)
        a = a + mulpos(u(li, mid), v(lj, mid));  // u >= 0, v >= 1
      else
        a = a + u(li, mid);
    }
    return a;
  }
};

__device__ __forceinline__ void entries_of(uint32_t code, const Problem& P, int* e) {
  for (int j = 0; j < P.d; ++j) e[j] = j * P.m + piece(code, j, P);
}

// accumulators of the child box (rest combined with the d piece terms)
template <class F>
__device__ __forceinline__ void child_acc(const Problem& P, const double* __restrict__ T, uint32_t code, Iv* A) {
#pragma unroll
  for (int k = 0; k < F::K; ++k) A[k] = get(T + H_REST + 2 * k);
  for (int j = 0; j < P.d; ++j) {
    const double* e = T + HDR + (size_t)(j * P.m + piece(code, j, P)) * ENT + E_T;
#pragma unroll
    for (int k = 0; k < F::K; ++k) A[k] = acc_comb<F>(k, A[k], get(e + 2 * k));
  }
}

__device__ __forceinline__ double child_width(const Problem& P, const double* __restrict__ T, uint32_t code) {
  double w = T[H_WREST];
  for (int j = 0; j < P.d; ++j) {
    const double* e = T + HDR + (size_t)(j * P.m + piece(code, j, P)) * ENT;
    w = fmax(w, __dsub_rn(e[E_HI], e[E_LO]));
  }
  return w;
}

// first-order test of PAPER.md lines 142-144 on the split variables of a
// child whose lower bound already passed; true = the child survives
template <class F>
__device__ __noinline__ bool child_mono_ok(const Problem& P, const double* __restrict__ T, uint32_t code) {
  const int d = P.d, m = P.m, n = P.n;
  const int c = (int)T[H_CHUNK];
  if constexpr (F::CHAIN) {
    int e[D_MAX];
    entries_of(code, P, e);
    LevyView V{T, e, d};
    LevyChunk q = levy_chunk(c, d, n);
    for (int j = 0; j < d; ++j) {
      int i = (c + j) % n;
      const double* ej = T + HDR + (size_t)e[j] * ENT;
      LevyVals me;
      me.u = get(ej + 2);
      me.v = get(ej + 4);
      me.s0 = get(ej + 6);
      me.du = get(ej + 8);
      me.sg = get(ej + 10);
      Iv up = i > 0 ? V.u(q.local(i - 1), false) : iv(0.0);
      Iv vn = i < n - 1 ? V.v(q.local(i + 1), false) : iv(0.0);
      Iv D = ObjLevy::deriv(me, up, vn, i, n);
      if ((D.lo > 0.0 && ej[E_LO] != P.l[i]) || (D.hi < 0.0 && ej[E_HI] != P.u[i])) return false;
    }
    return true;
  } else if constexpr (F::SEP) {
    for (int j = 0; j < d; ++j)
      if (T[HDR + (size_t)(j * m + piece(code, j, P)) * ENT + E_T + 4 * F::K + 2 * F::KG] != 0.0) return false;
    return true;
  } else {
    Iv A[2];
    child_acc<F>(P, T, code, A);
    typename F::Ctx cx = F::ctx(A, n);
    if constexpr (F::HASPROD) {
      // products without variable i: running prefix x precomputed suffix
      Iv suf[D_MAX + 1][2];
      Iv pre[2];
#pragma unroll
      for (int k = 0; k < F::K; ++k) {
        suf[d][k] = iv(1.0);
        pre[k] = get(T + H_REST + 2 * k);
      }
      for (int j = d - 1; j >= 0; --j) {
        const double* ej = T + HDR + (size_t)(j * m + piece(code, j, P)) * ENT + E_T;
#pragma unroll
        for (int k = 0; k < F::K; ++k)
          suf[j][k] = F::kind(k) == PROD ? get(ej + 2 * k) * suf[j + 1][k] : iv(0.0);
      }
      for (int j = 0; j < d; ++j) {
        int i = (c + j) % n;
        const double* ej = T + HDR + (size_t)(j * m + piece(code, j, P)) * ENT;
        Iv g[2], excl[2];
#pragma unroll
        for (int k = 0; k < F::KG; ++k) g[k] = get(ej + E_T + 4 * F::K + 2 * k);
#pragma unroll
        for (int k = 0; k < F::K; ++k) excl[k] = F::kind(k) == PROD ? pre[k] * suf[j + 1][k] : iv(0.0);
        Iv X{ej[E_LO], ej[E_HI]};
        Iv D = F::dfin(cx, g, X, i, n, excl);
        if ((D.lo > 0.0 && X.lo != P.l[i]) || (D.hi < 0.0 && X.hi != P.u[i])) return false;
#pragma unroll
        for (int k = 0; k < F::K; ++k)
          if (F::kind(k) == PROD) pre[k] = pre[k] * get(ej + E_T + 2 * k);
      }
    } else {
      for (int j = 0; j < d; ++j) {
        int i = (c + j) % n;
        const double* ej = T + HDR + (size_t)(j * m + piece(code, j, P)) * ENT;
        Iv g[2], excl[2] = {iv(0.0), iv(0.0)};
#pragma unroll
        for (int k = 0; k < F::KG; ++k) g[k] = get(ej + E_T + 4 * F::K + 2 * k);
        Iv X{ej[E_LO], ej[E_HI]};
        Iv D = F::dfin(cx, g, X, i, n, excl);
        if ((D.lo > 0.0 && X.lo != P.l[i]) || (D.hi < 0.0 && X.hi != P.u[i])) return false;
      }
    }
    return true;
  }
}

// The first-order test of child_mono_ok with one lane per split variable
// (called by all 32 lanes of a warp, d <= 16 lanes work): each lane repeats
// the serial function's shared steps (child accumulators, context, and for
// product accumulators its own left-to-right prefix and right-to-left
// suffix) in the same order, so every per-variable enclosure is bit-identical
// to child_mono_ok's and so is the decision.
template <class F>
__device__ __noinline__ bool child_mono_ok_warp(const Problem& P, const double* __restrict__ T, uint32_t code) {
  const int d = P.d, m = P.m, n = P.n;
  const int lane = threadIdx.x & 31;
  const int c = (int)T[H_CHUNK];
  bool bad = false;
  if (lane < d) {
    const int j = lane;
    const int i = (c + j) % n;
    if constexpr (F::CHAIN) {
      int e[D_MAX];
      entries_of(code, P, e);
      LevyView V{T, e, d};
      LevyChunk q = levy_chunk(c, d, n);
      const double* ej = T + HDR + (size_t)e[j] * ENT;
      LevyVals me;
      me.u = get(ej + 2);
      me.v = get(ej + 4);
      me.s0 = get(ej + 6);
      me.du = get(ej + 8);
      me.sg = get(ej + 10);
      Iv up = i > 0 ? V.u(q.local(i - 1), false) : iv(0.0);
      Iv vn = i < n - 1 ? V.v(q.local(i + 1), false) : iv(0.0);
      Iv D = ObjLevy::deriv(me, up, vn, i, n);
      bad = (D.lo > 0.0 && ej[E_LO] != P.l[i]) || (D.hi < 0.0 && ej[E_HI] != P.u[i]);
    } else if constexpr (F::SEP) {
      bad = T[HDR + (size_t)(j * m + piece(code, j, P)) * ENT + E_T + 4 * F::K + 2 * F::KG] != 0.0;
    } else {
      Iv A[2];
      child_acc<F>(P, T, code, A);
      typename F::Ctx cx = F::ctx(A, n);
      const double* ej = T + HDR + (size_t)(j * m + piece(code, j, P)) * ENT;
      Iv g[2], excl[2] = {iv(0.0), iv(0.0)};
#pragma unroll
      for (int k = 0; k < F::KG; ++k) g[k] = get(ej + E_T + 4 * F::K + 2 * k);
      if constexpr (F::HASPROD) {
        Iv pre[2], suf[2];
#pragma unroll
        for (int k = 0; k < F::K; ++k) {
          pre[k] = get(T + H_REST + 2 * k);
          suf[k] = iv(1.0);
        }
        for (int t = 0; t < j; ++t) {  // prefix: rest * t_0 * ... * t_{j-1}
          const double* et = T + HDR + (size_t)(t * m + piece(code, t, P)) * ENT + E_T;
#pragma unroll
          for (int k = 0; k < F::K; ++k)
            if (F::kind(k) == PROD) pre[k] = pre[k] * get(et + 2 * k);
        }
        for (int t = d - 1; t > j; --t) {  // suffix: t_{j+1} * (... * (t_{d-1} * 1))
          const double* et = T + HDR + (size_t)(t * m + piece(code, t, P)) * ENT + E_T;
#pragma unroll
          for (int k = 0; k < F::K; ++k)
            if (F::kind(k) == PROD) suf[k] = get(et + 2 * k) * suf[k];
        }
#pragma unroll
        for (int k = 0; k < F::K; ++k) excl[k] = F::kind(k) == PROD ? pre[k] * suf[k] : iv(0.0);
      }
      Iv X{ej[E_LO], ej[E_HI]};
      Iv D = F::dfin(cx, g, X, i, n, excl);
      bad = (D.lo > 0.0 && X.lo != P.l[i]) || (D.hi < 0.0 && X.hi != P.u[i]);
    }
  }
  return __ballot_sync(0xffffffffu, bad) == 0u;
}

// Pass 1: upper bound at the midpoint and lower bound of every child.
// A thread owns G = m^h consecutive children (all pieces of the h lowest
// split variables): the terms of the d - h higher variables are combined
// once per group.  Midpoint bounds are min-reduced (warp shuffle -> block ->
// one ordered-int atomicMin per block into the incumbent, line 134); lower
// bounds are stored per child for pass 2.
// GT = 8: bisection (m = 2, h = 3) with the group loop fully unrolled so the
// outer functions of the 8 children interleave (ILP); GT = 0: runtime G
// warp-aggregated append of child g to the potential-candidate list (k_fused)
__device__ __forceinline__ void pot_append(Ctl* ctl, uint32_t* pot, bool cond, uint32_t g) {
  const unsigned am = __activemask();
  const unsigned m = __ballot_sync(am, cond);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&ctl->npot, (unsigned long long)__popc(m));
  base = __shfl_sync(am, base, leader);
  if (cond) {
    const unsigned long long idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < (unsigned long long)PCAP) pot[idx] = g;
  }
}

template <class F, int GT>
__device__ __forceinline__ void child_eval_dev(const Problem& P, Ctl* __restrict__ ctl,
                                               const double* __restrict__ tab, int tab_stride,
                                               double* __restrict__ clb, uint64_t* zero_a, uint64_t* zero_b,
                                               long nzero, uint32_t* zero_ctr, unsigned int* zero_hist,
                                               uint32_t* pot = nullptr, const double* __restrict__ ppart = nullptr,
                                               uint64_t* __restrict__ pbits = nullptr) {
  if (ctl->done) return;
  if (zero_a) {  // descriptors and tickets of the following k_cand / k_emit,
                 // histograms and accumulators of the next k_list
    for (long i = (long)blockIdx.x * TPB + threadIdx.x; i < 3 * nzero; i += (long)gridDim.x * TPB) {
      if (i < nzero) zero_a[i] = 0;
      zero_b[i] = 0;
    }
    for (long i = (long)blockIdx.x * TPB + threadIdx.x; i < 16 * 256; i += (long)gridDim.x * TPB) zero_hist[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x < 4) zero_ctr[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->acc_live = ctl->acc_live2 = ctl->acc_live3 = 0;
      ctl->acc_min_key = ctl->acc_min_key2 = ctl->acc_min_key3 = ~0ull;
      ctl->acc_max_w = 0;
    }
  }
  const int d = P.d, m = GT ? 2 : P.m, n = P.n, h = GT ? 3 : P.h, G = GT ? GT : P.G;
  const long gpp = P.kids / G;
  const long ngroups = (long)ctl->B * gpp;
  const double gub0 = okey_inv(ctl->gub_key);  // incumbent before this iteration
  double best = CUDART_INF;
  // the tables of the (at most two) parents of a block's 256 groups are
  // staged in shared memory when they fit (bisection): one coalesced load
  // instead of a dependent L2 round trip per piece / chain term
  constexpr int TS = HDR + 2 * D_MAX * ENT;  // bisection tables (m = 2, d <= 16)
  __shared__ double s_tab[2][TS];
  for (long base = (long)blockIdx.x * TPB; base < ngroups; base += (long)gridDim.x * TPB) {
    const long gi = base + threadIdx.x;
    const double* __restrict__ Tsh = nullptr;
    int b0 = 0;
    {
      const long glast = min(base + TPB, ngroups) - 1;
      b0 = P.mbits ? (int)(base >> (P.kbits - h * P.mbits)) : (int)(base / gpp);
      const int b1 = P.mbits ? (int)(glast >> (P.kbits - h * P.mbits)) : (int)(glast / gpp);
      if (b1 - b0 <= 1 && tab_stride <= TS) {
        __syncthreads();  // the previous iteration's readers are done
        const int nb = b1 - b0 + 1;
        for (int t = threadIdx.x; t < nb * tab_stride; t += TPB)
          s_tab[t / tab_stride][t % tab_stride] = tab[(size_t)b0 * tab_stride + t];
        if (P.prest) {
          // rest accumulators of the parents from k_prep's slice partials;
          // also written to the global tables for the insertion pass (every
          // block writes the same bits)
          for (int j = 0; j < nb; ++j) {
            Iv ra[2], rm[2];
            double rw;
            combine_partials<F, TPB>(ppart, b0 + j, P.pslices, ra, rm, rw);
            if (threadIdx.x == 0) {
              double* Tg = const_cast<double*>(tab) + (size_t)(b0 + j) * tab_stride;
              for (int k = 0; k < 2; ++k) {
                put(&s_tab[j][H_REST + 2 * k], ra[k]);
                put(&s_tab[j][H_RESTM + 2 * k], rm[k]);
                put(Tg + H_REST + 2 * k, ra[k]);
                put(Tg + H_RESTM + 2 * k, rm[k]);
              }
              s_tab[j][H_WREST] = rw;
              Tg[H_WREST] = rw;
            }
          }
        }
        __syncthreads();
        Tsh = &s_tab[0][0];
      }
    }
    // potential-candidate bits of this thread's G children (lb <= GUB_old):
    // the bitmap of the sparse insertion (graph path, G = 8 only)
    uint32_t pm = 0;
    if (gi < ngroups) {
    const int b = P.mbits ? (int)(gi >> (P.kbits - h * P.mbits)) : (int)(gi / gpp);
    const uint32_t hcode = P.mbits ? (uint32_t)gi & (uint32_t)(gpp - 1) : (uint32_t)(gi % gpp);
    const double* __restrict__ T = Tsh ? Tsh + (size_t)(b - b0) * TS : tab + (size_t)b * tab_stride;
    if constexpr (F::CHAIN) {
      for (int q = 0; q < G; ++q) {
        int e[D_MAX];
        entries_of(hcode * (uint32_t)G + (uint32_t)q, P, e);
        LevyView V{T, e, d};
        const double lbq = canon_lb(ObjLevy::outer(V.acc(false), n).lo);
        clb[gi * G + q] = lbq;
        if (lbq <= gub0) best = fmin(best, ObjLevy::outer(V.acc(true), n).hi);
        if (pot) pot_append(ctl, pot, lbq <= gub0, (uint32_t)(gi * G + q));
      }
    } else {
      Iv A[2], Am[2];
#pragma unroll
      for (int k = 0; k < F::K; ++k) {
        A[k] = get(T + H_REST + 2 * k);
        Am[k] = get(T + H_RESTM + 2 * k);
      }
      const uint32_t code0 = hcode * (uint32_t)G;
      int j = h;
      // batches of 4 pieces: the loads of a batch are issued together (one
      // L2 round trip instead of four), the combination order is unchanged
      for (; j + 4 <= d; j += 4) {
        Iv t[4][2], tm[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double* e = T + HDR + (size_t)((j + u) * m + piece(code0, j + u, P)) * ENT + E_T;
#pragma unroll
          for (int k = 0; k < F::K; ++k) {
            t[u][k] = get(e + 2 * k);
            tm[u][k] = get(e + 2 * F::K + 2 * k);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < F::K; ++k) {
            A[k] = acc_comb<F>(k, A[k], t[u][k]);
            Am[k] = acc_comb<F>(k, Am[k], tm[u][k]);
          }
      }
      for (; j < d; ++j) {
        const double* e = T + HDR + (size_t)(j * m + piece(code0, j, P)) * ENT + E_T;
#pragma unroll
        for (int k = 0; k < F::K; ++k) {
          A[k] = acc_comb<F>(k, A[k], get(e + 2 * k));
          Am[k] = acc_comb<F>(k, Am[k], get(e + 2 * F::K + 2 * k));
        }
      }
#pragma unroll(GT ? GT : 1)
      for (int q = 0; q < G; ++q) {
        Iv B[2], Bm[2];
#pragma unroll
        for (int k = 0; k < F::K; ++k) {
          B[k] = A[k];
          Bm[k] = Am[k];
        }
#pragma unroll(GT ? 3 : 1)
        for (int j = 0; j < h; ++j) {
          const int p = GT ? ((q >> j) & 1) : piece((uint32_t)q, j, P);
          const double* e = T + HDR + (size_t)(j * m + p) * ENT + E_T;
#pragma unroll
          for (int k = 0; k < F::K; ++k) {
            B[k] = acc_comb<F>(k, B[k], get(e + 2 * k));
            Bm[k] = acc_comb<F>(k, Bm[k], get(e + 2 * F::K + 2 * k));
          }
        }
        // f(midpoint) >= lb: a child with lb > GUB_old cannot lower GUB
        const double lbq = canon_lb(outer_lo<F>(B, n));
        clb[gi * G + q] = lbq;
        if (lbq <= gub0) best = fmin(best, outer_hi<F>(Bm, n));
        if (pot) pot_append(ctl, pot, lbq <= gub0, (uint32_t)(gi * G + q));
        if (lbq <= gub0) pm |= 1u << q;
      }
    }
    }  // gi < ngroups
    if constexpr (GT == 8) {
      if (pbits) {
        // a warp's 32 groups are 256 consecutive children = 4 words; every
        // word below ceil(B m^d / 64) is written (zeros included), so the
        // bitmap needs no clearing between iterations
        const int lane = threadIdx.x & 31;
        unsigned long long v = (unsigned long long)pm << (8 * (lane & 7));
        v |= __shfl_xor_sync(0xffffffffu, v, 1);
        v |= __shfl_xor_sync(0xffffffffu, v, 2);
        v |= __shfl_xor_sync(0xffffffffu, v, 4);
        if ((lane & 7) == 0 && gi < ngroups) pbits[gi >> 3] = v;
        const unsigned np = __reduce_add_sync(0xffffffffu, (unsigned)__popc(pm));
        if (lane == 0 && np) atomicAdd(&ctl->npot, (unsigned long long)np);
      }
    }
  }
  __shared__ double s_m[TPB / 32];
  best = warp_min(best);
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < TPB / 32; ++w) best = fmin(best, s_m[w]);
    if (best < CUDART_INF) atomicMin(&ctl->gub_key, (unsigned long long)okey(best));
  }
}

template <class F, int GT>
__global__ void __launch_bounds__(TPB, 4) k_child_eval(Problem P, Ctl* __restrict__ ctl,
                                                               const double* __restrict__ tab, int tab_stride,
                                                               double* __restrict__ clb, uint64_t* zero_a,
                                                               uint64_t* zero_b, long nzero, uint32_t* zero_ctr,
                                                               unsigned int* zero_hist, const double* ppart,
                                                               uint64_t* pbits) {
  child_eval_dev<F, GT>(P, ctl, tab, tab_stride, clb, zero_a, zero_b, nzero, zero_ctr, zero_hist, nullptr, ppart,
                        pbits);
}

// Pass 2a: stable compaction of the candidates (children with lb <= GUB,
// line 140) into cand[] (decoupled look-back).
// next tile of a decoupled-look-back scan: a ticket (any launch) or, in a
// co-resident grid (STATIC), tile = block + k * grid -- every block walks its
// tiles in increasing order and a tile only waits on lower tiles, so no
// ticket atomics are needed
template <bool STATIC>
__device__ __forceinline__ uint32_t next_tile(uint32_t* tile_ctr, uint32_t k) {
  if constexpr (STATIC) {
    return blockIdx.x + k * gridDim.x;
  } else {
    __shared__ uint32_t s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    __syncthreads();
    return tile;
  }
}

template <bool STATIC = false>
__device__ void cand_dev(const Problem& P, Ctl* __restrict__ ctl, const double* __restrict__ clb,
                         uint32_t* __restrict__ cand, uint64_t* desc, uint32_t* tile_ctr) {
  for (uint32_t kt = 0;; ++kt) {
  const uint32_t tile = next_tile<STATIC>(tile_ctr, kt);
  const long total = (long)ctl->B * P.kids;
  const long ntiles = (total + TILE - 1) / TILE;
  if ((long)tile >= ntiles) break;  // tiles past the end: nobody waits on them
  const double gub = okey_inv(ctl->gub_key);
  const long g0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (g0 + q < total && clb[g0 + q] <= gub) f |= 1u << q;
  uint32_t c1[1] = {(uint32_t)__popc(f)}, ex[1], tot[1];
  block_exclusive_scan<1, TPB>(c1, ex, tot);
  uint64_t pfx[1];
  dl_lookback<1>(desc, tile, tot, pfx);
  uint64_t pos = pfx[0] + ex[0];
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (f & (1u << q)) cand[pos++] = (uint32_t)(g0 + q);
  if ((long)tile == ntiles - 1 && threadIdx.x == 0) ctl->ncand = pfx[0] + tot[0];
  }
}

// Pass 2b: first-order test (lines 142-144) of every candidate, one thread
// per candidate on a dense list (no divergence from pruned children).
template <class F>
__device__ void mono_dev(const Problem& P, const Ctl* __restrict__ ctl, const double* __restrict__ tab,
                         int tab_stride, const uint32_t* __restrict__ cand, uint8_t* __restrict__ ok) {
  const long nc = (long)ctl->ncand;
  for (long k = (long)blockIdx.x * TPB + threadIdx.x; k < nc; k += (long)gridDim.x * TPB) {
    ChildIdx ci = child_of(cand[k], P);
    ok[k] = (!P.mono || child_mono_ok<F>(P, tab + (size_t)ci.b * tab_stride, ci.code)) ? 1 : 0;
  }
}

// Pass 2c: insert the surviving candidates into L after its current end, in
// (parent, code) order (line 146), stable decoupled-look-back compaction.
__device__ void iter_end_dev(Ctl* ctl, long kids);
// the next k_fused list phase may take the single-block path: every live
// record is in the hot index (tau = ~0) and, with this iteration's survivors,
// it has at most min(bmax, LSMAX * TPB) entries (decided here, before the barrier,
// so that every block reads the same flag)
__device__ __forceinline__ void set_list_fast(Ctl* ctl, unsigned long long nsurv_hot) {
  const unsigned long long nh = ctl->nhot + nsurv_hot;
  ctl->list_fast =
      ctl->hot_valid && ctl->tau_key == ~0ull && nh <= ctl->bmax && nh <= (unsigned long long)(LSMAX * TPB);
}
// MONO: the first-order test of each candidate is evaluated here (fused
// kernel) instead of being read from ok[] (k_mono)
template <class F, bool MONO>
__device__ void emit_dev(const Problem& P, Ctl* __restrict__ ctl, const double* __restrict__ tab, int tab_stride,
                         const double* __restrict__ clb, const uint32_t* __restrict__ cand,
                         const uint8_t* __restrict__ ok, const int32_t* __restrict__ new_slot, Pool out,
                         uint64_t* desc, uint32_t* tile_ctr, bool finish, uint32_t* hot0, uint32_t* hot1) {
  // counters: 0 every survivor (-> L), 1 survivors with key < tau (-> hot index)
  PROBE_BEGIN
  uint32_t* hot = hot0 ? (ctl->hsel ? hot1 : hot0) : nullptr;
  const unsigned long long tau = ctl->tau_key;
  for (uint32_t kt = 0;; ++kt) {
  const uint32_t tile = next_tile<MONO>(tile_ctr, kt);  // the fused kernel (MONO) is co-resident
  const long nc = (long)ctl->ncand;
  const long ntiles = (nc + TILE - 1) / TILE;
  if (nc == 0) {
    if (tile == 0 && threadIdx.x == 0) {
      ctl->nsurv = 0;
      ctl->nsurv_hot = 0;
      if (finish) {
        ctl->pending_end = 1;
        set_list_fast(ctl, 0ull);
      }
    }
    break;
  }
  if ((long)tile >= ntiles) break;
  const long k0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  const long kbeg = (long)tile * TILE;
  // MONO: width and (separable f) first-order flags of the tile's candidates,
  // one warp per candidate with a lane per split variable
  __shared__ uint8_t s_ok[MONO ? TILE : 1];
  __shared__ double s_w[MONO ? TILE : 1];
  if constexpr (MONO) {
    const int cnt = (int)min((long)TILE, nc - kbeg);
    const int lane = threadIdx.x & 31;
    for (int q = threadIdx.x >> 5; q < cnt; q += TPB / 32) {
      ChildIdx ci = child_of(cand[kbeg + q], P);
      const double* T = tab + (size_t)ci.b * tab_stride;
      double wl = 0.0;
      bool bad = false;
      if (lane < P.d) {
        const double* e = T + HDR + (size_t)(lane * P.m + piece(ci.code, lane, P)) * ENT;
        wl = __dsub_rn(e[E_HI], e[E_LO]);
        if constexpr (F::SEP) bad = e[E_T + 4 * F::K + 2 * F::KG] != 0.0;
      }
      wl = warp_max(wl);
      const unsigned anybad = __ballot_sync(0xffffffffu, bad);
      if (lane == 0) {
        s_w[q] = fmax(T[H_WREST], wl);
        s_ok[q] = anybad == 0u;
      }
    }
    PROBE(1)
    __syncthreads();
    PROBE(2)
  }
  uint32_t f = 0, fh = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    bool okq = false;
    if (k0 + q < nc) {
      if constexpr (MONO) {
        if constexpr (F::SEP) {
          okq = !P.mono || s_ok[k0 + q - kbeg] != 0;
        } else {
          ChildIdx ci = child_of(cand[k0 + q], P);
          okq = !P.mono || child_mono_ok<F>(P, tab + (size_t)ci.b * tab_stride, ci.code);
        }
      } else {
        okq = ok[k0 + q] != 0;
      }
    }
    if (okq) {
      f |= 1u << q;
      if (hot && okey(clb[cand[k0 + q]]) < tau) fh |= 1u << q;
    }
  }
  PROBE(3)
  uint32_t c2[2] = {(uint32_t)__popc(f), (uint32_t)__popc(fh)}, ex[2], tot[2];
  block_exclusive_scan<2, TPB>(c2, ex, tot);
  PROBE(4)
  uint64_t pfx[2];
  dl_lookback<2>(desc, tile, tot, pfx);
  PROBE(5)
  const uint64_t base = ctl->pcount, cap = ctl->pool_cap, hbase = ctl->nhot;
  uint64_t pos = base + pfx[0] + ex[0], hpos = hbase + pfx[1] + ex[1];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    if (f & (1u << q)) {
      if (pos < cap) {
        uint32_t g = cand[k0 + q];
        ChildIdx ci = child_of(g, P);
        out.lb[pos] = clb[g];
        if constexpr (MONO)
          out.w[pos] = s_w[k0 + q - kbeg];
        else
          out.w[pos] = child_width(P, tab + (size_t)ci.b * tab_stride, ci.code);
        out.slot[pos] = new_slot[ci.b];
        out.code[pos] = ci.code;
        if (fh & (1u << q)) hot[hpos++] = (uint32_t)pos;
      }
      ++pos;
    }
  }
  if ((long)tile == ntiles - 1 && threadIdx.x == 0) {
    ctl->nsurv = pfx[0] + tot[0];
    ctl->nsurv_hot = pfx[1] + tot[1];
    if (base + pfx[0] + tot[0] > cap) {
      ctl->err = -2;  // IB_ENOSPACE
      ctl->done = 4;
    }
    // the iteration end is applied by the next k_list (other tiles may still
    // be reading pcount as their base here)
    if (finish) {
      ctl->pending_end = 1;
      set_list_fast(ctl, pfx[1] + tot[1]);
    }
  }
  PROBE(6)
  }
  PROBE(7)
  PROBE_END(0)
}

// k_fused, one block: the insertion pass when at most PCAP children had
// lb <= GUB at the iteration start (the candidates, lb <= final GUB, are
// among them).  Sorting the potential list by child index gives the same
// survivors in the same order as k_cand -> k_mono -> k_emit, without a scan
// over all children.
template <class F>
// Returns true when it also ran the next iteration's list phase (select):
// the common deep-dive case -- every live record is hot (tau = ~0), the hot
// index held nothing before this iteration's survivors and they fit one
// selection (<= min(bmax, TPB)) -- takes the iteration end and the list
// phase's decisions (stop test, batch size, selection of every live entry in
// list order) directly from the survivors in registers, with the same
// results as list_small_dev.
__device__ bool emit_small_dev(const Problem& P, Ctl* __restrict__ ctl, const double* __restrict__ tab,
                               int tab_stride, const double* __restrict__ clb, const int32_t* __restrict__ new_slot,
                               Pool out, const uint32_t* __restrict__ pot, int np, uint32_t* hot0, uint32_t* hot1,
                               bool try_select = false, long kids = 0, int32_t* sel_slot = nullptr,
                               uint32_t* sel_code = nullptr) {
  __shared__ uint32_t s_in[PCAP], s_g[PCAP];
  __shared__ uint8_t s_c[PCAP], s_ok[PCAP];
  __shared__ double s_w[PCAP];
  const int t = threadIdx.x, lane = t & 31;
  const double gub = okey_inv(ctl->gub_key);
  uint32_t* hot = ctl->hsel ? hot1 : hot0;
  const unsigned long long tau = ctl->tau_key;
  const uint32_t gin = t < np ? pot[t] : 0xffffffffu;
  if (t < PCAP) s_in[t] = gin;
  __syncthreads();
  if (t < np) {  // rank sort (child indices are distinct)
    int r = 0;
    for (int j = 0; j < np; ++j) r += s_in[j] < gin;
    s_g[r] = gin;
  }
  __syncthreads();
  const uint32_t g = t < np ? s_g[t] : 0u;
  const double lb = t < np ? clb[g] : CUDART_INF;
  const bool cand = t < np && lb <= gub;
  if (t < PCAP) s_c[t] = cand;
  // few candidates: first-order test with a warp per candidate (lane per
  // split variable); many: a thread per candidate (more of them at once)
  const bool warp_mono = __syncthreads_count(cand) <= TPB / 32;
  for (int k = t >> 5; warp_mono && k < np; k += TPB / 32) {
    if (!s_c[k]) continue;  // warp-uniform
    ChildIdx ci = child_of(s_g[k], P);
    const double* T = tab + (size_t)ci.b * tab_stride;
    double wl = 0.0;
    bool bad = false;
    if (lane < P.d) {
      const double* e = T + HDR + (size_t)(lane * P.m + piece(ci.code, lane, P)) * ENT;
      wl = __dsub_rn(e[E_HI], e[E_LO]);
      if constexpr (F::SEP) bad = e[E_T + 4 * F::K + 2 * F::KG] != 0.0;
    }
    wl = warp_max(wl);
    unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if constexpr (!F::SEP)
      if (warp_mono) anybad = (!P.mono || child_mono_ok_warp<F>(P, T, ci.code)) ? 0u : 1u;
    if (lane == 0) {
      s_w[k] = fmax(T[H_WREST], wl);
      s_ok[k] = anybad == 0u;
    }
  }
  __syncthreads();
  bool surv = false;
  if (cand) {
    if (warp_mono) {
      surv = !P.mono || s_ok[t] != 0;
    } else {  // many candidates: a thread per candidate
      ChildIdx ci = child_of(g, P);
      const double* T = tab + (size_t)ci.b * tab_stride;
      s_w[t] = child_width(P, T, ci.code);
      surv = !P.mono || child_mono_ok<F>(P, T, ci.code);
    }
  }
  const bool hotf = surv && hot0 && okey(lb) < tau;
  uint32_t c3[3] = {cand ? 1u : 0u, surv ? 1u : 0u, hotf ? 1u : 0u}, ex[3], tot[3];
  block_exclusive_scan<3, TPB>(c3, ex, tot);
  const uint64_t base = ctl->pcount, cap = ctl->pool_cap, hbase = ctl->nhot;
  const bool combined = try_select && hbase == 0 && ctl->hot_valid && tau == ~0ull && tot[2] == tot[1] &&
                        tot[1] <= ctl->bmax && tot[1] <= (uint32_t)TPB && base + tot[1] <= cap && !ctl->done;
  int32_t my_slot = 0;
  uint32_t my_code = 0;
  if (surv) {
    const uint64_t pos = base + ex[1];
    if (pos < cap) {
      ChildIdx ci = child_of(g, P);
      my_slot = new_slot[ci.b];
      my_code = ci.code;
      out.lb[pos] = lb;
      out.w[pos] = s_w[t];
      out.slot[pos] = my_slot;
      out.code[pos] = my_code;
      if (hotf) hot[hbase + ex[2]] = (uint32_t)pos;
    }
  }
  if (combined) {
    // iteration end (iter_end_dev) and the list phase (list_small_dev) on the
    // survivors: all of them are live (lb <= GUB) and form the hot index
    __shared__ unsigned long long s_mk;
    __shared__ double s_mw;
    if (t == 0) {
      s_mk = ~0ull;
      s_mw = 0.0;
    }
    __syncthreads();
    const unsigned long long key = surv ? okey(lb) : ~0ull;
    unsigned long long mk = key;
    double mw = surv ? s_w[t] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long q = __shfl_xor_sync(0xffffffffu, mk, o);
      mk = q < mk ? q : mk;
      mw = fmax(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    }
    if (lane == 0) {
      if (mk != ~0ull) atomicMin(&s_mk, mk);
      atomicMax((unsigned long long*)&s_mw, (unsigned long long)__double_as_longlong(mw));
    }
    __syncthreads();
    const unsigned long long nlive = tot[1], minkey = s_mk;
    const unsigned long long Bold = ctl->B, iter1 = ctl->iter + 1, free1 = ctl->free_top - Bold;
    unsigned long long bytes = 12ull * nlive;
    int done = 0;
    bool wpass = false;
    if (nlive == 0) {
      done = 3;
    } else if (__dsub_ru(gub, okey_inv(minkey)) <= ctl->eps_f) {
      wpass = true;
      bytes += 20ull * nlive;
      if (s_mw <= ctl->eps_x) done = 1;
    }
    if (!done && iter1 >= ctl->max_iter) done = 2;
    if (!done && free1 < nlive) done = 4;
    if (!done && surv) {  // selection: every live entry in list order
      sel_slot[ex[1]] = my_slot;
      sel_code[ex[1]] = my_code;
      out.lb[base + ex[1]] = CUDART_INF;  // removed from L
    }
    if (t == 0) {
      // iteration end
      ctl->ncand = tot[0];
      ctl->nsurv = tot[1];
      ctl->nsurv_hot = tot[2];
      ctl->sum_cand += tot[0];
      ctl->sum_pool += base;
      ctl->sum_B += Bold;
      ctl->free_top = free1;
      ctl->pcount = base + tot[1];
      ctl->iter = iter1;
      ctl->evals += Bold * (unsigned long long)kids;
      ctl->pending_end = 0;
      if (wpass) {
        ctl->nwidth += 1;
        const unsigned long long wb = (unsigned long long)__double_as_longlong(s_mw);
        if (wb > ctl->acc_max_w) ctl->acc_max_w = wb;
      }
      ctl->live = nlive;
      ctl->min_lb_key = minkey;
      if (done) {
        ctl->nhot = tot[2];  // the survivors stay in the hot index
        ctl->max_w_bits = ctl->acc_max_w;
        if (done == 4) ctl->err = -2;
        ctl->list_bytes += bytes;
        ctl->done = done;
      } else {
        bytes += 16ull * nlive;
        ctl->nhot_keep = 0;
        ctl->hsel ^= 1;
        ctl->nhot = 0;
        ctl->B = nlive;
        ctl->known = 0;
        ctl->prefix = 0;
        ctl->need = nlive;
        ctl->list_bytes += bytes;
      }
    }
    __syncthreads();
    return true;
  }
  if (t == 0) {
    ctl->ncand = tot[0];
    ctl->nsurv = tot[1];
    ctl->nsurv_hot = tot[2];
    if (base + tot[1] > cap) {
      ctl->err = -2;  // IB_ENOSPACE
      ctl->done = 4;
    }
    ctl->pending_end = 1;
    set_list_fast(ctl, tot[2]);
  }
  __syncthreads();
  return false;
}

// k_fused: candidates (lb <= GUB, line 140), first-order test (lines
// 142-144) and insertion into L (line 146) in one pass over the children of
// the batch, static tiles; the same survivors in the same order as
// k_cand -> k_mono -> k_emit.  Scan counters: 0 candidates, 1 survivors (-> L),
// 2 survivors with key < tau (-> hot index).  The descriptors (desc, 3 per
// tile) were zeroed by child_eval_dev.
template <class F>
__device__ void cand_emit_dev(const Problem& P, Ctl* __restrict__ ctl, const double* __restrict__ tab, int tab_stride,
                              const double* __restrict__ clb, const int32_t* __restrict__ new_slot, Pool out,
                              uint64_t* desc, uint32_t* hot0, uint32_t* hot1) {
  __shared__ uint32_t s_cidx[TILE];
  __shared__ uint8_t s_ok[TILE];
  __shared__ double s_w[TILE];
  uint32_t* hot = ctl->hsel ? hot1 : hot0;
  const unsigned long long tau = ctl->tau_key;
  const double gub = okey_inv(ctl->gub_key);
  const long total = (long)ctl->B * P.kids;
  const long ntiles = (total + TILE - 1) / TILE;
  const int lane = threadIdx.x & 31;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long g0 = tile * TILE + (long)threadIdx.x * IPT;
    uint32_t fc = 0;
    double lbv[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      lbv[q] = g0 + q < total ? clb[g0 + q] : CUDART_INF;
      if (g0 + q < total && lbv[q] <= gub) fc |= 1u << q;
    }
    uint32_t c1[1] = {(uint32_t)__popc(fc)}, ex1[1], tot1[1];
    block_exclusive_scan<1, TPB>(c1, ex1, tot1);
    {
      uint32_t pl = ex1[0];
#pragma unroll
      for (int q = 0; q < IPT; ++q)
        if (fc & (1u << q)) s_cidx[pl++] = (uint32_t)(g0 + q);
    }
    const int ncl = (int)tot1[0];
    __syncthreads();
    // widths (+ first-order flags): a warp per candidate, a lane per split
    // variable; with many candidates the non-separable test runs a thread
    // per candidate instead
    const bool warp_mono = ncl <= TPB / 32;
    for (int k = threadIdx.x >> 5; warp_mono && k < ncl; k += TPB / 32) {
      ChildIdx ci = child_of(s_cidx[k], P);
      const double* T = tab + (size_t)ci.b * tab_stride;
      double wl = 0.0;
      bool bad = false;
      if (lane < P.d) {
        const double* e = T + HDR + (size_t)(lane * P.m + piece(ci.code, lane, P)) * ENT;
        wl = __dsub_rn(e[E_HI], e[E_LO]);
        if constexpr (F::SEP) bad = e[E_T + 4 * F::K + 2 * F::KG] != 0.0;
      }
      wl = warp_max(wl);
      unsigned anybad = __ballot_sync(0xffffffffu, bad);
      if constexpr (!F::SEP)
        if (warp_mono) anybad = (!P.mono || child_mono_ok_warp<F>(P, T, ci.code)) ? 0u : 1u;
      if (lane == 0) {
        s_w[k] = fmax(T[H_WREST], wl);
        s_ok[k] = anybad == 0u;
      }
    }
    __syncthreads();
    uint32_t f = 0, fh = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int k = threadIdx.x * IPT + q;
      if (k < ncl) {
        bool okq;
        if (warp_mono) {
          okq = !P.mono || s_ok[k] != 0;
        } else {  // many candidates: a thread per candidate
          ChildIdx ci = child_of(s_cidx[k], P);
          const double* T = tab + (size_t)ci.b * tab_stride;
          s_w[k] = child_width(P, T, ci.code);
          okq = !P.mono || child_mono_ok<F>(P, T, ci.code);
        }
        if (okq) {
          f |= 1u << q;
          if (okey(clb[s_cidx[k]]) < tau) fh |= 1u << q;
        }
      }
    }
    uint32_t c3[3] = {threadIdx.x == 0 ? (uint32_t)ncl : 0u, (uint32_t)__popc(f), (uint32_t)__popc(fh)}, ex[3], tot[3];
    block_exclusive_scan<3, TPB>(c3, ex, tot);
    uint64_t pfx[3];
    dl_lookback<3>(desc, (uint32_t)tile, tot, pfx);
    const uint64_t base = ctl->pcount, cap = ctl->pool_cap, hbase = ctl->nhot;
    uint64_t pos = base + pfx[1] + ex[1], hpos = hbase + pfx[2] + ex[2];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      if (f & (1u << q)) {
        if (pos < cap) {
          const int k = threadIdx.x * IPT + q;
          const uint32_t g = s_cidx[k];
          ChildIdx ci = child_of(g, P);
          out.lb[pos] = clb[g];
          out.w[pos] = s_w[k];
          out.slot[pos] = new_slot[ci.b];
          out.code[pos] = ci.code;
          if (fh & (1u << q)) hot[hpos++] = (uint32_t)pos;
        }
        ++pos;
      }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
      ctl->ncand = pfx[0] + tot[0];
      ctl->nsurv = pfx[1] + tot[1];
      ctl->nsurv_hot = pfx[2] + tot[2];
      if (base + pfx[1] + tot[1] > cap) {
        ctl->err = -2;  // IB_ENOSPACE
        ctl->done = 4;
      }
      ctl->pending_end = 1;
      set_list_fast(ctl, pfx[2] + tot[2]);
    }
    __syncthreads();  // shared arrays are reused by the next tile
  }
}

#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_cand(const Problem P, Ctl* __restrict__ ctl, const double* __restrict__ clb,
                                              uint32_t* __restrict__ cand, uint64_t* desc, uint32_t* tile_ctr) {
  if (ctl->done) return;
  cand_dev(P, ctl, clb, cand, desc, tile_ctr);
}
#endif  // IBNB_OBJ_TU
template <class F>
__global__ void __launch_bounds__(TPB, 4) k_mono(Problem P, const Ctl* __restrict__ ctl, const double* __restrict__ tab,
                                                 int tab_stride, const uint32_t* __restrict__ cand,
                                                 uint8_t* __restrict__ ok) {
  if (ctl->done) return;
  mono_dev<F>(P, ctl, tab, tab_stride, cand, ok);
}
// Insertion (a5 + a6) in three phases of one cooperative kernel:
//  (A) every tile of TILE children lists its candidates (lb <= GUB, line 140)
//      in child order in its own slots of cand[] and counts them;
//  (B) grid barrier; the candidates of all tiles are numbered (a scan of the
//      tile counts in every block) and tested (first-order test, lines
//      142-144) by all warps of the grid, a warp per candidate and a lane
//      per split variable -- candidates crowd into the few tiles of the
//      parents near a minimiser, so a per-tile test would serialise there;
//      survivors are counted per tile (integer atomics);
//  (C) grid barrier; every block scans the tile survivor counts and
//      compacts its tiles' survivors into L at their stable positions.
// Sparse insertion (graph path, bisection with G = 8, at most SCAP potential
// candidates): the same candidates, first-order test and stable compaction
// as cand_emit_dev, but a tile covers SP_WORDS words of the potential bitmap
// written by k_child_eval (32,768 children) and only the children whose bit
// is set (lb <= GUB at the iteration start, a superset of the candidates
// lb <= GUB, line 140) are read: 32x fewer tiles in the look-back chain and
// 1/64 of the bytes.  Same survivors in the same order (bit-identical L).
constexpr int SP_WORDS = 64;       // 64-bit bitmap words per tile (4,096 children: a few candidates per tile,
                                   // one warp each -- the first-order tests spread over the grid)
constexpr int SCAP = 4096;         // potential candidates of one iteration
template <class F>
__device__ void cand_emit_sparse_dev(const Problem& P, Ctl* __restrict__ ctl, const double* __restrict__ tab,
                                     int tab_stride, const double* __restrict__ clb,
                                     const int32_t* __restrict__ new_slot, Pool out, const uint64_t* pbits,
                                     uint64_t* desc, uint32_t* hot0, uint32_t* hot1) {
  __shared__ uint32_t s_idx[SCAP];
  __shared__ uint8_t s_f[SCAP];
  __shared__ uint32_t s_cnt[3];
  uint32_t* hot = ctl->hsel ? hot1 : hot0;
  const unsigned long long tau = ctl->tau_key;
  const double gub = okey_inv(ctl->gub_key);
  const long total = (long)ctl->B * P.kids;
  const long nwords = (total + 63) / 64;
  const long ntiles = (nwords + SP_WORDS - 1) / SP_WORDS;
  const int t = threadIdx.x;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // (1) the potential candidates of the tile, in child order
    const long w0 = tile * SP_WORDS + 2 * t;
    const bool mine = 2 * t < SP_WORDS;
    const uint64_t a = mine && w0 < nwords ? __ldcg(&pbits[w0]) : 0ull;
    const uint64_t b = mine && w0 + 1 < nwords ? __ldcg(&pbits[w0 + 1]) : 0ull;
    uint32_t c1[1] = {(uint32_t)(__popcll(a) + __popcll(b))}, ex1[1], tot1[1];
    block_exclusive_scan<1, TPB>(c1, ex1, tot1);
    {
      uint32_t pos = ex1[0];
      for (uint64_t v = a; v; v &= v - 1) s_idx[pos++] = (uint32_t)(w0 * 64 + __ffsll((long long)v) - 1);
      for (uint64_t v = b; v; v &= v - 1) s_idx[pos++] = (uint32_t)((w0 + 1) * 64 + __ffsll((long long)v) - 1);
    }
    const int np = (int)tot1[0];
    if (t < 3) s_cnt[t] = 0;
    __syncthreads();
    // (2) candidates (lb <= GUB), a thread each
    {
      uint32_t nc = 0;
      for (int k = t; k < np; k += TPB) {
        const uint8_t f = clb[s_idx[k]] <= gub ? 1 : 0;
        s_f[k] = f;
        nc += f;
      }
      nc = __reduce_add_sync(0xffffffffu, nc);
      if ((t & 31) == 0 && nc) atomicAdd(&s_cnt[0], nc);
    }
    __syncthreads();
    // (3) the first-order test (lines 142-144): a warp per candidate (a lane
    // per split variable) when the tile has few, else a thread per candidate
    const int lane = t & 31;
    if (s_cnt[0] <= 4u * (TPB / 32)) {  // uniform
      for (int k = t >> 5; k < np; k += TPB / 32) {
        if (!(s_f[k] & 1)) continue;  // warp-uniform
        const uint32_t g = s_idx[k];
        ChildIdx ci = child_of(g, P);
        const double* T = tab + (size_t)ci.b * tab_stride;
        bool ok = true;
        if (P.mono) {
          if constexpr (F::SEP) {
            bool bad = false;
            if (lane < P.d)
              bad = T[HDR + (size_t)(lane * P.m + piece(ci.code, lane, P)) * ENT + E_T + 4 * F::K + 2 * F::KG] != 0.0;
            ok = __ballot_sync(0xffffffffu, bad) == 0u;
          } else {
            ok = child_mono_ok_warp<F>(P, T, ci.code);
          }
        }
        if (lane == 0 && ok) s_f[k] |= okey(clb[g]) < tau ? 6 : 2;
      }
    } else {
      for (int k = t; k < np; k += TPB) {
        if (!(s_f[k] & 1)) continue;
        const uint32_t g = s_idx[k];
        ChildIdx ci = child_of(g, P);
        if (!P.mono || child_mono_ok<F>(P, tab + (size_t)ci.b * tab_stride, ci.code))
          s_f[k] |= okey(clb[g]) < tau ? 6 : 2;
      }
    }
    __syncthreads();
    {
      uint32_t my1 = 0, my2 = 0;
      for (int k = t; k < np; k += TPB) {
        my1 += (s_f[k] >> 1) & 1;
        my2 += (s_f[k] >> 2) & 1;
      }
      my1 = __reduce_add_sync(0xffffffffu, my1);
      my2 = __reduce_add_sync(0xffffffffu, my2);
      if (lane == 0 && my1) atomicAdd(&s_cnt[1], my1);
      if (lane == 0 && my2) atomicAdd(&s_cnt[2], my2);
    }
    __syncthreads();
    uint32_t tot[3] = {s_cnt[0], s_cnt[1], s_cnt[2]};
    uint64_t pfx[3];
    dl_lookback<3>(desc, (uint32_t)tile, tot, pfx);
    // (3) stable compaction of the survivors into L (and the hot index)
    const uint64_t base = ctl->pcount, cap = ctl->pool_cap, hbase = ctl->nhot;
    uint64_t run = 0, hrun = 0;
    for (int k0 = 0; k0 < np; k0 += TPB) {
      const int k = k0 + t;
      const uint8_t f = k < np ? s_f[k] : 0;
      uint32_t c2[2] = {(uint32_t)((f >> 1) & 1), (uint32_t)((f >> 2) & 1)}, ex[2], tt[2];
      block_exclusive_scan<2, TPB>(c2, ex, tt);
      if (f & 2) {
        const uint64_t pos = base + pfx[1] + run + ex[0];
        if (pos < cap) {
          const uint32_t g = s_idx[k];
          ChildIdx ci = child_of(g, P);
          out.lb[pos] = clb[g];
          out.w[pos] = child_width(P, tab + (size_t)ci.b * tab_stride, ci.code);
          out.slot[pos] = new_slot[ci.b];
          out.code[pos] = ci.code;
          if (f & 4) hot[hbase + pfx[2] + hrun + ex[1]] = (uint32_t)pos;
        }
      }
      run += tt[0];
      hrun += tt[1];
    }
    if (tile == ntiles - 1 && t == 0) {
      ctl->ncand = pfx[0] + tot[0];
      ctl->nsurv = pfx[1] + tot[1];
      ctl->nsurv_hot = pfx[2] + tot[2];
      if (base + pfx[1] + tot[1] > cap) {
        ctl->err = -2;  // IB_ENOSPACE
        ctl->done = 4;
      }
      ctl->pending_end = 1;
      set_list_fast(ctl, pfx[2] + tot[2]);
    }
    __syncthreads();  // shared arrays are reused by the next tile
  }
}

// insertion in one pass (a5 + a6): candidates lb <= GUB, the first-order
// test, stable compaction of the survivors into L -- k_cand + k_mono + k_emit
// of the explicit-batch path as one cooperative kernel (static tiles with
// decoupled look-back, every block resident).  Measured against two- and
// three-phase variants (tile counts + grid barrier + scan, candidates tested
// by every warp of the grid): this single pass was the fastest.
template <class F>
__global__ void __launch_bounds__(TPB) k_insert(Problem P, IterBufs w) {
  if (w.ctl->done) return;
  if constexpr (!F::CHAIN) {
    // uniform: the potential bitmap exists (k_child_eval's G = 8 path) and
    // the potential candidates fit one tile's list
    const bool sparse = w.pbits && P.m == 2 && P.G == 8 && w.ctl->npot <= (unsigned long long)SCAP;
    if (w.tstamp && blockIdx.x == 0 && threadIdx.x == 0) {  // trace statistics
      atomicAdd(&w.tstamp[22], 1ull);
      atomicAdd(&w.tstamp[23], sparse ? 1ull : 0ull);
      atomicAdd(&w.tstamp[24], w.ctl->npot);
    }
    if (sparse) {
      cand_emit_sparse_dev<F>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.pbits, w.desc2, w.hot0,
                              w.hot1);
      return;
    }
  }
  cand_emit_dev<F>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.desc2, w.hot0, w.hot1);
}
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_emit(const Problem P, Ctl* __restrict__ ctl, const double* __restrict__ tab,
                                              int tab_stride, const double* __restrict__ clb,
                                              const uint32_t* __restrict__ cand, const uint8_t* __restrict__ ok,
                                              const int32_t* __restrict__ new_slot, Pool out, uint64_t* desc,
                                              uint32_t* tile_ctr, int finish, uint32_t* hot0, uint32_t* hot1) {
  if (ctl->done) return;
  emit_dev<ObjExample, false>(P, ctl, tab, tab_stride, clb, cand, ok, new_slot, out, desc, tile_ctr, finish != 0, hot0,
                              hot1);
}
#endif  // IBNB_OBJ_TU

// ============================================================ list L kernels
// Statistics of the live part of L (lb <= GUB, lines 136 and 148-150) and the
// histogram of the top 8 bits of the live lower bounds (radix pass 1).  The
// last block to finish (threadfence + ticket) takes the iteration's control
// decisions: stop test (line 148: every region narrower than eps_x; line
// 150: GUB - GLB <= eps_f), batch size B = min(live, bmax) (line 130, reading
// R1) and the first radix digit of the B-th smallest key.

// pick the radix digit of the B-th smallest key from hist with the whole
// block (256 threads, one bin each); zero hist
__device__ void block_pick_digit(Ctl* ctl, unsigned int* hist) {
  __shared__ unsigned long long s_inc[256];
  __shared__ int s_dig;
  const int t = threadIdx.x;
  unsigned long long h = t < 256 ? hist[t] : 0ull;
  if (t < 256) s_inc[t] = h;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // Hillis-Steele inclusive scan
    unsigned long long v = (t < 256 && t >= o) ? s_inc[t - o] : 0ull;
    __syncthreads();
    if (t < 256) s_inc[t] += v;
    __syncthreads();
  }
  const unsigned long long need = ctl->need;
  if (t == 0) s_dig = 255;
  __syncthreads();
  if (t < 256) {
    unsigned long long before = t ? s_inc[t - 1] : 0ull;
    if (before < need && s_inc[t] >= need) s_dig = t;
  }
  __syncthreads();
  if (t == 0) {
    int dig = s_dig;
    unsigned long long before = dig ? s_inc[dig - 1] : 0ull;
    unsigned long long cnt = s_inc[dig] - before;
    ctl->need = need - before;
    ctl->prefix = (ctl->prefix << 8) | (unsigned long long)dig;
    ctl->known += 8;
    if (cnt == ctl->need || ctl->known >= 64) ctl->resolved = 1;
  }
  if (t < 256) hist[t] = 0;
  __syncthreads();
}

// histogram increment aggregated over the lanes of a warp hitting the same bin
// (lower bounds cluster, so most lanes of a warp share a bin).  Must be
// called by all 32 lanes (callers loop with a warp-uniform condition).
__device__ __forceinline__ void hist_add(unsigned int* s_h, unsigned bin, bool valid) {
  const unsigned active = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned peers = __match_any_sync(active, bin);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&s_h[bin], (unsigned)__popc(peers));
}

__device__ __forceinline__ bool last_block(Ctl* ctl) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->blocks_done, 1u) == gridDim.x - 1;
  __syncthreads();
  return s_last;
}

// accumulate the statistics of this block's share of L into ctl->acc_* and
// the top-8-bit histogram of the live keys
template <bool WITH_W = true>
__device__ void stats_accum_dev(const Pool& p, Ctl* ctl, unsigned int* hist) {
  __shared__ unsigned int s_h[256];
  for (int i = threadIdx.x; i < 256; i += TPB) s_h[i] = 0;
  __syncthreads();
  const double gub = okey_inv(ctl->gub_key);
  const long cnt = (long)ctl->pcount;
  unsigned long long live = 0, mk = ~0ull;
  double mw = 0.0;
  // 4 independent loads in flight per thread (memory-level parallelism)
  const long gs = (long)gridDim.x * TPB;
  for (long r0 = (long)blockIdx.x * TPB + threadIdx.x; r0 - (long)(threadIdx.x & 31) < cnt; r0 += 4 * gs) {
    double lbv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) lbv[u] = r0 + u * gs < cnt ? p.lb[r0 + u * gs] : CUDART_INF;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = r0 + u * gs < cnt && lbv[u] <= gub;  // (GUB may be +inf)
      unsigned long long k = okey(lbv[u]);
      if (ok) {
        ++live;
        mk = k < mk ? k : mk;
        if (WITH_W) mw = fmax(mw, p.w[r0 + u * gs]);
      }
      hist_add(s_h, (unsigned)(k >> 56), ok);
    }
  }
  __shared__ unsigned long long s_l[TPB / 32], s_k[TPB / 32];
  __shared__ double s_w[TPB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(0xffffffffu, live, o);
    unsigned long long t = __shfl_xor_sync(0xffffffffu, mk, o);
    mk = t < mk ? t : mk;
    mw = fmax(mw, __shfl_xor_sync(0xffffffffu, mw, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_l[threadIdx.x >> 5] = live;
    s_k[threadIdx.x >> 5] = mk;
    s_w[threadIdx.x >> 5] = mw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < TPB / 32; ++w) {
      live += s_l[w];
      mk = s_k[w] < mk ? s_k[w] : mk;
      mw = fmax(mw, s_w[w]);
    }
    if (live) atomicAdd(&ctl->acc_live, live);
    atomicMin(&ctl->acc_min_key, mk);
    atomicMax(&ctl->acc_max_w, (unsigned long long)__double_as_longlong(mw));
  }
  for (int i = threadIdx.x; i < 256; i += TPB)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

// max width of the live records (only needed once the enclosure test passes)
__device__ __noinline__ void maxw_accum_dev(const Pool& p, Ctl* ctl) {
  const double gub = okey_inv(ctl->gub_key);
  const long cnt = (long)ctl->pcount;
  double mw = 0.0;
  const long gs = (long)gridDim.x * TPB;
  for (long r0 = (long)blockIdx.x * TPB + threadIdx.x; r0 - (long)(threadIdx.x & 31) < cnt; r0 += 4 * gs) {
    double lbv[4], wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = r0 + u * gs < cnt;
      lbv[u] = in ? p.lb[r0 + u * gs] : CUDART_INF;
      wv[u] = in ? p.w[r0 + u * gs] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r0 + u * gs < cnt && lbv[u] <= gub) mw = fmax(mw, wv[u]);
  }
  mw = warp_max(mw);
  if ((threadIdx.x & 31) == 0) atomicMax(&ctl->acc_max_w, (unsigned long long)__double_as_longlong(mw));
}

// max width of the live records listed in a hot index (all live records
// are there when tau = ~0)
__device__ __noinline__ void maxw_hot_dev(const Pool& p, const uint32_t* __restrict__ hot, long nh, Ctl* ctl) {
  const double gub = okey_inv(ctl->gub_key);
  double mw = 0.0;
  for (long k = (long)blockIdx.x * TPB + threadIdx.x; k < nh; k += (long)gridDim.x * TPB) {
    const uint32_t r = hot[k];
    if (p.lb[r] <= gub) mw = fmax(mw, p.w[r]);
  }
  mw = warp_max(mw);
  if ((threadIdx.x & 31) == 0) atomicMax(&ctl->acc_max_w, (unsigned long long)__double_as_longlong(mw));
}

// control decisions of an iteration, by one block after the statistics pass
// `wstage`: 0 = the max width was accumulated with the statistics (k_stats);
// 1 = first call of the cooperative kernel, widths not read yet: if the
// enclosure test GUB - GLB <= eps_f passes, ask for a width pass (returns
// with ctl->need_w = 1); 2 = second call, after the width pass.
__device__ void stats_control_dev(Ctl* ctl, unsigned int* hist, int wstage = 0) {
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    const double gub = okey_inv(ctl->gub_key);
    s_go = 0;
    if (wstage != 2) {
      ctl->blocks_done = 0;
      ctl->live = ctl->acc_live;
      ctl->min_lb_key = ctl->acc_min_key;
      ctl->acc_live = 0;
      ctl->acc_min_key = ~0ull;
    }
    if (wstage != 1) {
      ctl->max_w_bits = ctl->acc_max_w;
      ctl->acc_max_w = 0;
    }
    ctl->need_w = 0;
    const unsigned long long L = ctl->live;
    const double glb = okey_inv(ctl->min_lb_key);
    const bool encl = L > 0 && __dsub_ru(gub, glb) <= ctl->eps_f;
    if (L == 0) {
      ctl->done = 3;
    } else if (encl && wstage == 1) {
      ctl->need_w = 1;  // the width test decides: run the width pass first
      s_go = -1;
    } else if (encl && __longlong_as_double((long long)ctl->max_w_bits) <= ctl->eps_x) {
      ctl->done = 1;
    } else if (ctl->iter >= ctl->max_iter) {
      ctl->done = 2;
    } else {
      const unsigned long long B = L < ctl->bmax ? L : ctl->bmax;
      ctl->B = B;
      ctl->known = 0;
      ctl->prefix = 0;
      ctl->need = B;
      ctl->resolved = 1;
      if (ctl->free_top < B) {  // archive full
        ctl->err = -2;
        ctl->done = 4;
      } else if (L > ctl->bmax) {
        ctl->resolved = 0;
        s_go = 1;
      }
    }
  }
  __syncthreads();
  if (s_go == 1) {
    block_pick_digit(ctl, hist);
  } else if (s_go == 0) {
    for (int i = threadIdx.x; i < 256; i += TPB) hist[i] = 0;
    __syncthreads();
  }
}

#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_stats(Pool p, Ctl* ctl, unsigned int* hist) {
  if (ctl->done) return;
  stats_accum_dev(p, ctl, hist);
  if (!last_block(ctl)) return;
  stats_control_dev(ctl, hist);
}
#endif  // IBNB_OBJ_TU

// radix pass: histogram of the next digit among live records matching the
// known prefix; the last block picks the digit
__device__ void radix_accum_dev(const Pool& p, const Ctl* __restrict__ ctl, unsigned int* hist) {
  __shared__ unsigned int s_h[256];
  for (int i = threadIdx.x; i < 256; i += TPB) s_h[i] = 0;
  __syncthreads();
  const double gub = okey_inv(ctl->gub_key);
  const int known = ctl->known;
  const unsigned long long prefix = ctl->prefix;
  const int shift = 64 - known - 8;
  const long cnt = (long)ctl->pcount;
  const long gs = (long)gridDim.x * TPB;
  for (long r0 = (long)blockIdx.x * TPB + threadIdx.x; r0 - (long)(threadIdx.x & 31) < cnt; r0 += 4 * gs) {
    double lbv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) lbv[u] = r0 + u * gs < cnt ? p.lb[r0 + u * gs] : CUDART_INF;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      unsigned long long k = okey(lbv[u]);
      const bool ok = r0 + u * gs < cnt && lbv[u] <= gub && (k >> (64 - known)) == prefix;
      hist_add(s_h, (unsigned)((k >> shift) & 255u), ok);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += TPB)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_radix(Pool p, Ctl* __restrict__ ctl, unsigned int* hist) {
  if (ctl->done || ctl->resolved) return;
  radix_accum_dev(p, ctl, hist);
  if (!last_block(ctl)) return;
  if (threadIdx.x == 0) {
    ctl->blocks_done = 0;
    ctl->sum_radix += ctl->pcount;
  }
  block_pick_digit(ctl, hist);
}
#endif  // IBNB_OBJ_TU

// Selection (line 130): the B live records with the smallest (lb, position)
// are copied, in list order, to the batch arrays and marked dead in L
// (lb = +inf).  Kept records stay in place (lazy deletion).
__device__ void select_dev(const Pool& p, Ctl* __restrict__ ctl, int32_t* sel_slot, uint32_t* sel_code, uint64_t* desc,
                           uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile;
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  __syncthreads();
  const long cnt = (long)ctl->pcount;
  const long ntiles = (cnt + TILE - 1) / TILE;
  if ((long)tile >= ntiles) break;
  const double gub = okey_inv(ctl->gub_key);
  const int known = ctl->known;
  const unsigned long long prefix = ctl->prefix;
  const unsigned long long r_need = ctl->need;
  const bool all = known == 0;
  const long r0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  uint8_t cls[IPT];  // 0 lt (selected), 1 eq (tie class), 2 not selected
  uint32_t c2[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    long r = r0 + q;
    cls[q] = 2;
    if (r < cnt) {
      double lb = p.lb[r];
      if (lb <= gub) {
        if (all) {
          cls[q] = 0;
        } else {
          unsigned long long top = okey(lb) >> (64 - known);
          cls[q] = top < prefix ? 0 : (top == prefix ? 1 : 2);
        }
        if (cls[q] < 2) c2[cls[q]]++;
      }
    }
  }
  uint32_t ex[2], tot[2];
  block_exclusive_scan<2, TPB>(c2, ex, tot);
  uint64_t pfx[2];
  dl_lookback<2>(desc, tile, tot, pfx);
  uint64_t lt = pfx[0] + ex[0], eq = pfx[1] + ex[1];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    long r = r0 + q;
    int k = cls[q];
    if (k == 2) continue;
    bool sel;
    uint64_t pos = 0;
    if (k == 0) {
      sel = true;
      pos = lt + (eq < r_need ? eq : r_need);
      ++lt;
    } else {
      sel = eq < r_need;
      pos = lt + eq;
      ++eq;
    }
    if (sel) {
      sel_slot[pos] = p.slot[r];
      sel_code[pos] = p.code[r];
      p.lb[r] = CUDART_INF;  // removed from L
    }
  }
  }
}
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_select(Pool p, Ctl* __restrict__ ctl, int32_t* sel_slot, uint32_t* sel_code,
                                                uint64_t* desc, uint32_t* tile_ctr) {
  if (ctl->done) return;
  select_dev(p, ctl, sel_slot, sel_code, desc, tile_ctr);
}
#endif  // IBNB_OBJ_TU

// iteration end: the survivors become part of L
__device__ void iter_end_dev(Ctl* ctl, long kids) {
  if (ctl->done) return;
  ctl->sum_cand += ctl->ncand;
  ctl->sum_pool += ctl->pcount;
  ctl->sum_B += ctl->B;
  ctl->free_top -= ctl->B;  // archive slots taken by k_prep
  ctl->pcount += ctl->nsurv;
  ctl->nhot += ctl->nsurv_hot;
  ctl->iter += 1;
  ctl->evals += ctl->B * (unsigned long long)kids;
}
#ifndef IBNB_OBJ_TU
__global__ void k_iter_end(Ctl* ctl, long kids) { iter_end_dev(ctl, kids); }
#endif  // IBNB_OBJ_TU
#ifndef IBNB_OBJ_TU
__global__ void k_apply_pending(Ctl* ctl, long kids) {
  if (ctl->pending_end) {
    ctl->pending_end = 0;
    iter_end_dev(ctl, kids);
  }
}
#endif  // IBNB_OBJ_TU

// ===================================================== list L (cooperative)
// k_list runs the list phase of an iteration as one cooperative kernel; its
// steps are separated by grid-wide barriers (every block resident) and after
// a barrier the control block is re-read from L2.  k_fused calls the same
// device functions.
__device__ __forceinline__ int vload(const int* p) { return *(const volatile int*)p; }

// ------------------------------------------------------------ hot index of L
// The selection (line 130) only ever needs the smallest lower bounds: a
// position-ordered index of the live records with key < tau ("hot") is kept
// next to L, and statistics / radix select / selection run on it; it is
// rebuilt from a full pass over L (a "refill") only when it holds fewer than
// bmax live records.  Positions in L are insertion order, so selecting the B
// smallest (key, position) entries of the hot index is exactly the oracle's
// rule on the whole list (every cold key >= tau > every hot key).

// block-wide pick over a 256-bin histogram: smallest digit whose cumulative
// count reaches need; every thread gets (dig, before, cnt)
struct Pick {
  int dig;
  unsigned long long before, cnt, total;
};
__device__ __noinline__ Pick block_pick(const unsigned int* hist, unsigned long long need) {
  __shared__ unsigned long long s_inc[256];
  __shared__ Pick s_p;
  const int t = threadIdx.x;
  unsigned long long h = __ldcg(&hist[t]);
  s_inc[t] = h;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    unsigned long long v = t >= o ? s_inc[t - o] : 0ull;
    __syncthreads();
    s_inc[t] += v;
    __syncthreads();
  }
  if (t == 0) s_p.dig = 255;
  __syncthreads();
  unsigned long long before = t ? s_inc[t - 1] : 0ull;
  if (before < need && s_inc[t] >= need) s_p.dig = t;
  __syncthreads();
  if (t == 0) {
    int d = s_p.dig;
    s_p.before = d ? s_inc[d - 1] : 0ull;
    s_p.cnt = s_inc[d] - s_p.before;
    s_p.total = s_inc[255];
  }
  __syncthreads();
  Pick r = s_p;
  __syncthreads();
  return r;
}

// accumulate (live count, min key) of a set of records of L and the
// histogram of digit (64 - known - 8 .. 64 - known) of the live keys whose
// top `known` bits equal prefix.  idx == nullptr: records [0, n) of L.
__device__ __noinline__ void scan_keys_dev(const Pool& p, const uint32_t* __restrict__ idx, long n, double gub, int known,
                              unsigned long long prefix, unsigned int* hist, unsigned long long* acc_live,
                              unsigned long long* acc_min) {
  __shared__ unsigned int s_h[256];
  for (int i = threadIdx.x; i < 256; i += TPB) s_h[i] = 0;
  __syncthreads();
  const int shift = 64 - known - 8;
  unsigned long long live = 0, mk = ~0ull;
  const long gs = (long)gridDim.x * TPB;
  for (long r0 = (long)blockIdx.x * TPB + threadIdx.x; r0 - (long)(threadIdx.x & 31) < n; r0 += 4 * gs) {
    double lbv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long i = r0 + u * gs;
      lbv[u] = i < n ? p.lb[idx ? (long)idx[i] : i] : CUDART_INF;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long k = okey(lbv[u]);
      const bool ok = r0 + u * gs < n && lbv[u] <= gub && (known == 0 || (k >> (64 - known)) == prefix);
      if (ok) {
        ++live;
        mk = k < mk ? k : mk;
      }
      hist_add(s_h, (unsigned)((k >> shift) & 255u), ok);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += TPB)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
  if (acc_live) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      live += __shfl_xor_sync(0xffffffffu, live, o);
      unsigned long long t = __shfl_xor_sync(0xffffffffu, mk, o);
      mk = t < mk ? t : mk;
    }
    if ((threadIdx.x & 31) == 0) {
      if (live) atomicAdd(acc_live, live);
      atomicMin(acc_min, mk);
    }
  }
}

// refill: positions of the live records of L with key < tau, in order
__device__ __noinline__ void hot_collect_dev(const Pool& p, long n, double gub, unsigned long long tau, uint32_t* out,
                                unsigned long long* out_count, uint64_t* desc, uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    __syncthreads();
    const long ntiles = (n + TILE - 1) / TILE;
    if ((long)tile >= ntiles) break;
    const long r0 = (long)tile * TILE + (long)threadIdx.x * IPT;
    uint32_t f = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      if (r0 + q < n) {
        const double lb = p.lb[r0 + q];
        if (lb <= gub && okey(lb) < tau) f |= 1u << q;
      }
    }
    uint32_t c1[1] = {(uint32_t)__popc(f)}, ex[1], tot[1];
    block_exclusive_scan<1, TPB>(c1, ex, tot);
    uint64_t pfx[1];
    dl_lookback<1>(desc, tile, tot, pfx);
    uint64_t pos = pfx[0] + ex[0];
#pragma unroll
    for (int q = 0; q < IPT; ++q)
      if (f & (1u << q)) out[pos++] = (uint32_t)(r0 + q);
    if ((long)tile == ntiles - 1 && threadIdx.x == 0) *out_count = pfx[0] + tot[0];
  }
}

// selection (line 130) over the hot index: the B entries with the smallest
// (key, position) go to the batch and are removed from L (lb = +inf); the
// other live hot entries are kept, in order, in `hout`.  counters: 0 lt
// (selected), 1 eq (tie class), 2 gt (kept).  known == 0 selects all.
__device__ __noinline__ void hot_select_dev(const Pool& p, const uint32_t* __restrict__ hin, long n, uint32_t* hout, double gub,
                               int known, unsigned long long prefix, unsigned long long r_need, int32_t* sel_slot,
                               uint32_t* sel_code, unsigned long long* keep_count, uint64_t* desc,
                               uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    __syncthreads();
    const long ntiles = (n + TILE - 1) / TILE;
    if ((long)tile >= ntiles) break;
    const long i0 = (long)tile * TILE + (long)threadIdx.x * IPT;
    uint8_t cls[IPT];  // 0 lt, 1 eq, 2 gt, 3 dead
    uint32_t rr[IPT];
    uint32_t c3[3] = {0, 0, 0};
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      cls[q] = 3;
      rr[q] = 0;
      if (i0 + q < n) {
        rr[q] = hin[i0 + q];
        const double lb = p.lb[rr[q]];
        if (lb <= gub) {
          if (known == 0) {
            cls[q] = 0;
          } else {
            const unsigned long long top = okey(lb) >> (64 - known);
            cls[q] = top < prefix ? 0 : (top == prefix ? 1 : 2);
          }
          c3[cls[q]]++;
        }
      }
    }
    uint32_t ex[3], tot[3];
    block_exclusive_scan<3, TPB>(c3, ex, tot);
    uint64_t pfx[3];
    dl_lookback<3>(desc, tile, tot, pfx);
    uint64_t lt = pfx[0] + ex[0], eq = pfx[1] + ex[1], gt = pfx[2] + ex[2];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int k = cls[q];
      if (k == 3) continue;
      bool sel;
      uint64_t pos;
      if (k == 0) {
        sel = true;
        pos = lt + (eq < r_need ? eq : r_need);
        ++lt;
      } else if (k == 1) {
        sel = eq < r_need;
        pos = sel ? lt + eq : gt + (eq - r_need);
        ++eq;
      } else {
        sel = false;
        pos = gt + (eq > r_need ? eq - r_need : 0);
        ++gt;
      }
      if (sel) {
        sel_slot[pos] = p.slot[rr[q]];
        sel_code[pos] = p.code[rr[q]];
        p.lb[rr[q]] = CUDART_INF;  // removed from L
      } else {
        hout[pos] = rr[q];
      }
    }
    if ((long)tile == ntiles - 1 && threadIdx.x == 0) {
      const uint64_t e = pfx[1] + tot[1];
      *keep_count = pfx[2] + tot[2] + (e > r_need ? e - r_need : 0);
    }
  }
}

// One cooperative kernel per iteration for the list L (a1, a7): iteration
// end of the previous one, hot statistics (refill when short), stop test,
// batch size, radix select and selection.  Every block takes the same
// decisions from the same global values after each grid barrier; thread 0
// of block 0 records them in ctl.  hists: 16 x 256 zeroed counters (zeroed
// again by k_child_eval); the acc_* fields likewise.
// Single-block list phase (k_fused, when ctl->list_fast): the same decisions
// as list_dev when every live record is in a hot index of at most
// min(bmax, LSMAX * TPB) entries -- then live <= bmax, the selection takes every live
// entry in list order and no radix pass is needed.  Block 0 only.
__device__ void list_small_dev(const Pool& p, Ctl* ctl, uint32_t* hot0, uint32_t* hot1, int32_t* sel_slot,
                               uint32_t* sel_code, long kids) {
  __shared__ unsigned long long s_min;
  __shared__ double s_w;
  __shared__ uint32_t s_scan[TPB / 32];
  if (ctl->done) return;
  if (threadIdx.x == 0) {
    if (ctl->pending_end) {
      ctl->pending_end = 0;
      iter_end_dev(ctl, kids);
    }
    s_min = ~0ull;
    s_w = 0.0;
  }
  __syncthreads();
  const double gub = okey_inv(ctl->gub_key);
  const int hsel = ctl->hsel;
  const long nh = (long)ctl->nhot;
  const uint32_t* hin = hsel ? hot1 : hot0;
  const int t = threadIdx.x;
  // thread t owns the hot entries t * ls .. t * ls + ls - 1 (list order),
  // ls <= LSMAX (set_list_fast)
  const int ls = (int)((nh + TPB - 1) / TPB);
  uint32_t r[LSMAX];
  double lbv[LSMAX], wv[LSMAX];
  bool live[LSMAX];
  uint32_t cnt = 0;
  unsigned long long mk = ~0ull;
#pragma unroll
  for (int j = 0; j < LSMAX; ++j) {
    const long e = (long)t * ls + j;
    r[j] = 0;
    lbv[j] = CUDART_INF;
    wv[j] = 0.0;
    live[j] = false;
    if (j < ls && e < nh) {
      r[j] = hin[e];
      lbv[j] = p.lb[r[j]];
      wv[j] = p.w[r[j]];
      live[j] = lbv[j] <= gub;
    }
    if (live[j]) {
      ++cnt;
      const unsigned long long key = okey(lbv[j]);
      mk = key < mk ? key : mk;
    }
  }
  // live count (exclusive scan = selection position) and min key
  const int lane = t & 31, wid = t >> 5;
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long q = __shfl_xor_sync(0xffffffffu, mk, o);
    mk = q < mk ? q : mk;
  }
  if (lane == 31) s_scan[wid] = inc;
  if (lane == 0 && mk != ~0ull) atomicMin(&s_min, mk);
  __syncthreads();
  uint32_t before = 0, total = 0;
  for (int w2 = 0; w2 < TPB / 32; ++w2) {
    if (w2 < wid) before += s_scan[w2];
    total += s_scan[w2];
  }
  const uint32_t pos0 = before + inc - cnt;
  const unsigned long long nlive = total, minkey = s_min;
  unsigned long long bytes = 12ull * nh;
  int done = 0;
  if (nlive == 0) {
    done = 3;
  } else if (__dsub_ru(gub, okey_inv(minkey)) <= ctl->eps_f) {
    double mw = 0.0;
#pragma unroll
    for (int j = 0; j < LSMAX; ++j)
      if (live[j]) mw = fmax(mw, wv[j]);
    mw = warp_max(mw);
    if (lane == 0) atomicMax((unsigned long long*)&s_w, (unsigned long long)__double_as_longlong(mw));
    __syncthreads();
    bytes += 20ull * nh;
    if (t == 0) {
      ctl->nwidth += 1;
      const unsigned long long wb = (unsigned long long)__double_as_longlong(s_w);
      if (wb > ctl->acc_max_w) ctl->acc_max_w = wb;
    }
    if (s_w <= ctl->eps_x) done = 1;
  }
  if (!done && ctl->iter >= ctl->max_iter) done = 2;
  const unsigned long long B = nlive;  // nlive <= nh <= bmax
  if (!done && ctl->free_top < B) done = 4;
  if (done) {
    __syncthreads();
    if (t == 0) {
      ctl->live = nlive;
      ctl->min_lb_key = minkey;
      ctl->max_w_bits = ctl->acc_max_w;
      if (done == 4) ctl->err = -2;
      ctl->list_bytes += bytes;
      ctl->done = done;
    }
    return;
  }
  // selection (line 130): every live entry, in list order; L loses them
  {
    uint32_t pos = pos0;
#pragma unroll
    for (int j = 0; j < LSMAX; ++j) {
      if (live[j]) {
        sel_slot[pos] = p.slot[r[j]];
        sel_code[pos] = p.code[r[j]];
        p.lb[r[j]] = CUDART_INF;
        ++pos;
      }
    }
  }
  bytes += 16ull * nh;
  __syncthreads();
  if (t == 0) {
    ctl->nhot_keep = 0;
    ctl->hsel = hsel ^ 1;
    ctl->nhot = 0;
    ctl->B = B;
    ctl->live = nlive;
    ctl->min_lb_key = minkey;
    ctl->known = 0;
    ctl->prefix = 0;
    ctl->need = B;
    ctl->list_bytes += bytes;
  }
}

__device__ __noinline__ void list_dev(const Pool& p, Ctl* ctl, unsigned int* hists, int32_t* sel_slot, uint32_t* sel_code,
                         uint64_t* desc, uint64_t* desc2, uint32_t* tile_ctr, uint32_t* hot0, uint32_t* hot1,
                         long kids) {
  cg::grid_group grid = cg::this_grid();
  if (ctl->done) return;  // uniform: read before any block writes it
  const long gtid = (long)blockIdx.x * TPB + threadIdx.x, gsize = (long)gridDim.x * TPB;
  const bool lead = gtid == 0;
  if (lead && ctl->pending_end) {  // end of the previous iteration (k_emit)
    ctl->pending_end = 0;
    iter_end_dev(ctl, kids);
  }
  grid.sync();
  const double gub = okey_inv(ctl->gub_key);
  const long pc = (long)ctl->pcount;
  const unsigned long long bmax = ctl->bmax;
  int hsel = ctl->hsel;
  long nh = (long)ctl->nhot;
  unsigned long long tau = ctl->tau_key;
  const bool valid = ctl->hot_valid != 0;
  unsigned long long bytes = 0;
  {
    const long tl = (pc + TILE - 1) / TILE + 1;
    for (long i = gtid; i < 3 * tl; i += gsize) {
      desc2[i] = 0;
      if (i < tl) desc[i] = 0;
    }
    if (lead) {
      tile_ctr[0] = 0;
      tile_ctr[1] = 0;
    }
  }
  // statistics of the hot entries + histogram of their top 8 key bits
  unsigned long long live = 0, minkey = ~0ull;
  const unsigned int* hh = hists;
  if (valid) {
    scan_keys_dev(p, hsel ? hot1 : hot0, nh, gub, 0, 0, hists, &ctl->acc_live, &ctl->acc_min_key);
    bytes += 12ull * nh;
  }
  grid.sync();
  if (valid) {
    live = __ldcg(&ctl->acc_live);
    minkey = __ldcg(&ctl->acc_min_key);
  }
  if (!valid || (live < bmax && tau != ~0ull)) {
    // refill: histogram of all live keys of L, threshold tau for ~hot_target entries
    scan_keys_dev(p, nullptr, pc, gub, 0, 0, hists + 256, &ctl->acc_live2, &ctl->acc_min_key2);
    bytes += 8ull * pc;
    grid.sync();
    const unsigned long long total = __ldcg(&ctl->acc_live2), target = ctl->hot_target;
    unsigned long long new_tau = ~0ull;
    if (total > target) {
      Pick a = block_pick(hists + 256, target);
      if (a.before + a.cnt > 2 * target) {  // refine inside the boundary bucket
        scan_keys_dev(p, nullptr, pc, gub, 8, (unsigned long long)a.dig, hists + 512, nullptr, nullptr);
        bytes += 8ull * pc;
        grid.sync();
        Pick b2 = block_pick(hists + 512, target - a.before);
        const unsigned long long t16 = ((unsigned long long)a.dig << 8) | (unsigned long long)b2.dig;
        new_tau = t16 == 0xffffull ? ~0ull : (t16 + 1) << 48;
      } else {
        new_tau = a.dig == 255 ? ~0ull : ((unsigned long long)a.dig + 1) << 56;
      }
    }
    uint32_t* hout = hsel ? hot0 : hot1;
    hot_collect_dev(p, pc, gub, new_tau, hout, &ctl->nhot_keep, desc, tile_ctr);
    bytes += 8ull * pc;
    grid.sync();
    hsel ^= 1;
    nh = (long)__ldcg(&ctl->nhot_keep);
    tau = new_tau;
    if (lead) {
      ctl->hsel = hsel;
      ctl->nhot = (unsigned long long)nh;
      ctl->tau_key = tau;
      ctl->hot_valid = 1;
      ctl->live_total = total;
      ctl->sum_refill += (unsigned long long)pc;
      ctl->nrefill += 1;
      ctl->compact_hint = total < (unsigned long long)pc / 2;
      tile_ctr[1] = 0;
    }
    // statistics of the rebuilt hot index
    scan_keys_dev(p, hsel ? hot1 : hot0, nh, gub, 0, 0, hists + 2560, &ctl->acc_live3, &ctl->acc_min_key3);
    bytes += 12ull * nh;
    grid.sync();
    live = __ldcg(&ctl->acc_live3);
    minkey = __ldcg(&ctl->acc_min_key3);
    hh = hists + 2560;
  }
  // stop test (line 148: every region narrower than eps_x; line 150:
  // GUB - GLB <= eps_f); GLB = smallest hot key (all cold keys are larger)
  int done = 0;
  if (live == 0) {
    done = 3;  // the refill found no live record: L is empty
  } else if (__dsub_ru(gub, okey_inv(minkey)) <= ctl->eps_f) {
    if (tau == ~0ull) {  // every live record is in the hot index
      maxw_hot_dev(p, hsel ? hot1 : hot0, nh, ctl);
      bytes += 20ull * nh;
    } else {
      maxw_accum_dev(p, ctl);  // the width test decides: max width of all of L
      bytes += 16ull * pc;
    }
    if (lead) ctl->nwidth += 1;
    grid.sync();
    if (__longlong_as_double((long long)__ldcg(&ctl->acc_max_w)) <= ctl->eps_x) done = 1;
  }
  if (!done && ctl->iter >= ctl->max_iter) done = 2;
  const unsigned long long B = live < bmax ? live : bmax;
  if (!done && ctl->free_top < B) done = 4;  // archive full
  if (done) {
    if (lead) {
      ctl->live = live;
      ctl->min_lb_key = minkey;
      ctl->max_w_bits = ctl->acc_max_w;
      if (done == 4) ctl->err = -2;
      ctl->list_bytes += bytes;
      ctl->done = done;
    }
    return;
  }
  // radix select of the B-th smallest hot key (line 130, reading R1)
  int known = 0;
  unsigned long long prefix = 0, need = B;
  bool resolved = live <= bmax;
  if (!resolved) {
    Pick a = block_pick(hh, need);
    need -= a.before;
    prefix = (unsigned long long)a.dig;
    known = 8;
    resolved = a.cnt == need;
  }
  for (int pass = 1; pass < 8 && !resolved; ++pass) {
    unsigned int* hp = hists + (2 + pass) * 256;
    scan_keys_dev(p, hsel ? hot1 : hot0, nh, gub, known, prefix, hp, nullptr, nullptr);
    bytes += 12ull * nh;
    grid.sync();
    Pick a = block_pick(hp, need);
    need -= a.before;
    prefix = (prefix << 8) | (unsigned long long)a.dig;
    known += 8;
    resolved = a.cnt == need || known >= 64;
  }
  // selection + compaction of the hot index into the other buffer
  hot_select_dev(p, hsel ? hot1 : hot0, nh, hsel ? hot0 : hot1, gub, resolved && known == 0 ? 0 : known, prefix,
                 known == 0 ? 0ull : need, sel_slot, sel_code, &ctl->nhot_keep, desc2, tile_ctr + 1);
  bytes += 16ull * nh;
  grid.sync();
  if (lead) {
    ctl->hsel = hsel ^ 1;
    ctl->nhot = __ldcg(&ctl->nhot_keep);
    ctl->B = B;
    ctl->live = live;
    ctl->min_lb_key = minkey;
    ctl->known = known;
    ctl->prefix = prefix;
    ctl->need = need;
    ctl->list_bytes += bytes;
  }
}

#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_list(Pool p, Ctl* ctl, unsigned int* hists, int32_t* sel_slot,
                                              uint32_t* sel_code, uint64_t* desc, uint64_t* desc2, uint32_t* tile_ctr,
                                              uint32_t* hot0, uint32_t* hot1, long kids) {
  // potential-candidate count of this iteration's k_child_eval (read by
  // k_insert before this kernel runs again)
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->npot = 0ull;
  if (ctl->list_fast) {  // uniform: set by the previous insertion (emit)
    if (blockIdx.x == 0) list_small_dev(p, ctl, hot0, hot1, sel_slot, sel_code, kids);
    return;
  }
  list_dev(p, ctl, hists, sel_slot, sel_code, desc, desc2, tile_ctr, hot0, hot1, kids);
}
#endif  // IBNB_OBJ_TU

// multi-GPU exchange of the incumbent (2 doubles: GUB, finished flag)
#ifndef IBNB_OBJ_TU
__global__ void k_xchg_put(const Ctl* ctl, double* xchg) {
  xchg[0] = okey_inv(ctl->gub_key);
  xchg[1] = ctl->done ? 0.0 : -1.0;
}
#endif  // IBNB_OBJ_TU
#ifndef IBNB_OBJ_TU
__global__ void k_xchg_take(Ctl* ctl, const double* xchg) {
  unsigned long long k = okey(xchg[0]);
  if (k < ctl->gub_key) ctl->gub_key = k;
  ctl->gdone = xchg[1] == 0.0 ? 1 : 0;
}
#endif  // IBNB_OBJ_TU

// Stable 3-way partition of L with a host-given selection spec (ib_select,
// compaction of L, final output).  Live records (lb <= GUB) whose key's top
// `known` bits are < prefix are selected; those equal to prefix are selected
// while their rank among equals is < r_need; the other live records are
// kept.  known == 0 selects every live record; (known = 64, prefix = 0,
// r_need = 0) keeps every live record.  counters: 0 lt, 1 eq, 2 gt.
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_partition(Pool in, long cnt, const unsigned long long* gub_key,
                                                   int known, unsigned long long prefix,
                                                   unsigned long long r_need, int32_t* sel_slot,
                                                   uint32_t* sel_code, double* sel_lb, Pool keep,
                                                   uint64_t* desc, uint32_t* tile_ctr, uint64_t* keep_count,
                                                   long ntiles) {
  __shared__ uint32_t s_tile;
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  __syncthreads();
  if ((long)tile >= ntiles) break;
  const double gub = okey_inv(*gub_key);
  const long r0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  uint8_t cls[IPT];  // 0 lt, 1 eq, 2 gt, 3 drop
  uint32_t cnt3[3] = {0, 0, 0};
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    long r = r0 + q;
    cls[q] = 3;
    if (r < cnt) {
      double lb = in.lb[r];
      if (lb <= gub) {
        if (known == 0) {
          cls[q] = 0;
        } else {
          unsigned long long top = okey(lb) >> (64 - known);
          cls[q] = top < prefix ? 0 : (top == prefix ? 1 : 2);
        }
        cnt3[cls[q]]++;
      }
    }
  }
  uint32_t ex[3], tot[3];
  block_exclusive_scan<3, TPB>(cnt3, ex, tot);
  uint64_t pfx[3];
  dl_lookback<3>(desc, tile, tot, pfx);
  uint64_t lt = pfx[0] + ex[0], eq = pfx[1] + ex[1], gt = pfx[2] + ex[2];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    long r = r0 + q;
    int k = cls[q];
    if (k == 3) continue;
    bool sel;
    uint64_t pos;
    if (k == 0) {
      sel = true;
      pos = lt + (eq < r_need ? eq : r_need);
      ++lt;
    } else if (k == 1) {
      sel = eq < r_need;
      pos = sel ? lt + eq : gt + (eq - r_need);
      ++eq;
    } else {
      sel = false;
      pos = gt + (eq > r_need ? eq - r_need : 0);
      ++gt;
    }
    if (sel) {
      if (sel_slot) sel_slot[pos] = in.slot[r];
      if (sel_code) sel_code[pos] = in.code[r];
      if (sel_lb) sel_lb[pos] = in.lb[r];
    } else {
      keep.lb[pos] = in.lb[r];
      keep.w[pos] = in.w[r];
      keep.slot[pos] = in.slot[r];
      keep.code[pos] = in.code[r];
    }
  }
  if (tile == (uint32_t)(ntiles - 1) && threadIdx.x == 0 && keep_count) {
    uint64_t e = pfx[1] + tot[1];
    *keep_count = pfx[2] + tot[2] + (e > r_need ? e - r_need : 0);
  }
  }
}
#endif  // IBNB_OBJ_TU

// ---- archive slot garbage collection (mark from L, collect the unmarked)
// slots still needed: those of the live records (lb <= GUB); selected and
// ruled-out records (lazy deletion) are never read again
#ifndef IBNB_OBJ_TU
__global__ void k_gc_mark(Pool p, const Ctl* ctl, uint8_t* mark) {
  const long cnt = (long)ctl->pcount;
  const double gub = okey_inv(ctl->gub_key);
  for (long r = (long)blockIdx.x * blockDim.x + threadIdx.x; r < cnt; r += (long)gridDim.x * blockDim.x)
    if (p.lb[r] <= gub) mark[p.slot[r]] = 1;
}
#endif  // IBNB_OBJ_TU
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_gc_collect(const uint8_t* mark, long cap, int32_t* free_list,
                                                    uint64_t* desc, uint32_t* tile_ctr, Ctl* ctl, long ntiles) {
  __shared__ uint32_t s_tile;
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  __syncthreads();
  if ((long)tile >= ntiles) break;
  const long s0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (s0 + q < cap && !mark[s0 + q]) f |= 1u << q;
  uint32_t cnt[1] = {(uint32_t)__popc(f)}, ex[1], tot[1];
  block_exclusive_scan<1, TPB>(cnt, ex, tot);
  uint64_t pfx[1];
  dl_lookback<1>(desc, tile, tot, pfx);
  uint64_t pos = pfx[0] + ex[0];
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (f & (1u << q)) free_list[pos++] = (int32_t)(s0 + q);
  if (tile == (uint32_t)(ntiles - 1) && threadIdx.x == 0) ctl->free_top = pfx[0] + tot[0];
  }
}
#endif  // IBNB_OBJ_TU

// generic stable compaction of indices with key <= threshold (ib_compact_le)
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_compact_le(const double* keys, long cnt, double thr, int64_t* out_idx,
                                                    uint64_t* desc, uint32_t* tile_ctr, uint64_t* out_count,
                                                    long ntiles) {
  __shared__ uint32_t s_tile;
  for (;;) {
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  __syncthreads();
  if ((long)tile >= ntiles) break;
  const long s0 = (long)tile * TILE + (long)threadIdx.x * IPT;
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (s0 + q < cnt && keys[s0 + q] <= thr) f |= 1u << q;
  uint32_t c1[1] = {(uint32_t)__popc(f)}, ex[1], tot[1];
  block_exclusive_scan<1, TPB>(c1, ex, tot);
  uint64_t pfx[1];
  dl_lookback<1>(desc, tile, tot, pfx);
  uint64_t pos = pfx[0] + ex[0];
#pragma unroll
  for (int q = 0; q < IPT; ++q)
    if (f & (1u << q)) out_idx[pos++] = s0 + q;
  if (tile == (uint32_t)(ntiles - 1) && threadIdx.x == 0) *out_count = pfx[0] + tot[0];
  }
}
#endif  // IBNB_OBJ_TU

// materialise records (slot, code) of L into explicit boxes
#ifndef IBNB_OBJ_TU
__global__ void k_extract(Problem P, Pool p, long cnt, const double* A_lo, const double* A_hi,
                          const int32_t* sc, double* out_lo, double* out_hi, double* out_lb) {
  for (long r = blockIdx.x; r < cnt; r += gridDim.x) {
    int s = p.slot[r];
    uint32_t code = p.code[r];
    int psc = sc[s];
    for (int i = threadIdx.x; i < P.n; i += blockDim.x) {
      double a = A_lo[(size_t)s * P.ld + i], b = A_hi[(size_t)s * P.ld + i];
      if (code != CODE_WHOLE) {
        int jj = (i - psc + P.n) % P.n;
        if (jj < P.d) {
          int q = digit(code, jj, P.m);
          double a2 = part_point(a, b, P.m, q), b2 = part_point(a, b, P.m, q + 1);
          a = a2;
          b = b2;
        }
      }
      out_lo[(size_t)r * P.n + i] = a;
      out_hi[(size_t)r * P.n + i] = b;
    }
    if (threadIdx.x == 0 && out_lb) out_lb[r] = p.lb[r];
  }
}
#endif  // IBNB_OBJ_TU

// ========================================================= explicit batches
// f over explicit boxes: one warp per box, lanes stride over variables,
// warp-shuffle interval reduction (the "warp-cooperative sum").
template <class F>
__global__ void __launch_bounds__(TPB) k_eval_boxes(int n, long nbox, const double* __restrict__ lo,
                                                    const double* __restrict__ hi, long ld, double* out) {
  const long wbox = ((long)blockIdx.x * TPB + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wbox >= nbox) return;
  const double* bl = lo + wbox * ld;
  const double* bh = hi + wbox * ld;
  Iv acc[2];
  if constexpr (F::CHAIN) {
    acc[0] = iv(0.0);
    for (int i = lane; i < n; i += 32) {
      LevyVals v = ObjLevy::vals(Iv{bl[i], bh[i]});
      if (i == 0) acc[0] = acc[0] + v.s0;
      if (i <= n - 2) acc[0] = acc[0] + mulpos(v.u, ObjLevy::vals(Iv{bl[i + 1], bh[i + 1]}).v);
      if (i == n - 1) acc[0] = acc[0] + v.u;
    }
    warp_reduce_acc<ObjRastrigin>(acc);
    if (lane == 0) {
      Iv r = ObjLevy::outer(acc[0], n);
      out[2 * wbox] = r.lo;
      out[2 * wbox + 1] = r.hi;
    }
  } else {
#pragma unroll
    for (int k = 0; k < F::K; ++k) acc[k] = acc_ident<F>(k);
    for (int i = lane; i < n; i += 32) {
      Iv t[2];
      F::terms(Iv{bl[i], bh[i]}, i, n, t);
#pragma unroll
      for (int k = 0; k < F::K; ++k) acc[k] = acc_comb<F>(k, acc[k], t[k]);
    }
    warp_reduce_acc<F>(acc);
    if (lane == 0) {
      Iv r = F::outer(acc, n);
      out[2 * wbox] = r.lo;
      out[2 * wbox + 1] = r.hi;
    }
  }
}

// partial derivative enclosures: one warp per request (box index, variable)
template <class F>
__global__ void __launch_bounds__(TPB) k_eval_grad(int n, long nreq, const double* __restrict__ lo,
                                                   const double* __restrict__ hi, long ld,
                                                   const int64_t* __restrict__ req_box,
                                                   const int32_t* __restrict__ req_dim, double* out) {
  const long w = ((long)blockIdx.x * TPB + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nreq) return;
  const long bx = req_box[w];
  const int i = req_dim[w];
  const double* bl = lo + bx * ld;
  const double* bh = hi + bx * ld;
  Iv D;
  if constexpr (F::CHAIN) {
    LevyVals me = ObjLevy::vals(Iv{bl[i], bh[i]});
    Iv up = i > 0 ? ObjLevy::vals(Iv{bl[i - 1], bh[i - 1]}).u : iv(0.0);
    Iv vn = i < n - 1 ? ObjLevy::vals(Iv{bl[i + 1], bh[i + 1]}).v : iv(0.0);
    D = ObjLevy::deriv(me, up, vn, i, n);
  } else if constexpr (F::SEP) {
    D = F::dsep(Iv{bl[i], bh[i]}, i, n);
  } else {
    Iv acc[2], excl[2];
#pragma unroll
    for (int k = 0; k < F::K; ++k) acc[k] = excl[k] = acc_ident<F>(k);
    for (int j = lane; j < n; j += 32) {
      Iv t[2];
      F::terms(Iv{bl[j], bh[j]}, j, n, t);
#pragma unroll
      for (int k = 0; k < F::K; ++k) {
        acc[k] = acc_comb<F>(k, acc[k], t[k]);
        if (j != i) excl[k] = acc_comb<F>(k, excl[k], t[k]);
      }
    }
    warp_reduce_acc<F>(acc);
    warp_reduce_acc<F>(excl);
    Iv g[2];
    Iv X{bl[i], bh[i]};
    F::ding(X, i, n, g);
    typename F::Ctx cx = F::ctx(acc, n);
    D = F::dfin(cx, g, X, i, n, excl);
  }
  if (lane == 0) {
    out[2 * w] = D.lo;
    out[2 * w + 1] = D.hi;
  }
}

// ===================================================== fused persistent kernel
// Small batches (large n, few live regions): one cooperative launch runs up
// to `iters` whole iterations, the phases of each separated by grid
// barriers instead of kernel boundaries.  The phases are the same device
// functions as the multi-kernel path, in the same order, so both paths take
// identical decisions and produce identical results.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class F, int GT>
__global__ void __launch_bounds__(TPB, 1) k_fused(Problem P, IterBufs w, int iters, long nz) {
  cg::grid_group grid = cg::this_grid();
  const long kids = P.kids;
  // optional phase timer (IBNB_TRACE): block 0 accumulates ns per phase
  unsigned long long* ts = (w.tstamp && blockIdx.x == 0 && threadIdx.x == 0) ? w.tstamp : nullptr;
  unsigned long long* tw = (w.tstamp && threadIdx.x == 0) ? w.tstamp : nullptr;
  unsigned long long t0 = tw ? gtimer() : 0ull, tb = t0;
  // work(ph): this block's own work time in the phase (max over blocks is
  // accumulated per iteration); mark(ph): phase time seen by block 0
  const bool tracing = w.tstamp != nullptr;  // uniform over the block
  auto work = [&](int ph) {
    if (tracing) {
      __syncthreads();
      if (tw) atomicMax(&tw[16 + ph], gtimer() - tb);
    }
  };
  auto mark = [&](int ph) {
    if (tw) {
      unsigned long long t1 = gtimer();
      if (ts) {
        ts[ph] += t1 - t0;
        for (int k = 0; k < 6; ++k) {  // fold the per-iteration maxima
          ts[8 + k] += tw[16 + k];
          tw[16 + k] = 0;
        }
      }
      t0 = t1;
    }
  };
  bool need_list = true;  // the first iteration of a launch starts with its list phase
  for (int it = 0; it < iters; ++it) {
    if (need_list) {
      if (w.ctl->list_fast) {  // uniform: set before the last barrier
        if (blockIdx.x == 0) list_small_dev(w.pool, w.ctl, w.hot0, w.hot1, w.sel_slot, w.sel_code, kids);
      } else {
        list_dev(w.pool, w.ctl, w.hist, w.sel_slot, w.sel_code, w.desc, w.desc2, w.tile_ctr, w.hot0, w.hot1, kids);
      }
      work(0);
      grid.sync();
      if (tw) tb = gtimer();
      mark(0);
    }
    if (w.ctl->done) break;  // uniform: written before the barrier
    // every block read the last count before the previous barrier
    if (blockIdx.x == 0 && threadIdx.x == 0) w.ctl->npot = 0ull;
    const int nitems = (int)w.ctl->B * P.pslices;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int b = item / P.pslices;
      prep_item<F, TPB>(P, w.ctl, w.sel_slot, w.sel_code, w.new_slot, w.free_list, w.src_lo, w.src_hi, w.src_sc,
                        w.dst_lo, w.dst_hi, w.dst_sc, w.tab, w.tab_stride, w.ppart, w.pticket, b,
                        item - b * P.pslices);
    }
    work(1);
    grid.sync();
    if (tw) tb = gtimer();
    mark(1);
    child_eval_dev<F, GT>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.desc, w.desc2, nz, w.tile_ctr, w.hist, w.pot,
                          w.ppart);
    work(2);
    grid.sync();
    if (tw) tb = gtimer();
    mark(2);
    const unsigned long long npot = w.ctl->npot;  // uniform: complete before the barrier
    if (npot <= (unsigned long long)PCAP) {
      // few potential candidates: insertion and the next list phase on block 0
      need_list = true;
      if (blockIdx.x == 0) {
        const bool sel = emit_small_dev<F>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.pot, (int)npot,
                                           w.hot0, w.hot1, it + 1 < iters, kids, w.sel_slot, w.sel_code);
        if (it + 1 < iters) {
          const bool fast = sel || (w.ctl->list_fast != 0 && !w.ctl->done);
          if (fast && !sel) list_small_dev(w.pool, w.ctl, w.hot0, w.hot1, w.sel_slot, w.sel_code, kids);
          if (threadIdx.x == 0) w.ctl->list_pre = fast ? 1 : 0;
        }
      }
      work(3);
      grid.sync();
      if (tw) tb = gtimer();
      if (it + 1 < iters) need_list = w.ctl->list_pre == 0;
      mark(5);
      if (ts) ts[6] += 1;
      continue;
    }
    cand_emit_dev<F>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.desc2, w.hot0, w.hot1);
    work(3);
    // the last block to finish the insertion runs the next iteration's list
    // phase when it fits one block (no barrier between insertion and list)
    need_list = true;
    if (it + 1 < iters) {
      __shared__ int s_lastblk;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_lastblk = atomicAdd(&w.ctl->fused_ticket, 1u) == gridDim.x - 1;
      __syncthreads();
      if (s_lastblk) {
        __threadfence();
        const bool fast = w.ctl->list_fast != 0 && !w.ctl->done;
        if (fast) list_small_dev(w.pool, w.ctl, w.hot0, w.hot1, w.sel_slot, w.sel_code, kids);
        if (threadIdx.x == 0) {
          w.ctl->fused_ticket = 0u;
          w.ctl->list_pre = fast ? 1 : 0;
        }
      }
      work(5);
      grid.sync();
      if (tw) tb = gtimer();
      need_list = w.ctl->list_pre == 0;
    } else {
      grid.sync();
    }
    mark(5);
    if (ts) ts[6] += 1;
  }
}

IB_NS_END  // namespace ib
#include "chain.cuh"
#include "chainc.cuh"
IB_NS_BEGIN

// ================================================================ launchers
static inline unsigned grid_for(long items, int per_block, unsigned cap = 148u * 32u) {
  long g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (unsigned)(g < (long)cap ? g : cap);
}
static inline long tiles_for(long items) { return std::max(1L, (items + TILE - 1) / TILE); }
// persistent grid for the decoupled-look-back scans: blocks loop over tile tickets
static inline unsigned scan_grid(long items) { return (unsigned)std::min(tiles_for(items), 148L * 6); }

#define LAUNCH_OK return (int)cudaGetLastError()

// One iteration of the hot path, every kernel reading its sizes from ctl.
// pool_bound / batch_bound: host upper bounds of |L| and B * m^d for grids.
template <class F>
static void launch_prep_t(const Problem& P, const IterBufs& w, long nb, const int32_t* free_list, cudaStream_t st) {
  const unsigned g = (unsigned)(nb * P.pslices);
  if (P.n <= 64)
    k_prep<F, 32><<<g, 32, 0, st>>>(P, w.ctl, w.sel_slot, w.sel_code, w.new_slot, free_list, w.src_lo, w.src_hi,
                                     w.src_sc, w.dst_lo, w.dst_hi, w.dst_sc, w.tab, w.tab_stride, w.ppart, w.pticket);
  else
    k_prep<F, TPB><<<g, TPB, 0, st>>>(P, w.ctl, w.sel_slot, w.sel_code, w.new_slot, free_list, w.src_lo, w.src_hi,
                                       w.src_sc, w.dst_lo, w.dst_hi, w.dst_sc, w.tab, w.tab_stride, w.ppart,
                                       w.pticket);
}

template <class F>
static void launch_eval_t(const Problem& P, const IterBufs& w, long nkids, cudaStream_t st, bool zero = false) {
  unsigned g = grid_for(nkids / P.G, TPB, 148u * 16u);
  uint64_t* za = zero ? w.desc : nullptr;
  uint64_t* zb = zero ? w.desc2 : nullptr;
  long nz = tiles_for(nkids) + 1;
  if constexpr (!F::CHAIN) {  // the Levy chain never takes the G = 8 path
    if (P.m == 2 && P.G == 8) {
      k_child_eval<F, 8><<<g, TPB, 0, st>>>(P, w.ctl, w.tab, w.tab_stride, w.clb, za, zb, nz, w.tile_ctr, w.hist,
                                             w.ppart, zero ? w.pbits : nullptr);
      return;
    }
  }
  k_child_eval<F, 0><<<g, TPB, 0, st>>>(P, w.ctl, w.tab, w.tab_stride, w.clb, za, zb, nz, w.tile_ctr, w.hist,
                                         w.ppart, nullptr);
}

// k_list blocks for ~hint records: a power of two in [8, g_max]
static unsigned list_grid(long hint, unsigned g_max) {
  unsigned g = 8;
  while (g < g_max && (long)g * 2048 < hint) g <<= 1;
  return std::min(g, g_max);
}

// co-resident grid of a cooperative kernel (all blocks active at once)
static unsigned coop_grid(const void* fn, int per_sm_cap) {
  int nb = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, TPB, 0);
  nb = std::max(1, std::min(nb, per_sm_cap));
  return (unsigned)(nb * sms);
}
template <class K, class... A>
static cudaError_t coop_launch(K* fn, unsigned grid, cudaStream_t st, A... args) {
  void* argv[] = {(void*)&args...};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(TPB), argv, 0, st);
}

// ---------------------------------------------------------------- per objective
// The kernels templated on the objective are instantiated in one translation
// unit per objective (build.py compiles this file once more per fid with
// -DIBNB_OBJ_TU -DIBNB_FID=f); the common unit reaches them through a table
// of launchers (ObjLaunch) instead of instantiating all eleven itself.


template <class F>
struct ObjImpl {
  static void prep(const Problem& P, const IterBufs& w, long nb, const int32_t* fl, cudaStream_t st) {
    launch_prep_t<F>(P, w, nb, fl, st);
  }
  static void eval(const Problem& P, const IterBufs& w, long nk, cudaStream_t st, bool zero) {
    launch_eval_t<F>(P, w, nk, st, zero);
  }
  static int insert(const Problem& P, const IterBufs& w, long nitems, cudaStream_t st) {
    static unsigned g_max = 0;
    if (!g_max) g_max = coop_grid((const void*)k_insert<F>, 4);
    const unsigned g = (unsigned)std::min((long)g_max, tiles_for(nitems));
    return (int)coop_launch(k_insert<F>, g, st, P, w);
  }
  static void mono(const Problem& P, const IterBufs& w, long nitems, cudaStream_t st) {
    k_mono<F><<<grid_for(nitems, TPB, 148u * 12u), TPB, 0, st>>>(P, w.ctl, w.tab, w.tab_stride, w.cand, w.ok);
  }
  // `iters` iterations in one cooperative launch of k_fused (small batches)
  static int fused(const Problem& P, const IterBufs& w, int iters, long nz, unsigned grid, cudaStream_t st) {
    if constexpr (!F::CHAIN) {  // the Levy chain never takes the G = 8 path
      if (P.m == 2 && P.G == 8) return (int)coop_launch(k_fused<F, 8>, grid, st, P, w, iters, nz);
    }
    return (int)coop_launch(k_fused<F, 0>, grid, st, P, w, iters, nz);
  }
  // deep-dive chain (chain.cuh): one cooperative launch, one block per SM,
  // the block slices in dynamic shared memory (2 * per doubles)
  static int chain(const Problem& P, const IterBufs& w, const ChainBufs& cb0, int iters, unsigned sms,
                   cudaStream_t st) {
    // the slice (2 doubles per variable) and, when it fits, its term cache
    // (4K doubles per variable; not for the Levy chain sum)
    ChainBufs cb = cb0;
    // (Levy: u, v, s0 of the box and of the midpoint, 12 doubles per variable)
    const size_t tcb = sizeof(double) * (F::CHAIN ? 12 : 4 * F::K) * (size_t)cb.per;
    cb.tcache = sizeof(double) * 2 * (size_t)cb.per + tcb <= 110u * 1024u ? 1 : 0;
    if (const char* e = std::getenv("IBNB_TCACHE"))
      if (std::atoi(e) == 0) cb.tcache = 0;
    const size_t smem = sizeof(MitmTabs) + sizeof(double) * 2 * (size_t)cb.per + (cb.tcache ? tcb : 0);
    const bool mitm = P.mitm && !F::CHAIN;  // Levy: a thread per child at any d
    static size_t attr[2] = {0, 0};  // dynamic shared memory opted in so far (per instantiation)
    const void* fn = mitm ? (const void*)k_chain<F, !F::CHAIN> : (const void*)k_chain<F, false>;
    if (smem > attr[mitm ? 1 : 0]) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return (int)e;
      attr[mitm ? 1 : 0] = smem;
    }
    void* argv[] = {(void*)&P, (void*)&w, (void*)&cb, (void*)&iters};
    return (int)cudaLaunchCooperativeKernel(fn, dim3(sms), dim3(TPB), argv, smem, st);
  }
  template <int CS>
  static int chainc_cs(const Problem& P, const IterBufs& w, const ChainBufs& cb, int iters, cudaStream_t st) {
    if constexpr (!F::CHAIN) {
      const size_t smem = chainc_smem(cb.per);
      static size_t attr = 0;  // dynamic shared memory opted in so far (per instantiation)
      if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute((const void*)k_chainc<F, CS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        if (CS > 8) {
          e = cudaFuncSetAttribute((const void*)k_chainc<F, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
          if (e != cudaSuccess) return (int)e;
        }
        attr = smem;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CS);
      cfg.blockDim = dim3(TPB);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return (int)cudaLaunchKernelEx(&cfg, k_chainc<F, CS>, P, w, cb, iters);
    } else {
      return (int)cudaErrorInvalidValue;
    }
  }
  static int chainc(const Problem& P, const IterBufs& w, const ChainBufs& cb, int cs, int iters, cudaStream_t st) {
    return cs == 8 ? chainc_cs<8>(P, w, cb, iters, st) : chainc_cs<16>(P, w, cb, iters, st);
  }
  static void eval_boxes(int n, long nbox, const double* lo, const double* hi, long ld, double* out, unsigned g,
                         cudaStream_t st) {
    k_eval_boxes<F><<<g, TPB, 0, st>>>(n, nbox, lo, hi, ld, out);
  }
  static void eval_grad(int n, long nreq, const double* lo, const double* hi, long ld, const int64_t* req_box,
                        const int32_t* req_dim, double* out, unsigned g, cudaStream_t st) {
    k_eval_grad<F><<<g, TPB, 0, st>>>(n, nreq, lo, hi, ld, req_box, req_dim, out);
  }
  static const ObjLaunch* table() {
    static const ObjLaunch t{&prep, &eval, &mono, &insert, &fused, &chain, &chainc, &eval_boxes, &eval_grad};
    return &t;
  }
};

#ifdef IBNB_OBJ_TU
#if IBNB_FID == 0
using FObj = ObjExample;
#elif IBNB_FID == 1
using FObj = ObjAckley;
#elif IBNB_FID == 2
using FObj = ObjBelegundu;
#elif IBNB_FID == 3
using FObj = ObjBreiman;
#elif IBNB_FID == 4
using FObj = ObjFu;
#elif IBNB_FID == 5
using FObj = ObjGriewank;
#elif IBNB_FID == 6
using FObj = ObjLevy;
#elif IBNB_FID == 7
using FObj = ObjRastrigin;
#elif IBNB_FID == 8
using FObj = ObjSalomon;
#elif IBNB_FID == 9
using FObj = ObjStyblinski;
#elif IBNB_FID == 10
using FObj = ObjZabinsky;
#endif
IB_NS_END
namespace ib {  // the exported entry point, outside the per-objective namespace
const ObjLaunch* IBNB_CAT(obj_launch_, IBNB_FID)() { return ObjImpl<FObj>::table(); }
}  // namespace ib
#else  // the common translation unit
const ObjLaunch* obj_launch_0();
const ObjLaunch* obj_launch_1();
const ObjLaunch* obj_launch_2();
const ObjLaunch* obj_launch_3();
const ObjLaunch* obj_launch_4();
const ObjLaunch* obj_launch_5();
const ObjLaunch* obj_launch_6();
const ObjLaunch* obj_launch_7();
const ObjLaunch* obj_launch_8();
const ObjLaunch* obj_launch_9();
const ObjLaunch* obj_launch_10();
static const ObjLaunch* obj_launch(int fid) {
  static const ObjLaunch* tab[11] = {obj_launch_0(), obj_launch_1(), obj_launch_2(), obj_launch_3(),
                                     obj_launch_4(), obj_launch_5(), obj_launch_6(), obj_launch_7(),
                                     obj_launch_8(), obj_launch_9(), obj_launch_10()};
  return tab[fid];
}

// One iteration of the hot path: 4 launches (k_list, k_prep, k_child_eval,
// k_insert), every kernel reading its sizes and decisions from ctl.
// pool_bound / bmax: host upper bounds of |L| and B, used for grid sizes.
int launch_iteration(const Problem& P, const IterBufs& w, long pool_bound, long bmax, cudaStream_t st,
                     IterHook* hook, long list_hint) {
  const long kids = P.kids;
  static unsigned g_max = 0;
  if (!g_max) g_max = coop_grid((const void*)k_list, 8);
  // k_list grid: every loop is grid-strided, so any size is correct; size it
  // to the records it will scan (grid barriers get cheaper with fewer blocks)
  unsigned g_list = list_grid(list_hint, g_max);
  cudaError_t e;
  // statistics + stop test + batch size + radix select + selection (a1, a7)
  if (hook) hook->begin(3, pool_bound, st);
  e = coop_launch(k_list, g_list, st, w.pool, w.ctl, w.hist, w.sel_slot, w.sel_code, w.desc, w.desc2, w.tile_ctr,
                  w.hot0, w.hot1, kids);
  if (e != cudaSuccess) return (int)e;
  if (hook) hook->end(3, st);
  // partition (SPSD) + tables (a2, a3)
  if (hook) hook->begin(0, bmax, st);
  obj_launch(P.fid)->prep(P, w, bmax, w.free_list, st);
  if (hook) hook->end(0, st);
  // bounds of every child + incumbent (a3, a4); zeroes the scan descriptors
  if (hook) hook->begin(1, bmax * kids, st);
  obj_launch(P.fid)->eval(P, w, bmax * kids, st, true);
  if (hook) hook->end(1, st);
  if (hook) hook->exchange(st);
  // rule out (a5: lb > GUB, the first-order test) and insert the survivors
  // into L (a6), one pass
  if (hook) hook->begin(5, bmax * kids, st);
  const int ie = obj_launch(P.fid)->insert(P, w, bmax * kids, st);
  if (ie) return ie;
  if (hook) hook->end(5, st);
  LAUNCH_OK;
}

// `iters` iterations in one cooperative launch of k_fused (small batches)
int launch_fused(const Problem& P, const IterBufs& w, int iters, long bmax, cudaStream_t st) {
  const long nz = tiles_for(bmax * P.kids) + 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned grid = (unsigned)sms;  // one block per SM (launch bounds: co-resident)
  if (const char* e = std::getenv("IBNB_FUSE_GRID")) grid = (unsigned)std::max(1, std::min(atoi(e), sms));
  return obj_launch(P.fid)->fused(P, w, iters, nz, grid, st);
}

// deep-dive chain (chain.cuh): up to `iters` iterations in one cooperative
// launch, one block per SM, the block slices of the region in dynamic shared
// memory (2 * per doubles)
int launch_chain(const Problem& P, const IterBufs& w, const ChainBufs& cb, int iters, cudaStream_t st) {
  return obj_launch(P.fid)->chain(P, w, cb, iters, (unsigned)cb.grid, st);
}

size_t chainc_smem(int per) {
  return sizeof(MitmTabs) + sizeof(double) * (2 * (size_t)per + 2 * (size_t)DM_MAX * ENT + 2 * (size_t)PCAP) +
         sizeof(uint32_t) * 2 * (size_t)PCAP;
}

int launch_chainc(const Problem& P, const IterBufs& w, const ChainBufs& cb, int cs, int iters, cudaStream_t st) {
  return obj_launch(P.fid)->chainc(P, w, cb, cs, iters, st);
}

// steps a2-a6 only, for an explicit batch already in w (ib_branch): the
// parents are selected, ctl->B = nb, ctl->pcount = 0
int launch_branch(const Problem& P, const IterBufs& w, long nb, cudaStream_t st) {
  const long kids = P.kids;
  obj_launch(P.fid)->prep(P, w, nb, nullptr, st);
  obj_launch(P.fid)->eval(P, w, nb * kids, st, false);
  cudaMemsetAsync(w.desc, 0, sizeof(uint64_t) * (size_t)tiles_for(nb * kids), st);
  cudaMemsetAsync(w.desc2, 0, sizeof(uint64_t) * 2 * (size_t)tiles_for(nb * kids), st);
  cudaMemsetAsync(w.tile_ctr, 0, sizeof(uint32_t) * 4, st);
  k_cand<<<scan_grid(nb * kids), TPB, 0, st>>>(P, w.ctl, w.clb, w.cand, w.desc, w.tile_ctr);
  obj_launch(P.fid)->mono(P, w, nb * kids, st);
  k_emit<<<scan_grid(nb * kids), TPB, 0, st>>>(P, w.ctl, w.tab, w.tab_stride, w.clb, w.cand, w.ok,
                                                          w.new_slot, w.pool, w.desc2, w.tile_ctr + 1, 0, nullptr, nullptr);
  LAUNCH_OK;
}

#ifndef IBNB_OBJ_TU
__global__ void k_zero_w(Ctl* ctl) { ctl->acc_max_w = 0; }
#endif  // IBNB_OBJ_TU
#ifndef IBNB_OBJ_TU
__global__ void __launch_bounds__(TPB) k_final_w(Pool p, Ctl* ctl) { maxw_accum_dev(p, ctl); }
#endif  // IBNB_OBJ_TU
// max width of the live records into ctl->acc_max_w (final result)
int launch_final_width(Pool p, Ctl* ctl, long pool_bound, cudaStream_t st) {
  k_zero_w<<<1, 1, 0, st>>>(ctl);
  k_final_w<<<grid_for(pool_bound, TPB, 148u * 8u), TPB, 0, st>>>(p, ctl);
  LAUNCH_OK;
}

int launch_apply_pending(Ctl* ctl, long kids, cudaStream_t st) {
  k_apply_pending<<<1, 1, 0, st>>>(ctl, kids);
  LAUNCH_OK;
}

int launch_xchg_put(const Ctl* ctl, double* x, cudaStream_t st) {
  k_xchg_put<<<1, 1, 0, st>>>(ctl, x);
  LAUNCH_OK;
}
int launch_xchg_take(Ctl* ctl, const double* x, cudaStream_t st) {
  k_xchg_take<<<1, 1, 0, st>>>(ctl, x);
  LAUNCH_OK;
}

int launch_partition(Pool in, long cnt, const unsigned long long* gub_key, int known, unsigned long long prefix,
                     unsigned long long r_need, int32_t* sel_slot, uint32_t* sel_code, double* sel_lb, Pool keep,
                     uint64_t* desc, uint32_t* tile_ctr, uint64_t* keep_count, cudaStream_t st) {
  long ntiles = tiles_for(cnt);
  cudaMemsetAsync(desc, 0, sizeof(uint64_t) * 3 * (size_t)ntiles, st);
  cudaMemsetAsync(tile_ctr, 0, sizeof(uint32_t), st);
  k_partition<<<scan_grid(cnt), TPB, 0, st>>>(in, cnt, gub_key, known, prefix, r_need, sel_slot, sel_code, sel_lb,
                                                keep, desc, tile_ctr, keep_count, ntiles);
  LAUNCH_OK;
}

int launch_gc(Pool pool, Ctl* ctl, long pool_bound, uint8_t* mark, long cap, int32_t* free_list, uint64_t* desc,
              uint32_t* tile_ctr, cudaStream_t st) {
  cudaMemsetAsync(mark, 0, (size_t)cap, st);
  k_gc_mark<<<grid_for(pool_bound, TPB, 148u * 8u), TPB, 0, st>>>(pool, ctl, mark);
  long ntiles = tiles_for(cap);
  cudaMemsetAsync(desc, 0, sizeof(uint64_t) * (size_t)ntiles, st);
  cudaMemsetAsync(tile_ctr, 0, sizeof(uint32_t), st);
  k_gc_collect<<<scan_grid(cap), TPB, 0, st>>>(mark, cap, free_list, desc, tile_ctr, ctl, ntiles);
  LAUNCH_OK;
}

int launch_compact_le(const double* keys, long cnt, double thr, int64_t* out_idx, uint64_t* desc,
                      uint32_t* tile_ctr, uint64_t* out_count, cudaStream_t st) {
  if (cnt <= 0) {
    cudaMemsetAsync(out_count, 0, sizeof(uint64_t), st);
    LAUNCH_OK;
  }
  long ntiles = tiles_for(cnt);
  cudaMemsetAsync(desc, 0, sizeof(uint64_t) * (size_t)ntiles, st);
  cudaMemsetAsync(tile_ctr, 0, sizeof(uint32_t), st);
  k_compact_le<<<scan_grid(cnt), TPB, 0, st>>>(keys, cnt, thr, out_idx, desc, tile_ctr, out_count, ntiles);
  LAUNCH_OK;
}

int launch_extract(const Problem& P, Pool p, long cnt, const double* A_lo, const double* A_hi, const int32_t* sc,
                   double* out_lo, double* out_hi, double* out_lb, cudaStream_t st) {
  if (cnt > 0)
    k_extract<<<grid_for(cnt, 1, 148u * 16u), 128, 0, st>>>(P, p, cnt, A_lo, A_hi, sc, out_lo, out_hi, out_lb);
  LAUNCH_OK;
}

int launch_eval_boxes(int fid, int n, long nbox, const double* lo, const double* hi, long ld, double* out,
                      cudaStream_t st) {
  if (nbox <= 0) return 0;
  unsigned g = (unsigned)((nbox * 32 + TPB - 1) / TPB);
  obj_launch(fid)->eval_boxes(n, nbox, lo, hi, ld, out, g, st);
  LAUNCH_OK;
}

int launch_eval_grad(int fid, int n, long nreq, const double* lo, const double* hi, long ld,
                     const int64_t* req_box, const int32_t* req_dim, double* out, cudaStream_t st) {
  if (nreq <= 0) return 0;
  unsigned g = (unsigned)((nreq * 32 + TPB - 1) / TPB);
  obj_launch(fid)->eval_grad(n, nreq, lo, hi, ld, req_box, req_dim, out, g, st);
  LAUNCH_OK;
}

#ifdef IBNB_PROBE
int probe_read(unsigned long long* out) { return (int)cudaMemcpyFromSymbol(out, g_probe, sizeof(g_probe)); }
#endif
IB_NS_END  // namespace ib

IB_NS_BEGIN
// statistics + control + radix passes of an iteration on an explicit list
// (ib_select): leaves (known, prefix, need) of the B-th smallest key in ctl
int launch_select_only(Pool p, Ctl* ctl, unsigned int* hist, long n, cudaStream_t st) {
  cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned int), st);
  k_stats<<<grid_for(n, TPB, 148u * 8u), TPB, 0, st>>>(p, ctl, hist);
  for (int pass = 1; pass < 8; ++pass) k_radix<<<grid_for(n, TPB * 8, 148u * 4u), TPB, 0, st>>>(p, ctl, hist);
  LAUNCH_OK;
}
IB_NS_END  // namespace ib
#endif  // IBNB_OBJ_TU
