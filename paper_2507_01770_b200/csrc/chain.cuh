// chain.cuh -- k_chain: the deep-dive iteration kernel (included by
// bnb_kernels.cu after the phases it reuses).
//
// Regime: every iteration selects ONE region R (§3.1) and
// exactly one of its m^d subregions survives (lines 140-146), which becomes
// the next selected region.  This is the whole run of every paper function
// at n = 1,000 .. 10,000 once the R9 incumbent is known.  The
// iteration is then a chain of dependent steps, and what costs time is the
// number of grid-wide barriers and dependent memory round trips per step,
// not arithmetic.  k_chain keeps the state of the chain on chip and needs ONE
// grid barrier per iteration:
//
//  * every block holds its slice of the variables of R in shared memory and
//    the full table of R (rest accumulators + piece terms of the split
//    chunk c) in shared memory;
//  * phase 1 (between barriers), each block: (a) lower bound of its share of
//    the children (table combination, Eq. (3)-(6) natural
//    extension), midpoint upper bound for those with lb <= GUB (line 134),
//    potential candidates appended to a per-iteration list; (b) the partial
//    sum S_excl over its slice of the variables outside BOTH the current
//    chunk c and the next chunk c' = c + d (line 184): every child R' of R
//    has the same values there, so rest(R') = S_excl + the piece terms of
//    chunk c chosen by R' -- the O(n) reduction runs concurrently with the
//    child evaluation instead of before it; (c) the blocks owning chunk c'
//    tabulate its pieces (R' = R on c');
//  * barrier;
//  * phase 2, every block redundantly and deterministically (same inputs,
//    same order): incumbent GUB = min(previous, this iteration's midpoint
//    minimum), candidates lb <= GUB, first-order test (lines 142-144) and
//    widths, the survivor; the stop test (lines 148-150); the next table
//    (S_excl partials combined in a fixed order + chunk-c terms of the
//    survivor, chunk-c' entries from the owners) and the slice update.  No
//    block waits for another in phase 2, so the next phase 1 starts at once.
//
// Per-iteration buffers are triple (candidate lists, midpoint minima) or
// double (slice partials, next-chunk entries) buffered by iteration index so
// that a slow block still in phase 2 of iteration k never sees data of
// iteration k + 1.  Whenever the iteration does not continue the chain (no or
// several survivors, stop test, iteration budget), block 0 writes the
// control block, the table and the region to the archive exactly as the
// fused path would have them, and the insertion runs through the same
// emit_small_dev / cand_emit_dev as k_fused; the next launch (k_chain or
// k_fused) starts with its list phase.
//
// Requirements (checked by the host): m = 2, n >= 2 d, a non-chain objective,
// the list phase selects one region (every live record is in a hot index of
// one entry).  The accumulators are combined in a different order than the
// fused path (slice partials over 148 blocks, then the chunk terms), so the
// bounds agree with it and with the oracle to the parity tolerance, not bit
// for bit.
#pragma once

IB_NS_BEGIN

__device__ __forceinline__ bool in_chunk(int i, int c, int d, int n) { return ((i - c + n) % n) < d; }

// accumulator identity / combination for every objective (Levy, R11: one
// plain sum of chain terms)
template <class F>
__device__ __forceinline__ Iv ch_ident(int k) {
  if constexpr (F::CHAIN) return iv(0.0);
  else return acc_ident<F>(k);
}
template <class F>
__device__ __forceinline__ Iv ch_comb(int k, Iv a, Iv b) {
  if constexpr (F::CHAIN) return a + b;
  else return acc_comb<F>(k, a, b);
}

// doubles of a table entry that any reader of a chain table uses: bounds,
// box and midpoint terms, derivative ingredients, the separable flag (Levy:
// k_prep's layout up to s0 of the midpoint) -- phase 2 copies only these
// (every block reads the entries of the next chunk: L2 broadcast traffic)
template <class F>
__device__ __forceinline__ constexpr int ent_used() {
  if constexpr (F::CHAIN) return 18;
  else return E_T + 4 * F::K + 2 * F::KG + 1;
}
template <class F>
__device__ __forceinline__ void copy_entries(double* dst, const double* src, int dm) {
  constexpr int EU = ent_used<F>();
  for (int q = threadIdx.x; q < dm * EU; q += TPB) {
    const int j = q / EU, f = q - j * EU;
    dst[(size_t)j * ENT + f] = __ldcg(&src[(size_t)j * ENT + f]);
  }
}

// ------------------------------------------------------------------ Levy
// Levy (A11-A12, reading R11) in the chain: term i couples x_i and x_{i+1},
// so the chunk's table lists the affected chain terms (levy_desc, as k_prep
// writes them) and the child sums are taken over that list; a block's slice
// partial covers the pairs (i, i + 1) with i in its slice -- the value of
// x_{i1} (the next slice's first variable) is kept as a halo.
// Where the chunk's two neighbour variables live in the tables of the
// iteration buffers (tabn): the L slot at entry only, the R slot always.
constexpr int LEVY_TABN_L = DM_MAX * ENT - 16, LEVY_TABN_R = DM_MAX * ENT - 8;

// descriptors of the chain terms affected by chunk c (k_prep's list)
__device__ __forceinline__ void levy_desc(int c, int d, int n, double* T) {
  LevyChunk q = levy_chunk(c, d, n);
  int nt = 0;
  double* td = T + H_LEVY_T;
  if (q.inJ(0)) td[nt++] = (double)(0 * 65536 + q.local(0) * 256);
  const int ncand = d < n ? d + 1 : n;
  for (int t = 0; t < ncand; ++t) {
    const int i = d < n ? (c - 1 + t + n) % n : t;
    if (i > n - 2) continue;
    if (q.inJ(i) || q.inJ(i + 1)) td[nt++] = (double)(1 * 65536 + q.local(i) * 256 + q.local(i + 1));
  }
  if (q.inJ(n - 1)) td[nt++] = (double)(2 * 65536 + q.local(n - 1) * 256);
  T[H_LEVY_NT] = (double)nt;
  T[H_LEVY_LR] = (double)q.L;
  T[H_LEVY_LR + 1] = (double)q.R;
  T[H_CHUNK] = (double)c;
}

// the chunk is interior (x_1 and x_n outside it, both neighbours exist): its
// term list is L-pair, the d - 1 inner pairs, R-pair (levy_desc's result)
__device__ __forceinline__ bool levy_interior(int c, int d, int n) { return c >= 1 && c + d <= n - 1; }

// levy_desc by the lanes of a warp (same bits as levy_desc; interior chunks
// in parallel, the others on lane 0); __syncwarp before other lanes read
__device__ __forceinline__ void levy_desc_warp(int c, int d, int n, double* T) {
  const int lane = threadIdx.x & 31;
  if (levy_interior(c, d, n)) {
    if (lane <= d) {
      const int li = lane == 0 ? d : lane - 1, lj = lane == 0 ? 0 : (lane == d ? d + 1 : lane);
      T[H_LEVY_T + lane] = (double)(1 * 65536 + li * 256 + lj);
    }
    if (lane == 0) {
      T[H_LEVY_NT] = (double)(d + 1);
      T[H_LEVY_LR] = (double)(c - 1);
      T[H_LEVY_LR + 1] = (double)(c + d);
      T[H_CHUNK] = (double)c;
    }
  } else if (lane == 0) {
    levy_desc(c, d, n, T);
  }
}

// value of descriptor dsc for the child `code` (mid: at the midpoint values)
__device__ __forceinline__ Iv levy_term(const double* T, int dsc, uint32_t code, int d, bool mid) {
  const int kind = dsc >> 16, li = (dsc >> 8) & 255, lj = dsc & 255;
  auto ent = [&](int l) { return T + HDR + (size_t)(2 * l + ((code >> l) & 1u)) * ENT; };
  auto u = [&](int l) {
    return l < d ? get(ent(l) + (mid ? 12 : 2)) : get(T + H_LEVY_NB + 8 * (l - d) + (mid ? 4 : 0));
  };
  auto v = [&](int l) {
    return l < d ? get(ent(l) + (mid ? 14 : 4)) : get(T + H_LEVY_NB + 8 * (l - d) + (mid ? 6 : 2));
  };
  if (kind == 0) return get(ent(li) + (mid ? 16 : 6));
  if (kind == 1) return mulpos(u(li), v(lj));  // u >= 0, v >= 1
  return u(li);
}

// the child's chain sum: rest + the affected terms (list order, as LevyView)
__device__ __forceinline__ Iv levy_child_acc(const double* T, uint32_t code, int d, bool mid) {
  Iv a = get(T + (mid ? H_RESTM : H_REST));
  const int nt = (int)T[H_LEVY_NT];
  for (int t = 0; t < nt; ++t) a = a + levy_term(T, (int)T[H_LEVY_T + t], code, d, mid);
  return a;
}

// slice partial: the chain terms of the slice [i0, i1) that involve no
// variable of chunk c1 nor of chunk c2 (c2 < 0: none) -- pairs (i, i + 1),
// s0(x_0), u(x_{n-1}) -- box and midpoint, and the max width outside the
// chunks; (hlo, hhi): x_{i1} (halo, i1 < n)
template <class F>
__device__ __forceinline__ void chain_levy_partial(const Problem& P, const double* s_lo, const double* s_hi,
                                                   double hlo, double hhi, int i0, int i1, int c1, int c2,
                                                   double* part, double* keep) {
  const int n = P.n, d = P.d;
  Iv acc[2], accm[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) acc[k] = accm[k] = iv(0.0);
  double wmax = 0.0;
  constexpr int HB = TPB / 2;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  auto inC = [&](int i) { return in_chunk(i, c1, d, n) || (c2 >= 0 && in_chunk(i, c2, d, n)); };
  for (int i = i0 + hv; i < i1; i += HB) {
    const bool ci = inC(i);
    double a = s_lo[i - i0], bb = s_hi[i - i0];
    if (half == 1) a = bb = midpt(a, bb);
    const LevyVals v = ObjLevy::vals(Iv{a, bb});
    Iv r = iv(0.0);
    if (!ci) {
      if (half == 0) wmax = fmax(wmax, __dsub_rn(s_hi[i - i0], s_lo[i - i0]));
      if (i == 0) r = r + v.s0;
      if (i == n - 1) r = r + v.u;
    }
    if (i <= n - 2 && !ci && !inC(i + 1)) {
      double a1 = i + 1 < i1 ? s_lo[i + 1 - i0] : hlo, b1 = i + 1 < i1 ? s_hi[i + 1 - i0] : hhi;
      if (half == 1) a1 = b1 = midpt(a1, b1);
      r = r + mulpos(v.u, ObjLevy::vals(Iv{a1, b1}).v);
    }
    if (half == 0) acc[0] = acc[0] + r;
    else accm[0] = accm[0] + r;
  }
  block_reduce_prep<F, TPB>(acc, accm, wmax);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      put(part + 2 * k, acc[k]);
      put(part + 4 + 2 * k, accm[k]);
      put(keep + 2 * k, acc[k]);
      put(keep + 4 + 2 * k, accm[k]);
    }
    part[8] = keep[8] = wmax;
    part[9] = keep[9] = 0.0;
  }
}

// chain_levy_partial from the Levy value cache s_lc (u, v, s0 of the box,
// then of the midpoint, 12 doubles per slice variable: ObjLevy::vals of the
// current values, written when a variable changes) and the halo's v (box,
// midpoint) -- on warps 0..3 (named barrier 1) while warps 4..7 tabulate
// the next chunk; the same terms as chain_levy_partial (another thread
// mapping: another association, R10)
template <class F>
__device__ __forceinline__ void chain_levy_partial_cached128(const Problem& P, const double* s_lo, const double* s_hi,
                                                             const double* s_lc, Iv hvb, Iv hvm, int i0, int i1,
                                                             int c1, int c2, double* part, double* keep) {
  const int n = P.n, d = P.d;
  Iv acc = iv(0.0), accm = iv(0.0);
  double wmax = 0.0;
  constexpr int HB = 64;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  auto inC = [&](int i) { return in_chunk(i, c1, d, n) || (c2 >= 0 && in_chunk(i, c2, d, n)); };
  const int o = half == 0 ? 0 : 6;
  for (int i = i0 + hv; i < i1; i += HB) {
    const bool ci = inC(i);
    const double* lc = s_lc + (size_t)(i - i0) * 12 + o;
    Iv r = iv(0.0);
    if (!ci) {
      if (half == 0) wmax = fmax(wmax, __dsub_rn(s_hi[i - i0], s_lo[i - i0]));
      if (i == 0) r = r + get(lc + 4);
      if (i == n - 1) r = r + get(lc + 0);
    }
    if (i <= n - 2 && !ci && !inC(i + 1)) {
      const Iv v1 = i + 1 < i1 ? get(s_lc + (size_t)(i + 1 - i0) * 12 + o + 2) : (half == 0 ? hvb : hvm);
      r = r + mulpos(get(lc + 0), v1);
    }
    if (half == 0) acc = acc + r;
    else accm = accm + r;
  }
  Iv A[2] = {acc, iv(0.0)}, Am[2] = {accm, iv(0.0)};
  warp_reduce_prep<F>(A, Am, wmax);
  __shared__ Iv s_a[4], s_b[4];
  __shared__ double s_w[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_a[wid] = A[0];
    s_b[wid] = Am[0];
    s_w[wid] = wmax;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int w = 1; w < 4; ++w) {
      A[0] = A[0] + s_a[w];
      Am[0] = Am[0] + s_b[w];
      wmax = fmax(wmax, s_w[w]);
    }
    for (int k = 0; k < 2; ++k) {
      put(part + 2 * k, A[k]);
      put(part + 4 + 2 * k, Am[k]);
      put(keep + 2 * k, A[k]);
      put(keep + 4 + 2 * k, Am[k]);
    }
    part[8] = keep[8] = wmax;
    part[9] = keep[9] = 0.0;
  }
}

// the Levy values of variable x (box and midpoint: u v um vm) -> 8 doubles
__device__ __forceinline__ void levy_nb_vals(double a, double bb, double* out) {
  const LevyVals v = ObjLevy::vals(Iv{a, bb});
  const double xm = midpt(a, bb);
  const LevyVals vm = ObjLevy::vals(Iv{xm, xm});
  put(out + 0, v.u);
  put(out + 2, v.v);
  put(out + 4, vm.u);
  put(out + 6, vm.v);
}

// warp-aggregated append of (code, lb) to the iteration's candidate list
__device__ __forceinline__ void chain_append(unsigned long long* cnt, uint32_t* pc, double* pl, bool cond,
                                             uint32_t code, double lb, double* pw = nullptr, double wv = 0.0) {
  const unsigned am = __activemask();
  const unsigned mk = __ballot_sync(am, cond);
  if (!mk) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mk) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(mk));
  base = __shfl_sync(am, base, leader);
  if (cond) {
    const unsigned long long idx = base + __popc(mk & ((1u << lane) - 1u));
    if (idx < (unsigned long long)PCAP) {
      pc[idx] = code;
      pl[idx] = lb;
      if (pw) pw[idx] = wv;
    }
  }
}

// partial accumulators of a block's slice of region R (slice in s_lo / s_hi):
// box and midpoint terms of the variables NOT in chunk c1 (and, when c2 >= 0,
// not in chunk c2), max width of those variables -> part (thread 0)
template <class F>
__device__ __forceinline__ void chain_slice_partial(const Problem& P, const double* s_lo, const double* s_hi, int i0,
                                                    int i1, int c1, int c2, double* part, double* keep) {
  const int n = P.n, d = P.d;
  Iv acc[2], accm[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) acc[k] = accm[k] = iv(0.0);
#pragma unroll
  for (int k = 0; k < F::K; ++k) acc[k] = accm[k] = acc_ident<F>(k);
  double wmax = 0.0;
  constexpr int HB = TPB / 2;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  for (int i = i0 + hv; i < i1; i += HB) {
    if (in_chunk(i, c1, d, n) || (c2 >= 0 && in_chunk(i, c2, d, n))) continue;
    const double a = s_lo[i - i0], bb = s_hi[i - i0];
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
  block_reduce_prep<F, TPB>(acc, accm, wmax);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      put(part + 2 * k, acc[k]);
      put(part + 4 + 2 * k, accm[k]);
      put(keep + 2 * k, acc[k]);
      put(keep + 4 + 2 * k, accm[k]);
    }
    part[8] = keep[8] = wmax;
    part[9] = keep[9] = 0.0;
  }
}

// the same partial from the per-variable term cache s_tc (box terms then
// midpoint terms of each slice variable, 4K doubles: F::terms of the current
// values, written when a variable changes) -- the same combinations in the
// same order as chain_slice_partial, so the same bits, without evaluating
// any term
template <class F>
__device__ __forceinline__ void chain_slice_partial_cached(const Problem& P, const double* s_lo, const double* s_hi,
                                                           const double* s_tc, int i0, int i1, int c1, int c2,
                                                           double* part, double* keep) {
  const int n = P.n, d = P.d;
  constexpr int TC = 4 * F::K;
  Iv acc[2], accm[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) acc[k] = accm[k] = iv(0.0);
#pragma unroll
  for (int k = 0; k < F::K; ++k) acc[k] = accm[k] = acc_ident<F>(k);
  double wmax = 0.0;
  constexpr int HB = TPB / 2;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  for (int i = i0 + hv; i < i1; i += HB) {
    if (in_chunk(i, c1, d, n) || (c2 >= 0 && in_chunk(i, c2, d, n))) continue;
    const double* tc = s_tc + (size_t)(i - i0) * TC;
    if (half == 0) {
      wmax = fmax(wmax, __dsub_rn(s_hi[i - i0], s_lo[i - i0]));
#pragma unroll
      for (int k = 0; k < F::K; ++k) acc[k] = acc_comb<F>(k, acc[k], get(tc + 2 * k));
    } else {
#pragma unroll
      for (int k = 0; k < F::K; ++k) accm[k] = acc_comb<F>(k, accm[k], get(tc + 2 * F::K + 2 * k));
    }
  }
  block_reduce_prep<F, TPB>(acc, accm, wmax);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      put(part + 2 * k, acc[k]);
      put(part + 4 + 2 * k, accm[k]);
      put(keep + 2 * k, acc[k]);
      put(keep + 4 + 2 * k, accm[k]);
    }
    part[8] = keep[8] = wmax;
    part[9] = keep[9] = 0.0;
  }
}

// the cached partial on warps 0..3 only (named barrier 1), so that warps
// 4..7 of an owner block tabulate the next chunk meanwhile (another thread
// mapping than chain_slice_partial_cached: another association, R10)
template <class F>
__device__ __forceinline__ void chain_slice_partial_cached128(const Problem& P, const double* s_lo,
                                                              const double* s_hi, const double* s_tc, int i0, int i1,
                                                              int c1, int c2, double* part, double* keep) {
  const int n = P.n, d = P.d;
  constexpr int TC = 4 * F::K;
  Iv acc[2], accm[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) acc[k] = accm[k] = iv(0.0);
#pragma unroll
  for (int k = 0; k < F::K; ++k) acc[k] = accm[k] = acc_ident<F>(k);
  double wmax = 0.0;
  constexpr int HB = 64;
  const int hv = threadIdx.x % HB, half = threadIdx.x / HB;
  for (int i = i0 + hv; i < i1; i += HB) {
    if (in_chunk(i, c1, d, n) || (c2 >= 0 && in_chunk(i, c2, d, n))) continue;
    const double* tc = s_tc + (size_t)(i - i0) * TC;
    if (half == 0) {
      wmax = fmax(wmax, __dsub_rn(s_hi[i - i0], s_lo[i - i0]));
#pragma unroll
      for (int k = 0; k < F::K; ++k) acc[k] = acc_comb<F>(k, acc[k], get(tc + 2 * k));
    } else {
#pragma unroll
      for (int k = 0; k < F::K; ++k) accm[k] = acc_comb<F>(k, accm[k], get(tc + 2 * F::K + 2 * k));
    }
  }
  warp_reduce_prep<F>(acc, accm, wmax);
  __shared__ Iv s_a[4][2], s_b[4][2];
  __shared__ double s_w[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < F::K; ++k) {
      s_a[wid][k] = acc[k];
      s_b[wid][k] = accm[k];
    }
    s_w[wid] = wmax;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int w = 1; w < 4; ++w) {
#pragma unroll
      for (int k = 0; k < F::K; ++k) {
        acc[k] = acc_comb<F>(k, acc[k], s_a[w][k]);
        accm[k] = acc_comb<F>(k, accm[k], s_b[w][k]);
      }
      wmax = fmax(wmax, s_w[w]);
    }
    for (int k = 0; k < 2; ++k) {
      put(part + 2 * k, acc[k]);
      put(part + 4 + 2 * k, accm[k]);
      put(keep + 2 * k, acc[k]);
      put(keep + 4 + 2 * k, accm[k]);
    }
    part[8] = keep[8] = wmax;
    part[9] = keep[9] = 0.0;
  }
}

// first-order test of child `code` of the bisection table T (one thread):
// separable objectives read the per-entry flags, the others take
// child_mono_ok (bit-identical to the warp version of the other paths)
template <class F>
__device__ __forceinline__ bool chain_fo_ok(const Problem& P, const double* T, uint32_t code) {
  if constexpr (F::SEP) {
    for (int j = 0; j < P.d; ++j)
      if (T[HDR + (size_t)(2 * j + ((code >> j) & 1u)) * ENT + E_T + 4 * F::K + 2 * F::KG] != 0.0) return false;
    return true;
  } else {
    return child_mono_ok<F>(P, T, code);
  }
}

// i / per without an integer division (rper = 1 / per as float, corrected)
__device__ __forceinline__ int blk_of(int i, int per, float rper) {
  int q = __float2int_rz(__int2float_rn(i) * rper);
  if ((q + 1) * per <= i) ++q;
  if (q * per > i) --q;
  return q;
}

// chain_child_rank for slices of per >= d variables (every chunk meets at
// most two slices: those of its first and last variable), registers only
__device__ __forceinline__ int chain_child_rank_fast(int blk, int G, int per, float rper, int n, int d, int c,
                                                     int cn, int cprev, bool with_prev, int& nrank) {
  int bs[6];
  const int st[3] = {c, cn, with_prev ? cprev : c};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int e = st[q] + d - 1;
    if (e >= n) e -= n;
    bs[2 * q] = blk_of(st[q], per, rper);
    bs[2 * q + 1] = blk_of(e, per, rper);
  }
  int busy = 0, before = 0;
  bool me = false;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    bool dup = false;
#pragma unroll
    for (int z = 0; z < a; ++z) dup |= bs[z] == bs[a];
    if (!dup) {
      ++busy;
      before += bs[a] < blk ? 1 : 0;
      me |= bs[a] == blk;
    }
  }
  nrank = G - busy;
  if (2 * nrank < G) {  // degenerate (tiny grid): every block shares the children
    nrank = G;
    return blk;
  }
  return me ? -1 : blk - before;
}

// rank of block `blk` among the blocks whose slices (per variables each) meet
// none of the chunks c, cn and (k > 0) cprev -- the blocks with slice
// partials and chunk entries to compute leave the children to the others;
// -1 for a busy block.  nrank: the number of such blocks.
__device__ __forceinline__ int chain_child_rank(int blk, int G, int per, int n, int d, int c, int cn, int cprev,
                                                bool with_prev, int& nrank) {
  int ids[12];
  int nb = 0;
  const int starts[3] = {c, cn, cprev};
  for (int q = 0; q < (with_prev ? 3 : 2); ++q) {
    const int s = starts[q];
    const int e = s + d - 1;  // last variable, may pass n - 1 (wrap)
    int b0 = s / per, b1 = min(e, n - 1) / per;
    for (int b = b0; b <= b1 && nb < 12; ++b) ids[nb++] = b;
    if (e >= n)
      for (int b = 0; b <= (e - n) / per && nb < 12; ++b) ids[nb++] = b;
  }
  int busy = 0, before = 0;
  bool me = false;
  for (int a = 0; a < nb; ++a) {
    bool dup = false;
    for (int z = 0; z < a; ++z) dup |= ids[z] == ids[a];
    if (dup) continue;
    ++busy;
    if (ids[a] < blk) ++before;
    me |= ids[a] == blk;
  }
  nrank = G - busy;
  if (nb >= 12 || 2 * nrank < G) {  // degenerate (tiny slices): every block shares the children
    nrank = G;
    return blk;
  }
  return me ? -1 : blk - before;
}

// does chunk {c, ..., c + d - 1} (mod n) meet the slice [i0, i1)?
__device__ __forceinline__ bool meets(int i0, int i1, int c, int d, int n) {
  if (i0 >= i1) return false;
  const int e = c + d;  // exclusive end, may pass n (wrap)
  if (e <= n) return c < i1 && i0 < e;
  return (c < i1) || (i0 < e - n);
}

// children phase output: potential-candidate list of the iteration and the
// child lower bounds (clb[code], written for the listed children, or for
// every child when `all` -- the exit path's static-tile insertion)
struct ChainOut {
  unsigned long long* cnt;
  uint32_t* pc;
  double* pl;
  double* clb;
  bool all;
  unsigned long long* npot = nullptr;  // (IBNB_TRACE) children with lb <= GUB at the iteration start
  double* pw = nullptr;                // max width of each listed child (k_chain's phase 2 reads it)
};


// lower bound of a child from its accumulators B
template <class F>
__device__ __forceinline__ double chain_lb(const Problem& P, const Iv* B) {
  return canon_lb(outer_lo<F>(B, P.n));
}

// the rest of a child's evaluation (called by every lane of the warp, the
// child's lower bound lb already known; valid = false for a lane without a
// child): the midpoint sample (line 134) and the first-order test (lines
// 142-144) of a potential candidate (lb <= GUB at the iteration start,
// recombined from the midpoint terms -- rare), the append to the list; with
// o.all only the lower bound is stored
template <class F>
__device__ __forceinline__ void chain_leaf(const Problem& P, const double* T, double gub0, const ChainOut& o,
                                           uint32_t code, double lb, bool valid, double& best) {
  if (o.all) {
    if (valid) o.clb[code] = lb;
    return;
  }
  const bool pot = valid && lb <= gub0;
  bool keep = pot;
  double wv = 0.0;
  if (pot) {
    o.clb[code] = lb;
    // midpoint accumulators: rest + the d chunk terms as four interleaved
    // partial sums (a short dependence chain; another association of the
    // natural extension's sum, R10)
    Iv Bm[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < F::K; ++q) Bm[u][q] = u == 0 ? get(T + H_RESTM + 2 * q) : acc_ident<F>(q);
    for (int jj = 0; jj < P.d; jj += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (jj + u < P.d) {
          const double* e = T + HDR + (size_t)(2 * (jj + u) + ((code >> (jj + u)) & 1u)) * ENT;
#pragma unroll
          for (int q = 0; q < F::K; ++q) Bm[u][q] = acc_comb<F>(q, Bm[u][q], get(e + E_T + 2 * F::K + 2 * q));
          wv = fmax(wv, __dsub_rn(e[E_HI], e[E_LO]));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < F::K; ++q)
      Bm[0][q] = acc_comb<F>(q, acc_comb<F>(q, Bm[0][q], Bm[1][q]), acc_comb<F>(q, Bm[2][q], Bm[3][q]));
    best = fmin(best, outer_hi<F>(Bm[0], P.n));
    // the first-order test does not depend on GUB: taken here, so the list
    // holds only children it keeps (filtering first by the warp's smallest
    // midpoint value was measured slower: a 5-level shuffle per call)
    if constexpr (F::SEP)
      if (P.mono) keep = chain_fo_ok<F>(P, T, code);
  }
  if constexpr (!F::SEP) {
    // non-separable objectives: the warp's potential candidates one at a
    // time, a lane per split variable (child_mono_ok_warp, the decisions of
    // child_mono_ok): a serial test on one lane made its block the last at
    // the grid barrier (Levy: 0.32 -> 0.20 s)
    // Only when the warp has few of them: with many (Styblinski: ~7 per warp)
    // or product accumulators (Griewank, Zabinsky) the per-lane tests in
    // parallel are faster (measured: Griewank 0.38 s vs 1.75 s warp-only)
    if (P.mono) {
      const int lane = threadIdx.x & 31;
      unsigned pmask = __ballot_sync(0xffffffffu, pot);
      if (!F::HASPROD && __popc(pmask) <= 2) {
        bool ok_me = true;
        while (pmask) {
          const int src = __ffs(pmask) - 1;
          pmask &= pmask - 1;
          const uint32_t pc = __shfl_sync(0xffffffffu, code, src);
          const bool ok = child_mono_ok_warp<F>(P, T, pc);
          if (lane == src) ok_me = ok;
        }
        keep = pot && ok_me;
      } else if (pot) {
        keep = chain_fo_ok<F>(P, T, code);
      }
    }
  }
  if (o.npot) {  // trace statistics, one atomic per warp
    const unsigned am = __activemask(), pm = __ballot_sync(am, pot);
    if (pm && (threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(o.npot, (unsigned long long)__popc(pm));
  }
  chain_append(o.cnt, o.pc, o.pl, keep, code, lb, o.pw, wv);
}

// lower bounds of the 2^J children below accumulators A into lbs[idx ..]:
// bit J-1 first, then the lower bits (summation order: rest + tree(H .. d-1),
// then H-1 .. 0 for every child)
template <class F, int J>
struct ChainTree {
  __device__ __forceinline__ static void run(const Problem& P, const double* T, const Iv* A, double* lbs, int idx) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double* e = T + HDR + (size_t)(2 * (J - 1) + b) * ENT + E_T;
      Iv B[2];
#pragma unroll
      for (int q = 0; q < F::K; ++q) B[q] = acc_comb<F>(q, A[q], get(e + 2 * q));
      ChainTree<F, J - 1>::run(P, T, B, lbs, idx + (b << (J - 1)));
    }
  }
};
template <class F>
struct ChainTree<F, 0> {
  __device__ __forceinline__ static void run(const Problem& P, const double*, const Iv* A, double* lbs, int idx) {
    lbs[idx] = chain_lb<F>(P, A);
  }
};

// (rank, nrank): this block's share among the blocks that evaluate children
constexpr int TREE_SLOTS = 16;
template <class F, int H>
__device__ __forceinline__ double chain_children(const Problem& P, const double* T, double gub0, const ChainOut& o,
                                                 int rank = -1, int nrank = 0) {
  const int d = P.d;
  const int ng = 1 << (d - H);
  if (rank < 0) {
    rank = blockIdx.x;
    nrank = gridDim.x;
  }
  const int gpb = (ng + nrank - 1) / nrank;
  const int gb = rank * gpb, ge = min(ng, gb + gpb);
  double best = CUDART_INF;
  for (int g0 = gb; g0 < ge; g0 += TPB) {  // warp-uniform trip count (votes below)
    const int gi = g0 + threadIdx.x;
    const bool valid = gi < ge;
    const uint32_t code0 = (uint32_t)(valid ? gi : gb) << H;
    // the terms of variables H .. d-1 summed as a balanced tree (depth 4 over
    // TREE_SLOTS slots, identity padding; d - H <= 16): a short dependence chain instead of
    // d - H sequential combinations -- another association of the natural
    // extension's sum, rigorous (§2.1)
    Iv tt[TREE_SLOTS][2];
#pragma unroll
    for (int u = 0; u < TREE_SLOTS; ++u) {
      const int j = H + u;
#pragma unroll
      for (int q = 0; q < F::K; ++q) {
        if (j < d) {
          const double* e = T + HDR + (size_t)(2 * j + ((code0 >> j) & 1u)) * ENT + E_T;
          tt[u][q] = get(e + 2 * q);
        } else {
          tt[u][q] = acc_ident<F>(q);
        }
      }
    }
#pragma unroll
    for (int st = 1; st < TREE_SLOTS; st *= 2)
#pragma unroll
      for (int u = 0; u + st < TREE_SLOTS; u += 2 * st)
#pragma unroll
        for (int q = 0; q < F::K; ++q) tt[u][q] = acc_comb<F>(q, tt[u][q], tt[u + st][q]);
    Iv A[2];
#pragma unroll
    for (int q = 0; q < F::K; ++q) A[q] = acc_comb<F>(q, get(T + H_REST + 2 * q), tt[0][q]);
    double lbs[1 << H];
    ChainTree<F, H>::run(P, T, A, lbs, 0);
    if (o.all) {
#pragma unroll
      for (int q = 0; q < (1 << H); ++q)
        if (valid) o.clb[code0 | (uint32_t)q] = lbs[q];
      continue;
    }
    // potential candidates of this thread; the warp visits them one per
    // lane and round (usually one round) instead of every child slot
    uint32_t pm = 0;
#pragma unroll
    for (int q = 0; q < (1 << H); ++q) pm |= (valid && lbs[q] <= gub0) ? 1u << q : 0u;
    while (__any_sync(0xffffffffu, pm != 0)) {  // rare: a potential candidate in the warp
      const int q = pm ? __ffs(pm) - 1 : 0;
      double lq = lbs[0];
#pragma unroll
      for (int z = 1; z < (1 << H); ++z) lq = q == z ? lbs[z] : lq;
      chain_leaf<F>(P, T, gub0, o, code0 | (uint32_t)q, lq, pm != 0, best);
      pm &= pm - 1;
    }
  }
  return best;
}

// Levy children (R11): a thread per child, the chain sum over the affected
// terms (levy_child_acc); for a potential candidate the midpoint sum, the
// first-order test (child_mono_ok, k_prep's table layout) and the width
template <class F>
__device__ __forceinline__ double chain_children_levy(const Problem& P, const double* T, double gub0, const ChainOut& o,
                                                      int rank = -1, int nrank = 0) {
  if (rank < 0) {
    rank = blockIdx.x;
    nrank = gridDim.x;
  }
  const int d = P.d, n = P.n;
  const int nk = 1 << d;  // d <= 20: 32-bit division
  const int per = (nk + nrank - 1) / nrank;
  const long cb = (long)rank * per, ce = min((long)nk, cb + per);
  double best = CUDART_INF;
  // interior chunk: the d + 1 terms of every child tabulated per warp (the
  // same products in the same order as levy_child_acc: same bits)
  __shared__ Iv s_pair[TPB / 32][D_MAX + 1][4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool interior = levy_interior((int)T[H_CHUNK], d, n);
  if (interior) {
    for (int q = lane; q < 4 * (d + 1); q += 32) {
      const int tt = q >> 2, b = q & 3;
      Iv uu, vv;
      if (tt == 0) {  // x_{c-1} x_c: combo b = b_0 (b < 2)
        uu = get(T + H_LEVY_NB + 0);
        vv = get(T + HDR + (size_t)(b & 1) * ENT + 4);
      } else if (tt == d) {  // x_{c+d-1} x_{c+d}: combo b = b_{d-1}
        uu = get(T + HDR + (size_t)(2 * (d - 1) + (b & 1)) * ENT + 2);
        vv = get(T + H_LEVY_NB + 8 + 2);
      } else {  // x_{c+tt-1} x_{c+tt}: combo b = b_{tt-1} + 2 b_tt
        uu = get(T + HDR + (size_t)(2 * (tt - 1) + (b & 1)) * ENT + 2);
        vv = get(T + HDR + (size_t)(2 * tt + (b >> 1)) * ENT + 4);
      }
      s_pair[w][tt][b] = mulpos(uu, vv);
    }
    __syncwarp();
  }
  for (long c0 = cb; c0 < ce; c0 += blockDim.x) {  // warp-uniform trip count
    const long ci = c0 + threadIdx.x;
    const bool valid = ci < ce;
    const uint32_t code = (uint32_t)(valid ? ci : cb);
    Iv acc;
    if (interior) {
      acc = get(T + H_REST);
      acc = acc + s_pair[w][0][code & 1u];
      for (int tt = 1; tt < d; ++tt) acc = acc + s_pair[w][tt][((code >> (tt - 1)) & 1u) | (((code >> tt) & 1u) << 1)];
      acc = acc + s_pair[w][d][(code >> (d - 1)) & 1u];
    } else {
      acc = levy_child_acc(T, code, d, false);
    }
    const double lb = canon_lb(ObjLevy::outer(acc, n).lo);
    if (o.all) {
      if (valid) o.clb[code] = lb;
      continue;
    }
    const bool pot = valid && lb <= gub0;
    if (!__any_sync(0xffffffffu, pot)) continue;  // rare: a potential candidate in the warp
    if (o.npot) {  // trace statistics, one atomic per warp
      const unsigned pmk = __ballot_sync(0xffffffffu, pot);
      if ((threadIdx.x & 31) == 0) atomicAdd(o.npot, (unsigned long long)__popc(pmk));
    }
    // the warp's potential candidates one at a time: the midpoint sample on
    // the owning lane, the first-order test with a lane per split variable
    // (child_mono_ok_warp: the decisions of child_mono_ok) -- the serial
    // test of a chain objective made the survivor's block the last at the
    // grid barrier
    unsigned pmask = __ballot_sync(0xffffffffu, pot);
    while (pmask) {
      const int src = __ffs(pmask) - 1;
      pmask &= pmask - 1;
      const uint32_t pc = __shfl_sync(0xffffffffu, code, src);
      const double plb = __shfl_sync(0xffffffffu, lb, src);
      const bool keep = !P.mono || child_mono_ok_warp<F>(P, T, pc);
      if (lane == src) {
        o.clb[pc] = plb;
        best = fmin(best, ObjLevy::outer(levy_child_acc(T, pc, d, true), n).hi);
      }
      double wv = 0.0;
      if (lane < d) {
        const double* e = T + HDR + (size_t)(2 * lane + ((pc >> lane) & 1u)) * ENT;
        wv = __dsub_rn(e[E_HI], e[E_LO]);
      }
      wv = warp_max(wv);
      chain_append(o.cnt, o.pc, o.pl, keep && lane == src, pc, plb, o.pw, wv);
    }
  }
  return best;
}

// Meet in the middle (d >= 17): with the split variables cut into a low half
// (bits 0 .. dl-1 of the child code) and a high half (dl .. d-1), every
// child's accumulators are ONE combination  RH[h] (+) LO[l]  of two tables
// built per iteration and block:  RH[h] = rest (+) tree of the high-half
// terms chosen by h,  LO[l] = tree of the low-half terms chosen by l.  The
// natural interval extension of the sum (§2.1, Eq. 3-6) in another
// association: rigorous, equal to the oracle's left-to-right evaluation up
// to rounding (tests/tol.py).  A block builds LO in full and RH for the h of
// its own children only.
constexpr int MITM_BITS = 16;               // tree slots of one half (d - dl <= 16)
constexpr int MITM_MAX = 1024;              // entries of one table
struct MitmTabs {
  Iv lo[2][MITM_MAX];  // [accumulator][l]: consecutive l in consecutive lanes
  Iv rh[2][MITM_MAX];  // [accumulator][h - h0]: this block's high halves only
};

// split of the d bits: the low half is built by every block in full (2^dl
// entries), the high half only for the block's own children (~per / 2^dl):
// 2^dl ~ sqrt(per) minimises the table work per iteration (d = 18 on 145
// blocks: 64 + 29 entries instead of 512 + 4 with dl = d / 2)
__device__ __forceinline__ int mitm_dl(int d, int per) {
  int dl = (31 - __clz(max(per, 1))) / 2;  // largest dl with 4^dl <= per
  dl = max(dl, d - MITM_BITS);
  dl = min(dl, min(10, d - 1));
  return max(dl, 1);
}

// tree (+) of the terms of split variables j0 .. j0 + nb - 1, chosen by the
// bits of `bits` (identity-padded balanced tree over MITM_BITS slots)
template <class F>
__device__ __forceinline__ void mitm_tree(const double* T, int j0, int nb, uint32_t bits, Iv* A) {
  Iv tt[MITM_BITS][2];
#pragma unroll
  for (int u = 0; u < MITM_BITS; ++u)
#pragma unroll
    for (int q = 0; q < F::K; ++q) {
      if (u < nb) {
        const double* e = T + HDR + (size_t)(2 * (j0 + u) + ((bits >> u) & 1u)) * ENT + E_T;
        tt[u][q] = get(e + 2 * q);
      } else {
        tt[u][q] = acc_ident<F>(q);
      }
    }
#pragma unroll
  for (int st = 1; st < MITM_BITS; st *= 2)
#pragma unroll
    for (int u = 0; u + st < MITM_BITS; u += 2 * st)
#pragma unroll
      for (int q = 0; q < F::K; ++q) tt[u][q] = acc_comb<F>(q, tt[u][q], tt[u + st][q]);
#pragma unroll
  for (int q = 0; q < F::K; ++q) A[q] = tt[0][q];
}

// lower bounds of this block's share (rank of nrank) of the 2^d children of
// table T: builds the tables (all threads, synchronising), then a child per
// thread and step; returns this thread's midpoint minimum
template <class F>
__device__ __forceinline__ double chain_children_mitm(const Problem& P, const double* T, MitmTabs& M, double gub0,
                                                      const ChainOut& o, int rank = -1, int nrank = 0) {
  if (rank < 0) {
    rank = blockIdx.x;
    nrank = gridDim.x;
  }
  const int d = P.d;
  const int nk = 1 << d;  // d <= 20: 32-bit arithmetic (a 64-bit division per thread was 4 % of the samples)
  const int per = (nk + nrank - 1) / nrank;
  // the split depends on d and the grid only (the exit path's recomputation
  // over all blocks takes the same association)
  const int dl = mitm_dl(d, (nk + (int)gridDim.x - 1) / (int)gridDim.x), dh = d - dl;
  const long cb = (long)rank * per, ce = min((long)nk, cb + per);
  const uint32_t lmask = (1u << dl) - 1u;
  const int h0 = (int)(cb >> dl), h1 = ce > cb ? (int)((ce - 1) >> dl) : h0 - 1;
  const int nlo = 1 << dl, nrh = h1 - h0 + 1;
  __syncthreads();  // the previous readers of M are done
  for (int q = threadIdx.x; q < nlo + nrh; q += blockDim.x) {
    Iv A[2];
    if (q < nlo) {
      mitm_tree<F>(T, 0, dl, (uint32_t)q, A);
#pragma unroll
      for (int k = 0; k < F::K; ++k) M.lo[k][q] = A[k];
    } else {
      const int h = h0 + (q - nlo);
      mitm_tree<F>(T, dl, dh, (uint32_t)h, A);
#pragma unroll
      for (int k = 0; k < F::K; ++k) M.rh[k][h - h0] = acc_comb<F>(k, get(T + H_REST + 2 * k), A[k]);
    }
  }
  __syncthreads();
  double best = CUDART_INF;
  constexpr int U = 4;  // children per thread and step (independent loads)
  for (long c0 = cb; c0 < ce; c0 += (long)U * blockDim.x) {  // warp-uniform trip count
    double lbs[U];
    bool any = o.all;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long ci = c0 + threadIdx.x + (long)u * blockDim.x;
      const uint32_t code = (uint32_t)(ci < ce ? ci : cb);
      const uint32_t h = code >> dl, l = code & lmask;
      Iv B[2];
#pragma unroll
      for (int k = 0; k < F::K; ++k) B[k] = acc_comb<F>(k, M.rh[k][h - h0], M.lo[k][l]);
      lbs[u] = chain_lb<F>(P, B);
      any |= ci < ce && lbs[u] <= gub0;
    }
    if (o.all) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long ci = c0 + threadIdx.x + (long)u * blockDim.x;
        if (ci < ce) o.clb[ci] = lbs[u];
      }
      continue;
    }
    // potential candidates of this thread, visited one per lane and round
    uint32_t pm = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long ci = c0 + threadIdx.x + (long)u * blockDim.x;
      pm |= (ci < ce && lbs[u] <= gub0) ? 1u << u : 0u;
    }
    (void)any;
    while (__any_sync(0xffffffffu, pm != 0)) {  // rare: a potential candidate in the warp
      const int u = pm ? __ffs(pm) - 1 : 0;
      double lu = lbs[0];
#pragma unroll
      for (int z = 1; z < U; ++z) lu = u == z ? lbs[z] : lu;
      const long ci = c0 + threadIdx.x + (long)u * blockDim.x;
      chain_leaf<F>(P, T, gub0, o, (uint32_t)(pm ? ci : cb), lu, pm != 0, best);
      pm &= pm - 1;
    }
  }
  return best;
}

// entries of chunk c (pieces of its d variables) for the variables in this
// block's slice -> ent (global, d * m entries of ENT doubles)
template <class F>
__device__ __forceinline__ void chain_chunk_entries(const Problem& P, const double* s_lo, const double* s_hi, int i0,
                                                    int i1, int c, double* ent, bool with_left = false,
                                                    int tid = -1, int nth = TPB) {
  const int n = P.n, d = P.d, m = P.m;
  if (tid < 0) tid = threadIdx.x;
  for (int t = tid; t < 3 * d * m; t += nth) {
    const int e = t % (d * m), part = t / (d * m);
    const int j = e / m, p = e % m;
    const int i = (c + j) % n;
    if (i < i0 || i >= i1) continue;
    const double a = s_lo[i - i0], bb = s_hi[i - i0];
    const double pa = part_point(a, bb, m, p), pb = part_point(a, bb, m, p + 1);
    if constexpr (F::CHAIN) {  // k_prep's Levy entry layout
      double* en = ent + (size_t)e * ENT;
      if (part == 0) {
        const LevyVals v = ObjLevy::vals(Iv{pa, pb});
        en[E_LO] = pa;
        en[E_HI] = pb;
        put(en + 2, v.u);
        put(en + 4, v.v);
        put(en + 6, v.s0);
        put(en + 8, v.du);
        put(en + 10, v.sg);
      } else if (part == 1) {
        const double xm = midpt(pa, pb);
        const LevyVals vm = ObjLevy::vals(Iv{xm, xm});
        put(en + 12, vm.u);
        put(en + 14, vm.v);
        put(en + 16, vm.s0);
      }
    } else {
      piece_entry<F>(P, pa, pb, midpt(pa, pb), i, part, ent + (size_t)e * ENT);
    }
  }
  if constexpr (F::CHAIN) {
    // the chunk's right neighbour (and, with_left, its left one): the owner
    // of the variable writes its Levy values (k_prep's neighbour slots)
    const LevyChunk q = levy_chunk(c, d, n);
    if (tid == 0 && q.R >= i0 && q.R < i1) levy_nb_vals(s_lo[q.R - i0], s_hi[q.R - i0], ent + LEVY_TABN_R);
    if (with_left && tid == 0 && q.L >= i0 && q.L < i1)
      levy_nb_vals(s_lo[q.L - i0], s_hi[q.L - i0], ent + LEVY_TABN_L);
  }
}

// the G slice partials combined in a fixed order (deterministic: every block
// gets the same bits; results valid in thread 0).  L2 loads: the partials
// are rewritten by other blocks every second iteration.
template <class F>
__device__ __forceinline__ void chain_combine(const double* part, int G, Iv* acc, Iv* accm, double& wmax) {
  Iv ra[2], rm[2];
  double rw = 0.0;
#pragma unroll
  for (int k = 0; k < 2; ++k) ra[k] = rm[k] = iv(0.0);
#pragma unroll
  for (int k = 0; k < F::K; ++k) ra[k] = rm[k] = ch_ident<F>(k);
  for (int q = threadIdx.x; q < G; q += TPB) {
    const double* pt = part + (size_t)q * CH_PART;
#pragma unroll
    for (int k = 0; k < F::K; ++k) {
      ra[k] = ch_comb<F>(k, ra[k], Iv{__ldcg(pt + 2 * k), __ldcg(pt + 2 * k + 1)});
      rm[k] = ch_comb<F>(k, rm[k], Iv{__ldcg(pt + 4 + 2 * k), __ldcg(pt + 5 + 2 * k)});
    }
    rw = fmax(rw, __ldcg(pt + 8));
  }
  block_reduce_prep<F, TPB>(ra, rm, rw);
  for (int k = 0; k < 2; ++k) {
    acc[k] = ra[k];
    accm[k] = rm[k];
  }
  wmax = rw;
}

// MITM: the children by meet in the middle (d > 16) -- a template parameter so
// that each kernel holds only its own children code (instruction cache)
template <class F, bool MITM>
__global__ void __launch_bounds__(TPB, 1) k_chain(Problem P, IterBufs w, ChainBufs cb, int iters) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double s_dyn[];
  constexpr int TS = HDR + 2 * D_MAX * ENT;  // bisection tables (m = 2, d <= 16)
  __shared__ double s_T[2][TS];
  __shared__ Iv s_ra[TPB / 32][2], s_rm[TPB / 32][2];
  __shared__ double s_rw[TPB / 32];
  __shared__ double s_my[CH_PART];  // this block's last published slice partial
  __shared__ uint32_t s_code;
  __shared__ double s_lb, s_wsurv;
  __shared__ unsigned int s_ns[2];
  __shared__ double s_m[TPB / 32];
  Ctl* ctl = w.ctl;
  const int n = P.n, d = P.d, t = threadIdx.x, blk = blockIdx.x, G = gridDim.x;
  const int lane = t & 31;
  MitmTabs& M = *reinterpret_cast<MitmTabs*>(s_dyn);  // d >= 17: meet-in-the-middle tables
  double* s_lo = s_dyn + sizeof(MitmTabs) / sizeof(double);
  double* s_hi = s_lo + cb.per;
  double* s_tc = s_hi + cb.per;  // term cache (cb.tcache): 4K doubles per slice variable
  const bool tcache = cb.tcache != 0;
  const int i0 = blk * cb.per, i1 = min(n, i0 + cb.per);

  // ---- entry: list phase (block 0) -- the host launches k_chain only when
  // every live record is in a hot index of one entry
  if (blk == 0) list_small_dev(w.pool, ctl, w.hot0, w.hot1, w.sel_slot, w.sel_code, P.kids);
  grid.sync();
  if (__ldcg(&ctl->done) || __ldcg(&ctl->B) != 1ull) {  // uniform
    if (blk == 0 && t == 0) atomicAdd(&cb.exits[6], 1ull);
    return;
  }
  const unsigned long long iter0 = __ldcg(&ctl->iter), max_iter = ctl->max_iter;
  const unsigned long long pcount0 = __ldcg(&ctl->pcount);
  const double eps_f = ctl->eps_f, eps_x = ctl->eps_x;
  unsigned long long gub_key = __ldcg(&ctl->gub_key);
  // the selected region R0: materialise this block's slice (Eq. 8-11)
  int c;
  double hlo = 0.0, hhi = 0.0;  // Levy: x_{i1}, the first variable of the next slice
  {
    const int src = __ldcg(&w.sel_slot[0]);
    const uint32_t code = __ldcg(&w.sel_code[0]);
    const int psc = __ldcg(&w.src_sc[src]);
    c = (code == CODE_WHOLE) ? psc : (psc + d) % n;
    const double* slo = w.src_lo + (size_t)src * P.ld;
    const double* shi = w.src_hi + (size_t)src * P.ld;
    for (int i = i0 + t; i < i1; i += TPB) {
      double a = __ldcg(&slo[i]), bb = __ldcg(&shi[i]);
      if (code != CODE_WHOLE) {
        const int jj = (i - psc + n) % n;
        if (jj < d) {
          const int p = digit(code, jj, P.m);
          const double a2 = part_point(a, bb, P.m, p), b2 = part_point(a, bb, P.m, p + 1);
          a = a2;
          bb = b2;
        }
      }
      s_lo[i - i0] = a;
      s_hi[i - i0] = bb;
    }
    if constexpr (F::CHAIN) {  // Levy: x_{i1}, the halo (every thread, same bits)
      if (i1 < n) {
        hlo = __ldcg(&slo[i1]);
        hhi = __ldcg(&shi[i1]);
        if (code != CODE_WHOLE) {
          const int jj = (i1 - psc + n) % n;
          if (jj < d) {
            const int p = digit(code, jj, P.m);
            const double a2 = part_point(hlo, hhi, P.m, p), b2 = part_point(hlo, hhi, P.m, p + 1);
            hlo = a2;
            hhi = b2;
          }
        }
      }
    }
  }
  __syncthreads();
  Iv hvb = iv(1.0), hvm = iv(1.0);  // Levy: v of the halo x_{i1} (box, midpoint), every thread
  if constexpr (F::CHAIN) {
    if (tcache) {  // the Levy values of every slice variable (box and midpoint), once
      for (int i = i0 + t; i < i1; i += TPB) {
        const double a = s_lo[i - i0], bb = s_hi[i - i0], xm = midpt(a, bb);
        const LevyVals v = ObjLevy::vals(Iv{a, bb}), vm = ObjLevy::vals(Iv{xm, xm});
        double* lc = s_tc + (size_t)(i - i0) * 12;
        put(lc + 0, v.u);
        put(lc + 2, v.v);
        put(lc + 4, v.s0);
        put(lc + 6, vm.u);
        put(lc + 8, vm.v);
        put(lc + 10, vm.s0);
      }
      if (i1 < n) {
        const double xm = midpt(hlo, hhi);
        hvb = ObjLevy::vals(Iv{hlo, hhi}).v;
        hvm = ObjLevy::vals(Iv{xm, xm}).v;
      }
    }
  }
  if constexpr (!F::CHAIN)
  if (tcache) {  // the terms of every slice variable (box and midpoint), once
    for (int i = i0 + t; i < i1; i += TPB) {
      const double a = s_lo[i - i0], bb = s_hi[i - i0];
      Iv tb[2], tm[2];
      F::terms(Iv{a, bb}, i, n, tb);
      const double xm = midpt(a, bb);
      F::terms(Iv{xm, xm}, i, n, tm);
      double* tc = s_tc + (size_t)(i - i0) * 4 * F::K;
#pragma unroll
      for (int q = 0; q < F::K; ++q) {
        put(tc + 2 * q, tb[q]);
        put(tc + 2 * F::K + 2 * q, tm[q]);
      }
    }
  }
  // rest accumulators of R0 (variables outside chunk c) and its chunk entries
  if constexpr (F::CHAIN)
    chain_levy_partial<F>(P, s_lo, s_hi, hlo, hhi, i0, i1, c, -1, cb.part + ((size_t)1 * G + blk) * CH_PART, s_my);
  else
    chain_slice_partial<F>(P, s_lo, s_hi, i0, i1, c, -1, cb.part + ((size_t)1 * G + blk) * CH_PART, s_my);
  chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, c, cb.tabn, true);
  if (blk == 0 && t == 0) {
    for (int q = 0; q < 3; ++q) {
      cb.cnt[q] = 0ull;
      cb.gacc[q] = ~0ull;
    }
  }
  grid.sync();
  {
    double* T = s_T[0];
    Iv ra[2], rm[2];
    double rw;
    chain_combine<F>(cb.part + (size_t)1 * G * CH_PART, G, ra, rm, rw);
    if (t == 0) {
      for (int k = 0; k < 2; ++k) {
        put(T + H_REST + 2 * k, ra[k]);
        put(T + H_RESTM + 2 * k, rm[k]);
      }
      T[H_WREST] = rw;
      T[H_CHUNK] = (double)c;
      if constexpr (F::CHAIN) levy_desc(c, d, n, T);
    }
    copy_entries<F>(T + HDR, cb.tabn, d * P.m);
    if constexpr (F::CHAIN)
      if (t < 16) T[H_LEVY_NB + t] = __ldcg(&cb.tabn[LEVY_TABN_L + t]);  // L then R slot
  }
  __syncthreads();

  unsigned long long sum_cand = 0, nwidth = 0;
  int k = 0, why = 0, cprev = c;
  // phase timer (IBNB_TRACE): block 0, thread 0, ns per part into tstamp[26..31]
  unsigned long long* ts = (w.tstamp && blk == 0 && t == 0) ? w.tstamp : nullptr;
  unsigned long long tb = ts ? gtimer() : 0ull;
#define CH_TICK(slot)                      \
  if (ts) {                                \
    const unsigned long long tn = gtimer(); \
    ts[slot] += tn - tb;                   \
    tb = tn;                               \
  }
  // header of the current table in registers of every thread (the same bits
  // in every thread of every block; also in s_T for the rare readers)
  Iv hrest[2], hrestm[2];
  double hw;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    hrest[q] = get(s_T[0] + H_REST + 2 * q);
    hrestm[q] = get(s_T[0] + H_RESTM + 2 * q);
  }
  hw = s_T[0][H_WREST];
  if (t == 0) s_ns[0] = s_ns[1] = 0u;  // read after the first phase-2 barrier
  const float rper = 1.0f / (float)cb.per;
  const bool fast_rank = cb.per >= d;
  for (;; ++k) {
    const int sl = k % 3;
    double* T = s_T[k & 1];
    double* Tn = s_T[(k + 1) & 1];
    const int cn = (c + d) % n;
    const double gub0 = okey_inv(gub_key);
    // ================= phase 1
    const unsigned long long tp1 = (w.tstamp && t == 0) ? gtimer() : 0ull;  // per-role phase-1 times (trace)
    unsigned long long shared_old = ~0ull;
    if (blk == 0 && t == 0) {  // slot of the next iteration (last read before the previous barrier)
      cb.cnt[(k + 1) % 3] = 0ull;
      cb.gacc[(k + 1) % 3] = ~0ull;
      // multi-GPU: lower the shared incumbent word to this rank's GUB and
      // take the other ranks' back (one NVLink atomic; its value is needed
      // only at the end of the phase)
      if (cb.gshared) shared_old = atomicMin(cb.gshared, gub_key);
    }
    // (a) children: a thread owns the 2^H children of a code whose H low bits
    // are clear (enough groups for every thread of the grid, H <= 3)
    double best = CUDART_INF;
    int nrank = G;
    const int rank = fast_rank ? chain_child_rank_fast(blk, G, cb.per, rper, n, d, c, cn, cprev, k > 0, nrank)
                               : chain_child_rank(blk, G, cb.per, n, d, c, cn, cprev, k > 0, nrank);
    {
      ChainOut o{cb.cnt + sl, cb.pcode + (size_t)sl * PCAP, cb.plb + (size_t)sl * PCAP, w.clb, false,
                 w.tstamp ? cb.exits + 7 : nullptr, cb.pw + (size_t)sl * PCAP};
      if (rank >= 0) {
        if constexpr (F::CHAIN) best = chain_children_levy<F>(P, T, gub0, o, rank, nrank);
        else if constexpr (!MITM) best = chain_children<F, 1>(P, T, gub0, o, rank, nrank);
        else best = chain_children_mitm<F>(P, T, M, gub0, o, rank, nrank);
      }
    }
    CH_TICK(26)
    // (b) S_excl of R over this block's slice, outside chunks c and c'; a
    // slice that meets none of them (nor the chunk the last iteration changed)
    // republishes the bits of its previous partial (the full slice sum)
    bool ent_done = false;
    {
      double* dst = cb.part + ((size_t)(k & 1) * G + blk) * CH_PART;
      // (Levy: the slice's last pair reaches x_{i1}, so the halo counts)
      const int i1x = F::CHAIN ? min(n, i1 + 1) : i1;
      if (meets(i0, i1x, c, d, n) || meets(i0, i1x, cn, d, n) || (k > 0 && meets(i0, i1x, cprev, d, n))) {
        __syncthreads();  // the slice update of the last phase 2 (uniform: an owner block)
        if constexpr (F::CHAIN) {
          if (tcache) {  // warps 0..3 the partial from the value cache, warps 4..7 the entries of chunk c'
            if (t < 128)
              chain_levy_partial_cached128<F>(P, s_lo, s_hi, s_tc, hvb, hvm, i0, i1, c, cn, dst, s_my);
            else
              chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, cn, cb.tabn + (size_t)((k + 1) & 1) * DM_MAX * ENT,
                                     false, t - 128, TPB - 128);
            ent_done = true;
          } else {
            chain_levy_partial<F>(P, s_lo, s_hi, hlo, hhi, i0, i1, c, cn, dst, s_my);
          }
        } else if (tcache) {
          // warps 0..3 the partial, warps 4..7 the entries of chunk c'
          if (t < 128)
            chain_slice_partial_cached128<F>(P, s_lo, s_hi, s_tc, i0, i1, c, cn, dst, s_my);
          else
            chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, cn, cb.tabn + (size_t)((k + 1) & 1) * DM_MAX * ENT, false,
                                   t - 128, TPB - 128);
          ent_done = true;
        } else {
          chain_slice_partial<F>(P, s_lo, s_hi, i0, i1, c, cn, dst, s_my);
        }
      } else if (t < CH_PART) {
        dst[t] = s_my[t];
      }
    }
    // (c) entries of chunk c' (unchanged in every child of R)
    if (!ent_done) chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, cn, cb.tabn + (size_t)((k + 1) & 1) * DM_MAX * ENT);
    // (d) this block's midpoint minimum, ONE atomic per block (one word takes
    // every block's: per-warp atomics queue 8x as many at its L2 slice, and
    // the phase-2 load of the word waits behind them); block 0 also brings in
    // the incumbent shared with the other ranks (issued at the iteration
    // start).  The block barrier costs little: the grid barrier starts with one.
    {
      best = warp_min(best);
      if (lane == 0) s_m[t >> 5] = best;
      __syncthreads();
      if (t == 0) {
        for (int q = 1; q < TPB / 32; ++q) best = fmin(best, s_m[q]);
        if (best < CUDART_INF) atomicMin(&cb.gacc[sl], (unsigned long long)okey(best));
        if (shared_old != ~0ull) atomicMin(&cb.gacc[sl], shared_old);
      }
    }
    if (w.tstamp && t == 0) {  // phase-1 time by role: 16/17 blocks with slice work, 18/19 children only
      const int role = rank < 0 ? 16 : 18;
      atomicAdd(&w.tstamp[role], gtimer() - tp1);
      atomicAdd(&w.tstamp[role + 1], 1ull);
    }
    CH_TICK(27)
    grid.sync();
    CH_TICK(28)
    // ================= phase 2 (every block, same decisions)
    // every L2 load of the phase is issued first (one round trip): counts,
    // midpoint minimum, potential candidates, slice partials, the entries of
    // chunk c' (into Tn: the table of iteration k - 1 is no longer read)
    const unsigned long long np = __ldcg(&cb.cnt[sl]);
    const unsigned long long gk = __ldcg(&cb.gacc[sl]);
    uint32_t my_pc = 0;
    double my_pl = CUDART_INF, my_pw = 0.0;
    // the first 32 list slots with the other loads (one child is listed per
    // iteration in the deep dive); the rest only when the count says so
    if (t < 32) {
      my_pc = __ldcg(&cb.pcode[(size_t)sl * PCAP + t]);
      my_pl = __ldcg(&cb.plb[(size_t)sl * PCAP + t]);
      my_pw = __ldcg(&cb.pw[(size_t)sl * PCAP + t]);
    }
    Iv ra[2], rm[2];
    double rw = 0.0;
    {
#pragma unroll
      for (int q = 0; q < 2; ++q) ra[q] = rm[q] = iv(0.0);
#pragma unroll
      for (int q = 0; q < F::K; ++q) ra[q] = rm[q] = ch_ident<F>(q);
      const double* part = cb.part + (size_t)(k & 1) * G * CH_PART;
      for (int q = t; q < G; q += TPB) {  // G <= TPB: one partial per thread
        const double* pt = part + (size_t)q * CH_PART;
#pragma unroll
        for (int kk = 0; kk < F::K; ++kk) {
          ra[kk] = ch_comb<F>(kk, ra[kk], Iv{__ldcg(pt + 2 * kk), __ldcg(pt + 2 * kk + 1)});
          rm[kk] = ch_comb<F>(kk, rm[kk], Iv{__ldcg(pt + 4 + 2 * kk), __ldcg(pt + 5 + 2 * kk)});
        }
        rw = fmax(rw, __ldcg(pt + 8));
      }
      const double* en = cb.tabn + (size_t)((k + 1) & 1) * DM_MAX * ENT;
      copy_entries<F>(Tn + HDR, en, d * P.m);
      if constexpr (F::CHAIN)
        if (t < 8) Tn[H_LEVY_NB + 8 + t] = __ldcg(&en[LEVY_TABN_R + t]);  // R slot of chunk c'
    }
    if (gk < gub_key) gub_key = gk;
    const double gub = okey_inv(gub_key);
    if (ts) ts[25] += np;  // trace: potential candidates kept (first-order test passed) per iteration
    const bool fits = np <= (unsigned long long)PCAP;
    const int npi = fits ? (int)np : 0;
    if (npi > 32 && t >= 32 && t < npi) {  // uniform per block (np is the same everywhere)
      my_pc = __ldcg(&cb.pcode[(size_t)sl * PCAP + t]);
      my_pl = __ldcg(&cb.plb[(size_t)sl * PCAP + t]);
      my_pw = __ldcg(&cb.pw[(size_t)sl * PCAP + t]);
    }
    // warp level of the (fixed-order) reduction of the slice partials
    warp_reduce_prep<F>(ra, rm, rw);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < F::K; ++q) {
        s_ra[t >> 5][q] = ra[q];
        s_rm[t >> 5][q] = rm[q];
      }
      s_rw[t >> 5] = rw;
    }
    // candidates (lb <= GUB; the first-order test and the widths were taken
    // in phase 1), a thread each: the survivors are counted, the survivor's
    // code, bound and width are read back only when it is the only one
    if (t == 0) s_ns[(k + 1) & 1] = 0u;  // last read before this iteration's grid barrier
    if (t < npi && my_pl <= gub) {
      atomicAdd(&s_ns[k & 1], 1u);
      s_code = my_pc;
      s_lb = my_pl;
      s_wsurv = my_pw;
    }
    __syncthreads();  // the only block barrier of phase 2
    const unsigned ns = s_ns[k & 1];
    const uint32_t scode = s_code;
    const double slb = s_lb, swid = s_wsurv;
    bool cont = fits;
    why = 2;
    if (cont) {
      cont = ns == 1;
      why = ns == 0 ? 0 : 1;
      if (cont) {
        // the next list phase on the single live record (list_small_dev's
        // decisions): stop test (lines 148-150), iteration limit, budget
        if (__dsub_ru(gub, slb) <= eps_f) {
          nwidth += 1;
          if (fmax(hw, swid) <= eps_x) cont = false, why = 3;
        }
        if (cont && iter0 + (unsigned long long)k + 1 >= max_iter) cont = false, why = 4;
        if (cont && k + 1 >= iters) cont = false, why = 5;
      }
      if (cont) sum_cand += ns;
    }
    CH_TICK(29)
    if (!cont) break;  // uniform: every block took the same decisions
    // ---- continue: the survivor R' becomes the selected region.  Every
    // warp builds the header of R' itself, lanes in parallel: lane l < 8
    // holds warp l's partial of S_excl, lane j < d the terms of R' in chunk c
    // (not in c', n >= 2d); an xor butterfly leaves the same bits in every
    // lane of every warp of every block (commutative combinations): rest(R')
    // = S_excl + the chunk-c terms of R'
    {
      Iv A[2], Am[2];
      double W = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) A[q] = Am[q] = iv(0.0);
#pragma unroll
      for (int q = 0; q < F::K; ++q) {
        A[q] = lane < TPB / 32 ? s_ra[lane][q] : ch_ident<F>(q);
        Am[q] = lane < TPB / 32 ? s_rm[lane][q] : ch_ident<F>(q);
      }
      if (lane < TPB / 32) W = s_rw[lane];
      if constexpr (F::CHAIN) {
        // Levy: the terms of chunk c at the survivor, except the pair that
        // reaches into chunk c' (x_{c+d-1} x_{c+d}: the R neighbour)
        const int nt = (int)T[H_LEVY_NT];
        if (lane < nt) {
          const int dsc = (int)T[H_LEVY_T + lane];
          if (!((dsc >> 16) == 1 && (dsc & 255) == d + 1)) {
            A[0] = A[0] + levy_term(T, dsc, scode, d, false);
            Am[0] = Am[0] + levy_term(T, dsc, scode, d, true);
          }
        }
        if (lane < d) {
          const double* e = T + HDR + (size_t)(2 * lane + ((scode >> lane) & 1u)) * ENT;
          W = fmax(W, __dsub_rn(e[E_HI], e[E_LO]));
        }
      } else if (lane < d) {
        const double* e = T + HDR + (size_t)(2 * lane + ((scode >> lane) & 1u)) * ENT;
#pragma unroll
        for (int q = 0; q < F::K; ++q) {
          A[q] = acc_comb<F>(q, A[q], get(e + E_T + 2 * q));
          Am[q] = acc_comb<F>(q, Am[q], get(e + E_T + 2 * F::K + 2 * q));
        }
        W = fmax(W, __dsub_rn(e[E_HI], e[E_LO]));
      }
      warp_reduce_prep<F>(A, Am, W);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        hrest[q] = A[q];
        hrestm[q] = Am[q];
      }
      hw = W;
      // the header also in s_T for the readers of the table (children, the
      // first-order test, the exit path): every warp writes the same bits
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          put(Tn + H_REST + 2 * q, hrest[q]);
          put(Tn + H_RESTM + 2 * q, hrestm[q]);
        }
        Tn[H_WREST] = hw;
        Tn[H_CHUNK] = (double)cn;
        if constexpr (F::CHAIN) {
          // the term list of chunk c' and its left neighbour x_{c+d-1} (the
          // survivor's last piece); the right one came from its owner
          const double* e = T + HDR + (size_t)(2 * (d - 1) + ((scode >> (d - 1)) & 1u)) * ENT;
          put(Tn + H_LEVY_NB + 0, get(e + 2));
          put(Tn + H_LEVY_NB + 2, get(e + 4));
          put(Tn + H_LEVY_NB + 4, get(e + 12));
          put(Tn + H_LEVY_NB + 6, get(e + 14));
        }
      }
      if constexpr (F::CHAIN) levy_desc_warp(cn, d, n, Tn);
      __syncwarp();
    }
    // slice update: chunk c variables take the survivor's pieces (read by
    // this block's next slice partial after its barrier)
    for (int j = t; j < d; j += TPB) {
      const int i = (c + j) % n;
      if (i >= i0 && i < i1) {
        const double* e = T + HDR + (size_t)(2 * j + ((scode >> j) & 1u)) * ENT;
        s_lo[i - i0] = e[E_LO];
        s_hi[i - i0] = e[E_HI];
        if (tcache) {
          if constexpr (F::CHAIN) {  // the entry's Levy values (k_prep's layout: ObjLevy::vals of the piece)
            double* lc = s_tc + (size_t)(i - i0) * 12;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              lc[q] = e[2 + q];       // u v s0 of the box
              lc[6 + q] = e[12 + q];  // u v s0 of the midpoint
            }
          } else {  // the piece's terms are the entry's (piece_entry: same F::terms, same arguments)
            double* tc = s_tc + (size_t)(i - i0) * 4 * F::K;
#pragma unroll
            for (int q = 0; q < 4 * F::K; ++q) tc[q] = e[E_T + q];
          }
        }
      }
    }
    if constexpr (F::CHAIN) {  // the halo x_{i1} (every thread)
      if (i1 < n && in_chunk(i1, c, d, n)) {
        const int j = (i1 - c + n) % n;
        const double* e = T + HDR + (size_t)(2 * j + ((scode >> j) & 1u)) * ENT;
        hlo = e[E_LO];
        hhi = e[E_HI];
        hvb = get(e + 4);
        hvm = get(e + 14);
      }
    }
    cprev = c;
    c = cn;
    CH_TICK(30)
    if (ts) ts[31] += 1;
  }
#undef CH_TICK
  // ================= leave the chain at iteration k (all blocks)
  // iterations 0 .. k-1 ended inside the chain; iteration k is ended by the
  // insertion below and the next launch's list phase (pending end)
  double* T = s_T[k & 1];
  if (blk == 0 && t == 0) atomicAdd(&cb.exits[why], 1ull);
  const int slot = (int)w.free_list[__ldcg(&ctl->free_top) - 1];  // archive slot of R (prep's choice)
  for (int i = i0 + t; i < i1; i += TPB) {
    w.dst_lo[(size_t)slot * P.ld + i] = s_lo[i - i0];
    w.dst_hi[(size_t)slot * P.ld + i] = s_hi[i - i0];
  }
  if (blk == 0) {
    for (int q = t; q < w.tab_stride; q += TPB) w.tab[q] = T[q];
    if (t == 0) {
      w.new_slot[0] = slot;
      w.dst_sc[slot] = c;
      const unsigned long long K = (unsigned long long)k;
      ctl->gub_key = gub_key;
      ctl->iter = iter0 + K;
      ctl->evals += K * (unsigned long long)P.kids;
      ctl->sum_B += K;
      ctl->sum_cand += sum_cand;
      ctl->sum_pool += K * pcount0;
      ctl->nwidth += nwidth;
    }
    __syncthreads();
  }
  const unsigned long long np = __ldcg(&cb.cnt[k % 3]);
  if (np <= (unsigned long long)PCAP) {
    if (blk == 0) {
      __threadfence_block();
      emit_small_dev<F>(P, ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, cb.pcode + (size_t)(k % 3) * PCAP,
                        (int)np, w.hot0, w.hot1, false);
    }
    return;
  }
  // many potential candidates: the static-tile insertion pass over every child
  // (descriptors zeroed first; the phase wrote clb for listed children only,
  // so every child's lower bound is recomputed -- same bits)
  {
    const long nz = 3 * (((long)P.kids + TILE - 1) / TILE + 1);
    for (long q = (long)blk * TPB + t; q < nz; q += (long)G * TPB) w.desc2[q] = 0;
    ChainOut o{nullptr, nullptr, nullptr, w.clb, true};
    if constexpr (F::CHAIN) chain_children_levy<F>(P, T, 0.0, o);
    else if constexpr (!MITM) chain_children<F, 1>(P, T, 0.0, o);
    else chain_children_mitm<F>(P, T, M, 0.0, o);
  }
  grid.sync();
  cand_emit_dev<F>(P, ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.desc2, w.hot0, w.hot1);
}

IB_NS_END  // namespace ib
