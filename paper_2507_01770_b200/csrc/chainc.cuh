// chainc.cuh -- k_chainc: the deep-dive chain of k_chain (chain.cuh) on ONE
// thread-block cluster of CS CTAs (included by bnb_kernels.cu after
// chain.cuh, whose helpers it reuses).
//
// Same iteration, same decisions as k_chain (§3.1:
// select the single live region R, partition it along chunk c, bound the
// m^d children, sample the midpoints of those that can still lower GUB, rule
// out by GUB and by the first-order test, keep the single survivor), but the
// per-iteration exchange between CTAs goes through distributed shared memory
// and the cluster barrier instead of L2 and the grid barrier:
//
//  * phase 1, every CTA: its share of the children (potential candidates
//    appended to ITS OWN shared list), the slice partial S_excl of its
//    variables (own shared memory), the entries of chunk c' for the variables
//    it owns (own shared memory), its midpoint minimum;
//  * barrier.cluster (one per iteration);
//  * phase 2, every CTA redundantly: reads the CS counts, minima, partials and
//    lists and the chunk-c' entries from the owners' shared memory (DSMEM),
//    then takes k_chain's decisions in the same order.
//
// Exchange buffers are double buffered by iteration parity: a CTA in phase 2
// of iteration k has passed barrier k, so every CTA finished phase 2 of
// k - 1 and no one still reads the parity-(k+1) buffers it overwrites in
// phase 1 of k + 1.  Every path ends with a cluster barrier so that no CTA
// exits while another may read its shared memory.
//
// With CS = 16 CTAs an iteration costs a cluster barrier (~0.25 us measured,
// scripts/micro/sync_bench.cu) and DSMEM round trips instead of a 148-CTA
// grid barrier (~1.2 us) and L2 round trips; the arithmetic of the children
// (2^d lower bounds of d table terms each) and of the slices (n / CS
// variables per CTA) is small enough at n <= ~10^5 that the other 132 SMs
// would only add synchronisation.  Entry, exit and insertion are k_chain's.
#pragma once

IB_NS_BEGIN

template <class F, int CS>
__global__ void __launch_bounds__(TPB, 1) k_chainc(Problem P, IterBufs w, ChainBufs cb, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double s_dyn[];
  constexpr int TS = HDR + 2 * D_MAX * ENT;
  constexpr int XCAP = PCAP;  // potential candidates per CTA and iteration
  constexpr int XENT = DM_MAX * ENT;
  __shared__ double s_T[2][TS];
  __shared__ uint32_t s_pc[PCAP];
  __shared__ double s_pl[PCAP];
  __shared__ double s_my[CH_PART];
  __shared__ double x_part[2][CH_PART];
  __shared__ double x_best[2];
  __shared__ unsigned long long x_cnt[2];
  __shared__ unsigned int s_off[CS + 1];
  __shared__ unsigned long long s_gk;
  __shared__ int s_over;
  __shared__ Iv s_ra[2], s_rm[2];
  __shared__ double s_rw;
  __shared__ uint32_t s_code;
  __shared__ double s_lb, s_wsurv;
  __shared__ unsigned int s_nc, s_ns;
  Ctl* ctl = w.ctl;
  const int n = P.n, d = P.d, t = threadIdx.x, blk = blockIdx.x;
  const int lane = t & 31, wid = t >> 5;
  const int tabw = d * P.m * ENT;
  const int per = cb.per;
  MitmTabs& M = *reinterpret_cast<MitmTabs*>(s_dyn);
  double* s_lo = s_dyn + sizeof(MitmTabs) / sizeof(double);
  double* s_hi = s_lo + per;
  double* x_ent = s_lo + 2 * per;                       // [2][XENT]
  double* x_pl = x_ent + 2 * XENT;                      // [2][XCAP]
  uint32_t* x_pc = reinterpret_cast<uint32_t*>(x_pl + 2 * XCAP);  // [2][XCAP]
  const int i0 = blk * per, i1 = min(n, i0 + per);

  // ---- entry (k_chain's, the cluster barrier for the grid barrier)
  if (blk == 0) list_small_dev(w.pool, ctl, w.hot0, w.hot1, w.sel_slot, w.sel_code, P.kids);
  cl.sync();
  if (__ldcg(&ctl->done) || __ldcg(&ctl->B) != 1ull) {  // uniform
    if (blk == 0 && t == 0) atomicAdd(&cb.exits[6], 1ull);
    return;  // no CTA touched another's shared memory yet
  }
  const unsigned long long iter0 = __ldcg(&ctl->iter), max_iter = ctl->max_iter;
  const unsigned long long pcount0 = __ldcg(&ctl->pcount);
  const double eps_f = ctl->eps_f, eps_x = ctl->eps_x;
  unsigned long long gub_key = __ldcg(&ctl->gub_key);
  int c;
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
  }
  if (t == 0) x_cnt[0] = x_cnt[1] = 0ull;
  __syncthreads();
  chain_slice_partial<F>(P, s_lo, s_hi, i0, i1, c, -1, cb.part + ((size_t)1 * CS + blk) * CH_PART, s_my);
  chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, c, cb.tabn);
  cl.sync();
  {
    double* T = s_T[0];
    Iv ra[2], rm[2];
    double rw;
    chain_combine<F>(cb.part + (size_t)1 * CS * CH_PART, CS, ra, rm, rw);
    if (t == 0) {
      for (int q = 0; q < 2; ++q) {
        put(T + H_REST + 2 * q, ra[q]);
        put(T + H_RESTM + 2 * q, rm[q]);
      }
      T[H_WREST] = rw;
      T[H_CHUNK] = (double)c;
    }
    for (int q = t; q < tabw; q += TPB) T[HDR + q] = __ldcg(&cb.tabn[q]);
  }
  __syncthreads();

  unsigned long long sum_cand = 0, nwidth = 0;
  int k = 0, why = 0, cprev = c;
  bool fits = true;
  unsigned int total = 0;
  unsigned long long* ts = (w.tstamp && blk == 0 && t == 0) ? w.tstamp : nullptr;
  unsigned long long tb = ts ? gtimer() : 0ull;
#define CH_TICK(slot)                       \
  if (ts) {                                 \
    const unsigned long long tn = gtimer(); \
    ts[slot] += tn - tb;                    \
    tb = tn;                                \
  }
  for (;; ++k) {
    const int par = k & 1;
    double* T = s_T[par];
    double* Tn = s_T[par ^ 1];
    const int cn = (c + d) % n;
    const double gub0 = okey_inv(gub_key);
    // ================= phase 1 (this CTA's shares, into its own shared memory)
    double best = CUDART_INF;
    {
      ChainOut o{&x_cnt[par], x_pc + par * XCAP, x_pl + par * XCAP, w.clb, false};
      best = chain_children_mitm<F>(P, T, M, gub0, o);
    }
    CH_TICK(26)
    if (meets(i0, i1, c, d, n) || meets(i0, i1, cn, d, n) || (k > 0 && meets(i0, i1, cprev, d, n)))
      chain_slice_partial<F>(P, s_lo, s_hi, i0, i1, c, cn, x_part[par], s_my);
    else if (t < CH_PART)
      x_part[par][t] = s_my[t];
    chain_chunk_entries<F>(P, s_lo, s_hi, i0, i1, cn, x_ent + (par ^ 1) * XENT);
    {
      __shared__ double s_m[TPB / 32];
      best = warp_min(best);
      if (lane == 0) s_m[wid] = best;
      __syncthreads();
      if (t == 0) {
        for (int q = 1; q < TPB / 32; ++q) best = fmin(best, s_m[q]);
        x_best[par] = best;
      }
    }
    CH_TICK(27)
    cl.sync();
    CH_TICK(28)
    // ================= phase 2 (every CTA, same decisions): DSMEM reads
    if (wid == 0) {
      // counts -> offsets of the merged list (CTA rank order), minima
      unsigned long long cq = 0;
      double bq = CUDART_INF;
      if (lane < CS) {
        cq = *cl.map_shared_rank(&x_cnt[par], (unsigned)lane);
        bq = *cl.map_shared_rank(&x_best[par], (unsigned)lane);
      }
      const int over = __any_sync(0xffffffffu, cq > (unsigned long long)XCAP);
      unsigned int v = (unsigned int)min(cq, (unsigned long long)XCAP);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane < CS) s_off[lane + 1] = v;
      bq = warp_min(bq);
      if (lane == 0) {
        s_off[0] = 0;
        s_over = over;
        s_gk = bq < CUDART_INF ? okey(bq) : ~0ull;
      }
    } else if (wid == 1) {
      // slice partials, combined in CTA rank order (fixed: same bits in every CTA)
      Iv ra[2], rm[2];
      double rw = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) ra[q] = rm[q] = iv(0.0);
#pragma unroll
      for (int q = 0; q < F::K; ++q) ra[q] = rm[q] = acc_ident<F>(q);
      if (lane < CS) {
        const double* pt = cl.map_shared_rank(&x_part[par][0], (unsigned)lane);
#pragma unroll
        for (int kk = 0; kk < F::K; ++kk) {
          ra[kk] = acc_comb<F>(kk, ra[kk], Iv{pt[2 * kk], pt[2 * kk + 1]});
          rm[kk] = acc_comb<F>(kk, rm[kk], Iv{pt[4 + 2 * kk], pt[5 + 2 * kk]});
        }
        rw = fmax(rw, pt[8]);
      }
      warp_reduce_prep<F>(ra, rm, rw);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          s_ra[q] = ra[q];
          s_rm[q] = rm[q];
        }
        s_rw = rw;
      }
    }
    // entries of chunk c' from the CTAs owning its variables (into Tn: the
    // table of iteration k - 1 is no longer read)
    for (int q = t; q < tabw; q += TPB) {
      const int j = q / (P.m * ENT);
      const int owner = ((c + d + j) % n) / per;
      Tn[HDR + q] = cl.map_shared_rank(x_ent + (par ^ 1) * XENT, (unsigned)owner)[q];
    }
    if (t == 0) {
      s_nc = 0;
      s_ns = 0;
      x_cnt[par ^ 1] = 0ull;  // readers of parity k + 1 (phase 2 of k - 1) are done
    }
    __syncthreads();
    if (s_gk < gub_key) gub_key = s_gk;
    const double gub = okey_inv(gub_key);
    total = s_off[CS];
    fits = !s_over && total <= (unsigned int)PCAP;
    if (fits) {
      for (unsigned int q = t; q < total; q += TPB) {
        int r = 0;
        while (r + 1 < CS && s_off[r + 1] <= q) ++r;
        const unsigned int idx = q - s_off[r];
        s_pc[q] = cl.map_shared_rank(x_pc + par * XCAP, (unsigned)r)[idx];
        s_pl[q] = cl.map_shared_rank(x_pl + par * XCAP, (unsigned)r)[idx];
      }
    }
    __syncthreads();
    const int npi = fits ? (int)total : 0;
    for (int q = wid; q < npi; q += TPB / 32) {
      if (!(s_pl[q] <= gub)) continue;  // warp-uniform
      const uint32_t code = s_pc[q];
      double wl = 0.0;
      if (lane < d) {
        const double* e = T + HDR + (size_t)(2 * lane + ((code >> lane) & 1u)) * ENT;
        wl = __dsub_rn(e[E_HI], e[E_LO]);
      }
      wl = warp_max(wl);
      if (lane == 0) {
        atomicAdd(&s_nc, 1u);
        atomicAdd(&s_ns, 1u);
        s_code = code;
        s_lb = s_pl[q];
        s_wsurv = fmax(T[H_WREST], wl);
      }
    }
    __syncthreads();
    bool cont = fits;
    why = 2;
    if (cont) {
      const unsigned ns = s_ns;
      cont = ns == 1;
      why = ns == 0 ? 0 : 1;
      if (cont) {
        if (__dsub_ru(gub, s_lb) <= eps_f) {
          nwidth += 1;
          if (s_wsurv <= eps_x) cont = false, why = 3;
        }
        if (cont && iter0 + (unsigned long long)k + 1 >= max_iter) cont = false, why = 4;
        if (cont && k + 1 >= iters) cont = false, why = 5;
      }
      if (cont) sum_cand += s_nc;
    }
    CH_TICK(29)
    if (!cont) break;  // uniform
    const uint32_t scode = s_code;
    if (t == 0) {
      Iv ra[2], rm[2];
      double rw = s_rw;
      for (int q = 0; q < 2; ++q) {
        ra[q] = s_ra[q];
        rm[q] = s_rm[q];
      }
      for (int j = 0; j < d; ++j) {
        const double* e = T + HDR + (size_t)(2 * j + ((scode >> j) & 1u)) * ENT;
#pragma unroll
        for (int q = 0; q < F::K; ++q) {
          ra[q] = acc_comb<F>(q, ra[q], get(e + E_T + 2 * q));
          rm[q] = acc_comb<F>(q, rm[q], get(e + E_T + 2 * F::K + 2 * q));
        }
        rw = fmax(rw, __dsub_rn(e[E_HI], e[E_LO]));
      }
      for (int q = 0; q < 2; ++q) {
        put(Tn + H_REST + 2 * q, ra[q]);
        put(Tn + H_RESTM + 2 * q, rm[q]);
      }
      Tn[H_WREST] = rw;
      Tn[H_CHUNK] = (double)cn;
    }
    for (int j = t; j < d; j += TPB) {
      const int i = (c + j) % n;
      if (i >= i0 && i < i1) {
        const double* e = T + HDR + (size_t)(2 * j + ((scode >> j) & 1u)) * ENT;
        s_lo[i - i0] = e[E_LO];
        s_hi[i - i0] = e[E_HI];
      }
    }
    __syncthreads();
    cprev = c;
    c = cn;
    CH_TICK(30)
    if (ts) ts[31] += 1;
  }
#undef CH_TICK
  // ================= leave the chain at iteration k (k_chain's exit)
  double* T = s_T[k & 1];
  if (blk == 0 && t == 0) atomicAdd(&cb.exits[why], 1ull);
  const int slot = (int)w.free_list[__ldcg(&ctl->free_top) - 1];
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
  if (fits) {
    cl.sync();  // the archive row and the table are complete; DSMEM reads done
    if (blk == 0) {
      __threadfence_block();
      emit_small_dev<F>(P, ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, s_pc, (int)total, w.hot0, w.hot1,
                        false);
    }
    return;
  }
  {
    const long nz = 3 * (((long)P.kids + TILE - 1) / TILE + 1);
    for (long q = (long)blk * TPB + t; q < nz; q += (long)CS * TPB) w.desc2[q] = 0;
    ChainOut o{nullptr, nullptr, nullptr, w.clb, true};
    chain_children_mitm<F>(P, T, M, 0.0, o);
  }
  cl.sync();
  cand_emit_dev<F>(P, ctl, w.tab, w.tab_stride, w.clb, w.new_slot, w.pool, w.desc2, w.hot0, w.hot1);
}

IB_NS_END  // namespace ib
