// scan.cuh -- single-pass stable stream compaction: a shared-memory block
// scan plus decoupled look-back across tiles (Merrill & Garland's scheme),
// generalised to NC independent counters so that a 3-way stable partition
// (select / keep / tie) runs in one pass over the list.
//
// Tiles are numbered by an atomic ticket taken at block start, so a tile only
// ever waits on tiles that are already resident: no deadlock whatever order
// the hardware schedules blocks in.  Each tile publishes, per counter, one
// 64-bit descriptor word = (flag << 62) | value with a single atomic store,
// so flag and value are always observed together.
#pragma once
#include <stdint.h>

namespace ib {

constexpr uint64_t DL_FLAG_AGG = 1ull << 62;
constexpr uint64_t DL_FLAG_PFX = 2ull << 62;
constexpr uint64_t DL_VMASK = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t dl_load(const uint64_t* p) {
  return *(const volatile uint64_t*)p;
}
__device__ __forceinline__ void dl_store(uint64_t* p, uint64_t v) {
  atomicExch((unsigned long long*)p, (unsigned long long)v);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of per-thread counts (NC counters).
// Returns the exclusive prefix of this thread inside the block in `ex` and
// the block total in `tot` (valid in all threads).
template <int NC, int TPB>
__device__ __forceinline__ void block_exclusive_scan(const uint32_t (&cnt)[NC], uint32_t (&ex)[NC],
                                                     uint32_t (&tot)[NC]) {
  constexpr int NW = TPB / 32;
  __shared__ uint32_t s_warp[NC][NW];
  __shared__ uint32_t s_tot[NC];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t v = cnt[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    ex[c] = v - cnt[c];
    if (lane == 31) s_warp[c][wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint32_t v = lane < NW ? s_warp[c][lane] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane < NW) s_warp[c][lane] = incl - v;  // exclusive warp offsets
      if (lane == 31) s_tot[c] = incl;            // block total
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    ex[c] += s_warp[c][wid];
    tot[c] = s_tot[c];
  }
  __syncthreads();
}

// Decoupled look-back: given the block aggregate `agg` of tile `tile`,
// publish it and compute the exclusive prefix of the tile over all earlier
// tiles.  Must be called by all threads of the block; returns the prefix in
// every thread.
template <int NC>
__device__ __forceinline__ void dl_lookback(uint64_t* desc, uint32_t tile, const uint32_t (&agg)[NC],
                                            uint64_t (&pfx)[NC]) {
  __shared__ uint64_t s_pfx[NC];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int c = 0; c < NC; ++c) {
      uint64_t* dc = desc + c;  // descriptor of (tile t, counter c) at desc[t * NC + c]
      if (tile == 0) {
        if (lane == 0) {
          dl_store(dc, DL_FLAG_PFX | (uint64_t)agg[c]);
          s_pfx[c] = 0;
        }
        continue;
      }
      if (lane == 0) dl_store(dc + (size_t)tile * NC, DL_FLAG_AGG | (uint64_t)agg[c]);
      uint64_t run = 0;
      long p = (long)tile - 1;
      while (true) {
        long idx = p - lane;
        uint64_t d = idx >= 0 ? dl_load(dc + (size_t)idx * NC) : (DL_FLAG_PFX | 0ull);
        while (__any_sync(0xffffffffu, (d >> 62) == 0)) {
          if ((d >> 62) == 0) d = dl_load(dc + (size_t)idx * NC);
        }
        unsigned pm = __ballot_sync(0xffffffffu, (d >> 62) == 2);
        if (pm) {
          int first = __ffs(pm) - 1;
          run += warp_sum_u64(lane <= first ? (d & DL_VMASK) : 0ull);
          break;
        }
        run += warp_sum_u64(d & DL_VMASK);
        p -= 32;
      }
      if (lane == 0) {
        dl_store(dc + (size_t)tile * NC, DL_FLAG_PFX | (run + (uint64_t)agg[c]));
        s_pfx[c] = run;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) pfx[c] = s_pfx[c];
  __syncthreads();
}

}  // namespace ib
