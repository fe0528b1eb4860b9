// nmx_merge.cuh -- K10: merge-path element-wise addition of two sorted unique COO
// matrices (keys (src << 32) | dst, u64 counts). C = A + B is the union of the
// keys; a key present in both inputs gets the sum of its counts. The summed
// matrix of several windows is exactly
// build_matrices(stream, window_size=len(stream)) (traffic.py:221-242).
//
//   merge_partition_kernel  one thread per tile boundary: merge-path split of the
//                           diagonal d = t * kMgTile (binary search over A, B)
//   merge_add_kernel        one pass per 2048-position tile: A and B slices staged in
//                           shared memory, per-thread diagonal search + serial merge
//                           of 8 positions, duplicate combine (a key in both inputs
//                           sits on two adjacent positions, A first: the A copy keeps
//                           the sum, also across a tile boundary), tile offsets by
//                           decoupled lookback, compacted output staged in shared
//                           memory and written coalesced.
// Traffic: 16 B read + 16 B written per merged position (keys u64 + counts u64);
// a summed count beyond 2^63 - 1 (the reference's int64 values) is reported.
#pragma once
#include "nmx_msd.cuh"

namespace nmx {

constexpr int kMgThreads = 256;
#ifndef NMX_MG_IPT
#define NMX_MG_IPT 8
#endif
constexpr int kMgIPT = NMX_MG_IPT;  // positions per thread (A/B builds: -DNMX_MG_IPT=...)
constexpr int kMgTile = kMgThreads * kMgIPT;

// first i in [max(0, d - nb), min(d, na)] with a[i] > b[d - 1 - i] (ties: A first)
__device__ __forceinline__ uint64_t merge_split(const uint64_t* a, uint64_t na, const uint64_t* b, uint64_t nb,
                                                uint64_t d) {
  uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t i = (lo + hi) >> 1;
    if (a[i] <= b[d - 1 - i])
      lo = i + 1;
    else
      hi = i;
  }
  return lo;
}

__global__ void merge_partition_kernel(const uint64_t* __restrict__ ak, uint64_t na, const uint64_t* __restrict__ bk,
                                       uint64_t nb, uint64_t ntiles, uint64_t* __restrict__ split) {
  const uint64_t n = na + nb;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = t * kMgTile < n ? t * kMgTile : n;
    split[t] = merge_split(ak, na, bk, nb, d);
  }
}

// Shared-memory slices are padded (pad16): the per-thread serial merges read at a
// stride of ~4 items and the compacted writes at ~8, which would otherwise put a
// warp on a few banks.
constexpr int kMgPad = kMgTile + kMgTile / 16;
struct MergeSmem {
  uint64_t key[kMgPad];  // A slice [0, la), B slice [la, la + lb); later the compacted output
  uint64_t cnt[kMgPad];
  uint64_t fkey[kMgThreads], fcnt[kMgThreads], lkey[kMgThreads];  // each thread's first / last merged item
  uint8_t ffromb[kMgThreads];
  uint32_t wt[kWarps + 1];
  unsigned long long prefix;
  uint32_t tile;
  uint64_t prev_key, next_key;
  uint64_t next_cnt;
  int prev_valid, next_is_b, next_valid;
};

__global__ void __launch_bounds__(kMgThreads) merge_add_kernel(
    const uint64_t* __restrict__ ak, const uint64_t* __restrict__ ac, uint64_t na, const uint64_t* __restrict__ bk,
    const uint64_t* __restrict__ bc, uint64_t nb, const uint64_t* __restrict__ split, uint64_t* __restrict__ status,
    uint32_t epoch, uint32_t* __restrict__ tile_counter, uint64_t* __restrict__ ck, uint64_t* __restrict__ cc,
    unsigned long long* __restrict__ overflow, unsigned long long* __restrict__ total) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MergeSmem& S = *reinterpret_cast<MergeSmem*>(smem_raw);
  const int tid = threadIdx.x;
  if (tid == 0) S.tile = atomicAdd(tile_counter, 1u);  // dispatch order = lookback order
  __syncthreads();
  const uint32_t t = S.tile;
  const uint64_t n = na + nb;
  const uint64_t d0 = (uint64_t)t * kMgTile, d1 = d0 + kMgTile < n ? d0 + kMgTile : n;
  const uint64_t ia = split[t], ja = split[t + 1];
  const uint64_t ib = d0 - ia, jb = d1 - ja;
  const uint32_t la = (uint32_t)(ja - ia), lb = (uint32_t)(jb - ib), len = la + lb;
  for (uint32_t i = tid; i < la; i += kMgThreads) {
    S.key[pad16(i)] = ak[ia + i];
    S.cnt[pad16(i)] = ac[ia + i];
  }
  for (uint32_t i = tid; i < lb; i += kMgThreads) {
    S.key[pad16(la + i)] = bk[ib + i];
    S.cnt[pad16(la + i)] = bc[ib + i];
  }
  if (tid == 0) {
    // merged position d0 - 1 (its key decides whether our first B element is a duplicate)
    S.prev_valid = d0 > 0;
    if (d0 > 0) S.prev_key = (ia > 0 && (ib == 0 || ak[ia - 1] >= bk[ib - 1])) ? ak[ia - 1] : bk[ib - 1];
    // merged position d1 (a B duplicate of our last A element adds its count here)
    S.next_valid = d1 < n;
    S.next_is_b = 0;
    S.next_key = 0;
    S.next_cnt = 0;
    if (d1 < n) {
      if (ja < na && (jb >= nb || ak[ja] <= bk[jb])) {
        S.next_key = ak[ja];
      } else {
        S.next_key = bk[jb];
        S.next_cnt = bc[jb];
        S.next_is_b = 1;
      }
    }
  }
  __syncthreads();
  // per-thread merge of positions [q0, q1) of this tile, kept in registers
  const uint32_t q0 = min((uint32_t)tid * kMgIPT, len), q1 = min(q0 + kMgIPT, len), nq = q1 - q0;
  uint64_t k[kMgIPT], c[kMgIPT];
  uint32_t fromb = 0;  // bit q: position q0 + q comes from B
  {
    uint32_t lo = q0 > lb ? q0 - lb : 0, hi = min(q0, la);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (S.key[pad16(mid)] <= S.key[pad16(la + q0 - 1 - mid)])
        lo = mid + 1;
      else
        hi = mid;
    }
    uint32_t i = lo, j = q0 - lo;
    uint64_t ka = i < la ? S.key[pad16(i)] : ~0ull, kb = j < lb ? S.key[pad16(la + j)] : ~0ull;
#pragma unroll
    for (int q = 0; q < kMgIPT; ++q) {
      k[q] = 0;
      c[q] = 0;
      if ((uint32_t)q < nq) {
        const bool takeA = i < la && (j >= lb || ka <= kb);
        if (takeA) {
          k[q] = ka;
          c[q] = S.cnt[pad16(i)];
          ++i;
          ka = i < la ? S.key[pad16(i)] : ~0ull;
        } else {
          k[q] = kb;
          c[q] = S.cnt[pad16(la + j)];
          fromb |= 1u << q;
          ++j;
          kb = j < lb ? S.key[pad16(la + j)] : ~0ull;
        }
      }
    }
  }
  if (nq) {
    S.fkey[tid] = k[0];
    S.fcnt[tid] = c[0];
    S.ffromb[tid] = fromb & 1u;
    S.lkey[tid] = k[nq - 1];
  }
  __syncthreads();  // every merge has read the slices: they may be overwritten below
  // neighbours: the merged position before q0 and the one at q1
  const bool pv = tid ? true : S.prev_valid != 0;
  const uint64_t pk = tid ? S.lkey[tid - 1] : S.prev_key;
  const bool inner = q1 < len;
  const bool nv = inner || S.next_valid;
  const uint64_t nk = inner ? S.fkey[tid + 1] : S.next_key;
  const uint64_t nc = inner ? S.fcnt[tid + 1] : S.next_cnt;
  const bool nbf = inner ? S.ffromb[tid + 1] != 0 : S.next_is_b != 0;
  // a B element is dropped iff its merged predecessor has the same key (inputs are
  // unique, so duplicates are exactly adjacent A, B pairs); the A copy takes the sum
  uint32_t keep = 0, kept = 0;
#pragma unroll
  for (int q = 0; q < kMgIPT; ++q) {
    if ((uint32_t)q >= nq) continue;
    const bool isb = (fromb >> q) & 1u;
    const bool dup = isb && (q ? k[q - 1] == k[q] : (pv && pk == k[q]));
    if (dup) continue;
    const bool last = (uint32_t)q + 1 == nq;
    const bool nxb = last ? (nv && nbf && nk == k[q]) : (((fromb >> (q + 1)) & 1u) && k[q + 1] == k[q]);
    if (nxb) {
      c[q] += last ? nc : c[q + 1];
      if (c[q] > 0x7FFFFFFFFFFFFFFFull) atomicAdd(overflow, 1ull);  // both inputs < 2^63: no u64 wrap
    }
    keep |= 1u << q;
    ++kept;
  }
  uint32_t tot;
  uint32_t at = block_excl_scan<uint32_t>(kept, S.wt, &tot);
  if (tid < 32) {  // warp 0: publish, then a 32-wide lookback
    uint64_t* my = status + t;
    unsigned long long excl = 0;
    if (t == 0) {
      if (tid == 0) st_relaxed(my, st_pack(epoch, kFlagInc, tot));
    } else {
      if (tid == 0) st_relaxed(my, st_pack(epoch, kFlagAgg, tot));
      excl = lookback_exclusive_warp(status, t, 1, 0, epoch);
      if (tid == 0) st_relaxed(my, st_pack(epoch, kFlagInc, excl + tot));
    }
    if (tid == 0) {
      S.prefix = excl;
      if (d1 == n) *total = excl + tot;
    }
  }
  // compacted output staged in the (now free) slices, then written coalesced
#pragma unroll
  for (int q = 0; q < kMgIPT; ++q)
    if ((keep >> q) & 1u) {
      S.key[pad16(at)] = k[q];
      S.cnt[pad16(at)] = c[q];
      ++at;
    }
  __syncthreads();
  const unsigned long long base = S.prefix;
  for (uint32_t j = tid; j < tot; j += kMgThreads) {
    ck[base + j] = S.key[pad16(j)];
    cc[base + j] = S.cnt[pad16(j)];
  }
}

}  // namespace nmx
