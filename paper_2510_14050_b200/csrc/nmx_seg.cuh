// nmx_seg.cuh -- segmented MSD levels for the heavy buckets of the MSD path.
//
// The dense MSD levels (nmx_msd.cuh) split the keys by their top D bits into
// 2^D buckets; a bucket larger than a shared-memory group ("heavy": a power-law
// source with many packets, or a destination with a large fan-in) used to be
// finished by a full LSD sort. Here heavy buckets keep being partitioned by the
// next <= 7 key bits, one level at a time, with the parent of an item given by
// its POSITION (parents are contiguous ranges, offsets `poff`), not by a key
// prefix, so the bucket count never grows past (#heavy parents) x 128:
//
//   seg_count    per tile: child counts (parent-relative bins in shared memory)
//   seg_scan_*   classify every child: light (<= cap, goes to a shared-memory
//                group of this level) or big (next level); exclusive offsets of
//                both classes, compact list of the big children = next parents
//   seg_scatter  items -> light array (grouped by the local kernels) or big array
//   final level  count-only: every child is one key (rows: one link, emitted by
//                seg_emit_rows) or one destination (columns: fan-in + packet sum,
//                seg_emit_cols); nothing is moved
//
// Row keys are split on the remaining source bits first (children stay whole
// sources) and then on destination bits, where every parent is a single heavy
// source whose packets / fan-out are accumulated across groups in a SrcTable.
#pragma once
#include "nmx_msd.cuh"

namespace nmx {

constexpr int kSegMaxRel = 4;                              // parents per tile kept in shared memory
// digit bits per segmented level (at most). 8-bit levels (one level fewer over 32
// destination bits) measured no faster on cfg4: the 1024-bin tile scans and
// resets cost what the saved level moved (r02n, 59.0 vs 59.1 ms)
constexpr int kSegLevelBits = 7;
constexpr int kSegBins = kSegMaxRel << kSegLevelBits;     // 512 tile bins
constexpr int kSegCap = 1024;                              // light child: <= kSegCap items
constexpr int kSegScanItems = 4096;                        // children per scan block

// last parent p with poff[p] <= i (poff[0] = 0, non-decreasing; empty parents allowed)
__device__ __forceinline__ uint32_t seg_parent(const uint32_t* __restrict__ poff, uint32_t P, uint32_t i) {
  uint32_t a = 0, z = P - 1;
  while (a < z) {
    const uint32_t mid = (a + z + 1) >> 1;
    if (poff[mid] <= i)
      a = mid;
    else
      z = mid - 1;
  }
  return a;
}

template <typename KeyT>
__device__ __forceinline__ uint32_t seg_digit(KeyT key, int shift, uint32_t dmask) {
  return dmask ? (uint32_t)((uint64_t)key >> shift) & dmask : 0u;
}

// Child counts (FINAL: + per-child packet sums for (dst, count) items, or one
// representative key per child for row keys -- all keys of a final child are equal).
// PACKED: u64 column items (dst << 32 | count), summed like a value
template <typename KeyT, bool HAS_VAL, bool FINAL, bool PACKED = false>
__global__ void __launch_bounds__(kMsdThreads) seg_count_kernel(const KeyT* __restrict__ keys,
                                                               const uint32_t* __restrict__ vals, uint32_t m,
                                                               const uint32_t* __restrict__ poff, uint32_t P,
                                                               int shift, int dbits, uint32_t* __restrict__ ccnt,
                                                               unsigned long long* __restrict__ csum,
                                                               KeyT* __restrict__ rep) {
  constexpr bool SUM = FINAL && (HAS_VAL || PACKED);
  constexpr bool REP = FINAL && !HAS_VAL && !PACKED;
  __shared__ uint32_t cnt[kSegBins];
  __shared__ uint32_t sum[SUM ? kSegBins : 1];  // < 2^32 packets per call: 32-bit shared atomics
  __shared__ KeyT srep[REP ? kSegBins : 1];
  __shared__ uint32_t s_p0, s_bound[kSegMaxRel];
  const int tid = threadIdx.x;
  const int nbins = kSegMaxRel << dbits;
  for (int i = tid; i < nbins; i += kMsdThreads) {
    cnt[i] = 0;
    if (SUM) sum[i] = 0;
  }
  const uint32_t base = blockIdx.x * kMsdTile;
  if (tid == 0) {
    const uint32_t p0 = seg_parent(poff, P, base);
    s_p0 = p0;
#pragma unroll
    for (int k = 0; k < kSegMaxRel; ++k) s_bound[k] = p0 + 1 + k < P ? poff[p0 + 1 + k] : m;
  }
  KeyT k[kMsdIPT];
  uint32_t v[kMsdIPT];
#pragma unroll
  for (int i = 0; i < kMsdIPT; ++i) {
    const uint32_t idx = base + i * kMsdThreads + tid;
    const uint32_t j = idx < m ? idx : 0;
    k[i] = keys[j];
    v[i] = HAS_VAL ? vals[j] : PACKED ? (uint32_t)(uint64_t)k[i] : 0u;
  }
  __syncthreads();
  const uint32_t p0 = s_p0;
  const uint32_t dmask = (1u << dbits) - 1;
  uint32_t bd[kSegMaxRel];
#pragma unroll
  for (int q = 0; q < kSegMaxRel; ++q) bd[q] = s_bound[q];
  const bool one = bd[0] >= base + (uint32_t)kMsdTile;  // the whole tile in parent p0
  int bin[kMsdIPT];
#pragma unroll
  for (int i = 0; i < kMsdIPT; ++i) {
    const uint32_t idx = base + i * kMsdThreads + tid;
    bin[i] = -1;
    if (idx < m) {
      const uint32_t d = seg_digit(k[i], shift, dmask);
      uint32_t rel = 0;
      if (!one) {
#pragma unroll
        for (int q = 0; q < kSegMaxRel; ++q) rel += idx >= bd[q];
      }
      if (rel < kSegMaxRel) {
        bin[i] = (int)((rel << dbits) | d);
        if (REP) srep[bin[i]] = k[i];
      } else {  // a fifth parent inside one tile (tiny parents): direct global update
        const uint32_t c = (seg_parent(poff, P, idx) << dbits) | d;
        atomicAdd(ccnt + c, 1u);
        if (SUM) atomicAdd(csum + c, (unsigned long long)v[i]);
        if (REP) rep[c] = k[i];
      }
    }
  }
  // warp aggregation only for skewed warps (one hot link / destination)
  if (warp_skewed(bin[0])) {
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i) {
      if (SUM)
        agg_count_sum(cnt, sum, bin[i], v[i]);
      else
        agg_count(cnt, bin[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i)
      if (bin[i] >= 0) {
        atomicAdd(&cnt[bin[i]], 1u);
        if (SUM) atomicAdd(&sum[bin[i]], v[i]);
      }
  }
  __syncthreads();
  for (int bin = tid; bin < nbins; bin += kMsdThreads) {
    const uint32_t cb = cnt[bin];
    if (!cb) continue;
    const uint32_t c = ((p0 + (uint32_t)(bin >> dbits)) << dbits) | ((uint32_t)bin & dmask);
    atomicAdd(ccnt + c, cb);
    if (SUM) atomicAdd(csum + c, (unsigned long long)sum[bin]);
    if (REP) rep[c] = srep[bin];
  }
}

// ---- classification + exclusive offsets of the children ----------------------
// per child: light = size if size <= cap; big = size otherwise; packed
// (big << 32 | light) (each class total < 2^31, no carry), plus a big-child flag.
__device__ __forceinline__ void seg_class(uint32_t s, uint64_t& lb, uint32_t& f) {
  const bool big = s > (uint32_t)kSegCap;
  lb = big ? ((uint64_t)s << 32) : (uint64_t)s;
  f = big ? 1u : 0u;
}

__global__ void __launch_bounds__(256) seg_scan_sums_kernel(const uint32_t* __restrict__ ccnt, uint32_t C,
                                                           unsigned long long* __restrict__ bsum,
                                                           uint32_t* __restrict__ bflag) {
  __shared__ unsigned long long wt64[kWarps + 1];
  __shared__ uint32_t wt32[kWarps + 1];
  const uint32_t base = blockIdx.x * kSegScanItems;
  unsigned long long s = 0;
  uint32_t f = 0;
#pragma unroll 4
  for (int q = 0; q < kSegScanItems / 256; ++q) {
    const uint32_t i = base + q * 256 + threadIdx.x;
    if (i < C) {
      uint64_t lb;
      uint32_t ff;
      seg_class(ccnt[i], lb, ff);
      s += lb;
      f += ff;
    }
  }
  unsigned long long t64;
  uint32_t t32;
  block_excl_scan<unsigned long long>(s, wt64, &t64);
  block_excl_scan<uint32_t>(f, wt32, &t32);
  if (threadIdx.x == 0) {
    bsum[blockIdx.x] = t64;
    bflag[blockIdx.x] = t32;
  }
}

// one CTA: exclusive scan of the block sums in place; totals[0..2] = light, big, #big
__global__ void __launch_bounds__(1024) seg_scan_top_kernel(unsigned long long* __restrict__ bsum,
                                                           uint32_t* __restrict__ bflag, uint32_t nb,
                                                           uint32_t* __restrict__ totals) {
  __shared__ unsigned long long w64[33];
  __shared__ uint32_t w32[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long c64 = 0;
  uint32_t c32 = 0;
  for (uint32_t base = 0; base < nb; base += 1024) {
    const uint32_t i = base + tid;
    const unsigned long long x = i < nb ? bsum[i] : 0ull;
    const uint32_t y = i < nb ? bflag[i] : 0u;
    const unsigned long long ix = warp_incl_scan(x, lane);
    const uint32_t iy = warp_incl_scan(y, lane);
    if (lane == 31) w64[warp] = ix, w32[warp] = iy;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long a = w64[lane];
      const uint32_t bq = w32[lane];
      const unsigned long long ai = warp_incl_scan(a, lane);
      const uint32_t bi = warp_incl_scan(bq, lane);
      w64[lane] = ai - a;
      w32[lane] = bi - bq;
      if (lane == 31) w64[32] = ai, w32[32] = bi;
    }
    __syncthreads();
    if (i < nb) {
      bsum[i] = c64 + w64[warp] + ix - x;
      bflag[i] = c32 + w32[warp] + iy - y;
    }
    c64 += w64[32];
    c32 += w32[32];
    __syncthreads();
  }
  if (tid == 0) {
    totals[0] = (uint32_t)(c64 & 0xFFFFFFFFull);
    totals[1] = (uint32_t)(c64 >> 32);
    totals[2] = c32;
  }
}

// cursor[c] = light ? kLightBit | light offset : big offset; loff[0..C] = light
// offsets (loff[C] = light total); npoff[rank of big child] = its big offset
__global__ void __launch_bounds__(256) seg_scan_apply_kernel(const uint32_t* __restrict__ ccnt, uint32_t C,
                                                            const unsigned long long* __restrict__ bsum,
                                                            const uint32_t* __restrict__ bflag,
                                                            const uint32_t* __restrict__ totals,
                                                            uint32_t* __restrict__ cursor, uint32_t* __restrict__ loff,
                                                            uint32_t* __restrict__ npoff) {
  __shared__ unsigned long long wt64[kWarps + 1];
  __shared__ uint32_t wt32[kWarps + 1];
  constexpr int PER = kSegScanItems / 256;  // 16 consecutive children per thread
  const uint32_t base = blockIdx.x * kSegScanItems + threadIdx.x * PER;
  uint32_t sz[PER];
  unsigned long long s = 0;
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    sz[q] = base + q < C ? ccnt[base + q] : 0u;
    uint64_t lb;
    uint32_t ff;
    seg_class(sz[q], lb, ff);
    s += lb;
    f += ff;
  }
  unsigned long long t64;
  uint32_t t32;
  unsigned long long run = bsum[blockIdx.x] + block_excl_scan<unsigned long long>(s, wt64, &t64);
  uint32_t rank = bflag[blockIdx.x] + block_excl_scan<uint32_t>(f, wt32, &t32);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t c = base + q;
    if (c >= C) break;
    const uint32_t lo = (uint32_t)(run & 0xFFFFFFFFull), hi = (uint32_t)(run >> 32);
    const bool big = sz[q] > (uint32_t)kSegCap;
    cursor[c] = big ? hi : (kLightBit | lo);
    loff[c] = lo;
    if (big) npoff[rank++] = hi;
    uint64_t lb;
    uint32_t ff;
    seg_class(sz[q], lb, ff);
    run += lb;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) loff[C] = totals[0];
}

// C <= kSegSmallC: the whole classification in one block (chunks of 4096 with
// carries) -- one launch instead of three for small calls; same outputs + totals
constexpr uint32_t kSegSmallC = 2 * kSegScanItems;
__global__ void __launch_bounds__(256) seg_classify_small_kernel(const uint32_t* __restrict__ ccnt, uint32_t C,
                                                                uint32_t* __restrict__ totals,
                                                                uint32_t* __restrict__ cursor,
                                                                uint32_t* __restrict__ loff,
                                                                uint32_t* __restrict__ npoff) {
  __shared__ unsigned long long wt64[kWarps + 1];
  __shared__ uint32_t wt32[kWarps + 1];
  constexpr int PER = kSegScanItems / 256;
  unsigned long long carry64 = 0;
  uint32_t carry32 = 0;
  for (uint32_t chunk = 0; chunk < C; chunk += kSegScanItems) {
    const uint32_t base = chunk + threadIdx.x * PER;
    uint32_t sz[PER];
    unsigned long long s = 0;
    uint32_t f = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      sz[q] = base + q < C ? ccnt[base + q] : 0u;
      uint64_t lb;
      uint32_t ff;
      seg_class(sz[q], lb, ff);
      s += lb;
      f += ff;
    }
    unsigned long long t64;
    uint32_t t32;
    unsigned long long run = carry64 + block_excl_scan<unsigned long long>(s, wt64, &t64);
    uint32_t rank = carry32 + block_excl_scan<uint32_t>(f, wt32, &t32);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const uint32_t c = base + q;
      if (c >= C) break;
      const uint32_t lo = (uint32_t)(run & 0xFFFFFFFFull), hi = (uint32_t)(run >> 32);
      const bool big = sz[q] > (uint32_t)kSegCap;
      cursor[c] = big ? hi : (kLightBit | lo);
      loff[c] = lo;
      if (big) npoff[rank++] = hi;
      uint64_t lb;
      uint32_t ff;
      seg_class(sz[q], lb, ff);
      run += lb;
    }
    carry64 += t64;
    carry32 += t32;
  }
  if (threadIdx.x == 0) {
    totals[0] = (uint32_t)(carry64 & 0xFFFFFFFFull);
    totals[1] = (uint32_t)(carry64 >> 32);
    totals[2] = carry32;
    loff[C] = (uint32_t)(carry64 & 0xFFFFFFFFull);
  }
}

// group bounds and plans in one pass: group g = the buckets whose start lies in
// [g*S, (g+1)*S) (two binary searches per group); lightp: group count from the
// device-side light total, stored to *ngout
__global__ void group_plan_kernel(const uint32_t* __restrict__ off, uint32_t nb, uint32_t S, uint32_t ngroups,
                                  uint4* __restrict__ plan, const uint32_t* __restrict__ lightp,
                                  uint32_t* __restrict__ ngout) {
  if (lightp) {
    ngroups = (*lightp + S - 1) / S;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ngout = ngroups;
  }
  auto first_at = [&](uint64_t target) {
    uint32_t a = 0, z = nb;
    while (a < z) {
      const uint32_t mid = (a + z) >> 1;
      if (off[mid] < target)
        a = mid + 1;
      else
        z = mid;
    }
    return a;
  };
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
    const uint32_t b0 = first_at((uint64_t)g * S);
    const uint32_t b1 = g + 1 == ngroups ? nb : first_at((uint64_t)(g + 1) * S);
    plan[g] = make_uint4(off[b0], off[b1], b0, b1);
  }
}

// ---- scatter -----------------------------------------------------------------
template <typename KeyT, bool HAS_VAL>
struct SegSmem {
  KeyT stage[kMsdTile];
  uint32_t vstage[HAS_VAL ? kMsdTile : 1];
  uint32_t cnt[kSegBins];
  uint32_t tstart[kSegBins];
  uint32_t gbase[kSegBins];
  uint32_t wt[kMsdThreads / 32 + 1];
  uint32_t p0, bound[kSegMaxRel];
};

// Non-stable partition of each parent by `dbits` key bits at `shift`; light
// children land in (lout, lvout), big children in (bout, bvout). Ranking, the
// per-tile reservation atomics and the shared-memory staging follow
// msd_scatter_kernel. Parents are positional, so a staged item's parent is
// recovered from its staged position: the tile stages parent-major (bin = rel << dbits
// | digit), parent q's items start at tstart[q << dbits].
template <typename KeyT, bool HAS_VAL>
__global__ void __launch_bounds__(kMsdThreads, 5) seg_scatter_kernel(const KeyT* __restrict__ keys,
                                                                 const uint32_t* __restrict__ vals, uint32_t m,
                                                                 const uint32_t* __restrict__ poff, uint32_t P,
                                                                 int shift, int dbits, uint32_t* __restrict__ cursor,
                                                                 KeyT* __restrict__ lout, uint32_t* __restrict__ lvout,
                                                                 KeyT* __restrict__ bout, uint32_t* __restrict__ bvout) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<SegSmem<KeyT, HAS_VAL>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbins = kSegMaxRel << dbits;
  for (int i = tid; i < kSegBins; i += kMsdThreads) S.cnt[i] = 0;
  const uint32_t base = blockIdx.x * kMsdTile;
  if (tid == 0) {
    const uint32_t p0 = seg_parent(poff, P, base);
    S.p0 = p0;
#pragma unroll
    for (int k = 0; k < kSegMaxRel; ++k) S.bound[k] = p0 + 1 + k < P ? poff[p0 + 1 + k] : m;
  }
  KeyT k[kMsdIPT];
  uint32_t v[kMsdIPT];
  uint32_t idxs[kMsdIPT];
#pragma unroll
  for (int i = 0; i < kMsdIPT; ++i) {
    const uint32_t idx = base + (uint32_t)warp * 32 * kMsdIPT + (uint32_t)i * 32 + lane;
    idxs[i] = idx;
    const uint32_t j = idx < m ? idx : 0;
    k[i] = keys[j];
    v[i] = HAS_VAL ? vals[j] : 0u;
  }
  __syncthreads();
  const uint32_t p0 = S.p0;
  const uint32_t dmask = (1u << dbits) - 1;
  uint32_t bd[kSegMaxRel];
#pragma unroll
  for (int q = 0; q < kSegMaxRel; ++q) bd[q] = S.bound[q];
  int bin[kMsdIPT];
  uint32_t rank[kMsdIPT];
  // heavy parents usually cover whole tiles: then every key's parent is p0
  const bool one = bd[0] >= base + (uint32_t)kMsdTile;
#pragma unroll
  for (int i = 0; i < kMsdIPT; ++i) {
    bin[i] = -1;
    if (idxs[i] >= m) continue;
    const uint32_t d = seg_digit(k[i], shift, dmask);
    uint32_t rel = 0;
    if (!one) {
#pragma unroll
      for (int q = 0; q < kSegMaxRel; ++q) rel += idxs[i] >= bd[q];
    }
    if (rel < kSegMaxRel) {
      bin[i] = (int)((rel << dbits) | d);
    } else {
      const uint32_t c = (seg_parent(poff, P, idxs[i]) << dbits) | d;
      const uint32_t r = atomicAdd(cursor + c, 1u);
      const uint32_t pos = r & ~kLightBit;
      if (r & kLightBit) {
        lout[pos] = k[i];
        if (HAS_VAL) lvout[pos] = v[i];
      } else {
        bout[pos] = k[i];
        if (HAS_VAL) bvout[pos] = v[i];
      }
    }
  }
  if (warp_skewed(bin[0])) {
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i) rank[i] = agg_rank(S.cnt, bin[i]);
  } else {
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i)
      if (bin[i] >= 0) rank[i] = atomicAdd(&S.cnt[bin[i]], 1u);
  }
  __syncthreads();
  uint32_t resv[kSegBins / kMsdThreads];
#pragma unroll
  for (int q = 0; q < kSegBins / kMsdThreads; ++q) {
    const int i = tid + q * kMsdThreads;
    resv[q] = 0;
    if (i < nbins) {
      const uint32_t c = S.cnt[i];
      if (c) resv[q] = atomicAdd(cursor + (((p0 + (uint32_t)(i >> dbits)) << dbits) | ((uint32_t)i & dmask)), c);
    }
  }
  smem_excl_scan<kSegBins>(S.cnt, S.tstart, S.wt);
#pragma unroll
  for (int i = 0; i < kMsdIPT; ++i)
    if (bin[i] >= 0) {
      const uint32_t at = S.tstart[bin[i]] + rank[i];
      S.stage[at] = k[i];
      if (HAS_VAL) S.vstage[at] = v[i];
    }
#pragma unroll
  for (int q = 0; q < kSegBins / kMsdThreads; ++q) {
    const int i = tid + q * kMsdThreads;
    // light bit kept in bit 31; the position part wraps modulo 2^31 and is exact
    // once the staged index (>= tstart) is added back
    if (i < nbins && S.cnt[i]) S.gbase[i] = (resv[q] & kLightBit) | ((resv[q] - S.tstart[i]) & ~kLightBit);
  }
  __syncthreads();
  const uint32_t total = S.tstart[nbins - 1] + S.cnt[nbins - 1];
  uint32_t pst[kSegMaxRel - 1];  // staged start of parents 1 .. kSegMaxRel - 1
#pragma unroll
  for (int q = 1; q < kSegMaxRel; ++q) pst[q - 1] = S.tstart[q << dbits];
  for (uint32_t j = tid; j < total; j += kMsdThreads) {
    const KeyT key = S.stage[j];
    uint32_t rel = 0;
#pragma unroll
    for (int q = 0; q < kSegMaxRel - 1; ++q) rel += j >= pst[q];
    const uint32_t g = S.gbase[(rel << dbits) | seg_digit(key, shift, dmask)];
    const uint32_t pos = (g + j) & ~kLightBit;
    if (g & kLightBit) {
      lout[pos] = key;
      if (HAS_VAL) lvout[pos] = S.vstage[j];
    } else {
      bout[pos] = key;
      if (HAS_VAL) bvout[pos] = S.vstage[j];
    }
  }
}

// Groups spanning more than K buckets are cut into pieces of <= K buckets, so the
// grouping kernels can index sources / destinations directly (a piece covers at
// most K << dsb addresses): pieces per group, then (after an exclusive scan) the
// piece plans. The group count is the device-side *ngp.
__global__ void group_split_count_kernel(const uint32_t* __restrict__ gb, const uint32_t* __restrict__ ngp,
                                         uint32_t ng_max, uint32_t K, uint32_t* __restrict__ cnt) {
  const uint32_t ng = *ngp;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng_max; g += gridDim.x * blockDim.x)
    cnt[g] = g < ng ? max(1u, (gb[g + 1] - gb[g] + K - 1) / K) : 0u;
}
__global__ void seg_plan_split_kernel(const uint32_t* __restrict__ loff, const uint32_t* __restrict__ gb,
                                      const uint32_t* __restrict__ ngp, const uint32_t* __restrict__ poff, uint32_t K,
                                      uint4* __restrict__ plan) {
  const uint32_t ng = *ngp;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const uint32_t b0 = gb[g], b1 = gb[g + 1];
    uint32_t at = poff[g];
    if (b0 == b1) {
      plan[at] = make_uint4(loff[b0], loff[b0], b0, b0);
      continue;
    }
    const uint32_t span = b1 - b0, np = (span + K - 1) / K;  // np even pieces of <= K buckets
    for (uint32_t j = 0; j < np; ++j) {
      const uint32_t x = b0 + (uint32_t)((uint64_t)span * j / np), y = b0 + (uint32_t)((uint64_t)span * (j + 1) / np);
      plan[at++] = make_uint4(loff[x], loff[y], x, y);
    }
  }
}

// ---- final level emitters ------------------------------------------------------
// Rows: every non-empty child is one link (key rep[c], count ccnt[c]) of a
// heavy source: link statistics, its (dst, count) column entry (appended at
// *hcount), the column partition's first-level histogram, and the source's
// partial (fan-out 1, packets) -- summed per thread over runs of one source and
// per warp before the global table.
__global__ void __launch_bounds__(256) seg_emit_rows_kernel(const uint32_t* __restrict__ ccnt,
                                                           const uint64_t* __restrict__ rep, uint32_t C, int b,
                                                           uint64_t* __restrict__ hcol,
                                                           unsigned long long* __restrict__ hcount, int cshift,
                                                           uint32_t* __restrict__ chist,
                                                           unsigned long long* __restrict__ ccount,
                                                           unsigned long long* __restrict__ stats, SrcTable gsrc) {
  __shared__ uint32_t h[1 << kMsdMaxLevelBits];
  __shared__ uint32_t wt[kWarps + 1];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < (1 << kMsdMaxLevelBits)) h[tid] = 0;
  __syncthreads();
  constexpr int PER = 16;
  const uint64_t dmask = (1ull << b) - 1;
  unsigned long long a_valid = 0, a_links = 0, a_mlink = 0;
  // uniform trip count per block (ballots and block scans below)
  for (uint32_t base0 = blockIdx.x * 256 * PER; base0 < C; base0 += gridDim.x * 256 * PER) {
    const uint32_t base = base0 + tid * PER;
    uint32_t nz = 0;
    for (int q = 0; q < PER; ++q)
      if (base + q < C && ccnt[base + q]) ++nz;
    uint32_t tot;
    uint32_t at = block_excl_scan<uint32_t>(nz, wt, &tot);
    if (tid == 0 && tot) s_base = atomicAdd(hcount, (unsigned long long)tot);
    __syncthreads();
    const unsigned long long obase = s_base;
    uint32_t run_src = 0;
    unsigned long long run_v = 0;
    bool have = false;
    for (int q = 0; q < PER; ++q) {
      if (base + q >= C) break;
      const uint32_t cnt = ccnt[base + q];
      if (!cnt) continue;
      const uint64_t key = rep[base + q];
      const uint32_t src = (uint32_t)(key >> b), dst = (uint32_t)(key & dmask);
      a_valid += cnt;
      a_links += 1;
      a_mlink = max(a_mlink, (unsigned long long)cnt);
      const unsigned long long pos = obase + at++;
      hcol[pos] = ((uint64_t)dst << 32) | cnt;  // packed column item
      atomicAdd(&h[dst >> cshift], 1u);
      if (have && src != run_src) {  // a source boundary inside this thread's children
        gsrc.add(run_src, run_v);
        run_v = 0;
      }
      run_src = src;
      have = true;
      run_v += (1ull << 32) | cnt;
    }
    // open runs: lanes sharing the first open lane's source add once
    const uint32_t hm = __ballot_sync(FULL, have);
    if (hm) {
      const int leader = __ffs(hm) - 1;
      const uint32_t ls = __shfl_sync(FULL, run_src, leader);
      const bool same = have && run_src == ls;
      unsigned long long x = same ? run_v : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
      if (lane == leader) gsrc.add(ls, x);
      if (have && !same) gsrc.add(run_src, run_v);
    }
    __syncthreads();  // s_base reuse
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a_valid += __shfl_xor_sync(FULL, a_valid, o);
    a_links += __shfl_xor_sync(FULL, a_links, o);
    a_mlink = max(a_mlink, __shfl_xor_sync(FULL, a_mlink, o));
  }
  if (lane == 0 && a_links) {
    atomicAdd(ccount, a_links);
    atomicAdd(stats + S_VALID, a_valid);
    atomicAdd(stats + S_LINKS, a_links);
    atomicMax(stats + S_MAXLINK, a_mlink);
  }
  __syncthreads();
  if (tid < (1 << kMsdMaxLevelBits) && h[tid]) atomicAdd(chist + tid, h[tid]);
}

// Columns: every non-empty child is one destination: fan-in = entries, packets = sum
__global__ void __launch_bounds__(256) seg_emit_cols_kernel(const uint32_t* __restrict__ ccnt,
                                                           const unsigned long long* __restrict__ csum, uint32_t C,
                                                           unsigned long long* __restrict__ stats) {
  unsigned long long a_cnt = 0, a_fanin = 0, a_pk = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const uint32_t n = ccnt[c];
    if (!n) continue;
    a_cnt += 1;
    a_fanin = max(a_fanin, (unsigned long long)n);
    a_pk = max(a_pk, csum[c]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a_cnt += __shfl_xor_sync(FULL, a_cnt, o);
    a_fanin = max(a_fanin, __shfl_xor_sync(FULL, a_fanin, o));
    a_pk = max(a_pk, __shfl_xor_sync(FULL, a_pk, o));
  }
  if ((threadIdx.x & 31) == 0 && a_cnt) {
    atomicAdd(stats + S_DSTS, a_cnt);
    atomicMax(stats + S_MAXFANIN, a_fanin);
    atomicMax(stats + S_MAXDSTPK, a_pk);
  }
}

// heavy sources: one entry per source of the SrcTable
__global__ void __launch_bounds__(256) src_table_stats_kernel(SrcTable t, unsigned long long* __restrict__ stats) {
  unsigned long long a_srcs = 0, a_msrc = 0, a_mfan = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= t.mask + 1; i += gridDim.x * blockDim.x) {
    if (!t.keys[i]) continue;
    const unsigned long long v = t.vals[i];
    a_srcs += 1;
    a_msrc = max(a_msrc, v & 0xFFFFFFFFull);
    a_mfan = max(a_mfan, v >> 32);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a_srcs += __shfl_xor_sync(FULL, a_srcs, o);
    a_msrc = max(a_msrc, __shfl_xor_sync(FULL, a_msrc, o));
    a_mfan = max(a_mfan, __shfl_xor_sync(FULL, a_mfan, o));
  }
  if ((threadIdx.x & 31) == 0 && a_srcs) {
    atomicAdd(stats + S_SRCS, a_srcs);
    atomicMax(stats + S_MAXSRCPK, a_msrc);
    atomicMax(stats + S_MAXFANOUT, a_mfan);
  }
}

}  // namespace nmx
