// nmx_msd.cuh -- MSD partition + shared-memory grouping path for the summed matrix.
//
// The LSD path sorts all 2b key bits (8 + 4 onesweep passes at b = 32). Grouping
// only needs equal keys together, so here:
//   L1  msd_scatter<level 1>  packets -> keys grouped by the top D1 key bits
//   L2  msd_count2 + scan, msd_scatter<level 2>  -> grouped by the top D = D1+D2 bits
//       (buckets of ~2^10 keys; the top D bits are source bits, so every source
//       lies in one bucket)
//   LOC local_rows_kernel  per group of whole buckets: hash the keys into shared
//       memory (links with counts, sources with packets and fan-out), emit the
//       (dst, count) column entries in place, accumulate link + row statistics
// Buckets larger than the shared-memory capacity ("heavy", power-law hitters)
// are gathered and finished by the LSD path (onesweep + link_row_kernel).
// Both scatter levels are non-stable: a tile ranks keys with shared atomics and
// reserves each digit's output range with one global atomicAdd per digit, so
// there is no lookback chain; order inside a bucket is irrelevant to the
// statistics.
#pragma once
#include <cstddef>
#include <type_traits>
#include "nmx_kernels.cuh"

namespace nmx {

constexpr int kMsdThreads = 256;
constexpr int kMsdIPT = 8;
constexpr int kMsdTile = kMsdThreads * kMsdIPT;  // 2048 keys per scatter tile
constexpr int kMsdMaxBins = 2048;                // histogram bins of the first level (<= 2^11)
constexpr int kMsdLevelBits = 7;                 // digit bits per segmented (heavy) level
constexpr int kMsdMaxLevelBits = 8;              // dense levels: <= 8 bits (3 levels up to D = 24)
constexpr int kMsdScBins = 2 << kMsdMaxLevelBits;  // scatter bins: a tile spans <= 2 parent buckets
constexpr int kCount2Tiles = 4;                  // tiles per CTA of the next-level counting pass

// block exclusive scan of NB counters held in smem (512 threads, NB % 512 == 0 or NB <= 512)
template <int NB>
__device__ __forceinline__ void smem_excl_scan(uint32_t* cnt, uint32_t* out, uint32_t* wt) {
  constexpr int PER = (NB + kMsdThreads - 1) / kMsdThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t loc[PER];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int i = tid * PER + q;
    loc[q] = i < NB ? cnt[i] : 0u;
    s += loc[q];
  }
  uint32_t inc = warp_incl_scan(s, lane);
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < kMsdThreads / 32 ? wt[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v, lane);
    if (lane < kMsdThreads / 32) wt[lane] = vi - v;
  }
  __syncthreads();
  uint32_t run = wt[warp] + inc - s;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int i = tid * PER + q;
    if (i < NB) out[i] = run;
    run += loc[q];
  }
  __syncthreads();
}

// 8 items per thread as two quads (quad indices q0 and q0 + qstride)
__device__ __forceinline__ void quad_items(const PacketSrc& s, uint64_t q, uint64_t* k, uint32_t* v, bool* ok) {
  s.load_quad(q, k, ok);
  v[0] = v[1] = v[2] = v[3] = 0;
}
__device__ __forceinline__ void quad_items(const PacketSrcWin& s, uint64_t q, uint64_t* k, uint32_t* v, bool* ok) {
  s.load_quad(q, k, ok);
  v[0] = v[1] = v[2] = v[3] = 0;
}
template <typename KeyT, bool HAS_VAL>
__device__ __forceinline__ void quad_items(const KeySrc<KeyT, HAS_VAL>& s, uint64_t q, KeyT* k, uint32_t* v,
                                           bool* ok) {
#pragma unroll
  for (int t = 0; t < 4; ++t) ok[t] = s.load(4 * q + t, k[t], v[t]);
}
struct ColConcatSrc;
__device__ __forceinline__ void quad_items(const ColConcatSrc& s, uint64_t q, uint64_t* k, uint32_t* v, bool* ok);
template <typename Src, typename KeyT, int NQ = 2>
__device__ __forceinline__ void load_items(const Src& s, uint64_t q0, uint64_t qstride, KeyT* k, uint32_t* v,
                                           bool* ok) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) quad_items(s, q0 + q * qstride, k + 4 * q, v + 4 * q, ok + 4 * q);
}

// Level 1 (cursor indexed by the D1-bit digit) and level 2 (cursor indexed by
// the D-bit bucket id; a tile lies in one or two level-1 buckets, keys of further
// buckets take a per-key global atomic). KeyT u64 = packed row keys; KeyT u32
// with a u32 payload = column entries (dst, count).
template <typename KeyT, bool HAS_VAL, int NB = (2 << kMsdLevelBits), int TILE = kMsdTile>
struct MsdSmem {
  KeyT stage[TILE];
  uint32_t vstage[HAS_VAL ? TILE : 1];
  uint32_t cnt[NB];
  uint32_t tstart[NB];
  uint32_t gbase[NB];
  uint32_t wt[kMsdThreads / 32 + 1];
  uint64_t b1first;
  uint64_t e1, e2;  // NM_POS: ends of the tile's first two parents
};

// Narrowed column items (NM_*): after the first column level a u64 item
// (dst << 32 | count) travels as u32 (dst & (2^delta - 1)) << cb | (count - 1),
// delta = b - d1 destination bits below the first digit, cb = 32 - delta; the
// dropped prefix is the item's level-1 bucket, known from its position.
//   NM_OUT  first level: u64 items in, narrowed u32 items out (nw.nout)
//   NM_POS  later levels over u32 items: parents by position (nw.poff, nw.npar);
//           SPLIT heavy items leave widened back to u64 (nw.wout), parent id
//           >> nw.dlp = the level-1 bucket
constexpr int NM_NONE = 0, NM_OUT = 1, NM_POS = 2;
struct NarrowArgs {
  uint32_t* nout = nullptr;
  uint64_t* wout = nullptr;
  const uint32_t* poff = nullptr;
  uint32_t npar = 0;
  int delta = 0, cb = 0, dlp = 0;
  const uint4* tpar = nullptr;  // NM_POS: per tile {first parent, its end, the next parent's end, -}
  const uint32_t* big = nullptr;  // SPLIT: items in heavy buckets (0: every tile takes the light-only loop)
};
__device__ __forceinline__ uint32_t narrow_item(uint64_t e, int delta, int cb) {
  return ((uint32_t)(e >> 32) & ((1u << delta) - 1u)) << cb | ((uint32_t)e - 1u);
}
__device__ __forceinline__ uint64_t widen_item(uint32_t u, uint32_t l1, int delta, int cb) {
  const uint32_t dst = l1 << delta | u >> cb;
  return (uint64_t)dst << 32 | ((u & ((1u << cb) - 1u)) + 1u);
}
// last parent p in [lo, npar) with poff[p] <= i (poff[npar] = total)
__device__ __forceinline__ uint32_t find_parent(const uint32_t* poff, uint32_t lo, uint32_t npar, uint64_t i) {
  uint32_t a = lo, z = npar - 1;
  while (a < z) {
    const uint32_t mid = (a + z + 1) >> 1;
    if ((uint64_t)poff[mid] <= i)
      a = mid;
    else
      z = mid - 1;
  }
  return a;
}
// NM_POS tile table: one thread per 2048-item tile (a per-tile binary search inside
// the scatter would put ~log2(npar) dependent loads in front of every tile)
__global__ void tile_parents_kernel(const uint32_t* __restrict__ poff, uint32_t npar,
                                    const unsigned long long* __restrict__ mp, uint64_t ntiles,
                                    uint4* __restrict__ tpar, uint32_t tile = kMsdTile) {
  const uint64_t m = *mp;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = t * tile;
    if (base >= m) break;
    const uint32_t p0 = find_parent(poff, 0, npar, base);
    tpar[t] = make_uint4(p0, p0 + 1 < npar ? poff[p0 + 1] : 0xFFFFFFFFu, p0 + 2 < npar ? poff[p0 + 2] : 0xFFFFFFFFu, 0);
  }
}

// SPLIT (last level): cursor values with kLightBit set address the light
// output (out, vout), the others the heavy output (hout, hvout) -- buckets too
// large for a shared-memory group leave the dense levels already compacted.
constexpr uint32_t kLightBit = 0x80000000u;
// LB: digit-bit capacity (7, or 8 for the levels that save a whole level)
template <typename Src, typename KeyT, bool HAS_VAL, int LEVEL, bool SPLIT = false, int LB = kMsdLevelBits,
          int NM = NM_NONE, int IPT = kMsdIPT, bool HI = false>
__global__ void __launch_bounds__(kMsdThreads, IPT == 8 ? 5 : 3) msd_scatter_kernel(Src src, uint64_t n_items, KeyT* __restrict__ out,
                                                                   uint32_t* __restrict__ vout, int shift, int dbits,
                                                                   int bshift, uint32_t* __restrict__ cursor,
                                                                   KeyT* __restrict__ hout = nullptr,
                                                                   uint32_t* __restrict__ hvout = nullptr,
                                                                   NarrowArgs nw = NarrowArgs{}) {
  static_assert(NM != NM_OUT || (LEVEL == 1 && sizeof(KeyT) == 8 && !HAS_VAL), "NM_OUT: first level of u64 items");
  static_assert(NM != NM_POS || (LEVEL == 2 && sizeof(KeyT) == 4 && !HAS_VAL), "NM_POS: later levels of u32 items");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NBINS = 2 << LB;
  constexpr int TILE = kMsdThreads * IPT;
  auto& S = *reinterpret_cast<MsdSmem<KeyT, HAS_VAL, NBINS, TILE>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbins = LEVEL == 1 ? (1 << dbits) : (2 << dbits);
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  if constexpr (LEVEL == 2) {
    if (base >= src.size()) return;  // grid sized by an upper bound (KeySrcD)
  }
  // SPLIT without heavy buckets (the classification ran before this launch): every
  // cursor carries the light bit and the output loop needs no per-item light / heavy
  // branch. Loaded first so that its latency hides behind the tile's loads.
  const bool light_only = SPLIT && nw.big && *nw.big == 0;
  for (int i = tid; i < NBINS; i += kMsdThreads) S.cnt[i] = 0;
  if (LEVEL == 2 && tid == 0) {
    if constexpr (NM == NM_POS) {  // positions < 2^31: 0xFFFFFFFF = no such parent
      const uint4 tp = nw.tpar[blockIdx.x];
      S.b1first = tp.x;
      S.e1 = tp.y;
      S.e2 = tp.z;
    } else {
      KeyT k0 = 0;
      uint32_t v;
      src.load(base, k0, v);
      S.b1first = (uint64_t)k0 >> bshift;
    }
  }
  // issue every load of the tile before using any (memory-level parallelism);
  // order inside a tile is irrelevant to a non-stable partition
  KeyT k[IPT];
  uint32_t v[IPT];
  bool ok[IPT];
  uint32_t kidx[NM == NM_POS ? IPT : 1];  // NM_POS: item positions (< 2^31: n < 2^31 per call)
  if constexpr (LEVEL == 1) {
    load_items<Src, KeyT, IPT / 4>(src, base / 4 + tid, kMsdThreads, k, v, ok);
  } else if constexpr (NM == NM_POS) {
    // 16-byte loads: lane takes items 4 lane .. 4 lane + 3 of each 128-item slice
    const uint64_t wbase = base + (uint64_t)warp * 32 * IPT;
    const uint64_t nn = src.size();
    if (wbase + 32 * IPT <= nn) {
      const uint4* p = reinterpret_cast<const uint4*>(src.keys + wbase);
#pragma unroll
      for (int i = 0; i < IPT / 4; ++i) {
        const uint4 x = p[i * 32 + lane];
        k[4 * i] = x.x, k[4 * i + 1] = x.y, k[4 * i + 2] = x.z, k[4 * i + 3] = x.w;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          ok[4 * i + t] = true;
          v[4 * i + t] = 0;
          kidx[4 * i + t] = (uint32_t)wbase + (uint32_t)(i * 128 + 4 * lane + t);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        kidx[i] = (uint32_t)wbase + (uint32_t)(i * 32 + lane);
        ok[i] = src.load(wbase + (uint64_t)i * 32 + lane, k[i], v[i]);
      }
    }
  } else {
    const uint64_t wbase = base + (uint64_t)warp * 32 * IPT;
    if constexpr (sizeof(KeyT) == 8 && !HAS_VAL && std::is_same<Src, KeySrcD<KeyT, HAS_VAL>>::value) {
      // 16-byte loads: lane takes keys 2 lane, 2 lane + 1 of each 64-key slice
      const uint64_t nn = src.size();
      if (wbase + 32 * IPT <= nn) {
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(src.keys + wbase);
#pragma unroll
        for (int i = 0; i < IPT / 2; ++i) {
          const ulonglong2 x = p[i * 32 + lane];
          k[2 * i] = (KeyT)x.x;
          k[2 * i + 1] = (KeyT)x.y;
          ok[2 * i] = ok[2 * i + 1] = true;
          v[2 * i] = v[2 * i + 1] = 0;
        }
      } else {
#pragma unroll
        for (int i = 0; i < IPT; ++i) ok[i] = src.load(wbase + (uint64_t)i * 32 + lane, k[i], v[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < IPT; ++i) ok[i] = src.load(wbase + (uint64_t)i * 32 + lane, k[i], v[i]);
    }
  }
  __syncthreads();
  const uint64_t b1first = S.b1first;
  // NM_POS parent ends in registers: the stores and global atomics below may alias
  // shared memory as far as the compiler knows, so S.e1 / S.e2 would be reloaded per key
  const uint32_t e1 = NM == NM_POS ? (uint32_t)S.e1 : 0u, e2 = NM == NM_POS ? (uint32_t)S.e2 : 0u;
  const uint32_t dmask = (1u << dbits) - 1;
  // HI: u64 keys whose digit and parent fields lie in the high word (shift, bshift >= 32:
  // row keys and column items at b = 32) -- 32-bit shifts instead of 64-bit ones
  const int hs = HI ? shift - 32 : shift, hb = HI ? bshift - 32 : bshift;
  auto digit = [&](KeyT key) -> uint32_t {
    if constexpr (HI)
      return ((uint32_t)((uint64_t)key >> 32) >> hs) & dmask;
    else
      return (uint32_t)((uint64_t)key >> shift) & dmask;
  };
  // parent relative to the tile's first (< 2 for the binned ones; (key >> bshift) has <= 24 bits)
  auto parent_rel = [&](KeyT key) -> uint32_t {
    if constexpr (HI)
      return ((uint32_t)((uint64_t)key >> 32) >> hb) - (uint32_t)b1first;
    else
      return (uint32_t)(((uint64_t)key >> bshift) - b1first);
  };
  uint32_t rank[IPT];
  int bin[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    bin[i] = -1;
    if (ok[i]) {
      const uint32_t d = digit(k[i]);
      if (LEVEL == 1) {
        bin[i] = (int)d;
      } else if constexpr (NM == NM_POS) {
        const uint32_t ix = kidx[i];
        if (ix < e2) {
          bin[i] = (int)(((ix < e1 ? 0u : 1u) << dbits) | d);
        } else {  // third+ parent inside one tile: direct placement
          const uint32_t par = find_parent(nw.poff, (uint32_t)b1first + 2, nw.npar, ix);
          const uint32_t r = atomicAdd(cursor + (par << dbits | d), 1u);
          if (!SPLIT || (r & kLightBit)) {
            out[SPLIT ? r & ~kLightBit : r] = k[i];
          } else {
            nw.wout[r] = widen_item((uint32_t)k[i], par >> nw.dlp, nw.delta, nw.cb);
          }
        }
      } else {
        const uint32_t rel = parent_rel(k[i]);
        if (rel < 2) {
          bin[i] = (int)((rel << dbits) | d);
        } else {  // third+ level-1 bucket inside one tile: direct placement
          const uint32_t r = atomicAdd(cursor + (uint32_t)((uint64_t)k[i] >> shift), 1u);
          if (!SPLIT || (r & kLightBit)) {
            const uint32_t pos = SPLIT ? r & ~kLightBit : r;
            out[pos] = k[i];
            if (HAS_VAL) vout[pos] = v[i];
          } else {
            hout[r] = k[i];
            if (HAS_VAL) hvout[r] = v[i];
          }
        }
      }
    }
  }
  if (warp_skewed(bin[0])) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) rank[i] = agg_rank(S.cnt, bin[i]);
  } else {
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if (bin[i] >= 0) rank[i] = atomicAdd(&S.cnt[bin[i]], 1u);
  }
  __syncthreads();
  // reserve each digit's output range first: the global atomics are in flight
  // while the block scan and the staging run
  uint32_t resv[NBINS / kMsdThreads];
#pragma unroll
  for (int q = 0; q < NBINS / kMsdThreads; ++q) {
    const int i = tid + q * kMsdThreads;
    resv[q] = 0;
    if (i < nbins) {
      const uint32_t c = S.cnt[i];
      if (c) {
        const uint32_t g = LEVEL == 1
                               ? (uint32_t)i
                               : (uint32_t)(((b1first + (uint64_t)(i >> dbits)) << dbits) | (uint64_t)(i & dmask));
        resv[q] = atomicAdd(cursor + g, c);
      }
    }
  }
  smem_excl_scan<NBINS>(S.cnt, S.tstart, S.wt);
#pragma unroll
  for (int i = 0; i < IPT; ++i)
    if (bin[i] >= 0) {
      const uint32_t at = S.tstart[bin[i]] + rank[i];
      S.stage[at] = k[i];
      if (HAS_VAL) S.vstage[at] = v[i];
    }
#pragma unroll
  for (int q = 0; q < NBINS / kMsdThreads; ++q) {
    const int i = tid + q * kMsdThreads;
    if (i < nbins && S.cnt[i])
      S.gbase[i] = SPLIT ? (resv[q] & kLightBit) | ((resv[q] - S.tstart[i]) & ~kLightBit) : resv[q] - S.tstart[i];
  }
  __syncthreads();
  const uint32_t total = S.tstart[nbins - 1] + S.cnt[nbins - 1];
  // NM_POS: staged items are parent-major, so the second parent's start the same
  const uint32_t rel1 = NM == NM_POS ? S.tstart[1 << dbits] : 0u;
  if (light_only) {
    for (uint32_t j = tid; j < total; j += kMsdThreads) {
      const KeyT key = S.stage[j];
      int b;
      if (LEVEL == 1) {
        b = (int)digit(key);
      } else if constexpr (NM == NM_POS) {
        b = (int)(((j >= rel1 ? 1u : 0u) << dbits) | ((uint32_t)key >> shift & dmask));
      } else {
        b = (int)((parent_rel(key) << dbits) | digit(key));
      }
      const uint32_t pos = (S.gbase[b] + j) & ~kLightBit;
      if constexpr (NM == NM_OUT)
        nw.nout[pos] = narrow_item((uint64_t)key, nw.delta, nw.cb);
      else
        out[pos] = key;
      if (HAS_VAL) vout[pos] = S.vstage[j];
    }
    return;
  }
  for (uint32_t j = tid; j < total; j += kMsdThreads) {
    const KeyT key = S.stage[j];
    int b;
    uint32_t rel = 0;
    if (LEVEL == 1) {
      b = (int)digit(key);
    } else if constexpr (NM == NM_POS) {
      rel = j >= rel1 ? 1u : 0u;
      b = (int)((rel << dbits) | ((uint32_t)key >> shift & dmask));
    } else {
      b = (int)((parent_rel(key) << dbits) | digit(key));
    }
    const uint32_t g = S.gbase[b];
    if (!SPLIT || (g & kLightBit)) {
      const uint32_t pos = SPLIT ? (g + j) & ~kLightBit : g + j;
      if constexpr (NM == NM_OUT)
        nw.nout[pos] = narrow_item((uint64_t)key, nw.delta, nw.cb);
      else
        out[pos] = key;
      if (HAS_VAL) vout[pos] = S.vstage[j];
    } else {
      const uint32_t pos = (g + j) & ~kLightBit;  // position arithmetic is modulo 2^31
      if constexpr (NM == NM_POS)
        nw.wout[pos] = widen_item((uint32_t)key, ((uint32_t)b1first + rel) >> nw.dlp, nw.delta, nw.cb);
      else
        hout[pos] = key;
      if (HAS_VAL) hvout[pos] = S.vstage[j];
    }
  }
}

// level-1 histogram: top D1 bits of the key (+ valid count)
template <typename Src, typename KeyT>
__global__ void __launch_bounds__(256) msd_hist1_kernel(Src src, uint64_t n, int shift, uint32_t* __restrict__ hist1,
                                                       unsigned long long* __restrict__ gcount) {
  __shared__ uint32_t h[kMsdMaxBins];
  for (int i = threadIdx.x; i < kMsdMaxBins; i += 256) h[i] = 0;
  __syncthreads();
  uint32_t c = 0;
  constexpr int U = 8;
  const uint64_t stride = (uint64_t)gridDim.x * 256 * U;
  for (uint64_t base = (uint64_t)blockIdx.x * 256 * U; base < n; base += stride) {
    KeyT k[U];
    uint32_t v[U];
    bool ok[U];
    // two quads per thread: packets base + 4*(u*256 + tid) .. +4
    load_items<Src, KeyT>(src, base / 4 + threadIdx.x, 256, k, v, ok);
    int bin[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c += ok[u];
      bin[u] = ok[u] ? (int)(((uint64_t)k[u] >> shift) & (uint64_t)(kMsdMaxBins - 1)) : -1;
    }
    if (warp_skewed(bin[0])) {  // only skewed warps pay for the per-round aggregation
#pragma unroll
      for (int u = 0; u < U; ++u) agg_count(h, bin[u]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (bin[u] >= 0) atomicAdd(&h[bin[u]], 1u);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(gcount, (unsigned long long)c);
  __syncthreads();
  for (int i = threadIdx.x; i < kMsdMaxBins; i += 256)
    if (h[i]) atomicAdd(hist1 + i, h[i]);
}

// Levels 1 and 2 counted in one pass over the source: the joint histogram of the
// top cum2 = d1 + d2 key bits (<= 2^14 bins, dynamic shared memory) goes to
// hist2 -- exactly what msd_count2_kernel would count over the level-1 output --
// and its d1-row sums to hist1. One streaming pass instead of two.
constexpr int kJointMaxBits = 14;
constexpr int kH12Threads = 512;  // 3 CTAs (64 KB each) per SM: 1536 threads of loads in flight
template <typename Src, typename KeyT>
__global__ void __launch_bounds__(kH12Threads) msd_hist12_kernel(Src src, uint64_t n, int jshift, int jbits, int d2bits,
                                                        uint32_t* __restrict__ hist1, uint32_t* __restrict__ hist2,
                                                        unsigned long long* __restrict__ gcount) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
  const int nbins = 1 << jbits;
  for (int i = threadIdx.x; i < nbins; i += kH12Threads) h[i] = 0;
  __syncthreads();
  uint32_t c = 0;
  constexpr int U = 8;
  const uint64_t stride = (uint64_t)gridDim.x * kH12Threads * U;
  for (uint64_t base = (uint64_t)blockIdx.x * kH12Threads * U; base < n; base += stride) {
    KeyT k[U];
    uint32_t v[U];
    bool ok[U];
    load_items<Src, KeyT>(src, base / 4 + threadIdx.x, kH12Threads, k, v, ok);
    int bin[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c += ok[u];
      // masked: keys of out-of-range addresses (rejected after the pass) stay in bounds
      bin[u] = ok[u] ? (int)(((uint64_t)k[u] >> jshift) & (uint64_t)(nbins - 1)) : -1;
    }
    if (warp_skewed(bin[0])) {
#pragma unroll
      for (int u = 0; u < U; ++u) agg_count(h, bin[u]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (bin[u] >= 0) atomicAdd(&h[bin[u]], 1u);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(gcount, (unsigned long long)c);
  __syncthreads();
  // d2bits >= 5: the 32 bins of a warp share one level-1 digit
  for (int i = threadIdx.x; i < nbins; i += kH12Threads) {
    const uint32_t x = h[i];
    if (x) atomicAdd(hist2 + i, x);
    uint32_t r = x;
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
    if ((threadIdx.x & 31) == 0 && r) atomicAdd(hist1 + (i >> d2bits), r);
  }
}

// level-2 digit counts per level-1 bucket over the level-1 output
template <typename KeyT>
__global__ void __launch_bounds__(kMsdThreads) msd_count2_kernel(const KeyT* __restrict__ keys,
                                                                  const unsigned long long* __restrict__ mp, int shift,
                                                                  int dbits, int bshift, uint32_t* __restrict__ hist2) {
  const uint64_t m = *mp;  // valid count from the level-1 histogram (grid sized by an upper bound)
  if ((uint64_t)blockIdx.x * kMsdTile * kCount2Tiles >= m) return;
  // kCount2Tiles consecutive tiles per CTA share one shared histogram, so the
  // global flush costs one atomic per bin per 8192 keys instead of per 2048
  __shared__ uint32_t cnt[kMsdScBins];
  __shared__ uint64_t s_b1first;
  const int tid = threadIdx.x;
  for (int i = tid; i < kMsdScBins; i += kMsdThreads) cnt[i] = 0;
  const uint64_t base0 = (uint64_t)blockIdx.x * kMsdTile * kCount2Tiles;
  if (tid == 0) s_b1first = (uint64_t)keys[base0] >> bshift;
  __syncthreads();
  const uint32_t dmask = (1u << dbits) - 1;
  const uint64_t b1first = s_b1first;
  for (int t = 0; t < kCount2Tiles; ++t) {
    const uint64_t base = base0 + (uint64_t)t * kMsdTile;
    if (base >= m) break;
    // 32-bit index math inside the tile; one 64-bit shift per key (bshift = shift + dbits)
    const uint32_t rem = m - base < (uint64_t)kMsdTile ? (uint32_t)(m - base) : (uint32_t)kMsdTile;
    const KeyT* kt = keys + base;
    KeyT k[kMsdIPT];
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i) {
      const uint32_t o = (uint32_t)i * kMsdThreads + tid;
      k[i] = o < rem ? kt[o] : KeyT(0);
    }
    int bin[kMsdIPT];
#pragma unroll
    for (int i = 0; i < kMsdIPT; ++i) {
      const uint32_t o = (uint32_t)i * kMsdThreads + tid;
      bin[i] = -1;
      if (o < rem) {
        const uint64_t x = (uint64_t)k[i] >> shift;  // level-1 bucket id | digit
        const uint64_t rel = (x >> dbits) - b1first;
        if (rel < 2)
          bin[i] = (int)(((uint32_t)rel << dbits) | ((uint32_t)x & dmask));
        else
          atomicAdd(hist2 + (uint32_t)x, 1u);
      }
    }
    if (warp_skewed(bin[0])) {
#pragma unroll
      for (int i = 0; i < kMsdIPT; ++i) agg_count(cnt, bin[i]);
    } else {
#pragma unroll
      for (int i = 0; i < kMsdIPT; ++i)
        if (bin[i] >= 0) atomicAdd(&cnt[bin[i]], 1u);
    }
  }
  __syncthreads();
  const int nbins = 2 << dbits;
  for (int i = tid; i < nbins; i += kMsdThreads) {
    const uint32_t c = cnt[i];
    if (c) atomicAdd(hist2 + (((b1first + (uint64_t)(i >> dbits)) << dbits) | (uint64_t)(i & dmask)), c);
  }
}

// Levels 2 and 3 counted in one pass over the level-1 output: each CTA takes a
// contiguous range of `per_cta` items, cut at the level-1 parent boundaries (poff),
// and histograms the next jbits = d2 + d3 key bits of each parent segment in shared
// memory (64 KB: three CTAs per SM); hist3[parent << jbits | bin] receives the
// counts. One read of the items instead of two msd_count2 passes.
constexpr int kJointCountThreads = 512;
template <typename KeyT>
__global__ void __launch_bounds__(kJointCountThreads) msd_count23_kernel(const KeyT* __restrict__ keys,
                                                                        const unsigned long long* __restrict__ mp,
                                                                        const uint32_t* __restrict__ poff, uint32_t P,
                                                                        uint64_t per_cta, int shift3, int jbits,
                                                                        uint32_t* __restrict__ hist3) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
  __shared__ uint32_t s_p;
  const uint64_t m = *mp;
  const uint64_t lo = (uint64_t)blockIdx.x * per_cta;
  if (lo >= m) return;
  const uint64_t hi = m - lo < per_cta ? m : lo + per_cta;
  const int nb = 1 << jbits;
  const int tid = threadIdx.x;
  if (tid == 0) {  // last parent starting at or before lo
    uint32_t a = 0, z = P - 1;
    while (a < z) {
      const uint32_t mid = (a + z + 1) >> 1;
      if (poff[mid] <= lo)
        a = mid;
      else
        z = mid - 1;
    }
    s_p = a;
  }
  __syncthreads();
  const uint32_t jmask = (uint32_t)nb - 1;
  constexpr int U = 8;
  uint32_t p = s_p;
  for (uint64_t a = lo; a < hi; ++p) {  // uniform: one parent segment per round
    const uint64_t pe = p + 1 < P && (uint64_t)poff[p + 1] < hi ? (uint64_t)poff[p + 1] : hi;
    if (pe <= a) continue;
    for (int i = tid; i < nb; i += kJointCountThreads) h[i] = 0;
    __syncthreads();
    for (uint64_t base = a; base < pe; base += (uint64_t)kJointCountThreads * U) {
      KeyT k[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const uint64_t i = base + (uint64_t)r * kJointCountThreads + tid;
        k[r] = i < pe ? keys[i] : KeyT(0);
      }
#pragma unroll
      for (int r = 0; r < U; ++r)
        if (base + (uint64_t)r * kJointCountThreads + tid < pe)
          atomicAdd(&h[(uint32_t)((uint64_t)k[r] >> shift3) & jmask], 1u);
    }
    __syncthreads();
    for (int i = tid; i < nb; i += kJointCountThreads)
      if (h[i]) atomicAdd(hist3 + (((uint64_t)p << jbits) | (uint32_t)i), h[i]);
    __syncthreads();
    a = pe;
  }
}
// level-2 counts as row sums of the level-3 counts (2^d3 children per level-2 bucket)
__global__ void hist_fold_kernel(const uint32_t* __restrict__ hist3, uint32_t nb2, int d3bits, uint32_t* __restrict__ hist2) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nb2; j += gridDim.x * blockDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(hist3 + ((size_t)j << d3bits));
    uint32_t sum = 0;
    for (int q = 0; q < (1 << d3bits) / 4; ++q) {
      const uint4 v = row[q];
      sum += v.x + v.y + v.z + v.w;
    }
    hist2[j] = sum;
  }
}

// multi-CTA exclusive scan of n u32 counters (4096 per block, coalesced):
// scan_block_sums -> scan_top (one CTA over the block sums) -> scan_apply
constexpr int kScanItems = 4096;
__global__ void __launch_bounds__(256) scan_block_sums_kernel(const uint32_t* __restrict__ cnt, uint32_t n,
                                                             uint32_t* __restrict__ bsum) {
  __shared__ uint32_t wt[kWarps + 1];
  const uint32_t base = blockIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems / 256; ++q) {
    const uint32_t i = base + q * 256 + threadIdx.x;
    s += i < n ? cnt[i] : 0u;
  }
  uint32_t tot;
  block_excl_scan<uint32_t>(s, wt, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* __restrict__ bsum, uint32_t nb,
                                                       uint32_t* __restrict__ total) {
  __shared__ uint32_t wt[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nb; base += 1024) {
    const uint32_t i = base + tid;
    const uint32_t x = i < nb ? bsum[i] : 0u;
    const uint32_t inc = warp_incl_scan(x, lane);
    if (lane == 31) wt[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = wt[lane];
      const uint32_t vi = warp_incl_scan(v, lane);
      wt[lane] = vi - v;
      if (lane == 31) wt[32] = vi;
    }
    __syncthreads();
    if (i < nb) bsum[i] = carry + wt[warp] + inc - x;
    carry += wt[32];
    __syncthreads();
  }
  if (tid == 0) *total = carry;
}
// n <= kScanItems: the whole exclusive scan in one block (one launch instead of three)
__global__ void __launch_bounds__(256) scan_small_kernel(const uint32_t* __restrict__ cnt, uint32_t n,
                                                        uint32_t* __restrict__ off, uint32_t* __restrict__ cursor) {
  __shared__ uint32_t wt[kWarps + 1];
  constexpr int PER = kScanItems / 256;
  const uint32_t base = threadIdx.x * PER;
  uint32_t v[PER];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    v[q] = base + q < n ? cnt[base + q] : 0u;
    s += v[q];
  }
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(s, wt, &tot);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (base + q < n) {
      off[base + q] = run;
      if (cursor) cursor[base + q] = run;
    }
    run += v[q];
  }
  if (threadIdx.x == 0) off[n] = tot;
}

__global__ void __launch_bounds__(256) scan_apply_kernel(const uint32_t* __restrict__ cnt, uint32_t n,
                                                        const uint32_t* __restrict__ bexcl,
                                                        const uint32_t* __restrict__ total, uint32_t* __restrict__ off,
                                                        uint32_t* __restrict__ cursor) {
  __shared__ uint32_t wt[kWarps + 1];
  constexpr int PER = kScanItems / 256;  // 16 consecutive counters per thread
  const uint32_t base = blockIdx.x * kScanItems + threadIdx.x * PER;
  uint32_t v[PER];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    v[q] = base + q < n ? cnt[base + q] : 0u;
    s += v[q];
  }
  uint32_t tot;
  uint32_t run = bexcl[blockIdx.x] + block_excl_scan<uint32_t>(s, wt, &tot);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (base + q < n) {
      off[base + q] = run;
      if (cursor) cursor[base + q] = run;
    }
    run += v[q];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) off[n] = *total;
}

// group g covers the buckets whose start lies in [g*S, (g+1)*S)
// lightp != nullptr: the light total is on the device (deferred partition
// read-back); ngroups = ceil(light / S) is derived here and stored to *ngout
__global__ void group_bounds_kernel(const uint32_t* __restrict__ off, uint32_t nb, uint32_t S, uint32_t ngroups,
                                    uint32_t* __restrict__ gb, const uint32_t* __restrict__ lightp = nullptr,
                                    uint32_t* __restrict__ ngout = nullptr) {
  if (lightp) {
    ngroups = (*lightp + S - 1) / S;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ngout = ngroups;
  }
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g <= ngroups; g += gridDim.x * blockDim.x) {
    const uint64_t target = (uint64_t)g * S;
    uint32_t a = 0, z = nb;  // first bucket with off >= target (nb if none)
    while (a < z) {
      const uint32_t mid = (a + z) >> 1;
      if (off[mid] < target)
        a = mid + 1;
      else
        z = mid;
    }
    gb[g] = g == ngroups ? nb : a;
  }
}

// ---------------------------------------------------------------------------
// LOC: per group of buckets, shared-memory hash grouping
// ---------------------------------------------------------------------------
constexpr int kLocThreads = 512;
constexpr int kLocChunk = 1536;    // row groups: the light buckets whose start lies in one chunk
constexpr int kLocMaxKeys = 2560;  // light keys per row group (chunk + one light bucket of <= 1024)
constexpr int kLocColChunk = 1024; // column groups (fewer registers per item: 4 per thread)
constexpr int kLocColMaxKeys = 2048;
constexpr int kLocT1 = 3840;       // link table slots (load <= 2/3)
constexpr int kLocT2 = 3840;       // source table slots

// group plans are plain key ranges {klo, khi, -, -} (heavy buckets leave the
// dense levels separately, nmx_seg.cuh)
__device__ __forceinline__ uint32_t light_index(const uint4& p, uint32_t j) { return p.x + j; }
__device__ __forceinline__ uint32_t light_count(const uint4& p) { return p.y - p.x; }

constexpr int kLocPerThread = kLocMaxKeys / kLocThreads;  // 5 keys in registers per thread
constexpr int kLocColThreads = 256;  // 8 entries per thread: the per-group work is shared by fewer threads
constexpr int kLocColPerThread = kLocColMaxKeys / kLocColThreads;  // 8
static_assert(kLocColMaxKeys <= 2048 && kLocColMaxKeys * 511 < (1 << 20),
              "local_cols packs fan-in (bits 20+) and small-count packets (bits 0-19) in one word");
static_assert(kLocColPerThread <= 8, "local_cols packs per-slot flags into 8-bit fields");
constexpr int kBmWords = 4096;                             // 65536 two-bit saturating counters

// exact-table home slot in [0, n): 32-bit mix, then a multiply-high range reduction
__device__ __forceinline__ uint32_t hslot(uint64_t x, uint32_t n) {
  return __umulhi((uint32_t)x * 0x9E3779B1u ^ (uint32_t)(x >> 32) * 0xC2B2AE35u, n);
}
// 16-bit counter index of a 64-bit key: two 32-bit multiplies (a counter
// collision only sends a key through the exact table)
__device__ __forceinline__ uint32_t h16(uint64_t x) {
  return ((uint32_t)x * 0x9E3779B1u + (uint32_t)(x >> 32) * 0x85EBCA6Bu) >> 16;
}
// 16-bit counter index of a 32-bit value (sources, destinations): one IMAD
__device__ __forceinline__ uint32_t h16u(uint32_t x) { return (x * 0x9E3779B1u) >> 16; }
// count one occurrence in a 2-bit saturating counter (01 = once, 11 = twice or more)
__device__ __forceinline__ void bm_hit(uint32_t* bm, uint32_t h) {
  const uint32_t bit = 1u << ((h & 15) * 2);
  if (atomicOr(bm + (h >> 4), bit) & bit) atomicOr(bm + (h >> 4), bit << 1);
}
__device__ __forceinline__ bool bm_once(const uint32_t* bm, uint32_t h) {
  return ((bm[h >> 4] >> ((h & 15) * 2)) & 3u) == 1u;
}

// Global per-source accumulator for sources split across groups: open
// addressing over src + 1 (0 = empty), value = fan-out << 32 | packets (both
// < 2^32 since n < 2^32); slot mask + 1 is reserved for src 0xFFFFFFFF.
struct SrcTable {
  uint32_t* keys = nullptr;
  unsigned long long* vals = nullptr;
  uint32_t mask = 0;
  __device__ __forceinline__ void add(uint32_t src, unsigned long long v) const {
    if (src == 0xFFFFFFFFu) {
      keys[mask + 1] = 1u;
      atomicAdd(vals + mask + 1, v);
      return;
    }
    const uint32_t k = src + 1;
    uint32_t h = (uint32_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 40) & mask;
    for (;;) {
      const uint32_t c0 = atomicCAS(keys + h, 0u, k);
      if (c0 == 0u || c0 == k) {
        atomicAdd(vals + h, v);
        return;
      }
      h = (h + 1) & mask;
    }
  }
};

// direct source slots (source - first source of the group), aliasing bms + t2key + t2pf
constexpr uint32_t kLocDirect = kBmWords + 2 * kLocT2;
constexpr int kNoDirect = 127;
struct LocSmem {
  uint32_t bml[kBmWords];            // link-key hash counters
  unsigned long long t1key[kLocT1];  // exact link table for colliding keys: key + 1 (0 = empty)
  uint32_t t1cnt[kLocT1];
  // hashed source path: counters + exact table; direct path: kLocDirect slots of
  // packets | fan-out << 16 (all zero between groups in both modes)
  uint32_t bms[kBmWords];  // source hash counters
  uint32_t t2key[kLocT2];  // exact source table: src + 1 (0 = empty)
  uint32_t t2pf[kLocT2];   // packets (low 16 bits) | fan-out (high 16 bits), both <= 2048
  uint32_t sp_link, sp_src_pk, sp_src_fo;  // the all-ones key / source (cannot be stored +1)
  uint32_t one_fo;                          // PARTIAL single-source groups: fresh links
  uint4 plan[2];                           // current / next group (by iteration parity)
  uint32_t chist[1 << kMsdMaxLevelBits];   // first-level histogram of the emitted column entries
};
static_assert(offsetof(LocSmem, t2key) == offsetof(LocSmem, bms) + 4 * kBmWords &&
                  offsetof(LocSmem, t2pf) == offsetof(LocSmem, t2key) + 4 * kLocT2,
              "direct source slots span bms, t2key, t2pf");

// Per group (<= 2048 light keys, 4 per thread, in registers):
//   1. every key counts its key-hash and source-hash in two 2-bit saturating
//      counter arrays (two shared atomics, no probing);
//   2. a key whose key-hash counter reads "once" is a unique link of count 1; a
//      key whose source-hash counter reads "once" is a source with one packet and
//      one link. Only the others go through exact hash tables (linear probing);
//   3. every key writes its own column slot: (dst, count) for the first copy of a
//      link, a hole (count 0) for later copies; table creators report and clear.
// Groups are statically round-robined over persistent CTAs; thread 0 fetches the
// next group's plan during the counting and every thread loads its next keys
// into registers while the current group's results are written.
//
// Direct sources (dense levels, dsb != kNoDirect): a group's buckets (plan .z/.w)
// cover a contiguous source range; when it spans <= kLocDirect sources, each key
// adds packets | fresh-link << 16 to slot src - lo with one shared atomic (the
// first adder reports) -- no source counters, probing or all-ones special case.
// dsb = b - D: bucket id -> first source (bucket << dsb, or >> -dsb).
//
// PARTIAL (heavy sources split over several groups by destination-bit levels,
// nmx_seg.cuh): links are still complete per group, but each source's packets
// and fan-out are partial; they are summed per warp (all lanes usually share
// one source), per group in the exact source table, and per source in the
// global table `gsrc` (one atomic per source and group).
// link / row totals of a warp's lanes -> one set of atomics (every lane calls it)
__device__ __forceinline__ void flush_rows(unsigned long long* __restrict__ st, unsigned long long* __restrict__ ccount,
                                           uint32_t a_valid, uint32_t a_links, uint32_t a_srcs, uint32_t a_mlink,
                                           uint32_t a_msrc, uint32_t a_mfan) {
  if (a_srcs) {  // every counted source has >= 1 packet and >= 1 link
    a_msrc = max(a_msrc, 1u);
    a_mfan = max(a_mfan, 1u);
  }
  unsigned long long w_valid = a_valid, w_links = a_links, w_srcs = a_srcs;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    w_valid += __shfl_xor_sync(FULL, w_valid, o);
    w_links += __shfl_xor_sync(FULL, w_links, o);
    w_srcs += __shfl_xor_sync(FULL, w_srcs, o);
    a_mlink = max(a_mlink, __shfl_xor_sync(FULL, a_mlink, o));
    a_msrc = max(a_msrc, __shfl_xor_sync(FULL, a_msrc, o));
    a_mfan = max(a_mfan, __shfl_xor_sync(FULL, a_mfan, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (w_links) atomicAdd(ccount, w_links);
    if (w_valid) atomicAdd(st + S_VALID, w_valid);
    if (w_links) atomicAdd(st + S_LINKS, w_links);
    if (w_srcs) atomicAdd(st + S_SRCS, w_srcs);
    if (a_mlink) atomicMax(st + S_MAXLINK, (unsigned long long)a_mlink);
    if (a_msrc) atomicMax(st + S_MAXSRCPK, (unsigned long long)a_msrc);
    if (a_mfan) atomicMax(st + S_MAXFANOUT, (unsigned long long)a_mfan);
  }
}

// Phase 2 of local_rows_kernel for one key: its link (counter "once" = unique, else
// the exact link table) and, unless PARTIAL, its source (DIRECT: one slot per source
// of the group's range; else counters + exact source table). Returns the st bits
// (bit0 fast link, bit1 fresh table link, bit2 fast source, bit3 source creator).
template <bool PARTIAL, bool DIRECT>
__device__ __forceinline__ uint32_t rows_classify(LocSmem& s, uint32_t* dir, uint64_t key, uint32_t kh, int b,
                                                  uint64_t slo, uint32_t& hl, uint32_t& hs) {
  uint32_t st = 0;
  const uint32_t src = (uint32_t)(key >> b);
  bool fresh;
  if (bm_once(s.bml, kh)) {  // unique link (the all-ones key included)
    fresh = true;
    st |= 1;
  } else if (key == ~0ull) {  // key + 1 would wrap: its own counter
    fresh = atomicAdd(&s.sp_link, 1u) == 0;
    if (fresh) st |= 2;
  } else {
    const unsigned long long kk = key + 1;
    uint32_t h = hslot(kk, kLocT1);
    for (;;) {
      unsigned long long c0 = s.t1key[h];
      if (c0 == 0) {
        c0 = atomicCAS(&s.t1key[h], 0ull, kk);
        if (c0 == 0) {
          atomicAdd(&s.t1cnt[h], 1u);
          fresh = true;
          st |= 2;
          break;
        }
      }
      if (c0 == kk) {
        atomicAdd(&s.t1cnt[h], 1u);
        fresh = false;
        break;
      }
      h = h + 1 == kLocT1 ? 0 : h + 1;
    }
    hl = h;
  }
  if (PARTIAL) return st;  // sources: warp-aggregated by the caller
  if (DIRECT) {
    const uint32_t o = (uint32_t)(src - slo);
    if (atomicAdd(&dir[o], 1u | (fresh ? 0x10000u : 0u)) == 0) st |= 8;
    hs = o;
  } else if (src == 0xFFFFFFFFu) {
    atomicAdd(&s.sp_src_pk, 1u);
    if (fresh) atomicAdd(&s.sp_src_fo, 1u);
  } else if (bm_once(s.bms, h16u(src))) {
    st |= 4;
  } else {
    const uint32_t sk = src + 1;
    uint32_t h = hslot(sk, kLocT2);
    for (;;) {
      uint32_t c0 = s.t2key[h];
      if (c0 == 0) {
        c0 = atomicCAS(&s.t2key[h], 0u, sk);
        if (c0 == 0) {
          st |= 8;
          c0 = sk;
        }
      }
      if (c0 == sk) {
        atomicAdd(&s.t2pf[h], 1u | (fresh ? 0x10000u : 0u));
        break;
      }
      h = h + 1 == kLocT2 ? 0 : h + 1;
    }
    hs = h;
  }
  return st;
}

// Phase 3 of local_rows_kernel for one key: its column slot (dst << 32 | count, 0 =
// hole), link totals, the source report of its creator, and the clears.
template <bool PARTIAL, bool WIN, bool DIRECT>
__device__ __forceinline__ void rows_result(LocSmem& s, uint32_t* dir, uint64_t key, uint32_t kh, uint32_t st,
                                            uint32_t hl, uint32_t hs, uint32_t pos, int b, uint64_t* __restrict__ col,
                                            int cshift, int gwin, unsigned long long* __restrict__ stats,
                                            unsigned long long* __restrict__ ccount, const SrcTable& gsrc,
                                            uint32_t& a_valid, uint32_t& a_links, uint32_t& a_srcs, uint32_t& a_mlink,
                                            uint32_t& a_msrc, uint32_t& a_mfan) {
  uint32_t c = 0;
  if (st & 1) {
    c = 1;
  } else if (st & 2) {
    if (key == ~0ull) {
      c = s.sp_link;
    } else {
      c = s.t1cnt[hl];
      s.t1key[hl] = 0;
      s.t1cnt[hl] = 0;
    }
  }
  uint64_t ck = key & ((1ull << b) - 1);
  if constexpr (WIN) ck |= (key >> (2 * b)) << b;  // dst' = window << b | dst
  col[pos] = (ck << 32) | c;  // packed column slot (dst << 32 | count; 0 = hole)
  unsigned long long* sw = WIN ? stats + (size_t)S_COUNT * (key >> (2 * b)) : stats;  // straddling groups
  if (c) {
    atomicAdd(&s.chist[(uint32_t)ck >> cshift], 1u);  // the column partition's first level
    if (WIN && gwin < 0) {
      atomicAdd(ccount, 1ull);
      atomicAdd(sw + S_LINKS, 1ull);
      atomicAdd(sw + S_VALID, (unsigned long long)c);
      atomicMax(sw + S_MAXLINK, (unsigned long long)c);
    } else {
      a_links += 1;
      a_valid += c;
      a_mlink = max(a_mlink, c);
    }
  }
  if (!DIRECT && (st & 4)) {  // single-packet source (its maxima of 1 are folded in at the end)
    if (WIN && gwin < 0) {
      atomicAdd(sw + S_SRCS, 1ull);
      atomicMax(sw + S_MAXSRCPK, 1ull);
      atomicMax(sw + S_MAXFANOUT, 1ull);
    } else {
      a_srcs += 1;
    }
  } else if (st & 8) {
    const uint32_t pf = DIRECT ? dir[hs] : s.t2pf[hs];
    if (PARTIAL) {
      gsrc.add((uint32_t)(key >> b), ((unsigned long long)(pf >> 16) << 32) | (pf & 0xFFFFu));
    } else if (WIN && gwin < 0) {
      atomicAdd(sw + S_SRCS, 1ull);
      atomicMax(sw + S_MAXSRCPK, (unsigned long long)(pf & 0xFFFFu));
      atomicMax(sw + S_MAXFANOUT, (unsigned long long)(pf >> 16));
    } else {
      a_srcs += 1;
      a_msrc = max(a_msrc, pf & 0xFFFFu);
      a_mfan = max(a_mfan, pf >> 16);
    }
    if (DIRECT) {
      dir[hs] = 0;
    } else {
      s.t2key[hs] = 0;
      s.t2pf[hs] = 0;
    }
  }
  s.bml[kh >> 4] = 0;  // benign: every writer stores 0
}

// WIN (per-window statistics, analytics.py:109-130): keys carry the window id above
// the 2b address bits and the statistics go to stats[9 w ..]. A group whose buckets lie
// in one window (plan .z / .w >> wsh) accumulates in registers and flushes at its end;
// a group spanning windows (only at window edges) adds per key. Column entries carry
// the window above the destination (dst' = w << b | dst, b + wb <= 32).
template <bool PARTIAL, bool WIN = false>
__global__ void __launch_bounds__(kLocThreads, 2)
    local_rows_kernel(const uint64_t* __restrict__ keys, const uint4* __restrict__ plan, uint32_t ngroups, int b,
                      uint64_t* __restrict__ col, int cshift,
                      uint32_t* __restrict__ chist, unsigned long long* __restrict__ ccount,
                      unsigned long long* __restrict__ stats, SrcTable gsrc, int dsb,
                      const uint32_t* __restrict__ ngp = nullptr, int wsh = 0) {
  if (ngp) ngroups = *ngp;  // group count on the device (grid sized for the SMs)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LocSmem& s = *reinterpret_cast<LocSmem*>(smem_raw);
  // kLocDirect slots over bms, t2key, t2pf (contiguous members), addressed from the raw buffer
  uint32_t* dir = reinterpret_cast<uint32_t*>(smem_raw + offsetof(LocSmem, bms));
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kBmWords; i += kLocThreads) s.bml[i] = s.bms[i] = 0;
  if (tid < (1 << kMsdMaxLevelBits)) s.chist[tid] = 0;
  for (int i = tid; i < kLocT1; i += kLocThreads) {
    s.t1key[i] = 0;
    s.t1cnt[i] = 0;
  }
  for (int i = tid; i < kLocT2; i += kLocThreads) {
    s.t2key[i] = 0;
    s.t2pf[i] = 0;
  }
  if (tid == 0) {
    s.sp_link = s.sp_src_pk = s.sp_src_fo = s.one_fo = 0;
    if (blockIdx.x < ngroups) s.plan[0] = plan[blockIdx.x];
  }
  __syncthreads();
  uint64_t kr[kLocPerThread];
  uint32_t nmine = 0;
  if (blockIdx.x < ngroups) {
    const uint4 p = s.plan[0];
    const uint32_t nlight = light_count(p);
#pragma unroll
    for (int r = 0; r < kLocPerThread; ++r) {
      const uint32_t j = tid + r * kLocThreads;
      if (j < nlight) {
        kr[r] = keys[light_index(p, j)];
        ++nmine;
      }
    }
  }
  // per-thread totals in 32 bits (a thread sees < 2^32 keys; per-group maxima <= 2048)
  uint32_t a_valid = 0, a_links = 0, a_srcs = 0, a_mlink = 0, a_msrc = 0, a_mfan = 0;
  uint32_t it = 0;
  for (uint32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const uint32_t cur = it & 1;
    const uint32_t gn = g + gridDim.x;
    uint4 pnext = make_uint4(0, 0, 0, 0);
    if (tid == 0 && gn < ngroups) pnext = plan[gn];
    // source range of the group's buckets -> direct source slots when it fits
    uint64_t slo = 0;
    bool direct = false;
    if (!PARTIAL && dsb != kNoDirect) {
      const uint4 pc = s.plan[cur];
      uint64_t shi;
      if (dsb >= 0) {
        slo = (uint64_t)pc.z << dsb;
        shi = (uint64_t)pc.w << dsb;
      } else {
        slo = pc.z >> -dsb;
        shi = (uint64_t)((pc.w - 1) >> -dsb) + 1;
      }
      direct = shi - slo <= kLocDirect;
    }
    int gwin = 0;  // WIN: the group's window, -1 when its buckets span several
    if constexpr (WIN) {
      const uint4 pc = s.plan[cur];
      const uint32_t w0 = pc.z >> wsh, w1 = (pc.w > pc.z ? pc.w - 1 : pc.z) >> wsh;
      gwin = w0 == w1 ? (int)w0 : -1;
    }
    // 1. hash counters (the 16-bit counter indices stay in registers for phases 2-3)
    // (source counter indices are recomputed where the hashed source path needs them)
    uint32_t kh[kLocPerThread];
#pragma unroll
    for (int r = 0; r < kLocPerThread; ++r) {
      kh[r] = h16(kr[r]);
      if ((uint32_t)r < nmine) {
        bm_hit(s.bml, kh[r]);
        if (!PARTIAL && !direct) bm_hit(s.bms, h16u((uint32_t)(kr[r] >> b)));
      }
    }
    if (tid == 0) s.plan[cur ^ 1] = pnext;
    // PARTIAL: a group whose keys all share one source (a heavy source's slice)
    // sums it once per group instead of per warp and key
    bool single = false;
    if constexpr (PARTIAL) {
      const uint4 pc = s.plan[cur];
      bool mine_same = true;
      if (light_count(pc)) {
        const uint32_t src0 = (uint32_t)(keys[light_index(pc, 0)] >> b);
#pragma unroll
        for (int r = 0; r < kLocPerThread; ++r)
          if ((uint32_t)r < nmine && (uint32_t)(kr[r] >> b) != src0) mine_same = false;
      }
      single = __syncthreads_and(mine_same) != 0;
    } else {
      __syncthreads();
    }
    // next group's keys: issue the loads now, they land during phases 2-3
    const uint4 p = s.plan[cur];
    const uint4 pn = s.plan[cur ^ 1];
    uint64_t kn[kLocPerThread];
    uint32_t nnext = 0;
    if (gn < ngroups) {
      const uint32_t nl2 = light_count(pn);
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r) {
        const uint32_t j = tid + r * kLocThreads;
        if (j < nl2) {
          kn[r] = keys[light_index(pn, j)];
          ++nnext;
        }
      }
    }
    // 2. classify; exact tables for colliding keys only (the direct-slot and the
    // hashed-source bodies are separate loops: one uniform branch per group)
    uint32_t st[kLocPerThread];   // bit0 fast link, bit1 fresh (table creator), bit2 fast source, bit3 source creator
    uint32_t hl[kLocPerThread], hs[kLocPerThread];
    if (!PARTIAL && direct) {
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r)
        st[r] = (uint32_t)r < nmine ? rows_classify<PARTIAL, true>(s, dir, kr[r], kh[r], b, slo, hl[r], hs[r]) : 0u;
    } else {
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r)
        st[r] = (uint32_t)r < nmine ? rows_classify<PARTIAL, false>(s, dir, kr[r], kh[r], b, slo, hl[r], hs[r]) : 0u;
    }
    if constexpr (PARTIAL) {
      if (single) {  // fresh links of the group's one source: per warp, then one shared add
        uint32_t nf = 0;
#pragma unroll
        for (int r = 0; r < kLocPerThread; ++r) nf += ((uint32_t)r < nmine && (st[r] & 3u)) ? 1u : 0u;
        nf = __reduce_add_sync(FULL, nf);
        if (lane == 0 && nf) atomicAdd(&s.one_fo, nf);
      }
    }
    if constexpr (PARTIAL) if (!single) {
      // every lane runs every r (ballots): lanes sharing the warp leader's source
      // add once; the source-table creator (bit 8) flushes it after the barrier
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r) {
        const bool v = (uint32_t)r < nmine;
        const uint32_t src = v ? (uint32_t)(kr[r] >> b) : 0u;
        const bool fr = v && (st[r] & 3u);
        const uint32_t vm = __ballot_sync(FULL, v);
        if (!vm) continue;
        const int leader = __ffs(vm) - 1;
        const uint32_t ls = __shfl_sync(FULL, src, leader);
        const uint32_t same = __ballot_sync(FULL, v && src == ls);
        const uint32_t fm = __ballot_sync(FULL, fr);
        uint32_t add_pk = 0, add_fo = 0;
        if (same == vm) {
          if (lane == leader) add_pk = __popc(vm), add_fo = __popc(fm);
        } else if (v) {
          add_pk = 1, add_fo = fr ? 1u : 0u;
        }
        if (add_pk) {
          if (src == 0xFFFFFFFFu) {
            atomicAdd(&s.sp_src_pk, add_pk);
            atomicAdd(&s.sp_src_fo, add_fo);
          } else {
            const uint32_t sk = src + 1;
            uint32_t h = hslot(sk, kLocT2);
            for (;;) {
              uint32_t c0 = s.t2key[h];
              if (c0 == 0) {
                c0 = atomicCAS(&s.t2key[h], 0u, sk);
                if (c0 == 0) {
                  st[r] |= 8;
                  c0 = sk;
                }
              }
              if (c0 == sk) {
                atomicAdd(&s.t2pf[h], add_pk | (add_fo << 16));
                break;
              }
              h = h + 1 == kLocT2 ? 0 : h + 1;
            }
            hs[r] = h;
          }
        }
      }
    }
    __syncthreads();
    // 3. results: one column slot per key, creators report and clear
    if (!PARTIAL && direct) {
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r)
        if ((uint32_t)r < nmine)
          rows_result<PARTIAL, WIN, true>(s, dir, kr[r], kh[r], st[r], hl[r], hs[r],
                                          light_index(p, tid + r * kLocThreads), b, col, cshift, gwin, stats, ccount,
                                          gsrc, a_valid, a_links, a_srcs, a_mlink, a_msrc, a_mfan);
    } else {
#pragma unroll
      for (int r = 0; r < kLocPerThread; ++r)
        if ((uint32_t)r < nmine)
          rows_result<PARTIAL, WIN, false>(s, dir, kr[r], kh[r], st[r], hl[r], hs[r],
                                           light_index(p, tid + r * kLocThreads), b, col, cshift, gwin, stats, ccount,
                                           gsrc, a_valid, a_links, a_srcs, a_mlink, a_msrc, a_mfan);
      if (!PARTIAL) {  // source counters of the hashed path (a loop of its own, see local_cols_kernel)
#pragma unroll
        for (int r = 0; r < kLocPerThread; ++r)
          if ((uint32_t)r < nmine) s.bms[h16u((uint32_t)(kr[r] >> b)) >> 4] = 0;
      }
    }
    if (PARTIAL && single && tid == 0 && light_count(p))
      gsrc.add((uint32_t)(keys[light_index(p, 0)] >> b), ((unsigned long long)s.one_fo << 32) | light_count(p));
    if (tid == 0 && s.sp_src_pk) {
      if (PARTIAL) {
        gsrc.add(0xFFFFFFFFu, ((unsigned long long)s.sp_src_fo << 32) | s.sp_src_pk);
      } else if (WIN && gwin < 0) {  // source' 0xFFFFFFFF: the last window (b + wb = 32)
        unsigned long long* sw = stats + (size_t)S_COUNT * (0xFFFFFFFFu >> b);
        atomicAdd(sw + S_SRCS, 1ull);
        atomicMax(sw + S_MAXSRCPK, (unsigned long long)s.sp_src_pk);
        atomicMax(sw + S_MAXFANOUT, (unsigned long long)s.sp_src_fo);
      } else {
        a_srcs += 1;
        a_msrc = max(a_msrc, s.sp_src_pk);
        a_mfan = max(a_mfan, s.sp_src_fo);
      }
    }
    if constexpr (WIN) {
      if (gwin >= 0) {  // one window: this group's totals now
        flush_rows(stats + (size_t)S_COUNT * gwin, ccount, a_valid, a_links, a_srcs, a_mlink, a_msrc, a_mfan);
        a_valid = a_links = a_srcs = a_mlink = a_msrc = a_mfan = 0;
      }
    }
    __syncthreads();
    if (tid == 0) s.sp_link = s.sp_src_pk = s.sp_src_fo = s.one_fo = 0;  // not touched before the next barrier
#pragma unroll
    for (int r = 0; r < kLocPerThread; ++r) kr[r] = kn[r];
    nmine = nnext;
  }
  if (!WIN) flush_rows(stats, ccount, a_valid, a_links, a_srcs, a_mlink, a_msrc, a_mfan);
  __syncthreads();
  if (tid < (1 << kMsdMaxLevelBits) && s.chist[tid]) atomicAdd(chist + tid, s.chist[tid]);
}

// (dst, count) u32 pairs -> packed column items
__global__ void pack_cols_kernel(const uint32_t* __restrict__ dst, const uint32_t* __restrict__ cnt, uint64_t n,
                                 uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = ((uint64_t)dst[i] << 32) | cnt[i];
}

// packed column items (dst << 32 | count) from two arrays; a zero count is a hole
struct ColConcatSrc {
  const uint64_t* e1;
  uint64_t n1;
  const uint64_t* e2;
  uint64_t n2;
  uint64_t n;  // n1 + n2
  bool quad = false;  // e1 16-byte aligned
  __device__ __forceinline__ bool load(uint64_t i, uint64_t& item, uint32_t& val) const {
    const bool in = i < n;
    const uint64_t j = in ? i : 0;
    item = j < n1 ? e1[j] : e2[j - n1];
    val = 0;
    return in && (uint32_t)item != 0;
  }
  __device__ __forceinline__ bool load(uint64_t i, uint32_t& key, uint32_t& val) const {
    uint64_t e;
    const bool ok = load(i, e, val);
    key = (uint32_t)(e >> 32);
    val = (uint32_t)e;
    return ok;
  }
  __device__ __forceinline__ void load_quad(uint64_t q, uint64_t* item, bool* ok) const {
    const uint64_t i = 4 * q;
    if (quad && i + 4 <= n1) {
      const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(e1) + 2 * q);
      const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(e1) + 2 * q + 1);
      item[0] = a.x, item[1] = a.y, item[2] = b.x, item[3] = b.y;
#pragma unroll
      for (int t = 0; t < 4; ++t) ok[t] = (uint32_t)item[t] != 0;
    } else {
      uint32_t v;
#pragma unroll
      for (int t = 0; t < 4; ++t) ok[t] = load(i + t, item[t], v);
    }
  }
};

// the column partition moves packed u64 items (dst << 32 | count): one 8-byte
// stream per level (whole 128-byte runs per digit)
__device__ __forceinline__ void quad_items(const ColConcatSrc& s, uint64_t q, uint64_t* k, uint32_t* v, bool* ok) {
  s.load_quad(q, k, ok);
  v[0] = v[1] = v[2] = v[3] = 0;
}
// ---------------------------------------------------------------------------
// LOC (columns): per group of destination buckets, shared-memory hash of dst ->
// (fan-in, packets); heavy buckets go to the LSD column path
// ---------------------------------------------------------------------------
constexpr int kLocCT = 3072;
struct LocColSmem {
  uint32_t bm[kBmWords];          // destination hash counters
  uint32_t key[kLocCT];           // exact table for colliding destinations: dst + 1 (0 = empty)
  // fan-in and packets per destination: two native 32-bit shared atomics (a 64-bit
  // shared atomicAdd is a CAS loop, which a hot destination turns into a retry storm)
  uint32_t nfan[kLocCT], npk[kLocCT];
  uint32_t spf, spp;  // dst == 0xFFFFFFFF
  uint4 plan[2];
};
// direct destination slots: fan-in at words [0, kLocColDirect), packets at
// [kLocColDirect, 2 kLocColDirect) of bm .. npk (contiguous)
constexpr uint32_t kLocColDirect = (kBmWords + 3 * kLocCT) / 2;
static_assert(offsetof(LocColSmem, key) == offsetof(LocColSmem, bm) + 4 * kBmWords &&
                  offsetof(LocColSmem, npk) + 4 * kLocCT == offsetof(LocColSmem, bm) + 8 * kLocColDirect,
              "direct destination slots span bm .. npk");

// Same three phases as local_rows_kernel over (dst, count) column entries: a
// destination whose hash counter reads "once" has fan-in 1 and `count` packets.
// Direct destinations as in local_rows_kernel: groups whose buckets span
// <= kLocColDirect destinations (bucket << dsb) count in slots dst - lo.
__device__ __forceinline__ void flush_cols(unsigned long long* __restrict__ st, uint32_t a_cnt, uint32_t a_fanin,
                                           uint32_t a_pk) {
  if (a_cnt) a_fanin = max(a_fanin, 1u);
  unsigned long long w_cnt = a_cnt;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    w_cnt += __shfl_xor_sync(FULL, w_cnt, o);
    a_fanin = max(a_fanin, __shfl_xor_sync(FULL, a_fanin, o));
    a_pk = max(a_pk, __shfl_xor_sync(FULL, a_pk, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (w_cnt) atomicAdd(st + S_DSTS, w_cnt);
    if (a_fanin) atomicMax(st + S_MAXFANIN, (unsigned long long)a_fanin);
    if (a_pk) atomicMax(st + S_MAXDSTPK, (unsigned long long)a_pk);
  }
}

// WIN: entries carry dst' = window << wdb | dst; per-window statistics as in
// local_rows_kernel (group window = plan .z / .w >> wsh)
// NARROW: u32 items (NarrowArgs layout) in ce32; the destination prefix is the
// group's level-1 bucket (first bucket .z >> nw.dlp); a group whose buckets span
// level-1 buckets finds each item's by position in the light offsets nw.poff.
// The raw u32 is loaded with the prefetch and decoded only when the group starts
// (decoding at load time would wait for the load in the middle of the current group):
// the group's destination prefix once per group, two operations per item.
__device__ __forceinline__ void col_load(const uint64_t* ce, const uint32_t* ce32, bool narrow, const uint4& p,
                                         uint32_t j, uint32_t& d, uint32_t& c) {
  const uint32_t i = light_index(p, j);
  if (!narrow) {
    const uint64_t e = ce[i];
    d = (uint32_t)(e >> 32);
    c = (uint32_t)e;
  } else {
    d = ce32[i];
  }
}
// prefix (level-1 bucket << delta) of a group inside one level-1 bucket, else 0xFFFFFFFF
__device__ __forceinline__ uint32_t col_prefix(const NarrowArgs& nw, const uint4& p) {
  const uint32_t l1 = p.z >> nw.dlp;
  return p.w > p.z && ((p.w - 1) >> nw.dlp) != l1 ? 0xFFFFFFFFu : l1 << nw.delta;
}
// Items of a group inside one level-1 bucket keep only their low destination bits
// (d = u >> cb: injective there; direct slots are offset by the prefix instead), a
// group spanning level-1 buckets (rare) rebuilds whole destinations by position.
template <int PT>
__device__ __forceinline__ void col_decode_group(const NarrowArgs& nw, uint32_t pre, const uint4& p, uint32_t* d,
                                                 uint32_t* c) {
  const uint32_t cm = (1u << nw.cb) - 1u;
  if (pre != 0xFFFFFFFFu) {
#pragma unroll
    for (int r = 0; r < PT; ++r) {
      const uint32_t u = d[r];
      c[r] = (u & cm) + 1u;
      d[r] = u >> nw.cb;
    }
    return;
  }
  const uint32_t l1last = (p.w - 1) >> nw.dlp;
#pragma unroll
  for (int r = 0; r < PT; ++r) {
    const uint32_t u = d[r];
    const uint32_t i = light_index(p, threadIdx.x + r * blockDim.x);
    uint32_t l1 = p.z >> nw.dlp;
    for (uint32_t q = l1 + 1; q <= l1last && nw.poff[q << nw.dlp] <= i; ++q) l1 = q;
    c[r] = (u & cm) + 1u;
    d[r] = l1 << nw.delta | u >> nw.cb;
  }
}

template <bool WIN = false, bool NARROW = false>
__global__ void __launch_bounds__(kLocColThreads, 4)
    local_cols_kernel(const uint64_t* __restrict__ ce, const uint4* __restrict__ plan, uint32_t ngroups,
                      unsigned long long* __restrict__ stats, int dsb, const uint32_t* __restrict__ ngp = nullptr,
                      int wsh = 0, int wdb = 0, const uint32_t* __restrict__ ce32 = nullptr,
                      NarrowArgs nw = NarrowArgs{}) {
  if (ngp) ngroups = *ngp;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LocColSmem& s = *reinterpret_cast<LocColSmem*>(smem_raw);
  uint32_t* dfan = reinterpret_cast<uint32_t*>(smem_raw + offsetof(LocColSmem, bm));  // bm .. npk contiguous
  uint32_t* dpk = dfan + kLocColDirect;
  const int tid = threadIdx.x;
  for (int i = tid; i < kBmWords; i += kLocColThreads) s.bm[i] = 0;
  for (int i = tid; i < kLocCT; i += kLocColThreads) {
    s.key[i] = 0;
    s.nfan[i] = 0;
    s.npk[i] = 0;
  }
  if (tid == 0) {
    s.spf = s.spp = 0;
    if (blockIdx.x < ngroups) s.plan[0] = plan[blockIdx.x];
  }
  __syncthreads();
  uint32_t kr[kLocColPerThread], vr[kLocColPerThread];
  uint32_t nmine = 0;
  if (blockIdx.x < ngroups) {
    const uint4 p = s.plan[0];
    const uint32_t nlight = light_count(p);
#pragma unroll
    for (int r = 0; r < kLocColPerThread; ++r) {
      const uint32_t j = tid + r * kLocColThreads;
      if (j < nlight) {
        col_load(ce, ce32, NARROW, p, j, kr[r], vr[r]);
        ++nmine;
      }
    }
    if (NARROW) col_decode_group<kLocColPerThread>(nw, col_prefix(nw, p), p, kr, vr);
  }
  // per-thread totals in 32 bits (fan-in and packets of one destination < 2^32)
  uint32_t a_cnt = 0, a_fanin = 0, a_pk = 0;
  uint32_t it = 0;
  uint32_t cpre = NARROW && blockIdx.x < ngroups ? col_prefix(nw, s.plan[0]) : 0u;  // current group's prefix
  for (uint32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const uint32_t cur = it & 1;
    const uint32_t gn = g + gridDim.x;
    uint4 pnext = make_uint4(0, 0, 0, 0);
    if (tid == 0 && gn < ngroups) pnext = plan[gn];
    uint32_t dlo = 0;
    bool direct = false;
    if (dsb != kNoDirect) {
      const uint4 pc = s.plan[cur];
      dlo = pc.z << dsb;
      direct = ((uint64_t)pc.w << dsb) - dlo <= kLocColDirect;
      // items of a one-bucket group carry destinations without the prefix
      if (NARROW && cpre != 0xFFFFFFFFu) dlo -= cpre;
    }
    int gwin = 0;  // WIN: the group's window, -1 when its buckets span several
    if constexpr (WIN) {
      const uint4 pc = s.plan[cur];
      const uint32_t w0 = pc.z >> wsh, w1 = (pc.w > pc.z ? pc.w - 1 : pc.z) >> wsh;
      gwin = w0 == w1 ? (int)w0 : -1;
    }
    if (!direct) {
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r)
        if ((uint32_t)r < nmine) bm_hit(s.bm, h16u(kr[r]));  // one IMAD: recomputed below, not kept
    }
    if (tid == 0) s.plan[cur ^ 1] = pnext;
    __syncthreads();
    const uint4 pn = s.plan[cur ^ 1];
    uint32_t kn[kLocColPerThread], vn[kLocColPerThread];
    uint32_t nnext = 0;
    if (gn < ngroups) {
      const uint32_t nl2 = light_count(pn);
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r) {
        const uint32_t j = tid + r * kLocColThreads;
        if (j < nl2) {
          col_load(ce, ce32, NARROW, pn, j, kn[r], vn[r]);
          ++nnext;
        }
      }
    }
    uint32_t hh[kLocColPerThread];
    uint32_t stc = 0;  // bit r: fast, bit r+8: table creator
    // this destination's totals when entry r reports it (WIN edge groups: per entry)
    auto report = [&](int r, uint32_t fan, uint32_t pk) {
      if (WIN && gwin < 0) {  // a group at a window edge: straight to the entry's window
        unsigned long long* sw = stats + (size_t)S_COUNT * (kr[r] >> wdb);
        atomicAdd(sw + S_DSTS, 1ull);
        atomicMax(sw + S_MAXFANIN, (unsigned long long)fan);
        atomicMax(sw + S_MAXDSTPK, (unsigned long long)pk);
      } else {
        a_cnt += 1;
        a_fanin = max(a_fanin, fan);
        a_pk = max(a_pk, pk);
      }
    };
    if (direct) {  // direct slots: separate loops (one uniform branch per group)
      bool big = false;
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r) {
        if ((uint32_t)r >= nmine) continue;
        const uint32_t o = kr[r] - dlo;
        // one atomic: fan-in in bits 20+ (<= 2048 entries) | packets of counts < 512
        // (a group's sum of those stays < 2^20); larger counts add to dpk
        const uint32_t c = vr[r];
        const uint32_t small = c < 512u ? c : 0u;
        if (atomicAdd(&dfan[o], (1u << 20) | small) == 0) stc |= 256u << r;
        if (!small) {
          atomicAdd(&dpk[o], c);
          big = true;
        }
        hh[r] = o;
      }
      // dpk is all zero unless some entry of the group added to it: only then do the
      // creators read and clear it (uniform data: no count >= 512, half the slot traffic)
      if (__syncthreads_or(big)) {
#pragma unroll
        for (int r = 0; r < kLocColPerThread; ++r) {
          if ((uint32_t)r >= nmine || !(stc & (256u << r))) continue;
          const uint32_t f = dfan[hh[r]];
          report(r, f >> 20, (f & 0xFFFFFu) + dpk[hh[r]]);
          dfan[hh[r]] = 0;
          dpk[hh[r]] = 0;
        }
      } else {
#pragma unroll
        for (int r = 0; r < kLocColPerThread; ++r) {
          if ((uint32_t)r >= nmine || !(stc & (256u << r))) continue;
          const uint32_t f = dfan[hh[r]];
          report(r, f >> 20, f & 0xFFFFFu);
          dfan[hh[r]] = 0;
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r) {
        if ((uint32_t)r >= nmine) continue;
        const uint32_t d = kr[r];
        if (d == 0xFFFFFFFFu) {
          atomicAdd(&s.spf, 1u);
          atomicAdd(&s.spp, vr[r]);
        } else if (bm_once(s.bm, h16u(d))) {
          stc |= 1u << r;
        } else {
          const uint32_t dk = d + 1;
          uint32_t h = hslot(dk, kLocCT);
          for (;;) {
            uint32_t c0 = s.key[h];
            if (c0 == 0) {
              c0 = atomicCAS(&s.key[h], 0u, dk);
              if (c0 == 0) {
                stc |= 256u << r;
                c0 = dk;
              }
            }
            if (c0 == dk) {
              atomicAdd(&s.nfan[h], 1u);
              atomicAdd(&s.npk[h], vr[r]);
              break;
            }
            h = h + 1 == kLocCT ? 0 : h + 1;
          }
          hh[r] = h;
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r) {
        if ((uint32_t)r >= nmine) continue;
        if (stc & (1u << r)) {  // single-link destination (fan-in 1 folded in at the end)
          report(r, 1u, vr[r]);
        } else if (stc & (256u << r)) {
          report(r, s.nfan[hh[r]], s.npk[hh[r]]);
          s.key[hh[r]] = 0;
          s.nfan[hh[r]] = 0;
          s.npk[hh[r]] = 0;
        }
      }
#pragma unroll
      for (int r = 0; r < kLocColPerThread; ++r)  // hash counters: a loop of its own
        if ((uint32_t)r < nmine) s.bm[h16u(kr[r]) >> 4] = 0;
    }
    if (tid == 0 && s.spf) {
      if (WIN && gwin < 0) {
        unsigned long long* sw = stats + (size_t)S_COUNT * (0xFFFFFFFFu >> wdb);
        atomicAdd(sw + S_DSTS, 1ull);
        atomicMax(sw + S_MAXFANIN, (unsigned long long)s.spf);
        atomicMax(sw + S_MAXDSTPK, (unsigned long long)s.spp);
      } else {
        a_cnt += 1;
        a_fanin = max(a_fanin, s.spf);
        a_pk = max(a_pk, s.spp);
      }
    }
    if constexpr (WIN) {
      if (gwin >= 0) {
        flush_cols(stats + (size_t)S_COUNT * gwin, a_cnt, a_fanin, a_pk);
        a_cnt = a_fanin = a_pk = 0;
      }
    }
    __syncthreads();
    if (tid == 0) s.spf = s.spp = 0;
#pragma unroll
    for (int r = 0; r < kLocColPerThread; ++r) {
      kr[r] = kn[r];
      vr[r] = vn[r];
    }
    if (NARROW) {
      cpre = col_prefix(nw, pn);
      if (nnext) col_decode_group<kLocColPerThread>(nw, cpre, pn, kr, vr);
    }
    nmine = nnext;
  }
  if (!WIN) flush_cols(stats, a_cnt, a_fanin, a_pk);
}

}  // namespace nmx

namespace nmx {

// Unique keys of a sorted array with their run lengths, without a lookback
// chain: pass 1 counts run heads per tile, scan_counts gives every tile its first
// output index, pass 2 writes (key, start position) of each head through shared
// memory; run_counts_kernel turns start positions into counts.
constexpr int kUniqTile = 2048;
template <bool WRITE>
__global__ void __launch_bounds__(256) unique_heads_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                          uint32_t* __restrict__ tile_heads,
                                                          const uint32_t* __restrict__ tile_off,
                                                          uint64_t* __restrict__ ukeys, uint32_t* __restrict__ ustart) {
  __shared__ __align__(16) uint64_t sk[kUniqTile + kUniqTile / 16];
  __shared__ uint32_t ss[kUniqTile];
  __shared__ uint32_t wt[kWarps + 1];
  __shared__ uint64_t s_prev;
  const int tid = threadIdx.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * kUniqTile;
  const uint32_t cnt = (uint32_t)umin64(kUniqTile, n - t0);
  constexpr int PER = kUniqTile / 256;
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // coalesced load, padded for the blocked reads below
    const uint32_t i = q * 256 + tid;
    if (i < cnt) sk[pad16(i)] = keys[t0 + i];
  }
  if (tid == 0) s_prev = t0 ? keys[t0 - 1] : ~keys[0];
  __syncthreads();
  uint64_t k[PER];
  uint32_t hmask = 0, nh = 0;
  const uint32_t i0 = tid * PER;
  uint64_t prev = i0 == 0 ? s_prev : (i0 < cnt ? sk[pad16(i0 - 1)] : 0);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      k[q] = sk[pad16(i)];
      const bool h = k[q] != prev;
      hmask |= (uint32_t)h << q;
      nh += h;
      prev = k[q];
    }
  }
  uint32_t total;
  uint32_t at = block_excl_scan<uint32_t>(nh, wt, &total);  // (its barriers also end the sk reads)
  if (!WRITE) {
    if (tid == 0) tile_heads[blockIdx.x] = total;
    return;
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if ((hmask >> q) & 1u) {
      sk[at] = k[q];
      ss[at] = (uint32_t)(t0 + i0 + q);
      ++at;
    }
  }
  __syncthreads();
  const uint32_t base = tile_off[blockIdx.x];
  for (uint32_t j = tid; j < total; j += 256) {
    ukeys[base + j] = sk[j];
    ustart[base + j] = ss[j];
  }
}
__global__ void run_counts_kernel(const uint32_t* __restrict__ ustart, uint64_t u, uint64_t n,
                                  uint64_t* __restrict__ counts) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < u; j += (uint64_t)gridDim.x * blockDim.x)
    counts[j] = (j + 1 < u ? ustart[j + 1] : n) - ustart[j];
}

// link statistics of a COO (valid, links, max link)
__global__ void coo_link_stats_kernel(const uint64_t* __restrict__ cnt, uint64_t n,
                                      unsigned long long* __restrict__ stats) {
  unsigned long long v = 0, mx = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    v += cnt[i];
    mx = max(mx, (unsigned long long)cnt[i]);  // counts < 2^63: unsigned = signed order
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v += __shfl_xor_sync(FULL, v, o);
    mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(stats + S_VALID, v);
    atomicMax(stats + S_MAXLINK, mx);
  }
}

// destinations of a COO as (dst, count) column entries
// (counts narrowed: the caller checked max count <= 2^32 - 1)
__global__ void coo_col_entries_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cnt, uint64_t n,
                                       uint32_t* __restrict__ ck, uint32_t* __restrict__ cv) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    ck[i] = (uint32_t)keys[i];
    cv[i] = (uint32_t)cnt[i];
  }
}

// Row / column statistics of a COO whose counts exceed 32 bits (a summed matrix
// with a link of >= 2^32 packets): one open-addressing table per side keyed by
// address + 1 (0 = empty), packets and links summed with 64-bit atomics, then a
// reduction over the slots. The 32-bit grouping kernels pack counts into the low
// word of their items, so these rare matrices take this path instead.
__global__ void wide_table_add_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cnt, uint64_t n,
                                      int shift, unsigned long long* __restrict__ tkey,
                                      unsigned long long* __restrict__ tpk, unsigned long long* __restrict__ tln,
                                      uint64_t mask) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ((keys[i] >> shift) & 0xFFFFFFFFull) + 1;
    uint64_t h = ((k * 0x9E3779B97F4A7C15ull) >> 20) & mask;
    for (;;) {
      const unsigned long long c0 = atomicCAS(tkey + h, 0ull, k);
      if (c0 == 0ull || c0 == k) break;
      h = (h + 1) & mask;
    }
    atomicAdd(tpk + h, (unsigned long long)cnt[i]);
    atomicAdd(tln + h, 1ull);
  }
}
__global__ void wide_table_reduce_kernel(const unsigned long long* __restrict__ tkey,
                                         const unsigned long long* __restrict__ tpk,
                                         const unsigned long long* __restrict__ tln, uint64_t slots,
                                         unsigned long long* __restrict__ stats, int s_cnt, int s_len, int s_sum) {
  unsigned long long nz = 0, ml = 0, mp = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < slots; i += (uint64_t)gridDim.x * blockDim.x)
    if (tkey[i]) {
      ++nz;
      ml = max(ml, tln[i]);
      mp = max(mp, tpk[i]);
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    nz += __shfl_xor_sync(FULL, nz, o);
    ml = max(ml, __shfl_xor_sync(FULL, ml, o));
    mp = max(mp, __shfl_xor_sync(FULL, mp, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(stats + s_cnt, nz);
    atomicMax(stats + s_len, ml);
    atomicMax(stats + s_sum, mp);
  }
}

// owner partition (multi-GPU exchange 2) of column slots, holes skipped
struct ColConcatPart {
  ColConcatSrc s;
  uint32_t* out_ck;
  uint32_t* out_cv;
  __device__ __forceinline__ bool get(uint64_t i, uint32_t& hi, uint32_t& lo) const { return s.load(i, hi, lo); }
  __device__ __forceinline__ void put(uint64_t pos, uint32_t hi, uint32_t lo) const {
    out_ck[pos] = hi;
    out_cv[pos] = lo;
  }
};


// ---------------------------------------------------------------------------
// Sorted keys on the MSD machinery (COO builds: matrix_from_pairs / build_matrices,
// traffic.py:197-242, and anything else that needs the fully sorted packet keys):
// after the dense partition every light bucket is a contiguous range and buckets are
// in key order, so sorting each group of whole buckets in place sorts the array.
// Per group (<= kLocMaxKeys keys): striped load into shared memory, 8 keys per thread
// sorted in registers (19-comparator network), then merge-path rounds through shared
// memory (runs 8 -> 16 -> ... -> P * 8, P = active threads, a power of two), and a
// striped store back. Padding slots hold ~0 and sort last.
// ---------------------------------------------------------------------------
constexpr int kSortThreads = 512;
constexpr int kSortIPT = 8;
constexpr int kSortCap = kSortThreads * kSortIPT;  // 4096 >= kLocMaxKeys
static_assert(kSortCap >= kLocMaxKeys, "a row group must fit one sort tile");
constexpr int kSortBins = 2048;          // counting-sort bins of a group's key range
constexpr uint32_t kSortSmallBin = 32;   // groups with a larger bin take the merge rounds
constexpr int kSortKPT = (kLocMaxKeys + kSortThreads - 1) / kSortThreads;  // keys per thread (striped)
constexpr int kSortRaw = kLocMaxKeys + 2;  // a group's keys plus 16-byte alignment slack
struct SortSmem {
  uint64_t raw[2][kSortRaw];             // TMA-loaded keys of the current / next group
  uint64_t k[kSortCap + kSortCap / 16];  // pad16 layout
  uint32_t cnt[kSortBins];               // bin counts, then bin cursors (-> bin ends)
  uint32_t st0[kSortBins];               // bin starts
  uint32_t wt[kSortThreads / 32 + 1];
  uint32_t maxbin;
  uint64_t bar[2];                       // mbarriers of the two raw buffers
  uint4 pl[2];                           // plans of the current / next group
};
static_assert(offsetof(SortSmem, raw) % 16 == 0 && (kSortRaw * 8) % 16 == 0, "bulk-copy destinations 16-byte aligned");

// one thread: bulk-copy group p's keys (16-byte aligned cover of [p.x, p.y)) into raw[b]
__device__ __forceinline__ void sort_group_load(SortSmem& S, const uint64_t* keys, const uint4& p, int b) {
  if (p.y == p.x) return;
  const uint64_t a = (8ull * p.x) & ~15ull, e = (8ull * p.y + 15) & ~15ull;
  mbar_expect_tx(&S.bar[b], (uint32_t)(e - a));
  bulk_g2s(S.raw[b], reinterpret_cast<const unsigned char*>(keys) + a, (uint32_t)(e - a), &S.bar[b]);
}

__device__ __forceinline__ void cmpx(uint64_t& a, uint64_t& b) {
  const uint64_t x = a < b ? a : b, y = a < b ? b : a;
  a = x;
  b = y;
}
__device__ __forceinline__ void sort8(uint64_t* r) {
  cmpx(r[0], r[1]); cmpx(r[2], r[3]); cmpx(r[4], r[5]); cmpx(r[6], r[7]);
  cmpx(r[0], r[2]); cmpx(r[1], r[3]); cmpx(r[4], r[6]); cmpx(r[5], r[7]);
  cmpx(r[1], r[2]); cmpx(r[5], r[6]);
  cmpx(r[0], r[4]); cmpx(r[1], r[5]); cmpx(r[2], r[6]); cmpx(r[3], r[7]);
  cmpx(r[2], r[4]); cmpx(r[3], r[5]);
  cmpx(r[1], r[2]); cmpx(r[3], r[4]); cmpx(r[5], r[6]);
}

// Fast path: the group's keys lie in [b0 << rb, b1 << rb) (its buckets); a counting sort
// by the monotone bin (key - lo) >> s into 2048 bins, then each bin (a few keys when the
// keys spread) insertion-sorted by one thread. A group with a bin above kSortSmallBin keys
// (clustered keys) takes the merge rounds below instead.
__global__ void __launch_bounds__(kSortThreads, 2)
    local_sort_kernel(uint64_t* __restrict__ keys, const uint4* __restrict__ plan, const uint32_t* __restrict__ ngp,
                      int rb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
  const uint32_t ngroups = *ngp;
  const uint32_t tid = threadIdx.x;
  // the next group's keys arrive by TMA bulk copy (one thread, mbarrier completion)
  // while the current group is sorted
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init_fence();
    if (blockIdx.x < ngroups) {
      S.pl[0] = plan[blockIdx.x];
      sort_group_load(S, keys, S.pl[0], 0);
    }
  }
  __syncthreads();
  uint32_t phase = 0;  // bit b: parity of raw[b]'s next completion
  uint32_t it = 0;
  for (uint32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const int b = it & 1;
    const uint4 p = S.pl[b];
    if (tid == 0) {
      S.maxbin = 0;
      const uint32_t gn = g + gridDim.x;
      if (gn < ngroups) {  // raw[b ^ 1] was last read before the previous group's final barrier
        S.pl[b ^ 1] = plan[gn];
        fence_proxy_async_smem();
        sort_group_load(S, keys, S.pl[b ^ 1], b ^ 1);
      }
    }
    for (int i = tid; i < kSortBins; i += kSortThreads) S.cnt[i] = 0;
    const uint32_t cnt = p.y - p.x;
    if (!cnt) {  // uniform; nothing was loaded for it
      __syncthreads();
      continue;
    }
    mbar_wait(&S.bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const uint64_t* gk = S.raw[b] + (p.x & 1u);  // the group's keys in shared memory
    __syncthreads();
    {
      const uint64_t lo = (uint64_t)p.z << rb, range = (uint64_t)(p.w - p.z) << rb;
      const int sh = max(0, 64 - __clzll((long long)(range - 1)) - 11);  // (range - 1) >> sh < 2048
      uint64_t kr[kSortKPT];
      uint32_t bn[kSortKPT];
#pragma unroll
      for (int r = 0; r < kSortKPT; ++r) {
        const uint32_t j = tid + r * kSortThreads;
        if (j < cnt) {
          kr[r] = gk[j];
          bn[r] = (uint32_t)((kr[r] - lo) >> sh);
          atomicAdd(&S.cnt[bn[r]], 1u);
        }
      }
      __syncthreads();
      constexpr int PER = kSortBins / kSortThreads;  // 4 bins per thread
      uint32_t c4[PER], sum = 0, mx = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        c4[q] = S.cnt[tid * PER + q];
        sum += c4[q];
        mx = max(mx, c4[q]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
      if ((tid & 31) == 0) atomicMax(&S.maxbin, mx);
      uint32_t total;
      uint32_t ex = block_excl_scan_n<kSortThreads>(sum, S.wt, &total);
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        S.st0[tid * PER + q] = ex;
        S.cnt[tid * PER + q] = ex;
        ex += c4[q];
      }
      __syncthreads();
      if (S.maxbin <= kSortSmallBin) {
#pragma unroll
        for (int r = 0; r < kSortKPT; ++r) {
          const uint32_t j = tid + r * kSortThreads;
          if (j < cnt) S.k[pad16(atomicAdd(&S.cnt[bn[r]], 1u))] = kr[r];
        }
        __syncthreads();
        for (int bq = tid; bq < kSortBins; bq += kSortThreads) {
          const uint32_t b0 = S.st0[bq], b1 = S.cnt[bq];
          for (uint32_t i = b0 + 1; i < b1; ++i) {
            const uint64_t x = S.k[pad16(i)];
            uint32_t j = i;
            while (j > b0) {
              const uint64_t y = S.k[pad16(j - 1)];
              if (y <= x) break;
              S.k[pad16(j)] = y;
              --j;
            }
            S.k[pad16(j)] = x;
          }
        }
        __syncthreads();
        for (uint32_t i = tid; i < cnt; i += kSortThreads) keys[p.x + i] = S.k[pad16(i)];
        __syncthreads();
        continue;
      }
    }
    const uint32_t T = (cnt + kSortIPT - 1) / kSortIPT;
    uint32_t P = 1;
    while (P < T) P <<= 1;
    const uint32_t N = P * kSortIPT;
    for (uint32_t i = tid; i < N; i += kSortThreads) S.k[pad16(i)] = i < cnt ? gk[i] : ~0ull;
    __syncthreads();
    const bool act = tid < P;
    uint64_t r[kSortIPT];
    if (act) {
#pragma unroll
      for (int j = 0; j < kSortIPT; ++j) r[j] = S.k[pad16(tid * kSortIPT + j)];
      sort8(r);
    }
    for (uint32_t L = kSortIPT; L < N; L <<= 1) {
      __syncthreads();  // every read of the previous round is done
      if (act) {
#pragma unroll
        for (int j = 0; j < kSortIPT; ++j) S.k[pad16(tid * kSortIPT + j)] = r[j];
      }
      __syncthreads();
      if (act) {
        const uint32_t pos = tid * kSortIPT;
        const uint32_t a0 = pos & ~(2 * L - 1), b0 = a0 + L;  // runs A = [a0, a0 + L), B = [b0, b0 + L)
        const uint32_t d = pos - a0;                            // this thread's diagonal
        uint32_t lo = d > L ? d - L : 0, hi = d < L ? d : L;    // first i with A[i] > B[d - 1 - i]
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (S.k[pad16(a0 + mid)] <= S.k[pad16(b0 + d - 1 - mid)])
            lo = mid + 1;
          else
            hi = mid;
        }
        uint32_t i = lo, j = d - lo;
        uint64_t ka = i < L ? S.k[pad16(a0 + i)] : 0ull, kb = j < L ? S.k[pad16(b0 + j)] : 0ull;
#pragma unroll
        for (int q = 0; q < kSortIPT; ++q) {
          const bool takeA = i < L && (j >= L || ka <= kb);
          r[q] = takeA ? ka : kb;
          if (takeA) {
            ++i;
            ka = i < L ? S.k[pad16(a0 + i)] : 0ull;
          } else {
            ++j;
            kb = j < L ? S.k[pad16(b0 + j)] : 0ull;
          }
        }
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int j = 0; j < kSortIPT; ++j) S.k[pad16(tid * kSortIPT + j)] = r[j];
    }
    __syncthreads();
    for (uint32_t i = tid; i < cnt; i += kSortThreads) keys[p.x + i] = S.k[pad16(i)];
    __syncthreads();  // smem and plan are reused by the next group
  }
}

}  // namespace nmx
