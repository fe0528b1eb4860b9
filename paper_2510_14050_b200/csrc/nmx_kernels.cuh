// nmx_kernels.cuh -- the traffic-matrix hot path as sm_100a kernels.
//
// Pipeline for one call (n packets, b address bits, W windows, wb window bits):
//   K1  hist_kernel<PacketSrc>   ingest u32 src/dst (+valid) -> digit histograms of
//                                 every LSD pass of key = win<<2b | src<<b | dst
//   K2  onesweep_pass<...>       one stable 8-bit LSD pass per non-trivial digit;
//                                 the first pass packs keys straight from the packet
//                                 columns (traffic.py:205-207 `src*dim+dst`)
//   K3  rle_kernel               run-length encode sorted keys -> unique links
//                                 (np.unique(return_counts), traffic.py:207)
//   K5  row_kernel               per-link + per-source statistics (segmented over
//                                 src runs), emits (dst, count) for the columns and
//                                 their digit histograms (traffic.py:267-277)
//   K6  onesweep_pass<u32|u64,+count> then col_kernel: per-destination statistics
//                                 (traffic.py:279-283 bincount / add.at)
// Statistics land in a per-window u64[9] array (analytics.py:95-130 + the three
// Graph Challenge maxima).
#pragma once
#include "nmx_device.cuh"

namespace nmx {

// statistic slots (canonical order, oracle/netmeter_oracle.py STATS9_FIELDS)
enum : int {
  S_VALID = 0,
  S_LINKS = 1,
  S_MAXLINK = 2,
  S_SRCS = 3,
  S_MAXSRCPK = 4,
  S_MAXFANOUT = 5,
  S_DSTS = 6,
  S_MAXDSTPK = 7,
  S_MAXFANIN = 8,
  S_COUNT = 9
};

// ---------------------------------------------------------------------------
// item sources
// ---------------------------------------------------------------------------
// Raw packet columns -> packed key. Invalid packets are dropped here
// (traffic.py:238-240), their positions still define the windows.
struct PacketSrc {
  const uint32_t* src;
  const uint32_t* dst;
  const uint8_t* valid;  // may be null (all valid)
  uint64_t n;
  uint64_t window_size;  // 0 -> single window
  int b;                 // bits per address
  __device__ __forceinline__ bool load(uint64_t i, uint64_t& key, uint32_t& val) const {
    if (i >= n) return false;
    if (valid && !__ldg(valid + i)) return false;
    uint64_t k = ((uint64_t)__ldg(src + i) << b) | __ldg(dst + i);
    if (window_size) k |= (i / window_size) << (2 * b);
    key = k;
    val = 0;
    return true;
  }
};

template <typename KeyT, bool HAS_VAL>
struct KeySrc {
  const KeyT* keys;
  const uint32_t* vals;
  uint64_t n;
  __device__ __forceinline__ bool load(uint64_t i, KeyT& key, uint32_t& val) const {
    if (i >= n) return false;
    key = keys[i];
    val = HAS_VAL ? vals[i] : 0u;
    return true;
  }
};

// ---------------------------------------------------------------------------
// K1: digit histograms for every pass, plus the valid-item count
// ---------------------------------------------------------------------------
template <typename Src, typename KeyT>
__global__ void __launch_bounds__(kThreads) hist_kernel(Src src, uint64_t n, int npass, uint32_t* __restrict__ ghist,
                                                       unsigned long long* __restrict__ gcount) {
  __shared__ uint32_t h[8][kRadix];
  for (int i = threadIdx.x; i < 8 * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t cnt = 0;
  constexpr int U = 4;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * U;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * U; base < n; base += stride) {
    KeyT k[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t v;
      uint64_t kk = 0;
      ok[u] = src.load(base + (uint64_t)u * kThreads + threadIdx.x, *reinterpret_cast<KeyT*>(&kk), v);
      k[u] = *reinterpret_cast<KeyT*>(&kk);
      cnt += ok[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      for (int p = 0; p < npass; ++p) {
        const uint32_t d = (uint32_t)(k[u] >> (8 * p)) & 0xFFu;
        const uint32_t d0 = __shfl_sync(FULL, d, 0);
        if (__all_sync(FULL, ok[u] && d == d0)) {
          if (lane == 0) atomicAdd(&h[p][d0], 32u);
        } else if (ok[u]) {
          atomicAdd(&h[p][d], 1u);
        }
      }
    }
  }
  // warp-reduce the valid count
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if (lane == 0 && cnt) atomicAdd(gcount, (unsigned long long)cnt);
  __syncthreads();
  for (int i = threadIdx.x; i < npass * kRadix; i += kThreads) {
    uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(ghist + i, v);
  }
}

// exclusive scan of each pass's 256-bin histogram -> global bin base offsets
__global__ void __launch_bounds__(kThreads) bin_scan_kernel(const uint32_t* __restrict__ ghist, int npass,
                                                           uint32_t* __restrict__ gbase) {
  __shared__ uint32_t wt[kWarps + 1];
  for (int p = 0; p < npass; ++p) {
    uint32_t tot;
    uint32_t ex = block_excl_scan<uint32_t>(ghist[p * kRadix + threadIdx.x], wt, &tot);
    gbase[p * kRadix + threadIdx.x] = ex;
  }
}

// ---------------------------------------------------------------------------
// K2: one onesweep LSD pass (8-bit digit at `shift`), stable.
//   * tile id from an atomic counter (forward progress for the lookback)
//   * warp multisplit ranking with ballots into per-warp smem counters
//   * decoupled lookback per digit over epoch-tagged u64 status words
//   * keys staged in smem in digit order -> near-coalesced scatter
// ---------------------------------------------------------------------------
template <typename KeyT, bool HAS_VAL, int IPT>
struct PassSmem {
  KeyT keys[kThreads * IPT];
  uint32_t vals[HAS_VAL ? kThreads * IPT : 1];
  uint32_t whist[kWarps][kRadix];
  uint32_t tstart[kRadix];
  uint32_t gbase[kRadix];
  uint32_t wt[kWarps + 1];
  uint32_t tile;
};

template <typename Src, typename KeyT, bool HAS_VAL, int IPT>
__global__ void __launch_bounds__(kThreads) onesweep_pass(Src src, KeyT* __restrict__ keys_out,
                                                         uint32_t* __restrict__ vals_out, int shift,
                                                         const uint32_t* __restrict__ bin_base,
                                                         uint64_t* __restrict__ status, uint32_t epoch,
                                                         uint32_t* __restrict__ tile_counter) {
  constexpr int TILE = kThreads * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& s = *reinterpret_cast<PassSmem<KeyT, HAS_VAL, IPT>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s.tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&s.whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s.tile;
  const uint64_t base = (uint64_t)tile * TILE + (uint64_t)warp * 32 * IPT;

  KeyT k[IPT];
  uint32_t v[IPT];
  uint32_t okmask = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    uint64_t kk = 0;
    uint32_t vv = 0;
    bool ok = src.load(base + (uint64_t)i * 32 + lane, *reinterpret_cast<KeyT*>(&kk), vv);
    k[i] = *reinterpret_cast<KeyT*>(&kk);
    v[i] = vv;
    okmask |= (uint32_t)ok << i;
  }

  // rank within the warp (stable: item order is (i, lane))
  uint32_t rk[IPT];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool ok = (okmask >> i) & 1u;
    const uint32_t d = (uint32_t)(k[i] >> shift) & 0xFFu;
    const uint32_t peers = warp_digit_peers(d, ok);
    const int leader = ok ? __ffs(peers) - 1 : lane;
    uint32_t b = 0;
    if (ok && lane == leader) {
      b = s.whist[warp][d];
      s.whist[warp][d] = b + __popc(peers);
    }
    b = __shfl_sync(FULL, b, leader);
    rk[i] = b + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();

  // per-digit: exclusive over warps, tile count
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    uint32_t c = s.whist[w][tid];
    s.whist[w][tid] = cnt;
    cnt += c;
  }
  // publish + decoupled lookback (thread tid owns digit tid)
  uint64_t* my = status + (size_t)tile * kRadix + tid;
  uint64_t excl = 0;
  if (tile == 0) {
    st_relaxed(my, st_pack(epoch, kFlagInc, cnt));
  } else {
    st_relaxed(my, st_pack(epoch, kFlagAgg, cnt));
    excl = lookback_exclusive(status, tile, kRadix, tid, epoch);
    st_relaxed(my, st_pack(epoch, kFlagInc, excl + cnt));
  }
  uint32_t total;
  const uint32_t tstart = block_excl_scan<uint32_t>(cnt, s.wt, &total);
  s.tstart[tid] = tstart;
  s.gbase[tid] = bin_base[tid] + (uint32_t)excl - tstart;
  __syncthreads();

#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if ((okmask >> i) & 1u) {
      const uint32_t d = (uint32_t)(k[i] >> shift) & 0xFFu;
      const uint32_t lp = s.tstart[d] + s.whist[warp][d] + rk[i];
      s.keys[lp] = k[i];
      if (HAS_VAL) s.vals[lp] = v[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const uint32_t idx = j * kThreads + tid;
    if (idx < total) {
      const KeyT key = s.keys[idx];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      const uint32_t pos = s.gbase[d] + idx;
      keys_out[pos] = key;
      if (HAS_VAL) vals_out[pos] = s.vals[idx];
    }
  }
}

// ---------------------------------------------------------------------------
// K3: run-length encode sorted keys -> ukeys[u], ustart[u+1] (ustart[u] = m)
// ---------------------------------------------------------------------------
template <int IPT>
__global__ void __launch_bounds__(kThreads) rle_kernel(const uint64_t* __restrict__ keys, uint32_t m,
                                                      uint64_t* __restrict__ ukeys, uint32_t* __restrict__ ustart,
                                                      uint64_t* __restrict__ status, uint32_t epoch,
                                                      uint32_t* __restrict__ tile_counter,
                                                      uint32_t* __restrict__ d_u) {
  constexpr int TILE = kThreads * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* ss = reinterpret_cast<uint32_t*>(sk + TILE);
  __shared__ uint32_t wt[kWarps + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prev, s_excl;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, m - t0);
  for (int j = 0; j < IPT; ++j) {
    uint32_t i = j * kThreads + tid;
    if (i < cnt) sk[i] = keys[t0 + i];
  }
  if (tid == 0) s_prev = t0 ? keys[t0 - 1] : ~keys[0];
  __syncthreads();
  uint64_t k[IPT];
  uint32_t hmask = 0, nh = 0;
  uint64_t prev = tid ? (tid * IPT - 1 < cnt ? sk[tid * IPT - 1] : 0) : s_prev;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = tid * IPT + q;
    if (i < cnt) {
      k[q] = sk[i];
      const bool h = k[q] != prev;
      hmask |= (uint32_t)h << q;
      nh += h;
      prev = k[q];
    }
  }
  uint32_t total;
  uint32_t off = block_excl_scan<uint32_t>(nh, wt, &total);
  if (tid == 0) {
    uint64_t* my = status + tile;
    uint64_t ex = 0;
    if (tile == 0) {
      st_relaxed(my, st_pack(epoch, kFlagInc, total));
    } else {
      st_relaxed(my, st_pack(epoch, kFlagAgg, total));
      ex = lookback_exclusive(status, tile, 1, 0, epoch);
      st_relaxed(my, st_pack(epoch, kFlagInc, ex + total));
    }
    s_excl = ex;
  }
  __syncthreads();  // everyone done reading sk (k[] in registers)
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    if ((hmask >> q) & 1u) {
      sk[off] = k[q];
      ss[off] = (uint32_t)(t0 + tid * IPT + q);
      ++off;
    }
  }
  __syncthreads();
  const uint64_t ex = s_excl;
  for (int j = 0; j < IPT; ++j) {
    uint32_t i = j * kThreads + tid;
    if (i < total) {
      ukeys[ex + i] = sk[i];
      ustart[ex + i] = ss[i];
    }
  }
  if (tid == 0 && t0 + cnt == m) {
    *d_u = (uint32_t)(ex + total);
    ustart[ex + total] = m;
  }
}

// ---------------------------------------------------------------------------
// segmented reduction over one tile of sorted segment keys with weights.
// Shared by the row (segment = src) and column (segment = dst) kernels.
// Emits, per window: #segments, max segment length, max segment weight.
// Segments crossing tiles are stitched by a carry lookback (CarryStatus).
// ---------------------------------------------------------------------------
struct SegOut {
  int s_count, s_maxlen, s_maxsum;  // stat slots
  int wshift;                        // window = seg >> wshift (wshift >= 64 -> window 0)
};

__device__ __forceinline__ uint64_t window_of(uint64_t seg, int wshift) { return wshift >= 64 ? 0 : (seg >> wshift); }

template <int IPT>
struct SegSmem {
  uint64_t seg[kThreads * IPT];
  uint32_t w[kThreads * IPT];
};

template <int IPT>
__device__ void seg_tile(const SegSmem<IPT>& s, uint32_t cnt, uint32_t tile, bool head0, bool tail_closes,
                         CarryStatus* __restrict__ cstatus, uint32_t epoch, unsigned long long* __restrict__ stats,
                         SegOut o, Seg* sm_seg, uint64_t* sm_carry, unsigned long long* sm_red) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t win_first = window_of(s.seg[0], o.wshift);
  const uint64_t win_last = window_of(s.seg[cnt - 1], o.wshift);
  const bool uniform = win_first == win_last;

  // pass 1: thread aggregate
  Seg agg{0, 0, 0};
  uint32_t nheads = 0;
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = tid * IPT + q;
    if (i >= cnt) break;
    const bool h = i == 0 ? head0 : (s.seg[i] != s.seg[i - 1]);
    const uint32_t w = s.w[i];
    if (h) {
      agg = Seg{1, 1, w};
      ++nheads;
    } else {
      agg.len += 1;
      agg.sum += w;
    }
  }
  Seg total;
  Seg pre = block_excl_segscan(agg, sm_seg, &total);

  // carry-in for the tile's first segment (if it started in an earlier tile).
  // A tile with a head publishes its last segment's partial as final (INC)
  // at once; a tile without one publishes AGG, looks back, then INC.
  if (tid == 0) {
    CarryStatus* my = cstatus + tile;
    if (total.f) {
      st_relaxed(&my->inc_len, total.len);
      st_relaxed(&my->inc_sum, total.sum);
      st_release(&my->flag, ((uint64_t)epoch << 2) | kFlagInc);
    } else {
      st_relaxed(&my->agg_len, total.len);
      st_relaxed(&my->agg_sum, total.sum);
      st_release(&my->flag, ((uint64_t)epoch << 2) | kFlagAgg);
    }
    uint64_t clen = 0, csum = 0;
    if (!head0) {  // implies tile > 0
      for (int64_t p = (int64_t)tile - 1; p >= 0;) {
        const uint64_t f = ld_acquire(&cstatus[p].flag);
        if ((uint32_t)(f >> 2) != epoch) continue;
        if ((f & 3) == kFlagInc) {
          clen += ld_relaxed(&cstatus[p].inc_len);
          csum += ld_relaxed(&cstatus[p].inc_sum);
          break;
        }
        clen += ld_relaxed(&cstatus[p].agg_len);
        csum += ld_relaxed(&cstatus[p].agg_sum);
        --p;
      }
    }
    if (!total.f) {
      st_relaxed(&my->inc_len, clen + total.len);
      st_relaxed(&my->inc_sum, csum + total.sum);
      st_release(&my->flag, ((uint64_t)epoch << 2) | kFlagInc);
    }
    sm_carry[0] = clen;
    sm_carry[1] = csum;
  }
  __syncthreads();
  if (!pre.f) {  // still inside the tile's first segment: add the carry
    pre.len += (uint32_t)sm_carry[0];
    pre.sum += sm_carry[1];
  }

  // pass 2: close segments (segment lengths < 2^32: the API bounds m < 2^32)
  unsigned long long lmaxlen = 0, lmaxsum = 0;
  auto close_seg = [&](uint64_t seg, uint64_t len, uint64_t sum) {
    if (uniform) {
      lmaxlen = max(lmaxlen, (unsigned long long)len);
      lmaxsum = max(lmaxsum, (unsigned long long)sum);
    } else {
      const uint64_t wdw = window_of(seg, o.wshift);
      atomicMax(stats + wdw * S_COUNT + o.s_maxlen, (unsigned long long)len);
      atomicMax(stats + wdw * S_COUNT + o.s_maxsum, (unsigned long long)sum);
    }
  };
  Seg run = pre;
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = tid * IPT + q;
    if (i >= cnt) break;
    const bool h = i == 0 ? head0 : (s.seg[i] != s.seg[i - 1]);
    const uint32_t w = s.w[i];
    if (h) {
      if (i > 0) close_seg(s.seg[i - 1], run.len, run.sum);
      if (!uniform) atomicAdd(stats + window_of(s.seg[i], o.wshift) * S_COUNT + o.s_count, 1ull);
      run = Seg{1, 1, w};
    } else {
      run.len += 1;
      run.sum += w;
    }
    if (i == cnt - 1 && tail_closes) close_seg(s.seg[i], run.len, run.sum);
  }
  if (uniform) {
    // block reduce: count (sum), maxlen, maxsum
    unsigned long long c = nheads;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      c += __shfl_xor_sync(FULL, c, off);
      lmaxlen = max(lmaxlen, __shfl_xor_sync(FULL, lmaxlen, off));
      lmaxsum = max(lmaxsum, __shfl_xor_sync(FULL, lmaxsum, off));
    }
    const int warp = tid >> 5;
    if (lane == 0) {
      sm_red[warp * 3 + 0] = c;
      sm_red[warp * 3 + 1] = lmaxlen;
      sm_red[warp * 3 + 2] = lmaxsum;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long a = 0, b2 = 0, c2 = 0;
      for (int w = 0; w < kWarps; ++w) {
        a += sm_red[w * 3];
        b2 = max(b2, sm_red[w * 3 + 1]);
        c2 = max(c2, sm_red[w * 3 + 2]);
      }
      unsigned long long* st = stats + win_first * S_COUNT;
      if (a) atomicAdd(st + o.s_count, a);
      if (b2) atomicMax(st + o.s_maxlen, b2);
      if (c2) atomicMax(st + o.s_maxsum, c2);
    }
  }
}

// ---------------------------------------------------------------------------
// K5: links + rows. Items are unique links j in [0,u): key, count = ustart[j+1]-ustart[j].
// Writes the column keys (win<<b | dst) and counts, plus their digit histograms.
// ---------------------------------------------------------------------------
template <typename ColKeyT, int IPT>
__global__ void __launch_bounds__(kThreads) row_kernel(const uint64_t* __restrict__ ukeys,
                                                      const uint32_t* __restrict__ ustart, uint32_t u, int b,
                                                      int wb, ColKeyT* __restrict__ ckeys,
                                                      uint32_t* __restrict__ ccounts, int ncolpass,
                                                      uint32_t* __restrict__ colhist, CarryStatus* cstatus,
                                                      uint32_t epoch, uint32_t* __restrict__ tile_counter,
                                                      unsigned long long* __restrict__ stats) {
  constexpr int TILE = kThreads * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& s = *reinterpret_cast<SegSmem<IPT>*>(smem_raw);
  __shared__ uint32_t h[4][kRadix];  // <= 4 column passes when ColKeyT is u32; u64 uses up to 5 -> see host
  __shared__ uint32_t h5[kRadix * 4];
  __shared__ Seg sm_seg[kWarps + 1];
  __shared__ uint64_t sm_carry[2];
  __shared__ unsigned long long sm_red[kWarps * 3];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prevseg;
  __shared__ int s_head0, s_tailc;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < 4 * kRadix; i += kThreads) {
    (&h[0][0])[i] = 0;
    h5[i] = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, (uint64_t)u - t0);
  const uint64_t dmask = (b >= 64) ? ~0ull : ((1ull << b) - 1);
  const bool uniform_w = (wb == 0) || ((ukeys[t0] >> (2 * b)) == (ukeys[t0 + cnt - 1] >> (2 * b)));
  const uint64_t wfirst = wb ? (ukeys[t0] >> (2 * b)) : 0;

  unsigned long long links = 0, valid = 0, maxlink = 0;
  for (int j = 0; j < IPT; ++j) {
    const uint32_t i = j * kThreads + tid;
    if (i < cnt) {
      const uint64_t key = ukeys[t0 + i];
      const uint32_t c = ustart[t0 + i + 1] - ustart[t0 + i];
      const uint64_t wdw = wb ? (key >> (2 * b)) : 0;
      const ColKeyT ck = (ColKeyT)((wdw << b) | (key & dmask));
      ckeys[t0 + i] = ck;
      ccounts[t0 + i] = c;
      for (int p = 0; p < ncolpass; ++p) {
        const uint32_t d = (uint32_t)((uint64_t)ck >> (8 * p)) & 0xFFu;
        if (p < 4)
          atomicAdd(&h[p][d], 1u);
        else
          atomicAdd(&h5[(p - 4) * kRadix + d], 1u);
      }
      s.seg[i] = key >> b;
      s.w[i] = c;
      if (uniform_w) {
        links += 1;
        valid += c;
        maxlink = max(maxlink, (unsigned long long)c);
      } else {
        unsigned long long* st = stats + wdw * S_COUNT;
        atomicAdd(st + S_LINKS, 1ull);
        atomicAdd(st + S_VALID, (unsigned long long)c);
        atomicMax(st + S_MAXLINK, (unsigned long long)c);
      }
    }
  }
  if (tid == 0) {
    s_prevseg = t0 ? (ukeys[t0 - 1] >> b) : 0;
    s_head0 = t0 == 0 ? 1 : 0;
    const bool last = t0 + cnt == u;
    s_tailc = last ? 1 : ((ukeys[t0 + cnt] >> b) != (ukeys[t0 + cnt - 1] >> b));
  }
  __syncthreads();
  if (tid == 0 && t0) s_head0 = s.seg[0] != s_prevseg;
  if (uniform_w) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      links += __shfl_xor_sync(FULL, links, off);
      valid += __shfl_xor_sync(FULL, valid, off);
      maxlink = max(maxlink, __shfl_xor_sync(FULL, maxlink, off));
    }
    if ((tid & 31) == 0) {
      unsigned long long* st = stats + wfirst * S_COUNT;
      atomicAdd(st + S_LINKS, links);
      atomicAdd(st + S_VALID, valid);
      atomicMax(st + S_MAXLINK, maxlink);
    }
  }
  __syncthreads();
  for (int i = tid; i < ncolpass * kRadix; i += kThreads) {
    const int p = i / kRadix, d = i % kRadix;
    const uint32_t v = p < 4 ? h[p][d] : h5[(p - 4) * kRadix + d];
    if (v) atomicAdd(colhist + i, v);
  }
  seg_tile<IPT>(s, cnt, tile, s_head0 != 0, s_tailc != 0, cstatus, epoch, stats,
                SegOut{S_SRCS, S_MAXFANOUT, S_MAXSRCPK, wb ? b : 64}, sm_seg, sm_carry, sm_red);
}

// ---------------------------------------------------------------------------
// K6 (tail): destinations, segmented over sorted column keys.
// ---------------------------------------------------------------------------
template <typename ColKeyT, int IPT>
__global__ void __launch_bounds__(kThreads) col_kernel(const ColKeyT* __restrict__ ckeys,
                                                      const uint32_t* __restrict__ ccounts, uint32_t u, int b,
                                                      int wb, CarryStatus* cstatus, uint32_t epoch,
                                                      uint32_t* __restrict__ tile_counter,
                                                      unsigned long long* __restrict__ stats) {
  constexpr int TILE = kThreads * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& s = *reinterpret_cast<SegSmem<IPT>*>(smem_raw);
  __shared__ Seg sm_seg[kWarps + 1];
  __shared__ uint64_t sm_carry[2];
  __shared__ unsigned long long sm_red[kWarps * 3];
  __shared__ uint32_t s_tile;
  __shared__ int s_head0, s_tailc;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, (uint64_t)u - t0);
  for (int j = 0; j < IPT; ++j) {
    const uint32_t i = j * kThreads + tid;
    if (i < cnt) {
      s.seg[i] = (uint64_t)ckeys[t0 + i];
      s.w[i] = ccounts[t0 + i];
    }
  }
  if (tid == 0) {
    s_head0 = t0 == 0 ? 1 : ((uint64_t)ckeys[t0 - 1] != (uint64_t)ckeys[t0]);
    const bool last = t0 + cnt == u;
    s_tailc = last ? 1 : ((uint64_t)ckeys[t0 + cnt] != (uint64_t)ckeys[t0 + cnt - 1]);
  }
  __syncthreads();
  seg_tile<IPT>(s, cnt, tile, s_head0 != 0, s_tailc != 0, cstatus, epoch, stats,
                SegOut{S_DSTS, S_MAXFANIN, S_MAXDSTPK, wb ? b : 64}, sm_seg, sm_carry, sm_red);
}

// ---------------------------------------------------------------------------
// generators and the int64 reductions of the drop-in sum_reduce / max_scan
// ---------------------------------------------------------------------------
__global__ void gen_kernel(int kind, uint64_t seed, uint64_t offset, uint64_t n, uint64_t space,
                           uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  const uint64_t base = seed << 40;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = base + 2 * (offset + i);
    const uint64_t a = splitmix64(c), d = splitmix64(c + 1);
    uint32_t s32, d32;
    if (kind == 0) {
      s32 = (uint32_t)a;
      d32 = (uint32_t)(d >> 32);
    } else {
      s32 = octave32(a);
      d32 = octave32(d);
    }
    src[i] = scale32(s32, space);
    dst[i] = scale32(d32, space);
  }
}

// op 0: sum (wraps mod 2^64 like int64 np.add.reduce), op 1: max with INT64_MIN identity
__global__ void reduce_i64_kernel(const int64_t* __restrict__ x, uint64_t n, int op,
                                  unsigned long long* __restrict__ out) {
  long long acc = op == 0 ? 0 : INT64_MIN;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const long long v = x[i];
    acc = op == 0 ? (long long)((unsigned long long)acc + (unsigned long long)v) : max(acc, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const long long y = __shfl_xor_sync(FULL, acc, o);
    acc = op == 0 ? (long long)((unsigned long long)acc + (unsigned long long)y) : max(acc, y);
  }
  if ((threadIdx.x & 31) == 0) {
    if (op == 0)
      atomicAdd(out, (unsigned long long)acc);
    else
      atomicMax(reinterpret_cast<long long*>(out), acc);
  }
}

}  // namespace nmx
