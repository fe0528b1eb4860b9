// nmx_kernels.cuh -- the traffic-matrix hot path as sm_100a kernels.
//
// Pipeline for one call (n packets, b address bits, W windows, wb window bits):
//   K1  hist_kernel          ingest u32 src/dst (+valid) -> digit histograms of every
//                            LSD pass of key = win<<2b | src<<b | dst (one read)
//   K2  onesweep_pass        one stable 8-bit LSD pass per non-trivial digit; the
//                            first pass packs keys straight from the packet columns
//                            (traffic.py:205-207 `src*dim+dst`)
//   K3+K5 link_row_kernel    run-length encode the sorted keys into unique links
//                            (np.unique(return_counts), traffic.py:207) fused with the
//                            per-link and per-source statistics (traffic.py:267-277);
//                            emits compacted (win<<b|dst, count) column entries and
//                            their digit histograms
//   K6  onesweep_pass<+count> over the column entries, then col_kernel: per-destination
//                            statistics (traffic.py:279-283 bincount / add.at)
// Every cross-tile dependency is a decoupled lookback over tile-status words.
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

// padded index for blocked (thread-contiguous) shared-memory access: 16
// consecutive items per thread would otherwise put a warp on one bank
__device__ __forceinline__ uint32_t pad16(uint32_t i) { return i + (i >> 4); }

// ---------------------------------------------------------------------------
// item sources
// ---------------------------------------------------------------------------
// Raw packet columns -> packed key. Invalid packets are dropped here
// (traffic.py:238-240); their positions still define the windows.
struct PacketSrc {
  const uint32_t* src;
  const uint32_t* dst;
  const uint8_t* valid;  // may be null (all valid)
  uint64_t n;
  uint64_t window_size;  // 0 -> single window
  int b;                 // bits per address
  bool quad = false;     // src/dst 16-byte aligned (and valid 4-byte aligned): 128-bit loads allowed
  // addresses are masked to b bits when packed: an out-of-range address (rejected by
  // the address check, which a recorded graph runs beside the pipeline) can never
  // carry key bits that index past a bucket array or a shared-memory slot table
  __device__ __forceinline__ uint32_t am() const { return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u); }
  // four consecutive packets [4q, 4q+4) with two 128-bit loads (scalar at the tail)
  __device__ __forceinline__ void load_quad(uint64_t q, uint64_t* key, bool* ok) const {
    const uint64_t i = 4 * q;
    if (quad && i + 4 <= n && !window_size) {
      const uint4 s4 = __ldg(reinterpret_cast<const uint4*>(src) + q);
      const uint4 d4 = __ldg(reinterpret_cast<const uint4*>(dst) + q);
      uint32_t vv = 0x01010101u;
      if (valid) vv = __ldg(reinterpret_cast<const uint32_t*>(valid) + q);
      const uint32_t m = am();
      key[0] = ((uint64_t)(s4.x & m) << b) | (d4.x & m);
      key[1] = ((uint64_t)(s4.y & m) << b) | (d4.y & m);
      key[2] = ((uint64_t)(s4.z & m) << b) | (d4.z & m);
      key[3] = ((uint64_t)(s4.w & m) << b) | (d4.w & m);
      ok[0] = (vv & 0xFFu) != 0;
      ok[1] = (vv & 0xFF00u) != 0;
      ok[2] = (vv & 0xFF0000u) != 0;
      ok[3] = (vv & 0xFF000000u) != 0;
    } else {
      uint32_t v;
#pragma unroll
      for (int t = 0; t < 4; ++t) ok[t] = load(i + t, key[t], v);
    }
  }
  // branch-free: the loads are issued unconditionally (clamped index) so a
  // thread's whole tile of loads can be in flight at once
  __device__ __forceinline__ bool load(uint64_t i, uint64_t& key, uint32_t& val) const {
    const bool in = i < n;
    const uint64_t j = in ? i : 0;
    const uint32_t s = __ldg(src + j), d = __ldg(dst + j);
    bool ok = in;
    if (valid) ok = ok && __ldg(valid + j) != 0;
    uint64_t k = ((uint64_t)(s & am()) << b) | (d & am());
    if (window_size) k |= (j / window_size) << (2 * b);
    key = k;
    val = 0;
    return ok;
  }
};

// PacketSrc with window ids (window_size >= 4): quads keep their 128-bit loads and
// pay one division each (at most one window edge inside a quad). A separate type so
// the window-free kernels keep their exact code.
struct PacketSrcWin : PacketSrc {
  __device__ __forceinline__ void load_quad(uint64_t q, uint64_t* key, bool* ok) const {
    const uint64_t i = 4 * q;
    if (quad && i + 4 <= n) {
      const uint4 s4 = __ldg(reinterpret_cast<const uint4*>(src) + q);
      const uint4 d4 = __ldg(reinterpret_cast<const uint4*>(dst) + q);
      uint32_t vv = 0x01010101u;
      if (valid) vv = __ldg(reinterpret_cast<const uint32_t*>(valid) + q);
      const uint32_t m = am();
      const uint64_t w = i / window_size, edge = (w + 1) * window_size;
      const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        key[t] = ((i + t < edge ? w : w + 1) << (2 * b)) | ((uint64_t)(sv[t] & m) << b) | (dv[t] & m);
        ok[t] = ((vv >> (8 * t)) & 0xFFu) != 0;
      }
    } else {
      uint32_t v;
#pragma unroll
      for (int t = 0; t < 4; ++t) ok[t] = load(i + t, key[t], v);
    }
  }
};

template <typename KeyT, bool HAS_VAL>
struct KeySrc {
  const KeyT* keys;
  const uint32_t* vals;
  uint64_t n;
  __device__ __forceinline__ bool load(uint64_t i, KeyT& key, uint32_t& val) const {
    const bool in = i < n;
    const uint64_t j = in ? i : 0;
    key = keys[j];
    val = HAS_VAL ? vals[j] : 0u;
    return in;
  }
  __device__ __forceinline__ uint64_t size() const { return n; }
};

// KeySrc whose item count lives in device memory (written by an earlier kernel
// on the stream), so the host launches the next level without reading it back;
// grids are sized by an upper bound and tiles past the count exit at once
template <typename KeyT, bool HAS_VAL>
struct KeySrcD {
  const KeyT* keys;
  const uint32_t* vals;
  const unsigned long long* np;
  __device__ __forceinline__ bool load(uint64_t i, KeyT& key, uint32_t& val) const {
    const bool in = i < *np;
    const uint64_t j = in ? i : 0;
    key = keys[j];
    val = HAS_VAL ? vals[j] : 0u;
    return in;
  }
  __device__ __forceinline__ uint64_t size() const { return *np; }
};

// ---------------------------------------------------------------------------
// K1: digit histograms for every pass, plus the valid-item count
// ---------------------------------------------------------------------------
template <typename Src, int NPASS>
__global__ void __launch_bounds__(256) hist_kernel(Src src, uint32_t* __restrict__ ghist,
                                                  unsigned long long* __restrict__ gcount) {
  __shared__ uint32_t h[NPASS][kRadix];
  for (int i = threadIdx.x; i < NPASS * kRadix; i += 256) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t cnt = 0;
  constexpr int U = 4;
  const uint64_t n = src.n;
  const uint64_t stride = (uint64_t)gridDim.x * 256 * U;
  for (uint64_t base = (uint64_t)blockIdx.x * 256 * U; base < n; base += stride) {
    uint64_t k[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t v;
      ok[u] = src.load(base + (uint64_t)u * 256 + threadIdx.x, k[u], v);
      cnt += ok[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ok[u]) {
#pragma unroll
        for (int p = 0; p < NPASS; ++p) atomicAdd(&h[p][(uint32_t)(k[u] >> (8 * p)) & 0xFFu], 1u);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(gcount, (unsigned long long)cnt);
  __syncthreads();
  for (int i = threadIdx.x; i < NPASS * kRadix; i += 256) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(ghist + i, v);
  }
}

// exclusive scan of each pass's 256-bin histogram -> global bin base offsets
__global__ void __launch_bounds__(256) bin_scan_kernel(const uint32_t* __restrict__ ghist, int npass,
                                                      uint32_t* __restrict__ gbase) {
  __shared__ uint32_t wt[kWarps + 1];
  for (int p = 0; p < npass; ++p) {
    uint32_t tot;
    const uint32_t ex = block_excl_scan<uint32_t>(ghist[p * kRadix + threadIdx.x], wt, &tot);
    gbase[p * kRadix + threadIdx.x] = ex;
  }
}

// ---------------------------------------------------------------------------
// K2: one onesweep LSD pass (8-bit digit at `shift`), stable.
//   * tile id from an atomic counter (forward progress for the lookback)
//   * warp-level stable ranking into per-warp smem counters; peers of a digit
//     found either with 8 ballots (RANK_BALLOT) or one smem atomicOr of the
//     lane bit (RANK_ATOMIC_OR); match.any ranking measured 1.4-1.8x slower
//     (profiles/r02v_onesweep_variants.txt)
//   * decoupled lookback per digit over epoch-tagged u64 status words
//   * keys staged in smem in digit order -> near-coalesced scatter
// ---------------------------------------------------------------------------
enum { RANK_BALLOT = 0, RANK_ATOMIC_OR = 1 };

template <typename KeyT, bool HAS_VAL, int THREADS, int IPT>
struct PassSmem {
  static constexpr int W = THREADS / 32;
  KeyT keys[THREADS * IPT];
  uint32_t vals[HAS_VAL ? THREADS * IPT : 1];
  uint32_t whist[W][kRadix];
  uint32_t mm[W][kRadix];
  uint32_t tstart[kRadix];
  uint32_t gbase[kRadix];
  uint32_t wt[W + 1];
  uint32_t tile;
};

template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_scan_n(uint32_t x, uint32_t* wt, uint32_t* total) {
  constexpr int W = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = warp_incl_scan(x, lane);
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < W ? wt[lane] : 0u;
    const uint32_t vi = warp_incl_scan(v, lane);
    if (lane < W) wt[lane] = vi - v;
    if (lane == W - 1) wt[W] = vi;
  }
  __syncthreads();
  const uint32_t res = wt[warp] + inc - x;
  *total = wt[W];
  __syncthreads();
  return res;
}

template <typename Src, typename KeyT, bool HAS_VAL, int THREADS, int IPT, int RANK, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    onesweep_pass(Src src, KeyT* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int shift,
                  const uint32_t* __restrict__ bin_base, uint64_t* __restrict__ status, uint32_t epoch,
                  uint32_t* __restrict__ tile_counter) {
  constexpr int TILE = THREADS * IPT;
  constexpr int W = THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& s = *reinterpret_cast<PassSmem<KeyT, HAS_VAL, THREADS, IPT>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s.tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * kRadix; i += THREADS) {
    (&s.whist[0][0])[i] = 0;
    if (RANK == RANK_ATOMIC_OR) (&s.mm[0][0])[i] = 0;
  }
  __syncthreads();
  const uint32_t tile = s.tile;
  const uint64_t base = (uint64_t)tile * TILE + (uint64_t)warp * 32 * IPT;

  KeyT k[IPT];
  uint32_t v[HAS_VAL ? IPT : 1];
  uint32_t okmask = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    uint32_t vv = 0;
    const bool ok = src.load(base + (uint64_t)i * 32 + lane, k[i], vv);
    if (HAS_VAL) v[HAS_VAL ? i : 0] = vv;
    okmask |= (uint32_t)ok << i;
  }

  // stable rank within the warp: item order is (i, lane)
  uint32_t rk[(IPT + 1) / 2];  // two 16-bit ranks per register
  const uint32_t lt = lanemask_lt();
  const uint32_t lanebit = 1u << lane;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool ok = (okmask >> i) & 1u;
    const uint32_t d = (uint32_t)(k[i] >> shift) & 0xFFu;
    uint32_t peers;
    if (RANK == RANK_BALLOT) {
      peers = warp_digit_peers(d, ok);
    } else {
      volatile uint32_t* mp = &s.mm[warp][d];
      if (ok) atomicOr((uint32_t*)mp, lanebit);
      __syncwarp();
      peers = ok ? *mp : 0u;
      __syncwarp();
    }
    const int leader = ok ? __ffs(peers) - 1 : lane;
    uint32_t b = 0;
    if (ok && lane == leader) {
      b = s.whist[warp][d];
      s.whist[warp][d] = b + __popc(peers);
      if (RANK == RANK_ATOMIC_OR) s.mm[warp][d] = 0;
    }
    b = __shfl_sync(FULL, b, leader);
    const uint32_t r = b + __popc(peers & lt);
    if (i & 1)
      rk[i >> 1] |= r << 16;
    else
      rk[i >> 1] = r;
    __syncwarp();
  }
  __syncthreads();

  // per digit (threads < 256): exclusive over warps, tile count
  uint32_t cnt = 0;
  if (tid < kRadix) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = s.whist[w][tid];
      s.whist[w][tid] = cnt;
      cnt += c;
    }
  }
  // publish the tile's aggregate at once (thread tid owns digit tid); the lookback
  // waits until the tile is staged, so predecessors have had that long to publish
  // their inclusive prefixes
  uint64_t* my = status + (size_t)tile * kRadix + tid;
  if (tid < kRadix) st_relaxed(my, st_pack(epoch, tile == 0 ? kFlagInc : kFlagAgg, cnt));
  uint32_t total;
  const uint32_t tstart = block_excl_scan_n<THREADS>(cnt, s.wt, &total);
  if (tid < kRadix) s.tstart[tid] = tstart;
  __syncthreads();

#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if ((okmask >> i) & 1u) {
      const uint32_t d = (uint32_t)(k[i] >> shift) & 0xFFu;
      const uint32_t r = (i & 1) ? (rk[i >> 1] >> 16) : (rk[i >> 1] & 0xFFFFu);
      const uint32_t lp = s.tstart[d] + s.whist[warp][d] + r;
      s.keys[lp] = k[i];
      if (HAS_VAL) s.vals[lp] = v[HAS_VAL ? i : 0];
    }
  }
  if (tid < kRadix) {
    uint64_t excl = 0;
    if (tile != 0) {
      excl = lookback_exclusive(status, tile, kRadix, tid, epoch);
      st_relaxed(my, st_pack(epoch, kFlagInc, excl + cnt));
    }
    s.gbase[tid] = bin_base[tid] + (uint32_t)excl - tstart;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const uint32_t idx = j * THREADS + tid;
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
// Composite scan element of the fused link/row kernel (all counts < 2^32):
//   nh        number of link heads (-> output index of each unique link)
//   link seg  (llen)         run of equal keys: llen = packets on the link
//   src  seg  (slen, ssum)   run of equal sources: slen = packets of the
//                             source, ssum = link heads = fan-out
//   fl        bit0: a link head occurred, bit1: a source head occurred
// ---------------------------------------------------------------------------
struct LR {
  uint32_t nh, fl, llen, slen, ssum;
  __device__ __forceinline__ static LR identity() { return LR{0, 0, 0, 0, 0}; }
};
__device__ __forceinline__ LR lr_combine(const LR& a, const LR& b) {
  LR r;
  r.nh = a.nh + b.nh;
  r.fl = a.fl | b.fl;
  r.llen = (b.fl & 1) ? b.llen : a.llen + b.llen;
  r.slen = (b.fl & 2) ? b.slen : a.slen + b.slen;
  r.ssum = (b.fl & 2) ? b.ssum : a.ssum + b.ssum;
  return r;
}
__device__ __forceinline__ LR lr_shfl_up(const LR& x, int o) {
  LR y;
  y.nh = __shfl_up_sync(FULL, x.nh, o);
  y.fl = __shfl_up_sync(FULL, x.fl, o);
  y.llen = __shfl_up_sync(FULL, x.llen, o);
  y.slen = __shfl_up_sync(FULL, x.slen, o);
  y.ssum = __shfl_up_sync(FULL, x.ssum, o);
  return y;
}

// column segment (run of equal destinations): len = fan-in, sum = packets
struct CS {
  uint32_t f, len, sum;
  __device__ __forceinline__ static CS identity() { return CS{0, 0, 0}; }
};
__device__ __forceinline__ CS cs_combine(const CS& a, const CS& b) {
  return CS{a.f | b.f, b.f ? b.len : a.len + b.len, b.f ? b.sum : a.sum + b.sum};
}
__device__ __forceinline__ CS cs_shfl_up(const CS& x, int o) {
  return CS{__shfl_up_sync(FULL, x.f, o), __shfl_up_sync(FULL, x.len, o), __shfl_up_sync(FULL, x.sum, o)};
}

// generic exclusive block scan (256 threads) for LR / CS
template <typename T, T (*COMB)(const T&, const T&), T (*SHFL)(const T&, int)>
__device__ __forceinline__ T block_excl_scan_op(T x, T* sm, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = SHFL(inc, o);
    if (lane >= o) inc = COMB(y, inc);
  }
  T ex = SHFL(inc, 1);
  if (lane == 0) ex = T::identity();
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < kWarps ? sm[lane] : T::identity();
    T wi = w;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      T y = SHFL(wi, o);
      if (lane >= o) wi = COMB(y, wi);
    }
    T we = SHFL(wi, 1);
    if (lane == 0) we = T::identity();
    __syncwarp();
    if (lane < kWarps) sm[lane] = we;
    if (lane == kWarps - 1) sm[kWarps] = wi;
  }
  __syncthreads();
  const T res = COMB(sm[warp], ex);
  *total = sm[kWarps];
  __syncthreads();
  return res;
}

// Multi-word tile status for composite lookbacks: AGG and INC payloads in
// separate words (never rewritten within an epoch), flag stored last (release).
template <int NW>
struct TileStatus {
  uint32_t agg[NW];
  uint32_t inc[NW];
  uint64_t flag;  // epoch << 2 | {1 = AGG, 2 = INC}
};

__device__ __forceinline__ void st_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T, int NW>
__device__ __forceinline__ void publish(TileStatus<NW>* st, const T& x, uint32_t epoch, bool inclusive) {
  static_assert(sizeof(T) == 4 * NW, "status payload size");
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
  uint32_t* dst = inclusive ? st->inc : st->agg;
#pragma unroll
  for (int i = 0; i < NW; ++i) st_u32(dst + i, w[i]);
  st_release(&st->flag, ((uint64_t)epoch << 2) | (inclusive ? kFlagInc : kFlagAgg));
}

// exclusive prefix of tile `tile` (single thread)
template <typename T, int NW, T (*COMB)(const T&, const T&)>
__device__ __forceinline__ T lookback_op(TileStatus<NW>* status, uint32_t tile, uint32_t epoch) {
  T acc = T::identity();
  for (int64_t p = (int64_t)tile - 1; p >= 0;) {
    const uint64_t f = ld_acquire(&status[p].flag);
    if ((uint32_t)(f >> 2) != epoch) continue;
    T x;
    uint32_t* w = reinterpret_cast<uint32_t*>(&x);
    const bool inc = (f & 3) == kFlagInc;
    const uint32_t* srcw = inc ? status[p].inc : status[p].agg;
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = ld_u32(srcw + i);
    acc = COMB(x, acc);
    if (inc) break;
    --p;
  }
  return acc;
}

using LRStatus = TileStatus<5>;
using CSStatus = TileStatus<3>;

// ---------------------------------------------------------------------------
// K3+K5: links + rows, fused. Items are the sorted keys [0, m).
// ---------------------------------------------------------------------------
template <typename ColKeyT, int IPT>
__global__ void __launch_bounds__(256) link_row_kernel(const uint64_t* __restrict__ keys, uint32_t m, int b,
                                                      int wb, ColKeyT* __restrict__ ckeys,
                                                      uint32_t* __restrict__ ccounts, int ncolpass,
                                                      uint32_t* __restrict__ colhist, LRStatus* status,
                                                      uint32_t epoch, uint32_t* __restrict__ tile_counter,
                                                      unsigned long long* __restrict__ stats,
                                                      uint32_t* __restrict__ d_u) {
  constexpr int TILE = 256 * IPT;
  // staging: keys (padded, blocked reads), then reused for the column outputs
  __shared__ __align__(16) uint64_t sk[TILE + TILE / 16];
  __shared__ uint32_t sc[TILE];
  __shared__ uint32_t h[8][kRadix];
  __shared__ LR sm_lr[kWarps + 1];
  __shared__ LR s_excl;
  __shared__ unsigned long long sm_red[kWarps][6];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prev, s_next;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < ncolpass * kRadix; i += 256) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, m - t0);
  const bool last_tile = t0 + cnt == m;
  for (int j = 0; j < IPT; ++j) {
    const uint32_t i = j * 256 + tid;
    if (i < cnt) sk[pad16(i)] = keys[t0 + i];
  }
  if (tid == 0) {
    s_prev = t0 ? keys[t0 - 1] : ~keys[0];
    s_next = last_tile ? 0 : keys[t0 + cnt];
  }
  __syncthreads();
  const uint64_t first_key = sk[0], last_key = sk[pad16(cnt - 1)];
  const int b2 = 2 * b;
  const bool uniform = wb == 0 || (first_key >> b2) == (last_key >> b2);
  const uint64_t wfirst = wb ? (first_key >> b2) : 0;
  const uint64_t sprev = s_prev, snext = s_next;

  // pass 1: thread aggregate over its IPT consecutive keys
  uint64_t k[IPT];
  const uint32_t i0 = tid * IPT;
  uint64_t prev = i0 == 0 ? sprev : (i0 < cnt ? sk[pad16(i0 - 1)] : 0);
  const uint64_t prev0 = prev;
  LR agg = LR::identity();
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      k[q] = sk[pad16(i)];
      const uint32_t hl = k[q] != prev, hs = (k[q] >> b) != (prev >> b);
      agg = lr_combine(agg, LR{hl, hl | (hs << 1), 1, 1, hl});
      prev = k[q];
    }
  }
  LR total;
  const LR pre = block_excl_scan_op<LR, lr_combine, lr_shfl_up>(agg, sm_lr, &total);
  if (tid == 0) {
    LRStatus* my = status + tile;
    LR ex = LR::identity();
    if (tile == 0) {
      publish<LR, 5>(my, total, epoch, true);
    } else {
      publish<LR, 5>(my, total, epoch, false);
      ex = lookback_op<LR, 5, lr_combine>(status, tile, epoch);
      publish<LR, 5>(my, lr_combine(ex, total), epoch, true);
    }
    s_excl = ex;
    if (last_tile) *d_u = ex.nh + total.nh;
  }
  __syncthreads();  // sk is no longer read: reused as column staging below
  const LR ex = s_excl;
  // index of the link run containing the tile's first key
  const uint32_t jbase = ex.nh + (first_key != sprev ? 1u : 0u) - 1u;
  LR run = lr_combine(ex, pre);
  ColKeyT* sck = reinterpret_cast<ColKeyT*>(sk);
  const uint64_t dmask = (1ull << b) - 1;
  // local accumulators (uniform tile): valid, links, srcs, maxlink, maxsrcpk, maxfanout
  unsigned long long a_valid = 0, a_links = 0, a_srcs = 0, a_mlink = 0, a_msrc = 0, a_mfan = 0;
  auto win = [&](uint64_t key) -> uint64_t { return wb ? (key >> b2) : 0; };
  auto emit_link = [&](uint64_t key, uint32_t j, uint32_t count) {
    const uint32_t slot = j - jbase;
    sck[slot] = (ColKeyT)((win(key) << b) | (key & dmask));
    sc[slot] = count;
    if (uniform)
      a_mlink = max(a_mlink, (unsigned long long)count);
    else
      atomicMax(stats + win(key) * S_COUNT + S_MAXLINK, (unsigned long long)count);
  };
  auto close_src = [&](uint64_t key, uint32_t slen, uint32_t ssum) {
    if (uniform) {
      a_msrc = max(a_msrc, (unsigned long long)slen);
      a_mfan = max(a_mfan, (unsigned long long)ssum);
    } else {
      unsigned long long* st = stats + win(key) * S_COUNT;
      atomicMax(st + S_MAXSRCPK, (unsigned long long)slen);
      atomicMax(st + S_MAXFANOUT, (unsigned long long)ssum);
    }
  };
  prev = prev0;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      const uint64_t key = k[q];
      const uint32_t hl = key != prev, hs = (key >> b) != (prev >> b);
      if (hl && i != 0) emit_link(prev, run.nh - 1, run.llen);
      if (hs && i != 0) close_src(prev, run.slen, run.ssum);
      run = lr_combine(run, LR{hl, hl | (hs << 1), 1, 1, hl});
      if (uniform) {
        a_valid += 1;
        a_links += hl;
        a_srcs += hs;
      } else {
        unsigned long long* st = stats + win(key) * S_COUNT;
        atomicAdd(st + S_VALID, 1ull);
        if (hl) atomicAdd(st + S_LINKS, 1ull);
        if (hs) atomicAdd(st + S_SRCS, 1ull);
      }
      if (i == cnt - 1) {  // tile tail: close what ends at the tile boundary
        if (last_tile || snext != key) emit_link(key, run.nh - 1, run.llen);
        if (last_tile || (snext >> b) != (key >> b)) close_src(key, run.slen, run.ssum);
      }
      prev = key;
    }
  }
  if (uniform) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a_valid += __shfl_xor_sync(FULL, a_valid, o);
      a_links += __shfl_xor_sync(FULL, a_links, o);
      a_srcs += __shfl_xor_sync(FULL, a_srcs, o);
      a_mlink = max(a_mlink, __shfl_xor_sync(FULL, a_mlink, o));
      a_msrc = max(a_msrc, __shfl_xor_sync(FULL, a_msrc, o));
      a_mfan = max(a_mfan, __shfl_xor_sync(FULL, a_mfan, o));
    }
    if (lane == 0) {
      sm_red[warp][0] = a_valid;
      sm_red[warp][1] = a_links;
      sm_red[warp][2] = a_srcs;
      sm_red[warp][3] = a_mlink;
      sm_red[warp][4] = a_msrc;
      sm_red[warp][5] = a_mfan;
    }
  }
  __syncthreads();
  if (uniform && tid == 0) {
    unsigned long long r[6] = {0, 0, 0, 0, 0, 0};
    for (int w = 0; w < kWarps; ++w) {
      for (int x = 0; x < 3; ++x) r[x] += sm_red[w][x];
      for (int x = 3; x < 6; ++x) r[x] = max(r[x], sm_red[w][x]);
    }
    unsigned long long* st = stats + wfirst * S_COUNT;
    atomicAdd(st + S_VALID, r[0]);
    if (r[1]) atomicAdd(st + S_LINKS, r[1]);
    if (r[2]) atomicAdd(st + S_SRCS, r[2]);
    if (r[3]) atomicMax(st + S_MAXLINK, r[3]);
    if (r[4]) atomicMax(st + S_MAXSRCPK, r[4]);
    if (r[5]) atomicMax(st + S_MAXFANOUT, r[5]);
  }
  // column entries of the links closed in this tile: [jbase, jbase + nclosed)
  const uint32_t nclosed = (ex.nh + total.nh) - jbase - ((last_tile || snext != last_key) ? 0u : 1u);
  for (uint32_t j = tid; j < nclosed; j += 256) {
    const ColKeyT ck = sck[j];
    ckeys[jbase + j] = ck;
    ccounts[jbase + j] = sc[j];
    for (int p = 0; p < ncolpass; ++p) atomicAdd(&h[p][(uint32_t)((uint64_t)ck >> (8 * p)) & 0xFFu], 1u);
  }
  __syncthreads();
  for (int i = tid; i < ncolpass * kRadix; i += 256) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(colhist + i, v);
  }
}

// ---------------------------------------------------------------------------
// K6 (tail): destinations, segmented over the sorted column entries.
// ---------------------------------------------------------------------------
template <typename ColKeyT, int IPT>
__global__ void __launch_bounds__(256) col_kernel(const ColKeyT* __restrict__ ckeys,
                                                 const uint32_t* __restrict__ ccounts, uint32_t u, int b, int wb,
                                                 CSStatus* status, uint32_t epoch,
                                                 uint32_t* __restrict__ tile_counter,
                                                 unsigned long long* __restrict__ stats, int segshift = 0,
                                                 int s_cnt = S_DSTS, int s_len = S_MAXFANIN, int s_sum = S_MAXDSTPK) {
  constexpr int TILE = 256 * IPT;
  __shared__ __align__(16) uint64_t sk[TILE + TILE / 16];
  __shared__ uint32_t sw[TILE + TILE / 16];
  __shared__ CS sm_cs[kWarps + 1];
  __shared__ CS s_excl;
  __shared__ unsigned long long sm_red[kWarps][3];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prev, s_next;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, (uint64_t)u - t0);
  const bool last_tile = t0 + cnt == u;
  for (int j = 0; j < IPT; ++j) {
    const uint32_t i = j * 256 + tid;
    if (i < cnt) {
      sk[pad16(i)] = (uint64_t)ckeys[t0 + i] >> segshift;
      sw[pad16(i)] = ccounts[t0 + i];
    }
  }
  if (tid == 0) {
    s_prev = t0 ? ((uint64_t)ckeys[t0 - 1] >> segshift) : ~((uint64_t)ckeys[0] >> segshift);
    s_next = last_tile ? 0 : ((uint64_t)ckeys[t0 + cnt] >> segshift);
  }
  __syncthreads();
  const uint64_t first_key = sk[0], last_key = sk[pad16(cnt - 1)];
  const bool uniform = wb == 0 || (first_key >> b) == (last_key >> b);
  const uint64_t wfirst = wb ? (first_key >> b) : 0;
  const uint64_t snext = s_next;
  auto win = [&](uint64_t key) -> uint64_t { return wb ? (key >> b) : 0; };

  const uint32_t i0 = tid * IPT;
  uint64_t prev = i0 == 0 ? s_prev : (i0 < cnt ? sk[pad16(i0 - 1)] : 0);
  const uint64_t prev0 = prev;
  CS agg = CS::identity();
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      const uint64_t key = sk[pad16(i)];
      agg = cs_combine(agg, CS{key != prev, 1, sw[pad16(i)]});
      prev = key;
    }
  }
  CS total;
  const CS pre = block_excl_scan_op<CS, cs_combine, cs_shfl_up>(agg, sm_cs, &total);
  if (tid == 0) {
    CSStatus* my = status + tile;
    CS ex = CS::identity();
    if (tile == 0) {
      publish<CS, 3>(my, total, epoch, true);
    } else {
      publish<CS, 3>(my, total, epoch, false);
      ex = lookback_op<CS, 3, cs_combine>(status, tile, epoch);
      publish<CS, 3>(my, cs_combine(ex, total), epoch, true);
    }
    s_excl = ex;
  }
  __syncthreads();
  CS run = cs_combine(s_excl, pre);
  unsigned long long a_cnt = 0, a_len = 0, a_sum = 0;
  auto close = [&](uint64_t key, uint32_t len, uint32_t sum) {
    if (uniform) {
      a_len = max(a_len, (unsigned long long)len);
      a_sum = max(a_sum, (unsigned long long)sum);
    } else {
      unsigned long long* st = stats + win(key) * S_COUNT;
      atomicMax(st + s_len, (unsigned long long)len);
      atomicMax(st + s_sum, (unsigned long long)sum);
    }
  };
  prev = prev0;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      const uint64_t key = sk[pad16(i)];
      const uint32_t h = key != prev;
      if (h && i != 0) close(prev, run.len, run.sum);
      run = cs_combine(run, CS{h, 1, sw[pad16(i)]});
      if (uniform)
        a_cnt += h;
      else if (h)
        atomicAdd(stats + win(key) * S_COUNT + s_cnt, 1ull);
      if (i == cnt - 1 && (last_tile || snext != key)) close(key, run.len, run.sum);
      prev = key;
    }
  }
  if (uniform) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a_cnt += __shfl_xor_sync(FULL, a_cnt, o);
      a_len = max(a_len, __shfl_xor_sync(FULL, a_len, o));
      a_sum = max(a_sum, __shfl_xor_sync(FULL, a_sum, o));
    }
    if (lane == 0) {
      sm_red[warp][0] = a_cnt;
      sm_red[warp][1] = a_len;
      sm_red[warp][2] = a_sum;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long r0 = 0, r1 = 0, r2 = 0;
      for (int w = 0; w < kWarps; ++w) {
        r0 += sm_red[w][0];
        r1 = max(r1, sm_red[w][1]);
        r2 = max(r2, sm_red[w][2]);
      }
      unsigned long long* st = stats + wfirst * S_COUNT;
      if (r0) atomicAdd(st + s_cnt, r0);
      if (r1) atomicMax(st + s_len, r1);
      if (r2) atomicMax(st + s_sum, r2);
    }
  }
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

// ---------------------------------------------------------------------------
// owner partitions for the multi-GPU exchange:
// owner(x) = (fmix32(x) * G) >> 32 (murmur3 finaliser; oracle: distributed.owner)
// ---------------------------------------------------------------------------
constexpr int kMaxParts = 64;
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}
__host__ __device__ __forceinline__ int owner_of(uint32_t x, int parts) {
  return (int)(((uint64_t)fmix32(x) * (uint64_t)parts) >> 32);
}

// packets routed by owner(src); invalid packets are dropped
struct PacketPart {
  const uint32_t* src;
  const uint32_t* dst;
  const uint8_t* valid;
  uint32_t* out_src;
  uint32_t* out_dst;
  // (owner field, other field) of item i, written back as a pair by put
  __device__ __forceinline__ bool get(uint64_t i, uint32_t& hi, uint32_t& lo) const {
    hi = src[i];
    lo = dst[i];
    return !valid || valid[i];
  }
  __device__ __forceinline__ void put(uint64_t pos, uint32_t hi, uint32_t lo) const {
    out_src[pos] = hi;
    out_dst[pos] = lo;
  }
};
// column entries (dst, count) routed by owner(dst)
struct ColPart {
  const uint32_t* ck;
  const uint32_t* cv;
  uint32_t* out_ck;
  uint32_t* out_cv;
  __device__ __forceinline__ bool get(uint64_t i, uint32_t& hi, uint32_t& lo) const {
    hi = ck[i];
    lo = cv[i];
    return true;
  }
  __device__ __forceinline__ void put(uint64_t pos, uint32_t hi, uint32_t lo) const {
    out_ck[pos] = hi;
    out_cv[pos] = lo;
  }
};

// Tiled owner split (partition_items): 2048 items per CTA, 8 per thread with their loads
// issued first; warp-aggregated ranks per part (ballots for <= 8 parts, shared atomics
// otherwise), one global reservation per (tile, part), the tile staged by part in shared
// memory and written as runs (coalesced pairs of u32 columns).
// (A block-chunked loop of 256 items per round ran at ~400 warp instructions per 32
// items: 19 ms for 2^30 column entries.)
constexpr int kPartTile = 2048;
template <typename Item>
__device__ __forceinline__ void part_tile_load(const Item& it, uint64_t base, uint64_t n, int parts, uint32_t* hi,
                                               uint32_t* lo, int* o) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint64_t i = base + (uint64_t)r * 256 + threadIdx.x;
    const bool ok = i < n && it.get(i < n ? i : 0, hi[r], lo[r]);
    o[r] = ok ? owner_of(hi[r], parts) : -1;
  }
}
// rank of each item among its tile's items of the same part (cnt: per-part counters)
__device__ __forceinline__ uint32_t part_rank(uint32_t* cnt, int o, int parts) {
  if (parts > 8) return o >= 0 ? atomicAdd(&cnt[o], 1u) : 0u;
  const int lane = threadIdx.x & 31;
  uint32_t r = 0;
  for (int p = 0; p < parts; ++p) {
    const uint32_t mask = __ballot_sync(FULL, o == p);
    if (!mask) continue;
    const int leader = __ffs(mask) - 1;
    uint32_t b = 0;
    if (lane == leader) b = atomicAdd(&cnt[p], (uint32_t)__popc(mask));
    b = __shfl_sync(FULL, b, leader);
    if (o == p) r = b + __popc(mask & lanemask_lt());
  }
  return r;
}

template <typename Item>
__global__ void __launch_bounds__(256) part_tile_count_kernel(Item it, uint64_t n, int parts,
                                                             unsigned long long* __restrict__ counts) {
  __shared__ uint32_t sc[kMaxParts];
  if (threadIdx.x < kMaxParts) sc[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t base = (uint64_t)blockIdx.x * kPartTile; base < n; base += (uint64_t)gridDim.x * kPartTile) {
    uint32_t hi[8], lo[8];
    int o[8];
    part_tile_load(it, base, n, parts, hi, lo, o);
#pragma unroll
    for (int r = 0; r < 8; ++r) part_rank(sc, o[r], parts);
  }
  __syncthreads();
  if (threadIdx.x < parts && sc[threadIdx.x]) atomicAdd(counts + threadIdx.x, (unsigned long long)sc[threadIdx.x]);
}

template <typename Item>
__global__ void __launch_bounds__(256) part_tile_scatter_kernel(Item it, uint64_t n, int parts,
                                                               unsigned long long* __restrict__ cursor) {
  __shared__ uint64_t stage[kPartTile];
  __shared__ uint8_t spart[kPartTile];  // part of each staged item
  __shared__ uint32_t cnt[kMaxParts], tstart[kMaxParts + 1];
  __shared__ unsigned long long gb[kMaxParts];
  const int tid = threadIdx.x;
  const uint64_t base = (uint64_t)blockIdx.x * kPartTile;
  if (tid < kMaxParts) cnt[tid] = 0;
  uint32_t hi[8], lo[8];
  int o[8];
  part_tile_load(it, base, n, parts, hi, lo, o);
  __syncthreads();
  uint32_t rk[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) rk[r] = part_rank(cnt, o[r], parts);
  __syncthreads();
  if (tid < parts) gb[tid] = cnt[tid] ? atomicAdd(cursor + tid, (unsigned long long)cnt[tid]) : 0ull;
  if (tid == 0) {
    uint32_t run = 0;
    for (int p = 0; p < parts; ++p) {
      tstart[p] = run;
      run += cnt[p];
    }
    tstart[parts] = run;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r)
    if (o[r] >= 0) {
      const uint32_t at = tstart[o[r]] + rk[r];
      stage[at] = ((uint64_t)hi[r] << 32) | lo[r];
      spart[at] = (uint8_t)o[r];
    }
  __syncthreads();
  const uint32_t total = tstart[parts];
  for (uint32_t j = tid; j < total; j += 256) {
    const uint64_t v = stage[j];
    const uint32_t p = spart[j];
    it.put(gb[p] + (j - tstart[p]), (uint32_t)(v >> 32), (uint32_t)v);
  }
}

// digit histograms of received u32 column keys (multi-GPU column stage)
template <int NPASS>
__global__ void __launch_bounds__(256) hist_u32_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                                      uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[NPASS][kRadix];
  for (int i = threadIdx.x; i < NPASS * kRadix; i += 256) (&h[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
    const uint32_t k = keys[i];
#pragma unroll
    for (int p = 0; p < NPASS; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFFu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NPASS * kRadix; i += 256) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(ghist + i, v);
  }
}

// ---------------------------------------------------------------------------
// Materialisation (drop-in TrafficMatrix / FlatContainers)
// ---------------------------------------------------------------------------
// reduce-by-key with compacted outputs: for every run of equal (key >> shift)
// in a sorted array emit (segment key, length, sum of weights). This is
// np.unique(return_counts) (traffic.py:207), np.add.reduceat over rows
// (traffic.py:271-277) and bincount / np.add.at over columns (traffic.py:279-283).
struct RB {
  uint32_t nh, f, len, pad;
  unsigned long long sum;
  __device__ __forceinline__ static RB identity() { return RB{0, 0, 0, 0, 0ull}; }
};
__device__ __forceinline__ RB rb_combine(const RB& a, const RB& b) {
  return RB{a.nh + b.nh, a.f | b.f, b.f ? b.len : a.len + b.len, 0u, b.f ? b.sum : a.sum + b.sum};
}
__device__ __forceinline__ RB rb_shfl_up(const RB& x, int o) {
  return RB{__shfl_up_sync(FULL, x.nh, o), __shfl_up_sync(FULL, x.f, o), __shfl_up_sync(FULL, x.len, o), 0u,
            __shfl_up_sync(FULL, x.sum, o)};
}
using RBStatus = TileStatus<6>;

template <typename KeyT, int IPT>
__global__ void __launch_bounds__(256) rbk_kernel(const KeyT* __restrict__ keys, const uint32_t* __restrict__ w,
                                                 uint32_t n, int shift, unsigned long long* __restrict__ okeys,
                                                 uint32_t* __restrict__ olen, unsigned long long* __restrict__ osum,
                                                 RBStatus* status, uint32_t epoch, uint32_t* __restrict__ tile_counter,
                                                 uint32_t* __restrict__ d_count) {
  constexpr int TILE = 256 * IPT;
  __shared__ __align__(16) uint64_t sk[TILE + TILE / 16];
  __shared__ RB sm[kWarps + 1];
  __shared__ RB s_excl;
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prev, s_next;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * TILE;
  const uint32_t cnt = (uint32_t)umin64(TILE, (uint64_t)n - t0);
  const bool last_tile = t0 + cnt == n;
  for (int j = 0; j < IPT; ++j) {
    const uint32_t i = j * 256 + tid;
    if (i < cnt) sk[pad16(i)] = (uint64_t)keys[t0 + i] >> shift;
  }
  if (tid == 0) {
    const uint64_t k0 = (uint64_t)keys[t0] >> shift;
    s_prev = t0 ? ((uint64_t)keys[t0 - 1] >> shift) : ~k0;
    s_next = last_tile ? 0 : ((uint64_t)keys[t0 + cnt] >> shift);
  }
  __syncthreads();
  const uint32_t i0 = tid * IPT;
  uint64_t prev = i0 == 0 ? s_prev : (i0 < cnt ? sk[pad16(i0 - 1)] : 0);
  const uint64_t prev0 = prev;
  RB agg = RB::identity();
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      const uint64_t k = sk[pad16(i)];
      const uint32_t h = k != prev;
      agg = rb_combine(agg, RB{h, h, 1u, 0u, w ? (unsigned long long)w[t0 + i] : 1ull});
      prev = k;
    }
  }
  RB total;
  const RB pre = block_excl_scan_op<RB, rb_combine, rb_shfl_up>(agg, sm, &total);
  if (tid == 0) {
    RBStatus* my = status + tile;
    RB ex = RB::identity();
    if (tile == 0) {
      publish<RB, 6>(my, total, epoch, true);
    } else {
      publish<RB, 6>(my, total, epoch, false);
      ex = lookback_op<RB, 6, rb_combine>(status, tile, epoch);
      publish<RB, 6>(my, rb_combine(ex, total), epoch, true);
    }
    s_excl = ex;
    if (last_tile) *d_count = ex.nh + total.nh;
  }
  __syncthreads();
  RB run = rb_combine(s_excl, pre);
  const uint64_t snext = s_next;
  prev = prev0;
  auto emit = [&](uint64_t key, const RB& r) {
    const uint32_t j = r.nh - 1;
    okeys[j] = key;
    if (olen) olen[j] = r.len;
    if (osum) osum[j] = r.sum;
  };
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t i = i0 + q;
    if (i < cnt) {
      const uint64_t k = sk[pad16(i)];
      const uint32_t h = k != prev;
      if (h && i != 0) emit(prev, run);
      run = rb_combine(run, RB{h, h, 1u, 0u, w ? (unsigned long long)w[t0 + i] : 1ull});
      if (i == cnt - 1 && (last_tile || snext != k)) emit(k, run);
      prev = k;
    }
  }
}

// CSR -> per-nonzero row ids (np.repeat(arange(dim), diff(row_ptr)), traffic.py:268)
// plus u32 column/value columns for the column grouping
__global__ void csr_expand_kernel(const long long* __restrict__ row_ptr, uint64_t dim, const long long* __restrict__ col,
                                  const long long* __restrict__ val, uint64_t nnz, uint32_t* __restrict__ rows,
                                  uint32_t* __restrict__ ck, uint32_t* __restrict__ cv) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = dim;  // last r with row_ptr[r] <= k
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if ((uint64_t)row_ptr[mid] <= k)
        lo = mid;
      else
        hi = mid - 1;
    }
    rows[k] = (uint32_t)lo;
    ck[k] = (uint32_t)col[k];
    cv[k] = (uint32_t)val[k];
  }
}

// dense row_ptr of one window's slice of the packed COO (traffic.py:210-211)
__global__ void coo_rowptr_kernel(const uint64_t* __restrict__ keys, uint64_t lo, uint64_t hi, uint64_t wbase,
                                  int b, uint64_t dim, long long* __restrict__ row_ptr) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= dim; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t target = wbase + (r << b);  // r == 2^b reaches the next window
    uint64_t a = lo, z = hi;  // first index with key >= target
    while (a < z) {
      const uint64_t mid = (a + z) >> 1;
      if (keys[mid] < target)
        a = mid + 1;
      else
        z = mid;
    }
    row_ptr[r] = (long long)(a - lo);
  }
}

}  // namespace nmx
