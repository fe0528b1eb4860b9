// nmx_device.cuh -- device primitives shared by the traffic-matrix kernels (sm_100a).
//
// Everything here is integer work: warp ballots for digit multisplit, block
// scans, and the tile-status words of the decoupled-lookback scans.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nmx {

// stream-ordered store of a host-known count into device memory
__global__ void set_u64_kernel(unsigned long long* p, unsigned long long v) { *p = v; }

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;  // every tile kernel runs 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
static_assert(kRadix == kThreads, "one thread per digit in the lookback/scan phases");

// ---------------------------------------------------------------------------
// synthetic packet generators; identical integer functions in
// oracle/netmeter_oracle.py (gen_uniform / gen_powerlaw) and oracle/nmx_oracle.c
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint32_t octave32(uint64_t bits) {
  uint32_t e = (uint32_t)(bits >> 59);
  uint64_t rank = (1ull << e) | (bits & ((1ull << e) - 1));
  return (uint32_t)(rank * 0x9E3779B1ull);
}
__host__ __device__ __forceinline__ uint32_t scale32(uint32_t v, uint64_t space) {
  return space == (1ull << 32) ? v : (uint32_t)(((uint64_t)v * space) >> 32);
}

// ---------------------------------------------------------------------------
// lane / memory-order helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp-aggregated shared-memory counters for skewed (power-law) tiles: when all
// 32 lanes of a round carry the same bin (a tile of one heavy source or
// destination) one lane adds 32; otherwise every lane adds its own 1 (no extra
// dependency on the uniform path). Must be called by all 32 lanes; bin < 0 =
// no item. agg_rank returns the lane's rank within its bin.
// Cheap per-warp skew probe (one round): at least half the lanes share lane
// 0's bin. Only skewed warps pay for the per-round uniformity checks below.
__device__ __forceinline__ bool warp_skewed(int bin) {
  const int b0 = __shfl_sync(FULL, bin, 0);
  return b0 >= 0 && __popc(__ballot_sync(FULL, bin == b0)) >= 16;
}
__device__ __forceinline__ uint32_t agg_rank(uint32_t* cnt, int bin) {
  const int b0 = __shfl_sync(FULL, bin, 0);
  if (__all_sync(FULL, bin == b0) && b0 >= 0) {
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&cnt[b0], 32u);
    return __shfl_sync(FULL, base, 0) + (uint32_t)lane;
  }
  return bin >= 0 ? atomicAdd(&cnt[bin], 1u) : 0u;
}
__device__ __forceinline__ void agg_count(uint32_t* cnt, int bin) {
  const int b0 = __shfl_sync(FULL, bin, 0);
  if (__all_sync(FULL, bin == b0)) {
    if (b0 >= 0 && (threadIdx.x & 31) == 0) atomicAdd(&cnt[b0], 32u);
  } else if (bin >= 0) {
    atomicAdd(&cnt[bin], 1u);
  }
}
// + a 32-bit value per item (final column level: packet sums per destination; the
// sums stay below 2^32 since a call holds < 2^32 packets)
__device__ __forceinline__ void agg_count_sum(uint32_t* cnt, uint32_t* sum, int bin, uint32_t v) {
  const int b0 = __shfl_sync(FULL, bin, 0);
  if (__all_sync(FULL, bin == b0)) {
    if (b0 < 0) return;
    uint32_t x = v;
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&cnt[b0], 32u);
      atomicAdd(&sum[b0], x);
    }
  } else if (bin >= 0) {
    atomicAdd(&cnt[bin], 1u);
    atomicAdd(&sum[bin], v);
  }
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, 1-D) completing on a shared-memory mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// generic-proxy accesses to shared memory before this point are ordered before later
// async-proxy (bulk copy) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared, bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Tile status word for single-value lookback scans:
//   [63:42] epoch (22 bits, never 0 once written) | [41:40] flag | [39:0] value
// The epoch tag lets one status array serve every pass without a memset: a
// word whose epoch differs from the current launch's reads as "not ready".
constexpr uint64_t kFlagAgg = 1, kFlagInc = 2;
constexpr uint64_t kValueMask = (1ull << 40) - 1;
__device__ __forceinline__ uint64_t st_pack(uint32_t epoch, uint64_t flag, uint64_t v) {
  return ((uint64_t)epoch << 42) | (flag << 40) | (v & kValueMask);
}
__device__ __forceinline__ uint32_t st_epoch(uint64_t w) { return (uint32_t)(w >> 42); }
__device__ __forceinline__ uint64_t st_flag(uint64_t w) { return (w >> 40) & 3; }
__device__ __forceinline__ uint64_t st_value(uint64_t w) { return w & kValueMask; }

// Exclusive prefix over predecessors of `tile` for one lane of a lookback
// (status row stride `stride` words, column `col`). Spins until ready.
constexpr unsigned kLookbackBackoffNs = 64;
// Four predecessors are loaded per round (independent loads in flight) and consumed
// in order, so a chain of aggregate-only predecessors costs a quarter of the
// dependent L2 round trips of a one-word walk.
__device__ __forceinline__ uint64_t lookback_exclusive(const uint64_t* status, uint32_t tile, int stride, int col,
                                                       uint32_t epoch) {
  constexpr int V = 4;
  uint64_t excl = 0;
  int64_t p = (int64_t)tile - 1;
  while (p >= 0) {
    uint64_t w[V];
#pragma unroll
    for (int j = 0; j < V; ++j) w[j] = p - j >= 0 ? ld_relaxed(status + (size_t)(p - j) * stride + col) : 0ull;
    int adv = 0;
    bool done = false;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (done || adv != j) continue;  // stopped earlier in this round
      if (p - j < 0) {
        done = true;
      } else if (st_epoch(w[j]) == epoch) {
        excl += st_value(w[j]);
        adv = j + 1;
        if (st_flag(w[j]) == kFlagInc) done = true;
      }  // else: not published yet -- re-poll from p - j
    }
    if (done) break;
    if (!adv) __nanosleep(kLookbackBackoffNs);  // nothing published yet: yield the issue slots
    p -= adv;
  }
  return excl;
}

// Warp-cooperative lookback (every lane calls it with the same tile / column): lane
// l reads predecessor p - l, so one round covers 32 predecessors; the prefix stops at
// the nearest inclusive word or before the nearest unpublished one.
__device__ __forceinline__ uint64_t lookback_exclusive_warp(const uint64_t* status, uint32_t tile, int stride, int col,
                                                            uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t p = (int64_t)tile - 1;
  while (p >= 0) {
    const int64_t q = p - lane;
    const uint64_t w = q >= 0 ? ld_relaxed(status + (size_t)q * stride + col) : st_pack(epoch, kFlagInc, 0);
    const bool ready = st_epoch(w) == epoch;
    const uint32_t notready = __ballot_sync(FULL, !ready);
    const uint32_t inc = __ballot_sync(FULL, ready && st_flag(w) == kFlagInc);
    const int first_nr = notready ? __ffs(notready) - 1 : 32;
    const int first_inc = inc ? __ffs(inc) - 1 : 32;
    const int take = first_inc < first_nr ? first_inc + 1 : first_nr;  // lanes [0, take) are consumed
    uint64_t v = lane < take ? st_value(w) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    excl += v;
    if (first_inc < first_nr) break;
    if (!take) __nanosleep(kLookbackBackoffNs);
    p -= take;
  }
  return excl;
}

// Segmented-carry status (reduce-by-segment across tiles). The AGG and INC
// payloads live in separate words so a reader that saw flag == AGG can never
// pick up INC data written later (the data words are never rewritten within
// one epoch); the flag word is stored last with release semantics.
struct CarryStatus {
  uint64_t agg_len, agg_sum;
  uint64_t inc_len, inc_sum;
  uint64_t flag;  // epoch << 2 | {1 = AGG, 2 = INC}
  uint64_t pad[3];
};

// ---------------------------------------------------------------------------
// block scans (256 threads)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Exclusive block scan of one value per thread; returns the exclusive prefix,
// writes the block total to *total. `wtot` is kWarps words of shared memory.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T x, T* wtot, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(x, lane);
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T v = lane < kWarps ? wtot[lane] : T(0);
    T vi = warp_incl_scan(v, lane);
    if (lane < kWarps) wtot[lane] = vi - v;  // exclusive warp offsets
    if (lane == kWarps - 1) wtot[kWarps] = vi;
  }
  __syncthreads();
  T res = wtot[warp] + inc - x;
  *total = wtot[kWarps];
  __syncthreads();
  return res;
}

// Segmented scan element: f = a segment head occurred, (len, sum) = partial
// since the last head (or since the start when f == 0).
struct Seg {
  uint32_t f;
  uint32_t len;
  uint64_t sum;
};
__device__ __forceinline__ Seg seg_combine(const Seg& a, const Seg& b) {
  Seg r;
  r.f = a.f | b.f;
  r.len = b.f ? b.len : a.len + b.len;
  r.sum = b.f ? b.sum : a.sum + b.sum;
  return r;
}

// Exclusive segmented block scan; `sm` holds kWarps+1 Seg. Returns exclusive
// prefix for this thread; *total = inclusive total of the block.
__device__ __forceinline__ Seg block_excl_segscan(Seg x, Seg* sm, Seg* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Seg inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg y;
    y.f = __shfl_up_sync(FULL, inc.f, o);
    y.len = __shfl_up_sync(FULL, inc.len, o);
    y.sum = __shfl_up_sync(FULL, inc.sum, o);
    if (lane >= o) inc = seg_combine(y, inc);
  }
  Seg ex;
  ex.f = __shfl_up_sync(FULL, inc.f, 1);
  ex.len = __shfl_up_sync(FULL, inc.len, 1);
  ex.sum = __shfl_up_sync(FULL, inc.sum, 1);
  if (lane == 0) ex = Seg{0, 0, 0};
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Seg run{0, 0, 0};
    for (int w = 0; w < kWarps; ++w) {
      Seg t = sm[w];
      sm[w] = run;
      run = seg_combine(run, t);
    }
    sm[kWarps] = run;
  }
  __syncthreads();
  Seg res = seg_combine(sm[warp], ex);
  *total = sm[kWarps];
  __syncthreads();
  return res;
}

// Peers of this lane's 8-bit digit within the warp via 8 ballots (warp
// multisplit). MATCH.ANY measured ~60 cycles/instr/SM on B200 (profiles/
// r01_device_probe.txt), so ballots are the ranking primitive here.
__device__ __forceinline__ uint32_t warp_digit_peers(uint32_t d, bool ok) {
  uint32_t peers = __ballot_sync(FULL, ok);
#pragma unroll
  for (int b = 0; b < kRadixBits; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(FULL, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

}  // namespace nmx
