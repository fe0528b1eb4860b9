// nmx_api.cu -- context, workspace and the C ABI of libnmx.so (include/nmx.h).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened at run time (nccl_api)

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>
#include <immintrin.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <chrono>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/nmx.h"
#include "nmx_io.cuh"
#include "nmx_merge.cuh"
#include "nmx_text.cuh"
#include "nmx_seg.cuh"

using namespace nmx;

namespace {

thread_local std::string g_err;
thread_local bool g_capturing = false;  // a CUDA graph capture is open on this thread
// bumped whenever a device buffer is freed or moved: recorded graphs hold raw pointers
std::atomic<uint64_t> g_buf_gen{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

struct CudaError {
  cudaError_t e;
  const char* what;
  int line;
};

#define CK(x)                                              \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) throw CudaError{e_, #x, __LINE__}; \
  } while (0)
#define CK_LAUNCH() CK(cudaGetLastError())

constexpr int kIPT = 16;
constexpr int kTile = kThreads * kIPT;  // 4096 items per tile

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  // grow (never shrinks); returns true when (re)allocated (contents undefined / zeroed by caller)
  bool grow(size_t bytes) {
    if (bytes <= cap) return false;
    // a captured node may already point at the old buffer: the capture is abandoned
    if (g_capturing) throw std::runtime_error("buffer growth during graph capture");
    ++g_buf_gen;
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    // 1/8 headroom against regrowth, at most 256 MiB on the multi-GB buffers
    size_t want = std::max<size_t>(bytes + std::min<size_t>(bytes / 8, 256ull << 20), 1 << 16);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      want = bytes;
      CK(cudaMalloc(&p, want));
    }
    cap = want;
    return true;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
  void release() {
    if (p) {
      ++g_buf_gen;
      cudaFree(p);
    }
    p = nullptr;
    cap = 0;
  }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
};

// small device block layout (u32 words)
constexpr int kHist = 0;                    // 8*256 row-pass histograms
constexpr int kBase = kHist + 8 * kRadix;   // 8*256 row-pass bin bases
constexpr int kCHist = kBase + 8 * kRadix;  // 8*256 column-pass histograms
constexpr int kCBase = kCHist + 8 * kRadix; // 8*256 column-pass bin bases
constexpr int kCounters = kCBase + 8 * kRadix;  // 32 tile counters
constexpr int kU = kCounters + 32;          // unique-link count
constexpr int kGCount = kU + 2;             // u64 valid count (8-byte aligned)
constexpr int kSmallWords = kGCount + 2;

uint32_t ceil_log2(uint64_t x) {  // x >= 1
  uint32_t b = 0;
  while ((1ull << b) < x && b < 64) ++b;
  return b;
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  // once per (device, kernel, size): the attribute call costs host time on every launch
  static std::mutex mu;
  static std::map<std::tuple<int, const void*>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[std::make_tuple(dev, reinterpret_cast<const void*>(kernel))];
  if (have >= bytes) return;
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
}

}  // namespace

struct nmx_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t st = nullptr;
  std::mutex mu;
  DevBuf mpcnt, mpoff;  // group pieces (seg_plan_groups_dev with a bucket cap)
  DevBuf parS, parD, pcolD, pcolC;  // out-of-core source / destination part arenas (> 2^31 packets)
  DevBuf mscan, mch, mgh, mplan, keysA, keysB, keysC, keysD, cgk, cgv, cgk2, cgv2, colL_dst, colL_cnt, mcur, moff, mhist2, mgb, mheavy, mdst, ckA, ckB, cvA, cvB, status, lrstatus, csstatus, small, part, rbstatus, mkeys, mlen, msum,
      ckeys2, clen2, csum2, frows, stats, in_src, in_dst, in_valid,
      red, ws0, ws1, wd0, wd1, wv0, wv1, wr0, wr1, rmax, anAk, anAv, anBk, anBv, anHead, anHoff, anDistinct,
      anFirst, anFlag, anFoff, anPerm, anCode, txt, tcnt, toff, tends, tntok, tvals, tnb, tnboff, thdr, tbad, trows,
      tcols, tval, tlen, tloff, msplit, lightK, lightCK, lightCV, sccnt, scur, sloff, spoffA, spoffB, srep, ssum, sbsum, sbflag, stot, gsk, gsv,
      hcount;
  uint32_t epoch = 0;
  cudaStream_t st2 = nullptr;  // copy stream of the streamed path
  cudaEvent_t evc[2] = {nullptr, nullptr}, evu[2] = {nullptr, nullptr}, evs = nullptr;
  // nmx_stats9_host_batches: two device input slots, copy-done / slot-free events
  DevBuf bat_s[2], bat_d[2], bat_v[2];
  DevBuf mhist3;  // level-3 counts of msd_count23_kernel
  DevBuf moff1;   // level-1 offsets kept for the positional levels of narrowed column items
  DevBuf mtpar;   // per-tile parents of those levels (tile_parents_kernel)
  cudaEvent_t evbc[2] = {nullptr, nullptr}, evbu[2] = {nullptr, nullptr};
  uint32_t* h_small = nullptr;  // pinned mirror of `small`
  unsigned long long* h_scr = nullptr;  // pinned scalars read back mid-pipeline (one round trip each)
  unsigned long long* scr() {
    if (!h_scr) CK(cudaMallocHost(&h_scr, 64 * sizeof(unsigned long long)));
    return h_scr;
  }
  unsigned long long* h_stats = nullptr;
  size_t h_stats_cap = 0;
  void* h_wide = nullptr;  // pinned u32 / u8 slots of the int64-column entry
  size_t wide_cap = 0;
  cudaEvent_t ev[40];
  int nev = 0;
  // deferred partition read-back (msd_partition(defer) -> msd_partition_wait)
  cudaEvent_t evw = nullptr;
  bool joint_ready = false;  // streamed windows left the level-2 counts in mhist2
  int scr_off = 0;            // scr() slots of the pending partition read-back (rows 0, columns 8)
  // CUDA graphs of whole small calls (run_pipeline_msd_graph), keyed by inputs and size
  struct CallGraph {
    const void *s, *d, *v;
    uint64_t n, space;
    uint64_t window;  // 0: summed matrix; else the per-window statistics of windows of this size
    cudaGraphExec_t exec;
    uint64_t gen;  // g_buf_gen when recorded
    int launches;  // kernels in the graph
  };
  std::vector<CallGraph> graphs;
  bool capturing = false;
  bool had_heavy = false;  // the last call sent buckets through the segmented levels
  uint64_t pend_bytes_per_m = 0;
  int pend_L = 0;
  float last_total_ms = 0, last_sort_ms = 0;
  float last_stage_ms[8] = {0};
  int last_nstage = 0;
  int last_sort_launches = 0, last_launches = 0;
  int launches = 0;
  // materialised outputs (drop-in TrafficMatrix / FlatContainers)
  uint64_t coo_nnz = 0, flat_nnz = 0, flat_r = 0, flat_c = 0;
  int coo_b = 0;
  int msd_levels = 0;
  // anonymize state between nmx_anonymize_begin and nmx_anonymize_finish
  uint64_t an_m = 0, an_k = 0;
  const uint32_t* an_pos = nullptr;

  uint32_t next_epoch() {
    if (++epoch >= (1u << 22)) {
      if (status.p) CK(cudaMemsetAsync(status.p, 0, status.cap, st));
      if (lrstatus.p) CK(cudaMemsetAsync(lrstatus.p, 0, lrstatus.cap, st));
      if (csstatus.p) CK(cudaMemsetAsync(csstatus.p, 0, csstatus.cap, st));
      epoch = 1;
    }
    return epoch;
  }
  void grow_status(size_t tiles_x_cols) {
    if (status.grow(tiles_x_cols * sizeof(uint64_t))) CK(cudaMemsetAsync(status.p, 0, status.cap, st));
  }
  void grow_hstats(size_t words) {
    if (words <= h_stats_cap) return;
    ++g_buf_gen;
    if (h_stats) cudaFreeHost(h_stats);
    h_stats = nullptr;
    CK(cudaMallocHost(&h_stats, words * sizeof(unsigned long long)));
    h_stats_cap = words;
  }
  void mark() {
    if (!capturing) CK(cudaEventRecord(ev[nev++], st));
  }
  // dominant-kernel accounting (event pairs around each launch of the class)
  cudaEvent_t evk[64];
  int nevk = 0;
  uint64_t dom_bytes = 0;
  float dom_ms = 0;
  int dom_launches = 0;
  const char* dom_name = "";
  bool dom_cur = false;
  // the first kernel class that reports in a call owns the accounting
  void dom_begin(const char* nm) {
    if (capturing) {
      dom_cur = false;
      return;
    }
    if (!dom_name[0]) dom_name = nm;
    dom_cur = strcmp(dom_name, nm) == 0 && nevk + 2 <= 64;
    if (dom_cur) CK(cudaEventRecord(evk[nevk], st));
  }
  // per launch: algorithmic bytes (known now, or bytes per valid item `bpi` resolved
  // when the partition's valid count comes back) and the event-pair time
  uint64_t dom_lbytes[32] = {};
  uint32_t dom_lbpi[32] = {};
  float dom_lms[32] = {};
  void dom_end(uint64_t bytes, uint32_t bpi = 0) {
    if (!dom_cur) return;
    CK(cudaEventRecord(evk[nevk + 1], st));
    dom_lbytes[nevk / 2] = bytes;
    dom_lbpi[nevk / 2] = bpi;
    nevk += 2;
    dom_bytes += bytes;
    ++dom_launches;
  }
  void dom_resolve(uint64_t m) {  // launches waiting for their item count
    for (int k = 0; k < nevk / 2; ++k)
      if (dom_lbpi[k] && !dom_lbytes[k]) dom_lbytes[k] = (uint64_t)dom_lbpi[k] * m;
  }
};

// device-resident sorted unique COO: keys (src<<32)|dst, u64 counts in [1, 2^63)
// (the reference's int64 matrix values, traffic.py:140-194)
struct nmx_coo {
  int device = 0;
  uint64_t nnz = 0;
  uint64_t* keys = nullptr;
  uint64_t* counts = nullptr;
};

extern "C" nmx_coo* coo_alloc(nmx_ctx* c, uint64_t nnz);  // stream-ordered COO storage (below)

namespace {

uint64_t tiles_of(uint64_t items, int tile = kTile) { return (items + tile - 1) / tile; }

// onesweep pass configurations (THREADS, IPT, ranking, min blocks/SM); the
// default was picked by the sweep in profiles/ (NMX_PASS_VARIANT overrides).
constexpr int kDefaultVariant = 5;
constexpr int kMinPassTile = 2048;  // smallest THREADS*IPT among the variants
int pass_variant() {
  static const int v = [] {
    const char* e = getenv("NMX_PASS_VARIANT");
    return e ? atoi(e) : kDefaultVariant;
  }();
  return v;
}

template <typename Src, typename KeyT, bool HAS_VAL, int THREADS, int IPT, int RANK, int MINB>
void launch_pass_v(nmx_ctx* c, const Src& src, uint64_t items, KeyT* out, uint32_t* vout, int shift,
                   const uint32_t* binbase, uint32_t* counter) {
  using S = PassSmem<KeyT, HAS_VAL, THREADS, IPT>;
  auto kern = onesweep_pass<Src, KeyT, HAS_VAL, THREADS, IPT, RANK, MINB>;
  set_smem(kern, sizeof(S));
  const uint64_t t = tiles_of(items, THREADS * IPT);
  if (!t) return;
  c->dom_begin("onesweep_pass");
  kern<<<(unsigned)t, THREADS, sizeof(S), c->st>>>(src, out, vout, shift, binbase, c->status.as<uint64_t>(),
                                                     c->next_epoch(), counter);
  CK_LAUNCH();
  c->dom_end(items * 2 * (sizeof(KeyT) + (HAS_VAL ? 4 : 0)));
  ++c->launches;
}

template <typename Src, typename KeyT, bool HAS_VAL>
void launch_pass(nmx_ctx* c, const Src& src, uint64_t items, KeyT* out, uint32_t* vout, int shift,
                 const uint32_t* binbase, uint32_t* counter) {
#define NMX_PV(T, I, R, M) \
  launch_pass_v<Src, KeyT, HAS_VAL, T, I, R, M>(c, src, items, out, vout, shift, binbase, counter)
  switch (pass_variant()) {
    case 1: NMX_PV(256, 16, RANK_ATOMIC_OR, 1); break;
    case 2: NMX_PV(256, 8, RANK_BALLOT, 3); break;
    case 3: NMX_PV(256, 8, RANK_ATOMIC_OR, 3); break;
    case 4: NMX_PV(512, 8, RANK_BALLOT, 2); break;
    case 5: NMX_PV(512, 8, RANK_ATOMIC_OR, 2); break;
    case 6: NMX_PV(256, 12, RANK_BALLOT, 2); break;
    case 7: NMX_PV(256, 12, RANK_ATOMIC_OR, 2); break;
    case 0: NMX_PV(256, 16, RANK_BALLOT, 1); break;
    default: NMX_PV(512, 8, RANK_ATOMIC_OR, 2); break;
  }
#undef NMX_PV
}

constexpr int kSegIPT = 8;  // link_row / col kernels: 2048 items per tile
constexpr int kSegTile = 256 * kSegIPT;

// LSD onesweep sort of u entries (ColKeyT keys in ckA, u32 values in cvA; their
// digit histograms already in small[kCHist]) -> sorted pointers.
template <typename ColKeyT>
std::pair<ColKeyT*, uint32_t*> sort_col_entries(nmx_ctx* c, uint32_t u, int nbits, uint32_t* d_small) {
  const int ncolpass = (nbits + 7) / 8;
  ColKeyT* ck = c->ckA.as<ColKeyT>();
  uint32_t* cv = c->cvA.as<uint32_t>();
  bin_scan_kernel<<<1, 256, 0, c->st>>>(d_small + kCHist, ncolpass, d_small + kCBase);
  CK_LAUNCH();
  ++c->launches;
  CK(cudaMemcpyAsync(c->h_small + kCHist, d_small + kCHist, sizeof(uint32_t) * ncolpass * kRadix,
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->grow_status(tiles_of(u, kMinPassTile) * kRadix);
  int idx = 0;
  for (int p = 0; p < ncolpass; ++p) {
    const uint32_t* hp = c->h_small + kCHist + p * kRadix;
    bool trivial = false;
    for (int d = 0; d < kRadix; ++d)
      if (hp[d] == u) trivial = true;
    if (trivial) continue;
    ColKeyT* ok = (idx & 1) ? c->ckA.as<ColKeyT>() : c->ckB.as<ColKeyT>();
    uint32_t* ov = (idx & 1) ? c->cvA.as<uint32_t>() : c->cvB.as<uint32_t>();
    KeySrc<ColKeyT, true> src{ck, cv, u};
    launch_pass<KeySrc<ColKeyT, true>, ColKeyT, true>(c, src, u, ok, ov, 8 * p, d_small + kCBase + p * kRadix,
                                                      d_small + kCounters + 16 + idx);
    ck = ok;
    cv = ov;
    ++idx;
  }
  return {ck, cv};
}

template <typename ColKeyT>
void column_phase(nmx_ctx* c, uint32_t u, int b, int wb, uint32_t* d_small) {
  auto sorted = sort_col_entries<ColKeyT>(c, u, b + wb, d_small);
  c->mark();  // column sort end
  col_kernel<ColKeyT, kSegIPT><<<(unsigned)tiles_of(u, kSegTile), 256, 0, c->st>>>(
      sorted.first, sorted.second, u, b, wb, c->csstatus.as<CSStatus>(), c->next_epoch(), d_small + kCounters + 26,
      c->stats.as<unsigned long long>());
  CK_LAUNCH();
  ++c->launches;
}

template <typename ColKeyT>
void launch_link_row(nmx_ctx* c, const uint64_t* keys, uint32_t m, int b, int wb, uint32_t* d_small) {
  const int ncolpass = (b + wb + 7) / 8;
  link_row_kernel<ColKeyT, kSegIPT><<<(unsigned)tiles_of(m, kSegTile), 256, 0, c->st>>>(
      keys, m, b, wb, c->ckA.as<ColKeyT>(), c->cvA.as<uint32_t>(), ncolpass, d_small + kCHist,
      c->lrstatus.as<LRStatus>(), c->next_epoch(), d_small + kCounters + 25, c->stats.as<unsigned long long>(),
      d_small + kU);
  CK_LAUNCH();
  ++c->launches;
}

template <typename Src>
void launch_hist(nmx_ctx* c, const Src& ps, int npass, uint32_t* d_small) {
  const uint64_t want = (ps.n + 1023) / 1024;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)c->sms * 8));
  auto* gcount = reinterpret_cast<unsigned long long*>(d_small + kGCount);
  switch (npass) {
#define NMX_HCASE(P) \
  case P: hist_kernel<Src, P><<<grid, 256, 0, c->st>>>(ps, d_small + kHist, gcount); break;
    NMX_HCASE(1) NMX_HCASE(2) NMX_HCASE(3) NMX_HCASE(4) NMX_HCASE(5) NMX_HCASE(6) NMX_HCASE(7) NMX_HCASE(8)
#undef NMX_HCASE
    default: throw std::runtime_error("bad pass count");
  }
  CK_LAUNCH();
  ++c->launches;
}

// ---- pipeline stages -------------------------------------------------------
void stage_begin(nmx_ctx* c, uint64_t W) {
  c->nev = 0;
  c->nevk = 0;
  c->dom_bytes = 0;
  c->dom_ms = 0;
  c->dom_launches = 0;
  c->dom_name = "";
  c->launches = 0;
  c->last_sort_launches = 0;
  c->last_sort_ms = 0;
  c->had_heavy = false;
  c->small.grow(kSmallWords * sizeof(uint32_t));
  if (!c->h_small) CK(cudaMallocHost(&c->h_small, kSmallWords * sizeof(uint32_t)));
  c->stats.grow(W * S_COUNT * sizeof(unsigned long long));
  c->grow_hstats(W * S_COUNT);
  c->mark();  // 0: start
  CK(cudaMemsetAsync(c->small.p, 0, kSmallWords * sizeof(uint32_t), c->st));
  CK(cudaMemsetAsync(c->stats.p, 0, W * S_COUNT * sizeof(unsigned long long), c->st));
}

void stage_finish(nmx_ctx* c, uint64_t W) {
  CK(cudaMemcpyAsync(c->h_stats, c->stats.p, W * S_COUNT * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     c->st));
  if (c->capturing) return;  // a graph replay is timed and waited on by its caller
  c->mark();  // end
  CK(cudaStreamSynchronize(c->st));
  CK(cudaEventElapsedTime(&c->last_total_ms, c->ev[0], c->ev[c->nev - 1]));
  if (c->nev >= 3 && c->last_sort_launches) CK(cudaEventElapsedTime(&c->last_sort_ms, c->ev[1], c->ev[2]));
  c->last_nstage = 0;
  for (int i = 0; i + 1 < c->nev && i < 8; ++i) CK(cudaEventElapsedTime(&c->last_stage_ms[i], c->ev[i], c->ev[i + 1]));
  c->last_nstage = std::min(c->nev - 1, 8);
  c->last_launches = c->launches;
  c->dom_ms = 0;
  for (int i = 0; i + 1 < c->nevk; i += 2) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, c->evk[i], c->evk[i + 1]));
    c->dom_ms += t;
    c->dom_lms[i / 2] = t;
  }
}

struct RowsOut {
  uint64_t m;  // valid packets
  uint32_t u;  // unique links (column entries in ckA/cvA, link order)
  bool wide;   // column keys are u64
};

// hist -> onesweep row sort -> fused link/row kernel. Link + row statistics
// accumulate into c->stats; the column entries are left in c->ckA / c->cvA.
bool sort_rows_msd(nmx_ctx* c, const PacketSrc& ps, int kb, uint64_t* m_out, uint64_t** keys_out);
// the packed keys of the valid packets, fully sorted (m valid): the MSD partition +
// per-group shared-memory sort when the inputs allow it, else the LSD onesweep passes.
// kb_used: key bits that can be nonzero (default 2b + wb)
uint64_t* sort_rows(nmx_ctx* c, const PacketSrc& ps, int b, int wb, uint64_t* m_out, int kb_used = 0) {
  {
    uint64_t* k = nullptr;
    if (sort_rows_msd(c, ps, kb_used ? kb_used : 2 * b + wb, m_out, &k)) return k;
  }
  const uint64_t n = ps.n;
  const int kb = 2 * b + wb;
  const int npass = (kb + 7) / 8;
  uint32_t* d_small = c->small.as<uint32_t>();
  launch_hist(c, ps, npass, d_small);
  bin_scan_kernel<<<1, 256, 0, c->st>>>(d_small + kHist, npass, d_small + kBase);
  CK_LAUNCH();
  ++c->launches;
  CK(cudaMemcpyAsync(c->h_small, d_small, kSmallWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const uint64_t m = *reinterpret_cast<unsigned long long*>(c->h_small + kGCount);
  *m_out = m;
  if (m == 0) return nullptr;
  if (m >= (1ull << 32)) throw std::runtime_error("more than 2^32-1 valid packets in one call");

  std::vector<int> active;
  for (int p = 0; p < npass; ++p) {
    const uint32_t* hp = c->h_small + kHist + p * kRadix;
    bool trivial = false;
    for (int d = 0; d < kRadix; ++d)
      if (hp[d] == m) trivial = true;
    if (!trivial) active.push_back(p);
  }
  if (active.empty()) active.push_back(0);  // still need one pass to pack the keys
  c->keysA.grow(m * 8);
  c->keysB.grow(m * 8);
  c->grow_status(tiles_of(std::max(n, m), kMinPassTile) * kRadix);
  c->mark();  // 1: sort start
  uint64_t* keys = nullptr;
  for (size_t i = 0; i < active.size(); ++i) {
    const int p = active[i];
    uint64_t* out = (i & 1) ? c->keysB.as<uint64_t>() : c->keysA.as<uint64_t>();
    if (i == 0) {
      launch_pass<PacketSrc, uint64_t, false>(c, ps, n, out, nullptr, 8 * p, d_small + kBase + p * kRadix,
                                              d_small + kCounters + i);
    } else {
      KeySrc<uint64_t, false> ks{keys, nullptr, m};
      launch_pass<KeySrc<uint64_t, false>, uint64_t, false>(c, ks, m, out, nullptr, 8 * p,
                                                            d_small + kBase + p * kRadix, d_small + kCounters + i);
    }
    keys = out;
  }
  c->last_sort_launches = (int)active.size();
  c->mark();  // 2: sort end
  return keys;
}

RowsOut stage_rows(nmx_ctx* c, const PacketSrc& ps, int b, int wb) {
  uint64_t m = 0;
  uint64_t* keys = sort_rows(c, ps, b, wb, &m);
  const bool wide = b + wb > 32;
  if (m == 0) return RowsOut{0, 0, wide};
  uint32_t* d_small = c->small.as<uint32_t>();
  c->ckA.grow(m * (wide ? 8 : 4));
  c->ckB.grow(m * (wide ? 8 : 4));
  c->cvA.grow(m * 4);
  c->cvB.grow(m * 4);
  if (c->lrstatus.grow(tiles_of(m, kSegTile) * sizeof(LRStatus)))
    CK(cudaMemsetAsync(c->lrstatus.p, 0, c->lrstatus.cap, c->st));
  if (c->csstatus.grow(tiles_of(m, kSegTile) * sizeof(CSStatus)))
    CK(cudaMemsetAsync(c->csstatus.p, 0, c->csstatus.cap, c->st));
  if (wide)
    launch_link_row<uint64_t>(c, keys, (uint32_t)m, b, wb, d_small);
  else
    launch_link_row<uint32_t>(c, keys, (uint32_t)m, b, wb, d_small);
  c->mark();  // 3: link/row end
  CK(cudaMemcpyAsync(c->h_small + kU, d_small + kU, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RowsOut{m, c->h_small[kU], wide};
}

// column sort + column kernel over the u entries in c->ckA / c->cvA (whose
// digit histograms are in small[kCHist]).
void stage_cols(nmx_ctx* c, uint32_t u, int b, int wb, bool wide) {
  if (!u) return;
  uint32_t* d_small = c->small.as<uint32_t>();
  c->grow_status(tiles_of(u, kMinPassTile) * kRadix);
  if (wide)
    column_phase<uint64_t>(c, u, b, wb, d_small);
  else
    column_phase<uint32_t>(c, u, b, wb, d_small);
}

// reduce-by-key launch; returns the number of segments (host sync)
template <typename KeyT>
uint32_t run_rbk(nmx_ctx* c, const KeyT* keys, const uint32_t* w, uint32_t n, int shift, unsigned long long* okeys,
                 uint32_t* olen, unsigned long long* osum, int counter) {
  if (!n) return 0;
  uint32_t* d_small = c->small.as<uint32_t>();
  if (c->rbstatus.grow(tiles_of(n, kSegTile) * sizeof(RBStatus)))
    CK(cudaMemsetAsync(c->rbstatus.p, 0, c->rbstatus.cap, c->st));
  rbk_kernel<KeyT, kSegIPT><<<(unsigned)tiles_of(n, kSegTile), 256, 0, c->st>>>(
      keys, w, n, shift, okeys, olen, osum, c->rbstatus.as<RBStatus>(), c->next_epoch(), d_small + kCounters + counter,
      d_small + kU);
  CK_LAUNCH();
  ++c->launches;
  uint32_t r = 0;
  CK(cudaMemcpyAsync(&r, d_small + kU, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return r;
}

// ---- MSD partition + shared-memory grouping (nmx_msd.cuh) -------------------
// used for the summed matrix when 2^20 <= n <= 2^30 and the D MSD bits are all
// source bits; NMX_PATH=lsd forces the LSD path.
int msd_bits(uint64_t n, int b) {
  const char* e = getenv("NMX_PATH");
  if (e && std::string(e) == "lsd") return 0;
  // positions carry a light flag in bit 31 (nmx_seg.cuh): at most 2^31 keys; from
  // 2^16 packets the MSD path (fewer host round trips) beats the LSD sort
  if (n < (1ull << 16) || n > (1ull << 31)) return 0;
  const int D = std::min(22, std::max(11, (int)ceil_log2(n) - 9));
  return D <= b ? D : 0;
}

// LSD onesweep sort of n (u32 key, u32 value) pairs (nbits significant key bits)
std::pair<uint32_t*, uint32_t*> sort_u32_pairs(nmx_ctx* c, uint32_t* k, uint32_t* v, uint64_t n, int nbits,
                                               uint32_t* k2, uint32_t* v2) {
  uint32_t* d_small = c->small.as<uint32_t>();
  const int npass = (nbits + 7) / 8;
  CK(cudaMemsetAsync(d_small + kCHist, 0, sizeof(uint32_t) * 8 * kRadix, c->st));
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 1023) / 1024, (uint64_t)c->sms * 8));
  switch (npass) {
    case 1: hist_u32_kernel<1><<<grid, 256, 0, c->st>>>(k, n, d_small + kCHist); break;
    case 2: hist_u32_kernel<2><<<grid, 256, 0, c->st>>>(k, n, d_small + kCHist); break;
    case 3: hist_u32_kernel<3><<<grid, 256, 0, c->st>>>(k, n, d_small + kCHist); break;
    default: hist_u32_kernel<4><<<grid, 256, 0, c->st>>>(k, n, d_small + kCHist); break;
  }
  CK_LAUNCH();
  bin_scan_kernel<<<1, 256, 0, c->st>>>(d_small + kCHist, npass, d_small + kCBase);
  CK_LAUNCH();
  CK(cudaMemcpyAsync(c->h_small + kCHist, d_small + kCHist, sizeof(uint32_t) * npass * kRadix, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  c->grow_status(tiles_of(n, kMinPassTile) * kRadix);
  int idx = 0;
  for (int p = 0; p < npass; ++p) {
    const uint32_t* hp = c->h_small + kCHist + p * kRadix;
    bool trivial = false;
    for (int d = 0; d < kRadix; ++d)
      if (hp[d] == n) trivial = true;
    if (trivial) continue;
    KeySrc<uint32_t, true> src{k, v, n};
    launch_pass<KeySrc<uint32_t, true>, uint32_t, true>(c, src, n, k2, v2, 8 * p, d_small + kCBase + p * kRadix,
                                                        d_small + kCounters + 16 + idx);
    std::swap(k, k2);
    std::swap(v, v2);
    ++idx;
  }
  return {k, v};
}

// Two-level non-stable MSD partition of the valid items of `src` (kb-bit keys)
// by their top D bits. Leaves bucket offsets in c->moff (2^D + 1 entries) and
// returns the partitioned keys / values and the number of valid items.
// exclusive scan of n counters -> off[0..n] (off[n] = total) and cursor = off
void scan_counts(nmx_ctx* c, const uint32_t* cnt, uint32_t n, uint32_t* off, uint32_t* cursor) {
  if (n <= (uint32_t)kScanItems) {
    scan_small_kernel<<<1, 256, 0, c->st>>>(cnt, n, off, cursor);
    CK_LAUNCH();
    ++c->launches;
    return;
  }
  const uint32_t nb = (n + kScanItems - 1) / kScanItems;
  c->mscan.grow(((size_t)nb + 4) * 4);
  uint32_t* bsum = c->mscan.as<uint32_t>();
  scan_block_sums_kernel<<<nb, 256, 0, c->st>>>(cnt, n, bsum);
  CK_LAUNCH();
  scan_top_kernel<<<1, 1024, 0, c->st>>>(bsum, nb, bsum + nb);
  CK_LAUNCH();
  scan_apply_kernel<<<nb, 256, 0, c->st>>>(cnt, n, bsum, bsum + nb, off, cursor);
  CK_LAUNCH();
  c->launches += 3;
}

// NMX_COUNT23=0 keeps two msd_count2 passes (A/B runs)
bool count23_enabled() {
  static const bool v = [] {
    const char* e = getenv("NMX_COUNT23");
    return !(e && e[0] == '0');
  }();
  return v;
}

int msd_first_bits(int D) {
  const int L = (D + kMsdMaxLevelBits - 1) / kMsdMaxLevelBits;
  return D / L + (0 < D % L ? 1 : 0);
}

// dense scatter launch with the bin capacity of this level's digit width
template <typename Src, typename KeyT, bool HAS_VAL, int LEVEL, bool SPLIT, int NM, int IPT, bool HI>
void launch_msd_scatter_impl(nmx_ctx* c, int dbits, uint64_t tiles, const Src& src, uint64_t n, KeyT* out, uint32_t* vout,
                        int shift, int bshift, uint32_t* cursor, KeyT* hout, uint32_t* hvout,
                        const NarrowArgs& nw) {
  if (dbits > kMsdLevelBits) {
    auto k = msd_scatter_kernel<Src, KeyT, HAS_VAL, LEVEL, SPLIT, kMsdMaxLevelBits, NM, IPT, HI>;
    constexpr size_t sm = sizeof(MsdSmem<KeyT, HAS_VAL, (2 << kMsdMaxLevelBits), kMsdThreads * IPT>);
    set_smem(k, sm);
    k<<<(unsigned)tiles, kMsdThreads, sm, c->st>>>(src, n, out, vout, shift, dbits, bshift, cursor, hout, hvout, nw);
  } else {
    auto k = msd_scatter_kernel<Src, KeyT, HAS_VAL, LEVEL, SPLIT, kMsdLevelBits, NM, IPT, HI>;
    constexpr size_t sm = sizeof(MsdSmem<KeyT, HAS_VAL, (2 << kMsdLevelBits), kMsdThreads * IPT>);
    set_smem(k, sm);
    k<<<(unsigned)tiles, kMsdThreads, sm, c->st>>>(src, n, out, vout, shift, dbits, bshift, cursor, hout, hvout, nw);
  }
}

// later-level u64 keys whose digit / parent fields lie in the high word take the 32-bit
// shift body (level 2: 3.58 / 3.61 -> 3.50 / 3.56 ms; the first levels measured slower
// with it, 3.57 -> 3.76 ms: profiles/r02bz/)
template <typename Src, typename KeyT, bool HAS_VAL, int LEVEL, bool SPLIT = false, int NM = NM_NONE,
          int IPT = kMsdIPT>
void launch_msd_scatter(nmx_ctx* c, int dbits, uint64_t tiles, const Src& src, uint64_t n, KeyT* out, uint32_t* vout,
                        int shift, int bshift, uint32_t* cursor, KeyT* hout = nullptr, uint32_t* hvout = nullptr,
                        const NarrowArgs& nw = NarrowArgs{}) {
  if constexpr (sizeof(KeyT) == 8) {
    if (LEVEL == 2 && shift >= 32 && bshift >= 32) {
      launch_msd_scatter_impl<Src, KeyT, HAS_VAL, LEVEL, SPLIT, NM, IPT, true>(c, dbits, tiles, src, n, out, vout, shift,
                                                                              bshift, cursor, hout, hvout, nw);
      return;
    }
  }
  launch_msd_scatter_impl<Src, KeyT, HAS_VAL, LEVEL, SPLIT, NM, IPT, false>(c, dbits, tiles, src, n, out, vout, shift,
                                                                           bshift, cursor, hout, hvout, nw);
}

struct SegTotals {
  uint32_t light, big, nbig;
};

// classify C child counts (light <= kSegCap, big otherwise): cursors with the
// light bit in scur, light offsets in sloff[0..C], big offsets (= next parents)
// compacted into npoff; totals in stot (seg_classify: read back to the host)
void seg_classify_enqueue(nmx_ctx* c, const uint32_t* ccnt, uint32_t C, uint32_t* npoff) {
  c->scur.grow(((size_t)C + 8) * 4);
  c->sloff.grow(((size_t)C + 8) * 4);
  c->stot.grow(64);
  if (C <= kSegSmallC) {
    seg_classify_small_kernel<<<1, 256, 0, c->st>>>(ccnt, C, c->stot.as<uint32_t>(), c->scur.as<uint32_t>(),
                                                    c->sloff.as<uint32_t>(), npoff);
    CK_LAUNCH();
    ++c->launches;
    return;
  }
  const uint32_t nb = (C + kSegScanItems - 1) / kSegScanItems;
  c->sbsum.grow(((size_t)nb + 8) * 8);
  c->sbflag.grow(((size_t)nb + 8) * 4);
  c->stot.grow(64);
  seg_scan_sums_kernel<<<nb, 256, 0, c->st>>>(ccnt, C, c->sbsum.as<unsigned long long>(), c->sbflag.as<uint32_t>());
  CK_LAUNCH();
  seg_scan_top_kernel<<<1, 1024, 0, c->st>>>(c->sbsum.as<unsigned long long>(), c->sbflag.as<uint32_t>(), nb,
                                             c->stot.as<uint32_t>());
  CK_LAUNCH();
  seg_scan_apply_kernel<<<nb, 256, 0, c->st>>>(ccnt, C, c->sbsum.as<unsigned long long>(), c->sbflag.as<uint32_t>(),
                                               c->stot.as<uint32_t>(), c->scur.as<uint32_t>(), c->sloff.as<uint32_t>(),
                                               npoff);
  CK_LAUNCH();
  c->launches += 3;
}
SegTotals seg_classify(nmx_ctx* c, const uint32_t* ccnt, uint32_t C, uint32_t* npoff) {
  seg_classify_enqueue(c, ccnt, C, npoff);
  auto* h = reinterpret_cast<SegTotals*>(c->scr());
  CK(cudaMemcpyAsync(h, c->stot.p, sizeof(SegTotals), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return *h;
}

// level widths of a D-bit dense partition: the fewest levels of <= 8 bits, split
// evenly (7-bit levels keep a digit's run in a 2048-key tile ~16 keys long; an
// 8-bit level is only used where it saves a whole level: D = 15, 16, 22-24);
// returns the number of levels
int msd_level_bits(int D, int* dl, int* cum) {
  const int L = (D + kMsdMaxLevelBits - 1) / kMsdMaxLevelBits;
  for (int l = 0, acc = 0; l < L; ++l) {
    dl[l] = D / L + (l < D % L ? 1 : 0);
    acc += dl[l];
    cum[l] = acc;
  }
  return L;
}

// last-level split of the dense MSD partition: light buckets stay in the level
// output, heavy ones (> kSegCap) go compacted to (hk, hv), their offsets to spoffA
struct MsdSplit {
  void* hk = nullptr;
  uint32_t* hv = nullptr;
  SegTotals t{};
};

// Waits for a partition's read-back (work queued after it keeps the GPU busy
// meanwhile): returns m, fills split->t.
uint64_t msd_partition_wait(nmx_ctx* c, MsdSplit* split) {
  if (c->capturing) {  // inside a graph: no heavy buckets assumed, checked after the replay
    if (split) split->t = SegTotals{0, 0, 0};
    return 1;
  }
  CK(cudaEventSynchronize(c->evw));
  const unsigned long long* h = c->scr() + c->scr_off;
  const uint64_t m = h[0];
  if (split) {
    split->t = c->pend_L > 1 ? *reinterpret_cast<const SegTotals*>(h + 1) : SegTotals{};
    if (getenv("NMX_DEBUG"))
      fprintf(stderr, "dense split m=%llu light=%u big=%u nbig=%u\n", (unsigned long long)m, split->t.light,
              split->t.big, split->t.nbig);
  }
  c->dom_bytes += c->pend_bytes_per_m * m;
  c->dom_resolve(m);
  return m;
}

// defer: return 0 at once; the caller queues more work (sized from device-side
// totals) and then calls msd_partition_wait
template <typename Src, typename KeyT, bool HAS_VAL>
uint64_t msd_partition(nmx_ctx* c, const Src& src, uint64_t n, int kb, int D, KeyT* outA, uint32_t* voutA,
                       KeyT* outB, uint32_t* voutB, KeyT** res_k, uint32_t** res_v,
                       const uint32_t* prehist = nullptr, MsdSplit* split = nullptr, uint64_t pre_m = 0,
                       bool defer = false) {
  int dl[8], cum[8];
  const int L = msd_level_bits(D, dl, cum);
  const uint32_t nb = 1u << D;
  uint32_t* d_small = c->small.as<uint32_t>();
  auto* gcount = reinterpret_cast<unsigned long long*>(d_small + kGCount);
  c->mcur.grow(((size_t)nb + 8) * 4);
  c->moff.grow(((size_t)nb + 8) * 4);
  c->mhist2.grow(((size_t)nb + 8) * 4);
  uint32_t* cur = c->mcur.as<uint32_t>();
  uint32_t* off = c->moff.as<uint32_t>();
  constexpr uint64_t kItem = sizeof(KeyT) + (HAS_VAL ? 4 : 0);  // 8 B per item in and out
  bool joint = false;  // level-2 counts already in mhist2 (msd_hist12_kernel)
  if (pre_m) {
    joint = c->joint_ready;
    c->joint_ready = false;
  }
  *res_k = outA;
  *res_v = voutA;
  if (pre_m) {
    // level 1 already done window by window into outA (msd_window_level1)
  } else if (prehist) {  // first-level histogram (+ count) filled by the producer of `src`
    CK(cudaMemcpyAsync(d_small + kHist, prehist, sizeof(uint32_t) * kMsdMaxBins, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(gcount, prehist + kMsdMaxBins, 8, cudaMemcpyDeviceToDevice, c->st));
  } else {
    CK(cudaMemsetAsync(d_small + kHist, 0, sizeof(uint32_t) * kMsdMaxBins, c->st));
    CK(cudaMemsetAsync(gcount, 0, 8, c->st));
    // levels 1 + 2 counted together when the per-CTA flush of the joint bins
    // stays below 1/16 of the keys (large inputs)
    if (L >= 2 && cum[1] <= kJointMaxBits && dl[1] >= 5 && n >= ((uint64_t)c->sms * 3 << (cum[1] + 4))) {
      joint = true;
      CK(cudaMemsetAsync(c->mhist2.p, 0, sizeof(uint32_t) << cum[1], c->st));
      auto k = msd_hist12_kernel<Src, KeyT>;
      const size_t sm = sizeof(uint32_t) << cum[1];
      set_smem(k, sm);
      const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 2047) / 2048, (uint64_t)c->sms * 3));
      k<<<hgrid, kH12Threads, sm, c->st>>>(src, n, kb - cum[1], cum[1], dl[1], d_small + kHist,
                                           c->mhist2.as<uint32_t>(),
                                   gcount);
    } else {
      const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 2047) / 2048, (uint64_t)c->sms * 8));
      msd_hist1_kernel<Src, KeyT><<<hgrid, 256, 0, c->st>>>(src, n, kb - dl[0], d_small + kHist, gcount);
    }
    CK_LAUNCH();
  }
  // The valid count m stays on the device (gcount) until the last level's split
  // totals come back: later levels size their grids by n and read m there, so
  // the whole dense partition is queued without a host round trip.
  int dom_pending = 0;  // dominant-class launches whose bytes (2 kItem m each) wait for m
  if (pre_m) {
    set_u64_kernel<<<1, 1, 0, c->st>>>(gcount, pre_m);
    CK_LAUNCH();
    ++c->launches;
  } else {
    scan_counts(c, d_small + kHist, 1u << dl[0], off, cur);
    c->launches += 2;
    c->dom_begin("msd_scatter");
    launch_msd_scatter<Src, KeyT, HAS_VAL, 1>(c, dl[0], tiles_of(n, kMsdTile), src, n, outA, voutA, kb - dl[0], 0,
                                              cur);
    CK_LAUNCH();
    dom_pending += c->dom_cur;
    c->dom_end(0, 2 * kItem);
    ++c->launches;
  }
  KeyT* in_k = outA;
  uint32_t* in_v = voutA;
  KeyT* out_k = outB;
  uint32_t* out_v = voutB;
  // three levels without the joint level-1/2 counts (the column partition): levels 2
  // and 3 counted in one pass over the level-1 output (msd_count23_kernel)
  const bool joint23 = !joint && !pre_m && !HAS_VAL && L == 3 && dl[1] + dl[2] <= kJointMaxBits && dl[2] >= 2 &&
                       n >= (1ull << 27) && !c->capturing && count23_enabled();
  if (joint23) {
    c->mhist3.grow(((size_t)(1u << cum[2]) + 8) * 4);
    CK(cudaMemsetAsync(c->mhist3.p, 0, (size_t)4 << cum[2], c->st));
    auto k = msd_count23_kernel<KeyT>;
    const int jbits = dl[1] + dl[2];
    const size_t sm = (size_t)4 << jbits;
    set_smem(k, sm);
    constexpr uint64_t kPer = 1ull << 20;
    k<<<(unsigned)((n + kPer - 1) / kPer), kJointCountThreads, sm, c->st>>>(
        outA, gcount, off, 1u << dl[0], kPer, kb - cum[2], jbits, c->mhist3.as<uint32_t>());
    CK_LAUNCH();
    hist_fold_kernel<<<(unsigned)std::max(1u, std::min(((1u << cum[1]) + 255) / 256, (uint32_t)c->sms * 4)), 256, 0,
                       c->st>>>(c->mhist3.as<uint32_t>(), 1u << cum[1], dl[2], c->mhist2.as<uint32_t>());
    CK_LAUNCH();
    c->launches += 2;
  }
  for (int l = 1; l < L; ++l) {
    const int shift = kb - cum[l], bshift = kb - cum[l - 1];
    const uint32_t nbl = 1u << cum[l];
    uint32_t* h2 = joint23 && l == 2 ? c->mhist3.as<uint32_t>() : c->mhist2.as<uint32_t>();
    if (!(joint && l == 1) && !joint23) {
      CK(cudaMemsetAsync(h2, 0, (size_t)nbl * 4, c->st));
      msd_count2_kernel<KeyT><<<(unsigned)tiles_of(n, kMsdTile * kCount2Tiles), kMsdThreads, 0, c->st>>>(
          in_k, gcount, shift, dl[l], bshift, h2);
      CK_LAUNCH();
    }
    KeySrcD<KeyT, HAS_VAL> ks{in_k, in_v, gcount};
    if (split && l + 1 == L) {  // heavy buckets leave compacted (nmx_seg.cuh continues them)
      c->spoffA.grow(((size_t)std::min<uint64_t>(nbl, n / (kSegCap + 1) + 1) + 8) * 4);
      seg_classify_enqueue(c, h2, nbl, c->spoffA.as<uint32_t>());
      c->dom_begin("msd_scatter");
      NarrowArgs sw;
      sw.big = c->stot.as<uint32_t>() + 1;  // SegTotals.big of the classification just queued
      launch_msd_scatter<KeySrcD<KeyT, HAS_VAL>, KeyT, HAS_VAL, 2, true>(
          c, dl[l], tiles_of(n, kMsdTile), ks, n, out_k, out_v, shift, bshift, c->scur.as<uint32_t>(),
          reinterpret_cast<KeyT*>(split->hk), split->hv, sw);
    } else {
      scan_counts(c, h2, nbl, off, cur);
      c->dom_begin("msd_scatter");
      launch_msd_scatter<KeySrcD<KeyT, HAS_VAL>, KeyT, HAS_VAL, 2>(c, dl[l], tiles_of(n, kMsdTile), ks, n, out_k,
                                                                   out_v, shift, bshift, cur);
    }
    CK_LAUNCH();
    dom_pending += c->dom_cur;
    c->dom_end(0, 2 * kItem);
    c->launches += 3;
    std::swap(in_k, out_k);
    std::swap(in_v, out_v);
  }
  *res_k = in_k;
  *res_v = in_v;
  c->msd_levels = L;
  // one round trip for the whole partition: m and (with a split) its totals
  unsigned long long* h = c->scr() + c->scr_off;  // [0] m, [1..2] split totals
  if (split) CK(cudaMemcpyAsync(h + 1, c->stot.p, sizeof(SegTotals), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(h, gcount, 8, cudaMemcpyDeviceToHost, c->st));
  if (!c->evw) CK(cudaEventCreateWithFlags(&c->evw, cudaEventDisableTiming));
  if (!c->capturing) CK(cudaEventRecord(c->evw, c->st));
  c->pend_bytes_per_m = (uint64_t)dom_pending * 2 * kItem;
  c->pend_L = L;
  return defer ? 0 : msd_partition_wait(c, split);
}

// Column partition with narrowed items (NarrowArgs, nmx_msd.cuh): level 1 reads the
// u64 (dst << 32 | count) items and writes u32 items (dst bits below the level-1
// digit | count - 1); levels 2 and 3 are counted in one pass and move 4-byte items
// with positional parents; heavy destination buckets leave widened back to u64
// (split->hk) for the segmented levels. Per item: 12 + 4 + 8 + 8 bytes over the
// levels instead of 16 + 8 + 16 + 16. The caller has checked col_narrow_bits()
// (three levels, every count <= 2^cb). Deferred like msd_partition (defer = true).
// items per thread of the u32 column levels (4-byte items: a 4096-item tile stages in
// the bytes of a 2048-item u64 tile, digit runs twice as long)
#ifndef NMX_POS_IPT
#define NMX_POS_IPT 8
#endif
constexpr int kPosIPT = NMX_POS_IPT;
constexpr int kPosTile = kMsdThreads * kPosIPT;
int col_narrow_bits(int b, int D) {
  int dl[8], cum[8];
  if (msd_level_bits(D, dl, cum) != 3 || dl[1] + dl[2] > kJointMaxBits || dl[2] < 2) return 0;
  const int delta = b - dl[0];
  return delta >= 8 && delta <= 31 ? 32 - delta : 0;  // count bits
}

void msd_partition_cols_narrow(nmx_ctx* c, const ColConcatSrc& src, uint64_t n, int b, int D, const uint32_t* prehist,
                               MsdSplit* split, uint32_t* k32A, uint32_t* k32B) {
  int dl[8], cum[8];
  msd_level_bits(D, dl, cum);
  const int kb = b + 32, delta = b - dl[0], cb = 32 - delta;
  uint32_t* d_small = c->small.as<uint32_t>();
  auto* gcount = reinterpret_cast<unsigned long long*>(d_small + kGCount);
  const uint32_t nb = 1u << D;
  c->mcur.grow(((size_t)nb + 8) * 4);
  c->moff.grow(((size_t)nb + 8) * 4);
  c->mhist2.grow(((size_t)nb + 8) * 4);
  c->moff1.grow(((size_t)(1u << dl[0]) + 8) * 4);
  c->mhist3.grow(((size_t)(1u << cum[2]) + 8) * 4);
  uint32_t* cur = c->mcur.as<uint32_t>();
  uint32_t* off = c->moff.as<uint32_t>();
  uint32_t* off1 = c->moff1.as<uint32_t>();
  CK(cudaMemcpyAsync(d_small + kHist, prehist, sizeof(uint32_t) * kMsdMaxBins, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(gcount, prehist + kMsdMaxBins, 8, cudaMemcpyDeviceToDevice, c->st));
  NarrowArgs nw;
  nw.delta = delta;
  nw.cb = cb;
  uint64_t bpi = 0;  // dominant-class bytes per valid item
  // level 1: u64 items -> u32
  scan_counts(c, d_small + kHist, 1u << dl[0], off1, cur);
  c->dom_begin("msd_scatter");
  nw.nout = k32A;
  launch_msd_scatter<ColConcatSrc, uint64_t, false, 1, false, NM_OUT>(c, dl[0], tiles_of(n, kMsdTile), src, n,
                                                                      nullptr, nullptr, kb - dl[0], 0, cur, nullptr,
                                                                      nullptr, nw);
  CK_LAUNCH();
  bpi += c->dom_cur ? 12 : 0;
  c->dom_end(0, 12);
  // levels 2 + 3 counted jointly over the u32 items (parents = level-1 buckets by position)
  CK(cudaMemsetAsync(c->mhist3.p, 0, (size_t)4 << cum[2], c->st));
  {
    auto k = msd_count23_kernel<uint32_t>;
    const int jbits = dl[1] + dl[2];
    const size_t sm = (size_t)4 << jbits;
    set_smem(k, sm);
    constexpr uint64_t kPer = 1ull << 20;
    k<<<(unsigned)((n + kPer - 1) / kPer), kJointCountThreads, sm, c->st>>>(
        k32A, gcount, off1, 1u << dl[0], kPer, kb - cum[2] - delta, jbits, c->mhist3.as<uint32_t>());
    CK_LAUNCH();
    hist_fold_kernel<<<(unsigned)std::max(1u, std::min(((1u << cum[1]) + 255) / 256, (uint32_t)c->sms * 4)), 256, 0,
                       c->st>>>(c->mhist3.as<uint32_t>(), 1u << cum[1], dl[2], c->mhist2.as<uint32_t>());
    CK_LAUNCH();
  }
  // level 2: u32 -> u32, parents = level-1 buckets (tiles of kPosIPT items per thread)
  const uint64_t ntiles = tiles_of(n, kPosTile);
  c->mtpar.grow((size_t)(ntiles + 1) * 16);
  const unsigned tgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ntiles + 255) / 256, (uint64_t)c->sms * 8));
  nw.tpar = c->mtpar.as<uint4>();
  scan_counts(c, c->mhist2.as<uint32_t>(), 1u << cum[1], off, cur);
  nw.nout = nullptr;
  nw.poff = off1;
  nw.npar = 1u << dl[0];
  tile_parents_kernel<<<tgrid, 256, 0, c->st>>>(off1, nw.npar, gcount, ntiles, c->mtpar.as<uint4>(), kPosTile);
  CK_LAUNCH();
  c->dom_begin("msd_scatter");
  launch_msd_scatter<KeySrcD<uint32_t, false>, uint32_t, false, 2, false, NM_POS, kPosIPT>(
      c, dl[1], ntiles, KeySrcD<uint32_t, false>{k32A, nullptr, gcount}, n, k32B, nullptr,
      kb - cum[1] - delta, 0, cur, nullptr, nullptr, nw);
  CK_LAUNCH();
  bpi += c->dom_cur ? 8 : 0;
  c->dom_end(0, 8);
  // level 3 with the light / heavy split: parents = level-2 buckets (their offsets in off)
  c->spoffA.grow(((size_t)std::min<uint64_t>(1u << cum[2], n / (kSegCap + 1) + 1) + 8) * 4);
  seg_classify_enqueue(c, c->mhist3.as<uint32_t>(), 1u << cum[2], c->spoffA.as<uint32_t>());
  nw.poff = off;
  nw.npar = 1u << cum[1];
  nw.wout = reinterpret_cast<uint64_t*>(split->hk);
  nw.dlp = dl[1];
  nw.big = c->stot.as<uint32_t>() + 1;
  tile_parents_kernel<<<tgrid, 256, 0, c->st>>>(off, nw.npar, gcount, ntiles, c->mtpar.as<uint4>(), kPosTile);
  CK_LAUNCH();
  c->dom_begin("msd_scatter");
  launch_msd_scatter<KeySrcD<uint32_t, false>, uint32_t, false, 2, true, NM_POS, kPosIPT>(
      c, dl[2], ntiles, KeySrcD<uint32_t, false>{k32B, nullptr, gcount}, n, k32A, nullptr,
      kb - cum[2] - delta, 0, c->scur.as<uint32_t>(), nullptr, nullptr, nw);
  CK_LAUNCH();
  bpi += c->dom_cur ? 8 : 0;
  c->dom_end(0, 8);
  c->launches += 7;  // + the scans and the classification (counted there)
  c->msd_levels = 3;
  unsigned long long* h = c->scr() + c->scr_off;  // [0] m, [1..2] split totals
  CK(cudaMemcpyAsync(h + 1, c->stot.p, sizeof(SegTotals), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(h, gcount, 8, cudaMemcpyDeviceToHost, c->st));
  if (!c->evw) CK(cudaEventCreateWithFlags(&c->evw, cudaEventDisableTiming));
  CK(cudaEventRecord(c->evw, c->st));
  c->pend_bytes_per_m = bpi;
  c->pend_L = 3;
}

// ---- segmented MSD levels over heavy buckets (nmx_seg.cuh) ------------------
// split `bits` into ceil(bits / seg_level_bits()) near-equal level widths
// (NMX_SEG_BITS=7 restores the 7-bit segmented levels, for A/B measurements)
int seg_level_bits() {
  static const int v = [] {
    const char* e = getenv("NMX_SEG_BITS");
    const int x = e ? atoi(e) : kSegLevelBits;
    return x >= 4 && x <= kSegLevelBits ? x : kSegLevelBits;
  }();
  return v;
}
int split_levels(int bits, int* out) {
  if (bits <= 0) return 0;
  const int lb = seg_level_bits();
  const int L = (bits + lb - 1) / lb;
  for (int l = 0; l < L; ++l) out[l] = bits / L + (l < bits % L ? 1 : 0);
  return L;
}

// count + classify one level of P positional parents (m items) into C = P << dbits
// children; leaves child counts in sccnt, cursors in scur, light offsets in
// sloff, next parents in `npoff`
template <typename KeyT, bool HAS_VAL>
SegTotals seg_level_plan(nmx_ctx* c, const KeyT* k, const uint32_t* v, uint32_t m, const uint32_t* poff, uint32_t P,
                         int shift, int dbits, uint32_t* npoff) {
  const uint32_t C = P << dbits;
  c->sccnt.grow(((size_t)C + 8) * 4);
  uint32_t* ccnt = c->sccnt.as<uint32_t>();
  CK(cudaMemsetAsync(ccnt, 0, (size_t)C * 4, c->st));
  seg_count_kernel<KeyT, HAS_VAL, false><<<(unsigned)tiles_of(m, kMsdTile), kMsdThreads, 0, c->st>>>(
      k, v, m, poff, P, shift, dbits, ccnt, nullptr, nullptr);
  CK_LAUNCH();
  ++c->launches;
  return seg_classify(c, ccnt, C, npoff);
}

// shared-memory groups over this level's light children (loff = sloff, C children)
// the same with the light total still on the device (stot[0], deferred
// partition read-back): plans for at most `upper` keys; returns the device
// group count for the grouping kernel
// K > 0: groups are cut into pieces of <= K buckets (direct-slot eligibility)
const uint32_t* seg_plan_groups_dev(nmx_ctx* c, uint32_t C, uint64_t upper, uint32_t S, uint32_t K = 0) {
  const uint64_t ng_max = (upper + S - 1) / S;
  // a piece could never exceed K buckets; small calls keep their few launches
  if (K >= C || upper < (1ull << 26)) K = 0;
  const uint64_t np_max = ng_max + (K ? (uint64_t)C / K + 2 : 0);
  c->mgb.grow(((size_t)ng_max + 2) * 4);
  c->mplan.grow(((size_t)np_max + 2) * 16);
  uint32_t* ngp = c->stot.as<uint32_t>() + 12;
  const unsigned g1 = (unsigned)std::min<uint64_t>((ng_max + 256) / 256, (uint64_t)c->sms * 8);
  if (!K) {  // bounds and plans in one pass
    group_plan_kernel<<<g1, 256, 0, c->st>>>(c->sloff.as<uint32_t>(), C, S, 0, c->mplan.as<uint4>(),
                                             c->stot.as<uint32_t>(), ngp);
    CK_LAUNCH();
    ++c->launches;
    return ngp;
  }
  group_bounds_kernel<<<g1, 256, 0, c->st>>>(c->sloff.as<uint32_t>(), C, S, 0, c->mgb.as<uint32_t>(),
                                             c->stot.as<uint32_t>(), ngp);
  CK_LAUNCH();
  c->mpcnt.grow(((size_t)ng_max + 2) * 4);
  c->mpoff.grow(((size_t)ng_max + 2) * 4);
  group_split_count_kernel<<<g1, 256, 0, c->st>>>(c->mgb.as<uint32_t>(), ngp, (uint32_t)ng_max, K,
                                                  c->mpcnt.as<uint32_t>());
  CK_LAUNCH();
  scan_counts(c, c->mpcnt.as<uint32_t>(), (uint32_t)ng_max, c->mpoff.as<uint32_t>(), nullptr);
  seg_plan_split_kernel<<<g1, 256, 0, c->st>>>(c->sloff.as<uint32_t>(), c->mgb.as<uint32_t>(), ngp,
                                               c->mpoff.as<uint32_t>(), K, c->mplan.as<uint4>());
  CK_LAUNCH();
  c->launches += 4;
  return c->mpoff.as<uint32_t>() + ng_max;  // the piece count (scan total)
}

uint32_t seg_plan_groups(nmx_ctx* c, uint32_t C, uint32_t light, uint32_t S) {
  const uint32_t ngroups = (light + S - 1) / S;
  c->mgb.grow(((size_t)ngroups + 2) * 4);
  c->mplan.grow(((size_t)ngroups + 2) * 16);
  const unsigned g1 = (unsigned)std::min<uint64_t>((ngroups + 256) / 256, (uint64_t)c->sms * 8);
  group_plan_kernel<<<g1, 256, 0, c->st>>>(c->sloff.as<uint32_t>(), C, S, ngroups, c->mplan.as<uint4>(), nullptr,
                                           nullptr);
  CK_LAUNCH();
  ++c->launches;
  return ngroups;
}

// Heavy row buckets (mh keys in keysC, nheavy parents at spoffA):
// levels over the remaining b - D source bits (children stay whole sources,
// local_rows_kernel<false>), then over the b destination bits (every parent is
// one source: local_rows_kernel<true> with the SrcTable), final level
// count-only (one link per child). Column entries go to ckA / cvA; returns
// their number.
uint64_t heavy_rows(nmx_ctx* c, uint64_t mh, uint32_t nheavy, int b, int D, int cshift, uint32_t* chist,
                    unsigned long long* ccount) {
  // Key fields per level (shift, width): one level of the remaining source bits
  // (children stay whole sources: NORMAL groups), then the destination bits
  // (parents mostly one heavy source: PARTIAL groups + SrcTable), then the last
  // source bits in the count-only final level, where every child is one key.
  // Heavy parents are dominated by one source, so the low source bits carry
  // almost no entropy and would only re-copy the bucket if split first.
  int w[16], sh[16];
  bool part[16];
  int L = 0;
  const int r = b - D;                          // source bits below the dense prefix
  int r0 = r > 0 ? std::min(r, std::min((r + 1) / 2, seg_level_bits())) : 0;
  if (const char* e = getenv("NMX_HEAVY_R0")) r0 = std::max(0, std::min(r, atoi(e)));  // A/B runs
  if (r0) w[L] = r0, sh[L] = 2 * b - D - r0, part[L] = false, ++L;
  {
    int dw[8];
    const int Ld = split_levels(b, dw);
    for (int i = 0, at = b; i < Ld; ++i) {
      at -= dw[i];
      w[L] = dw[i], sh[L] = at, part[L] = true, ++L;
    }
  }
  const int rlow = r - r0;                      // low source bits, last (the final level is count-only)
  {
    int lw[8];
    const int Ll = split_levels(rlow, lw);
    for (int i = 0, at = b + rlow; i < Ll; ++i) {
      at -= lw[i];
      w[L] = lw[i], sh[L] = at, part[L] = true, ++L;
    }
  }
  c->lightK.grow(mh * 8);
  uint32_t* poff = c->spoffA.as<uint32_t>();
  uint64_t* in = c->keysC.as<uint64_t>();
  uint64_t* out = c->keysD.as<uint64_t>();
  uint64_t* hcol = c->ckA.as<uint64_t>();  // packed column items of the heavy sources
  uint32_t P = nheavy, m = (uint32_t)mh;
  uint64_t lbase = 0;
  SrcTable gsrc;
  bool table = false;
  set_smem(seg_scatter_kernel<uint64_t, false>, sizeof(SegSmem<uint64_t, false>));
  set_smem(local_rows_kernel<false>, sizeof(LocSmem));
  set_smem(local_rows_kernel<true>, sizeof(LocSmem));
  for (int l = 0; l < L && m; ++l) {
    const int dbits = w[l];
    const bool partial = part[l];  // sources may be split over several children
    if (partial && !table) {       // at most 2^rlow sources per parent of the first destination level
      const uint64_t bound = std::min<uint64_t>(m, (uint64_t)P << rlow);
      uint32_t cap = 1024;
      while (cap < 2 * bound + 16) cap <<= 1;
      c->gsk.grow(((size_t)cap + 2) * 4);
      c->gsv.grow(((size_t)cap + 2) * 8);
      CK(cudaMemsetAsync(c->gsk.p, 0, ((size_t)cap + 2) * 4, c->st));
      CK(cudaMemsetAsync(c->gsv.p, 0, ((size_t)cap + 2) * 8, c->st));
      gsrc.keys = c->gsk.as<uint32_t>();
      gsrc.vals = c->gsv.as<unsigned long long>();
      gsrc.mask = cap - 1;
      table = true;
    }
    const int shift = sh[l];
    const uint32_t C = P << dbits;
    if (l + 1 == L) {  // final level: count only, one link per child
      c->sccnt.grow(((size_t)C + 8) * 4);
      c->srep.grow(((size_t)C + 8) * 8);
      c->hcount.grow(64);
      uint32_t* ccnt = c->sccnt.as<uint32_t>();
      CK(cudaMemsetAsync(ccnt, 0, (size_t)C * 4, c->st));
      CK(cudaMemsetAsync(c->hcount.p, 0, 8, c->st));
      seg_count_kernel<uint64_t, false, true><<<(unsigned)tiles_of(m, kMsdTile), kMsdThreads, 0, c->st>>>(
          in, nullptr, m, poff, P, shift, dbits, ccnt, nullptr, c->srep.as<uint64_t>());
      CK_LAUNCH();
      const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((C + 4095) / 4096, (uint64_t)c->sms * 4));
      seg_emit_rows_kernel<<<g, 256, 0, c->st>>>(ccnt, c->srep.as<uint64_t>(), C, b, hcol + lbase,
                                                 c->hcount.as<unsigned long long>(), cshift, chist,
                                                 ccount, c->stats.as<unsigned long long>(), gsrc);
      CK_LAUNCH();
      c->launches += 2;
      unsigned long long* hc = c->scr();
      CK(cudaMemcpyAsync(hc, c->hcount.p, 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      lbase += *hc;
      m = 0;
      break;
    }
    DevBuf& nb = (l & 1) ? c->spoffA : c->spoffB;
    // next parents: at most min(C, m / (kSegCap + 1)) big children
    nb.grow(((size_t)std::min<uint64_t>(C, m / (kSegCap + 1) + 1) + 8) * 4);
    uint32_t* npoff = nb.as<uint32_t>();
    const SegTotals t = seg_level_plan<uint64_t, false>(c, in, nullptr, m, poff, P, shift, dbits, npoff);
    if (getenv("NMX_DEBUG"))
      fprintf(stderr, "heavy_rows l=%d P=%u m=%u C=%u dbits=%d shift=%d light=%u big=%u nbig=%u\n", l, P, m, C, dbits,
              shift, t.light, t.big, t.nbig);
    seg_scatter_kernel<uint64_t, false><<<(unsigned)tiles_of(m, kMsdTile), kMsdThreads,
                                          sizeof(SegSmem<uint64_t, false>), c->st>>>(
        in, nullptr, m, poff, P, shift, dbits, c->scur.as<uint32_t>(), c->lightK.as<uint64_t>() + lbase, nullptr, out,
        nullptr);
    CK_LAUNCH();
    ++c->launches;
    if (t.light) {
      const uint32_t ngroups = seg_plan_groups(c, C, t.light, kLocChunk);
      const unsigned grid = (unsigned)std::min<uint64_t>(ngroups, (uint64_t)c->sms * 2);
      if (partial)
        local_rows_kernel<true><<<grid, kLocThreads, sizeof(LocSmem), c->st>>>(
            c->lightK.as<uint64_t>() + lbase, c->mplan.as<uint4>(), ngroups, b, hcol + lbase,
            cshift, chist, ccount, c->stats.as<unsigned long long>(), gsrc, kNoDirect);
      else
        local_rows_kernel<false><<<grid, kLocThreads, sizeof(LocSmem), c->st>>>(
            c->lightK.as<uint64_t>() + lbase, c->mplan.as<uint4>(), ngroups, b, hcol + lbase,
            cshift, chist, ccount, c->stats.as<unsigned long long>(), gsrc, kNoDirect);
      CK_LAUNCH();
      ++c->launches;
    }
    lbase += t.light;
    std::swap(in, out);
    poff = npoff;
    P = t.nbig;
    m = t.big;
  }
  if (table) {
    const uint32_t ents = gsrc.mask + 2;
    src_table_stats_kernel<<<(unsigned)std::min<uint64_t>((ents + 255) / 256, (uint64_t)c->sms * 4), 256, 0, c->st>>>(
        gsrc, c->stats.as<unsigned long long>());
    CK_LAUNCH();
    ++c->launches;
  }
  return lbase;
}

// Heavy destination buckets ((dst, count) entries in cgk / cgv, nheavy
// parents at spoffA): levels over the remaining b - Dc destination bits
// (children stay whole destinations, local_cols_kernel), final level
// count-only with packet sums (one destination per child).
void heavy_cols(nmx_ctx* c, uint64_t ch, uint32_t nheavy, int b, int Dc) {
  // packed items (dst << 32 | count): key bits [32, 32 + b)
  int w[8];
  int L = split_levels(b - Dc, w);
  if (!L) w[L++] = 0;  // the dense levels already isolate single destinations
  c->lightCK.grow(ch * 8);
  uint32_t* poff = c->spoffA.as<uint32_t>();
  uint64_t* ink = c->cgk.as<uint64_t>();
  uint64_t* outk = c->cgk2.as<uint64_t>();
  uint64_t* light = c->lightCK.as<uint64_t>();
  uint32_t P = nheavy, m = (uint32_t)ch;
  uint64_t lbase = 0;
  int consumed = Dc;
  set_smem(seg_scatter_kernel<uint64_t, false>, sizeof(SegSmem<uint64_t, false>));
  set_smem(local_cols_kernel<false>, sizeof(LocColSmem));
  for (int l = 0; l < L && m; ++l) {
    const int dbits = w[l];
    consumed += dbits;
    const int shift = b + 32 - consumed;
    const uint32_t C = P << dbits;
    if (l + 1 == L) {
      c->sccnt.grow(((size_t)C + 8) * 4);
      c->ssum.grow(((size_t)C + 8) * 8);
      uint32_t* ccnt = c->sccnt.as<uint32_t>();
      CK(cudaMemsetAsync(ccnt, 0, (size_t)C * 4, c->st));
      CK(cudaMemsetAsync(c->ssum.p, 0, (size_t)C * 8, c->st));
      seg_count_kernel<uint64_t, false, true, true><<<(unsigned)tiles_of(m, kMsdTile), kMsdThreads, 0, c->st>>>(
          ink, nullptr, m, poff, P, shift, dbits, ccnt, c->ssum.as<unsigned long long>(), nullptr);
      CK_LAUNCH();
      const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((C + 255) / 256, (uint64_t)c->sms * 8));
      seg_emit_cols_kernel<<<g, 256, 0, c->st>>>(ccnt, c->ssum.as<unsigned long long>(), C,
                                                 c->stats.as<unsigned long long>());
      CK_LAUNCH();
      c->launches += 2;
      break;
    }
    DevBuf& nb = (l & 1) ? c->spoffA : c->spoffB;
    nb.grow(((size_t)std::min<uint64_t>(C, m / (kSegCap + 1) + 1) + 8) * 4);
    uint32_t* npoff = nb.as<uint32_t>();
    const SegTotals t = seg_level_plan<uint64_t, false>(c, ink, nullptr, m, poff, P, shift, dbits, npoff);
    seg_scatter_kernel<uint64_t, false><<<(unsigned)tiles_of(m, kMsdTile), kMsdThreads,
                                          sizeof(SegSmem<uint64_t, false>), c->st>>>(
        ink, nullptr, m, poff, P, shift, dbits, c->scur.as<uint32_t>(), light + lbase, nullptr, outk, nullptr);
    CK_LAUNCH();
    ++c->launches;
    if (t.light) {
      const uint32_t ngroups = seg_plan_groups(c, C, t.light, kLocColChunk);
      const unsigned grid = (unsigned)std::min<uint64_t>(ngroups, (uint64_t)c->sms * 4);
      local_cols_kernel<false><<<grid, kLocColThreads, sizeof(LocColSmem), c->st>>>(
          light + lbase, c->mplan.as<uint4>(), ngroups, c->stats.as<unsigned long long>(), kNoDirect);
      CK_LAUNCH();
      ++c->launches;
    }
    lbase += t.light;
    std::swap(ink, outk);
    poff = npoff;
    P = t.nbig;
    m = t.big;
  }
}

// Column statistics of (dst, count) entries (holes allowed) read through `cs`,
// whose arrays may alias ckA / cvA (the first level reads them all before the
// second level writes ckA / cvA): MSD partition by destination bits ->
// shared-memory grouping -> heavy destinations via LSD + col_kernel.
// wb > 0 (windowed): entries are dst' = window << (b - wb) | dst with b = address bits
// + wb; returns false (nothing more queued) when a heavy destination bucket needs the
// segmented levels, which keep no per-window statistics -- the caller reruns the call
// on the LSD path.
// NMX_NARROW=0 keeps the u64 column items on every level (A/B runs)
bool narrow_enabled() {
  static const bool v = [] {
    const char* e = getenv("NMX_NARROW");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool msd_columns(nmx_ctx* c, const ColConcatSrc& cs, int b, int Dc, const uint32_t* prehist, int wb = 0) {
  // the levels move packed u64 items (dst << 32 | count, key bits [32, 32 + b))
  // through the row key buffers, free once the row half is queued
  uint64_t* ce = nullptr;
  uint32_t* unused = nullptr;
  const uint64_t need = cs.n;
  c->keysA.grow(need * 8);
  c->keysB.grow(need * 8);
  c->cgk.grow(need * 8);
  MsdSplit sp;
  sp.hk = c->cgk.p;
  c->scr_off = 8;  // its read-back beside the row partition's (both live in one graph)
  // Narrowed items after level 1 when every count fits cb bits: prehist means the
  // entries come from this call's row half, whose largest link count (stats field 2)
  // is on the device once the row kernels are done -- one short host wait.
  NarrowArgs nw;
  bool narrow = false;
  if (prehist && !wb && !c->capturing && cs.n >= (1ull << 27) && narrow_enabled()) {
    if (const int cb = col_narrow_bits(b, Dc)) {
      unsigned long long* h = c->scr() + 12;
      CK(cudaMemcpyAsync(h, c->stats.as<unsigned long long>() + S_MAXLINK, 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      narrow = *h >= 1 && *h - 1 < (1ull << cb);
      if (narrow) {
        int dl[8], cum[8];
        msd_level_bits(Dc, dl, cum);
        nw.delta = b - dl[0];
        nw.cb = cb;
        nw.dlp = Dc - dl[0];
      }
    }
  }
  if (narrow)
    msd_partition_cols_narrow(c, cs, cs.n, b, Dc, prehist, &sp, c->keysA.as<uint32_t>(), c->keysB.as<uint32_t>());
  else
    msd_partition<ColConcatSrc, uint64_t, false>(c, cs, cs.n, b + 32, Dc, c->keysA.as<uint64_t>(), nullptr,
                                                 c->keysB.as<uint64_t>(), nullptr, &ce, &unused, prehist, &sp, 0, true);
  c->mark();  // column partition end
  {
    const uint32_t* ngp = seg_plan_groups_dev(c, 1u << Dc, cs.n, kLocColChunk,
                                              b - Dc < 31 ? kLocColDirect >> (b - Dc) : 0);
    if (narrow) {
      nw.poff = c->sloff.as<uint32_t>();
      set_smem(local_cols_kernel<false, true>, sizeof(LocColSmem));
      local_cols_kernel<false, true><<<c->sms * 4, kLocColThreads, sizeof(LocColSmem), c->st>>>(
          nullptr, c->mplan.as<uint4>(), 0, c->stats.as<unsigned long long>(), b - Dc, ngp, 0, 0,
          c->keysA.as<uint32_t>(), nw);
    } else if (wb) {
      set_smem(local_cols_kernel<true>, sizeof(LocColSmem));
      local_cols_kernel<true><<<c->sms * 4, kLocColThreads, sizeof(LocColSmem), c->st>>>(
          ce, c->mplan.as<uint4>(), 0, c->stats.as<unsigned long long>(), b - Dc, ngp, Dc - wb, b - wb);
    } else {
      set_smem(local_cols_kernel<false>, sizeof(LocColSmem));
      local_cols_kernel<false><<<c->sms * 4, kLocColThreads, sizeof(LocColSmem), c->st>>>(
          ce, c->mplan.as<uint4>(), 0, c->stats.as<unsigned long long>(), b - Dc, ngp);
    }
    CK_LAUNCH();
    ++c->launches;
  }
  c->mark();  // local columns end
  const uint64_t u = msd_partition_wait(c, &sp);
  c->scr_off = 0;
  if (sp.t.big) c->had_heavy = true;
  if (!u) return true;
  if (sp.t.big) {  // heavy destination buckets: segmented MSD levels (nmx_seg.cuh)
    if (wb) return false;
    c->cgk2.grow((size_t)sp.t.big * 8);
    heavy_cols(c, sp.t.big, sp.t.nbig, b, Dc);
  }
  return true;
}

// Level 1 of the dense row partition for one window of packets (streaming):
// its keys land in `out` (the window's region of the arena keysA), partitioned
// by the top dl[0] key bits; later levels only need every tile to span few
// level-1 buckets, which window-contiguous regions satisfy. Returns the window's
// valid packets (host sync; the scatter stays queued).
uint64_t msd_window_level1(nmx_ctx* c, const PacketSrc& ps, int kb, int D, uint64_t* out, uint32_t* joint) {
  int dl[8], cum[8];
  msd_level_bits(D, dl, cum);
  uint32_t* d_small = c->small.as<uint32_t>();
  auto* gcount = reinterpret_cast<unsigned long long*>(d_small + kGCount);
  c->mcur.grow(((size_t)(1u << D) + 8) * 4);
  c->moff.grow(((size_t)(1u << D) + 8) * 4);
  CK(cudaMemsetAsync(d_small + kHist, 0, sizeof(uint32_t) * kMsdMaxBins, c->st));
  CK(cudaMemsetAsync(gcount, 0, 8, c->st));
  const uint64_t n = ps.n;
  if (joint) {  // level-2 counts accumulate over the windows (hidden under the copies)
    auto k = msd_hist12_kernel<PacketSrc, uint64_t>;
    const size_t sm = sizeof(uint32_t) << cum[1];
    set_smem(k, sm);
    const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096, (uint64_t)c->sms * 3));
    k<<<hgrid, kH12Threads, sm, c->st>>>(ps, n, kb - cum[1], cum[1], dl[1], d_small + kHist, joint, gcount);
  } else {
    const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 2047) / 2048, (uint64_t)c->sms * 8));
    msd_hist1_kernel<PacketSrc, uint64_t><<<hgrid, 256, 0, c->st>>>(ps, n, kb - dl[0], d_small + kHist, gcount);
  }
  CK_LAUNCH();
  scan_counts(c, d_small + kHist, 1u << dl[0], c->moff.as<uint32_t>(), c->mcur.as<uint32_t>());
  unsigned long long* hm = c->scr();
  CK(cudaMemcpyAsync(hm, gcount, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const unsigned long long m = *hm;
  if (m) {
    launch_msd_scatter<PacketSrc, uint64_t, false, 1>(c, dl[0], tiles_of(n, kMsdTile), ps, n, out, nullptr,
                                                      kb - dl[0], 0, c->mcur.as<uint32_t>());
    CK_LAUNCH();
  }
  return m;
}

// Row half of the MSD path: partition the packed keys by source bits, group them
// in shared memory (links + rows into c->stats), heavy buckets through the
// segmented levels. Returns the column entries ((dst, count) slots, holes = count
// 0) as a ColConcatSrc; *chist_out = their first-level histogram + count.
// pre_m > 0: keysA already holds the level-1 partition of pre_m valid keys
// (streamed windows); n bounds the buffers. Empty (n1 = n2 = 0) if no valid packet.
// window_size > 0 (wb window bits, b + wb <= 32): keys w << 2b | src << b | dst, the
// top D key bits = wb window bits + D - wb source bits, statistics per window; a heavy
// row bucket sets *aborted (the caller reruns the call on the LSD path).
ColConcatSrc msd_rows(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                      int b, int D, uint64_t pre_m, uint32_t** chist_out, int wb = 0, uint64_t window_size = 0,
                      bool* aborted = nullptr) {
  const int kb = 2 * b + wb;
  const int bs = b + wb;  // source' = window << b | src
  // every buffer the step needs is sized up front (n bounds m, u and the heavy parts)
  c->keysA.grow(n * 8);
  c->keysB.grow(n * 8);
  c->keysC.grow(n * 8);
  c->colL_dst.grow(n * 8);  // packed column slots of the light groups
  c->ckA.grow(n * 8);       // packed column items of the heavy sources
  c->mch.grow((kMsdMaxBins + 4) * 4);
  uint32_t* chist = c->mch.as<uint32_t>();
  *chist_out = chist;
  auto* ccount = reinterpret_cast<unsigned long long*>(chist + kMsdMaxBins);
  CK(cudaMemsetAsync(chist, 0, (kMsdMaxBins + 4) * 4, c->st));

  PacketSrc ps{d_src, d_dst, d_valid, n, wb ? window_size : 0, b};
  ps.quad = !(((uintptr_t)d_src | (uintptr_t)d_dst) & 15) && !((uintptr_t)d_valid & 3);
  c->mark();  // 1: row partition start
  uint64_t* keys = nullptr;
  uint32_t* dummy = nullptr;
  MsdSplit sp;
  sp.hk = c->keysC.p;
  // the partition's totals come back while the light groups run (plans and
  // group count derived on the device)
  if (wb)
    msd_partition<PacketSrcWin, uint64_t, false>(c, PacketSrcWin{ps}, n, kb, D, c->keysA.as<uint64_t>(), nullptr,
                                                 c->keysB.as<uint64_t>(), nullptr, &keys, &dummy, nullptr, &sp, pre_m,
                                                 true);
  else
    msd_partition<PacketSrc, uint64_t, false>(c, ps, n, kb, D, c->keysA.as<uint64_t>(), nullptr,
                                              c->keysB.as<uint64_t>(), nullptr, &keys, &dummy, nullptr, &sp, pre_m,
                                              true);
  c->last_sort_launches = c->msd_levels;
  c->mark();  // 2: row partition end
  ColConcatSrc cs{c->colL_dst.as<uint64_t>(), 0, c->ckA.as<uint64_t>(), 0, 0};
  cs.quad = true;  // context buffers are cudaMalloc-aligned
  const uint32_t nb = 1u << D;
  const int Dc = std::min(D, bs);
  const int cshift = bs - msd_first_bits(Dc);
  if (c->capturing)  // light count unknown while recording: every slot past it must read as a hole
    CK(cudaMemsetAsync(c->colL_dst.p, 0, n * 8, c->st));
  {
    const uint32_t* ngp = seg_plan_groups_dev(c, nb, pre_m ? pre_m : n, kLocChunk,
                                              bs - D < 31 ? kLocDirect >> (bs - D) : 0);
    if (wb) {
      set_smem(local_rows_kernel<false, true>, sizeof(LocSmem));
      local_rows_kernel<false, true><<<c->sms * 2, kLocThreads, sizeof(LocSmem), c->st>>>(
          keys, c->mplan.as<uint4>(), 0, b, c->colL_dst.as<uint64_t>(), cshift, chist,
          ccount, c->stats.as<unsigned long long>(), SrcTable{}, bs - D, ngp, D - wb);
    } else {
      set_smem(local_rows_kernel<false>, sizeof(LocSmem));
      local_rows_kernel<false><<<c->sms * 2, kLocThreads, sizeof(LocSmem), c->st>>>(
          keys, c->mplan.as<uint4>(), 0, b, c->colL_dst.as<uint64_t>(), cshift, chist,
          ccount, c->stats.as<unsigned long long>(), SrcTable{}, b - D, ngp);
    }
    CK_LAUNCH();
    ++c->launches;
  }
  c->mark();  // 3: local rows end
  const uint64_t m = msd_partition_wait(c, &sp);
  if (c->capturing) {  // the column partition reads all n slots (holes skipped)
    cs.n1 = cs.n = n;
    return cs;
  }
  if (!m) return cs;
  uint64_t uh = 0;
  if (sp.t.big) c->had_heavy = true;
  if (sp.t.big && wb) {  // heavy buckets keep no per-window statistics: LSD path instead
    if (aborted) *aborted = true;
    return cs;
  }
  if (sp.t.big) {  // heavy row buckets: segmented MSD levels (nmx_seg.cuh)
    c->keysD.grow((size_t)sp.t.big * 8);
    uh = heavy_rows(c, sp.t.big, sp.t.nbig, b, D, cshift, chist, ccount);
  }
  c->mark();  // 4: heavy rows end
  cs.n1 = sp.t.light;
  cs.n2 = uh;
  cs.n = sp.t.light + uh;
  return cs;
}

void run_pipeline_msd(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                      int b, int D, uint64_t pre_m = 0) {
  stage_begin(c, 1);
  uint32_t* chist = nullptr;
  const ColConcatSrc cs = msd_rows(c, d_src, d_dst, d_valid, n, b, D, pre_m, &chist);
  // ---- columns: MSD partition of the (dst, count) entries by destination bits ----
  if (cs.n) msd_columns(c, cs, b, std::min(D, b), chist);
  stage_finish(c, 1);
}

// Sorted packet keys on the MSD machinery (COO builds): dense partition of the top D
// key bits, then local_sort_kernel per group of whole light buckets, in place. Returns
// false (the LSD sort runs instead; nothing the caller sees was written) for small or
// narrow inputs and when a bucket is heavy (> kSegCap keys).
bool sort_rows_msd(nmx_ctx* c, const PacketSrc& ps, int kb, uint64_t* m_out, uint64_t** keys_out) {
  const uint64_t n = ps.n;
  const int D = msd_bits(n, kb);
  if (!D) return false;
  c->keysA.grow(n * 8);
  c->keysB.grow(n * 8);
  c->keysC.grow(n * 8);
  c->mark();  // 1: sort start
  uint64_t* keys = nullptr;
  uint32_t* dummy = nullptr;
  MsdSplit sp;
  sp.hk = c->keysC.p;
  // window ids (window_size < 4 keeps the scalar per-packet loads of PacketSrc)
  const uint64_t m =
      ps.window_size >= 4
          ? msd_partition<PacketSrcWin, uint64_t, false>(c, PacketSrcWin{ps}, n, kb, D, c->keysA.as<uint64_t>(),
                                                         nullptr, c->keysB.as<uint64_t>(), nullptr, &keys, &dummy,
                                                         nullptr, &sp, 0, false)
          : msd_partition<PacketSrc, uint64_t, false>(c, ps, n, kb, D, c->keysA.as<uint64_t>(), nullptr,
                                                      c->keysB.as<uint64_t>(), nullptr, &keys, &dummy, nullptr, &sp,
                                                      0, false);
  if (sp.t.big) {  // the LSD sort starts from zeroed histograms and re-marks its stages
    CK(cudaMemsetAsync(c->small.p, 0, kSmallWords * sizeof(uint32_t), c->st));
    c->nev = 1;
    return false;
  }
  *m_out = m;
  *keys_out = m ? keys : nullptr;
  if (m) {
    const uint32_t* ngp = seg_plan_groups_dev(c, 1u << D, n, kLocChunk, 0);
    set_smem(local_sort_kernel, sizeof(SortSmem));
    local_sort_kernel<<<c->sms * 2, kSortThreads, sizeof(SortSmem), c->st>>>(keys, c->mplan.as<uint4>(), ngp, kb - D);
    CK_LAUNCH();
    ++c->launches;
  }
  c->last_sort_launches = c->msd_levels + 1;
  c->mark();  // 2: sort end
  return true;
}

// Per-window statistics on the MSD path (analytics.py:109-130 analyze_dataset of
// build_matrices(stream, W), traffic.py:221-242): the window id rides above the
// address bits of the row keys and above the destination of the column entries, so
// the partitions never mix windows; the grouping kernels add into stats[9 w ..].
// Needs b + wb <= 32 (anonymized address spaces). Returns false, with nothing
// reported, when a heavy bucket appears (the caller takes the LSD path).
constexpr uint64_t kWinMsdMinWindow = 1ull << 12;
bool run_pipeline_msd_windows(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                              uint64_t n, int b, uint64_t window_size, uint64_t W) {
  const int wb = (int)ceil_log2(W);
  if (b + wb > 32 || window_size < kWinMsdMinWindow) return false;
  const int D = msd_bits(n, b + wb);
  if (!D || D < wb + 4) return false;
  stage_begin(c, W);
  uint32_t* chist = nullptr;
  bool aborted = false;
  const ColConcatSrc cs = msd_rows(c, d_src, d_dst, d_valid, n, b, D, 0, &chist, wb, window_size, &aborted);
  if (aborted) return false;
  if (cs.n && !msd_columns(c, cs, b + wb, std::min(D, b + wb), chist, wb)) return false;
  stage_finish(c, W);
  return true;
}

// ---- small calls as one CUDA graph -------------------------------------------
// A call of n <= 2^24 packets is ~20 short kernels and three host round trips
// (partition read-backs, result). Its launch sequence depends only on (n, b) as long
// as no bucket is heavy, so after one ordinary call the sequence is recorded once --
// address check, row partition, shared-memory groups, column partition, column
// groups, and the D2H of the statistics and of both partitions' heavy totals -- and
// later calls on the same inputs replay it with one launch and one wait. A replay
// whose totals report a heavy bucket (its work is not in the graph) is discarded and
// the call reruns the ordinary way.
void launch_max_addr(nmx_ctx* c, const uint32_t* s, const uint32_t* d, uint64_t n);
constexpr uint64_t kGraphMaxN = 1ull << 24;
constexpr int kGraphSlots = 8;
constexpr int kScrMaxAddr = 16;  // scr() slot of the replay's largest address

bool graph_eligible(uint64_t n) {
  static const bool off = getenv("NMX_NO_GRAPHS") != nullptr;
  return !off && n >= 1 && n <= kGraphMaxN;
}

nmx_ctx::CallGraph* graph_find(nmx_ctx* c, const void* s, const void* d, const void* v, uint64_t n, uint64_t space,
                               uint64_t window = 0) {
  const uint64_t gen = g_buf_gen.load();
  for (size_t i = 0; i < c->graphs.size();) {  // a buffer moved since recording: stale
    if (c->graphs[i].gen != gen) {
      cudaGraphExecDestroy(c->graphs[i].exec);
      c->graphs.erase(c->graphs.begin() + i);
    } else {
      ++i;
    }
  }
  for (auto& g : c->graphs)
    if (g.s == s && g.d == d && g.v == v && g.n == n && g.space == space && g.window == window) return &g;
  return nullptr;
}

// replay: 1 = statistics in h_stats, 0 = a heavy bucket (rerun), NMX_EINVAL = bad address
int graph_replay(nmx_ctx* c, nmx_ctx::CallGraph* g, uint64_t space) {
  c->nev = c->nevk = 0;
  c->dom_name = "";
  c->dom_launches = 0;
  c->dom_bytes = 0;
  c->scr()[kScrMaxAddr] = 0;  // the replay writes its low 4 bytes
  c->mark();
  CK(cudaGraphLaunch(g->exec, c->st));
  c->mark();
  CK(cudaStreamSynchronize(c->st));
  unsigned long long* h = c->scr();
  if (space < (1ull << 32) && h[kScrMaxAddr] >= space)
    return fail(NMX_EINVAL, "addresses must lie in [0, address_space): found %llu >= %llu", h[kScrMaxAddr],
                (unsigned long long)space);
  const SegTotals* rt = reinterpret_cast<const SegTotals*>(h + 1);
  const SegTotals* ct = reinterpret_cast<const SegTotals*>(h + 9);
  if (rt->big || ct->big) return 0;
  CK(cudaEventElapsedTime(&c->last_total_ms, c->ev[0], c->ev[1]));
  c->last_nstage = 1;
  c->last_stage_ms[0] = c->last_total_ms;
  c->last_sort_ms = 0;
  c->last_launches = g->launches;  // the recorded kernels (one graph launch)
  return 1;
}

// record the call's launch sequence (after an ordinary call sized every buffer)
bool run_pipeline_msd_windows(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                              uint64_t n, int b, uint64_t window_size, uint64_t W);
// window > 0: the windowed MSD pipeline (per-window statistics, W windows)
void graph_capture(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                   int b, int D, uint64_t space, uint64_t window = 0) {
  // every buffer the recording touches at its recorded size (the ordinary call sized
  // them for its own, possibly smaller, light totals)
  c->cgk.grow(n * 8);
  c->rmax.grow(64);
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  c->capturing = g_capturing = true;
  bool ok = true;
  int launched = 0;
  try {
    if (space < (1ull << 32)) {
      CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
      launch_max_addr(c, d_src, d_dst, n);
      CK(cudaMemcpyAsync(c->scr() + kScrMaxAddr, c->rmax.p, 4, cudaMemcpyDeviceToHost, c->st));
    }
    c->launches = space < (1ull << 32) ? 1 : 0;
    if (window) {
      if (!run_pipeline_msd_windows(c, d_src, d_dst, d_valid, n, b, window, (n + window - 1) / window)) ok = false;
    } else {
      run_pipeline_msd(c, d_src, d_dst, d_valid, n, b, D);  // stage_begin resets the count
    }
    launched = c->launches + (space < (1ull << 32) ? 1 : 0);
  } catch (...) {
    ok = false;
  }
  c->capturing = g_capturing = false;
  c->scr_off = 0;
  const cudaError_t e = cudaStreamEndCapture(c->st, &graph);
  if (!ok || e != cudaSuccess || !graph) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if ((int)c->graphs.size() >= kGraphSlots) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back({d_src, d_dst, d_valid, n, space, window, exec, g_buf_gen.load(), launched});
}

// The whole pipeline over packet columns already on the device. Writes W*9
// statistics (u64) into c->h_stats. Windows: window_size == 0 -> one window.
void run_pipeline(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                  int b, uint64_t window_size, uint64_t W) {
  if (W == 1) {
    const int D = msd_bits(n, b);
    if (D) return run_pipeline_msd(c, d_src, d_dst, d_valid, n, b, D);
  } else if (run_pipeline_msd_windows(c, d_src, d_dst, d_valid, n, b, window_size, W)) {
    return;
  }
  const int wb = W > 1 ? (int)ceil_log2(W) : 0;
  stage_begin(c, W);
  PacketSrc ps{d_src, d_dst, d_valid, n, W > 1 ? window_size : 0, b};
  const RowsOut r = stage_rows(c, ps, b, wb);
  stage_cols(c, r.u, b, wb, r.wide);
  stage_finish(c, W);
}

// ---- owner partitions for the multi-GPU exchange ----------
// returns per-part counts on the host; items scattered part-contiguously
// base_add (host, optional): part p's items go to absolute positions base_add[p] + ..
// (separate per-part arenas) instead of part-contiguously from 0
// cap_left (host, optional): part p may take at most cap_left[p] items (checked
// before anything is written; std::length_error otherwise)
template <typename Item>
void partition_items(nmx_ctx* c, const Item& it, uint64_t n, int nparts, uint64_t* counts_host,
                     const uint64_t* base_add = nullptr, const uint64_t* cap_left = nullptr) {
  c->part.grow(2 * kMaxParts * sizeof(unsigned long long));
  auto* d_counts = c->part.as<unsigned long long>();
  auto* d_cursor = d_counts + kMaxParts;
  CK(cudaMemsetAsync(d_counts, 0, kMaxParts * sizeof(unsigned long long), c->st));
  const uint64_t tiles = (n + kPartTile - 1) / kPartTile;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)c->sms * 8));
  part_tile_count_kernel<Item><<<grid, 256, 0, c->st>>>(it, n, nparts, d_counts);
  CK_LAUNCH();
  unsigned long long hc[kMaxParts];
  CK(cudaMemcpyAsync(hc, d_counts, sizeof(hc), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (cap_left)
    for (int p = 0; p < nparts; ++p)
      if (hc[p] > cap_left[p]) throw std::length_error("part capacity exceeded (skewed owner split)");
  unsigned long long base[kMaxParts], acc = 0;
  for (int p = 0; p < nparts; ++p) {
    base[p] = base_add ? base_add[p] : acc;
    acc += hc[p];
    counts_host[p] = hc[p];
  }
  CK(cudaMemcpyAsync(d_cursor, base, sizeof(unsigned long long) * nparts, cudaMemcpyHostToDevice, c->st));
  part_tile_scatter_kernel<Item><<<(unsigned)std::max<uint64_t>(tiles, 1), 256, 0, c->st>>>(it, n, nparts, d_cursor);
  CK_LAUNCH();
  c->launches += 2;
  CK(cudaStreamSynchronize(c->st));
}

template <typename F>
int guarded(nmx_ctx* c, F&& f) {
  if (!c) return fail(NMX_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  try {
    CK(cudaSetDevice(c->device));
    return f();
  } catch (const CudaError& e) {
    cudaGetLastError();
    return fail(NMX_ECUDA, "CUDA error %s (%s) at nmx_api.cu:%d", cudaGetErrorString(e.e), e.what, e.line);
  } catch (const std::bad_alloc&) {
    return fail(NMX_ENOMEM, "host allocation failed");
  } catch (const std::length_error& e) {
    return fail(NMX_ENOMEM, "%s", e.what());
  } catch (const std::exception& e) {
    return fail(NMX_EINVAL, "%s", e.what());
  }
}

int check_space(uint64_t address_space, int& b) {
  if (address_space < 1 || address_space > (1ull << 32))
    return fail(NMX_EINVAL, "address_space must lie in [1, 2^32], got %llu", (unsigned long long)address_space);
  b = std::max<int>(1, (int)ceil_log2(address_space));
  return NMX_OK;
}

void copy_out9(const unsigned long long* s, int64_t* out, uint64_t W) {
  for (uint64_t i = 0; i < W * S_COUNT; ++i) out[i] = (int64_t)s[i];
}

int check_maxaddr(nmx_ctx* c, uint64_t space);

// Addresses >= address_space -> NMX_EINVAL before any key is packed (PacketStream,
// traffic.py:56-64): an out-of-range address would carry bits above the 2b-bit key
// and index past the partition's bucket arrays. Free at address_space = 2^32.
void launch_max_addr(nmx_ctx* c, const uint32_t* s, const uint32_t* d, uint64_t n) {
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n / 4 + 255) / 256, (uint64_t)c->sms * 8));
  max_addr_kernel<<<grid, 256, 0, c->st>>>(s, d, n, c->rmax.as<unsigned int>());
  CK_LAUNCH();
  ++c->launches;
}
int check_addresses(nmx_ctx* c, const uint32_t* s, const uint32_t* d, uint64_t n, uint64_t space) {
  if (space >= (1ull << 32) || !n) return NMX_OK;
  c->rmax.grow(64);
  CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
  launch_max_addr(c, s, d, n);
  return check_maxaddr(c, space);
}

int stats_device_impl(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                      uint64_t space, uint64_t window_size, int64_t* out) {
  int b;
  if (int r = check_space(space, b)) return r;
  if (n >= (1ull << 32)) return fail(NMX_EINVAL, "n must be < 2^32 per call, got %llu", (unsigned long long)n);
  if (!out) return fail(NMX_EINVAL, "null output");
  if (n == 0) {
    if (window_size == 0) std::fill(out, out + S_COUNT, 0);
    return NMX_OK;
  }
  if (!d_src || !d_dst) return fail(NMX_EINVAL, "null packet columns");
  for (DevBuf* d : {&c->parS, &c->parD, &c->pcolD, &c->pcolC}) d->release();  // a previous out-of-core call's arenas
  const bool whole = window_size == 0 || window_size >= n;
  const int Dg = whole && graph_eligible(n) ? msd_bits(n, b) : 0;
  if (Dg) {  // small call: replay its recorded graph (address check included)
    if (nmx_ctx::CallGraph* g = graph_find(c, d_src, d_dst, d_valid, n, space)) {
      const int r = graph_replay(c, g, space);
      if (r < 0) return r;
      if (r == 1) {
        copy_out9(c->h_stats, out, 1);
        return NMX_OK;
      }
    }
  }
  // small windowed calls on the MSD path (per-window statistics) replay a recorded graph too
  const uint64_t Wg = whole ? 1 : (n + window_size - 1) / window_size;
  const int wbg = Wg > 1 ? (int)ceil_log2(Wg) : 0;
  const bool gw = !whole && graph_eligible(n) && b + wbg <= 32 && window_size >= kWinMsdMinWindow &&
                  msd_bits(n, b + wbg) >= wbg + 4;
  if (gw) {
    if (nmx_ctx::CallGraph* g = graph_find(c, d_src, d_dst, d_valid, n, space, window_size)) {
      const int r = graph_replay(c, g, space);
      if (r < 0) return r;
      if (r == 1) {
        copy_out9(c->h_stats, out, Wg);
        return NMX_OK;
      }
    }
  }
  if (int r = check_addresses(c, d_src, d_dst, n, space)) return r;
  if (whole) {
    run_pipeline(c, d_src, d_dst, d_valid, n, b, 0, 1);
    copy_out9(c->h_stats, out, 1);
    if (Dg && !c->had_heavy && !graph_find(c, d_src, d_dst, d_valid, n, space))
      graph_capture(c, d_src, d_dst, d_valid, n, b, Dg, space);
    return NMX_OK;
  }
  const uint64_t W = (n + window_size - 1) / window_size;
  const int wb = (int)ceil_log2(W);
  if (2 * b + wb <= 64) {
    run_pipeline(c, d_src, d_dst, d_valid, n, b, window_size, W);
    copy_out9(c->h_stats, out, W);
    if (gw && !c->had_heavy && !graph_find(c, d_src, d_dst, d_valid, n, space, window_size))
      graph_capture(c, d_src, d_dst, d_valid, n, b, 0, space, window_size);
    return NMX_OK;
  }
  // keys too wide to carry the window id: one window per pipeline run
  for (uint64_t t = 0; t < W; ++t) {
    const uint64_t lo = t * window_size, len = std::min(window_size, n - lo);
    run_pipeline(c, d_src + lo, d_dst + lo, d_valid ? d_valid + lo : nullptr, len, b, 0, 1);
    copy_out9(c->h_stats, out + t * S_COUNT, 1);
  }
  return NMX_OK;
}

// Host windows of packets: u32 src / dst columns (+ u8 valid or NULL per window),
// or raw 9-byte packet-file records (traffic.py:25) when `rec` is set.
struct HostWindows {
  const uint32_t* const* src = nullptr;
  const uint32_t* const* dst = nullptr;
  const uint8_t* const* valid = nullptr;
  const uint8_t* const* rec = nullptr;
  const uint64_t* lens = nullptr;
  uint64_t nwin = 0;
  // producer mode (the reference's int64 columns): window k is written by fill(k, slot)
  // into pinned slot k & 1 (whose previous copy must have left first) right before
  // its copy; src[k] / dst[k] / valid[k] then point at that slot
  std::function<void(uint64_t, int)> fill;
};

// pinned staging of the producer mode: the window's previous use of the slot must
// have been copied out before the producer overwrites it
void produce_window(nmx_ctx* c, const HostWindows& hw, uint64_t k, bool* pin_used) {
  if (!hw.fill) return;
  const int sl = (int)(k & 1);
  if (pin_used[sl]) CK(cudaEventSynchronize(c->evc[sl]));
  hw.fill(k, sl);
  pin_used[sl] = true;
}

// device records -> columns; the largest address seen is max-reduced into *maxaddr
void unpack_records(nmx_ctx* c, const uint8_t* rec, uint64_t n, uint32_t* s, uint32_t* d, uint8_t* v,
                    unsigned int* maxaddr) {
  if (!n) return;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n / 4 + 256) / 256, (uint64_t)c->sms * 8));
  unpack_records_kernel<<<grid, 256, 0, c->st>>>(rec, n, s, d, v, maxaddr);
  CK_LAUNCH();
  ++c->launches;
}

int check_maxaddr(nmx_ctx* c, uint64_t space) {
  unsigned int mx = 0;
  CK(cudaMemcpyAsync(&mx, c->rmax.p, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if ((uint64_t)mx >= space)
    return fail(NMX_EINVAL, "addresses must lie in [0, address_space): found %u >= %llu", mx,
                (unsigned long long)space);
  return NMX_OK;
}

// Streamed summed-matrix statistics (BASELINE config 5; also nmx_stats9_host and
// packet files): windows of host packets are copied on a second stream into two
// alternating device slots; the H2D copy of window k+1 overlaps the level-1 MSD
// partition of window k into the arena keysA, and the remaining levels, the
// shared-memory groups and the column statistics run once over the sum.
int stream_parts_impl(nmx_ctx* c, const HostWindows& hw, uint64_t N, uint64_t wmax, uint64_t space, bool any_valid,
                      int64_t* out);

int stream_impl(nmx_ctx* c, const HostWindows& hw, uint64_t space, int64_t* out) {
  int b;
  if (int r = check_space(space, b)) return r;
  const bool recs = hw.rec != nullptr;
  if (!out || (hw.nwin && (!hw.lens || (!recs && (!hw.src || !hw.dst))))) return fail(NMX_EINVAL, "null argument");
  uint64_t N = 0, wmax = 0;
  bool any_valid = recs;
  for (uint64_t k = 0; k < hw.nwin; ++k) {
    const bool null_cols = recs ? !hw.rec[k] : (!hw.src[k] || !hw.dst[k]);
    if (hw.lens[k] && null_cols) return fail(NMX_EINVAL, "null packet data in window %llu", (unsigned long long)k);
    N += hw.lens[k];
    wmax = std::max(wmax, hw.lens[k]);
    any_valid = any_valid || (hw.valid && hw.valid[k]);
  }
  if (N >= (1ull << 35)) return fail(NMX_EINVAL, "n must be < 2^35 per device, got %llu", (unsigned long long)N);
  // above 2^31 packets the out-of-core part split (NMX_PARTS_MIN lowers the threshold for tests)
  const char* pm = getenv("NMX_PARTS_MIN");
  const uint64_t parts_min = pm ? strtoull(pm, nullptr, 10) : (1ull << 31);
  if (N > parts_min) return stream_parts_impl(c, hw, N, wmax, space, any_valid, out);
  for (DevBuf* d : {&c->parS, &c->parD, &c->pcolD, &c->pcolC}) d->release();  // a previous out-of-core call's arenas
  const bool range = recs || space < (1ull << 32);  // address range checked on the device
  if (range) {
    c->rmax.grow(64);
    CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
  }
  const int D = msd_bits(N, b);
  if (!D) {  // small (or address space too narrow for the MSD path): one device call
    c->in_src.grow(std::max<uint64_t>(N, 1) * 4 + 16);
    c->in_dst.grow(std::max<uint64_t>(N, 1) * 4 + 16);
    if (any_valid) c->in_valid.grow(std::max<uint64_t>(N, 1) + 16);
    if (recs) c->wr0.grow(std::max<uint64_t>(wmax, 1) * 9 + 16);
    uint64_t at = 0;
    for (uint64_t k = 0; k < hw.nwin; ++k) {
      const uint64_t L = hw.lens[k];
      if (!L) continue;
      if (hw.fill) {  // the pinned slot is reused every other window: wait for its last copy
        CK(cudaStreamSynchronize(c->st));
        hw.fill(k, (int)(k & 1));
      }
      if (recs) {  // window by window through one record slot (offsets stay 16-byte aligned only at 0)
        CK(cudaMemcpyAsync(c->wr0.p, hw.rec[k], L * 9, cudaMemcpyHostToDevice, c->st));
        c->ws0.grow(L * 4 + 16);
        c->wd0.grow(L * 4 + 16);
        c->wv0.grow(L + 16);
        unpack_records(c, c->wr0.as<uint8_t>(), L, c->ws0.as<uint32_t>(), c->wd0.as<uint32_t>(), c->wv0.as<uint8_t>(),
                       c->rmax.as<unsigned int>());
        CK(cudaMemcpyAsync(c->in_src.as<uint32_t>() + at, c->ws0.p, L * 4, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(c->in_dst.as<uint32_t>() + at, c->wd0.p, L * 4, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(c->in_valid.as<uint8_t>() + at, c->wv0.p, L, cudaMemcpyDeviceToDevice, c->st));
      } else {
        CK(cudaMemcpyAsync(c->in_src.as<uint32_t>() + at, hw.src[k], L * 4, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(c->in_dst.as<uint32_t>() + at, hw.dst[k], L * 4, cudaMemcpyHostToDevice, c->st));
        if (any_valid) {
          if (hw.valid[k])
            CK(cudaMemcpyAsync(c->in_valid.as<uint8_t>() + at, hw.valid[k], L, cudaMemcpyHostToDevice, c->st));
          else
            CK(cudaMemsetAsync(c->in_valid.as<uint8_t>() + at, 1, L, c->st));
        }
      }
      at += L;
    }
    if (recs)
      if (int r = check_maxaddr(c, space)) return r;
    return stats_device_impl(c, c->in_src.as<uint32_t>(), c->in_dst.as<uint32_t>(),
                             any_valid ? c->in_valid.as<uint8_t>() : nullptr, N, space, 0, out);
  }
  if (!c->st2) CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!c->evc[i]) CK(cudaEventCreateWithFlags(&c->evc[i], cudaEventDisableTiming));
    if (!c->evu[i]) CK(cudaEventCreateWithFlags(&c->evu[i], cudaEventDisableTiming));
  }
  if (!c->evs) CK(cudaEventCreate(&c->evs));
  c->small.grow(kSmallWords * sizeof(uint32_t));  // level-1 histograms before run_pipeline_msd's stage_begin
  c->keysA.grow(N * 8);  // the arena: level-1 partitions of every window, back to back
  // levels 1 + 2 counted per window (joint histogram) when the dense split allows it
  uint32_t* joint = nullptr;
  {
    int dl[8], cum[8];
    const int L = msd_level_bits(D, dl, cum);
    c->mhist2.grow(((size_t)(1u << D) + 8) * 4);  // the size msd_partition asks for: no reallocation
    if (L >= 2 && cum[1] <= kJointMaxBits && dl[1] >= 5) {
      joint = c->mhist2.as<uint32_t>();
      CK(cudaMemsetAsync(joint, 0, sizeof(uint32_t) << cum[1], c->st));
    }
  }
  c->joint_ready = false;
  DevBuf* ws[2] = {&c->ws0, &c->ws1};
  DevBuf* wd[2] = {&c->wd0, &c->wd1};
  DevBuf* wv[2] = {&c->wv0, &c->wv1};
  DevBuf* wr[2] = {&c->wr0, &c->wr1};
  for (int i = 0; i < 2; ++i) {
    ws[i]->grow(wmax * 4 + 16);
    wd[i]->grow(wmax * 4 + 16);
    if (any_valid) wv[i]->grow(wmax + 16);
    if (recs) wr[i]->grow(wmax * 9 + 16);
  }
  CK(cudaEventRecord(c->evs, c->st));
  CK(cudaStreamWaitEvent(c->st2, c->evs, 0));  // copies start after the caller's prior work
  bool used[2] = {false, false};
  bool pin_used[2] = {false, false};
  auto enqueue_copy = [&](uint64_t k) {
    const int sl = (int)(k & 1);
    produce_window(c, hw, k, pin_used);
    if (used[sl]) CK(cudaStreamWaitEvent(c->st2, c->evu[sl], 0));
    const uint64_t L = hw.lens[k];
    if (L && recs) {
      CK(cudaMemcpyAsync(wr[sl]->p, hw.rec[k], L * 9, cudaMemcpyHostToDevice, c->st2));
    } else if (L) {
      CK(cudaMemcpyAsync(ws[sl]->p, hw.src[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      CK(cudaMemcpyAsync(wd[sl]->p, hw.dst[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      if (hw.valid && hw.valid[k]) CK(cudaMemcpyAsync(wv[sl]->p, hw.valid[k], L, cudaMemcpyHostToDevice, c->st2));
    }
    CK(cudaEventRecord(c->evc[sl], c->st2));
  };
  if (hw.nwin) enqueue_copy(0);
  uint64_t M = 0;
  for (uint64_t k = 0; k < hw.nwin; ++k) {
    if (k + 1 < hw.nwin) enqueue_copy(k + 1);
    const int sl = (int)(k & 1);
    CK(cudaStreamWaitEvent(c->st, c->evc[sl], 0));
    const uint64_t L = hw.lens[k];
    if (L) {
      if (recs)
        unpack_records(c, wr[sl]->as<uint8_t>(), L, ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(),
                       wv[sl]->as<uint8_t>(), c->rmax.as<unsigned int>());
      else if (range)
        launch_max_addr(c, ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(), L);
      const uint8_t* v = (recs || (hw.valid && hw.valid[k])) ? wv[sl]->as<uint8_t>() : nullptr;
      PacketSrc ps{ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(), v, L, 0, b};
      ps.quad = true;  // slots are cudaMalloc-aligned
      M += msd_window_level1(c, ps, 2 * b, D, c->keysA.as<uint64_t>() + M, joint);
    }
    CK(cudaEventRecord(c->evu[sl], c->st));
    used[sl] = true;
  }
  if (range)
    if (int r = check_maxaddr(c, space)) return r;
  if (!M) {
    CK(cudaStreamSynchronize(c->st));
    std::fill(out, out + S_COUNT, 0);
    return NMX_OK;
  }
  c->joint_ready = joint != nullptr;
  run_pipeline_msd(c, nullptr, nullptr, nullptr, N, b, D, M);
  CK(cudaEventElapsedTime(&c->last_total_ms, c->evs, c->ev[c->nev - 1]));  // whole streamed call
  copy_out9(c->h_stats, out, 1);
  return NMX_OK;
}

int stats_host_impl(nmx_ctx* c, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                    uint64_t space, uint64_t window_size, int64_t* out) {
  if (window_size == 0 && n >= (1ull << 20) && n < (1ull << 35) && src && dst) {
    // H2D in chunks overlapped with the level-1 partition of the previous chunk
    constexpr uint64_t kChunk = 1ull << 25;
    std::vector<const uint32_t*> ss, dd;
    std::vector<const uint8_t*> vv;
    std::vector<uint64_t> ll;
    for (uint64_t lo = 0; lo < n; lo += kChunk) {
      ss.push_back(src + lo);
      dd.push_back(dst + lo);
      vv.push_back(valid ? valid + lo : nullptr);
      ll.push_back(std::min(kChunk, n - lo));
    }
    HostWindows hw;
    hw.src = ss.data();
    hw.dst = dd.data();
    hw.valid = valid ? vv.data() : nullptr;
    hw.lens = ll.data();
    hw.nwin = ll.size();
    return stream_impl(c, hw, space, out);
  }
  if (n && (!src || !dst)) return fail(NMX_EINVAL, "null packet columns");
  if (n >= (1ull << 32)) return fail(NMX_EINVAL, "n must be < 2^32 per call, got %llu", (unsigned long long)n);
  if (n) {
    c->in_src.grow(n * 4);
    c->in_dst.grow(n * 4);
    CK(cudaMemcpyAsync(c->in_src.p, src, n * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->in_dst.p, dst, n * 4, cudaMemcpyHostToDevice, c->st));
    if (valid) {
      c->in_valid.grow(n);
      CK(cudaMemcpyAsync(c->in_valid.p, valid, n, cudaMemcpyHostToDevice, c->st));
    }
  }
  return stats_device_impl(c, c->in_src.as<uint32_t>(), c->in_dst.as<uint32_t>(),
                           valid ? c->in_valid.as<uint8_t>() : nullptr, n, space, window_size, out);
}

// Independent host batches back to back (a stream of analyses, the way a sensor feed
// arrives): batch k+1's H2D copy runs on the copy stream into the other of two device
// slots while batch k's device pipeline runs on the context stream, so a sequence of
// batches is bound by the host link, not by copy + compute. Batch k's nine statistics
// land in out[9k, 9k + 9). Each batch is one stats_device_impl call (summed matrix of
// its packets); a failing batch stops the sequence with its error.
int stats_host_batches_impl(nmx_ctx* c, uint64_t nb, const uint32_t* const* src, const uint32_t* const* dst,
                            const uint8_t* const* valid, const uint64_t* lens, uint64_t space, int64_t* out) {
  int b;
  if (int r = check_space(space, b)) return r;
  if (nb && (!src || !dst || !lens || !out)) return fail(NMX_EINVAL, "null argument");
  uint64_t nmax = 0;
  bool any_valid = false;
  for (uint64_t k = 0; k < nb; ++k) {
    if (lens[k] >= (1ull << 32))
      return fail(NMX_EINVAL, "n must be < 2^32 per batch, got %llu in batch %llu", (unsigned long long)lens[k],
                  (unsigned long long)k);
    if (lens[k] && (!src[k] || !dst[k])) return fail(NMX_EINVAL, "null packet columns in batch %llu", (unsigned long long)k);
    nmax = std::max(nmax, lens[k]);
    any_valid = any_valid || (valid && valid[k]);
  }
  if (!nb) return NMX_OK;
  if (!c->st2) CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!c->evbc[i]) CK(cudaEventCreateWithFlags(&c->evbc[i], cudaEventDisableTiming));
    if (!c->evbu[i]) CK(cudaEventCreateWithFlags(&c->evbu[i], cudaEventDisableTiming));
    c->bat_s[i].grow(std::max<uint64_t>(nmax, 1) * 4 + 16);
    c->bat_d[i].grow(std::max<uint64_t>(nmax, 1) * 4 + 16);
    if (any_valid) c->bat_v[i].grow(std::max<uint64_t>(nmax, 1) + 16);
  }
  if (!c->evs) CK(cudaEventCreate(&c->evs));
  CK(cudaEventRecord(c->evs, c->st));
  CK(cudaStreamWaitEvent(c->st2, c->evs, 0));  // copies start after the caller's prior work
  bool used[2] = {false, false};
  auto enqueue_copy = [&](uint64_t k) {
    const int sl = (int)(k & 1);
    if (used[sl]) CK(cudaStreamWaitEvent(c->st2, c->evbu[sl], 0));  // batch k-2 is done with the slot
    const uint64_t L = lens[k];
    if (L) {
      CK(cudaMemcpyAsync(c->bat_s[sl].p, src[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      CK(cudaMemcpyAsync(c->bat_d[sl].p, dst[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      if (valid && valid[k]) CK(cudaMemcpyAsync(c->bat_v[sl].p, valid[k], L, cudaMemcpyHostToDevice, c->st2));
    }
    CK(cudaEventRecord(c->evbc[sl], c->st2));
  };
  enqueue_copy(0);
  int rc = NMX_OK;
  for (uint64_t k = 0; k < nb && rc == NMX_OK; ++k) {
    if (k + 1 < nb) enqueue_copy(k + 1);
    const int sl = (int)(k & 1);
    CK(cudaStreamWaitEvent(c->st, c->evbc[sl], 0));
    const uint8_t* v = (valid && valid[k]) ? c->bat_v[sl].as<uint8_t>() : nullptr;
    rc = stats_device_impl(c, c->bat_s[sl].as<uint32_t>(), c->bat_d[sl].as<uint32_t>(), v, lens[k], space, 0,
                           out + k * S_COUNT);
    CK(cudaEventRecord(c->evbu[sl], c->st));
    used[sl] = true;
  }
  CK(cudaStreamSynchronize(c->st2));  // no copy outlives the call (host buffers are borrowed)
  return rc;
}

// int64 -> u32 narrowing of the reference's columns into pinned slots: returns whether
// an address lies outside [0, space). With AVX2, 8 packets per step and non-temporal
// 16-byte stores (the pinned slots are only read back by the DMA engine, so no
// read-for-ownership of their lines).
__attribute__((target("avx2"))) static bool narrow_u32_avx2(const int64_t* s, const int64_t* d, uint32_t* os,
                                                           uint32_t* od, uint64_t n, uint64_t space) {
  uint64_t i = 0, orr = 0;
  // scalar head until the outputs are 16-byte aligned
  for (; i < n && (((uintptr_t)(os + i) | (uintptr_t)(od + i)) & 15); ++i) {
    const uint64_t x = (uint64_t)s[i], y = (uint64_t)d[i];
    orr |= (x >= space) | (y >= space);
    os[i] = (uint32_t)x;
    od[i] = (uint32_t)y;
  }
  const __m256i lim = _mm256_set1_epi64x((long long)(space - 1) ^ (long long)0x8000000000000000ull);
  const __m256i sgn = _mm256_set1_epi64x((long long)0x8000000000000000ull);
  const __m256i pick = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i bad = _mm256_setzero_si256();
  for (; i + 4 <= n; i += 4) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i y = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(d + i));
    // unsigned x > space - 1 via the sign-flipped signed compare
    bad = _mm256_or_si256(bad, _mm256_cmpgt_epi64(_mm256_xor_si256(x, sgn), lim));
    bad = _mm256_or_si256(bad, _mm256_cmpgt_epi64(_mm256_xor_si256(y, sgn), lim));
    _mm_stream_si128(reinterpret_cast<__m128i*>(os + i),
                     _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(x, pick)));
    _mm_stream_si128(reinterpret_cast<__m128i*>(od + i),
                     _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(y, pick)));
  }
  orr |= !_mm256_testz_si256(bad, bad);
  for (; i < n; ++i) {
    const uint64_t x = (uint64_t)s[i], y = (uint64_t)d[i];
    orr |= (x >= space) | (y >= space);
    os[i] = (uint32_t)x;
    od[i] = (uint32_t)y;
  }
  _mm_sfence();
  return orr != 0;
}
static bool narrow_u32(const int64_t* s, const int64_t* d, uint32_t* os, uint32_t* od, uint64_t n, uint64_t space) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) return narrow_u32_avx2(s, d, os, od, n, space);
  uint64_t orr = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t x = (uint64_t)s[i], y = (uint64_t)d[i];
    orr |= (x >= space) | (y >= space);
    os[i] = (uint32_t)x;
    od[i] = (uint32_t)y;
  }
  return orr != 0;
}

// T host threads (the caller is thread 0) reused across jobs: run(f) calls f(t, T) on
// every thread and returns when all are done
struct NarrowPool {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(unsigned, unsigned)> job;
  uint64_t gen = 0;
  unsigned pending = 0, nt;
  bool stop = false;
  explicit NarrowPool(unsigned n) : nt(std::max(1u, n)) {
    for (unsigned t = 1; t < nt; ++t)
      th.emplace_back([this, t] {
        uint64_t seen = 0;
        for (;;) {
          std::function<void(unsigned, unsigned)> f;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return stop || gen != seen; });
            if (stop) return;
            seen = gen;
            f = job;
          }
          f(t, nt);
          std::lock_guard<std::mutex> lk(mu);
          if (--pending == 0) done_cv.notify_one();
        }
      });
  }
  void run(const std::function<void(unsigned, unsigned)>& f) {
    {
      std::lock_guard<std::mutex> lk(mu);
      job = f;
      pending = nt - 1;
      ++gen;
    }
    cv.notify_all();
    f(0, nt);
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return pending == 0; });
  }
  ~NarrowPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& x : th) x.join();
  }
};

// The reference's own columns (PacketStream: int64 src / dst, bool valid): narrowed to
// u32 on the host by a few threads per window, into two pinned slots that alternate,
// while the previous window is copied and partitioned -- the drop-in analytics.stats9
// without a pageable int64 -> u32 pass in numpy before the call.
constexpr uint64_t kWideWindow = 1ull << 24;
int stats_host_i64_impl(nmx_ctx* c, const int64_t* src, const int64_t* dst, const uint8_t* valid, uint64_t n,
                        uint64_t space, int64_t* out) {
  int b;
  if (int r = check_space(space, b)) return r;
  if (n && (!src || !dst)) return fail(NMX_EINVAL, "null packet columns");
  if (!n) {
    std::fill(out, out + S_COUNT, 0);
    return NMX_OK;
  }
  const uint64_t W = std::min<uint64_t>(kWideWindow, n);
  const uint64_t nwin = (n + W - 1) / W;
  // pinned slots: u32 src, u32 dst, u8 valid per packet, two of each
  const size_t slot = W * 9 + 64;
  if (c->wide_cap < 2 * slot) {
    if (c->h_wide) CK(cudaFreeHost(c->h_wide));
    c->h_wide = nullptr;
    c->wide_cap = 0;
    CK(cudaMallocHost(&c->h_wide, 2 * slot));
    c->wide_cap = 2 * slot;
  }
  unsigned char* base = static_cast<unsigned char*>(c->h_wide);
  uint32_t* ps[2] = {reinterpret_cast<uint32_t*>(base), reinterpret_cast<uint32_t*>(base + slot)};
  uint32_t* pd[2] = {ps[0] + W, ps[1] + W};
  uint8_t* pv[2] = {reinterpret_cast<uint8_t*>(pd[0] + W), reinterpret_cast<uint8_t*>(pd[1] + W)};
  std::vector<const uint32_t*> sp(nwin), dp(nwin);
  std::vector<const uint8_t*> vp(nwin);
  std::vector<uint64_t> lens(nwin);
  for (uint64_t k = 0; k < nwin; ++k) {
    sp[k] = ps[k & 1];
    dp[k] = pd[k & 1];
    vp[k] = valid ? pv[k & 1] : nullptr;
    lens[k] = std::min(W, n - k * W);
  }
  const unsigned hw_threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<bool> bad{false};
  // one pool for the whole call (a window is 2^24 packets: spawning threads per window
  // cost more than the narrowing of a small one)
  const unsigned T = (unsigned)std::min<uint64_t>(hw_threads, (W + 65535) / 65536);
  NarrowPool pool(T);
  HostWindows hw;
  hw.src = sp.data();
  hw.dst = dp.data();
  hw.valid = valid ? vp.data() : nullptr;
  hw.lens = lens.data();
  hw.nwin = nwin;
  hw.fill = [&](uint64_t k, int sl) {
    const uint64_t lo = k * W, L = lens[k];
    pool.run([&](unsigned t, unsigned nt) {
      const uint64_t a = (L * t / nt) & ~7ull, z = t + 1 == nt ? L : (L * (t + 1) / nt) & ~7ull;
      if (narrow_u32(src + lo + a, dst + lo + a, ps[sl] + a, pd[sl] + a, z - a, space)) bad = true;
      if (valid) memcpy(pv[sl] + a, valid + lo + a, z - a);
    });
  };
  const int rc = stream_impl(c, hw, space, out);
  if (bad) return fail(NMX_EINVAL, "addresses must lie in [0, address_space)");
  return rc;
}

// ---- multi-GPU shard stages; callers hold the context lock ----
// link + row statistics (fields 0-5) of the packets whose sources this rank owns,
// and its unique links' (dst, count) column entries routed by owner(dst)
int shard_rows_impl(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t space, int nparts,
                    uint32_t* d_out_dst, uint32_t* d_out_count, uint64_t* counts, int64_t* out,
                    const uint64_t* base_add = nullptr, const uint64_t* cap_left = nullptr) {
  int b;
  if (int r = check_space(space, b)) return r;
  std::fill(out, out + S_COUNT, 0);
  std::fill(counts, counts + nparts, 0);
  if (!n) return NMX_OK;
  if (int r = check_addresses(c, d_src, d_dst, n, space)) return r;
  stage_begin(c, 1);
  if (const int D = msd_bits(n, b)) {  // MSD rows; column slots (holes skipped) by owner(dst)
    uint32_t* chist = nullptr;
    const ColConcatSrc cs = msd_rows(c, d_src, d_dst, nullptr, n, b, D, 0, &chist);
    if (cs.n) {
      ColConcatPart it{cs, d_out_dst, d_out_count};
      partition_items(c, it, cs.n, nparts, counts, base_add, cap_left);
    }
  } else {
    PacketSrc ps{d_src, d_dst, nullptr, n, 0, b};
    const RowsOut r = stage_rows(c, ps, b, 0);
    if (r.u) {
      ColPart it{c->ckA.as<uint32_t>(), c->cvA.as<uint32_t>(), d_out_dst, d_out_count};
      partition_items(c, it, r.u, nparts, counts, base_add, cap_left);
    }
  }
  stage_finish(c, 1);
  copy_out9(c->h_stats, out, 1);
  return NMX_OK;
}

// column statistics (fields 6-8) of the received column entries of this rank's destinations
int shard_cols_impl(nmx_ctx* c, const uint32_t* d_dst, const uint32_t* d_count, uint64_t u, uint64_t space,
                    int64_t* out) {
  int b;
  if (int r = check_space(space, b)) return r;
  std::fill(out, out + S_COUNT, 0);
  if (!u) return NMX_OK;
  if (int r = check_addresses(c, d_dst, d_dst, u, space)) return r;
  stage_begin(c, 1);
  c->ckA.grow(u * 4);
  c->ckB.grow(u * 4);
  c->cvA.grow(u * 4);
  c->cvB.grow(u * 4);
  if (const int Dc = msd_bits(u, b)) {  // MSD column partition + shared-memory groups
    c->colL_dst.grow(u * 8);
    pack_cols_kernel<<<c->sms * 8, 256, 0, c->st>>>(d_dst, d_count, u, c->colL_dst.as<uint64_t>());
    CK_LAUNCH();
    ++c->launches;
    ColConcatSrc cs{c->colL_dst.as<uint64_t>(), u, nullptr, 0, u};
    cs.quad = true;
    msd_columns(c, cs, b, Dc, nullptr);
    stage_finish(c, 1);
    copy_out9(c->h_stats, out, 1);
    return NMX_OK;
  }
  if (c->csstatus.grow(tiles_of(u, kSegTile) * sizeof(CSStatus)))
    CK(cudaMemsetAsync(c->csstatus.p, 0, c->csstatus.cap, c->st));
  CK(cudaMemcpyAsync(c->ckA.p, d_dst, u * 4, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(c->cvA.p, d_count, u * 4, cudaMemcpyDeviceToDevice, c->st));
  const int ncolpass = (b + 7) / 8;
  uint32_t* d_small = c->small.as<uint32_t>();
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((u + 1023) / 1024, (uint64_t)c->sms * 8));
  switch (ncolpass) {
    case 1: hist_u32_kernel<1><<<grid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), u, d_small + kCHist); break;
    case 2: hist_u32_kernel<2><<<grid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), u, d_small + kCHist); break;
    case 3: hist_u32_kernel<3><<<grid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), u, d_small + kCHist); break;
    default: hist_u32_kernel<4><<<grid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), u, d_small + kCHist); break;
  }
  CK_LAUNCH();
  ++c->launches;
  stage_cols(c, (uint32_t)u, b, 0, false);
  stage_finish(c, 1);
  copy_out9(c->h_stats, out, 1);
  return NMX_OK;
}

// Out-of-core summed statistics of more than 2^31 packets on one device (BASELINE
// config 5: 2^32 packets streamed from pinned host memory): the sharded pipeline of
// SURVEY.md 8(e) with its ranks run one after another on this context. Every window is
// partitioned on arrival into P source-part arenas by owner(src) = (fmix32(src) P) >> 32
// (a part holds whole sources, < 2^31 packets); each part's links and rows are finished
// by the MSD row half, its unique links' (dst, count) routed by owner(dst) into P
// column-part arenas; each column part is finished by the MSD column half. Parts are
// disjoint by source / destination, so the statistics combine by SUM / MAX -- exactly
// the one-pass result (bit-identical, tests/golden/full_size.json cfg5 cases).
int stream_parts_impl(nmx_ctx* c, const HostWindows& hw, uint64_t N, uint64_t wmax, uint64_t space, bool any_valid,
                      int64_t* out) {
  const bool recs = hw.rec != nullptr;
  const bool range = recs || space < (1ull << 32);
  int P = 2;
  auto cap_of = [&](int parts) { return N / parts + N / (4 * (uint64_t)parts) + (1ull << 22); };
  while (cap_of(P) >= (1ull << 31) - (1ull << 22)) P *= 2;
  if (P > kMaxParts) return fail(NMX_EINVAL, "too many packets for one device");
  const uint64_t cap = cap_of(P);
  // the part arenas come first: workspace grown by earlier (larger single-pass) calls is
  // dropped and regrown at part size; part-sized workspace (an earlier out-of-core call's)
  // is kept -- reallocating tens of GB per call cost ~0.5 s
  const size_t part_ws = (size_t)cap * 8 + (size_t)cap / 8 * 8 + (512ull << 20);
  for (DevBuf* d : {&c->keysA, &c->keysB, &c->keysC, &c->keysD, &c->colL_dst, &c->ckA, &c->ckB, &c->cvA, &c->cvB,
                    &c->cgk, &c->cgk2, &c->in_src, &c->in_dst, &c->in_valid, &c->lightK})
    if (d->cap > part_ws) d->release();
  for (DevBuf* d : {&c->pcolD, &c->pcolC})
    if (d->cap > (size_t)P * cap * 4 + (512ull << 20)) d->release();
  c->parS.grow((size_t)P * cap * 4);
  c->parD.grow((size_t)P * cap * 4);
  if (range) {
    c->rmax.grow(64);
    CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
  }
  if (!c->st2) CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!c->evc[i]) CK(cudaEventCreateWithFlags(&c->evc[i], cudaEventDisableTiming));
    if (!c->evu[i]) CK(cudaEventCreateWithFlags(&c->evu[i], cudaEventDisableTiming));
  }
  if (!c->evs) CK(cudaEventCreate(&c->evs));
  DevBuf* ws[2] = {&c->ws0, &c->ws1};
  DevBuf* wd[2] = {&c->wd0, &c->wd1};
  DevBuf* wv[2] = {&c->wv0, &c->wv1};
  DevBuf* wr[2] = {&c->wr0, &c->wr1};
  for (int i = 0; i < 2; ++i) {
    ws[i]->grow(wmax * 4 + 16);
    wd[i]->grow(wmax * 4 + 16);
    if (any_valid) wv[i]->grow(wmax + 16);
    if (recs) wr[i]->grow(wmax * 9 + 16);
  }
  CK(cudaEventRecord(c->evs, c->st));
  CK(cudaStreamWaitEvent(c->st2, c->evs, 0));
  bool used[2] = {false, false};
  bool pin_used[2] = {false, false};
  auto enqueue_copy = [&](uint64_t k) {
    const int sl = (int)(k & 1);
    produce_window(c, hw, k, pin_used);
    if (used[sl]) CK(cudaStreamWaitEvent(c->st2, c->evu[sl], 0));
    const uint64_t L = hw.lens[k];
    if (L && recs) {
      CK(cudaMemcpyAsync(wr[sl]->p, hw.rec[k], L * 9, cudaMemcpyHostToDevice, c->st2));
    } else if (L) {
      CK(cudaMemcpyAsync(ws[sl]->p, hw.src[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      CK(cudaMemcpyAsync(wd[sl]->p, hw.dst[k], L * 4, cudaMemcpyHostToDevice, c->st2));
      if (hw.valid && hw.valid[k]) CK(cudaMemcpyAsync(wv[sl]->p, hw.valid[k], L, cudaMemcpyHostToDevice, c->st2));
    }
    CK(cudaEventRecord(c->evc[sl], c->st2));
  };
  // NMX_DEBUG: wall-clock phase times (each phase end synchronizes the stream)
  const bool dbg = getenv("NMX_DEBUG") != nullptr;
  auto t_phase = std::chrono::steady_clock::now();
  auto phase_done = [&](const char* what) {
    if (!dbg) return;
    CK(cudaStreamSynchronize(c->st));
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "stream_parts %s: %.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t_phase).count());
    t_phase = t;
  };
  // 1. windows -> source-part arenas (the copy of window k+1 overlaps window k's split)
  uint64_t fill[kMaxParts] = {0}, base[kMaxParts], left[kMaxParts], cnt[kMaxParts];
  if (hw.nwin) enqueue_copy(0);
  for (uint64_t k = 0; k < hw.nwin; ++k) {
    if (k + 1 < hw.nwin) enqueue_copy(k + 1);
    const int sl = (int)(k & 1);
    CK(cudaStreamWaitEvent(c->st, c->evc[sl], 0));
    const uint64_t L = hw.lens[k];
    if (L) {
      if (recs)
        unpack_records(c, wr[sl]->as<uint8_t>(), L, ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(),
                       wv[sl]->as<uint8_t>(), c->rmax.as<unsigned int>());
      else if (range)
        launch_max_addr(c, ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(), L);
      const uint8_t* v = (recs || (hw.valid && hw.valid[k])) ? wv[sl]->as<uint8_t>() : nullptr;
      for (int p = 0; p < P; ++p) {
        base[p] = p * cap + fill[p];
        left[p] = cap - fill[p];
      }
      PacketPart it{ws[sl]->as<uint32_t>(), wd[sl]->as<uint32_t>(), v, c->parS.as<uint32_t>(), c->parD.as<uint32_t>()};
      partition_items(c, it, L, P, cnt, base, left);  // host-synchronous: the next copy is already queued
      for (int p = 0; p < P; ++p) fill[p] += cnt[p];
    }
    CK(cudaEventRecord(c->evu[sl], c->st));
    used[sl] = true;
  }
  if (range)
    if (int r = check_maxaddr(c, space)) return r;
  phase_done("1 copies + owner(src) split");
  // 2. rows per source part; column entries -> destination-part arenas
  c->pcolD.grow((size_t)P * cap * 4);
  c->pcolC.grow((size_t)P * cap * 4);
  uint64_t cfill[kMaxParts] = {0};
  int64_t tot[S_COUNT] = {0};
  static const bool kSum[S_COUNT] = {true, true, false, true, false, false, true, false, false};
  auto fold = [&](const int64_t* s9, int lo, int hi) {
    for (int i = lo; i < hi; ++i) tot[i] = kSum[i] ? tot[i] + s9[i] : std::max(tot[i], s9[i]);
  };
  for (int p = 0; p < P; ++p) {
    if (!fill[p]) continue;
    for (int q = 0; q < P; ++q) {
      base[q] = q * cap + cfill[q];
      left[q] = cap - cfill[q];
    }
    int64_t row9[S_COUNT];
    if (int r = shard_rows_impl(c, c->parS.as<uint32_t>() + p * cap, c->parD.as<uint32_t>() + p * cap, fill[p], space,
                                P, c->pcolD.as<uint32_t>(), c->pcolC.as<uint32_t>(), cnt, row9, base, left))
      return r;
    for (int q = 0; q < P; ++q) cfill[q] += cnt[q];
    fold(row9, 0, 6);
    if (dbg) {
      fprintf(stderr, "  part %d: %llu packets, device %.2f ms, stages", p, (unsigned long long)fill[p], c->last_total_ms);
      for (int i = 0; i < c->last_nstage; ++i) fprintf(stderr, " %.2f", c->last_stage_ms[i]);
      fprintf(stderr, "\n");
    }
  }
  phase_done("2 rows per source part");
  // 3. columns per destination part
  for (int q = 0; q < P; ++q) {
    if (!cfill[q]) continue;
    int64_t col9[S_COUNT];
    if (int r = shard_cols_impl(c, c->pcolD.as<uint32_t>() + q * cap, c->pcolC.as<uint32_t>() + q * cap, cfill[q],
                                space, col9))
      return r;
    fold(col9, 6, 9);
  }
  phase_done("3 columns per destination part");
  std::copy(tot, tot + S_COUNT, out);
  c->last_nstage = 0;
  return NMX_OK;
}

// ---- device groups: one process driving G contexts ----------
// A group is G ranks, each an nmx_ctx (its own stream and workspace) on a device;
// virtual ranks may share a device. nmx_group_stats9_* run one host thread per
// rank through the owner(src) / owner(dst) pipeline of distributed.py, with the two
// all-to-all exchanges done in-library as peer copies (cudaMemcpyPeerAsync: NVLink /
// NVSwitch between distinct B200s, a device-local copy between virtual ranks) and
// cross-stream events instead of a host round trip through NCCL.

// barrier that a failing rank can abort (the others then unwind instead of hanging)
struct GroupBarrier {
  std::mutex mu;
  std::condition_variable cv;
  int n = 0, waiting = 0;
  uint64_t gen = 0;
  bool aborted = false;
  void arrive() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw std::runtime_error("group aborted by another rank");
    const uint64_t g = gen;
    if (++waiting == n) {
      waiting = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (aborted) throw std::runtime_error("group aborted by another rank");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct GroupRank {
  nmx_ctx* ctx = nullptr;
  DevBuf ps, pd;    // exchange 1 send: packets by owner(src)
  DevBuf rs, rd;    // exchange 1 receive
  DevBuf cs, cc;    // exchange 2 send: column entries by owner(dst)
  DevBuf qs, qc;    // exchange 2 receive
  DevBuf hs, hd, hv;  // host variant: this rank's span on the device
  uint64_t cnt1[kMaxParts] = {0}, cnt2[kMaxParts] = {0};
  int64_t st[S_COUNT] = {0};
  cudaEvent_t ev = nullptr;
  int rc = NMX_OK;
  std::string err;
};

}  // namespace

struct nmx_group {
  int g = 0;
  std::vector<int> devices;
  std::vector<GroupRank> ranks;
  std::mutex mu;  // one group call at a time
  GroupBarrier bar;
  uint64_t last_x1 = 0, last_x2 = 0;  // bytes moved by the last call's exchanges
};

namespace {

// exchange `k` of rank r: its part p (count cnt[p], at offset sum_{q<p} cnt[q] of the
// send buffers) goes to rank p at offset sum_{r'<r} cnt_{r'}[p]; two u32 columns.
void group_exchange(nmx_group* G, int r, DevBuf GroupRank::*sa, DevBuf GroupRank::*sb, DevBuf GroupRank::*ra,
                    DevBuf GroupRank::*rb, uint64_t (GroupRank::*cnt)[kMaxParts], uint64_t* recv_total) {
  GroupRank& me = G->ranks[r];
  // receive size, then buffers grown before anyone writes into them
  uint64_t tot = 0;
  for (int q = 0; q < G->g; ++q) tot += (G->ranks[q].*cnt)[r];
  (me.*ra).grow(std::max<uint64_t>(tot, 1) * 4);
  (me.*rb).grow(std::max<uint64_t>(tot, 1) * 4);
  *recv_total = tot;
  G->bar.arrive();  // every receive buffer exists
  uint64_t soff = 0;
  for (int p = 0; p < G->g; ++p) {
    const uint64_t len = (me.*cnt)[p];
    if (len) {
      uint64_t roff = 0;
      for (int q = 0; q < r; ++q) roff += (G->ranks[q].*cnt)[p];
      GroupRank& peer = G->ranks[p];
      const int sdev = me.ctx->device, ddev = peer.ctx->device;
      CK(cudaMemcpyPeerAsync((peer.*ra).as<uint32_t>() + roff, ddev,
                             (me.*sa).as<uint32_t>() + soff, sdev, len * 4, me.ctx->st));
      CK(cudaMemcpyPeerAsync((peer.*rb).as<uint32_t>() + roff, ddev, (me.*sb).as<uint32_t>() + soff, sdev, len * 4,
                             me.ctx->st));
    }
    soff += len;
  }
  CK(cudaEventRecord(me.ev, me.ctx->st));
  G->bar.arrive();  // every send is queued (events recorded)
  for (int q = 0; q < G->g; ++q)
    if (q != r) CK(cudaStreamWaitEvent(me.ctx->st, G->ranks[q].ev, 0));
}

// rank r's share of a group call; d_src / d_dst / d_valid = its n packets on its device
void group_rank_run(nmx_group* G, int r, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                    uint64_t n, uint64_t space) {
  GroupRank& me = G->ranks[r];
  nmx_ctx* c = me.ctx;
  const int g = G->g;
  // exchange 1: valid packets by owner(src)
  me.ps.grow(std::max<uint64_t>(n, 1) * 4);
  me.pd.grow(std::max<uint64_t>(n, 1) * 4);
  std::fill(me.cnt1, me.cnt1 + kMaxParts, 0);
  std::fill(me.cnt2, me.cnt2 + kMaxParts, 0);
  if (n) {
    if (int rc = check_addresses(c, d_src, d_dst, n, space)) throw std::runtime_error(g_err);
    PacketPart it{d_src, d_dst, d_valid, me.ps.as<uint32_t>(), me.pd.as<uint32_t>()};
    partition_items(c, it, n, g, me.cnt1);
  }
  G->bar.arrive();  // counts published
  uint64_t m = 0;
  group_exchange(G, r, &GroupRank::ps, &GroupRank::pd, &GroupRank::rs, &GroupRank::rd, &GroupRank::cnt1, &m);
  // links + rows of this rank's sources; column entries by owner(dst)
  me.cs.grow(std::max<uint64_t>(m, 1) * 4);
  me.cc.grow(std::max<uint64_t>(m, 1) * 4);
  int64_t row9[S_COUNT], col9[S_COUNT];
  if (m >= (1ull << 32)) throw std::runtime_error("more than 2^32-1 packets routed to one rank");
  if (int rc = shard_rows_impl(c, me.rs.as<uint32_t>(), me.rd.as<uint32_t>(), m, space, g, me.cs.as<uint32_t>(),
                               me.cc.as<uint32_t>(), me.cnt2, row9))
    throw std::runtime_error(g_err);
  G->bar.arrive();  // counts published
  uint64_t u = 0;
  group_exchange(G, r, &GroupRank::cs, &GroupRank::cc, &GroupRank::qs, &GroupRank::qc, &GroupRank::cnt2, &u);
  if (int rc = shard_cols_impl(c, me.qs.as<uint32_t>(), me.qc.as<uint32_t>(), u, space, col9))
    throw std::runtime_error(g_err);
  CK(cudaStreamSynchronize(c->st));
  for (int i = 0; i < S_COUNT; ++i) me.st[i] = i < 6 ? row9[i] : col9[i];
}

// one host thread per rank; results combined as the final SUM / MAX all-reduce
int group_run(nmx_group* G, const std::function<void(int)>& body, int64_t* out) {
  std::lock_guard<std::mutex> lk(G->mu);
  G->bar.n = G->g;
  G->bar.waiting = 0;
  G->bar.aborted = false;
  std::vector<std::thread> th;
  for (int r = 0; r < G->g; ++r) {
    G->ranks[r].rc = NMX_OK;
    th.emplace_back([G, r, &body] {
      GroupRank& me = G->ranks[r];
      std::lock_guard<std::mutex> clk(me.ctx->mu);
      try {
        CK(cudaSetDevice(me.ctx->device));
        if (!me.ev) CK(cudaEventCreateWithFlags(&me.ev, cudaEventDisableTiming));
        body(r);
      } catch (const CudaError& e) {
        cudaGetLastError();
        me.rc = NMX_ECUDA;
        char b[256];
        snprintf(b, sizeof(b), "rank %d: CUDA error %s (%s) at nmx_api.cu:%d", r, cudaGetErrorString(e.e), e.what,
                 e.line);
        me.err = b;
        G->bar.abort();
      } catch (const std::bad_alloc&) {
        me.rc = NMX_ENOMEM;
        me.err = "host allocation failed";
        G->bar.abort();
      } catch (const std::exception& e) {
        me.rc = NMX_EINVAL;
        me.err = std::string("rank ") + std::to_string(r) + ": " + e.what();
        G->bar.abort();
      }
    });
  }
  for (auto& t : th) t.join();
  // the first real failure wins over the "aborted by another rank" echoes
  int rc = NMX_OK;
  std::string msg;
  for (auto& rk : G->ranks)
    if (rk.rc != NMX_OK && (rc == NMX_OK || msg.find("aborted") != std::string::npos) &&
        rk.err.find("aborted by another rank") == std::string::npos) {
      rc = rk.rc;
      msg = rk.err;
    }
  if (rc == NMX_OK)
    for (auto& rk : G->ranks)
      if (rk.rc != NMX_OK) rc = rk.rc, msg = rk.err;
  if (rc != NMX_OK) return fail(rc, "%s", msg.c_str());
  static const bool kSum[S_COUNT] = {true, true, false, true, false, false, true, false, false};
  for (int i = 0; i < S_COUNT; ++i) {
    int64_t v = 0;
    for (auto& rk : G->ranks) v = kSum[i] ? v + rk.st[i] : std::max(v, rk.st[i]);
    out[i] = v;
  }
  G->last_x1 = G->last_x2 = 0;
  for (auto& rk : G->ranks)
    for (int p = 0; p < G->g; ++p) {
      G->last_x1 += rk.cnt1[p] * 8;
      G->last_x2 += rk.cnt2[p] * 8;
    }
  return NMX_OK;
}

// ---- NCCL communicators: one process per GPU -----------------
// The multi-process form of the sharded pipeline: each rank is a process with its own
// nmx_ctx and one NCCL communicator. Both all-to-all exchanges are grouped
// ncclSend / ncclRecv on the context stream (src and dst columns of a part in one
// group, so NCCL moves them together over NVLink / NVSwitch), the per-part counts an
// ncclAllGather, and the final combine two ncclAllReduce (SUM, MAX) on int64 -- no
// host staging, no torch on the data path.
struct CommBufs {
  DevBuf ps, pd, rs, rd, cs, cc, qs, qc, hs, hd, hv, cnt, red;
};

// libnccl is opened on first use instead of linked: a process that also imports
// torch must share torch's NCCL (same soname, newer symbols), so NMX_NCCL_LIB
// (set by _lib.Communicator to the bundled nvidia-nccl library when present) wins
// over the system libnccl.so.2.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};
const NcclApi* nccl_api() {
  static std::once_flag once;
  static NcclApi api;
  static bool ok = false;
  std::call_once(once, [] {
    const char* want = getenv("NMX_NCCL_LIB");
    void* h = want && *want ? dlopen(want, RTLD_NOW | RTLD_GLOBAL) : nullptr;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    bool all = true;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      all = all && f;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    ok = all;
  });
  if (!ok) throw std::runtime_error("NCCL library not found (libnccl.so.2 / NMX_NCCL_LIB)");
  return &api;
}

#define NK(x)                                                                                          \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + nccl_api()->GetErrorString(r_)); \
  } while (0)

}  // namespace

struct nmx_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
  CommBufs b;
  uint64_t last_x1 = 0, last_x2 = 0;
};

namespace {

// rank r sends part p of (sa, sb) (cnt[p] items, parts back to back) to rank p and
// receives every rank's part r into (ra, rb) in rank order; returns the items received
uint64_t comm_exchange(nmx_comm* K, nmx_ctx* c, const uint32_t* sa, const uint32_t* sb, const uint64_t* cnt,
                       DevBuf& ra, DevBuf& rb) {
  const int g = K->nranks, r = K->rank;
  K->b.cnt.grow((size_t)(g + 1) * g * 8);
  auto* dc = K->b.cnt.as<unsigned long long>();
  std::vector<unsigned long long> mine(cnt, cnt + g), all((size_t)g * g);
  CK(cudaMemcpyAsync(dc + (size_t)g * g, mine.data(), g * 8, cudaMemcpyHostToDevice, c->st));
  NK(nccl_api()->AllGather(dc + (size_t)g * g, dc, g, ncclUint64, K->comm, c->st));
  CK(cudaMemcpyAsync(all.data(), dc, (size_t)g * g * 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  uint64_t tot = 0;
  for (int q = 0; q < g; ++q) tot += all[(size_t)q * g + r];
  ra.grow(std::max<uint64_t>(tot, 1) * 4);
  rb.grow(std::max<uint64_t>(tot, 1) * 4);
  NK(nccl_api()->GroupStart());
  uint64_t soff = 0, roff = 0;
  for (int p = 0; p < g; ++p) {
    const uint64_t sl = cnt[p], rl = all[(size_t)p * g + r];
    if (sl) {
      NK(nccl_api()->Send(sa + soff, sl, ncclUint32, p, K->comm, c->st));
      NK(nccl_api()->Send(sb + soff, sl, ncclUint32, p, K->comm, c->st));
    }
    if (rl) {
      NK(nccl_api()->Recv(ra.as<uint32_t>() + roff, rl, ncclUint32, p, K->comm, c->st));
      NK(nccl_api()->Recv(rb.as<uint32_t>() + roff, rl, ncclUint32, p, K->comm, c->st));
    }
    soff += sl;
    roff += rl;
  }
  NK(nccl_api()->GroupEnd());
  return tot;
}

// this rank's share: exchange 1 (owner(src)), links + rows, exchange 2 (owner(dst)),
// columns, SUM / MAX all-reduce of the nine statistics
int comm_run(nmx_comm* K, nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
             uint64_t n, uint64_t space, int64_t* out) {
  const int g = K->nranks;
  uint64_t cnt1[kMaxParts] = {0}, cnt2[kMaxParts] = {0};
  K->b.ps.grow(std::max<uint64_t>(n, 1) * 4);
  K->b.pd.grow(std::max<uint64_t>(n, 1) * 4);
  if (n) {
    if (int rc = check_addresses(c, d_src, d_dst, n, space)) return rc;
    PacketPart it{d_src, d_dst, d_valid, K->b.ps.as<uint32_t>(), K->b.pd.as<uint32_t>()};
    partition_items(c, it, n, g, cnt1);
  }
  const uint64_t m = comm_exchange(K, c, K->b.ps.as<uint32_t>(), K->b.pd.as<uint32_t>(), cnt1, K->b.rs, K->b.rd);
  if (m >= (1ull << 32)) throw std::runtime_error("more than 2^32-1 packets routed to one rank");
  K->b.cs.grow(std::max<uint64_t>(m, 1) * 4);
  K->b.cc.grow(std::max<uint64_t>(m, 1) * 4);
  int64_t row9[S_COUNT], col9[S_COUNT];
  if (int rc = shard_rows_impl(c, K->b.rs.as<uint32_t>(), K->b.rd.as<uint32_t>(), m, space, g,
                               K->b.cs.as<uint32_t>(), K->b.cc.as<uint32_t>(), cnt2, row9))
    return rc;
  const uint64_t u = comm_exchange(K, c, K->b.cs.as<uint32_t>(), K->b.cc.as<uint32_t>(), cnt2, K->b.qs, K->b.qc);
  if (int rc = shard_cols_impl(c, K->b.qs.as<uint32_t>(), K->b.qc.as<uint32_t>(), u, space, col9)) return rc;
  static const bool kSum[S_COUNT] = {true, true, false, true, false, false, true, false, false};
  int64_t sv[2 * S_COUNT];
  for (int i = 0; i < S_COUNT; ++i) {
    const int64_t v = i < 6 ? row9[i] : col9[i];
    sv[i] = kSum[i] ? v : 0;
    sv[S_COUNT + i] = kSum[i] ? 0 : v;
  }
  K->b.red.grow(2 * S_COUNT * 8);
  auto* dr = K->b.red.as<int64_t>();
  CK(cudaMemcpyAsync(dr, sv, sizeof(sv), cudaMemcpyHostToDevice, c->st));
  NK(nccl_api()->GroupStart());
  NK(nccl_api()->AllReduce(dr, dr, S_COUNT, ncclInt64, ncclSum, K->comm, c->st));
  NK(nccl_api()->AllReduce(dr + S_COUNT, dr + S_COUNT, S_COUNT, ncclInt64, ncclMax, K->comm, c->st));
  NK(nccl_api()->GroupEnd());
  CK(cudaMemcpyAsync(sv, dr, sizeof(sv), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (int i = 0; i < S_COUNT; ++i) out[i] = kSum[i] ? sv[i] : sv[S_COUNT + i];
  K->last_x1 = K->last_x2 = 0;
  for (int p = 0; p < g; ++p) {
    K->last_x1 += cnt1[p] * 8;
    K->last_x2 += cnt2[p] * 8;
  }
  return NMX_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int nmx_version(void) { return 1; }

const char* nmx_last_error(void) { return g_err.c_str(); }

int nmx_device_count(int* count) {
  if (!count) return fail(NMX_EINVAL, "null count");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(NMX_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  }
  return NMX_OK;
}

int nmx_create(int device, nmx_ctx** out) {
  if (!out) return fail(NMX_EINVAL, "null out");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(NMX_ENODEV, "no CUDA device visible");
  }
  if (device < 0 || device >= n) return fail(NMX_EINVAL, "device %d out of range [0,%d)", device, n);
  nmx_ctx* c = new (std::nothrow) nmx_ctx();
  if (!c) return fail(NMX_ENOMEM, "context allocation failed");
  c->device = device;
  try {
    CK(cudaSetDevice(device));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    if (p.major < 10) {
      delete c;
      return fail(NMX_ENODEV, "device %d is sm_%d%d; libnmx.so is built for sm_100a only", device, p.major, p.minor);
    }
    c->sms = p.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    for (auto& e : c->evk) CK(cudaEventCreate(&e));
  } catch (const CudaError& e) {
    cudaGetLastError();
    delete c;
    return fail(NMX_ECUDA, "CUDA error %s (%s)", cudaGetErrorString(e.e), e.what);
  }
  *out = c;
  return NMX_OK;
}

void nmx_destroy(nmx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  for (DevBuf* b : {&c->mpcnt, &c->mpoff, &c->mscan, &c->mch, &c->mgh, &c->mplan, &c->keysA, &c->keysB, &c->keysC, &c->keysD, &c->cgk, &c->cgv, &c->cgk2, &c->cgv2, &c->colL_dst, &c->colL_cnt, &c->mcur, &c->moff,
                    &c->mhist2, &c->mgb, &c->mheavy, &c->mdst, &c->ckA, &c->ckB, &c->cvA, &c->cvB, &c->status, &c->lrstatus,
                    &c->csstatus, &c->part, &c->rbstatus, &c->mkeys, &c->mlen, &c->msum, &c->ckeys2, &c->clen2, &c->csum2,
                    &c->frows, &c->small, &c->stats, &c->in_src, &c->in_dst, &c->in_valid, &c->red, &c->ws0, &c->ws1,
                    &c->wd0, &c->wd1, &c->wv0, &c->wv1, &c->wr0, &c->wr1, &c->bat_s[0], &c->bat_s[1], &c->bat_d[0],
                    &c->bat_d[1], &c->bat_v[0], &c->bat_v[1], &c->mhist3, &c->moff1, &c->mtpar})
    b->release();
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->h_wide) cudaFreeHost(c->h_wide);
  if (c->h_small) cudaFreeHost(c->h_small);
  if (c->h_scr) cudaFreeHost(c->h_scr);
  if (c->evw) cudaEventDestroy(c->evw);
  if (c->h_stats) cudaFreeHost(c->h_stats);
  for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->evk) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->evc[0], c->evc[1], c->evu[0], c->evu[1], c->evs, c->evbc[0], c->evbc[1], c->evbu[0],
                        c->evbu[1]})
    if (e) cudaEventDestroy(e);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
}

void* nmx_stream(nmx_ctx* c) { return c ? (void*)c->st : nullptr; }

int nmx_synchronize(nmx_ctx* c) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_malloc(nmx_ctx* c, uint64_t bytes, void** dptr) {
  if (!dptr) return fail(NMX_EINVAL, "null out");
  return guarded(c, [&] {
    cudaError_t e = cudaMalloc(dptr, std::max<uint64_t>(bytes, 1));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(NMX_ENOMEM, "cudaMalloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    }
    return NMX_OK;
  });
}

int nmx_free(nmx_ctx* c, void* dptr) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->st));
    CK(cudaFree(dptr));
    return NMX_OK;
  });
}

int nmx_host_alloc(uint64_t bytes, void** hptr) {
  if (!hptr) return fail(NMX_EINVAL, "null out");
  cudaError_t e = cudaMallocHost(hptr, std::max<uint64_t>(bytes, 1));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(NMX_ENOMEM, "cudaMallocHost(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
  }
  return NMX_OK;
}

int nmx_host_free(void* hptr) {
  cudaError_t e = cudaFreeHost(hptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(NMX_ECUDA, "cudaFreeHost failed: %s", cudaGetErrorString(e));
  }
  return NMX_OK;
}

int nmx_memcpy_h2d(nmx_ctx* c, void* dst, const void* src, uint64_t bytes) {
  return guarded(c, [&] {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_memcpy_d2h(nmx_ctx* c, void* dst, const void* src, uint64_t bytes) {
  return guarded(c, [&] {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_generate(nmx_ctx* c, int kind, uint64_t seed, uint64_t offset, uint64_t n, uint64_t address_space,
                 uint32_t* d_src, uint32_t* d_dst) {
  if (kind != NMX_GEN_UNIFORM && kind != NMX_GEN_POWERLAW) return fail(NMX_EINVAL, "unknown generator %d", kind);
  if (address_space < 1 || address_space > (1ull << 32)) return fail(NMX_EINVAL, "address_space out of range");
  return guarded(c, [&] {
    if (!n) return NMX_OK;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 16);
    gen_kernel<<<grid, 256, 0, c->st>>>(kind, seed, offset, n, address_space, d_src, d_dst);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_stats9_device(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid, uint64_t n,
                      uint64_t address_space, int64_t out[9]) {
  return guarded(c, [&] { return stats_device_impl(c, d_src, d_dst, d_valid, n, address_space, 0, out); });
}

int nmx_stats9_host(nmx_ctx* c, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                    uint64_t address_space, int64_t out[9]) {
  return guarded(c, [&] { return stats_host_impl(c, src, dst, valid, n, address_space, 0, out); });
}

int nmx_stats9_host_batches(nmx_ctx* c, uint64_t nbatch, const uint32_t* const* src, const uint32_t* const* dst,
                            const uint8_t* const* valid, const uint64_t* lens, uint64_t address_space, int64_t* out) {
  return guarded(c, [&] { return stats_host_batches_impl(c, nbatch, src, dst, valid, lens, address_space, out); });
}

int nmx_stats9_host_i64(nmx_ctx* c, const int64_t* src, const int64_t* dst, const uint8_t* valid, uint64_t n,
                        uint64_t address_space, int64_t out[9]) {
  if (!out) return fail(NMX_EINVAL, "null output");
  return guarded(c, [&] { return stats_host_i64_impl(c, src, dst, valid, n, address_space, out); });
}

int nmx_stream_stats9(nmx_ctx* c, const uint32_t* const* src, const uint32_t* const* dst, const uint8_t* const* valid,
                      const uint64_t* lens, uint64_t nwin, uint64_t address_space, int64_t out[9]) {
  HostWindows hw;
  hw.src = src;
  hw.dst = dst;
  hw.valid = valid;
  hw.lens = lens;
  hw.nwin = nwin;
  return guarded(c, [&] { return stream_impl(c, hw, address_space, out); });
}

int nmx_stream_records(nmx_ctx* c, const uint8_t* const* rec, const uint64_t* lens, uint64_t nwin,
                       uint64_t address_space, int64_t out[9]) {
  if (nwin && !rec) return fail(NMX_EINVAL, "null record windows");
  HostWindows hw;
  hw.rec = rec;
  hw.lens = lens;
  hw.nwin = nwin;
  return guarded(c, [&] { return stream_impl(c, hw, address_space, out); });
}

int nmx_unpack_records(nmx_ctx* c, const uint8_t* d_rec, uint64_t n, uint32_t* d_src, uint32_t* d_dst,
                       uint8_t* d_valid, uint64_t address_space) {
  if (n && (!d_rec || !d_src || !d_dst || !d_valid)) return fail(NMX_EINVAL, "null argument");
  if (((uintptr_t)d_rec & 3) || ((uintptr_t)d_src & 15) || ((uintptr_t)d_dst & 15) || ((uintptr_t)d_valid & 3))
    return fail(NMX_EINVAL, "records need 4-byte, src/dst 16-byte, valid 4-byte alignment");
  return guarded(c, [&] {
    int b;
    if (int r = check_space(address_space, b)) return r;
    c->rmax.grow(64);
    CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
    unpack_records(c, d_rec, n, d_src, d_dst, d_valid, c->rmax.as<unsigned int>());
    return check_maxaddr(c, address_space);
  });
}

int nmx_anonymize_begin(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t* k_out) {
  if (!k_out || (n && (!d_src || !d_dst))) return fail(NMX_EINVAL, "null argument");
  if (n >= (1ull << 31)) return fail(NMX_EINVAL, "anonymize takes < 2^31 packets per call, got %llu",
                                     (unsigned long long)n);
  return guarded(c, [&] {
    stage_begin(c, 1);
    const uint64_t m = 2 * n;
    c->an_m = m;
    c->an_k = 0;
    c->an_pos = nullptr;
    *k_out = 0;
    if (!n) {
      stage_finish(c, 1);
      return NMX_OK;
    }
    for (DevBuf* bf : {&c->anAk, &c->anAv, &c->anBk, &c->anBv, &c->anHead, &c->anFlag}) bf->grow(m * 4 + 16);
    c->anHoff.grow((m + 1) * 4 + 16);
    c->anFoff.grow((m + 1) * 4 + 16);
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, (uint64_t)c->sms * 16));
    anon_pairs_kernel<<<g, 256, 0, c->st>>>(d_src, d_dst, n, c->anAk.as<uint32_t>(), c->anAv.as<uint32_t>());
    CK_LAUNCH();
    // stable LSD sort of (address, position): positions stay ascending inside a run
    auto sorted = sort_u32_pairs(c, c->anAk.as<uint32_t>(), c->anAv.as<uint32_t>(), m, 32, c->anBk.as<uint32_t>(),
                                 c->anBv.as<uint32_t>());
    anon_heads_kernel<<<g, 256, 0, c->st>>>(sorted.first, m, c->anHead.as<uint32_t>());
    CK_LAUNCH();
    scan_counts(c, c->anHead.as<uint32_t>(), (uint32_t)m, c->anHoff.as<uint32_t>(), nullptr);
    uint32_t k = 0;
    CK(cudaMemcpyAsync(&k, c->anHoff.as<uint32_t>() + m, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->anDistinct.grow((uint64_t)k * 4 + 16);
    c->anFirst.grow((uint64_t)k * 4 + 16);
    CK(cudaMemsetAsync(c->anFlag.p, 0, m * 4, c->st));
    anon_uniques_kernel<<<g, 256, 0, c->st>>>(sorted.first, sorted.second, c->anHead.as<uint32_t>(),
                                              c->anHoff.as<uint32_t>(), m, c->anDistinct.as<uint32_t>(),
                                              c->anFirst.as<uint32_t>(), c->anFlag.as<uint32_t>());
    CK_LAUNCH();
    scan_counts(c, c->anFlag.as<uint32_t>(), (uint32_t)m, c->anFoff.as<uint32_t>(), nullptr);
    c->launches += 3;
    c->an_k = k;
    c->an_pos = sorted.second;
    *k_out = k;
    return NMX_OK;
  });
}

int nmx_anonymize_finish(nmx_ctx* c, const uint32_t* perm, uint32_t* d_src_out, uint32_t* d_dst_out,
                         uint32_t* distinct_out, uint32_t* code_out) {
  return guarded(c, [&] {
    const uint64_t k = c->an_k, m = c->an_m;
    if (!k) {
      stage_finish(c, 1);
      return NMX_OK;
    }
    if (!perm || !d_src_out || !d_dst_out || !c->an_pos) return fail(NMX_EINVAL, "null argument or no begin");
    c->anPerm.grow(k * 4 + 16);
    c->anCode.grow(k * 4 + 16);
    CK(cudaMemcpyAsync(c->anPerm.p, perm, k * 4, cudaMemcpyHostToDevice, c->st));
    const unsigned gk = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((k + 255) / 256, (uint64_t)c->sms * 16));
    anon_codes_kernel<<<gk, 256, 0, c->st>>>(c->anFirst.as<uint32_t>(), c->anFoff.as<uint32_t>(),
                                             c->anPerm.as<uint32_t>(), k, c->anCode.as<uint32_t>());
    CK_LAUNCH();
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, (uint64_t)c->sms * 16));
    anon_scatter_kernel<<<g, 256, 0, c->st>>>(c->an_pos, c->anHead.as<uint32_t>(), c->anHoff.as<uint32_t>(), m,
                                              c->anCode.as<uint32_t>(), d_src_out, d_dst_out);
    CK_LAUNCH();
    c->launches += 2;
    if (distinct_out) CK(cudaMemcpyAsync(distinct_out, c->anDistinct.p, k * 4, cudaMemcpyDeviceToHost, c->st));
    if (code_out) CK(cudaMemcpyAsync(code_out, c->anCode.p, k * 4, cudaMemcpyDeviceToHost, c->st));
    c->an_pos = nullptr;
    c->an_k = 0;
    stage_finish(c, 1);
    return NMX_OK;
  });
}

// ---- text matrix files (nmx_text.cuh, traffic.py:295-367) -------------------
int nmx_parse_matrix_text(nmx_ctx* c, const char* text, uint64_t T, int64_t info[8], nmx_coo** out) {
  if (!out || !info || (T && !text)) return fail(NMX_EINVAL, "null argument");
  *out = nullptr;
  std::fill(info, info + 8, 0);
  auto diag = [&](int64_t code, uint64_t line) {
    info[3] = code;
    info[4] = (int64_t)line;
    return NMX_OK;
  };
  if (T == 0) return diag(TXT_HEADER, 1);
  if (T >= (1ull << 40)) return fail(NMX_EINVAL, "text larger than 2^40 bytes");
  return guarded(c, [&] {
    c->txt.grow(T + 16);
    CK(cudaMemcpyAsync(c->txt.p, text, T, cudaMemcpyHostToDevice, c->st));
    const uint64_t nb = (T + kTextChunk - 1) / kTextChunk;
    c->tcnt.grow((nb + 8) * 4);
    c->toff.grow((nb + 8) * 4);
    c->tbad.grow(TR_N * 8);
    auto* red = c->tbad.as<unsigned long long>();
    CK(cudaMemsetAsync(red, 0xFF, TR_N * 8, c->st));  // min-reductions start at UINT64_MAX
    CK(cudaMemsetAsync(red + TR_ENC, 0, 8, c->st));
    text_nl_count_kernel<<<(unsigned)nb, 256, 0, c->st>>>(c->txt.as<char>(), T, c->tcnt.as<uint32_t>());
    CK_LAUNCH();
    scan_counts(c, c->tcnt.as<uint32_t>(), (uint32_t)nb, c->toff.as<uint32_t>(), nullptr);
    uint32_t nl = 0;
    CK(cudaMemcpyAsync(&nl, c->toff.as<uint32_t>() + nb, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    // a text not ending on a break has one more (open) line
    const unsigned char tail = (unsigned char)text[T - 1];
    const bool closed = tail == '\n' || tail == '\r' || tail == '\v' || tail == '\f' || (tail >= 0x1c && tail <= 0x1e);
    const uint64_t L = (uint64_t)nl + (closed ? 0 : 1);
    c->tends.grow((L + 8) * 8);
    text_nl_write_kernel<<<(unsigned)nb, 256, 0, c->st>>>(c->txt.as<char>(), T, c->toff.as<uint32_t>(),
                                                          c->tends.as<uint64_t>());
    CK_LAUNCH();
    if (!closed) CK(cudaMemcpyAsync(c->tends.as<uint64_t>() + L - 1, &T, 8, cudaMemcpyHostToDevice, c->st));
    c->tntok.grow(L + 16);
    c->tvals.grow((L + 8) * 24);
    c->tnb.grow((L + 8) * 4);
    c->tnboff.grow((L + 8) * 4);
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((L + 255) / 256, (uint64_t)c->sms * 16));
    text_parse_lines_kernel<<<g, 256, 0, c->st>>>(c->txt.as<char>(), c->tends.as<uint64_t>(), L,
                                                  c->tntok.as<uint8_t>(), c->tvals.as<long long>(), red);
    CK_LAUNCH();
    text_nonblank_kernel<<<g, 256, 0, c->st>>>(c->tntok.as<uint8_t>(), L, c->tnb.as<uint32_t>());
    CK_LAUNCH();
    scan_counts(c, c->tnb.as<uint32_t>(), (uint32_t)L, c->tnboff.as<uint32_t>(), nullptr);
    c->launches += 5;
    uint32_t nbl = 0;
    unsigned long long r[TR_N];
    CK(cudaMemcpyAsync(&nbl, c->tnboff.as<uint32_t>() + L, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(r, red, sizeof(r), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (r[TR_ENC]) return diag(TXT_ENCODING, 0);
    if (nbl == 0) return diag(TXT_HEADER, 1);
    // header = first nonblank line (traffic.py:322-333 order of checks)
    const uint64_t l0 = r[TR_HEAD];
    uint8_t t0 = 0;
    long long h[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(&t0, c->tntok.as<uint8_t>() + l0, 1, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(h, c->tvals.as<long long>() + 3 * l0, 24, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if ((t0 & 0x7F) != 2 || (t0 & 0x80)) return diag(TXT_HEADER, l0 + 1);
    info[0] = h[0];
    info[1] = h[1];
    if (h[0] < 1) return diag(TXT_DIM, l0 + 1);
    if (h[1] < 0) return diag(TXT_NNZ, l0 + 1);
    const uint64_t entries = nbl - 1;
    info[2] = (int64_t)entries;
    nmx_coo* o = coo_alloc(c, entries);
    c->tloff.grow((entries + 8) * 4);
    text_entries_kernel<<<g, 256, 0, c->st>>>(c->tntok.as<uint8_t>(), c->tvals.as<long long>(),
                                              c->tnboff.as<uint32_t>(), L, h[0],
                                              reinterpret_cast<unsigned long long*>(o->keys), o->counts,
                                              c->tloff.as<uint32_t>(), red);
    CK_LAUNCH();
    if (entries > 1) {
      const unsigned gn =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((entries + 255) / 256, (uint64_t)c->sms * 16));
      text_order_kernel<<<gn, 256, 0, c->st>>>(reinterpret_cast<const unsigned long long*>(o->keys),
                                               c->tloff.as<uint32_t>(), entries, red);
      CK_LAUNCH();
    }
    c->launches += 2;
    CK(cudaMemcpyAsync(r, red, sizeof(r), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    const unsigned long long none = ~0ull;
    int64_t code = TXT_OK;
    uint64_t line = 0;
    if (r[TR_TOK] != none) {
      code = (int64_t)(r[TR_TOK] & 15);
      line = r[TR_TOK] >> 4;
    } else if ((uint64_t)h[1] != entries) {
      code = TXT_COUNT;
    } else if (r[TR_BOUNDS] != none) {
      code = TXT_BOUNDS, line = r[TR_BOUNDS];
    } else if (r[TR_VALUE] != none) {
      code = TXT_VALUE, line = r[TR_VALUE];
    } else if (r[TR_ORDER] != none) {
      code = TXT_ORDER, line = r[TR_ORDER];
    } else if (h[0] > (1ll << 32)) {  // row / col beyond the 32-bit key halves
      code = TXT_WIDE, line = l0 + 1;
    }
    if (code != TXT_OK) {
      nmx_coo_free(o);
      return diag(code, line);
    }
    *out = o;
    return NMX_OK;
  });
}

int nmx_format_matrix_text(nmx_ctx* c, const int64_t* rows, const int64_t* cols, const int64_t* vals, uint64_t nnz,
                           char* out, uint64_t cap, uint64_t* bytes) {
  if (!bytes || (nnz && (!rows || !cols || !vals))) return fail(NMX_EINVAL, "null argument");
  return guarded(c, [&] {
    *bytes = 0;
    if (!nnz) return NMX_OK;
    c->trows.grow(nnz * 8);
    c->tcols.grow(nnz * 8);
    c->tval.grow(nnz * 8);
    c->tlen.grow((nnz + 8) * 4);
    c->tloff.grow((nnz + 8) * 8);
    CK(cudaMemcpyAsync(c->trows.p, rows, nnz * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->tcols.p, cols, nnz * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->tval.p, vals, nnz * 8, cudaMemcpyHostToDevice, c->st));
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nnz + 255) / 256, (uint64_t)c->sms * 16));
    auto* R = c->trows.as<unsigned long long>();
    auto* Cc = c->tcols.as<unsigned long long>();
    auto* V = c->tval.as<unsigned long long>();
    text_line_len_kernel<<<g, 256, 0, c->st>>>(R, Cc, V, nnz, c->tlen.as<uint32_t>());
    CK_LAUNCH();
    // line offsets: the u32 scan gives offsets < 2^32; the text stays below 4 GiB per call
    if (nnz >= (1ull << 32) / 64) throw std::runtime_error("matrix too large for one text call");
    c->toff.grow((nnz + 8) * 4);
    scan_counts(c, c->tlen.as<uint32_t>(), (uint32_t)nnz, c->toff.as<uint32_t>(), nullptr);
    uint32_t total = 0;
    CK(cudaMemcpyAsync(&total, c->toff.as<uint32_t>() + nnz, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    *bytes = total;
    if (!out || cap < total) return NMX_OK;
    c->txt.grow((uint64_t)total + 16);
    widen_offsets_kernel<<<g, 256, 0, c->st>>>(c->toff.as<uint32_t>(), nnz, c->tloff.as<unsigned long long>());
    CK_LAUNCH();
    text_write_lines_kernel<<<g, 256, 0, c->st>>>(R, Cc, V, nnz, c->tloff.as<unsigned long long>(), c->txt.as<char>());
    CK_LAUNCH();
    CK(cudaMemcpyAsync(out, c->txt.p, total, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->launches += 4;
    return NMX_OK;
  });
}

int nmx_window_stats9_device(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                             uint64_t n, uint64_t address_space, uint64_t window_size, int64_t* out) {
  if (window_size < 1) return fail(NMX_EINVAL, "window_size must be >= 1");
  return guarded(c, [&] {
    if (n == 0) return NMX_OK;
    if (window_size >= n) return stats_device_impl(c, d_src, d_dst, d_valid, n, address_space, 0, out);
    return stats_device_impl(c, d_src, d_dst, d_valid, n, address_space, window_size, out);
  });
}

int nmx_window_stats9_host(nmx_ctx* c, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                           uint64_t address_space, uint64_t window_size, int64_t* out) {
  if (window_size < 1) return fail(NMX_EINVAL, "window_size must be >= 1");
  return guarded(c, [&] {
    if (n == 0) return NMX_OK;
    return stats_host_impl(c, src, dst, valid, n, address_space, window_size >= n ? 0 : window_size, out);
  });
}

int nmx_reduce_i64(nmx_ctx* c, const int64_t* data, uint64_t n, int op, int64_t* out) {
  if (op != NMX_REDUCE_SUM && op != NMX_REDUCE_MAX) return fail(NMX_EINVAL, "unknown reduce op %d", op);
  if (!out) return fail(NMX_EINVAL, "null output");
  return guarded(c, [&] {
    c->red.grow(n * 8 + 64);
    unsigned long long init = op == NMX_REDUCE_SUM ? 0ull : (unsigned long long)INT64_MIN;
    unsigned long long* d_out = reinterpret_cast<unsigned long long*>(c->red.as<int64_t>() + n);
    CK(cudaMemcpyAsync(d_out, &init, 8, cudaMemcpyHostToDevice, c->st));
    if (n) {
      CK(cudaMemcpyAsync(c->red.p, data, n * 8, cudaMemcpyHostToDevice, c->st));
      const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 8);
      reduce_i64_kernel<<<grid, 256, 0, c->st>>>(c->red.as<int64_t>(), n, op, d_out);
      CK_LAUNCH();
    }
    unsigned long long r;
    CK(cudaMemcpyAsync(&r, d_out, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    *out = (int64_t)r;
    return NMX_OK;
  });
}

int nmx_partition_packets(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                          uint64_t n, int nparts, uint32_t* d_out_src, uint32_t* d_out_dst, uint64_t* counts) {
  if (nparts < 1 || nparts > kMaxParts) return fail(NMX_EINVAL, "nparts must lie in [1, %d]", kMaxParts);
  if (!counts) return fail(NMX_EINVAL, "null counts");
  return guarded(c, [&] {
    if (!n) {
      std::fill(counts, counts + nparts, 0);
      return NMX_OK;
    }
    PacketPart it{d_src, d_dst, d_valid, d_out_src, d_out_dst};
    partition_items(c, it, n, nparts, counts);
    return NMX_OK;
  });
}

int nmx_shard_rows(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t address_space,
                   int nparts, uint32_t* d_out_dst, uint32_t* d_out_count, uint64_t* counts, int64_t out[9]) {
  if (nparts < 1 || nparts > kMaxParts) return fail(NMX_EINVAL, "nparts must lie in [1, %d]", kMaxParts);
  if (!counts || !out) return fail(NMX_EINVAL, "null output");
  int b;
  if (int r = check_space(address_space, b)) return r;
  if (n >= (1ull << 32)) return fail(NMX_EINVAL, "n must be < 2^32 per call");
  return guarded(c, [&] {
    return shard_rows_impl(c, d_src, d_dst, n, address_space, nparts, d_out_dst, d_out_count, counts, out);
  });
}

int nmx_shard_cols(nmx_ctx* c, const uint32_t* d_dst, const uint32_t* d_count, uint64_t u, uint64_t address_space,
                   int64_t out[9]) {
  if (!out) return fail(NMX_EINVAL, "null output");
  int b;
  if (int r = check_space(address_space, b)) return r;
  if (u >= (1ull << 32)) return fail(NMX_EINVAL, "u must be < 2^32 per call");
  return guarded(c, [&] { return shard_cols_impl(c, d_dst, d_count, u, address_space, out); });
}

int nmx_coo_build(nmx_ctx* c, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                  uint64_t address_space, uint64_t window_size, uint64_t* nnz) {
  if (!nnz) return fail(NMX_EINVAL, "null output");
  int b;
  if (int r = check_space(address_space, b)) return r;
  if (n >= (1ull << 32)) return fail(NMX_EINVAL, "n must be < 2^32 per call");
  return guarded(c, [&] {
    *nnz = 0;
    c->coo_nnz = 0;
    c->coo_b = b;
    if (!n) return NMX_OK;
    const uint64_t W = (window_size && window_size < n) ? (n + window_size - 1) / window_size : 1;
    const int wb = W > 1 ? (int)ceil_log2(W) : 0;
    if (2 * b + wb > 64) return fail(NMX_EINVAL, "2*bits + window bits exceed 64; build windows separately");
    c->in_src.grow(n * 4);
    c->in_dst.grow(n * 4);
    CK(cudaMemcpyAsync(c->in_src.p, src, n * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->in_dst.p, dst, n * 4, cudaMemcpyHostToDevice, c->st));
    if (valid) {
      c->in_valid.grow(n);
      CK(cudaMemcpyAsync(c->in_valid.p, valid, n, cudaMemcpyHostToDevice, c->st));
    }
    if (int r = check_addresses(c, c->in_src.as<uint32_t>(), c->in_dst.as<uint32_t>(), n, address_space)) return r;
    stage_begin(c, 1);
    PacketSrc ps{c->in_src.as<uint32_t>(), c->in_dst.as<uint32_t>(), valid ? c->in_valid.as<uint8_t>() : nullptr, n,
                 W > 1 ? window_size : 0, b};
    uint64_t m = 0;
    uint64_t* keys = sort_rows(c, ps, b, wb, &m);
    if (m) {
      c->mkeys.grow(m * 8);
      c->mlen.grow(m * 4);
      c->coo_nnz = run_rbk<uint64_t>(c, keys, nullptr, (uint32_t)m, 0, c->mkeys.as<unsigned long long>(),
                                     c->mlen.as<uint32_t>(), nullptr, 27);
    }
    stage_finish(c, 1);
    *nnz = c->coo_nnz;
    return NMX_OK;
  });
}

int nmx_coo_fetch(nmx_ctx* c, uint64_t* keys, int64_t* counts) {
  return guarded(c, [&] {
    const uint64_t u = c->coo_nnz;
    if (!u) return NMX_OK;
    if (keys) CK(cudaMemcpyAsync(keys, c->mkeys.p, u * 8, cudaMemcpyDeviceToHost, c->st));
    std::vector<uint32_t> tmp(counts ? u : 0);
    if (counts) CK(cudaMemcpyAsync(tmp.data(), c->mlen.p, u * 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (uint64_t i = 0; counts && i < u; ++i) counts[i] = tmp[i];
    return NMX_OK;
  });
}

int nmx_coo_rowptr(nmx_ctx* c, uint64_t lo, uint64_t hi, uint64_t window, uint64_t dim, int64_t* row_ptr) {
  if (!row_ptr) return fail(NMX_EINVAL, "null output");
  return guarded(c, [&] {
    if (hi < lo || hi > c->coo_nnz) return fail(NMX_EINVAL, "slice [%llu,%llu) outside the COO", (unsigned long long)lo,
                                                 (unsigned long long)hi);
    const int b = c->coo_b;
    if (dim > (1ull << b)) return fail(NMX_EINVAL, "dim exceeds the address space of the COO");
    DevBuf& out = c->frows;
    out.grow((dim + 1) * 8);
    const uint64_t wbase = 2 * b < 64 ? (window << (2 * b)) : 0;
    const unsigned grid = (unsigned)std::min<uint64_t>((dim + 256) / 256, (uint64_t)c->sms * 16);
    coo_rowptr_kernel<<<grid, 256, 0, c->st>>>(c->mkeys.as<uint64_t>(), lo, hi, wbase, b, dim,
                                               out.as<long long>());
    CK_LAUNCH();
    CK(cudaMemcpyAsync(row_ptr, out.p, (dim + 1) * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_flat_build(nmx_ctx* c, const int64_t* row_ptr, uint64_t dim, const int64_t* col_idx, const int64_t* values,
                   uint64_t nnz, uint64_t* r_out, uint64_t* c_out) {
  if (!r_out || !c_out) return fail(NMX_EINVAL, "null output");
  if (nnz >= (1ull << 32) || dim >= (1ull << 32)) return fail(NMX_EINVAL, "nnz and dim must be < 2^32");
  for (uint64_t k = 0; k < nnz; ++k)
    if (values[k] < 1 || values[k] > 0xFFFFFFFFll) return fail(NMX_EINVAL, "values must lie in [1, 2^32)");
  return guarded(c, [&] {
    *r_out = *c_out = 0;
    c->flat_nnz = nnz;
    c->flat_r = c->flat_c = 0;
    if (!nnz) return NMX_OK;
    stage_begin(c, 1);
    uint32_t* d_small = c->small.as<uint32_t>();
    // upload CSR
    c->in_src.grow((dim + 1) * 8);
    c->in_dst.grow(nnz * 16);
    long long* d_rp = c->in_src.as<long long>();
    long long* d_col = c->in_dst.as<long long>();
    long long* d_val = d_col + nnz;
    CK(cudaMemcpyAsync(d_rp, row_ptr, (dim + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_col, col_idx, nnz * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_val, values, nnz * 8, cudaMemcpyHostToDevice, c->st));
    c->frows.grow(nnz * 4);
    c->ckA.grow(nnz * 4);
    c->ckB.grow(nnz * 4);
    c->cvA.grow(nnz * 4);
    c->cvB.grow(nnz * 4);
    const unsigned grid = (unsigned)std::min<uint64_t>((nnz + 255) / 256, (uint64_t)c->sms * 16);
    csr_expand_kernel<<<grid, 256, 0, c->st>>>(d_rp, dim, d_col, d_val, nnz, c->frows.as<uint32_t>(),
                                                c->ckA.as<uint32_t>(), c->cvA.as<uint32_t>());
    CK_LAUNCH();
    // rows: CSR order is row-sorted -> reduce by row (np.add.reduceat, traffic.py:271-277)
    c->mkeys.grow(nnz * 8);
    c->mlen.grow(nnz * 4);
    c->msum.grow(nnz * 8);
    c->flat_r = run_rbk<uint32_t>(c, c->frows.as<uint32_t>(), c->cvA.as<uint32_t>(), (uint32_t)nnz, 0,
                                  c->mkeys.as<unsigned long long>(), c->mlen.as<uint32_t>(),
                                  c->msum.as<unsigned long long>(), 28);
    // columns: sort (col, value) then reduce by column (bincount / np.add.at, traffic.py:279-283)
    const int cb = std::max<int>(1, (int)ceil_log2(std::max<uint64_t>(dim, 2)));
    const int ncolpass = (cb + 7) / 8;
    const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nnz + 1023) / 1024, (uint64_t)c->sms * 8));
    switch (ncolpass) {
      case 1: hist_u32_kernel<1><<<hgrid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), nnz, d_small + kCHist); break;
      case 2: hist_u32_kernel<2><<<hgrid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), nnz, d_small + kCHist); break;
      case 3: hist_u32_kernel<3><<<hgrid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), nnz, d_small + kCHist); break;
      default: hist_u32_kernel<4><<<hgrid, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), nnz, d_small + kCHist); break;
    }
    CK_LAUNCH();
    auto sorted = sort_col_entries<uint32_t>(c, (uint32_t)nnz, cb, d_small);
    c->ckeys2.grow(nnz * 8);
    c->clen2.grow(nnz * 4);
    c->csum2.grow(nnz * 8);
    c->flat_c = run_rbk<uint32_t>(c, sorted.first, sorted.second, (uint32_t)nnz, 0,
                                  c->ckeys2.as<unsigned long long>(), c->clen2.as<uint32_t>(),
                                  c->csum2.as<unsigned long long>(), 29);
    stage_finish(c, 1);
    *r_out = c->flat_r;
    *c_out = c->flat_c;
    return NMX_OK;
  });
}

int nmx_flat_fetch(nmx_ctx* c, int64_t* edge_src, int64_t* row_ids, int64_t* row_nnz, int64_t* row_sum,
                   int64_t* col_ids, int64_t* col_nnz, int64_t* col_sum) {
  return guarded(c, [&] {
    const uint64_t nnz = c->flat_nnz, r = c->flat_r, cc = c->flat_c;
    std::vector<uint32_t> rows(nnz), rl(r), cl(cc);
    std::vector<unsigned long long> rk(r), rs(r), ck(cc), cs(cc);
    if (nnz) CK(cudaMemcpyAsync(rows.data(), c->frows.p, nnz * 4, cudaMemcpyDeviceToHost, c->st));
    if (r) {
      CK(cudaMemcpyAsync(rk.data(), c->mkeys.p, r * 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(rl.data(), c->mlen.p, r * 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(rs.data(), c->msum.p, r * 8, cudaMemcpyDeviceToHost, c->st));
    }
    if (cc) {
      CK(cudaMemcpyAsync(ck.data(), c->ckeys2.p, cc * 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(cl.data(), c->clen2.p, cc * 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(cs.data(), c->csum2.p, cc * 8, cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    for (uint64_t i = 0; edge_src && i < nnz; ++i) edge_src[i] = rows[i];
    for (uint64_t i = 0; i < r; ++i) {
      if (row_ids) row_ids[i] = (int64_t)rk[i];
      if (row_nnz) row_nnz[i] = rl[i];
      if (row_sum) row_sum[i] = (int64_t)rs[i];
    }
    for (uint64_t i = 0; i < cc; ++i) {
      if (col_ids) col_ids[i] = (int64_t)ck[i];
      if (col_nnz) col_nnz[i] = cl[i];
      if (col_sum) col_sum[i] = (int64_t)cs[i];
    }
    return NMX_OK;
  });
}

// COO storage is stream-ordered (cudaMallocAsync / cudaFreeAsync from the device's
// default pool, kept resident): a plain cudaFree would synchronise the whole
// device and serialise the overlapped H2D copies of the streamed path.
nmx_coo* coo_alloc(nmx_ctx* c, uint64_t nnz) {
  static bool pool_ready[64] = {false};
  if (c->device < 64 && !pool_ready[c->device]) {
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
    uint64_t keep = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    pool_ready[c->device] = true;
  }
  nmx_coo* o = new nmx_coo();
  o->device = c->device;
  o->nnz = nnz;
  if (nnz) {
    CK(cudaMallocAsync(reinterpret_cast<void**>(&o->keys), nnz * 8, c->st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&o->counts), nnz * 8, c->st));
  }
  return o;
}

int nmx_coo_from_packets(nmx_ctx* c, const uint32_t* d_src, const uint32_t* d_dst, const uint8_t* d_valid,
                         uint64_t n, nmx_coo** out) {
  if (!out) return fail(NMX_EINVAL, "null output");
  if (n >= (1ull << 32)) return fail(NMX_EINVAL, "n must be < 2^32 per call");
  return guarded(c, [&] {
    stage_begin(c, 1);
    uint64_t m = 0;
    uint64_t u = 0;
    if (n) {
      PacketSrc ps{d_src, d_dst, d_valid, n, 0, 32};
      // keys (src << 32 | dst) only use 32 + bits(max address) bits: the MSD levels
      // take their digits from there (a narrow address space would otherwise leave
      // every key in one bucket)
      c->rmax.grow(64);
      CK(cudaMemsetAsync(c->rmax.p, 0, 4, c->st));
      launch_max_addr(c, d_src, d_dst, n);
      unsigned int mx = 0;
      CK(cudaMemcpyAsync(&mx, c->rmax.p, 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      uint64_t* keys = sort_rows(c, ps, 32, 0, &m, 32 + (int)ceil_log2((uint64_t)mx + 1));
      if (m) {
        const uint64_t tiles = (m + kUniqTile - 1) / kUniqTile;
        c->mhist2.grow((tiles + 8) * 4);
        c->moff.grow((tiles + 8) * 4);
        unique_heads_kernel<false><<<(unsigned)tiles, 256, 0, c->st>>>(keys, m, c->mhist2.as<uint32_t>(), nullptr,
                                                                      nullptr, nullptr);
        CK_LAUNCH();
        scan_counts(c, c->mhist2.as<uint32_t>(), (uint32_t)tiles, c->moff.as<uint32_t>(), nullptr);
        uint32_t uu = 0;
        CK(cudaMemcpyAsync(&uu, c->moff.as<uint32_t>() + tiles, 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        u = uu;
        c->mlen.grow(u * 4 + 8);
        nmx_coo* o = coo_alloc(c, u);
        unique_heads_kernel<true><<<(unsigned)tiles, 256, 0, c->st>>>(keys, m, nullptr, c->moff.as<uint32_t>(),
                                                                     o->keys, c->mlen.as<uint32_t>());
        CK_LAUNCH();
        run_counts_kernel<<<(unsigned)std::min<uint64_t>((u + 255) / 256, (uint64_t)c->sms * 16), 256, 0, c->st>>>(
            c->mlen.as<uint32_t>(), u, m, o->counts);
        CK_LAUNCH();
        c->launches += 3;
        stage_finish(c, 1);
        *out = o;
        return NMX_OK;
      }
    }
    nmx_coo* o = coo_alloc(c, u);
    stage_finish(c, 1);
    *out = o;
    return NMX_OK;
  });
}

int nmx_coo_upload(nmx_ctx* c, const uint64_t* keys, const int64_t* counts, uint64_t nnz, nmx_coo** out) {
  if (!out || (nnz && (!keys || !counts))) return fail(NMX_EINVAL, "null argument");
  for (uint64_t i = 0; i < nnz; ++i)
    if (counts[i] < 1) return fail(NMX_EINVAL, "COO counts must be >= 1");
  return guarded(c, [&] {
    nmx_coo* o = coo_alloc(c, nnz);
    if (nnz) {
      CK(cudaMemcpyAsync(o->keys, keys, nnz * 8, cudaMemcpyHostToDevice, c->st));
      CK(cudaMemcpyAsync(o->counts, counts, nnz * 8, cudaMemcpyHostToDevice, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    *out = o;
    return NMX_OK;
  });
}

int nmx_coo_merge_add(nmx_ctx* c, const nmx_coo* a, const nmx_coo* b, nmx_coo** out) {
  if (!a || !b || !out) return fail(NMX_EINVAL, "null argument");
  return guarded(c, [&] {
    stage_begin(c, 1);
    const uint64_t n = a->nnz + b->nnz;
    if (n >= (1ull << 32)) throw std::runtime_error("merged matrix would exceed 2^32-1 links");
    const uint64_t tiles = (n + kMgTile - 1) / kMgTile;
    nmx_coo* o = coo_alloc(c, n);  // capacity na + nb; nnz set below
    if (tiles) {
      c->msplit.grow((tiles + 2) * 8);
      c->part.grow(64);
      auto* ovf = c->part.as<unsigned long long>();
      CK(cudaMemsetAsync(ovf, 0, 16, c->st));
      c->grow_status(tiles + 1);
      const unsigned pg = (unsigned)std::min<uint64_t>((tiles + 256) / 256, (uint64_t)c->sms * 8);
      merge_partition_kernel<<<pg, 256, 0, c->st>>>(a->keys, a->nnz, b->keys, b->nnz, tiles,
                                                    c->msplit.as<uint64_t>());
      CK_LAUNCH();
      set_smem(merge_add_kernel, sizeof(MergeSmem));
      c->dom_begin("merge_add");
      merge_add_kernel<<<(unsigned)tiles, kMgThreads, sizeof(MergeSmem), c->st>>>(
          a->keys, a->counts, a->nnz, b->keys, b->counts, b->nnz, c->msplit.as<uint64_t>(),
          c->status.as<uint64_t>(), c->next_epoch(), c->small.as<uint32_t>() + kCounters + 28, o->keys, o->counts,
          ovf, ovf + 1);
      CK_LAUNCH();
      c->dom_end(16 * n);  // + 16 B per output link, added below
      c->launches += 2;
      unsigned long long res[2] = {0, 0};
      CK(cudaMemcpyAsync(res, ovf, 16, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      c->dom_bytes += 16 * (uint64_t)res[1];
      if (c->dom_cur) c->dom_lbytes[c->nevk / 2 - 1] += 16 * (uint64_t)res[1];
      o->nnz = res[1];
      if (res[0]) {
        nmx_coo_free(o);
        return fail(NMX_EINVAL, "merged link count exceeds 2^63-1");
      }
    }
    stage_finish(c, 1);
    *out = o;
    return NMX_OK;
  });
}

int nmx_coo_stats9(nmx_ctx* c, const nmx_coo* a, int64_t out[9]) {
  if (!a || !out) return fail(NMX_EINVAL, "null argument");
  return guarded(c, [&] {
    stage_begin(c, 1);
    const uint64_t u = a->nnz;
    if (u) {
      if (u >= (1ull << 32)) throw std::runtime_error("COO too large for one statistics call");
      uint32_t* d_small = c->small.as<uint32_t>();
      unsigned long long* st = c->stats.as<unsigned long long>();
      const unsigned grid = (unsigned)std::min<uint64_t>((u + 255) / 256, (uint64_t)c->sms * 8);
      coo_link_stats_kernel<<<grid, 256, 0, c->st>>>(a->counts, u, st);
      CK_LAUNCH();
      CK(cudaMemcpyAsync(st + S_LINKS, &u, 8, cudaMemcpyHostToDevice, c->st));
      unsigned long long maxc = 0;
      CK(cudaMemcpyAsync(&maxc, st + S_MAXLINK, 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      if (maxc > 0xFFFFFFFFull) {  // a link of >= 2^32 packets: 64-bit tables
        if (u > (1ull << 28)) throw std::runtime_error("COO with counts >= 2^32 and more than 2^28 links");
        uint64_t slots = 1;
        while (slots < 2 * u) slots <<= 1;
        c->cgk.grow(slots * 24);
        auto* tk = c->cgk.as<unsigned long long>();
        for (int side = 0; side < 2; ++side) {
          CK(cudaMemsetAsync(tk, 0, slots * 24, c->st));
          wide_table_add_kernel<<<grid, 256, 0, c->st>>>(a->keys, a->counts, u, side ? 0 : 32, tk, tk + slots,
                                                         tk + 2 * slots, slots - 1);
          CK_LAUNCH();
          const unsigned rg = (unsigned)std::min<uint64_t>((slots + 255) / 256, (uint64_t)c->sms * 8);
          wide_table_reduce_kernel<<<rg, 256, 0, c->st>>>(tk, tk + slots, tk + 2 * slots, slots, st,
                                                          side ? S_DSTS : S_SRCS, side ? S_MAXFANIN : S_MAXFANOUT,
                                                          side ? S_MAXDSTPK : S_MAXSRCPK);
          CK_LAUNCH();
        }
        c->launches += 5;
        stage_finish(c, 1);
        copy_out9(c->h_stats, out, 1);
        return NMX_OK;
      }
      // columns: (dst, count) entries; their 32-bit counts (key order) also feed the row segments
      c->ckA.grow(u * 4);
      c->cvA.grow(u * 4);
      c->ckB.grow(u * 4);
      c->cvB.grow(u * 4);
      coo_col_entries_kernel<<<grid, 256, 0, c->st>>>(a->keys, a->counts, u, c->ckA.as<uint32_t>(),
                                                      c->cvA.as<uint32_t>());
      CK_LAUNCH();
      if (c->csstatus.grow(tiles_of(u, kSegTile) * sizeof(CSStatus)))
        CK(cudaMemsetAsync(c->csstatus.p, 0, c->csstatus.cap, c->st));
      // rows: segments of equal src over the sorted keys (fan-out = links, packets = counts)
      col_kernel<uint64_t, kSegIPT><<<(unsigned)tiles_of(u, kSegTile), 256, 0, c->st>>>(
          a->keys, c->cvA.as<uint32_t>(), (uint32_t)u, 32, 0, c->csstatus.as<CSStatus>(), c->next_epoch(),
          d_small + kCounters + 27, st, 32, S_SRCS, S_MAXFANOUT, S_MAXSRCPK);
      CK_LAUNCH();
      const int Dc = std::min(21, std::max(11, (int)ceil_log2(u) - 9));
      if (u >= (1ull << 20)) {  // MSD partition + shared-memory grouping
        c->colL_dst.grow(u * 8);
        pack_cols_kernel<<<c->sms * 8, 256, 0, c->st>>>(c->ckA.as<uint32_t>(), c->cvA.as<uint32_t>(), u,
                                                        c->colL_dst.as<uint64_t>());
        CK_LAUNCH();
        ColConcatSrc cs{c->colL_dst.as<uint64_t>(), u, nullptr, 0, u};
        cs.quad = true;
        msd_columns(c, cs, 32, Dc, nullptr);
      } else {
        auto sorted = sort_u32_pairs(c, c->ckA.as<uint32_t>(), c->cvA.as<uint32_t>(), u, 32, c->ckB.as<uint32_t>(),
                                     c->cvB.as<uint32_t>());
        col_kernel<uint32_t, kSegIPT><<<(unsigned)tiles_of(u, kSegTile), 256, 0, c->st>>>(
            sorted.first, sorted.second, (uint32_t)u, 32, 0, c->csstatus.as<CSStatus>(), c->next_epoch(),
            d_small + kCounters + 26, st);
        CK_LAUNCH();
      }
      c->launches += 4;
    }
    stage_finish(c, 1);
    copy_out9(c->h_stats, out, 1);
    return NMX_OK;
  });
}

int nmx_coo_reserve(nmx_ctx* c, uint64_t bytes) {
  return guarded(c, [&] {
    nmx_coo* probe = coo_alloc(c, 0);  // configures the pool (release threshold = keep)
    delete probe;
    void* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<uint64_t>(bytes, 1), c->st));
    CK(cudaFreeAsync(p, c->st));
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

int nmx_coo_nnz(const nmx_coo* a, uint64_t* nnz) {
  if (!a || !nnz) return fail(NMX_EINVAL, "null argument");
  *nnz = a->nnz;
  return NMX_OK;
}

int nmx_coo_download(nmx_ctx* c, const nmx_coo* a, uint64_t* keys, int64_t* counts) {
  if (!a) return fail(NMX_EINVAL, "null argument");
  return guarded(c, [&] {
    if (!a->nnz) return NMX_OK;
    if (keys) CK(cudaMemcpyAsync(keys, a->keys, a->nnz * 8, cudaMemcpyDeviceToHost, c->st));
    if (counts) CK(cudaMemcpyAsync(counts, a->counts, a->nnz * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return NMX_OK;
  });
}

void nmx_coo_free(nmx_coo* a) {
  if (!a) return;
  cudaSetDevice(a->device);
  // stream-ordered on the legacy stream: ordered after every prior launch that
  // could read the matrix on blocking streams; the context streams are
  // non-blocking, so callers free only after their synchronous calls returned
  if (a->keys) cudaFreeAsync(a->keys, 0);
  if (a->counts) cudaFreeAsync(a->counts, 0);
  delete a;
}

int nmx_last_kernel_class(nmx_ctx* c, float* ms, int* launches, uint64_t* bytes, char* name, int name_cap) {
  if (!c) return fail(NMX_EINVAL, "null context");
  if (ms) *ms = c->dom_ms;
  if (launches) *launches = c->dom_launches;
  if (bytes) *bytes = c->dom_bytes;
  if (name && name_cap > 0) snprintf(name, name_cap, "%s", c->dom_name);
  return NMX_OK;
}

int nmx_last_kernel_launches(nmx_ctx* c, int cap, float* ms, uint64_t* bytes, int* count) {
  if (!c || cap < 0) return fail(NMX_EINVAL, "null context or negative capacity");
  const int k = std::min(cap, c->nevk / 2);
  for (int i = 0; i < k; ++i) {
    if (ms) ms[i] = c->dom_lms[i];
    if (bytes) bytes[i] = c->dom_lbytes[i];
  }
  if (count) *count = c->nevk / 2;
  return NMX_OK;
}

int nmx_last_stages(nmx_ctx* c, float* ms, int cap) {
  if (!c) return fail(NMX_EINVAL, "null context");
  const int k = std::min(cap, c->last_nstage);
  for (int i = 0; i < k; ++i) ms[i] = c->last_stage_ms[i];
  return k;
}

int nmx_last_timing(nmx_ctx* c, float* total_ms, float* sort_ms, int* sort_launches, int* kernel_launches) {
  if (!c) return fail(NMX_EINVAL, "null context");
  if (total_ms) *total_ms = c->last_total_ms;
  if (sort_ms) *sort_ms = c->last_sort_ms;
  if (sort_launches) *sort_launches = c->last_sort_launches;
  if (kernel_launches) *kernel_launches = c->last_launches;
  return NMX_OK;
}


// ---- device groups -----------------------------------------------------------
int nmx_group_create(const int* devices, int g, nmx_group** out) {
  if (!out || !devices) return fail(NMX_EINVAL, "null argument");
  *out = nullptr;
  if (g < 1 || g > kMaxParts) return fail(NMX_EINVAL, "group size must lie in [1, %d], got %d", kMaxParts, g);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(NMX_ENODEV, "no CUDA device");
  }
  for (int r = 0; r < g; ++r)
    if (devices[r] < 0 || devices[r] >= ndev)
      return fail(NMX_EINVAL, "rank %d: device %d out of range (%d visible)", r, devices[r], ndev);
  auto* G = new (std::nothrow) nmx_group();
  if (!G) return fail(NMX_ENOMEM, "host allocation failed");
  G->g = g;
  G->devices.assign(devices, devices + g);
  G->ranks = std::vector<GroupRank>(g);
  for (int r = 0; r < g; ++r) {
    if (int rc = nmx_create(devices[r], &G->ranks[r].ctx)) {
      nmx_group_destroy(G);
      return rc;
    }
  }
  // NVLink peer access between the distinct devices of the group (copies fall back
  // to staging through the host path of cudaMemcpyPeer when a pair has none)
  for (int a = 0; a < g; ++a)
    for (int b = 0; b < g; ++b) {
      const int da = devices[a], db = devices[b];
      if (da == db) continue;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, da, db) == cudaSuccess && ok) {
        cudaSetDevice(da);
        const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e != cudaSuccess) cudaGetLastError();  // already enabled
      }
    }
  *out = G;
  return NMX_OK;
}

void nmx_group_destroy(nmx_group* G) {
  if (!G) return;
  for (auto& rk : G->ranks) {
    if (!rk.ctx) continue;
    cudaSetDevice(rk.ctx->device);
    if (rk.ev) cudaEventDestroy(rk.ev);
    for (DevBuf* b : {&rk.ps, &rk.pd, &rk.rs, &rk.rd, &rk.cs, &rk.cc, &rk.qs, &rk.qc, &rk.hs, &rk.hd, &rk.hv})
      b->release();
    nmx_destroy(rk.ctx);
    rk.ctx = nullptr;
  }
  delete G;
}

int nmx_group_size(const nmx_group* G, int* g) {
  if (!G || !g) return fail(NMX_EINVAL, "null argument");
  *g = G->g;
  return NMX_OK;
}

int nmx_group_context(nmx_group* G, int rank, nmx_ctx** out) {
  if (!G || !out) return fail(NMX_EINVAL, "null argument");
  if (rank < 0 || rank >= G->g) return fail(NMX_EINVAL, "rank %d out of range", rank);
  *out = G->ranks[rank].ctx;
  return NMX_OK;
}

int nmx_group_stats9_device(nmx_group* G, const uint32_t* const* d_src, const uint32_t* const* d_dst,
                            const uint8_t* const* d_valid, const uint64_t* n, uint64_t address_space, int64_t out[9]) {
  if (!G || !d_src || !d_dst || !n || !out) return fail(NMX_EINVAL, "null argument");
  int b;
  if (int r = check_space(address_space, b)) return r;
  for (int r = 0; r < G->g; ++r) {
    if (n[r] >= (1ull << 32)) return fail(NMX_EINVAL, "rank %d: n must be < 2^32 per rank", r);
    if (n[r] && (!d_src[r] || !d_dst[r])) return fail(NMX_EINVAL, "rank %d: null packet columns", r);
  }
  return group_run(
      G, [&](int r) { group_rank_run(G, r, d_src[r], d_dst[r], d_valid ? d_valid[r] : nullptr, n[r], address_space); },
      out);
}

int nmx_group_stats9_host(nmx_group* G, const uint32_t* src, const uint32_t* dst, const uint8_t* valid, uint64_t n,
                          uint64_t address_space, uint64_t batch_count, int64_t out[9]) {
  if (!G || !out || (n && (!src || !dst))) return fail(NMX_EINVAL, "null argument");
  if (batch_count < 1) return fail(NMX_EINVAL, "batch_count must be >= 1");
  int b;
  if (int r = check_space(address_space, b)) return r;
  return group_run(
      G,
      [&](int r) {
        // partition_even (partitioning.py:62-70): rank r's contiguous span, remainder to the front
        const uint64_t q = n / G->g, rem = n % G->g;
        const uint64_t len = q + ((uint64_t)r < rem ? 1 : 0), off = r * q + std::min<uint64_t>(r, rem);
        GroupRank& me = G->ranks[r];
        nmx_ctx* c = me.ctx;
        me.hs.grow(std::max<uint64_t>(len, 1) * 4);
        me.hd.grow(std::max<uint64_t>(len, 1) * 4);
        if (valid) me.hv.grow(std::max<uint64_t>(len, 1));
        // b_n streaming chunks per rank (batch_table, partitioning.py:89-98)
        const uint64_t bq = len / batch_count, brem = len % batch_count;
        for (uint64_t k = 0, at = 0; k < batch_count; ++k) {
          const uint64_t bl = bq + (k < brem ? 1 : 0);
          if (!bl) continue;
          CK(cudaMemcpyAsync(me.hs.as<uint32_t>() + at, src + off + at, bl * 4, cudaMemcpyHostToDevice, c->st));
          CK(cudaMemcpyAsync(me.hd.as<uint32_t>() + at, dst + off + at, bl * 4, cudaMemcpyHostToDevice, c->st));
          if (valid)
            CK(cudaMemcpyAsync(me.hv.as<uint8_t>() + at, valid + off + at, bl, cudaMemcpyHostToDevice, c->st));
          at += bl;
        }
        group_rank_run(G, r, me.hs.as<uint32_t>(), me.hd.as<uint32_t>(), valid ? me.hv.as<uint8_t>() : nullptr, len,
                       address_space);
      },
      out);
}

int nmx_comm_unique_id(uint8_t* id) {
  if (!id) return fail(NMX_EINVAL, "null id");
  static_assert(sizeof(ncclUniqueId) == NMX_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  const NcclApi* api = nullptr;
  try {
    api = nccl_api();
  } catch (const std::exception& e) {
    return fail(NMX_ENODEV, "%s", e.what());
  }
  const ncclResult_t r = api->GetUniqueId(&u);
  if (r != ncclSuccess) return fail(NMX_ECUDA, "ncclGetUniqueId: %s", api->GetErrorString(r));
  memcpy(id, &u, sizeof(u));
  return NMX_OK;
}

int nmx_comm_init(nmx_ctx* c, const uint8_t* id, int nranks, int rank, nmx_comm** out) {
  if (!id || !out) return fail(NMX_EINVAL, "null argument");
  if (nranks < 1 || nranks > kMaxParts || rank < 0 || rank >= nranks)
    return fail(NMX_EINVAL, "need 1 <= nranks <= %d and 0 <= rank < nranks", kMaxParts);
  *out = nullptr;
  return guarded(c, [&] {
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    auto* K = new nmx_comm();
    K->nranks = nranks;
    K->rank = rank;
    K->device = c->device;
    const ncclResult_t r = nccl_api()->CommInitRank(&K->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      delete K;
      return fail(NMX_ECUDA, "ncclCommInitRank: %s", nccl_api()->GetErrorString(r));
    }
    *out = K;
    return NMX_OK;
  });
}

void nmx_comm_destroy(nmx_comm* K) {
  if (!K) return;
  cudaSetDevice(K->device);
  if (K->comm) nccl_api()->CommDestroy(K->comm);  // init succeeded, so the library is open
  delete K;
}

int nmx_stats9_sharded(nmx_ctx* c, nmx_comm* K, const uint32_t* d_src, const uint32_t* d_dst,
                       const uint8_t* d_valid, uint64_t n, uint64_t address_space, int64_t out[9]) {
  if (!K || !out || (n && (!d_src || !d_dst))) return fail(NMX_EINVAL, "null argument");
  if (K->device != (c ? c->device : -1)) return fail(NMX_EINVAL, "communicator and context on different devices");
  int b;
  if (int r = check_space(address_space, b)) return r;
  return guarded(c, [&] { return comm_run(K, c, d_src, d_dst, d_valid, n, address_space, out); });
}

int nmx_stats9_sharded_host(nmx_ctx* c, nmx_comm* K, const uint32_t* src, const uint32_t* dst,
                            const uint8_t* valid, uint64_t n, uint64_t address_space, int64_t out[9]) {
  if (!K || !out || (n && (!src || !dst))) return fail(NMX_EINVAL, "null argument");
  if (K->device != (c ? c->device : -1)) return fail(NMX_EINVAL, "communicator and context on different devices");
  int b;
  if (int r = check_space(address_space, b)) return r;
  return guarded(c, [&] {
    K->b.hs.grow(std::max<uint64_t>(n, 1) * 4);
    K->b.hd.grow(std::max<uint64_t>(n, 1) * 4);
    if (valid) K->b.hv.grow(std::max<uint64_t>(n, 1));
    if (n) {
      CK(cudaMemcpyAsync(K->b.hs.p, src, n * 4, cudaMemcpyHostToDevice, c->st));
      CK(cudaMemcpyAsync(K->b.hd.p, dst, n * 4, cudaMemcpyHostToDevice, c->st));
      if (valid) CK(cudaMemcpyAsync(K->b.hv.p, valid, n, cudaMemcpyHostToDevice, c->st));
    }
    return comm_run(K, c, K->b.hs.as<uint32_t>(), K->b.hd.as<uint32_t>(), valid ? K->b.hv.as<uint8_t>() : nullptr,
                    n, address_space, out);
  });
}

int nmx_comm_last_exchange(nmx_comm* K, uint64_t* bytes1, uint64_t* bytes2) {
  if (!K) return fail(NMX_EINVAL, "null communicator");
  if (bytes1) *bytes1 = K->last_x1;
  if (bytes2) *bytes2 = K->last_x2;
  return NMX_OK;
}

int nmx_group_last_exchange(nmx_group* G, uint64_t* bytes1, uint64_t* bytes2) {
  if (!G) return fail(NMX_EINVAL, "null group");
  if (bytes1) *bytes1 = G->last_x1;
  if (bytes2) *bytes2 = G->last_x2;
  return NMX_OK;
}

}  // extern "C"
