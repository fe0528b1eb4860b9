/* Bounded-RAM chunked packed-key oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * This file is the checker, never the product: it is compiled by
 * __graft_entry__.build() into oracle/_build/libnmx_oracle.so and loaded only by
 * tests/, tools/ and oracle/make_full_size.py (through oracle/big.py).  The
 * product package never links or loads it.
 *
 * What it restates (citations relative to /root/reference/pkg/src/netmeter):
 *
 *   build_matrices(stream, len(stream))      traffic.py:221-242  (one window, invalid dropped)
 *     matrix_from_pairs: unique(src*dim+dst)  traffic.py:197-218  (links = runs of equal keys)
 *   to_flat: weights, out_degrees, row_sums   traffic.py:263-284  (per-source runs)
 *            in_degrees, col_sums             traffic.py:285-292  (per-destination groups)
 *   analyze_matrix + 3 x max_scan             analytics.py:89-106 (sum / count / max, empty -> 0)
 *
 * with the packed key (src << 32) | dst, which orders exactly like src*dim+dst
 * for every dim <= 2^32.  It never materialises the
 * whole stream: the packets are regenerated (or re-read) once per bucket.
 *
 *   rows    : for each bucket of source addresses, gather key = src<<32|dst of the
 *             bucket's valid packets, sort, and run-length encode: every run is a
 *             link (count = run length); runs of equal src give the source's
 *             packets and fan-out.  Buckets hold disjoint sources, so the
 *             statistics combine by sum / max.
 *   columns : the same with key = dst<<32|src, bucketed by destination: runs of
 *             equal key are links again, runs of equal dst give the destination's
 *             packets and fan-in (its number of distinct links).
 *
 * valid_packets and unique_links come out of both halves and must agree; that
 * is asserted (return code -3 on a mismatch).
 *
 * The generators restate oracle/netmeter_oracle.py gen_uniform / gen_powerlaw
 * bit for bit: counter c = (seed << 40) + 2i (mod 2^64),
 * src from splitmix64(c), dst from splitmix64(c + 1); the power-law "octave"
 * map; multiply-shift scaling onto [0, address_space).
 *
 * Parity pinning: tests/test_oracle.py checks this file against the reference-
 * generated splitmix64 goldens (tests/golden/golden.json, 2^16 .. 2^24, made by
 * the real netmeter package) and against stats9_packed at 2^26.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KIND_UNIFORM 0
#define KIND_POWERLAW 1

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint32_t octave(uint64_t bits) {
  uint64_t e = bits >> 59;
  uint64_t rank = (1ull << e) | (bits & ((1ull << e) - 1ull));
  return (uint32_t)(rank * 0x9E3779B1ull);
}

static inline uint32_t scale(uint32_t v, uint64_t space) {
  if (space == (1ull << 32)) return v;
  return (uint32_t)(((uint64_t)v * space) >> 32);
}

/* One packet source: either the counter-based generator or borrowed arrays. */
typedef struct {
  int kind; /* -1 = arrays */
  uint64_t seed_base, offset, n, space;
  const uint32_t *src, *dst;
  const uint8_t *valid;
} source_t;

static inline int packet(const source_t *s, uint64_t i, uint32_t *a, uint32_t *b) {
  if (s->kind < 0) {
    if (s->valid && !s->valid[i]) return 0;
    *a = s->src[i];
    *b = s->dst[i];
    return 1;
  }
  uint64_t c = s->seed_base + 2ull * (s->offset + i);
  uint64_t x = splitmix64(c), y = splitmix64(c + 1ull);
  if (s->kind == KIND_UNIFORM) {
    *a = scale((uint32_t)x, s->space);
    *b = scale((uint32_t)(y >> 32), s->space);
  } else {
    *a = scale(octave(x), s->space);
    *b = scale(octave(y), s->space);
  }
  return 1;
}

/* LSD radix sort of u64 keys, 11-bit digits, passes whose digit is constant skipped. */
static void radix_sort(uint64_t *a, uint64_t *tmp, uint64_t n) {
  if (n < 2) return;
  if (n < 64) { /* insertion sort */
    for (uint64_t i = 1; i < n; i++) {
      uint64_t v = a[i], j = i;
      while (j > 0 && a[j - 1] > v) { a[j] = a[j - 1]; j--; }
      a[j] = v;
    }
    return;
  }
  uint64_t *src = a, *dst = tmp;
  static const int D = 11;
  uint64_t *cnt = (uint64_t *)malloc(sizeof(uint64_t) << D);
  for (int shift = 0; shift < 64; shift += D) {
    memset(cnt, 0, sizeof(uint64_t) << D);
    uint64_t mask = (1ull << D) - 1;
    for (uint64_t i = 0; i < n; i++) cnt[(src[i] >> shift) & mask]++;
    int trivial = 0;
    for (uint64_t d = 0; d <= mask; d++)
      if (cnt[d] == n) trivial = 1;
    if (trivial) continue;
    uint64_t s = 0;
    for (uint64_t d = 0; d <= mask; d++) { uint64_t c = cnt[d]; cnt[d] = s; s += c; }
    for (uint64_t i = 0; i < n; i++) dst[cnt[(src[i] >> shift) & mask]++] = src[i];
    uint64_t *t = src; src = dst; dst = t;
  }
  if (src != a) memcpy(a, src, n * sizeof(uint64_t));
  free(cnt);
}

typedef struct {
  int64_t valid, links, max_link, groups, max_group_pk, max_group_nnz;
} half_t;

/* Run-length statistics of a sorted key range whose groups (key >> 32) do not cross it. */
static void reduce_sorted(const uint64_t *k, uint64_t n, half_t *h) {
  uint64_t i = 0;
  while (i < n) {
    uint64_t g = k[i] >> 32;
    int64_t gpk = 0, gnnz = 0;
    while (i < n && (k[i] >> 32) == g) {
      uint64_t key = k[i], j = i + 1;
      while (j < n && k[j] == key) j++;
      int64_t c = (int64_t)(j - i);
      h->links++;
      if (c > h->max_link) h->max_link = c;
      gpk += c;
      gnnz++;
      i = j;
    }
    h->valid += gpk;
    h->groups++;
    if (gpk > h->max_group_pk) h->max_group_pk = gpk;
    if (gnnz > h->max_group_nnz) h->max_group_nnz = gnnz;
  }
}

static int bits_of(uint64_t space) {
  int b = 0;
  while (b < 32 && (1ull << b) < space) b++;
  return b;
}

/* One half: key = major<<32 | minor, buckets by the top bucket_bits of the major
 * address, sub-buckets by the next 8 bits (sorted independently in parallel). */
static int run_half(const source_t *s, int swap, int bucket_bits, half_t *out) {
  int b = s->kind < 0 ? 32 : bits_of(s->space);
  if (bucket_bits > b) bucket_bits = b;
  int shift = b - bucket_bits;                /* major >> shift = bucket */
  int sub_bits = shift < 8 ? shift : 8;       /* sub-bucket = (major >> sub_shift) & mask */
  int sub_shift = shift - sub_bits;
  uint64_t nb = 1ull << bucket_bits, ns = 1ull << sub_bits;
  int T = omp_get_max_threads();
  uint64_t chunk = (s->n + T - 1) / T;
  if (chunk == 0) chunk = 1;
  /* per-thread-chunk bucket histogram (one generation pass) */
  uint64_t *hist = (uint64_t *)calloc((size_t)T * nb, sizeof(uint64_t));
  if (!hist) return -1;
#pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    uint64_t lo = (uint64_t)t * chunk, hi = lo + chunk < s->n ? lo + chunk : s->n;
    uint64_t *h = hist + (size_t)t * nb;
    for (uint64_t i = lo; i < hi; i++) {
      uint32_t a, c;
      if (!packet(s, i, &a, &c)) continue;
      uint32_t major = swap ? c : a;
      h[(uint64_t)major >> shift]++;
    }
  }
  uint64_t maxb = 0;
  for (uint64_t k = 0; k < nb; k++) {
    uint64_t tot = 0;
    for (int t = 0; t < T; t++) tot += hist[(size_t)t * nb + k];
    if (tot > maxb) maxb = tot;
  }
  uint64_t *keys = (uint64_t *)malloc((maxb ? maxb : 1) * sizeof(uint64_t));
  uint64_t *tmp = (uint64_t *)malloc((maxb ? maxb : 1) * sizeof(uint64_t));
  uint64_t *subc = (uint64_t *)malloc((ns + 1) * sizeof(uint64_t));
  uint64_t *toff = (uint64_t *)malloc((size_t)T * sizeof(uint64_t));
  if (!keys || !tmp || !subc || !toff) { free(hist); free(keys); free(tmp); free(subc); free(toff); return -1; }
  memset(out, 0, sizeof(*out));
  for (uint64_t bk = 0; bk < nb; bk++) {
    uint64_t tot = 0;
    for (int t = 0; t < T; t++) { toff[t] = tot; tot += hist[(size_t)t * nb + bk]; }
    if (tot == 0) continue;
#pragma omp parallel num_threads(T)
    {
      int t = omp_get_thread_num();
      uint64_t lo = (uint64_t)t * chunk, hi = lo + chunk < s->n ? lo + chunk : s->n;
      uint64_t w = toff[t];
      for (uint64_t i = lo; i < hi; i++) {
        uint32_t a, c;
        if (!packet(s, i, &a, &c)) continue;
        uint32_t major = swap ? c : a, minor = swap ? a : c;
        if (((uint64_t)major >> shift) != bk) continue;
        keys[w++] = ((uint64_t)major << 32) | minor;
      }
    }
    /* sub-bucket scatter (serial counting sort on 8 address bits) */
    memset(subc, 0, (ns + 1) * sizeof(uint64_t));
    uint64_t smask = ns - 1;
    for (uint64_t i = 0; i < tot; i++) subc[((keys[i] >> 32) >> sub_shift & smask) + 1]++;
    for (uint64_t d = 0; d < ns; d++) subc[d + 1] += subc[d];
    {
      uint64_t *cur = (uint64_t *)malloc(ns * sizeof(uint64_t));
      memcpy(cur, subc, ns * sizeof(uint64_t));
      for (uint64_t i = 0; i < tot; i++) tmp[cur[(keys[i] >> 32) >> sub_shift & smask]++] = keys[i];
      free(cur);
    }
    half_t acc = {0, 0, 0, 0, 0, 0};
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
    for (uint64_t d = 0; d < ns; d++) {
      uint64_t lo = subc[d], len = subc[d + 1] - lo;
      if (!len) continue;
      radix_sort(tmp + lo, keys + lo, len);
      half_t h = {0, 0, 0, 0, 0, 0};
      reduce_sorted(tmp + lo, len, &h);
#pragma omp critical
      {
        acc.valid += h.valid;
        acc.links += h.links;
        acc.groups += h.groups;
        if (h.max_link > acc.max_link) acc.max_link = h.max_link;
        if (h.max_group_pk > acc.max_group_pk) acc.max_group_pk = h.max_group_pk;
        if (h.max_group_nnz > acc.max_group_nnz) acc.max_group_nnz = h.max_group_nnz;
      }
    }
    out->valid += acc.valid;
    out->links += acc.links;
    out->groups += acc.groups;
    if (acc.max_link > out->max_link) out->max_link = acc.max_link;
    if (acc.max_group_pk > out->max_group_pk) out->max_group_pk = acc.max_group_pk;
    if (acc.max_group_nnz > out->max_group_nnz) out->max_group_nnz = acc.max_group_nnz;
  }
  free(hist); free(keys); free(tmp); free(subc); free(toff);
  return 0;
}

static int stats9(const source_t *s, int bucket_bits, int64_t out[9]) {
  half_t r, c;
  int rc = run_half(s, 0, bucket_bits, &r);
  if (rc) return rc;
  rc = run_half(s, 1, bucket_bits, &c);
  if (rc) return rc;
  if (r.valid != c.valid || r.links != c.links || r.max_link != c.max_link) return -3;
  out[0] = r.valid;          /* valid_packets            sum(weights)       analytics.py:101 */
  out[1] = r.links;          /* unique_links             len(edges)         analytics.py:102 */
  out[2] = r.max_link;       /* max_link_packets         max_scan(weights)  analytics.py:89-92 */
  out[3] = r.groups;         /* unique_sources           len(row_sums)      analytics.py:103 */
  out[4] = r.max_group_pk;   /* max_source_packets       max_scan(row_sums[:,1]) */
  out[5] = r.max_group_nnz;  /* max_fanout               max(out_degrees)   analytics.py:104 */
  out[6] = c.groups;         /* unique_destinations      len(col_sums)      analytics.py:105 */
  out[7] = c.max_group_pk;   /* max_destination_packets  max_scan(col_sums[:,1]) */
  out[8] = c.max_group_nnz;  /* max_fanin                max(in_degrees)    analytics.py:106 */
  return 0;
}

/* Nine statistics of the summed matrix of generated packets [offset, offset+n). */
int nmx_oracle_stats9_gen(int kind, uint64_t seed, uint64_t offset, uint64_t n, uint64_t space,
                          int bucket_bits, int64_t out[9]) {
  if ((kind != KIND_UNIFORM && kind != KIND_POWERLAW) || space < 1 || space > (1ull << 32)) return -2;
  source_t s = {kind, seed << 40, offset, n, space, NULL, NULL, NULL};
  return stats9(&s, bucket_bits, out);
}

/* Nine statistics of borrowed u32 columns (valid may be NULL = all valid). */
int nmx_oracle_stats9_pairs(const uint32_t *src, const uint32_t *dst, const uint8_t *valid, uint64_t n,
                            int bucket_bits, int64_t out[9]) {
  source_t s = {-1, 0, 0, n, 1ull << 32, src, dst, valid};
  return stats9(&s, bucket_bits, out);
}

/* The generator alone (chunk-addressable), for cross-checking gen_uniform / gen_powerlaw. */
int nmx_oracle_generate(int kind, uint64_t seed, uint64_t offset, uint64_t n, uint64_t space, uint32_t *src,
                        uint32_t *dst) {
  if ((kind != KIND_UNIFORM && kind != KIND_POWERLAW) || space < 1 || space > (1ull << 32)) return -2;
  source_t s = {kind, seed << 40, offset, n, space, NULL, NULL, NULL};
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; i++) packet(&s, i, &src[i], &dst[i]);
  return 0;
}

int nmx_oracle_threads(void) { return omp_get_max_threads(); }
