// nmx_text.cuh -- the reference's text matrix files on the device.
//
// Format (traffic.py:295-367): header "dim nnz", then one "row col value" line
// per nonzero, sorted row-major, no duplicates; written with single spaces and
// '\n'. The reference parses it line by line in Python (the dominant cost of its
// CLI end-to-end time).
//
// Parse: newline positions (per-block counts -> scan -> per-block write), one
// thread per line tokenises up to three integers; nonblank lines are compacted
// (header first), entries validated (3 tokens, bounds, value >= 1, strictly
// increasing row*dim+col) straight into a device COO. The fast path accepts
// only digits, '+'/'-' signs, ' ', '\t' and '\n'; anything else (and any
// validation failure) is reported so the host re-parses with the exact
// reference semantics and error messages.
// Format: per-entry decimal lengths -> exclusive scan -> one thread per line.
#pragma once
#include "nmx_device.cuh"

namespace nmx {

constexpr int kTextChunk = 8192;  // bytes per block of the newline passes

__global__ void __launch_bounds__(256) text_nl_count_kernel(const char* __restrict__ buf, uint64_t T,
                                                           uint32_t* __restrict__ bcount) {
  __shared__ uint32_t wt[kWarps + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kTextChunk;
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < kTextChunk; i += 256) {
    const uint64_t p = base + i;
    if (p < T && buf[p] == '\n') ++c;
  }
  uint32_t tot;
  block_excl_scan<uint32_t>(c, wt, &tot);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// ends[k] = position of the k-th '\n' (blocked: thread t scans bytes [32t, 32t+32) of the chunk)
__global__ void __launch_bounds__(256) text_nl_write_kernel(const char* __restrict__ buf, uint64_t T,
                                                           const uint32_t* __restrict__ boff,
                                                           uint64_t* __restrict__ ends) {
  __shared__ uint32_t wt[kWarps + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kTextChunk + threadIdx.x * (kTextChunk / 256);
  uint32_t c = 0;
  for (int i = 0; i < kTextChunk / 256; ++i) {
    const uint64_t p = base + i;
    if (p < T && buf[p] == '\n') ++c;
  }
  uint32_t tot;
  uint32_t at = boff[blockIdx.x] + block_excl_scan<uint32_t>(c, wt, &tot);
  for (int i = 0; i < kTextChunk / 256; ++i) {
    const uint64_t p = base + i;
    if (p < T && buf[p] == '\n') ends[at++] = p;
  }
}

// Line l spans [l ? ends[l-1] + 1 : 0, ends[l]) (ends[L-1] = T for an unterminated
// last line). ntok[l] = tokens (capped at 4), vals[3l..3l+2] the first three.
// bad |= 1: a byte outside the fast-path alphabet or a malformed / oversized token.
__global__ void text_parse_lines_kernel(const char* __restrict__ buf, const uint64_t* __restrict__ ends, uint64_t L,
                                        uint8_t* __restrict__ ntok, long long* __restrict__ vals,
                                        unsigned int* __restrict__ bad) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = l ? ends[l - 1] + 1 : 0, z = ends[l];
    int nt = 0;
    long long v[3] = {0, 0, 0};
    bool in = false, neg = false, digits = false, fail = false;
    unsigned long long acc = 0;
    auto finish = [&]() {
      if (!digits || acc > 0x7FFFFFFFFFFFFFFFull) fail = true;
      if (nt < 3) v[nt] = neg ? -(long long)acc : (long long)acc;
      ++nt;
      in = neg = digits = false;
      acc = 0;
    };
    for (uint64_t p = a; p < z; ++p) {
      const char ch = buf[p];
      if (ch == ' ' || ch == '\t') {
        if (in) finish();
      } else if (ch >= '0' && ch <= '9') {
        if (!in) in = true;
        if (acc > 0x0CCCCCCCCCCCCCCCull) fail = true;  // would exceed int64 soon; exact text on the host
        acc = acc * 10 + (unsigned)(ch - '0');
        digits = true;
      } else if ((ch == '-' || ch == '+') && !in) {
        in = true;
        neg = ch == '-';
      } else {
        fail = true;  // any other byte (incl. '\r', '_', letters): host re-parse
        if (in) finish();
      }
    }
    if (in) finish();
    ntok[l] = (uint8_t)(nt > 4 ? 4 : nt);
    vals[3 * l] = v[0];
    vals[3 * l + 1] = v[1];
    vals[3 * l + 2] = v[2];
    if (fail) atomicOr(bad, 1u);
  }
}

__global__ void text_nonblank_kernel(const uint8_t* __restrict__ ntok, uint64_t L, uint32_t* __restrict__ nb) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x)
    nb[l] = ntok[l] ? 1u : 0u;
}

// nonblank line j (= nboff[l]): j == 0 -> header (2 tokens), else entry j - 1 (3 tokens)
// -> COO key (row << 32 | col) and u32 count; validation flags into *bad (bit 1: token
// counts, bit 2: bounds / values / order); header tokens to hdr[0..1]
__global__ void text_entries_kernel(const uint8_t* __restrict__ ntok, const long long* __restrict__ vals,
                                    const uint32_t* __restrict__ nboff, uint64_t L, long long* __restrict__ hdr,
                                    unsigned long long* __restrict__ keys, uint32_t* __restrict__ cnt,
                                    unsigned int* __restrict__ bad) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x) {
    if (!ntok[l]) continue;
    const uint32_t j = nboff[l];
    const long long* t = vals + 3 * l;
    if (j == 0) {
      if (ntok[l] != 2) atomicOr(bad, 2u);
      hdr[0] = t[0];
      hdr[1] = t[1];
      continue;
    }
    if (ntok[l] != 3) {
      atomicOr(bad, 2u);
      continue;
    }
    if (t[0] < 0 || t[1] < 0 || t[0] >= (1ll << 31) || t[1] >= (1ll << 31) || t[2] < 1 || t[2] > 0xFFFFFFFFll) {
      atomicOr(bad, 4u);  // the host decides which message (bounds vs value) applies
      keys[j - 1] = 0;
      cnt[j - 1] = 0;
      continue;
    }
    keys[j - 1] = ((unsigned long long)t[0] << 32) | (unsigned long long)t[1];
    cnt[j - 1] = (uint32_t)t[2];
  }
}

// rows / cols inside [0, dim) and keys strictly increasing
__global__ void text_check_kernel(const unsigned long long* __restrict__ keys, uint64_t nnz, long long dim,
                                  unsigned int* __restrict__ bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    if ((long long)(k >> 32) >= dim || (long long)(k & 0xFFFFFFFFull) >= dim) atomicOr(bad, 4u);
    if (i && keys[i - 1] >= k) atomicOr(bad, 4u);
  }
}

// ---- formatting --------------------------------------------------------------
__global__ void widen_offsets_kernel(const uint32_t* __restrict__ off32, uint64_t n, unsigned long long* __restrict__ off) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    off[i] = off32[i];
}
__device__ __forceinline__ uint32_t dec_len(unsigned long long v) {
  uint32_t n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}
__device__ __forceinline__ char* dec_put(char* p, unsigned long long v, uint32_t n) {
  for (uint32_t i = n; i > 0; --i) {
    p[i - 1] = (char)('0' + v % 10);
    v /= 10;
  }
  return p + n;
}

__global__ void text_line_len_kernel(const unsigned long long* __restrict__ rows,
                                     const unsigned long long* __restrict__ cols,
                                     const unsigned long long* __restrict__ vals, uint64_t nnz,
                                     uint32_t* __restrict__ len) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (uint64_t)gridDim.x * blockDim.x)
    len[i] = dec_len(rows[i]) + dec_len(cols[i]) + dec_len(vals[i]) + 3;
}

__global__ void text_write_lines_kernel(const unsigned long long* __restrict__ rows,
                                        const unsigned long long* __restrict__ cols,
                                        const unsigned long long* __restrict__ vals, uint64_t nnz,
                                        const unsigned long long* __restrict__ off, char* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (uint64_t)gridDim.x * blockDim.x) {
    char* p = out + off[i];
    p = dec_put(p, rows[i], dec_len(rows[i]));
    *p++ = ' ';
    p = dec_put(p, cols[i], dec_len(cols[i]));
    *p++ = ' ';
    p = dec_put(p, vals[i], dec_len(vals[i]));
    *p = '\n';
  }
}

}  // namespace nmx
