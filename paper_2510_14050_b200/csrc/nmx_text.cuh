// nmx_text.cuh -- the reference's text matrix files on the device.
//
// Format (traffic.py:295-367): header "dim nnz", then one "row col value" line
// per nonzero, sorted row-major, no duplicates. The reference reads it with
// str.splitlines() / str.split() / int() line by line in Python (the dominant cost of
// its CLI end-to-end time); here the whole file is tokenised,
// converted and validated on the device, including the diagnosis of malformed files:
//
//   lines   : breaks are the ASCII line boundaries of str.splitlines() -- '\n', '\r',
//             "\r\n" (one break), '\v', '\f', '\x1c', '\x1d', '\x1e'; blank lines are
//             dropped but keep their number (error messages cite physical lines);
//   tokens  : separated by ASCII whitespace (' ', '\t', '\x1f' and the '\n' of "\r\n");
//             an integer is int()'s ASCII grammar [+-]?d(_?d)* within int64
//             (the reference stores entries in an int64 array);
//   checks  : in the reference's precedence -- header, per line field count then
//             integer syntax (first failing line), entry count, bounds, value >= 1,
//             strict row-major order -- each as a min-reduction over line numbers.
// Bytes >= 0x80 (non-ASCII whitespace or digits) are flagged: the caller normalises
// such text once (str.split semantics) and parses again on the device.
// Format: per-entry decimal lengths -> exclusive scan -> one thread per line.
#pragma once
#include "nmx_device.cuh"

namespace nmx {

constexpr int kTextChunk = 8192;  // bytes per block of the newline passes

// diagnosis codes (include/nmx.h NMX_TXT_*)
enum TextErr : uint32_t {
  TXT_OK = 0,
  TXT_HEADER = 1,
  TXT_DIM = 2,
  TXT_NNZ = 3,
  TXT_FIELDS = 4,
  TXT_INTEGERS = 5,
  TXT_COUNT = 6,
  TXT_BOUNDS = 7,
  TXT_VALUE = 8,
  TXT_ORDER = 9,
  TXT_WIDE = 10,
  TXT_ENCODING = 11,
};
// per-file reductions (u64 each): first (line << 4 | code) of field / integer errors,
// first line of bounds / value / order / wide errors, non-ASCII flag, first nonblank line
enum TextRed { TR_TOK = 0, TR_BOUNDS, TR_VALUE, TR_ORDER, TR_WIDE, TR_ENC, TR_HEAD, TR_N };

__device__ __forceinline__ bool text_break(const char* buf, uint64_t p) {
  const unsigned char ch = (unsigned char)buf[p];
  if (ch == '\n') return !(p > 0 && buf[p - 1] == '\r');
  return ch == '\r' || ch == '\v' || ch == '\f' || (ch >= 0x1c && ch <= 0x1e);
}
__device__ __forceinline__ bool text_space(unsigned char ch) {
  return ch == ' ' || ch == '\t' || ch == 0x1f || ch == '\n';
}

__global__ void __launch_bounds__(256) text_nl_count_kernel(const char* __restrict__ buf, uint64_t T,
                                                           uint32_t* __restrict__ bcount) {
  __shared__ uint32_t wt[kWarps + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kTextChunk;
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < kTextChunk; i += 256) {
    const uint64_t p = base + i;
    if (p < T && text_break(buf, p)) ++c;
  }
  uint32_t tot;
  block_excl_scan<uint32_t>(c, wt, &tot);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// ends[k] = position of the k-th break (blocked: thread t scans bytes [32t, 32t+32) of the chunk)
__global__ void __launch_bounds__(256) text_nl_write_kernel(const char* __restrict__ buf, uint64_t T,
                                                           const uint32_t* __restrict__ boff,
                                                           uint64_t* __restrict__ ends) {
  __shared__ uint32_t wt[kWarps + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kTextChunk + threadIdx.x * (kTextChunk / 256);
  uint32_t c = 0;
  for (int i = 0; i < kTextChunk / 256; ++i) {
    const uint64_t p = base + i;
    if (p < T && text_break(buf, p)) ++c;
  }
  uint32_t tot;
  uint32_t at = boff[blockIdx.x] + block_excl_scan<uint32_t>(c, wt, &tot);
  for (int i = 0; i < kTextChunk / 256; ++i) {
    const uint64_t p = base + i;
    if (p < T && text_break(buf, p)) ends[at++] = p;
  }
}

// Line l spans [l ? ends[l-1] + 1 : 0, ends[l]) (ends[L-1] = T for an unterminated
// last line). ntok[l] = tokens (capped at 4) | 0x80 if one of the first three is not an
// int64 integer; vals[3l..3l+2] the first three values.
__global__ void text_parse_lines_kernel(const char* __restrict__ buf, const uint64_t* __restrict__ ends, uint64_t L,
                                        uint8_t* __restrict__ ntok, long long* __restrict__ vals,
                                        unsigned long long* __restrict__ red) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = l ? ends[l - 1] + 1 : 0, z = ends[l];
    int nt = 0;
    long long v[3] = {0, 0, 0};
    bool in = false, neg = false, ok = true, invalid = false, enc = false;
    int last = 0;  // 0 start, 1 digit, 2 underscore, 3 sign
    unsigned long long acc = 0;
    auto finish = [&]() {
      const bool good = ok && last == 1 && acc <= (neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull);
      if (nt < 3) {
        v[nt] = good ? (neg ? (long long)(0ull - acc) : (long long)acc) : 0;
        if (!good) invalid = true;
      }
      ++nt;
      in = neg = false;
      ok = true;
      last = 0;
      acc = 0;
    };
    for (uint64_t p = a; p < z; ++p) {
      const unsigned char ch = (unsigned char)buf[p];
      if (text_space(ch)) {
        if (in) finish();
        continue;
      }
      if (ch >= 0x80) enc = true;
      if (!in) in = true;
      if (ch >= '0' && ch <= '9') {
        if (acc > 0x0CCCCCCCCCCCCCCCull) ok = false;  // beyond int64 (the reference's OverflowError)
        acc = acc * 10 + (unsigned)(ch - '0');
        last = 1;
      } else if (ch == '_' && last == 1) {
        last = 2;
      } else if ((ch == '-' || ch == '+') && last == 0 && ok) {  // a sign only at the token start
        neg = ch == '-';
        last = 3;
      } else {
        ok = false;
      }
    }
    if (in) finish();
    ntok[l] = (uint8_t)((nt > 4 ? 4 : nt) | (invalid ? 0x80 : 0));
    vals[3 * l] = v[0];
    vals[3 * l + 1] = v[1];
    vals[3 * l + 2] = v[2];
    if (enc) atomicOr(red + TR_ENC, 1ull);
    if (nt) atomicMin(red + TR_HEAD, (unsigned long long)l);
  }
}

__global__ void text_nonblank_kernel(const uint8_t* __restrict__ ntok, uint64_t L, uint32_t* __restrict__ nb) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x)
    nb[l] = (ntok[l] & 0x7F) ? 1u : 0u;
}

// entry lines (nonblank j >= 1) -> COO key (row << 32 | col), int64 value and the
// line number; the first field / integer error as (line << 4 | code), the first
// bounds and value lines (1-based physical line numbers)
__global__ void text_entries_kernel(const uint8_t* __restrict__ ntok, const long long* __restrict__ vals,
                                    const uint32_t* __restrict__ nboff, uint64_t L, long long dim,
                                    unsigned long long* __restrict__ keys, uint64_t* __restrict__ cnt,
                                    uint32_t* __restrict__ eline, unsigned long long* __restrict__ red) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t t = ntok[l];
    if (!(t & 0x7F)) continue;
    const uint32_t j = nboff[l];
    if (j == 0) continue;  // the header (checked on the host)
    const unsigned long long line = l + 1;
    const long long* v = vals + 3 * l;
    eline[j - 1] = (uint32_t)line;
    keys[j - 1] = 0;
    cnt[j - 1] = 0;
    if ((t & 0x7F) != 3) {
      atomicMin(red + TR_TOK, line << 4 | TXT_FIELDS);
      continue;
    }
    if (t & 0x80) {
      atomicMin(red + TR_TOK, line << 4 | TXT_INTEGERS);
      continue;
    }
    if (v[0] < 0 || v[0] >= dim || v[1] < 0 || v[1] >= dim) {
      atomicMin(red + TR_BOUNDS, line);
      continue;
    }
    if (v[2] < 1) atomicMin(red + TR_VALUE, line);
    keys[j - 1] = ((unsigned long long)v[0] << 32) | (unsigned long long)v[1];
    cnt[j - 1] = (uint64_t)v[2];
  }
}

// keys strictly increasing (row-major, no duplicates): first offending line
__global__ void text_order_kernel(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ eline,
                                  uint64_t nnz, unsigned long long* __restrict__ red) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < nnz; i += (uint64_t)gridDim.x * blockDim.x)
    if (keys[i - 1] >= keys[i]) atomicMin(red + TR_ORDER, (unsigned long long)eline[i]);
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
