// nmx_io.cuh -- packet-file records on the device.
//
// The reference's binary packet file is an array of 9-byte little-endian
// records {u32 src, u32 dst, u8 valid} (traffic.py:25 _PACKET_DTYPE,
// write_packets / read_packets traffic.py:370-388). Records are streamed to the
// device as raw bytes (9 B/packet, no host-side conversion) and unpacked into
// the u32 / u32 / u8 columns the pipeline reads: four records = 36 bytes = nine
// aligned 32-bit words per thread, split with funnel shifts, written as 128-bit
// src / dst stores and one 32-bit valid store. Every address (valid or not) is
// range-checked like PacketStream.__post_init__ (traffic.py:56-64) through a
// max-reduction.
#pragma once
#include "nmx_device.cuh"

namespace nmx {

__device__ __forceinline__ uint32_t rec_u32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// rec: 4-byte aligned; src / dst 16-byte aligned, valid 4-byte aligned
__global__ void __launch_bounds__(256) unpack_records_kernel(const uint8_t* __restrict__ rec, uint64_t n,
                                                            uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                            uint8_t* __restrict__ valid,
                                                            unsigned int* __restrict__ maxaddr) {
  uint32_t mx = 0;
  const uint64_t nq = (n + 3) / 4;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
    if (4 * q + 4 <= n) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(rec) + 9 * q;
      uint32_t x[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) x[i] = __ldg(w + i);
      // record r starts at byte 9r: r = 0 at word 0, r = 1 at byte 1 of word 2,
      // r = 2 at byte 2 of word 4, r = 3 at byte 3 of word 6
      const uint4 s4 = make_uint4(x[0], __funnelshift_r(x[2], x[3], 8), __funnelshift_r(x[4], x[5], 16),
                                  __funnelshift_r(x[6], x[7], 24));
      const uint4 d4 = make_uint4(x[1], __funnelshift_r(x[3], x[4], 8), __funnelshift_r(x[5], x[6], 16),
                                  __funnelshift_r(x[7], x[8], 24));
      const uint32_t v4 = ((x[2] & 0xFFu) != 0) | (((x[4] >> 8) & 0xFFu) != 0) << 8 |
                          (((x[6] >> 16) & 0xFFu) != 0) << 16 | ((x[8] >> 24) != 0) << 24;
      reinterpret_cast<uint4*>(src)[q] = s4;
      reinterpret_cast<uint4*>(dst)[q] = d4;
      reinterpret_cast<uint32_t*>(valid)[q] = v4;
      mx = max(mx, max(max(max(s4.x, s4.y), max(s4.z, s4.w)), max(max(d4.x, d4.y), max(d4.z, d4.w))));
    } else {
      for (uint64_t i = 4 * q; i < n; ++i) {
        const uint8_t* r = rec + 9 * i;
        const uint32_t s = rec_u32(r), d = rec_u32(r + 4);
        src[i] = s;
        dst[i] = d;
        valid[i] = r[8] != 0;
        mx = max(mx, max(s, d));
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxaddr, mx);
}

}  // namespace nmx

namespace nmx {

// ---------------------------------------------------------------------------
// anonymize (traffic.py:107-137) on the device, SURVEY.md 8(f) f3.
// Addresses of the interleaved stream e = 2p (src of packet p), 2p + 1 (dst)
// are stably sorted with their positions; run heads give the distinct addresses
// and their first positions; the first-seen rank of an address is the number of
// first positions before its own (a flag scan over positions); its code is
// perm[rank] with perm = default_rng(key).permutation(k) drawn by the caller.
// ---------------------------------------------------------------------------
__global__ void anon_pairs_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t n,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ pos) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    reinterpret_cast<uint2*>(keys)[p] = make_uint2(src[p], dst[p]);
    reinterpret_cast<uint2*>(pos)[p] = make_uint2((uint32_t)(2 * p), (uint32_t)(2 * p + 1));
  }
}

// head[j] = 1 where a new address starts in the sorted keys
__global__ void anon_heads_kernel(const uint32_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ head) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x)
    head[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1u : 0u;
}

// per head j (uid = hoff[j]): distinct[uid] = address, first[uid] = its first
// position (stable sort: the run's first element), flag[first] = 1
__global__ void anon_uniques_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ pos,
                                    const uint32_t* __restrict__ head, const uint32_t* __restrict__ hoff, uint64_t m,
                                    uint32_t* __restrict__ distinct, uint32_t* __restrict__ first,
                                    uint32_t* __restrict__ flag) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[j]) continue;
    const uint32_t u = hoff[j];
    distinct[u] = keys[j];
    first[u] = pos[j];
    flag[pos[j]] = 1u;
  }
}

// code[u] = perm[rank(u)], rank(u) = number of first positions before first[u]
__global__ void anon_codes_kernel(const uint32_t* __restrict__ first, const uint32_t* __restrict__ foff,
                                  const uint32_t* __restrict__ perm, uint64_t k, uint32_t* __restrict__ code) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < k; u += (uint64_t)gridDim.x * blockDim.x)
    code[u] = perm[foff[first[u]]];
}

// relabel: element j of the sorted stream (address run uid = hoff[j] + head[j] - 1)
// writes its code back to its packet position
__global__ void anon_scatter_kernel(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ head,
                                    const uint32_t* __restrict__ hoff, uint64_t m, const uint32_t* __restrict__ code,
                                    uint32_t* __restrict__ src_out, uint32_t* __restrict__ dst_out) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = pos[j];
    const uint32_t c = code[hoff[j] + head[j] - 1];
    if (e & 1u)
      dst_out[e >> 1] = c;
    else
      src_out[e >> 1] = c;
  }
}


// Largest address of u32 src / dst columns (every packet, valid or not, like
// PacketStream.__post_init__, traffic.py:56-64), max-reduced into *maxaddr. Run by
// every device entry whose address_space is below 2^32 before any key is packed:
// an out-of-range address would otherwise carry bits above the 2b-bit key.
__global__ void __launch_bounds__(256) max_addr_kernel(const uint32_t* __restrict__ src,
                                                       const uint32_t* __restrict__ dst, uint64_t n,
                                                       unsigned int* __restrict__ maxaddr) {
  uint32_t mx = 0;
  const bool vec = !(((uintptr_t)src | (uintptr_t)dst) & 15);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const uint64_t nq = n / 4;
    for (uint64_t q = i0; q < nq; q += stride) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(src) + q);
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(dst) + q);
      mx = max(mx, max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w))));
    }
    for (uint64_t i = 4 * nq + i0; i < n; i += stride) mx = max(mx, max(src[i], dst[i]));
  } else {
    for (uint64_t i = i0; i < n; i += stride) mx = max(mx, max(src[i], dst[i]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxaddr, mx);
}

}  // namespace nmx
