// DSMEM atomic throughput probe (developer tool): random u64 adds into a table that is
// distributed over the shared memory of a thread-block cluster, against the same adds
// into the CTA's own shared memory and into an L2-resident global table.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe/dsmem_probe tools/probe/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int kSlotsPerCta = 8192;  // u64 slots: 64 KB per CTA

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void red_add_u64(uint32_t a, unsigned long long v) {
  asm volatile("red.shared::cluster.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_u32(uint32_t a, uint32_t v) {
  asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// mode 0: remote (cluster-wide table), 1: local smem only, 2: remote with warp-aggregation
template <int CL>
__global__ void __launch_bounds__(1024) dsmem_kernel(uint64_t iters, unsigned long long* out, int mode) {
  extern __shared__ unsigned long long tab[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kSlotsPerCta; i += blockDim.x) tab[i] = 0;
  cl.sync();
  uint32_t h = mix(blockIdx.x * 1024 + threadIdx.x);
  for (uint64_t it = 0; it < iters; ++it) {
    h = mix(h + (uint32_t)it);
    const uint32_t slot = h & (kSlotsPerCta * CL - 1);
    const unsigned rank = mode == 1 ? cl.block_rank() : slot / kSlotsPerCta;
    if (mode == 4) {  // plain shared-memory u32 atomics on the CTA's own table
      atomicAdd(reinterpret_cast<uint32_t*>(tab) + (slot % (2 * kSlotsPerCta)), 1u);
      continue;
    }
    const uint32_t a = mapa(smem_u32(tab + (slot % kSlotsPerCta)), rank);
    if (mode == 3)
      red_add_u32(a, 1u);
    else
      red_add_u64(a, (1ull << 32) | 1ull);
  }
  cl.sync();
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < kSlotsPerCta; i += blockDim.x) s += tab[i];
  atomicAdd(out, s);
}

__global__ void gmem_kernel(uint64_t iters, unsigned long long* tab, uint32_t mask) {
  uint32_t h = mix(blockIdx.x * 1024 + threadIdx.x);
  for (uint64_t it = 0; it < iters; ++it) {
    h = mix(h + (uint32_t)it);
    atomicAdd(tab + (h & mask), (1ull << 32) | 1ull);
  }
}

template <int CL>
void run(int mode, int sms) {
  auto k = dsmem_kernel<CL>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlotsPerCta * 8);
  if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long* out;
  cudaMalloc(&out, 8);
  cudaMemset(out, 0, 8);
  const int grid = (sms / CL) * CL;
  const uint64_t iters = 4096;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = kSlotsPerCta * 8;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, iters, out, mode);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, out, mode);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)grid * 1024 * iters;
  printf("cluster %2d mode %d grid %d: %s %.3f ms, %.2f Gop/s, %.3f op/clk/SM @1.965GHz\n", CL, mode, grid,
         cudaGetErrorString(err), ms, ops / ms / 1e6, ops / (ms * 1e-3) / grid / 1.965e9);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8>(1, sms);
  run<8>(0, sms);
  run<8>(3, sms);
  run<8>(4, sms);
  run<4>(0, sms);
  run<2>(0, sms);
  run<16>(0, sms);
  for (uint32_t lg : {20, 23}) {
    unsigned long long* tab;
    cudaMalloc(&tab, (8ull << lg));
    cudaMemset(tab, 0, 8ull << lg);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint64_t iters = 1024;
    gmem_kernel<<<sms * 2, 1024>>>(iters, tab, (1u << lg) - 1);
    cudaEventRecord(e0);
    gmem_kernel<<<sms * 2, 1024>>>(iters, tab, (1u << lg) - 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)sms * 2 * 1024 * iters;
    printf("global table 2^%u u64: %.3f ms, %.2f Gop/s, %.3f op/clk/SM\n", lg, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / 1.965e9);
    cudaFree(tab);
  }
  return 0;
}
