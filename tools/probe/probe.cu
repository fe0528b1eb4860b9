// Throwaway device probe: props, cub sort comparator, smem-atomic histogram rate, H2D bandwidth.
#include <cstdio>
#include <cstdint>
#include <cub/cub.cuh>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

__device__ __forceinline__ uint64_t sm64(uint64_t x){ x+=0x9E3779B97F4A7C15ull; x=(x^(x>>30))*0xBF58476D1CE4E5B9ull; x=(x^(x>>27))*0x94D049BB133111EBull; return x^(x>>31);}
__global__ void gen(uint64_t* k, size_t n){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) k[i]=sm64(i);}
__global__ void copyk(const uint4* a, uint4* b, size_t n){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];}
template<int NDIG>
__global__ void hist(const uint64_t* k, size_t n, unsigned* gh){
  __shared__ unsigned h[NDIG][256];
  for(int i=threadIdx.x;i<NDIG*256;i+=blockDim.x) (&h[0][0])[i]=0;
  __syncthreads();
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ uint64_t x=k[i];
#pragma unroll
    for(int d=0;d<NDIG;d++) atomicAdd(&h[d][(x>>(8*d))&255],1u);}
  __syncthreads();
  for(int i=threadIdx.x;i<NDIG*256;i+=blockDim.x) atomicAdd(gh+i,(&h[0][0])[i]);
}
__global__ void matchk(const uint64_t* k, size_t n, unsigned* out){
  unsigned acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ uint64_t x=k[i];
#pragma unroll
    for(int d=0;d<8;d++){ unsigned m=__match_any_sync(0xffffffffu,(unsigned)(x>>(8*d))&255); acc+=__popc(m);} }
  if(acc==0xdeadbeef) out[0]=acc;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("dev %s sms %d smemPerSM %zu smemOptin %zu l2 %d mem %zu GB clock %d\n",p.name,p.multiProcessorCount,p.sharedMemPerMultiprocessor,p.sharedMemPerBlockOptin,p.l2CacheSize,p.totalGlobalMem>>30,p.clockRate);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for(int lg: {24,27,30}){
    size_t n=1ull<<lg; uint64_t *k,*k2; CK(cudaMalloc(&k,n*8)); CK(cudaMalloc(&k2,n*8));
    gen<<<148*8,256>>>(k,n);
    void* tmp=nullptr; size_t tb=0; cub::DeviceRadixSort::SortKeys(tmp,tb,k,k2,(int)n); CK(cudaMalloc(&tmp,tb));
    for(int r=0;r<3;r++){ cudaEventRecord(a); cub::DeviceRadixSort::SortKeys(tmp,tb,k,k2,(int)n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("cub sort u64 2^%d: %.3f ms  %.2f Gkeys/s\n",lg,ms,n/ms/1e6);
    for(int r=0;r<3;r++){ cudaEventRecord(a); cub::DeviceRadixSort::SortKeys(tmp,tb,(uint32_t*)k,(uint32_t*)k2,(int)n); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("cub sort u32 2^%d: %.3f ms  %.2f Gkeys/s\n",lg,ms,n/ms/1e6);
    cudaFree(tmp);
    unsigned* gh; CK(cudaMalloc(&gh,8*256*4));
    for(int r=0;r<3;r++){ cudaEventRecord(a); hist<8><<<148*4,512>>>(k,n,gh); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("hist8 smem atomics 2^%d: %.3f ms  %.1f GB/s read, %.2f Gatom/s\n",lg,ms,n*8/ms/1e6,n*8/ms/1e6);
    for(int r=0;r<3;r++){ cudaEventRecord(a); hist<1><<<148*4,512>>>(k,n,gh); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("hist1 2^%d: %.3f ms  %.1f GB/s read\n",lg,ms,n*8/ms/1e6);
    for(int r=0;r<3;r++){ cudaEventRecord(a); matchk<<<148*4,512>>>(k,n,gh); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("match8 2^%d: %.3f ms  %.2f Gmatch/s\n",lg,ms,n*8/ms/1e6);
    for(int r=0;r<3;r++){ cudaEventRecord(a); copyk<<<148*8,256>>>((uint4*)k,(uint4*)k2,n/2); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    printf("copy 2^%d u64: %.3f ms  %.1f GB/s\n",lg,ms,2.0*n*8/ms/1e6);
    cudaFree(k); cudaFree(k2); cudaFree(gh);
  }
  size_t hb=1ull<<31; void* h; CK(cudaMallocHost(&h,hb)); void* d; CK(cudaMalloc(&d,hb));
  for(int r=0;r<3;r++){ cudaEventRecord(a); cudaMemcpyAsync(d,h,hb,cudaMemcpyHostToDevice); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
  printf("H2D pinned 2GB: %.1f GB/s\n",hb/ms/1e6);
  for(int r=0;r<3;r++){ cudaEventRecord(a); cudaMemcpyAsync(h,d,hb,cudaMemcpyDeviceToHost); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
  printf("D2H pinned 2GB: %.1f GB/s\n",hb/ms/1e6);
  return 0;
}
