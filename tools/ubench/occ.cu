// Occupancy probe: does a kernel's use of tcgen05 (TMEM) or its launch bounds
// limit resident CTAs per SM?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_plain(float* o) { extern __shared__ float s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); o[threadIdx.x] = s[threadIdx.x ^ 1]; }
__global__ void __launch_bounds__(512, 1) k_tmem(float* o) {
  __shared__ uint32_t slot;
  extern __shared__ float s[];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  s[threadIdx.x] = threadIdx.x; __syncthreads(); o[threadIdx.x] = s[threadIdx.x ^ 1];
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(slot) : "memory");
}
template <typename K> void probe(const char* name, K k) {
  for (int thr : {128, 256, 512}) for (int sm : {16384, 55000, 111000}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, thr, sm);
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
    printf("%s thr %d smem %d -> %d CTAs/SM (%s) regs %d\n", name, thr, sm, n, cudaGetErrorString(e), fa.numRegs);
  }
}
int main() { probe("plain", k_plain); probe("tmem", k_tmem); return 0; }
