// Is compute-sanitizer synccheck's "Barrier error detected. Missing init."
// on the fused kernels (profiles/r2_sanitizer.md) caused by tcgen05.alloc?
// Three minimal kernels, each checked by synccheck / racecheck:
//   plain  : __syncthreads only
//   tmem   : tcgen05.alloc / relinquish / dealloc around a __syncthreads
//   tmemio : the same plus a tcgen05.st / ld round trip of every lane
// Run: nvcc -gencode arch=compute_100a,code=sm_100a -O2 san_tmem.cu -o san_tmem &&
//      compute-sanitizer --tool synccheck ./san_tmem <mode>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (MODE > 0 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (MODE > 0) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MODE > 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v = threadIdx.x;
  if (MODE == 2 && warp < 4) {
    const uint32_t ta = slot + ((uint32_t)(32 * warp) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(ta), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(ta) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }
  if (MODE > 0) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MODE > 0 && warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(slot) : "memory");
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  uint32_t* d;
  cudaMalloc(&d, 4 * 256 * sizeof(uint32_t));
  if (mode == 0) k<0><<<4, 256>>>(d);
  else if (mode == 1) k<1><<<4, 256>>>(d);
  else k<2><<<4, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[256];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 256; ++i) bad += h[i] != (uint32_t)i;
  printf("mode %d: %s, mismatches %d\n", mode, cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
