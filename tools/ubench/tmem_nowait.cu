// Probe (sm_100a): are tcgen05.ld destination registers scoreboarded by
// ptxas, i.e. is a consumer issued without tcgen05.wait::ld still ordered
// after the load's completion?  Each thread stores a distinct pattern into its
// TMEM lane, then loads it back and consumes it with no wait, rotating through
// several columns so a stale register would be caught.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD16(ta, r) asm volatile( \
  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]), \
    "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(ta))
#define ST16(ta, r) asm volatile( \
  "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
  :: "r"(ta), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]), \
    "r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory")

__global__ void __launch_bounds__(512, 1) probe(int iters, unsigned* bad, long long* cyc, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tl = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  for (int c = 0; c < 8; ++c) {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = (threadIdx.x << 12) ^ (c << 6) ^ i;
    ST16(tl + 16 * c, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  unsigned nbad = 0;
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int c0 = it & 7, c1 = (it + 3) & 7, c2 = (it + 5) & 7;
    uint32_t a[16], b[16], d[16];
    LD16(tl + 16 * c0, a);
    LD16(tl + 16 * c1, b);
    LD16(tl + 16 * c2, d);
    if (mode == 1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      nbad += a[i] != ((threadIdx.x << 12) ^ (c0 << 6) ^ i);
      nbad += b[i] != ((threadIdx.x << 12) ^ (c1 << 6) ^ i);
      nbad += d[i] != ((threadIdx.x << 12) ^ (c2 << 6) ^ i);
      acc += a[i] + b[i] + d[i];
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  atomicAdd(bad, nbad + (acc == 0x12345678u));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot) : "memory");
}

int main() {
  unsigned* bad;
  long long* cyc;
  cudaMalloc(&bad, 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(bad, 0, 4);
    probe<<<148, 512>>>(2000, bad, cyc, mode);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned h = 0;
    long long c[148];
    cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    printf("%s: mismatches %u, %.1f cycles/iter (%s)\n", mode ? "with wait::ld" : "no wait::ld  ", h, c[0] / 2000.0,
           cudaGetErrorString(e));
  }
  return 0;
}
