// Microbenchmark (sm_100a): TMEM tcgen05.ld / tcgen05.st throughput per SM vs
// shared-memory LDS.128, plus a correctness probe of unaligned-column TMEM
// loads.  Decides whether the SS-CGA gather can be fed from TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(slot))), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}

#define LD16(ta, r) asm volatile( \
  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]), \
    "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(ta))
#define ST16(ta, r) asm volatile( \
  "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
  :: "r"(ta), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]), \
    "r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory")
#define WAITLD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define WAITST() asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory")

// mode 0: TMEM ld x16 (4 in flight then wait); 1: TMEM st x16; 2: LDS.128;
// 3: TMEM ld x16 with unaligned column offsets (stride 3).
__global__ void bw(int mode, int iters, unsigned* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  const int colbase = (warp >> 2) * 128;  // warps sharing a lane quadrant use disjoint columns
  unsigned acc = 0;
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
  ST16(tb + colbase, r);
  WAITST();
  const float4* s4 = reinterpret_cast<const float4*>(sm);
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0 || mode == 3) {
    const int step = mode == 0 ? 16 : 3;
    for (int it = 0; it < iters; ++it) {
      uint32_t a[16], b[16], c[16], d[16];
      const int o = (it * step) & 63;
      LD16(tb + colbase + o, a);
      LD16(tb + colbase + ((o + 16) & 63), b);
      LD16(tb + colbase + ((o + 32) & 63), c);
      LD16(tb + colbase + ((o + 48) & 63), d);
      WAITLD();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc ^= a[i] + b[i] + c[i] + d[i];
    }
  } else if (mode == 1) {
    for (int it = 0; it < iters; ++it) {
      r[it & 15] += 1;
      ST16(tb + colbase + ((it * 16) & 63), r);
      ST16(tb + colbase + ((it * 16 + 16) & 63), r);
      ST16(tb + colbase + ((it * 16 + 32) & 63), r);
      ST16(tb + colbase + ((it * 16 + 48) & 63), r);
    }
    WAITST();
  } else {
    for (int it = 0; it < iters; ++it) {
      const int base = (threadIdx.x + it * 37) & 2047;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        float4 w = s4[(base + m * 512) & 4095];
        acc ^= __float_as_uint(w.x) + __float_as_uint(w.y) + __float_as_uint(w.z) + __float_as_uint(w.w);
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (mode == 3 && blockIdx.x == 0 && warp == 0) {
    // unaligned probe: stored value at column c of lane L = tid*16 + (c - colbase) for c in [colbase, colbase+16)
    uint32_t q[16];
    LD16(tb + colbase + 5, q);  // columns 5..20 (11..15 beyond the first store are garbage, check 0..10)
    WAITLD();
    unsigned bad = 0;
    for (int i = 0; i < 11; ++i) bad += q[i] != (uint32_t)(threadIdx.x * 16 + 5 + i);
    out[gridDim.x * blockDim.x + lane] = bad;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned* out;
  long long* cyc;
  CK(cudaMalloc(&out, (size_t)(sms * 512 + 64) * 4));
  CK(cudaMalloc(&cyc, sms * 8));
  CK(cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
  const char* names[] = {"tmem ld x16 (aligned)", "tmem st x16", "smem LDS.128", "tmem ld x16 (col stride 3)"};
  for (int threads : {128, 256, 512}) {
    for (int mode = 0; mode < 4; ++mode) {
      const int iters = 4096;
      bw<<<sms, threads, 65536>>>(mode, iters, out, cyc);
      CK(cudaDeviceSynchronize());
      bw<<<sms, threads, 65536>>>(mode, iters, out, cyc);
      CK(cudaDeviceSynchronize());
      long long h[256];
      CK(cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < sms; ++i) avg += h[i];
      avg /= sms;
      // bytes per CTA: tmem modes 4 x16 per iter = 4*16*4 B per thread; smem 8 x 16 B per thread
      double bytes = (double)threads * iters * (mode == 2 ? 8 * 16 : 4 * 64);
      printf("threads %3d  %-28s  %8.1f B/clk/SM  (%.0f cycles)\n", threads, names[mode], bytes / avg, avg);
      if (mode == 3) {
        unsigned bad[32];
        CK(cudaMemcpy(bad, out + sms * threads, 128, cudaMemcpyDeviceToHost));
        unsigned s = 0;
        for (int i = 0; i < 32; ++i) s += bad[i];
        printf("    unaligned-column tcgen05.ld mismatches: %u\n", s);
      }
    }
  }
  return 0;
}
