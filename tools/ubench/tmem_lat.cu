// Microbenchmark (sm_100a): latency-bound TMEM access patterns of the CG
// elementwise steps, 512-thread CTA, 1 CTA/SM, per warp per "step":
//   mode 0: 4 chunks x [3 x LDTM.x8 -> wait -> 8 FFMA2 -> 2 x STTM.x8]        (E = 4, as the kernel)
//   mode 1: 2 chunks x [3 x LDTM.x16 -> wait -> 16 FFMA2 -> 2 x STTM.x16]     (E = 8)
//   mode 2: 12 x LDTM.x8 issued, one wait, 32 FFMA2, 8 x STTM.x8              (all loads up front)
//   mode 3: single LDTM.x8 -> wait round trip (latency)
//   mode 4: mode 0 + tcgen05.wait::st after every chunk
// Reports cycles per step per warp (all 16 warps running the same pattern).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD8(ta, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]) : "r"(ta))
#define ST8(ta, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" \
  :: "r"(ta), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]) : "memory")
#define WAITLD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define WAITST() asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory")

template <int N> __device__ __forceinline__ void tie(uint32_t (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ void fma2(uint32_t& a0, uint32_t& a1, uint32_t b0, uint32_t b1, float s) {
  unsigned long long acc, x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "r"(a0), "r"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(b0), "r"(b1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(y) : "f"(s));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(y));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a0), "=r"(a1) : "l"(acc));
}

__global__ void __launch_bounds__(512, 1) lat_kernel(int mode, int iters, long long* out, float s) {
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
  const uint32_t tl = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 32);
  const uint32_t tA = tl, tB = tl + 128, tC = tl + 256;  // three 32-column regions per warp
  uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < 4; ++c) { ST8(tA + 8 * c, z); ST8(tB + 8 * c, z); ST8(tC + 8 * c, z); }
  WAITST();
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0 || mode == 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t a[8], b[8], d[8];
        LD8(tA + 8 * c, a); LD8(tB + 8 * c, b); LD8(tC + 8 * c, d);
        WAITLD(); tie(a); tie(b); tie(d);
#pragma unroll
        for (int i = 0; i < 4; ++i) { fma2(a[2 * i], a[2 * i + 1], b[2 * i], b[2 * i + 1], s); fma2(d[2 * i], d[2 * i + 1], b[2 * i], b[2 * i + 1], s); }
        ST8(tA + 8 * c, a); ST8(tC + 8 * c, d);
        if (mode == 4) WAITST();
      }
    } else if (mode == 1) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t a[8], b[8], d[8], a2[8], b2[8], d2[8];
        LD8(tA + 16 * c, a); LD8(tB + 16 * c, b); LD8(tC + 16 * c, d);
        LD8(tA + 16 * c + 8, a2); LD8(tB + 16 * c + 8, b2); LD8(tC + 16 * c + 8, d2);
        WAITLD(); tie(a); tie(b); tie(d); tie(a2); tie(b2); tie(d2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          fma2(a[2 * i], a[2 * i + 1], b[2 * i], b[2 * i + 1], s); fma2(d[2 * i], d[2 * i + 1], b[2 * i], b[2 * i + 1], s);
          fma2(a2[2 * i], a2[2 * i + 1], b2[2 * i], b2[2 * i + 1], s); fma2(d2[2 * i], d2[2 * i + 1], b2[2 * i], b2[2 * i + 1], s);
        }
        ST8(tA + 16 * c, a); ST8(tC + 16 * c, d); ST8(tA + 16 * c + 8, a2); ST8(tC + 16 * c + 8, d2);
      }
    } else if (mode == 2) {
      uint32_t a[4][8], b[4][8], d[4][8];
#pragma unroll
      for (int c = 0; c < 4; ++c) { LD8(tA + 8 * c, a[c]); LD8(tB + 8 * c, b[c]); LD8(tC + 8 * c, d[c]); }
      WAITLD();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tie(a[c]); tie(b[c]); tie(d[c]);
#pragma unroll
        for (int i = 0; i < 4; ++i) { fma2(a[c][2 * i], a[c][2 * i + 1], b[c][2 * i], b[c][2 * i + 1], s); fma2(d[c][2 * i], d[c][2 * i + 1], b[c][2 * i], b[c][2 * i + 1], s); }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) { ST8(tA + 8 * c, a[c]); ST8(tC + 8 * c, d[c]); }
    } else {
      uint32_t a[8];
      LD8(tA + (it & 3) * 8, a);
      WAITLD(); tie(a);
      if (a[0] == 12345u) out[1000] = a[1];
    }
  }
  WAITST();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot) : "memory");
}

int main() {
  long long* out;
  cudaMalloc(&out, 2048 * 8);
  const char* names[] = {"E=4 chunks (kernel pattern)", "E=8 chunks", "all loads up front", "single LDTM.x8 round trip",
                         "E=4 + wait::st per chunk"};
  for (int thr : {32, 128, 512}) for (int mode = 0; mode < 5; ++mode) {
    const int iters = 1000;
    lat_kernel<<<148, thr>>>(mode, iters, out, 1.0001f);
    cudaDeviceSynchronize();
    lat_kernel<<<148, thr>>>(mode, iters, out, 1.0001f);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("threads %3d  %-32s %8.1f cycles/step (%s)\n", thr, names[mode], avg / 148 / iters, cudaGetErrorString(e));
  }
  return 0;
}
