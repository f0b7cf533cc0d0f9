// Microbenchmark (sm_100a): shared-memory read throughput per SM by route,
// with the access pattern of the Doppler-tap runs (tap_elem): every thread
// reads a 16-row run (eight 16-byte words) of an extended column, lanes spread
// over columns of stride CS rows.  One 512-thread CTA per SM, clusters of 2,
// the whole GPU busy.
//   mode 0: LDS.128 (own CTA, shared::cta address)
//   mode 1: ld.shared::cluster.v4 at this CTA's own rank (mapa to self)
//   mode 2: ld.shared::cluster.v4 at the peer CTA
//   mode 3: per lane: even lanes LDS from own, odd lanes DSMEM from the peer
//   mode 4: generic LD through a generic pointer to own shared memory
//   mode 5: ld.shared::cluster.v4 at the peer, coalesced (lane i at +16 i: 512 B per warp)
//   mode 6: ld.shared::cluster.v2 at the peer (8-byte words, the kernel's pattern)
//   mode 7: st.shared::cluster.v4 to the peer (push), the kernel's pattern
//   mode 8: st.shared::cluster.v4 to the peer, coalesced
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kCS = 874;    // column stride in complex values (cfg3's extended column)
constexpr int kCols = 16;   // columns per CTA
constexpr int kSmem = kCols * kCS * 8 + 64;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t map_rank(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ float4 ldc4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) bw(int mode, int iters, float* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* col = reinterpret_cast<float2*>(sm + 16);
  for (int i = threadIdx.x; i < kCols * kCS; i += blockDim.x) col[i] = make_float2(i * 1e-3f, 1.f);
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ln = (warp & 3) * 32 + lane;           // TMEM-lane-like index
  const int c = ln % kCols, seg = ln / kCols;       // lanes spread over columns (the kernel's layout)
  const int row0 = 64 + seg * 64 + (warp >> 2) * 16;
  const unsigned rank = cluster_rank(), peer = rank ^ 1u;
  const uint32_t own = smem_addr(col + c * kCS + row0);
  const uint32_t self_c = map_rank(own, rank), peer_c = map_rank(own, peer);
  const uint32_t peer_co = map_rank(smem_addr(sm + 16 + (warp * 32 + lane) * 16), peer);  // coalesced
  const float4* gen = reinterpret_cast<const float4*>(col + c * kCS + row0);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t off = (uint32_t)((it * 5) & 31) * 16u;  // move the run a little
    float4 w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t o = off + 16u * k;
      if (mode == 0) w[k] = lds4(own + o);
      else if (mode == 1) w[k] = ldc4(self_c + o);
      else if (mode == 2) w[k] = ldc4(peer_c + o);
      else if (mode == 3) w[k] = (lane & 1) ? ldc4(peer_c + o) : lds4(own + o);
      else if (mode == 4) w[k] = gen[(off >> 4) + k];
      else if (mode == 5) w[k] = ldc4(peer_co + 512u * k + (uint32_t)(it & 7) * 4096u);
      else if (mode == 6) {
        float2 a, b;
        asm volatile("ld.shared::cluster.v2.f32 {%0,%1}, [%2];" : "=f"(a.x), "=f"(a.y) : "r"(peer_c + o) : "memory");
        asm volatile("ld.shared::cluster.v2.f32 {%0,%1}, [%2];" : "=f"(b.x), "=f"(b.y) : "r"(peer_c + o + 8u) : "memory");
        w[k] = make_float4(a.x, a.y, b.x, b.y);
      } else {
        const uint32_t d = mode == 7 ? peer_c + o : peer_co + 512u * k + (uint32_t)(it & 7) * 4096u;
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(d), "f"(acc.x), "f"(acc.y), "f"(acc.z), "f"(acc.w) : "memory");
        w[k] = make_float4(1.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc.x += w[k].x; acc.y += w[k].y; acc.z += w[k].z; acc.w += w[k].w; }
  }
  const long long t1 = clock64();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  const int grid = (nsm / 2) * 2, iters = 4096;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&cyc, grid * sizeof(long long)));
  long long* h = new long long[grid];
  const char* names[] = {"LDS.128 own", "ld.shared::cluster own rank", "ld.shared::cluster peer", "half lanes LDS own, half DSMEM peer", "generic LD own",
                         "ld.shared::cluster peer coalesced", "ld.shared::cluster.v2 peer", "st.shared::cluster peer", "st.shared::cluster peer coalesced"};
  for (int mode = 0; mode < 9; ++mode) {
    bw<<<grid, 512, kSmem>>>(mode, 64, out, cyc);  // warm-up
    CK(cudaDeviceSynchronize());
    bw<<<grid, 512, kSmem>>>(mode, iters, out, cyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
    const double bytes = 512.0 * iters * 8 * 16;  // per CTA
    printf("mode %d %-40s %8.1f cycles/iter  %6.1f B/clk/SM\n", mode, names[mode], mean / iters, bytes / mean);
  }
  return 0;
}
