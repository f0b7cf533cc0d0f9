// Microbenchmark (sm_100a): cost of the synchronisation primitives one CG
// half-iteration of the fused SS-CGA kernel uses, per call, 512-thread CTAs,
// 1 CTA per SM, clusters of 1/2/4:
//   0 __syncthreads
//   1 barrier.cluster arrive.release + wait.acquire
//   2 same, arrive split from wait by a __syncthreads (the kernel's pattern)
//   3 mode 2 + a DSMEM push (st.shared::cluster) of one pair per warp before it
//   4 mode 3 + tcgen05 wait::st / fence::before / fence::after around it
//   5 barrier.cluster arrive.relaxed + wait (no release/acquire)
//   6 fence.acq_rel.cluster + relaxed arrive + wait
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rank_() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

__global__ void __launch_bounds__(512, 1) sync_kernel(int mode, int iters, long long* out) {
  __shared__ float2 slot[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t C = gridDim.x > 0 ? 0 : 0;
  uint32_t csz;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csz));
  (void)C;
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode >= 3 && mode <= 4 && lane < (int)csz) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&slot[(rank_() * 16 + warp) & 63]), ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((uint32_t)lane));
      asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" :: "r"(ra), "f"((float)it), "f"(1.f) : "memory");
    }
    if (mode == 4) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    switch (mode) {
      case 0: __syncthreads(); break;
      case 1:
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        break;
      case 5:
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
        break;
      case 6:
        asm volatile("fence.acq_rel.cluster;\nbarrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
        break;
      default:
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        __syncthreads();
        if (mode == 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        break;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long* out;
  cudaMalloc(&out, 1024 * 8);
  const char* names[] = {"syncthreads", "cluster arrive.release+wait.acquire", "split (arrive, syncthreads, wait)",
                         "split + DSMEM push", "split + push + tcgen05 fences", "cluster relaxed arrive+wait",
                         "fence.acq_rel.cluster + relaxed"};
  for (int C : {1, 2, 4}) {
    for (int mode = 0; mode < 7; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148 / C * C);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int iters = 2000;
      cudaLaunchKernelEx(&cfg, sync_kernel, mode, iters, out);
      cudaError_t e = cudaDeviceSynchronize();
      cudaLaunchKernelEx(&cfg, sync_kernel, mode, iters, out);
      e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148 / C * C; ++i) avg += h[i];
      avg /= 148 / C * C;
      printf("C=%d  %-40s %8.1f cycles/call  (%s)\n", C, names[mode], avg / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
