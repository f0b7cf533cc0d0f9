// Measured CTA co-residency of tcgen05 (TMEM-allocating) kernels.
//
// cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 CTA/SM for any
// kernel containing tcgen05.alloc (occ.cu).  This probe measures what the
// hardware actually does: an oversubscribed grid (4 CTAs per SM requested)
// where every CTA allocates `cols` TMEM columns, stamps %smid and
// %globaltimer at entry and exit and spins ~50 us in between.  The maximum
// number of CTAs whose [start, end) intervals overlap on one SM is the real
// residency.  Run: nvcc -gencode arch=compute_100a,code=sm_100a -O2 resident.cu -o resident && ./resident
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

template <bool TMEM>
__global__ void probe(uint64_t* rec, int cols, int spin_ns) {
  __shared__ uint32_t slot;
  extern __shared__ float s[];
  const uint64_t t0 = gtime();
  if (TMEM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  s[threadIdx.x] = threadIdx.x;
  while (gtime() - t0 < (uint64_t)spin_ns) {
  }
  __syncthreads();
  if (TMEM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(cols) : "memory");
  const uint64_t t1 = gtime();
  if (threadIdx.x == 0) {
    rec[3 * blockIdx.x] = smid();
    rec[3 * blockIdx.x + 1] = t0;
    rec[3 * blockIdx.x + 2] = t1;
  }
}

template <bool TMEM>
void run(const char* name, int threads, int smem, int cols, int cluster) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nblk = 4 * nsm;
  uint64_t* d;
  cudaMalloc(&d, sizeof(uint64_t) * 3 * nblk);
  auto k = probe<TMEM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int occ = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, cols, 50000);
  cudaError_t e2 = cudaDeviceSynchronize();
  std::vector<uint64_t> h(3 * nblk);
  cudaMemcpy(h.data(), d, sizeof(uint64_t) * 3 * nblk, cudaMemcpyDeviceToHost);
  cudaFree(d);
  // max overlap per SM (sweep over interval end points)
  int best = 0;
  std::vector<int> per(nsm, 0);
  for (int sm = 0; sm < nsm; ++sm) {
    std::vector<std::pair<uint64_t, int>> ev;
    for (int b = 0; b < nblk; ++b)
      if ((int)h[3 * b] == sm) {
        ev.push_back({h[3 * b + 1], 1});
        ev.push_back({h[3 * b + 2], -1});
      }
    std::sort(ev.begin(), ev.end());
    int cur = 0, mx = 0;
    for (auto& p : ev) {
      cur += p.second;
      mx = std::max(mx, cur);
    }
    per[sm] = mx;
    best = std::max(best, mx);
  }
  uint64_t tmin = ~0ull, tmax = 0;
  for (int b = 0; b < nblk; ++b) {
    tmin = std::min(tmin, h[3 * b + 1]);
    tmax = std::max(tmax, h[3 * b + 2]);
  }
  int hist[9] = {0};
  for (int sm = 0; sm < nsm; ++sm) hist[std::min(per[sm], 8)]++;
  printf("%-6s threads %4d smem %6d cols %3d cluster %d | occupancy API %d | launch %s/%s | max resident/SM %d "
         "(SMs by residency 1:%d 2:%d 3:%d 4:%d) | makespan %.1f us for %d CTAs of 50 us\n",
         name, threads, smem, cols, cluster, occ, cudaGetErrorString(e), cudaGetErrorString(e2), best, hist[1],
         hist[2], hist[3], hist[4], (tmax - tmin) / 1e3, nblk);
}

int main() {
  run<false>("plain", 512, 100000, 0, 1);
  run<true>("tmem", 512, 100000, 256, 1);
  run<true>("tmem", 512, 100000, 128, 1);
  run<true>("tmem", 256, 60000, 128, 1);
  run<true>("tmem", 512, 100000, 256, 2);
  run<true>("tmem", 512, 100000, 256, 4);
  run<true>("tmem", 256, 100000, 256, 2);
  return 0;
}
