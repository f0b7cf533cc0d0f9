// Device helpers shared by the ddb kernels: complex arithmetic on interleaved
// (re, im) pairs, exact-phase twiddles, warp reductions and the thread-block
// cluster / DSMEM primitives the fused solver is built on (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ddb {

template <typename T> struct VecOf;
template <> struct VecOf<float> { using type = float2; };
template <> struct VecOf<double> { using type = double2; };
template <typename T> using Vec = typename VecOf<T>::type;

template <typename V> __device__ __forceinline__ V cmake(decltype(V::x) re, decltype(V::x) im) {
  V r; r.x = re; r.y = im; return r;
}
template <typename V> __device__ __forceinline__ V czero() { return cmake<V>(0, 0); }
template <typename V> __device__ __forceinline__ V cconj(V a) { return cmake<V>(a.x, -a.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return cmake<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc += a * b
template <typename V> __device__ __forceinline__ void cfma(V& acc, V a, V b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
template <typename V> __device__ __forceinline__ auto cabs2(V a) -> decltype(a.x) {
  return a.x * a.x + a.y * a.y;
}
template <typename V> __device__ __forceinline__ V cscale(V a, decltype(V::x) s) {
  return cmake<V>(a.x * s, a.y * s);
}
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return cmake<V>(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return cmake<V>(a.x - b.x, a.y - b.y); }

// e^{j 2 pi e / period} for an integer phase index already reduced mod period.
// Working from the reduced integer keeps the phase exact (no drift with MN),
// which is how sparse.py:118-121 defines it (2 pi / MN times an integer).
__device__ __forceinline__ float2 twiddle(float, int e, int period) {
  float s, c;
  int ee = 2 * e > period ? e - period : e;  // map to (-period/2, period/2]
  sincospif(2.0f * (float)ee / (float)period, &s, &c);
  return make_float2(c, s);
}
__device__ __forceinline__ double2 twiddle(double, int e, int period) {
  double s, c;
  int ee = 2 * e > period ? e - period : e;
  sincospi(2.0 * (double)ee / (double)period, &s, &c);
  return make_double2(c, s);
}

__device__ __forceinline__ int mod_pos(int a, int m) {
  int r = a % m;
  return r < 0 ? r + m : r;
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- thread-block cluster primitives (PTX ISA: mapa, ld.shared::cluster,
//      barrier.cluster) ----------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Map a shared::cta address of this CTA to the same offset in CTA `rank`.
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float2 ld_cluster(float2*, uint32_t caddr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_cluster(double2*, uint32_t caddr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ float ld_cluster_scalar(float*, uint32_t caddr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ double ld_cluster_scalar(double*, uint32_t caddr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(caddr) : "memory");
  return v;
}

}  // namespace ddb
