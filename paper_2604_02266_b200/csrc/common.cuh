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

// |re + j im| exactly as numpy evaluates np.abs on complex arrays (its SIMD
// loop: larger * sqrt(fma(r, r, 1)), r = smaller / larger), so decisions that
// hinge on last-ulp distance ties (hard_demod's argmin, detect_paths'
// threshold and ordering) come out bit-identical to the reference.
__device__ __forceinline__ double np_cabs(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double big = fmax(a, b), small = fmin(a, b);
  if (big == 0.0 || isinf(big)) return big;
  const double r = __ddiv_rn(small, big);
  return __dmul_rn(big, __dsqrt_rn(__fma_rn(r, r, 1.0)));
}
__device__ __forceinline__ float np_cabs(float re, float im) {
  const float a = fabsf(re), b = fabsf(im);
  const float big = fmaxf(a, b), small = fminf(a, b);
  if (big == 0.f || isinf(big)) return big;
  const float r = __fdiv_rn(small, big);
  return __fmul_rn(big, __fsqrt_rn(__fmaf_rn(r, r, 1.f)));
}

// Transmitted label of symbol q: one byte per symbol, or bps bits per symbol
// packed LSB-first within bytes (bps 2 or 4, so a symbol never straddles bytes).
__device__ __forceinline__ unsigned tx_label_at(const uint8_t* txl, size_t q, int bps, int packed) {
  if (!packed) return txl[q];
  const size_t bit = q * (size_t)bps;
  return (txl[bit >> 3] >> (bit & 7)) & ((1u << bps) - 1u);
}
__device__ __forceinline__ const uint8_t* tx_label_ptr(const uint8_t* txl, size_t q, int bps, int packed) {
  return txl + (packed ? (q * (size_t)bps >> 3) : q);
}

// ---- packed complex MAC on sm_100 FFMA2: acc (re, im) += c * v as two
//      fma.rn.f32x2; ptxas folds the broadcast of c.re / c.im and the swapped,
//      partially negated v into the FFMA2 operand modifiers.
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ void cmac2(unsigned long long& acc, float cr, float ci, float2 v) {
  const unsigned long long V = pack2(v.x, v.y), S = pack2(v.y, v.x);
  const unsigned long long X = pack2(cr, cr), Y = pack2(-ci, ci);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(X), "l"(V));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(Y), "l"(S));
}

// Accumulator abstraction: packed u64 for fp32 (FFMA2), double2 for fp64.
template <typename T> struct Acc;
template <> struct Acc<float> {
  using type = unsigned long long;
  __device__ static __forceinline__ type zero() { return 0ull; }
  __device__ static __forceinline__ void mac(type& a, float2 c, float2 v) { cmac2(a, c.x, c.y, v); }
  __device__ static __forceinline__ float2 get(type a) { return unpack2(a); }
};
template <> struct Acc<double> {
  using type = double2;
  __device__ static __forceinline__ type zero() { return make_double2(0.0, 0.0); }
  __device__ static __forceinline__ void mac(type& a, double2 c, double2 v) {
    a.x = fma(c.x, v.x, a.x);
    a.x = fma(-c.y, v.y, a.x);
    a.y = fma(c.x, v.y, a.y);
    a.y = fma(c.y, v.x, a.y);
  }
  __device__ static __forceinline__ double2 get(type a) { return a; }
};

__device__ __forceinline__ int mod_pos(int a, int m) {
  int r = a % m;
  return r < 0 ? r + m : r;
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- tensor memory (TMEM, sm_100): per-CTA 128 lanes x 512 columns x 32 bit.
// Used here as the home of the CG solution vector x: thread t of warp w owns
// lane 32 (w % 4) + (t % 32) and a private run of columns, so every access is
// lane-local (tcgen05.ld/st .32x32b) and needs no cross-thread ordering.
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(slot))), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int NR> __device__ __forceinline__ void tmem_ld(uint32_t ta, uint32_t (&r)[NR]);
template <int NR> __device__ __forceinline__ void tmem_st(uint32_t ta, const uint32_t (&r)[NR]);
template <> __device__ __forceinline__ void tmem_ld<2>(uint32_t ta, uint32_t (&r)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(ta));
}
template <> __device__ __forceinline__ void tmem_ld<4>(uint32_t ta, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
}
template <> __device__ __forceinline__ void tmem_ld<8>(uint32_t ta, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
}
template <> __device__ __forceinline__ void tmem_ld<16>(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
}
template <> __device__ __forceinline__ void tmem_ld<32>(uint32_t ta, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
}
// tcgen05.wait::ld.  ptxas tracks tcgen05.ld destinations on a scoreboard
// (the wait compiles to a scoreboard wait), so consumers of the loaded
// registers are ordered after it; the register array only documents which
// load the wait is for.
template <int W> __device__ __forceinline__ void tmem_wait_ld_tie(uint32_t (&)[W]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <> __device__ __forceinline__ void tmem_st<2>(uint32_t ta, const uint32_t (&r)[2]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" :: "r"(ta), "r"(r[0]), "r"(r[1]) : "memory");
}
template <> __device__ __forceinline__ void tmem_st<4>(uint32_t ta, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
               :: "r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
template <> __device__ __forceinline__ void tmem_st<8>(uint32_t ta, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
template <> __device__ __forceinline__ void tmem_st<16>(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};"
      :: "r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
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

// ---- mbarrier + 1-D bulk copies (TMA engine, cp.async.bulk): a global ->
// shared copy completes on an mbarrier with a transaction count.
__device__ __forceinline__ void mbar_init(void* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(void* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(smem_addr(mb)), "r"(parity) : "memory");
}
// the same with cluster-scope acquire (an mbarrier that other CTAs arrive on)
__device__ __forceinline__ void mbar_wait_cluster(void* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(smem_addr(mb)), "r"(parity) : "memory");
}
// arrive on another CTA's mbarrier (cluster address), releasing this CTA's prior accesses
__device__ __forceinline__ void mbar_arrive_remote(uint32_t mb) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mb) : "memory");
}
// generic-proxy accesses of shared memory before, async-proxy (bulk copy) after
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, void* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(mb)) : "memory");
}
// Push `bytes` of this CTA's shared memory to a cluster address (another CTA's
// shared memory) with the bulk-copy engine, completing on that CTA's mbarrier.
__device__ __forceinline__ void bulk_s2c(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "r"(smem_addr(src)), "r"(bytes), "r"(mb) : "memory");
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
__device__ __forceinline__ float4 ld_cluster4(uint32_t caddr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_cluster(double2*, uint32_t caddr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster(uint32_t caddr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" :: "r"(caddr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t caddr, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" :: "r"(caddr), "d"(v.x), "d"(v.y) : "memory");
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
