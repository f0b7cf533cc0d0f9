// Device pieces shared by the fused SS-CGA kernels (sscga.cu: row-major
// on-chip slices; sscga_tm.cu: TMEM-resident operands): the per-frame tap
// entry, FFMA2 gather runs, split cluster barriers, deterministic cluster-wide
// reductions, packed CG vector arithmetic and the clock64 phase timer.
#pragma once

#include "common.cuh"
#include "internal.h"

namespace ddb {
// Per-frame tap entry: offsets and both direction's row-invariant gain factor,
// hf = h W_MN^{-d_l d_k} (forward) and hh = conj(h) (hermitian), so a thread
// only adds its own row's W_MN^{-+d_l k} (skipped when d_l == 0).  off is the
// tap's shift in the row-major on-chip slices, d_k RS + d_l elements: the
// forward gather of row k reads thread_base + off, the hermitian one - off.
template <typename T> struct PathEnt;
template <> struct __align__(16) PathEnt<double> {
  int dk, dl, off, pad;
  double2 hf, hh;
  __device__ double2 coef(bool herm) const { return herm ? hh : hf; }
};
// fp32: gains stored as FFMA2-ready quads (g.x, g.x, -g.y, g.y), so a 128-bit
// load yields the register pairs of both packed MACs directly.
template <> struct __align__(16) PathEnt<float> {
  int dk, dl, off, pad;
  float4 hf, hh;
  __device__ float2 coef(bool herm) const {
    const float4 q = herm ? hh : hf;
    return make_float2(q.x, q.w);
  }
};
__device__ __forceinline__ float4 quad(float2 g) { return make_float4(g.x, g.x, -g.y, g.y); }
__device__ __forceinline__ double2 quad(double2 g) { return g; }


// (x mod m) for x in (-m, 2m)
__device__ __forceinline__ int wrap1(int x, int m) {
  x = x < 0 ? x + m : x;
  return x >= m ? x - m : x;
}


// Contiguous run of LC source columns starting at rp (16-byte aligned row,
// offset `odd` elements): 128-bit loads, two complex values each; an odd start
// loads one extra aligned chunk and uses the other halves (register naming only).
// acc += c v with c given as the FFMA2 operand pairs X = (c.x, c.x), Y = (-c.y, c.y)
__device__ __forceinline__ void cmacxy(unsigned long long& acc, unsigned long long X, unsigned long long Y,
                                       float a, float b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(X), "l"(pack2(a, b)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(Y), "l"(pack2(b, a)));
}
template <int LC>
__device__ __forceinline__ void gather_run(const float2* rp, bool odd, unsigned long long X, unsigned long long Y,
                                           unsigned long long (&acc)[LC]) {
  if constexpr (LC == 1) {
    const float2 v = rp[0];
    cmacxy(acc[0], X, Y, v.x, v.y);
  } else {
    if (!odd) {
      const float4* q = reinterpret_cast<const float4*>(rp);
#pragma unroll
      for (int m = 0; m < LC / 2; ++m) {
        const float4 w = q[m];
        cmacxy(acc[2 * m], X, Y, w.x, w.y);
        cmacxy(acc[2 * m + 1], X, Y, w.z, w.w);
      }
    } else {
      const float4* q = reinterpret_cast<const float4*>(rp - 1);
      float4 w = q[0];
      cmacxy(acc[0], X, Y, w.z, w.w);
#pragma unroll
      for (int m = 1; m < LC / 2; ++m) {
        w = q[m];
        cmacxy(acc[2 * m - 1], X, Y, w.x, w.y);
        cmacxy(acc[2 * m], X, Y, w.z, w.w);
      }
      w = q[LC / 2];
      cmacxy(acc[LC - 1], X, Y, w.x, w.y);
    }
  }
}
template <int LC>
__device__ __forceinline__ void gather_run(const double2* rp, bool, double2 c, double2 (&acc)[LC]) {
#pragma unroll
  for (int j = 0; j < LC; ++j) Acc<double>::mac(acc[j], c, rp[j]);
}


template <typename T>
__device__ __forceinline__ void cl_sync(int C) {
  if (C > 1) cluster_sync_all();
  else __syncthreads();
}

// Reduction buffers: [2 kinds][2 parities][kPushSlots] pairs.  red_read sums
// `total` per-warp pairs of slot in a fixed order (the one-CTA case of the
// two-level reduction below, and the pull of peers' pairs for large clusters).
constexpr int kPushSlots = 64;

// Cluster-wide total (after the cluster barrier's wait); identical in every warp.
template <typename T>
__device__ __forceinline__ Vec<T> red_read(const Vec<T>* slot, int C, int nwarps, int lane) {
  using V = Vec<T>;
  const int total = C * nwarps;
  V s = czero<V>();
  if (total <= kPushSlots) {
    // every lane sums all the cluster's per-warp pairs from local shared memory
    // (broadcast loads, four fixed-order partial sums): no shuffles on the
    // critical path, bit-identical result everywhere
    V q0 = czero<V>(), q1 = czero<V>(), q2 = czero<V>(), q3 = czero<V>();
    if constexpr (sizeof(T) == 4) {
      const float4* s4 = reinterpret_cast<const float4*>(slot);
      const int n4 = total / 2;
      int i = 0;
      for (; i + 1 < n4; i += 2) {
        const float4 w = s4[i], z = s4[i + 1];
        q0 = cadd(q0, make_float2(w.x, w.y));
        q1 = cadd(q1, make_float2(w.z, w.w));
        q2 = cadd(q2, make_float2(z.x, z.y));
        q3 = cadd(q3, make_float2(z.z, z.w));
      }
      if (i < n4) {
        const float4 w = s4[i];
        q0 = cadd(q0, make_float2(w.x, w.y));
        q1 = cadd(q1, make_float2(w.z, w.w));
      }
      if (total & 1) q2 = cadd(q2, slot[total - 1]);
    } else {
      int i = 0;
      for (; i + 1 < total; i += 2) {
        q0 = cadd(q0, slot[i]);
        q1 = cadd(q1, slot[i + 1]);
      }
      if (i < total) q2 = cadd(q2, slot[i]);
    }
    return cadd(cadd(q0, q1), cadd(q2, q3));
  } else {
    // pull mode: lane i starts at cluster slot i = (rank, warp)
    const int r0 = lane < total ? lane / nwarps : C;
    const int w0 = lane < total ? lane - (lane / nwarps) * nwarps : 0;
    const uint32_t base = smem_addr(slot);
    for (int r = r0, w = w0; r < C;) {
      s = cadd(s, ld_cluster(static_cast<V*>(nullptr), map_rank(base + w * (int)sizeof(V), r)));
      w += 32;
      while (w >= nwarps) { w -= nwarps; ++r; }
    }
  }
  s.x = warp_sum(s.x);
  s.y = warp_sum(s.y);
  return s;
}

// Two-level deterministic cluster reduction of a pair (e.g. ||u||^2, ||p||^2).
// base = this reduction's buffer (kind, parity): base[0 .. 32) per-warp
// partials of this CTA, base[32 + r] CTA r's total.
//   red_stage       (before the barrier)  every warp publishes its partial;
//   cl_arrive_red   (the barrier's arrive half) after the CTA barrier one warp
//                   (fold_warp) folds the CTA's partials with a fixed xor-tree
//                   (bit-identical in every lane) and pushes the total to every
//                   CTA of the cluster, then its cluster arrive releases it --
//                   and, being after the CTA barrier, every warp's shared-memory
//                   writes with it; the other warps arrive relaxed
//                   (cluster-scope fences are the most expensive part of a
//                   cluster barrier).  `relaxed` is kept for the callers' sake;
//   red_total       (after the wait) the C totals summed in rank order, so every
//                   warp of every CTA holds the same bits and takes the same branch.
// One CTA (C == 1) reads the per-warp partials directly instead.
// The warp that folds the CTA's partials and pushes the total: one of a
// middle row block when there are several (the first and last row blocks of a
// TMEM segment carry most shared-memory taps, so they arrive last): cfg3
// 17.06 -> 17.55 G symbols/s with warp 8 (profiles/r2_experiments.md).
__device__ __forceinline__ int fold_warp(int nwarps) { return nwarps >= 12 ? 8 : (nwarps >= 8 ? 4 : 0); }

template <typename T>
__device__ __forceinline__ void red_stage(Vec<T> part, Vec<T>* base, int warp, int lane) {
  part.x = warp_sum(part.x);
  part.y = warp_sum(part.y);
  if (lane == 0) base[warp] = part;
}
__device__ __forceinline__ void cl_arrive_sem(bool release) {
  if (release) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  else asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
template <typename T, bool TMEM_FENCES>
__device__ __forceinline__ void cl_arrive_red(int C, Vec<T>* base, int nwarps, int warp, int lane, int rank,
                                              bool relaxed, int fold = -1) {
  if constexpr (TMEM_FENCES) {
    tmem_wait_st();
    tmem_fence_before();
  }
  __syncthreads();
  if (C > 1) {
    const int fw = fold >= 0 ? fold : TMEM_FENCES ? fold_warp(nwarps) : 0;  // (the row-slice kernel: warp 0 measured best)
    if (warp == fw) {
      Vec<T> t = lane < nwarps ? base[lane] : czero<Vec<T>>();
      t.x = warp_sum(t.x);
      t.y = warp_sum(t.y);
      if (lane < C) st_cluster(map_rank(smem_addr(base + 32 + rank), (uint32_t)lane), t);
    }
    // the CTA barrier above orders every warp's shared-memory writes before the
    // folding warp's cluster-scope release (cumulative), so one release serves
    // the DSMEM readers of frames with Doppler taps too; every other warp
    // arrives relaxed (cfg3det 8.5 -> 9.0 G symbols/s; the release fences of
    // all warps were 8 % of its stall samples)
    (void)relaxed;
    cl_arrive_sem(warp == fw);
  }
  if constexpr (TMEM_FENCES) tmem_fence_after();
}
template <typename T>
__device__ __forceinline__ Vec<T> red_total(int C, const Vec<T>* base, int nwarps) {
  if (C == 1) return red_read<T>(base, 1, nwarps, 0);
  Vec<T> t = base[32];
  for (int r = 1; r < C; ++r) t = cadd(t, base[32 + r]);
  return t;
}

// Split cluster barrier: arrive (release) -> CTA barrier -> ... -> wait (acquire).
__device__ __forceinline__ void cl_arrive(int C) {
  if (C > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
}
__device__ __forceinline__ void cl_wait(int C) {
  if (C > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---- packed elementwise CG arithmetic (FFMA2 for fp32)
// y + a x (a real, broadcast)
__device__ __forceinline__ float2 axpy(float2 y, float a, float2 x) {
  unsigned long long r = pack2(y.x, y.y);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(pack2(a, a)), "l"(pack2(x.x, x.y)));
  return unpack2(r);
}
__device__ __forceinline__ double2 axpy(double2 y, double a, double2 x) {
  return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}
// n += (v.x^2, v.y^2); the norm is n.x + n.y
__device__ __forceinline__ void nacc(float2& n, float2 v) {
  unsigned long long r = pack2(n.x, n.y);
  const unsigned long long p = pack2(v.x, v.y);
  asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r) : "l"(p));
  n = unpack2(r);
}
__device__ __forceinline__ void nacc(double2& n, double2 v) {
  n.x = fma(v.x, v.x, n.x);
  n.y = fma(v.y, v.y, n.y);
}


// Phase timer (measurement builds of a launch only: SolveArgs::prof != null):
// thread 0 of each CTA attributes clock64 intervals to the phase being run.
enum Phase { kSetup, kArrive, kMvmLocal, kWait, kMvmRemote, kRead, kStep1, kStep3, kEpilogue, kTail };
struct ProfSm {
  long long acc[kProfPhases];
  long long t;
  int cur, pad;
};
// Attribute the cycles since the last mark to the running phase and switch to
// `next`.  State lives in shared memory, so production launches (prof null)
// carry no registers for it.
__device__ __forceinline__ void prof_mark(const long long* prof, ProfSm* ps, int next) {
  if (prof != nullptr && threadIdx.x == 0) {
    const long long now = clock64();
    ps->acc[ps->cur] += now - ps->t;
    ps->t = now;
    ps->cur = next;
  }
}
__device__ __forceinline__ void prof_init(const long long* prof, ProfSm* ps) {
  if (prof != nullptr && threadIdx.x == 0) {
    for (int i = 0; i < kProfPhases; ++i) ps->acc[i] = 0;
    ps->cur = kTail;
    ps->t = clock64();
  }
}
__device__ __forceinline__ void prof_store(long long* prof, const ProfSm* ps) {
  if (prof != nullptr && threadIdx.x == 0)
    for (int i = 0; i < kProfPhases; ++i) prof[(size_t)blockIdx.x * kProfPhases + i] = ps->acc[i];
}


}  // namespace ddb
