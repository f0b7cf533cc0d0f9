// Fused SS-CGA solve: matrix-free structured-sparse operator + fixed-Xi
// conjugate gradient + demod epilogue, one thread-block cluster per frame.
//
// Reference algorithm: equalize.py:43-77 (cga_equalize) on the operator of
// sparse.py:91-160.  Nothing of H_dd is stored: for tap p (k_p, l_p, h_p) with
// offsets d_k = K0 - k_p, d_l = L0 - l_p (sparse.py:35-37) the forward product
// is, for output (k, l),
//     a = k + d_k,  n = floor(a / M),  k_s = a - n M
//     u[k, l] += h_p W_MN^{-d_l k_s} W_N^{n l} v[k_s, (l + d_l) mod N]
// and the Hermitian product is, with a = k - d_k, n = floor(a / M), k_s = a - n M,
//     u[k, l] += conj(h_p) W_MN^{d_l (k - n M)} W_N^{n l} v[k_s, (l - d_l) mod N]
// (W_X^e = exp(j 2 pi e / X); both are the closed forms of the tables built by
// sparse.py:124-144, checked entry-by-entry in tests/test_oracle.py).  The
// coefficient of a (tap, delay row) pair is the same for every Doppler column
// except for the quasi-periodic wrap twist W_N^{n l}, which only rows whose
// source wraps across the delay period see.
//
// Layout: frame q = l M + k (grid.py:86-95).  The cluster's CTA r owns the
// Doppler columns [r Lcta, (r+1) Lcta); inside it thread (k, g) owns delay row
// k of the LC columns g LC .. g LC + LC - 1.  Shared memory holds this CTA's
// slice of p (gathered by H), u = H p (gathered by H^H) and x; the residual c
// and the MVM accumulators live in registers.  Gathers whose source column is
// owned by another CTA of the cluster read it through DSMEM
// (ld.shared::cluster), so no halo copies are needed.
//
// CG step, per iteration (equalize.py:59-76):
//   u = H p;             ||u||^2 reduced cluster-wide          (barrier B)
//   denom = ||u||^2 + lam ||p||^2  (= Re p^H (H^H H + lam I) p, equalize.py:60-64,
//   evaluated from the forward product so it needs no extra barrier)
//   denom == 0 -> exact convergence (equalize.py:64-67)
//   ap = H^H u + lam p;  x += alpha p;  c -= alpha ap;  ||c||^2  (barrier C)
//   p = c + beta p;      ||p||^2                              (barrier A)
// Reductions are deterministic: every warp of every CTA sums the same
// per-warp partials in the same order, so all CTAs take identical branches.
#include "common.cuh"
#include "demod.cuh"
#include "internal.h"

namespace ddb {

struct Ctx {
  int k;        // delay row owned by this thread
  int g;        // column group inside the CTA
  int rank;     // CTA rank in the cluster
  int colbase;  // global Doppler column of this thread's first column
  bool active;  // padding threads (M * G not a multiple of 32) compute but never store
};

// acc[j] = (H v)[k, colbase + j]  (HERM = false)  or  (H^H v)[k, colbase + j]
template <typename T, int LC, bool HERM>
__device__ __forceinline__ void ss_mvm_cluster(const SolveArgs& a, const Ctx& cx, int P0, int P,
                                               const Vec<T>* __restrict__ buf,
                                               const Vec<T>* __restrict__ tw, Vec<T> (&acc)[LC]) {
  using V = Vec<T>;
  const int M = a.M, N = a.N, MN = a.MN, Lcta = a.Lcta;
  const V* gains = reinterpret_cast<const V*>(a.ph);
#pragma unroll
  for (int j = 0; j < LC; ++j) acc[j] = czero<V>();
  const uint32_t buf_s = smem_addr(buf);
  const int first_col = cx.rank * Lcta;
  for (int p = 0; p < P; ++p) {
    const int kp = __ldg(a.pk + P0 + p);
    const int lp = __ldg(a.pl + P0 + p);
    V h = __ldg(gains + P0 + p);
    const int dk = a.K0 - kp, dl = a.L0 - lp;
    const int ar = HERM ? cx.k - dk : cx.k + dk;
    const int n = ar < 0 ? -1 : (ar >= M ? 1 : 0);
    const int ks = ar - n * M;
    int e;
    if (HERM) {
      e = mod_pos(dl * (cx.k - n * M), MN);
      h = cconj(h);
    } else {
      e = mod_pos(-dl * ks, MN);
    }
    const V coef = cmul(h, twiddle(T(0), e, MN));
    const int base = mod_pos(cx.colbase + (HERM ? -dl : dl), N);
    const int loc0 = base - first_col;
    const bool fast = (n == 0) && loc0 >= 0 && loc0 + LC <= Lcta;
    if (__all_sync(0xffffffffu, fast)) {
      // every column local and contiguous, no wrap twist: pure gather-FMA
      const V* s = buf + loc0 * M + ks;
#pragma unroll
      for (int j = 0; j < LC; ++j) cfma(acc[j], coef, s[j * M]);
    } else {
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        int ls = base + j;
        if (ls >= N) ls -= N;
        const int owner = ls / Lcta;
        const int lloc = ls - owner * Lcta;
        V v;
        if (owner == cx.rank) {
          v = buf[lloc * M + ks];
        } else {
          v = ld_cluster(static_cast<V*>(nullptr),
                         map_rank(buf_s + (uint32_t)((lloc * M + ks) * (int)sizeof(V)), owner));
        }
        V cj = coef;
        if (n != 0) {
          V t = tw[cx.colbase + j];
          if (n < 0) t = cconj(t);
          cj = cmul(coef, t);
        }
        cfma(acc[j], cj, v);
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ void cl_sync(int C) {
  if (C > 1) cluster_sync_all();
  else __syncthreads();
}

// Deterministic cluster-wide sum.  slot: this CTA's [32] partial array for the
// reduction kind / parity in use.  Contains the barrier.
template <typename T>
__device__ __forceinline__ T cluster_sum(T part, T* slot, int C, int nwarps, int lane, int warp) {
  T v = warp_sum(part);
  if (lane == 0) slot[warp] = v;
  cl_sync<T>(C);
  const int total = C * nwarps;
  const uint32_t base = smem_addr(slot);
  T s = T(0);
  for (int i = lane; i < total; i += 32) {
    const int r = i / nwarps, w = i - r * nwarps;
    s += (C > 1) ? ld_cluster_scalar(static_cast<T*>(nullptr), map_rank(base + w * (int)sizeof(T), r))
                 : slot[w];
  }
  return warp_sum(s);
}

template <typename T, int LC>
__global__ void __launch_bounds__(sscga_max_threads(sizeof(T), LC), 1) sscga_kernel(const SolveArgs a) {
  using V = Vec<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = a.M;
  const int nelem = a.Lcta * M;
  V* pbuf = reinterpret_cast<V*>(smem);
  V* ubuf = pbuf + nelem;
  V* xbuf = ubuf + nelem;
  T* red = reinterpret_cast<T*>(xbuf + nelem);  // [3 kinds][2 parities][32 warps]
  V* tw = reinterpret_cast<V*>(red + 3 * 2 * 32);  // W_N^l, l in [0, N)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  Ctx cx;
  cx.rank = a.C > 1 ? (int)cluster_rank() : 0;
  cx.active = tid < a.active_threads;
  const int t = cx.active ? tid : 0;
  cx.k = t % M;
  cx.g = t / M;
  cx.colbase = cx.rank * a.Lcta + cx.g * LC;

  for (int l = tid; l < a.N; l += blockDim.x) tw[l] = twiddle(T(0), l, a.N);
  __syncthreads();

  const V* y = reinterpret_cast<const V*>(a.y);
  V* xo = reinterpret_cast<V*>(a.x);
  T* cnorm = reinterpret_cast<T*>(a.cnorm);
  V* snaps = reinterpret_cast<V*>(a.snaps);
  const T* lamv = reinterpret_cast<const T*>(a.lam);
  const T* nvar = reinterpret_cast<const T*>(a.nvar);
  const bool lead = (cx.rank == 0 && tid == 0);
  const int stride = a.iters + 1;
  int par[3] = {0, 0, 0};  // 0: ||p||^2, 1: ||u||^2, 2: ||c||^2

  for (int f = blockIdx.x / a.C; f < a.B; f += a.n_clusters) {
    const int P0 = __ldg(a.off + f);
    const int P = __ldg(a.off + f + 1) - P0;
    const size_t fo = (size_t)f * a.MN;

    if (P <= 0) {  // EmptyChannel (sparse.py:126-127): flag it, no NaNs
      if (cx.active) {
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const size_t q = fo + (size_t)(cx.colbase + j) * M + cx.k;
          xo[q] = czero<V>();
          if (a.labels) a.labels[q] = 0;
          if (a.llr)
            for (int b = 0; b < a.bps; ++b) a.llr[q * a.bps + b] = 0.f;
        }
      }
      if (lead) {
        if (cnorm) for (int i = 0; i < stride; ++i) cnorm[(size_t)f * stride + i] = T(0);
        if (a.itdone) a.itdone[f] = 0;
        if (a.status) a.status[f] = 1;
        if (a.berr) a.berr[f] = a.bps * a.MN / 2;  // harness.py:173 scoring of a failed packet
      }
      continue;
    }
    const T lam = lamv[f];

    // y -> ubuf (own columns); b = H^H y is gathered from it
    if (cx.active) {
#pragma unroll
      for (int j = 0; j < LC; ++j)
        ubuf[(cx.g * LC + j) * M + cx.k] = y[fo + (size_t)(cx.colbase + j) * M + cx.k];
    }
    if (lead && a.berr) a.berr[f] = 0;
    cl_sync<T>(a.C);

    V acc[LC], c[LC];
    ss_mvm_cluster<T, LC, true>(a, cx, P0, P, ubuf, tw, acc);  // b = H^H y (equalize.py:52)
    T part = T(0);
#pragma unroll
    for (int j = 0; j < LC; ++j) {
      c[j] = acc[j];
      if (cx.active) {
        const int o = (cx.g * LC + j) * M + cx.k;
        pbuf[o] = acc[j];
        xbuf[o] = czero<V>();
        part += cabs2(acc[j]);
      }
    }
    T cn = cluster_sum<T>(part, red + (0 * 2 + par[0]) * 32, a.C, nwarps, lane, warp);
    par[0] ^= 1;
    T pp = cn;
    if (lead && cnorm) cnorm[(size_t)f * stride] = cn;

    int done = 0;
    bool exact = false;
    for (int it = 0; it < a.iters; ++it) {
      ss_mvm_cluster<T, LC, false>(a, cx, P0, P, pbuf, tw, acc);  // u = H p
      part = T(0);
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        if (cx.active) {
          ubuf[(cx.g * LC + j) * M + cx.k] = acc[j];
          part += cabs2(acc[j]);
        }
      }
      const T uu = cluster_sum<T>(part, red + (1 * 2 + par[1]) * 32, a.C, nwarps, lane, warp);
      par[1] ^= 1;
      const T denom = uu + lam * pp;
      if (denom == T(0)) {  // equalize.py:64-67
        exact = true;
        break;
      }
      const T alpha = cn / denom;
      ss_mvm_cluster<T, LC, true>(a, cx, P0, P, ubuf, tw, acc);  // H^H u
      part = T(0);
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        if (cx.active) {
          const int o = (cx.g * LC + j) * M + cx.k;
          const V pj = pbuf[o];
          const V ap = cadd(acc[j], cscale(pj, lam));
          const V xj = cadd(xbuf[o], cscale(pj, alpha));
          xbuf[o] = xj;
          c[j] = csub(c[j], cscale(ap, alpha));
          part += cabs2(c[j]);
          if (snaps)
            snaps[((size_t)f * a.iters + it) * a.MN + (size_t)(cx.colbase + j) * M + cx.k] = xj;
        }
      }
      const T nn = cluster_sum<T>(part, red + (2 * 2 + par[2]) * 32, a.C, nwarps, lane, warp);
      par[2] ^= 1;
      const T beta = nn / cn;
      part = T(0);
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        if (cx.active) {
          const int o = (cx.g * LC + j) * M + cx.k;
          const V pj = cadd(c[j], cscale(pbuf[o], beta));
          pbuf[o] = pj;
          part += cabs2(pj);
        }
      }
      cn = nn;
      done = it + 1;
      if (lead && cnorm) cnorm[(size_t)f * stride + done] = cn;
      if (done < a.iters) {
        pp = cluster_sum<T>(part, red + (0 * 2 + par[0]) * 32, a.C, nwarps, lane, warp);
        par[0] ^= 1;
      }
    }
    if (lead) {
      if (cnorm) for (int i = done + 1; i < stride; ++i) cnorm[(size_t)f * stride + i] = T(0);
      if (a.itdone) a.itdone[f] = done;
      if (a.status) a.status[f] = exact ? 2 : 0;
    }

    // epilogue: x_hat out, fused hard decisions / LLRs / bit errors
    T scale = T(1);
    if (a.bps) {
      const T nv = nvar ? nvar[f] : lam;
      scale = nv > T(0) ? T(1) / nv : T(1);
    }
    int errs = 0;
    if (cx.active) {
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        const size_t q = fo + (size_t)(cx.colbase + j) * M + cx.k;
        const V xj = xbuf[(cx.g * LC + j) * M + cx.k];
        xo[q] = xj;
        if (a.bps) {
          const int lab = qam_demod_symbol<T>(xj.x, xj.y, a.bps, scale, a.llr ? a.llr + q * a.bps : nullptr);
          if (a.labels) a.labels[q] = (uint8_t)lab;
          if (a.txl) errs += __popc((unsigned)(lab ^ a.txl[q]));
        }
      }
    }
    if (a.berr) {
      errs = warp_sum(errs);
      if (lane == 0 && errs) atomicAdd(a.berr + f, errs);
    }
  }
}

size_t sscga_smem_bytes(int M, int N, int C, int elem_bytes) {
  const size_t vb = 2 * (size_t)elem_bytes;
  const size_t lcta = (size_t)N / C;
  return 3 * lcta * M * vb + 3 * 2 * 32 * (size_t)elem_bytes + (size_t)N * vb;
}

template <typename T, int LC>
static cudaError_t launch_lc(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  auto kern = sscga_kernel<T, LC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, s.smem);
  if (e != cudaSuccess) return e;
  if (s.cluster > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(s.threads);
  cfg.dynamicSmemBytes = s.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = s.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be co-resident, capped by the batch
  cfg.gridDim = dim3(s.cluster);
  int max_clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
  if (e != cudaSuccess) return e;
  if (max_clusters < 1) return cudaErrorInvalidConfiguration;
  const int nclu = a.B < max_clusters ? a.B : max_clusters;
  a.n_clusters = nclu;
  cfg.gridDim = dim3(nclu * s.cluster);
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename T>
cudaError_t launch_sscga(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  if (a.B == 0) return cudaSuccess;
  switch (s.lc) {
    case 1: return launch_lc<T, 1>(a, s, st);
    case 2: return launch_lc<T, 2>(a, s, st);
    case 4: return launch_lc<T, 4>(a, s, st);
    case 8: return launch_lc<T, 8>(a, s, st);
    case 16:
      if constexpr (sizeof(T) == 4) return launch_lc<T, 16>(a, s, st);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int LC>
static cudaError_t occ_lc(const LaunchShape& s, int* n) {
  auto kern = sscga_kernel<T, LC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, s.smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, s.threads, s.smem);
}

template <typename T>
cudaError_t sscga_occupancy(const LaunchShape& s, int* n) {
  switch (s.lc) {
    case 1: return occ_lc<T, 1>(s, n);
    case 2: return occ_lc<T, 2>(s, n);
    case 4: return occ_lc<T, 4>(s, n);
    case 8: return occ_lc<T, 8>(s, n);
    case 16:
      if constexpr (sizeof(T) == 4) return occ_lc<T, 16>(s, n);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

template cudaError_t launch_sscga<float>(SolveArgs, const LaunchShape&, cudaStream_t);
template cudaError_t launch_sscga<double>(SolveArgs, const LaunchShape&, cudaStream_t);
template cudaError_t sscga_occupancy<float>(const LaunchShape&, int*);
template cudaError_t sscga_occupancy<double>(const LaunchShape&, int*);

// ---------------------------------------------------------------------------
// Matrix-free batched operator over global memory (ss_mvm / ss_mvm_hermitian,
// sparse.py:147-160, without tables).  One thread per output element.
template <typename T, bool HERM>
__global__ void ss_apply_kernel(int M, int N, const int* __restrict__ off, const int* __restrict__ pk,
                                const int* __restrict__ pl, const Vec<T>* __restrict__ ph,
                                const Vec<T>* __restrict__ v, Vec<T>* __restrict__ out) {
  using V = Vec<T>;
  const int MN = M * N;
  const int f = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= MN) return;
  const int k = q % M, l = q / M;
  const int K0 = M / 2, L0 = N / 2;
  const int P0 = off[f], P1 = off[f + 1];
  const V* vf = v + (size_t)f * MN;
  V acc = czero<V>();
  for (int p = P0; p < P1; ++p) {
    const int dk = K0 - pk[p], dl = L0 - pl[p];
    V h = ph[p];
    const int ar = HERM ? k - dk : k + dk;
    const int n = ar < 0 ? -1 : (ar >= M ? 1 : 0);
    const int ks = ar - n * M;
    int e;
    if (HERM) {
      e = mod_pos(dl * (k - n * M) + n * M * l, MN);
      h = cconj(h);
    } else {
      e = mod_pos(-dl * ks + n * M * l, MN);
    }
    const int ls = mod_pos(l + (HERM ? -dl : dl), N);
    cfma(acc, cmul(h, twiddle(T(0), e, MN)), vf[ls * M + ks]);
  }
  out[(size_t)f * MN + q] = acc;
}

template <typename T>
cudaError_t launch_ss_apply(int B, int M, int N, const int* off, const int* pk, const int* pl,
                            const void* ph, const void* v, void* out, bool herm, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  using V = Vec<T>;
  const int MN = M * N;
  dim3 grid((MN + 255) / 256, B);
  if (herm)
    ss_apply_kernel<T, true><<<grid, 256, 0, st>>>(M, N, off, pk, pl, (const V*)ph, (const V*)v, (V*)out);
  else
    ss_apply_kernel<T, false><<<grid, 256, 0, st>>>(M, N, off, pk, pl, (const V*)ph, (const V*)v, (V*)out);
  return cudaGetLastError();
}

template cudaError_t launch_ss_apply<float>(int, int, int, const int*, const int*, const int*,
                                            const void*, const void*, void*, bool, cudaStream_t);
template cudaError_t launch_ss_apply<double>(int, int, int, const int*, const int*, const int*,
                                             const void*, const void*, void*, bool, cudaStream_t);

}  // namespace ddb
