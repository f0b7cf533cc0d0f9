// API-parity kernels around the fused solve:
//   K4 table materialisation   (sparse.py:124-144 build_ss_channel)
//   K5 table-driven MVM        (sparse.py:147-160 ss_mvm / ss_mvm_hermitian)
//   K6 demod                   (grid.py:172-183 hard_demod; Gray-QAM max-log LLR)
//   f1 path detection          (sparse.py:69-88 detect_paths)
#include "common.cuh"
#include "demod.cuh"
#include "internal.h"

namespace ddb {

// ---- K4: one thread per (tap, output index); fp64 like the reference tables.
// fwd_col   = forward_index (sparse.py:91-96)
// fwd_coef  = coefficient   (sparse.py:107-121), phase index reduced mod MN
// herm_row  = inverse_index (sparse.py:99-104)
// herm_coef = conj(fwd_coef[p, herm_row])  (sparse.py:139), evaluated in place
__device__ __forceinline__ void fwd_entry(int M, int N, int kp, int lp, int q, int* col, int* e) {
  const int MN = M * N, K0 = M / 2, L0 = N / 2;
  const int k = q % M, l = q / M;
  const int dk = K0 - kp, dl = L0 - lp;
  const int a = k + dk;
  const int n = a < 0 ? -1 : (a >= M ? 1 : 0);
  const int ks = a - n * M;
  *col = mod_pos(l + dl, N) * M + ks;
  *e = mod_pos(-dl * ks + n * M * l, MN);
}

__global__ void build_tables_kernel(int M, int N, int P, const int* __restrict__ pk,
                                    const int* __restrict__ pl, const double2* __restrict__ ph,
                                    double2* fwd_coef, int* fwd_col, double2* herm_coef, int* herm_row) {
  const int MN = M * N;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)P * MN) return;
  const int p = (int)(i / MN), q = (int)(i - (long long)p * MN);
  const int kp = pk[p], lp = pl[p];
  const double2 h = ph[p];
  int col, e;
  fwd_entry(M, N, kp, lp, q, &col, &e);
  fwd_col[i] = col;
  fwd_coef[i] = cmul(h, twiddle(0.0, e, MN));
  // inverse map: the row whose forward source is q
  const int K0 = M / 2, L0 = N / 2;
  const int dk = K0 - kp, dl = L0 - lp;
  const int k = q % M, l = q / M;
  const int row = mod_pos(l - dl, N) * M + mod_pos(k - dk, M);
  herm_row[i] = row;
  int col2, e2;
  fwd_entry(M, N, kp, lp, row, &col2, &e2);
  herm_coef[i] = cconj(cmul(h, twiddle(0.0, e2, MN)));
}

cudaError_t launch_build_tables(int M, int N, int P, const int* pk, const int* pl, const void* ph,
                                void* fwd_coef, int* fwd_col, void* herm_coef, int* herm_row,
                                cudaStream_t st) {
  const long long total = (long long)P * M * N;
  if (total == 0) return cudaSuccess;
  const int bs = 256;
  const long long nb = (total + bs - 1) / bs;
  build_tables_kernel<<<(unsigned)nb, bs, 0, st>>>(M, N, P, pk, pl, (const double2*)ph,
                                                   (double2*)fwd_coef, fwd_col, (double2*)herm_coef,
                                                   herm_row);
  return cudaGetLastError();
}

// ---- K5: u[q] = sum_p coef[p, q] v[index[p, q]] (einsum "pq,pq->q", sparse.py:152)
__global__ void mvm_tables_kernel(int size, int P, const double2* __restrict__ coef,
                                  const int* __restrict__ idx, const double2* __restrict__ v,
                                  double2* __restrict__ u) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= size) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int p = 0; p < P; ++p) {
    const size_t o = (size_t)p * size + q;
    cfma(acc, coef[o], v[idx[o]]);
  }
  u[q] = acc;
}

cudaError_t launch_mvm_tables(int size, int P, const void* coef, const int* idx, const void* v,
                              void* u, cudaStream_t st) {
  if (size == 0) return cudaSuccess;
  mvm_tables_kernel<<<(size + 255) / 256, 256, 0, st>>>(size, P, (const double2*)coef, idx,
                                                        (const double2*)v, (double2*)u);
  return cudaGetLastError();
}

// ---- K6a: nearest point over an arbitrary table, lowest label on ties
//      (grid.py:172-183: argmin of |v - s|^2, numpy argmin keeps the first).
template <typename T>
__global__ void hard_demod_kernel(long long count, const Vec<T>* __restrict__ x,
                                  const Vec<T>* __restrict__ pts, int npts, int* __restrict__ labels) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const Vec<T> v = x[i];
  int best = 0;
  T bestd = T(0);
  for (int s = 0; s < npts; ++s) {
    const Vec<T> pt = pts[s];
    // np.abs(v - s) ** 2, rounded exactly as numpy does it
    const T m = np_cabs(v.x - pt.x, v.y - pt.y);
    const T d = m * m;
    if (s == 0 || d < bestd) { bestd = d; best = s; }
  }
  labels[i] = best;
}

template <typename T>
cudaError_t launch_hard_demod(long long count, const void* x, const void* pts, int npts, int* labels,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const long long nb = (count + 255) / 256;
  hard_demod_kernel<T><<<(unsigned)nb, 256, 0, st>>>(count, (const Vec<T>*)x, (const Vec<T>*)pts,
                                                      npts, labels);
  return cudaGetLastError();
}
template cudaError_t launch_hard_demod<float>(long long, const void*, const void*, int, int*, cudaStream_t);
template cudaError_t launch_hard_demod<double>(long long, const void*, const void*, int, int*, cudaStream_t);

// ---- K6b: Gray-QAM slicer + max-log LLR (same device code as the fused epilogue)
template <typename T>
__global__ void qam_demod_kernel(long long count, const Vec<T>* __restrict__ x, int bps, T scale,
                                 uint8_t* labels, float* llr) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const Vec<T> v = x[i];
  const int lab = qam_demod_symbol<T>(v.x, v.y, bps, scale, llr ? llr + i * bps : nullptr);
  if (labels) labels[i] = (uint8_t)lab;
}

template <typename T>
cudaError_t launch_qam_demod(long long count, const void* x, int bps, double nvar, uint8_t* labels,
                             float* llr, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const T scale = nvar > 0 ? T(1.0 / nvar) : T(1);
  const long long nb = (count + 255) / 256;
  qam_demod_kernel<T><<<(unsigned)nb, 256, 0, st>>>(count, (const Vec<T>*)x, bps, scale, labels, llr);
  return cudaGetLastError();
}
template cudaError_t launch_qam_demod<float>(long long, const void*, int, double, uint8_t*, float*, cudaStream_t);
template cudaError_t launch_qam_demod<double>(long long, const void*, int, double, uint8_t*, float*, cudaStream_t);

// ---- f1: detect_paths (sparse.py:69-88), one CTA per frame.
// peak = max |h|; keep |h| > theta * peak (strict); candidates are compacted
// in row-major (k, l) order (np.nonzero on the (M, N) frame) and ranked by
// descending |h| with ties kept in that order (argsort kind="stable").
constexpr int kDetectThreads = 1024;

__device__ __forceinline__ double block_max(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? scratch[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) scratch[0] = v;
  }
  __syncthreads();
  v = scratch[0];
  __syncthreads();
  return v;
}

// |h| is evaluated once per bin into shared memory when the frame fits (else
// re-read), candidates are compacted in row-major order with warp ballots over
// coalesced bin ranges, then ranked.
__global__ void __launch_bounds__(kDetectThreads) detect_paths_kernel(
    int M, int N, const double2* __restrict__ heff, double theta, int max_paths, int cap, int mag_smem,
    int* count, int* pk, int* pl, double2* ph) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = M * N;
  double* mag = reinterpret_cast<double*>(smem);                        // [n] when mag_smem
  int* cidx = reinterpret_cast<int*>(mag + (mag_smem ? n : 0));         // [cap]
  __shared__ double dscratch[32];
  __shared__ int wcount[32];
  __shared__ int running;
  const int f = blockIdx.x;
  const double2* h = heff + (size_t)f * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double peak = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double m = np_cabs(h[i].x, h[i].y);
    if (mag_smem) mag[i] = m;
    peak = fmax(peak, m);
  }
  peak = block_max(peak, dscratch);  // (contains the barriers that publish mag)
  if (peak == 0.0) {  // sparse.py:81-82
    if (threadIdx.x == 0) count[f] = 0;
    return;
  }
  const double thr = theta * peak;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  // order-preserving compaction of {i : |h_i| > thr} (np.nonzero on the (M, N) frame)
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool keep = i < n && (mag_smem ? mag[i] : np_cabs(h[i].x, h[i].y)) > thr;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int before = running;
    for (int w = 0; w < warp; ++w) before += wcount[w];
    const int pos = before + __popc(bal & ((1u << lane) - 1u));
    if (keep && pos < cap) cidx[pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = running;
      for (int w = 0; w < nw; ++w) t += wcount[w];
      running = t;
    }
    __syncthreads();
  }
  const int total = running;
  if (threadIdx.x == 0) count[f] = total > cap ? -1 : total;
  if (total > cap) return;  // -1: candidate list exceeds shared memory; host reports it
  // descending |h|, ties in row-major order (argsort kind="stable")
  for (int c = threadIdx.x; c < total; c += blockDim.x) {
    const int ic = cidx[c];
    const double m = mag_smem ? mag[ic] : np_cabs(h[ic].x, h[ic].y);
    int rank = 0;
    for (int o = 0; o < total; ++o) {
      const int io = cidx[o];
      const double mo = mag_smem ? mag[io] : np_cabs(h[io].x, h[io].y);
      rank += (mo > m) || (mo == m && o < c);
    }
    if (rank < max_paths) {
      const size_t out = (size_t)f * max_paths + rank;
      pk[out] = ic / N;
      pl[out] = ic - (ic / N) * N;
      ph[out] = h[ic];
    }
  }
}

cudaError_t launch_detect_paths(int B, int M, int N, const void* heff, double theta, int max_paths,
                                int* count, int* pk, int* pl, void* ph, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int n = M * N;
  const int budget = optin - 2048;  // static shared memory of the kernel
  // keep the frame's magnitudes on chip when they leave room for a candidate list
  const int mag_smem = (size_t)n * sizeof(double) + 4096 * sizeof(int) <= (size_t)budget ? 1 : 0;
  int cap = (budget - (mag_smem ? n * (int)sizeof(double) : 0)) / (int)sizeof(int);
  if (cap > n) cap = n;
  const size_t smem = (mag_smem ? (size_t)n * sizeof(double) : 0) + (size_t)cap * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(detect_paths_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  detect_paths_kernel<<<B, kDetectThreads, smem, st>>>(M, N, (const double2*)heff, theta, max_paths, cap, mag_smem,
                                                       count, pk, pl, (double2*)ph);
  return cudaGetLastError();
}

}  // namespace ddb

namespace ddb {

// ---- FP32 roofline probe: pure FMA chains (8 independent per thread) so the
// bench can state the measured FP32 peak of the box it runs on.  mode 0:
// scalar FFMA with register operands; mode 1: packed FFMA2 (fma.rn.f32x2).
template <int MODE>
__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float m, float c) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  if (MODE == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], m, c);
    }
  } else {
    unsigned long long p[4], mm, cc;
    asm("mov.b64 %0, {%1, %1};" : "=l"(mm) : "f"(m));
    asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
#pragma unroll
    for (int i = 0; i < 4; ++i) asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(mm), "l"(cc));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) asm("mov.b64 {%0, %1}, %2;" : "=f"(a[2 * i]), "=f"(a[2 * i + 1]) : "l"(p[i]));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[blockIdx.x] = s;  // keep the chains alive
}

cudaError_t launch_fp32_probe(int mode, int blocks, int iters, float* out, cudaStream_t st) {
  if (mode == 0) fp32_probe_kernel<0><<<blocks, 256, 0, st>>>(out, iters, 0.999f, 1e-3f);
  else fp32_probe_kernel<1><<<blocks, 256, 0, st>>>(out, iters, 0.999f, 1e-3f);
  return cudaGetLastError();
}

}  // namespace ddb
