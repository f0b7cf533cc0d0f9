// Receiver front end: the discrete Zak transform of a
// received frame as the compact GEMM of zak.py:50-55 (dzt_gemm), optionally
// fused with the point-pilot channel estimate of pilot.py:40-49
// (estimate_heff: times the twist kernel of pilot.py:29-37, divided by the
// pilot amplitude).
//
//   Y[k, l] = sum_i y[k + i M] K[i, l],   K = build_zak_kernel(N) (zak.py:33-47)
//            = (1/sqrt N) e^{-j 2 pi i l / N}, or any caller-supplied N x N kernel
//   heff[k, l] = Y[k, l] e^{-j 2 pi K0 (l - L0) / (M N)} / amplitude
//
// One CTA per (frame, tile of TK delay rows): the N time blocks of the tile are
// staged in shared memory with loads coalesced along delay, the kernel matrix
// next to them; each thread owns one delay row and a block of Doppler columns
// (register-blocked when 4 | N), so the y value it reads is its own
// (conflict-free) and the kernel entries are warp broadcasts.  Phases come
// from exact integer indices (no drift with MN).  Roofline: HBM, 16 bytes in
// and out per element at fp32 (32 at fp64), N complex MACs per element.
#include "common.cuh"
#include "internal.h"

namespace ddb {

namespace {

constexpr int kTk = 64;        // delay rows per CTA
constexpr int kDztThreads = 256;

template <typename T, bool COLMAJOR, bool PILOT>
__global__ void __launch_bounds__(kDztThreads) dzt_kernel(int M, int N, const Vec<T>* __restrict__ y,
                                                          const Vec<T>* __restrict__ kern, int sgn, T inv_amp,
                                                          Vec<T>* __restrict__ out) {
  using V = Vec<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  V* ys = reinterpret_cast<V*>(smem);  // [N][kTk]
  V* kk = ys + (size_t)N * kTk;        // [N][N]
  const int f = blockIdx.y;
  const int k0 = blockIdx.x * kTk;
  const int MN = M * N;
  const V* yf = y + (size_t)f * MN;
  const T rs = T(1) / sqrt(T(N));
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    if (kern) {
      kk[idx] = kern[idx];
    } else {
      const int i = idx / N, l = idx - (idx / N) * N;
      kk[idx] = cscale(twiddle(T(0), mod_pos(sgn * ((i * l) % N), N), N), rs);
    }
  }
  for (int idx = threadIdx.x; idx < N * kTk; idx += blockDim.x) {
    const int i = idx / kTk, kl = idx - i * kTk;
    const int k = k0 + kl;
    ys[idx] = k < M ? yf[k + (size_t)i * M] : czero<V>();
  }
  __syncthreads();
  const int kl = threadIdx.x % kTk;
  const int k = k0 + kl;
  if (k >= M) return;
  const int groups = blockDim.x / kTk;
  for (int l = threadIdx.x / kTk; l < N; l += groups) {
    V acc = czero<V>();
    for (int i = 0; i < N; ++i) cfma(acc, ys[i * kTk + kl], kk[i * N + l]);
    if constexpr (PILOT) {
      // e^{-j 2 pi K0 (l - L0) / (M N)}, exact integer phase (pilot.py:29-37)
      const long long e = (long long)(M / 2) * (l - N / 2);
      const int er = (int)(((-e) % MN + MN) % MN);
      acc = cscale(cmul(acc, twiddle(T(0), er, MN)), inv_amp);
    }
    if constexpr (COLMAJOR) out[(size_t)f * MN + (size_t)l * M + k] = acc;
    else out[(size_t)f * MN + (size_t)k * N + l] = acc;
  }
}

// Register-blocked variant for N = 4 NB: thread (delay row, quarter of the
// Doppler columns) keeps NB accumulators; per time block it reads its own
// y value once and the NB kernel entries as warp broadcasts, so shared-memory
// traffic per complex MAC drops ~5x and the kernel becomes FMA/HBM bound.
template <typename T, bool COLMAJOR, bool PILOT, int NB>
__global__ void __launch_bounds__(kDztThreads) dzt_blk_kernel(int M, int N, const Vec<T>* __restrict__ y,
                                                              const Vec<T>* __restrict__ kern, int sgn, T inv_amp,
                                                              Vec<T>* __restrict__ out) {
  using V = Vec<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  V* ys = reinterpret_cast<V*>(smem);  // [N][kTk]
  V* kk = ys + (size_t)N * kTk;        // [N][N]
  const int f = blockIdx.y;
  const int k0 = blockIdx.x * kTk;
  const int MN = M * N;
  const V* yf = y + (size_t)f * MN;
  const T rs = T(1) / sqrt(T(N));
  V* wn = kk + (size_t)N * N;  // [N]: W_N^{sgn e} / sqrt(N), the only distinct kernel values
  for (int e = threadIdx.x; e < N; e += blockDim.x) wn[e] = cscale(twiddle(T(0), mod_pos(sgn * e, N), N), rs);
  for (int idx = threadIdx.x; idx < N * kTk; idx += blockDim.x) {
    const int i = idx / kTk, kl = idx - i * kTk;
    const int k = k0 + kl;
    ys[idx] = k < M ? yf[k + (size_t)i * M] : czero<V>();
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    const int i = idx / N, l = idx - (idx / N) * N;
    kk[idx] = kern ? kern[idx] : wn[(i * l) % N];
  }
  __syncthreads();
  const int kl = threadIdx.x % kTk;
  const int k = k0 + kl;
  const int l0 = (threadIdx.x / kTk) * NB;  // warp-uniform (kTk >= 32)
  V acc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j] = czero<V>();
#pragma unroll 4
  for (int i = 0; i < N; ++i) {
    const V v = ys[i * kTk + kl];
    const V* kr = kk + i * N + l0;
#pragma unroll
    for (int j = 0; j < NB; ++j) cfma(acc[j], v, kr[j]);
  }
  if (k >= M) return;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int l = l0 + j;
    V r = acc[j];
    if constexpr (PILOT) {
      const long long e = (long long)(M / 2) * (l - N / 2);
      const int er = (int)(((-e) % MN + MN) % MN);
      r = cscale(cmul(r, twiddle(T(0), er, MN)), inv_amp);
    }
    if constexpr (COLMAJOR) out[(size_t)f * MN + (size_t)l * M + k] = r;
    else out[(size_t)f * MN + (size_t)k * N + l] = r;
  }
}

// Default kernel (build_zak_kernel(N), N a power of two): the same transform
// as a radix-2 FFT along the N time blocks of every delay row, log2 N stages
// of N/2 butterflies in shared memory instead of N complex MACs per element
// (the GEMM form is kept for caller-supplied kernels).  The input is stored in
// bit-reversed block order while it is loaded, so the decimation-in-time
// stages leave the Doppler columns in natural order; twiddles come from exact
// integer phases.  Same result to rounding (parity tolerances 1e-12 fp64).
template <typename T, bool COLMAJOR, bool PILOT, typename VIN = Vec<T>>
__global__ void __launch_bounds__(kDztThreads) dzt_fft_kernel(int M, int N, int logn, const VIN* __restrict__ y,
                                                              int sgn, T inv_amp, Vec<T>* __restrict__ out) {
  using V = Vec<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  V* xs = reinterpret_cast<V*>(smem);  // [N][kTk], block index bit-reversed
  V* wn = xs + (size_t)N * kTk;        // [N/2]: W_N^{sgn e} (sgn -1: dzt, +1: idzt)
  V* twist = wn + N / 2;               // [N] (PILOT): e^{-j2pi K0 (l - L0)/MN} / amplitude, per Doppler column
  const int f = blockIdx.y;
  const int k0 = blockIdx.x * kTk;
  const int MN = M * N;
  const VIN* yf = y + (size_t)f * MN;
  for (int e = threadIdx.x; e < N / 2; e += blockDim.x) wn[e] = twiddle(T(0), mod_pos(sgn * e, N), N);
  if constexpr (PILOT) {
    for (int l = threadIdx.x; l < N; l += blockDim.x) {
      const long long e = (long long)(M / 2) * (l - N / 2);
      const int er = (int)(((-e) % MN + MN) % MN);
      twist[l] = cscale(twiddle(T(0), er, MN), inv_amp);
    }
  }
  for (int idx = threadIdx.x; idx < N * kTk; idx += blockDim.x) {
    const int i = idx / kTk, kl = idx - i * kTk;
    const int k = k0 + kl;
    const int ir = (int)(__brev((unsigned)i) >> (32 - logn));
    V v = czero<V>();
    if (k < M) {
      const VIN t = yf[k + (size_t)i * M];
      v = cmake<V>(t.x, t.y);
    }
    xs[ir * kTk + kl] = v;
  }
  __syncthreads();
  const int kl = threadIdx.x % kTk;
  const int g0 = threadIdx.x / kTk, groups = blockDim.x / kTk;
  for (int st = 0; st < logn; ++st) {
    const int half = 1 << st;
    for (int bf = g0; bf < N / 2; bf += groups) {
      const int grp = bf >> st, pos = bf & (half - 1);
      const int i0 = (grp << (st + 1)) + pos, i1 = i0 + half;
      const V w = wn[pos << (logn - 1 - st)];
      const V a0 = xs[i0 * kTk + kl];
      const V t = cmul(w, xs[i1 * kTk + kl]);
      xs[i0 * kTk + kl] = cadd(a0, t);
      xs[i1 * kTk + kl] = csub(a0, t);
    }
    __syncthreads();
  }
  const T rs = T(1) / sqrt(T(N));
  const int k = k0 + kl;
  if (k >= M) return;
  for (int l = g0; l < N; l += groups) {
    V r = cscale(xs[l * kTk + kl], rs);
    if constexpr (PILOT) r = cmul(r, twist[l]);  // twist constant along delay (pilot.py:29-37)
    if constexpr (COLMAJOR) out[(size_t)f * MN + (size_t)l * M + k] = r;
    else out[(size_t)f * MN + (size_t)k * N + l] = r;
  }
}

template <typename T, bool COLMAJOR, bool PILOT>
cudaError_t launch_dzt_t(int B, int M, int N, const void* y, const void* kern, int sgn, double amp, void* out,
                         cudaStream_t st) {
  using V = Vec<T>;
  const size_t smem = ((size_t)N * kTk + (size_t)N * N + N) * sizeof(V);
  dim3 grid((M + kTk - 1) / kTk, B);
  const int groups = kDztThreads / kTk;
  auto run = [&](auto kfn) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, kDztThreads, smem, st>>>(M, N, (const V*)y, (const V*)kern, sgn, T(1.0 / amp), (V*)out);
    return cudaGetLastError();
  };
  if (!kern && N >= 2 && (N & (N - 1)) == 0) {  // default kernel, power-of-two N: FFT
    int logn = 0;
    while ((1 << logn) < N) ++logn;
    const size_t fsmem = ((size_t)N * kTk + N / 2 + N) * sizeof(V);
    cudaError_t e = cudaFuncSetAttribute(dzt_fft_kernel<T, COLMAJOR, PILOT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    if (e != cudaSuccess) return e;
    dzt_fft_kernel<T, COLMAJOR, PILOT><<<grid, kDztThreads, fsmem, st>>>(M, N, logn, (const V*)y, sgn,
                                                                        T(1.0 / amp), (V*)out);
    return cudaGetLastError();
  }
  if (N % groups == 0) {
    switch (N / groups) {
      case 1: return run(dzt_blk_kernel<T, COLMAJOR, PILOT, 1>);
      case 2: return run(dzt_blk_kernel<T, COLMAJOR, PILOT, 2>);
      case 4: return run(dzt_blk_kernel<T, COLMAJOR, PILOT, 4>);
      case 8: return run(dzt_blk_kernel<T, COLMAJOR, PILOT, 8>);
      case 16: return run(dzt_blk_kernel<T, COLMAJOR, PILOT, 16>);
      default: break;
    }
  }
  return run(dzt_kernel<T, COLMAJOR, PILOT>);
}

template <typename T>
__global__ void estimate_heff_kernel(long long count, const Vec<T>* __restrict__ ydd, const Vec<T>* __restrict__ tw,
                                     T inv_amp, Vec<T>* __restrict__ heff) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    heff[i] = cscale(cmul(ydd[i], tw[i]), inv_amp);
}

}  // namespace

// fp64 arithmetic on complex64 samples (the pilot path: no separate widening
// pass); default kernel, power-of-two N.
template <bool COLMAJOR, bool PILOT>
cudaError_t launch_dzt_mixed_t(int B, int M, int N, const void* y, double amp, void* out, cudaStream_t st) {
  int logn = 0;
  while ((1 << logn) < N) ++logn;
  const size_t fsmem = ((size_t)N * kTk + N / 2 + N) * sizeof(double2);
  auto kfn = dzt_fft_kernel<double, COLMAJOR, PILOT, float2>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
  if (e != cudaSuccess) return e;
  dim3 grid((M + kTk - 1) / kTk, B);
  kfn<<<grid, kDztThreads, fsmem, st>>>(M, N, logn, (const float2*)y, -1, 1.0 / amp, (double2*)out);
  return cudaGetLastError();
}

cudaError_t launch_dzt_mixed(int B, int M, int N, const void* y, int colmajor, int pilot, double amp, void* out,
                             cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  if (N < 2 || (N & (N - 1))) return cudaErrorInvalidValue;
  const int sel = (colmajor ? 1 : 0) | (pilot ? 2 : 0);
  switch (sel) {
    case 0: return launch_dzt_mixed_t<false, false>(B, M, N, y, amp, out, st);
    case 1: return launch_dzt_mixed_t<true, false>(B, M, N, y, amp, out, st);
    case 2: return launch_dzt_mixed_t<false, true>(B, M, N, y, amp, out, st);
    default: return launch_dzt_mixed_t<true, true>(B, M, N, y, amp, out, st);
  }
}

cudaError_t launch_dzt(int dtype_f64, int B, int M, int N, const void* y, const void* kern, int colmajor, int pilot,
                       int inverse, double amp, void* out, cudaStream_t st) {
  const int sgn = inverse ? 1 : -1;
  if (B == 0) return cudaSuccess;
  const int sel = (colmajor ? 1 : 0) | (pilot ? 2 : 0);
  if (dtype_f64) {
    switch (sel) {
      case 0: return launch_dzt_t<double, false, false>(B, M, N, y, kern, sgn, amp, out, st);
      case 1: return launch_dzt_t<double, true, false>(B, M, N, y, kern, sgn, amp, out, st);
      case 2: return launch_dzt_t<double, false, true>(B, M, N, y, kern, sgn, amp, out, st);
      default: return launch_dzt_t<double, true, true>(B, M, N, y, kern, sgn, amp, out, st);
    }
  }
  switch (sel) {
    case 0: return launch_dzt_t<float, false, false>(B, M, N, y, kern, sgn, amp, out, st);
    case 1: return launch_dzt_t<float, true, false>(B, M, N, y, kern, sgn, amp, out, st);
    case 2: return launch_dzt_t<float, false, true>(B, M, N, y, kern, sgn, amp, out, st);
    default: return launch_dzt_t<float, true, true>(B, M, N, y, kern, sgn, amp, out, st);
  }
}

cudaError_t launch_estimate_heff(int dtype_f64, long long count, const void* ydd, const void* twist, double amp,
                                 void* heff, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const int blocks = (int)((count + 255) / 256 < 148 * 16 ? (count + 255) / 256 : 148 * 16);
  if (dtype_f64)
    estimate_heff_kernel<double><<<blocks, 256, 0, st>>>(count, (const double2*)ydd, (const double2*)twist,
                                                         1.0 / amp, (double2*)heff);
  else
    estimate_heff_kernel<float><<<blocks, 256, 0, st>>>(count, (const float2*)ydd, (const float2*)twist,
                                                        (float)(1.0 / amp), (float2*)heff);
  return cudaGetLastError();
}

}  // namespace ddb
