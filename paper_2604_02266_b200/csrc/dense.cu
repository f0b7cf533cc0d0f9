// Dense LMMSE baseline, small grids only (MN <= 4096,
// sparse.py DENSE_GUARD): the effective-channel frame thresholded as
// threshold_frame (sparse.py:163-169) and expanded to the full MN x MN DD
// channel matrix of build_dense_hdd (sparse.py:172-206).  The Gram matrix and
// its Cholesky solve (equalize.py:80-94) are library calls on the host side
// (cuBLAS / cuSOLVER through torch), as the survey allows for this
// off-hot-path cross-check.
//
// Entry (row q' = l' M + k', column q = l M + k): the unique wrap pair
// n = floor((k' - k + K0) / M), m = floor((l' - l + L0) / N) puts
// (dk, dl) = (k' - k - n M, l' - l - m N) in the signed fundamental range; the
// entry is heff[K0 + dk, L0 + dl] e^{j 2 pi (dl (k + n M) + n l M) / MN}, the
// phase taken from the exact integer exponent mod MN.  Roofline: HBM writes
// of 8 / 16 bytes per entry (the frame is L1/L2 resident).
#include "common.cuh"
#include "internal.h"

namespace ddb {

namespace {

constexpr int kDnThreads = 256;

// One CTA per frame: peak |h| (numpy's abs) and the strict threshold.
template <typename T>
__global__ void __launch_bounds__(kDnThreads) threshold_kernel(int MN, const Vec<T>* __restrict__ heff, double theta,
                                                             Vec<T>* __restrict__ out) {
  __shared__ double part[kDnThreads / 32];
  const Vec<T>* h = heff + (size_t)blockIdx.x * MN;
  Vec<T>* o = out + (size_t)blockIdx.x * MN;
  double m = 0.0;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) m = fmax(m, np_cabs((double)h[i].x, (double)h[i].y));
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
  __syncthreads();
  double peak = 0.0;
  for (int w = 0; w < kDnThreads / 32; ++w) peak = fmax(peak, part[w]);
  const double thr = theta * peak;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    const Vec<T> v = h[i];
    const bool keep = peak == 0.0 || np_cabs((double)v.x, (double)v.y) > thr;  // sparse.py:165-168
    o[i] = keep ? v : czero<Vec<T>>();
  }
}

// grid (MN / kDnThreads column tiles, MN rows, B); thread = one column of one row.
template <typename T>
__global__ void __launch_bounds__(kDnThreads) dense_hdd_kernel(int M, int N, const Vec<T>* __restrict__ heff,
                                                             Vec<T>* __restrict__ H) {
  const int MN = M * N, K0 = M / 2, L0 = N / 2;
  const int f = blockIdx.z;
  const int row = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= MN) return;
  const int kr = row % M, lr = row / M, kc = col % M, lc = col / M;
  const int n = (int)floor((double)(kr - kc + K0) / M);
  const int m = (int)floor((double)(lr - lc + L0) / N);
  const int dk = kr - kc - n * M, dl = lr - lc - m * N;
  const Vec<T> tap = heff[(size_t)f * MN + (size_t)(K0 + dk) * N + (L0 + dl)];  // (M, N) row-major frame
  Vec<T> v = czero<Vec<T>>();
  if (tap.x != T(0) || tap.y != T(0)) {
    const long long e = (long long)dl * (kc + (long long)n * M) + (long long)n * lc * M;
    const int er = (int)(((e % MN) + MN) % MN);
    v = cmul(tap, twiddle(T(0), er, MN));
  }
  H[((size_t)f * MN + row) * MN + col] = v;
}

}  // namespace

cudaError_t launch_threshold_frame(int dtype_f64, int B, int MN, const void* heff, double theta, void* out,
                                   cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  if (dtype_f64)
    threshold_kernel<double><<<B, kDnThreads, 0, st>>>(MN, (const double2*)heff, theta, (double2*)out);
  else
    threshold_kernel<float><<<B, kDnThreads, 0, st>>>(MN, (const float2*)heff, theta, (float2*)out);
  return cudaGetLastError();
}

cudaError_t launch_build_dense(int dtype_f64, int B, int M, int N, const void* heff, void* H, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int MN = M * N;
  dim3 grid((MN + kDnThreads - 1) / kDnThreads, MN, B);
  if (dtype_f64)
    dense_hdd_kernel<double><<<grid, kDnThreads, 0, st>>>(M, N, (const double2*)heff, (double2*)H);
  else
    dense_hdd_kernel<float><<<grid, kDnThreads, 0, st>>>(M, N, (const float2*)heff, (float2*)H);
  return cudaGetLastError();
}

}  // namespace ddb
