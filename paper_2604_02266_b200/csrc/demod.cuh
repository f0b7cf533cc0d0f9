// Gray-QAM hard decisions and max-log LLRs on the reference's constellations
// (grid.py:98-154): label bits are MSB first, even bit positions drive I and
// odd ones Q; per axis the Gray PAM levels follow TS 38.211 in the recursive
// form of grid.py:98-109,
//     level(c0..c_{ba-1}) = (1 - 2 c0) * mag,  mag = 2^{ba-m} - (1 - 2 c_m) mag'
// divided by the rms norm sqrt(2 (4^ba - 1) / 3) (sqrt2, sqrt10, sqrt42), as
// make_constellation does (grid.py:151).  ba = 1, 2 reproduce qpsk / qam16
// exactly; ba = 3 (64-QAM) is the build extension the north star asks for
// (the reference rejects qam64, tests/test_grid.py:85-87), so its parity is
// pinned only through the LLR-sign == hard-decision identity.
//
// Nearest-point decisions on a separable Gray grid reduce to a per-axis
// argmin; taking the lowest axis index on ties reproduces hard_demod's
// lowest-label tie rule (grid.py:172-183).  Everything is specialised on the
// bits per axis at compile time, so the levels are immediates.
#pragma once

#include "common.cuh"

namespace ddb {

template <int BA> __host__ __device__ constexpr int qam_level(int i) {
  int mag = 1;
  for (int m = BA - 1; m >= 1; --m) {
    const int cm = (i >> (BA - 1 - m)) & 1;
    mag = (1 << (BA - m)) - (1 - 2 * cm) * mag;
  }
  return (1 - 2 * ((i >> (BA - 1)) & 1)) * mag;
}
template <int BA> __host__ __device__ constexpr double qam_norm() {
  return BA == 1 ? 1.4142135623730951 : (BA == 2 ? 3.1622776601683795 : 6.48074069840786);
}

// One axis: returns the axis index (bits MSB first); writes BA LLRs to llr[2m]
// (interleaved with the other axis) when llr != nullptr.
template <typename T, int BA>
__device__ __forceinline__ int qam_axis(T v, T scale, float* llr) {
  constexpr int L = 1 << BA;
  T d[L];
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const T a = T((double)qam_level<BA>(i) / qam_norm<BA>());
    d[i] = (v - a) * (v - a);
  }
  int best = 0;
  T bestd = d[0];
#pragma unroll
  for (int i = 1; i < L; ++i)
    if (d[i] < bestd) { bestd = d[i]; best = i; }
  if (llr) {
#pragma unroll
    for (int m = 0; m < BA; ++m) {
      T d1 = T(3.0e38), d0 = T(3.0e38);
#pragma unroll
      for (int i = 0; i < L; ++i) {
        if ((i >> (BA - 1 - m)) & 1) d1 = d[i] < d1 ? d[i] : d1;
        else d0 = d[i] < d0 ? d[i] : d0;
      }
      llr[2 * m] = (float)((d1 - d0) * scale);
    }
  }
  return best;
}

template <typename T, int BA>
__device__ __forceinline__ int qam_symbol(T re, T im, T scale, float* llr) {
  const int ii = qam_axis<T, BA>(re, scale, llr);
  const int qi = qam_axis<T, BA>(im, scale, llr ? llr + 1 : nullptr);
  int label = 0;
#pragma unroll
  for (int m = 0; m < BA; ++m) {
    label |= ((ii >> (BA - 1 - m)) & 1) << (2 * BA - 1 - 2 * m);
    label |= ((qi >> (BA - 1 - m)) & 1) << (2 * BA - 2 - 2 * m);
  }
  return label;
}

// Runtime-dispatched form (standalone kernels); bps in {2, 4, 6}.
template <typename T>
__device__ __forceinline__ int qam_demod_symbol(T re, T im, int bps, T scale, float* llr) {
  switch (bps) {
    case 2: return qam_symbol<T, 1>(re, im, scale, llr);
    case 4: return qam_symbol<T, 2>(re, im, scale, llr);
    default: return qam_symbol<T, 3>(re, im, scale, llr);
  }
}

}  // namespace ddb
