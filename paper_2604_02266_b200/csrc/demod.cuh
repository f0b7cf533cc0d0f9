// Gray-QAM hard decisions and max-log LLRs on the reference's constellations
// (grid.py:98-154): label bits are MSB first, even bit positions drive I and
// odd ones Q; per axis the Gray PAM levels follow TS 38.211 in the recursive
// form of grid.py:98-109,
//     level(c0..c_{ba-1}) = (1 - 2 c0) * mag,  mag = 2^{ba-m} - (1 - 2 c_m) mag'
// with unit mean symbol energy (norm sqrt(2 (4^ba - 1) / 3): sqrt2, sqrt10,
// sqrt42).  ba = 1, 2 reproduce qpsk / qam16 exactly; ba = 3 (64-QAM) is the
// build extension the north star asks for (the reference rejects qam64,
// tests/test_grid.py:85-87), so its parity is pinned only through the
// LLR-sign == hard-decision identity.
//
// Nearest-point decisions for a separable Gray grid reduce to a per-axis
// argmin; taking the lowest axis index on ties reproduces the lowest-label
// tie rule of hard_demod (grid.py:172-183).
#pragma once

#include "common.cuh"

namespace ddb {

__device__ __forceinline__ int qam_axis_level(int i, int ba) {
  int mag = 1;
  for (int m = ba - 1; m >= 1; --m) {
    const int cm = (i >> (ba - 1 - m)) & 1;
    mag = (1 << (ba - m)) - (1 - 2 * cm) * mag;
  }
  const int c0 = (i >> (ba - 1)) & 1;
  return (1 - 2 * c0) * mag;
}

// One axis: v is the normalised component.  Writes the axis index (bits MSB
// first) and, if llr != nullptr, ba LLRs with stride 2 (interleaved I/Q).
template <typename T>
__device__ __forceinline__ int qam_axis(T v, int ba, T inv_norm, T scale, float* llr) {
  T dmin1[3], dmin0[3];
#pragma unroll
  for (int m = 0; m < 3; ++m) { dmin1[m] = T(3.0e38); dmin0[m] = dmin1[m]; }
  int best = 0;
  T bestd = T(0);
  const int nlev = 1 << ba;
  for (int i = 0; i < nlev; ++i) {
    const T a = T(qam_axis_level(i, ba)) * inv_norm;
    const T d = (v - a) * (v - a);
    if (i == 0 || d < bestd) { bestd = d; best = i; }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      if (m < ba) {
        if ((i >> (ba - 1 - m)) & 1) dmin1[m] = d < dmin1[m] ? d : dmin1[m];
        else dmin0[m] = d < dmin0[m] ? d : dmin0[m];
      }
    }
  }
  if (llr) {
#pragma unroll
    for (int m = 0; m < 3; ++m)
      if (m < ba) llr[2 * m] = (float)((dmin1[m] - dmin0[m]) * scale);
  }
  return best;
}

// Returns the constellation label of x; writes bps LLRs to llr if non-null.
template <typename T>
__device__ __forceinline__ int qam_demod_symbol(T re, T im, int bps, T scale, float* llr) {
  const int ba = bps >> 1;
  const T norm2 = T(2) * T((1 << (2 * ba)) - 1) / T(3);
  const T inv_norm = T(1) / sqrt(norm2);
  const int ii = qam_axis<T>(re, ba, inv_norm, scale, llr);
  const int qi = qam_axis<T>(im, ba, inv_norm, scale, llr ? llr + 1 : nullptr);
  int label = 0;
  for (int m = 0; m < ba; ++m) {
    const int cm = (ii >> (ba - 1 - m)) & 1;
    const int dm = (qi >> (ba - 1 - m)) & 1;
    label |= cm << (bps - 1 - 2 * m);
    label |= dm << (bps - 2 - 2 * m);
  }
  return label;
}

}  // namespace ddb
