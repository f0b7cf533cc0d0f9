// Frame synthesis on the device: the transmit side and
// the channel of one packet of harness.py:141-149 for a whole batch, so the
// end-to-end receiver can be fed at HBM speed instead of through PCIe.
//
//   modulate       grid.py:157-169   labels -> Gray-QAM points (grid.py:126-154)
//   idzt           zak.py:14-21      ddb_dzt with DDB_DZT_INVERSE (frontend.cu)
//   apply_channel  channel.py:95-103 y[i] = sum_p h_p x[(i - k_p) mod MN]
//                                          e^{j 2 pi nu_p (i / B - tau_p)}
//   add_awgn       channel.py:106-119 y + sigma/sqrt(2) (n1 + j n2),
//                                    sigma^2 = mean|y|^2 / 10^(snr/10)
//
// apply_channel is a gather over P circular shifts of the frame with a
// fractional-Doppler phase ramp per path: the ramp's phase is formed in fp64
// from the continuous delay and Doppler (as numpy does), reduced to one turn
// and evaluated with sincospi, so fp64 output matches the reference to
// rounding.  Roofline: HBM, 8 (fp32) / 16 (fp64) bytes read and written per
// sample; the P shifted reads of a tile hit L1/L2.
//
// AWGN draws are counter-based (Philox4x32-10 keyed by the seed, counter =
// (sample pair, frame)), so a batch is reproducible for a seed and any launch
// shape.  The reference's numpy stream is not reproduced:
// parity for the noise is distributional.  The per-frame signal power is a
// fixed-order reduction (deterministic).
#include "common.cuh"
#include "demod.cuh"
#include "internal.h"

namespace ddb {

namespace {

constexpr int kChThreads = 256;
constexpr int kChPerThread = 8;     // consecutive samples per thread
constexpr int kChPathCap = 64;      // paths staged in shared memory per frame

template <typename T, int BA>
__global__ void modulate_kernel(long long count, const uint8_t* __restrict__ labels, Vec<T>* __restrict__ out) {
  constexpr int MASK = (1 << BA) - 1;
  const T inv = T(1.0 / qam_norm<BA>());
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = labels[i];
    int ii = 0, qi = 0;  // even label bits (MSB first) drive I, odd ones Q (grid.py:139-146)
#pragma unroll
    for (int m = 0; m < BA; ++m) {
      ii = (ii << 1) | ((s >> (2 * BA - 1 - 2 * m)) & 1);
      qi = (qi << 1) | ((s >> (2 * BA - 2 - 2 * m)) & 1);
    }
    out[i] = cmake<Vec<T>>(T(qam_level<BA>(ii & MASK)) * inv, T(qam_level<BA>(qi & MASK)) * inv);
  }
}

struct ChPath {
  double nu, tau;  // Doppler (Hz), delay (s)
  double2 h;       // gain
  double2 step;    // e^{j 2 pi nu / B}: the ramp's advance per sample
  int k;           // delay bin
  int pad;
};

// One CTA per (frame, tile of kChThreads * kChPerThread samples).  Each thread
// takes kChPerThread consecutive samples: the ramp is evaluated exactly
// (sincospi of the phase reduced to one turn) at the first and advanced by
// one fp64 complex multiply per sample after it.
template <typename T>
__global__ void __launch_bounds__(kChThreads) apply_channel_kernel(int MN, double inv_bw, const Vec<T>* __restrict__ x,
                                                                 const int* __restrict__ off,
                                                                 const int* __restrict__ kbin,
                                                                 const double* __restrict__ nu,
                                                                 const double* __restrict__ tau,
                                                                 const Vec<T>* __restrict__ gain,
                                                                 Vec<T>* __restrict__ y) {
  using V = Vec<T>;
  __shared__ ChPath ps[kChPathCap];
  const int f = blockIdx.y;
  const int p0 = off[f], P = off[f + 1] - p0;
  const V* xf = x + (size_t)f * MN;
  V* yf = y + (size_t)f * MN;
  const int i0 = (blockIdx.x * kChThreads + threadIdx.x) * kChPerThread;
  double2 acc[kChPerThread];
#pragma unroll
  for (int j = 0; j < kChPerThread; ++j) acc[j] = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < P; c0 += kChPathCap) {
    const int n = min(kChPathCap, P - c0);
    __syncthreads();
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const V g = gain[p0 + c0 + p];
      const double v = nu[p0 + c0 + p];
      double ds = v * inv_bw, ss, cs;
      ds -= rint(ds);
      sincospi(2.0 * ds, &ss, &cs);
      ps[p] = ChPath{v, tau[p0 + c0 + p], make_double2(g.x, g.y), make_double2(cs, ss),
                     mod_pos(kbin[p0 + c0 + p], MN), 0};
    }
    __syncthreads();
    if (i0 >= MN) continue;
    for (int p = 0; p < n; ++p) {
      const ChPath e = ps[p];
      double ph = e.nu * ((double)i0 * inv_bw - e.tau);  // turns: nu (i / B - tau)
      ph -= rint(ph);
      double s, c;
      sincospi(2.0 * ph, &s, &c);
      double2 w = make_double2(e.h.x * c - e.h.y * s, e.h.x * s + e.h.y * c);  // h e^{j 2 pi ph}
      int src = i0 - e.k;
      if (src < 0) src += MN;
#pragma unroll
      for (int j = 0; j < kChPerThread; ++j) {
        if (i0 + j >= MN) break;
        const V v = xf[src];
        acc[j].x += w.x * (double)v.x - w.y * (double)v.y;
        acc[j].y += w.x * (double)v.y + w.y * (double)v.x;
        w = make_double2(w.x * e.step.x - w.y * e.step.y, w.x * e.step.y + w.y * e.step.x);
        if (++src == MN) src = 0;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kChPerThread; ++j)
    if (i0 + j < MN) yf[i0 + j] = cmake<V>(T(acc[j].x), T(acc[j].y));
}

// Mean power of each frame: fixed-order block reduction in fp64.
template <typename T>
__global__ void __launch_bounds__(kChThreads) frame_power_kernel(long long L, const Vec<T>* __restrict__ y,
                                                               double* __restrict__ power) {
  __shared__ double part[kChThreads / 32];
  const Vec<T>* yf = y + (size_t)blockIdx.x * L;
  double s = 0.0;
  for (long long i = threadIdx.x; i < L; i += blockDim.x) {
    const Vec<T> v = yf[i];
    s += (double)v.x * v.x + (double)v.y * v.y;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kChThreads / 32; ++w) t += part[w];
    power[blockIdx.x] = t / (double)L;
  }
}

// Philox4x32-10 (Salmon et al., SC'11).
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// Two standard normals from two 32-bit words (Box-Muller, u1 in (0, 1]).
__device__ __forceinline__ double2 box_muller(uint32_t a, uint32_t b) {
  const double u1 = ((double)a + 1.0) * 2.3283064365386963e-10;
  const double u2 = (double)b * 2.3283064365386963e-10;
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(r * c, r * s);
}

// y + sigma/sqrt(2) (n1 + j n2) per frame; each thread draws one Philox block
// (4 words) for a pair of samples.
template <typename T>
__global__ void awgn_kernel(long long L, const Vec<T>* __restrict__ y, const double* __restrict__ power,
                            double inv_snr, uint2 key, Vec<T>* __restrict__ out) {
  const int f = blockIdx.y;
  const double sc = sqrt(power[f] * inv_snr) * 0.70710678118654752;
  const Vec<T>* yf = y + (size_t)f * L;
  Vec<T>* of = out + (size_t)f * L;
  for (long long pr = blockIdx.x * (long long)blockDim.x + threadIdx.x; 2 * pr < L;
       pr += (long long)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32(make_uint4((uint32_t)pr, (uint32_t)(pr >> 32), (uint32_t)f, 0x5eedu), key);
    const double2 n0 = box_muller(w.x, w.y), n1 = box_muller(w.z, w.w);
    const long long i = 2 * pr;
    Vec<T> a = yf[i];
    of[i] = cmake<Vec<T>>(T((double)a.x + sc * n0.x), T((double)a.y + sc * n0.y));
    if (i + 1 < L) {
      a = yf[i + 1];
      of[i + 1] = cmake<Vec<T>>(T((double)a.x + sc * n1.x), T((double)a.y + sc * n1.y));
    }
  }
}

int grid_1d(long long n, int per_block) {
  const long long b = (n + per_block - 1) / per_block;
  return (int)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace

cudaError_t launch_modulate(int dtype_f64, long long count, const uint8_t* labels, int bps, void* out,
                            cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const int g = grid_1d(count, 256);
  if (dtype_f64) {
    switch (bps) {
      case 2: modulate_kernel<double, 1><<<g, 256, 0, st>>>(count, labels, (double2*)out); break;
      case 4: modulate_kernel<double, 2><<<g, 256, 0, st>>>(count, labels, (double2*)out); break;
      default: modulate_kernel<double, 3><<<g, 256, 0, st>>>(count, labels, (double2*)out); break;
    }
  } else {
    switch (bps) {
      case 2: modulate_kernel<float, 1><<<g, 256, 0, st>>>(count, labels, (float2*)out); break;
      case 4: modulate_kernel<float, 2><<<g, 256, 0, st>>>(count, labels, (float2*)out); break;
      default: modulate_kernel<float, 3><<<g, 256, 0, st>>>(count, labels, (float2*)out); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_apply_channel(int dtype_f64, int B, int MN, double bandwidth, const void* x, const int* off,
                                 const int* kbin, const double* nu, const double* tau, const void* gain, void* y,
                                 cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  dim3 grid((MN + kChThreads * kChPerThread - 1) / (kChThreads * kChPerThread), B);
  if (dtype_f64)
    apply_channel_kernel<double><<<grid, kChThreads, 0, st>>>(MN, 1.0 / bandwidth, (const double2*)x, off, kbin, nu,
                                                              tau, (const double2*)gain, (double2*)y);
  else
    apply_channel_kernel<float><<<grid, kChThreads, 0, st>>>(MN, 1.0 / bandwidth, (const float2*)x, off, kbin, nu,
                                                             tau, (const float2*)gain, (float2*)y);
  return cudaGetLastError();
}

cudaError_t launch_add_awgn(int dtype_f64, int B, long long L, const void* y, double snr_db, unsigned long long seed,
                            double* power, void* out, cudaStream_t st) {
  if (B == 0 || L == 0) return cudaSuccess;
  const double inv_snr = 1.0 / pow(10.0, snr_db / 10.0);
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  dim3 grid(grid_1d((L + 1) / 2, 256) / 8 + 1, B);
  if (dtype_f64) {
    frame_power_kernel<double><<<B, kChThreads, 0, st>>>(L, (const double2*)y, power);
    awgn_kernel<double><<<grid, 256, 0, st>>>(L, (const double2*)y, power, inv_snr, key, (double2*)out);
  } else {
    frame_power_kernel<float><<<B, kChThreads, 0, st>>>(L, (const float2*)y, power);
    awgn_kernel<float><<<grid, 256, 0, st>>>(L, (const float2*)y, power, inv_snr, key, (float2*)out);
  }
  return cudaGetLastError();
}

}  // namespace ddb
