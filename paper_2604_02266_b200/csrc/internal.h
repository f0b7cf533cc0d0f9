// Internal (non-ABI) declarations shared by the ddb translation units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ddb {

// Everything the fused SS-CGA kernel needs for one batch (device pointers).
struct SolveArgs {
  int B, M, N, MN, K0, L0, iters;
  int C;              // cluster size (CTAs per frame)
  int Lcta;           // Doppler columns per CTA = N / C
  int active_threads; // M * (Lcta / LC); blockDim is this rounded up to 32
  int n_clusters;     // persistent clusters in the grid
  int S;              // rows of the extended p/u buffers = M + H
  int RS;             // row stride in complex elements (row_stride())
  int H;              // quasi-periodic halo capacity (rows) of p/u
  int TL, TH;         // two-level W_MN twiddle tables: e = hi * TL + lo
  int pcap;           // per-frame tap table capacity in shared memory
  int tcols;          // TMEM columns allocated per CTA (x lives in TMEM)
  // TMEM-operand kernel (sscga_tm.cu) only
  int G;              // delay rows per TMEM lane segment (M / segments per column)
  int WQ;             // warps per TMEM lane quarter (threads = 128 WQ)
  int CS;             // column stride (complex elements) of the column-major extended slices
  int stream_y;       // 1: a frame's y arrives by cp.async.bulk into the u slice during the previous frame
  int split;          // 1: lean frames go to the lean instantiation, the rest to the general one; 0: general only
  int gd;             // TMEM kernel: ghost depth (boundary columns per side pushed to the neighbours; 0: none)
  const int* off;
  const int* pk;
  const int* pl;
  const void* ph;
  const void* y;
  const void* lam;
  void* x;
  void* cnorm;
  int* itdone;
  uint8_t* status;
  void* snaps;
  int bps;
  uint8_t* labels;
  float* llr;
  const void* nvar;
  const uint8_t* txl;
  int txpk;          // tx labels packed bps bits per symbol (bps 2 or 4)
  int* berr;
  long long* prof;  // optional per-CTA phase cycle counters [gridDim.x][kProfPhases]
};

constexpr int kProfPhases = 12;
constexpr int kProfWarpBase = 4096;  // per-warp timers of measurement builds: prof[4096 + (cta * 16 + warp) * 8 + k]

struct LaunchShape {
  int cluster, lcta, lc, threads, smem, halo, tl, th, pcap, tcols;
  int kind;        // 0: row-slice kernel (sscga.cu), 1: TMEM-operand kernel (sscga_tm.cu),
                   // 2: workspace-backed kernels (sscga_global.cu)
  int g, wq, rows, cs;  // kind 1: segment rows, warps per lane quarter, rows per thread, column stride
  int gd = 0;           // kind 1: ghost depth (SolveArgs::gd)
};
// Ghost columns (TMEM kernel): clusters of at least this many CTAs, up to this
// many columns per side.
constexpr int kGhostMinC = 4;
constexpr int kGhostMaxDepth = 4;

// TMEM columns for the thread-private runs of x, p and the own-element copies
// of c and u: (warps per lane quarter) x 4 runs x (32-bit words per run),
// rounded to the allocator's power-of-two granularity (>= 32).
constexpr int sscga_tmem_cols(int threads, int lc, int elem_bytes) {
  int need = ((threads / 32 + 3) / 4) * 4 * lc * 2 * elem_bytes / 4;
  int c = 32;
  while (c < need) c *= 2;
  return c;
}

// Thread ceiling of the fused kernel instantiation (its __launch_bounds__):
// per-thread column runs of >= 32 bytes of real data need > 64 registers,
// so those instantiations cap at 512 threads.
constexpr int sscga_max_threads(int elem_bytes, int lc) { return elem_bytes * lc >= 32 ? 512 : 1024; }

// Row stride (complex elements) of the on-chip row-major slices: the Lcta
// columns padded so that a row is a multiple of 16 bytes and == 16 (mod 32),
// which makes 8 consecutive rows hit 8 distinct 16-byte bank groups (LDS.128
// conflict-free when consecutive lanes own consecutive rows).
__host__ __device__ constexpr int row_stride(int lcta, int elem_bytes) {
  return (((lcta * 2 * elem_bytes + 31) / 32) * 32 + 16) / (2 * elem_bytes);
}

// Shared-memory layout of the fused kernel (byte offsets, 16-byte aligned).
struct SmemLayout {
  size_t p, u, x, tlo, thi, tw, ptab, red, q, total;  // q: the TMEM kernel's frame list
  size_t gh = 0, ghmb = 0;  // TMEM kernel, clusters: ghost columns of c and u and their mbarriers
};
SmemLayout sscga_layout(int M, int N, int C, int elem_bytes, int H, int TL, int TH, int pcap);
void twiddle_split(int MN, int* TL, int* TH);

template <typename T>
cudaError_t launch_sscga(SolveArgs a, const LaunchShape& s, cudaStream_t st);

// TMEM-operand kernel (fp32): layout of its shared memory and launch.
SmemLayout sscga_tm_layout(int M, int Lcta, int N, int CS, int TL, int TH, int pcap, int gd);
cudaError_t launch_sscga_tm(SolveArgs a, const LaunchShape& s, cudaStream_t st);
cudaError_t sscga_tm_occupancy(const LaunchShape& s, int* ctas_per_sm);

// Workspace-backed path for grids beyond a cluster's on-chip memory (sscga_global.cu).
size_t align_up(size_t v, size_t a);
size_t sscga_global_workspace(int dtype_f64, int B, int M, int N);
template <typename T>
cudaError_t launch_sscga_global(const SolveArgs& a, void* workspace, cudaStream_t st);

template <typename T>
cudaError_t sscga_occupancy(const LaunchShape& s, int* ctas_per_sm);

template <typename T>
cudaError_t launch_ss_apply(int B, int M, int N, const int* off, const int* pk, const int* pl,
                            const void* ph, const void* v, void* out, bool herm, cudaStream_t st);

cudaError_t launch_build_tables(int M, int N, int P, const int* pk, const int* pl, const void* ph,
                                void* fwd_coef, int* fwd_col, void* herm_coef, int* herm_row,
                                cudaStream_t st);
cudaError_t launch_mvm_tables(int size, int P, const void* coef, const int* idx, const void* v,
                              void* u, cudaStream_t st);
template <typename T>
cudaError_t launch_hard_demod(long long count, const void* x, const void* pts, int npts,
                              int* labels, cudaStream_t st);
template <typename T>
cudaError_t launch_qam_demod(long long count, const void* x, int bps, double nvar,
                             uint8_t* labels, float* llr, cudaStream_t st);
cudaError_t launch_detect_paths(int B, int M, int N, const void* heff, double theta,
                                int max_paths, int* count, int* pk, int* pl, void* ph,
                                cudaStream_t st);

// Receiver front end (frontend.cu): Zak transform (+ fused pilot estimate),
// elementwise pilot estimate on a DD frame.
cudaError_t launch_dzt(int dtype_f64, int B, int M, int N, const void* y, const void* kern, int colmajor, int pilot,
                       int inverse, double amp, void* out, cudaStream_t st);
cudaError_t launch_dzt_mixed(int B, int M, int N, const void* y, int colmajor, int pilot, double amp, void* out,
                             cudaStream_t st);
cudaError_t launch_estimate_heff(int dtype_f64, long long count, const void* ydd, const void* twist, double amp,
                                 void* heff, cudaStream_t st);

// FP32 FMA throughput probe: blocks x 256 threads x iters x 256 FMAs.
cudaError_t launch_modulate(int dtype_f64, long long count, const uint8_t* labels, int bps, void* out,
                            cudaStream_t st);
cudaError_t launch_apply_channel(int dtype_f64, int B, int MN, double bandwidth, const void* x, const int* off,
                                 const int* kbin, const double* nu, const double* tau, const void* gain, void* y,
                                 cudaStream_t st);
cudaError_t launch_add_awgn(int dtype_f64, int B, long long L, const void* y, double snr_db, unsigned long long seed,
                            double* power, void* out, cudaStream_t st);
cudaError_t launch_threshold_frame(int dtype_f64, int B, int MN, const void* heff, double theta, void* out,
                                   cudaStream_t st);
cudaError_t launch_build_dense(int dtype_f64, int B, int M, int N, const void* heff, void* H, cudaStream_t st);
cudaError_t launch_paths_csr(int B, int max_paths, const int* count, const int* pk, const int* pl, const void* ph,
                             int dtype_f64, int* off, int* k, int* l, void* g, int* stats, cudaStream_t st);
cudaError_t launch_fp32_probe(int mode, int blocks, int iters, float* out, cudaStream_t st);

}  // namespace ddb
