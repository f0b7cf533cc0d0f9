/*
 * ddb.h — C ABI of the B200-native SS-CGA delay-Doppler equalizer.
 *
 * Every entry point takes plain device pointers and sizes (no torch types),
 * is non-blocking on the caller's CUDA stream, allocates nothing on the hot
 * path, and returns a ddb_status; on failure ddb_last_error() returns a
 * thread-local human-readable message.
 *
 * Reference interface each entry point replaces (paths are relative to the
 * reference package, /root/reference/pkg/src/ddlink):
 *
 *   ddb_sscga_solve      equalize.py:43-77   cga_equalize(ch, y_dd, cfg)
 *                        (fused with grid.py:172-183 hard_demod, the
 *                        harness.py:198 bit-error count, and the build-defined
 *                        max-log LLR soft demod that north_star adds)
 *   ddb_ss_apply         sparse.py:147-160   ss_mvm / ss_mvm_hermitian, matrix-free
 *   ddb_build_tables     sparse.py:124-144   build_ss_channel (+ forward_index 91-96,
 *                                            inverse_index 99-104, coefficient 107-121)
 *   ddb_ss_mvm_tables    sparse.py:147-160   ss_mvm / ss_mvm_hermitian on explicit tables
 *   ddb_hard_demod       grid.py:172-183     hard_demod (nearest point, lowest label on ties)
 *   ddb_qam_demod        grid.py:98-183      Gray-QAM slicer + max-log LLR (build-defined)
 *   ddb_dzt              zak.py:50-55        dzt_gemm (kernel of zak.py:33-47 or caller's),
 *                        fused with pilot.py:40-49 estimate_heff (twist of pilot.py:29-37)
 *   ddb_estimate_heff    pilot.py:40-49      estimate_heff on a DD frame
 *   ddb_detect_paths     sparse.py:69-88     detect_paths (strict relative threshold,
 *                                            stable descending-magnitude order)
 *   ddb_paths_csr        harness.py:159-163  taps -> build_ss_channel's input, batched as CSR
 *   ddb_dzt + INVERSE    zak.py:14-21        idzt (transmit side, frame synthesis)
 *   ddb_modulate         grid.py:157-169     modulate (labels -> constellation points)
 *   ddb_apply_channel    channel.py:95-103   apply_channel (delay shift + Doppler ramp)
 *   ddb_add_awgn         channel.py:106-119  add_awgn (own counter-based RNG)
 *   ddb_threshold_frame  sparse.py:163-169   threshold_frame (dense LMMSE baseline)
 *   ddb_build_dense_hdd  sparse.py:172-206   build_dense_hdd (dense LMMSE baseline)
 *
 * Layouts (identical to the reference's numpy layouts):
 *   complex values are interleaved (re, im) of the problem dtype;
 *   DD vectors are column-major flattened frames, q = l*M + k (grid.py:86-95);
 *   per-frame paths are CSR: path_offsets[b] .. path_offsets[b+1].
 */
#ifndef DDB_H
#define DDB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDB_ABI_VERSION 3

typedef enum {
  DDB_OK = 0,
  DDB_ERR_INVALID = 1,     /* bad argument (null pointer, negative size, ...)  */
  DDB_ERR_SHAPE = 2,       /* grid geometry rejected (odd M/N, too small, ...)  */
  DDB_ERR_UNSUPPORTED = 3, /* valid request outside what the build supports    */
  DDB_ERR_CUDA = 4,        /* CUDA runtime / launch failure                      */
  DDB_ERR_WORKSPACE = 5    /* workspace missing or too small                     */
} ddb_status;

typedef enum { DDB_F32 = 0, DDB_F64 = 1 } ddb_dtype;

/* frame status bits written to ddb_sscga_outputs.status */
#define DDB_FRAME_EMPTY_CHANNEL 0x1u /* P == 0: EmptyChannel (sparse.py:23-24, 126-127) */
#define DDB_FRAME_EXACT_CONVERGED 0x2u /* curvature exactly zero (equalize.py:64-67) */

/* One batch of independent frames sharing one grid.  All pointers are device
 * pointers.  Replaces the (ch, y_dd, cfg) triple of cga_equalize
 * (equalize.py:43): ch.paths -> CSR path arrays, y_dd -> y row, cfg.lam -> lam,
 * cfg.iterations -> iterations. */
typedef struct {
  int32_t batch;                /* number of frames B (>= 0)                      */
  int32_t M, N;                 /* grid (grid.py:14-31): even, >= 2                */
  int32_t iterations;           /* fixed CG iteration count Xi (>= 1)              */
  int32_t dtype;                /* ddb_dtype of y, gains, lam, x, c_norm           */
  const int32_t* path_offsets;  /* [B+1] CSR offsets into the path arrays          */
  const int32_t* path_k;        /* [n_paths] absolute delay index k_p in [0, M)    */
  const int32_t* path_l;        /* [n_paths] absolute Doppler index l_p in [0, N)  */
  const void* path_gain;        /* [n_paths] complex gain h_p                      */
  const void* y;                /* [B, M*N] complex received DD vector             */
  const void* lam;              /* [B] real ridge term (1/SNR, 0 = none)           */
} ddb_sscga_problem;

typedef struct {
  void* x;                  /* [B, M*N] complex equalized symbols (required)        */
  void* c_norm;             /* [B, iterations+1] real residual trace, or NULL;
                               entries past iterations_done are written as 0     */
  int32_t* iterations_done; /* [B] completed iterations (= len(c_norm)-1), or NULL   */
  uint8_t* status;          /* [B] DDB_FRAME_* bits, or NULL                        */
  void* snapshots;          /* [B, iterations, M*N] complex x after each iteration
                               (CgaConfig.profile, equalize.py:74-76), or NULL   */
  /* fused demod epilogue; bits_per_symbol == 0 disables it */
  int32_t bits_per_symbol;  /* 0, 2 (QPSK), 4 (16-QAM), 6 (64-QAM, build extension) */
  uint8_t* labels;          /* [B, M*N] hard-decision labels (bits MSB first), or NULL */
  float* llr;               /* [B, M*N, bits] max-log LLRs (>0 favours bit 0), or NULL */
  const void* noise_var;    /* [B] real LLR noise variance, or NULL (-> lam; 1 if 0) */
  const uint8_t* tx_labels; /* [B, M*N] transmitted labels, or NULL                 */
  int32_t* bit_errors;      /* [B] Hamming distance rx vs tx bits (needs tx_labels) */
  int32_t tx_labels_packed; /* 1: tx_labels carry bits_per_symbol bits per symbol,
                               LSB-first within bytes ([B, M*N*bps/8] bytes; bps 2 or 4),
                               0: one byte per symbol                              */
} ddb_sscga_outputs;

/* Launch plan chosen for a grid/dtype (exposed for tests and tooling). */
typedef struct {
  int32_t cluster;           /* CTAs per frame (thread-block cluster size)          */
  int32_t cols_per_cta;      /* Doppler columns owned by each CTA (N / cluster)     */
  int32_t cols_per_thread;   /* columns per thread (each thread owns one delay row) */
  int32_t threads;           /* threads per CTA                                     */
  int32_t smem_bytes;        /* dynamic shared memory per CTA                       */
  int32_t ctas_per_sm;       /* occupancy reported by the CUDA runtime (0 on CPU)   */
  int32_t halo_rows;         /* quasi-periodic extension rows kept around c and u   */
  int32_t kernel;            /* 0: row-slice kernel, 1: TMEM-operand kernel (fp32),
                                2: workspace-backed kernels (grids beyond a cluster) */
  int32_t rows_per_thread;   /* delay rows per thread (TMEM-operand kernel), else 1 */
} ddb_plan;

/* ---- library ------------------------------------------------------------ */
int32_t ddb_abi_version(void);
const char* ddb_last_error(void);
const char* ddb_build_info(void);

/* ---- planning / workspace ----------------------------------------------- */
int32_t ddb_sscga_plan(int32_t M, int32_t N, int32_t dtype, ddb_plan* out);
/* Bytes of device workspace ddb_sscga_solve needs for this problem: 0 for the
 * fused kernels (all CG state on chip); for grids beyond a 16-CTA cluster's
 * on-chip memory (e.g. the paper's 16384 x 32) the c, u, p vectors of every
 * frame plus per-block partials.  Pass it as `workspace` (DDB_ERR_WORKSPACE
 * if missing or too small). */
size_t ddb_sscga_workspace_bytes(const ddb_sscga_problem* prob);

/* ---- fused solve: coefficients on the fly + fixed-Xi CG + demod ---------- */
int32_t ddb_sscga_solve(const ddb_sscga_problem* prob, const ddb_sscga_outputs* out,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---- matrix-free operator: out = H v (hermitian=0) or H^H v (hermitian=1),
 *      batched over prob->batch frames; v is prob->y.  (sparse.py:147-160) */
int32_t ddb_ss_apply(const ddb_sscga_problem* prob, void* out, int32_t hermitian,
                     void* stream);

/* ---- table materialisation, fp64 only (sparse.py:124-144):
 *      fwd_coef/herm_coef complex128 [P, MN], fwd_col/herm_row int32 [P, MN] */
int32_t ddb_build_tables(int32_t M, int32_t N, int32_t n_paths, const int32_t* path_k,
                         const int32_t* path_l, const void* path_gain, void* fwd_coef,
                         int32_t* fwd_col, void* herm_coef, int32_t* herm_row,
                         void* stream);

/* ---- table-driven MVM, fp64 (sparse.py:147-160):
 *      u[q] = sum_p coef[p, q] * v[index[p, q]] */
int32_t ddb_ss_mvm_tables(int32_t size, int32_t n_paths, const void* coef,
                          const int32_t* index, const void* v, void* u, void* stream);

/* ---- nearest-point hard demod over an arbitrary constellation table
 *      (grid.py:172-183); ties go to the lowest label.  x, points in dtype. */
int32_t ddb_hard_demod(int64_t count, int32_t dtype, const void* x, const void* points,
                       int32_t n_points, int32_t* labels, void* stream);

/* ---- Gray-QAM slicer + max-log LLR on the reference's constellations
 *      (grid.py:98-154; 64-QAM is a build extension).  x is complex dtype
 *      [count]; noise_var is a scalar; labels/llr may be NULL. */
int32_t ddb_qam_demod(int64_t count, int32_t dtype, const void* x, int32_t bits_per_symbol,
                      double noise_var, uint8_t* labels, float* llr, void* stream);

/* ---- path detection (sparse.py:69-88), fp64: heff complex128 [B, M, N]
 *      (row-major k, l as the reference's (M, N) frame).  Writes per-frame
 *      counts and up to max_paths taps per frame in descending |h| order
 *      (stable w.r.t. row-major position).  count[b] > max_paths means the
 *      frame was truncated. */
int32_t ddb_detect_paths(int32_t batch, int32_t M, int32_t N, const void* heff, double theta,
                         int32_t max_paths, int32_t* count, int32_t* path_k,
                         int32_t* path_l, void* path_gain, void* stream);

/* ---- detected taps -> the solver's CSR, on the device: count [B] and the
 *      ranked rows [B, max_paths] of ddb_detect_paths become path_offsets
 *      [B+1] (exclusive scan of the stored rows, clamp(count, 0, max_paths))
 *      and csr_k / csr_l / csr_gain (gain in `dtype`), each sized for
 *      B * max_paths.
 *      stats [3] receives the minimum and maximum count (a negative minimum:
 *      a frame overflowed the candidate list; maximum > max_paths: truncated)
 *      and the number of rows stored, so a caller checks and sizes the batch
 *      with one 12-byte read. */
int32_t ddb_paths_csr(int32_t batch, int32_t max_paths, const int32_t* count, const int32_t* path_k,
                      const int32_t* path_l, const void* path_gain, int32_t dtype, int32_t* path_offsets,
                      int32_t* csr_k, int32_t* csr_l, void* csr_gain, int32_t* stats, void* stream);

/* ---- receiver front end.
 *      ddb_dzt: y_time complex [B, M*N] received samples (time index k + i*M,
 *      grid.py check_signal); kernel complex [N, N] row-major (i, l) or NULL for
 *      build_zak_kernel(N) = e^{-j2pi i l/N}/sqrt(N) (zak.py:33-47); out complex
 *      [B, M*N].  flags: DDB_DZT_COLMAJOR writes the flattened vector
 *      q = l*M + k (grid.py:86-95), else the (M, N) frame row-major as dzt_gemm
 *      returns it; DDB_DZT_PILOT also multiplies by the twist kernel
 *      e^{-j2pi K0 (l-L0)/(MN)} and divides by `amplitude` (estimate_heff). */
#define DDB_DZT_COLMAJOR 1
#define DDB_DZT_PILOT 2
#define DDB_DZT_INPUT_F32 4  /* dtype f64 with complex64 y_time (fp64 arithmetic on
                                single-precision samples); default kernel, power-of-two N */
#define DDB_DZT_INVERSE 8    /* idzt (zak.py:14-21): x[k + nM] = (1/sqrt N) sum_l X[k,l] e^{+j2pi n l/N};
                                y_time is then the flattened DD vector q = l*M + k and out the
                                time samples (needs DDB_DZT_COLMAJOR, the default kernel) */
int32_t ddb_dzt(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* y_time, const void* kernel,
                int32_t flags, double amplitude, void* out, void* stream);

/* ---- estimate_heff (pilot.py:40-49) on DD frames: heff = y_dd * twist / amplitude
 *      elementwise over `count` complex values of the dtype (amplitude > 0). */
int32_t ddb_estimate_heff(int64_t count, int32_t dtype, const void* y_dd, const void* twist, double amplitude,
                          void* heff, void* stream);

/* ---- host-buffer round trips for one frame (the numpy drop-ins the
 *      reference calls once per packet, harness.py:156-159): every pointer is
 *      HOST memory (complex128 = interleaved double pairs); one call copies the
 *      inputs into a per-thread device scratch, runs the kernel above and
 *      copies the result back, with one stream synchronisation.  The
 *      reference's receive path pays one such round trip per function.
 *      ddb_host_dzt            zak.py:50-55   y [M*N] -> out (M, N) row-major;
 *                                             kernel [N, N] or NULL (default)
 *      ddb_host_estimate_heff  pilot.py:40-49 y_dd, twist [count] -> heff
 *      ddb_host_detect_paths   sparse.py:69-88 heff (M, N) -> *count taps
 *                                             (k, l, gain) ranked; capacity
 *                                             max_paths (M*N returns all) */
int32_t ddb_host_dzt(int32_t M, int32_t N, const void* y_time, const void* kernel, void* out);
int32_t ddb_host_estimate_heff(int64_t count, const void* y_dd, const void* twist, double amplitude, void* heff);
int32_t ddb_host_detect_paths(int32_t M, int32_t N, const void* heff, double theta, int32_t max_paths,
                              int32_t* count, int32_t* path_k, int32_t* path_l, void* path_gain);

/* ---- frame synthesis on the device: the transmit
 *      side and channel of one packet (harness.py:141-149) for a batch.
 *      ddb_modulate        grid.py:157-169  labels [count] (bits MSB first,
 *                          as `groups @ weights`) -> points of
 *                          make_constellation (grid.py:126-154), complex dtype.
 *      ddb_apply_channel   channel.py:95-103 on time-domain frames x [B, M*N]:
 *                          y[i] = sum_p h_p x[(i - k_p) mod MN]
 *                                 e^{j2pi nu_p (i / bandwidth - tau_p)}
 *                          paths as CSR (path_offsets [B+1]; delay_bin int32,
 *                          doppler_hz / delay_s float64, gain complex dtype);
 *                          phases in fp64.  y must not alias x.
 *      ddb_add_awgn        channel.py:106-119: out = y + sigma/sqrt(2) (n1 + j n2),
 *                          sigma^2 = mean_frame |y|^2 / 10^(snr_db/10), per frame of
 *                          frame_len samples; counter-based normals (Philox4x32-10,
 *                          seed) -- the reference's numpy stream is not reproduced.
 *                          snr_db = +inf copies (the noiseless sentinel).
 *                          frame_power: device float64 [batch] scratch (receives
 *                          the per-frame mean power).  out may alias y. */
int32_t ddb_modulate(int64_t count, int32_t dtype, const uint8_t* labels, int32_t bits_per_symbol, void* out,
                     void* stream);
int32_t ddb_apply_channel(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* x,
                          const int32_t* path_offsets, const int32_t* delay_bin, const double* doppler_hz,
                          const double* delay_s, const void* gain, double bandwidth_hz, void* y, void* stream);
int32_t ddb_add_awgn(int32_t batch, int64_t frame_len, int32_t dtype, const void* y, double snr_db, uint64_t seed,
                     double* frame_power, void* out, void* stream);

/* ---- dense LMMSE baseline, MN <= 4096.
 *      ddb_threshold_frame  sparse.py:163-169: zero every bin of heff [B, M, N]
 *                           (row-major (M, N) frames) with |h| <= theta * peak
 *                           (peak 0: copy).
 *      ddb_build_dense_hdd  sparse.py:172-206: H [B, MN, MN] row-major (row
 *                           q' = l'M + k', column q = lM + k) from heff frames.
 *      The Gram matrix and Cholesky solve of lmmse_equalize (equalize.py:80-94)
 *      are library calls (cuBLAS / cuSOLVER) in the host mirror. */
int32_t ddb_threshold_frame(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* heff, double theta,
                            void* out, void* stream);
int32_t ddb_build_dense_hdd(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* heff, void* H,
                            void* stream);

/* ---- measurement helper (not a reference interface): FP32 FMA throughput
 *      probe used by bench.py to state the measured FP32 roofline.  Launches
 *      blocks x 256 threads, each doing iters x 256 FMAs (mode 0: FFMA,
 *      mode 1: packed FFMA2, mode 2: DFMA, the fp64 rate).  scratch: device
 *      float[blocks]. */
int32_t ddb_probe_fp32(int32_t mode, int32_t blocks, int32_t iters, float* scratch, void* stream);

/* ---- measurement helper (not a reference interface): ddb_sscga_solve with
 *      clock64 phase accounting on thread 0 of every CTA.  phase_cycles:
 *      device int64 [4736][12], zero-initialised by the caller; row = CTA,
 *      columns = setup, arrive, mvm_local, wait, mvm_remote, read, step1,
 *      step3, epilogue, tail. */
int32_t ddb_sscga_profile_phases(const ddb_sscga_problem* prob, const ddb_sscga_outputs* out,
                                 long long* phase_cycles, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DDB_H */
