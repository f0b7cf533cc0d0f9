// C ABI (include/ddb.h): argument validation, launch planning, error state.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/ddb.h"
#include "internal.h"

#include <cmath>

namespace {

thread_local std::string g_err;

int32_t fail(int32_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int32_t cuda_fail(cudaError_t e, const char* where) {
  return fail(DDB_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

int32_t ok() {
  g_err.clear();
  return DDB_OK;
}

int32_t check_grid(int32_t M, int32_t N) {
  // GridConfig.__post_init__ (grid.py:23-29)
  if (M < 2 || N < 2) return fail(DDB_ERR_SHAPE, "grid must be at least 2x2, got (%d,%d)", M, N);
  if ((M & 1) || (N & 1))
    return fail(DDB_ERR_SHAPE, "M and N must be even so the pilot sits on a bin center, got (%d,%d)", M, N);
  if ((long long)M * N >= (1LL << 29)) return fail(DDB_ERR_UNSUPPORTED, "grid too large: M*N=%lld", (long long)M * N);
  return DDB_OK;
}

int smem_optin() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    return 232448;  // sm_100: 227 KiB opt-in per block
  }
  return v;
}

// TMEM-operand kernel (sscga_tm.cu, fp32): 128 TMEM lanes = Lcta columns x
// S segments of G = M / S delay rows, G <= 64 so that c | u | p | x fit the
// 512 lane columns; WQ warps per lane quarter, R = G / WQ rows per thread.
// The smallest cluster that fits (largest segment G: most d_l = 0 taps read
// TMEM); then the WQ that puts the most frames on an SM.  tcgen05 CTAs do
// co-reside (tools/ubench/resident.cu: 2 x 256 or 4 x 128 TMEM columns per
// SM) although the occupancy API reports 1, so a CTA of 128 or 256 threads
// whose shared memory is capped to its share of the SM runs 2-4 frames per SM
// (cfg1 5.4 -> 12.9, cfg2 13.0 -> 15.8 G symbols/s, profiles/r2_residency.md).
// Ties keep the larger CTA.  The halo then takes the rest of the CTA's share
// (at least min(M, 64) rows: the Veh-A delay spread is <= 39 bins at M = 512).
constexpr int kTmRegs128 = 96;  // sscga_tm.cu: __launch_bounds__(128, 5) for 128-thread plans
bool make_plan_tm(int32_t M, int32_t N, ddb::LaunchShape* s) {
  const char* env_k = getenv("DDB_KERNEL");
  if (env_k && env_k[0] == 'r') return false;  // DDB_KERNEL=row: force the row-slice kernel
  const int cap = smem_optin();
  const int pcap = 64;
  int TL = 0, TH = 0;
  ddb::twiddle_split(M * N, &TL, &TH);
  // delay shifts |d_k| <= M / 2 (sparse.py:35-37): a halo of M / 2 rows covers
  // every shift; 64 covers the Veh-A delay spread (<= 39 bins at M = 512)
  const int hmin = M / 2 < 64 ? M / 2 : 64;
  const char* env_c = getenv("DDB_PLAN_C");
  const char* env_wq = getenv("DDB_PLAN_WQ");
  const char* env_cap = getenv("DDB_PLAN_SMEM_CAP");
  const int cmin = env_c ? atoi(env_c) : 1;
  for (int C = 1; C <= 16; C *= 2) {
    if (N % C || C < cmin) continue;
    const int lcta = N / C;
    if (128 % lcta) continue;
    const int S = 128 / lcta;
    if (M % S) continue;
    const int G = M / S;
    if (G > 64 || G % 2) continue;
    auto cs_of = [&](int h) { int cs = M + 2 * h + 2; return cs % 4 == 2 ? cs : cs + 2; };
    // ghost columns (clusters of kGhostMinC+ CTAs): as deep as the shared memory allows
    // with the minimum halo (DDB_NO_GHOST: none)
    int gd = 0;
    auto smem_of = [&](int h) { return ddb::sscga_tm_layout(M, lcta, N, cs_of(h), TL, TH, pcap, gd).total; };
    if (C >= ddb::kGhostMinC && !getenv("DDB_NO_GHOST")) {
      gd = lcta < ddb::kGhostMaxDepth ? lcta : ddb::kGhostMaxDepth;
      while (gd > 0 && smem_of(hmin) > (size_t)cap) --gd;
    }
    if (smem_of(hmin) > (size_t)cap) continue;
    int tc = 32;
    while (tc < 8 * G) tc *= 2;
    int best_wq = 0, best_n = 0, best_h = 0;
    for (int w = 4; w >= 1; w /= 2) {
      if (G % w || (env_wq && atoi(env_wq) != w)) continue;
      const int r = G / w;
      if (r != 4 && r != 8 && r != 16) continue;
      const int threads = 128 * w;
      // frames per SM: TMEM columns, threads (<= 128 registers each), shared memory
      int n = 512 / tc;
      // registers per thread: 128 (the kernel's launch bounds), 96 for 128-thread
      // CTAs (their instantiations are bounded for five CTAs per SM)
      const int regs = threads == 128 ? kTmRegs128 : 128;
      if (65536 / (threads * regs) < n) n = 65536 / (threads * regs);
      int share = 0, h = 0;
      for (; n >= 1; --n) {
        share = 233472 / n - 1024;  // 228 KiB per SM, 1 KiB reserved per CTA
        if (share > cap) share = cap;
        if (env_cap && atoi(env_cap) < share) share = atoi(env_cap);
        if (smem_of(hmin) <= (size_t)share) break;
      }
      if (n < 1) continue;
      h = M;
      while (h > hmin && smem_of(h) > (size_t)share) h -= 2;
      if (n > best_n) { best_n = n; best_wq = w; best_h = h; }
    }
    if (!best_wq) continue;
    int h = best_h;
    if (const char* env_h = getenv("DDB_PLAN_H")) h = h < atoi(env_h) ? h : atoi(env_h);
    h &= ~1;
    s->kind = 1;
    s->cluster = C;
    s->lcta = lcta;
    s->lc = 1;
    s->g = G;
    s->wq = best_wq;
    s->rows = G / best_wq;
    s->threads = 128 * best_wq;
    s->halo = h;
    s->cs = cs_of(h);
    s->gd = gd;
    s->tl = TL;
    s->th = TH;
    s->pcap = pcap;
    s->tcols = tc;
    s->smem = (int)smem_of(h);
    // keep (CTAs per SM) x (TMEM columns per CTA) <= 512 so tcgen05.alloc never
    // waits on a co-resident CTA: pad the shared memory of small CTAs
    const int max_ctas = 512 / tc;
    int floor_smem = 233472 / (max_ctas + 1) - 1024 + 16;
    if (floor_smem > cap) floor_smem = cap;
    if (s->smem < floor_smem) s->smem = floor_smem;
    return true;
  }
  return false;
}

// Workspace-backed kernels (sscga_global.cu): any grid; the CG vectors live in
// a caller-provided workspace (ddb_sscga_workspace_bytes).
int32_t plan_global(int32_t M, int32_t N, ddb::LaunchShape* s) {
  *s = ddb::LaunchShape{};
  s->kind = 2;
  s->cluster = 1;
  s->lcta = N;
  s->lc = 1;
  s->threads = 256;
  ddb::twiddle_split(M * N, &s->tl, &s->th);
  return DDB_OK;
}

// Smallest cluster whose CTAs can hold their column slice of p, u and x in
// shared memory; then the widest per-thread column run that keeps at least
// 256 threads per CTA within the register file.
int32_t make_plan(int32_t M, int32_t N, int32_t dtype, ddb::LaunchShape* s) {
  *s = ddb::LaunchShape{};
  const char* env_k = getenv("DDB_KERNEL");
  if (env_k && env_k[0] == 'g') return plan_global(M, N, s);  // DDB_KERNEL=global (tests / A-B)
  if (dtype == DDB_F32 && make_plan_tm(M, N, s)) return DDB_OK;
  const int eb = dtype == DDB_F64 ? 8 : 4;
  const int cap = smem_optin();
  const int lcmax = dtype == DDB_F64 ? 8 : 16;
  const int pcap = 64;  // larger tap sets read their entries from global memory
  int TL = 0, TH = 0;
  ddb::twiddle_split(M * N, &TL, &TH);
  const int hmin = M < 64 ? M : 64;  // Veh-A delay spread is <= 39 bins at M = 512
  // tuning overrides (benchmarks only): DDB_PLAN_C = minimum cluster size,
  // DDB_PLAN_LC = columns per thread (ignored when it does not fit)
  const char* env_c = getenv("DDB_PLAN_C");
  const char* env_lc = getenv("DDB_PLAN_LC");
  const int cmin = env_c ? atoi(env_c) : 1;
  const int force_lc = env_lc ? atoi(env_lc) : 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int C = 1; C <= 16; C *= 2) {
      if (N % C || C < cmin) continue;
      const int lcta = N / C;
      const size_t base = ddb::sscga_layout(M, N, C, eb, 0, TL, TH, pcap).total;
      if (base > (size_t)cap) continue;
      long long h = (long long)(cap - base) / (2LL * lcta * 2 * eb);
      while (h > 0 && ddb::sscga_layout(M, N, C, eb, (int)h, TL, TH, pcap).total > (size_t)cap) --h;
      if (h > M) h = M;  // a delay shift spans at most M - 1 rows
      if (const char* env_h = getenv("DDB_PLAN_H")) h = h < atoi(env_h) ? h : atoi(env_h);
      if (pass == 0 && h < hmin) continue;
      const int target = M * lcta < 256 ? M * lcta : 256;
      int best = 0;
      for (int lc = lcmax; lc >= 1; lc /= 2) {
        if (lcta % lc) continue;
        const int active = M * (lcta / lc);
        const int threads = (active + 31) / 32 * 32;
        if (threads > ddb::sscga_max_threads(eb, lc)) continue;
        if (force_lc && lc != force_lc) continue;
        if (active >= target || force_lc) { best = lc; break; }
      }
      if (!best) continue;
      s->cluster = C;
      s->lcta = lcta;
      s->lc = best;
      s->threads = (M * (lcta / best) + 31) / 32 * 32;
      s->halo = (int)h;
      s->tl = TL;
      s->th = TH;
      s->pcap = pcap;
      s->tcols = ddb::sscga_tmem_cols(s->threads, best, eb);
      s->smem = (int)ddb::sscga_layout(M, N, C, eb, (int)h, TL, TH, pcap).total;
      // keep (CTAs per SM) x (TMEM columns per CTA) <= 512 so tcgen05.alloc never
      // waits on a co-resident CTA: pad tiny CTAs' shared memory accordingly
      // 228 KiB per SM, 1 KiB reserved per CTA: at most 512 / tcols CTAs fit
      const int max_ctas = 512 / s->tcols;
      int floor_smem = 233472 / (max_ctas + 1) - 1024 + 16;
      if (floor_smem > cap) floor_smem = cap;
      if (s->smem < floor_smem) s->smem = floor_smem;
      return DDB_OK;
    }
  }
  return plan_global(M, N, s);
}

}  // namespace

extern "C" {

int32_t ddb_abi_version(void) { return DDB_ABI_VERSION; }

const char* ddb_last_error(void) { return g_err.c_str(); }

const char* ddb_build_info(void) {
#define DDB_STR2(x) #x
#define DDB_STR(x) DDB_STR2(x)
  static const char info[] = "ddb sm_100a; nvcc " DDB_STR(__CUDACC_VER_MAJOR__) "." DDB_STR(
      __CUDACC_VER_MINOR__) "." DDB_STR(__CUDACC_VER_BUILD__);
  return info;
}

int32_t ddb_sscga_plan(int32_t M, int32_t N, int32_t dtype, ddb_plan* out) {
  if (!out) return fail(DDB_ERR_INVALID, "null plan pointer");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  int32_t r = check_grid(M, N);
  if (r) return r;
  ddb::LaunchShape s;
  r = make_plan(M, N, dtype, &s);
  if (r) return r;
  out->cluster = s.cluster;
  out->cols_per_cta = s.lcta;
  out->cols_per_thread = s.lc;
  out->threads = s.threads;
  out->smem_bytes = s.smem;
  out->ctas_per_sm = 0;
  out->halo_rows = s.halo;
  out->kernel = s.kind;
  out->rows_per_thread = s.kind == 1 ? s.rows : 1;
  int n = 0;
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0) {
    cudaError_t e = s.kind == 2          ? (n = 0, cudaSuccess)
                    : s.kind == 1        ? ddb::sscga_tm_occupancy(s, &n)
                    : dtype == DDB_F64 ? ddb::sscga_occupancy<double>(s, &n)
                                       : ddb::sscga_occupancy<float>(s, &n);
    if (e == cudaSuccess) out->ctas_per_sm = n;
  }
  cudaGetLastError();
  return ok();
}

size_t ddb_sscga_workspace_bytes(const ddb_sscga_problem* prob) {
  if (!prob || prob->batch <= 0 || (prob->dtype != DDB_F32 && prob->dtype != DDB_F64)) return 0;
  if (check_grid(prob->M, prob->N)) return 0;
  ddb::LaunchShape s;
  if (make_plan(prob->M, prob->N, prob->dtype, &s)) return 0;
  // the fused kernels keep all CG state on chip; the workspace path keeps c, u, p in HBM
  return s.kind == 2 ? ddb::sscga_global_workspace(prob->dtype == DDB_F64, prob->batch, prob->M, prob->N) : 0;
}

static int32_t solve_impl(const ddb_sscga_problem* prob, const ddb_sscga_outputs* out, long long* prof,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (!prob || !out) return fail(DDB_ERR_INVALID, "null problem/outputs");
  if (prob->batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (prob->iterations < 1) return fail(DDB_ERR_INVALID, "need at least one iteration");  // equalize.py:26-27
  if (prob->dtype != DDB_F32 && prob->dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", prob->dtype);
  int32_t r = check_grid(prob->M, prob->N);
  if (r) return r;
  if (prob->batch == 0) return ok();
  if (!prob->path_offsets || !prob->y || !prob->lam || !out->x)
    return fail(DDB_ERR_INVALID, "null required pointer (path_offsets, y, lam, x)");
  if (!prob->path_k || !prob->path_l || !prob->path_gain)
    return fail(DDB_ERR_INVALID, "null path arrays");
  const int bps = out->bits_per_symbol;
  if (bps != 0 && bps != 2 && bps != 4 && bps != 6)
    return fail(DDB_ERR_INVALID, "bits_per_symbol must be 0, 2, 4 or 6, got %d", bps);
  if (out->bit_errors && (!out->tx_labels || bps == 0))
    return fail(DDB_ERR_INVALID, "bit_errors needs tx_labels and bits_per_symbol > 0");
  if ((out->labels || out->llr) && bps == 0)
    return fail(DDB_ERR_INVALID, "labels/llr need bits_per_symbol > 0");
  if (out->tx_labels_packed && bps != 2 && bps != 4)
    return fail(DDB_ERR_INVALID, "packed tx labels need bits_per_symbol 2 or 4, got %d", bps);
  ddb::LaunchShape s;
  r = make_plan(prob->M, prob->N, prob->dtype, &s);
  if (r) return r;
  ddb::SolveArgs a = {};
  a.B = prob->batch;
  a.M = prob->M;
  a.N = prob->N;
  a.MN = prob->M * prob->N;
  a.K0 = prob->M / 2;
  a.L0 = prob->N / 2;
  a.iters = prob->iterations;
  a.C = s.cluster;
  a.Lcta = s.lcta;
  a.active_threads = prob->M * (s.lcta / s.lc);
  a.S = prob->M + s.halo;
  a.RS = ddb::row_stride(s.lcta, prob->dtype == DDB_F64 ? 8 : 4);
  a.H = s.halo;
  a.TL = s.tl;
  a.TH = s.th;
  a.pcap = s.pcap;
  a.tcols = s.tcols;
  a.G = s.g;
  a.WQ = s.wq;
  a.CS = s.cs;
  a.gd = s.kind == 1 ? s.gd : 0;
  if (s.kind == 1) a.active_threads = s.threads;
  // TMEM kernel: frames' y streamed by cp.async.bulk (16-byte aligned y; DDB_NO_TMA=1 for A/B runs)
  a.stream_y = s.kind == 1 && (reinterpret_cast<uintptr_t>(prob->y) & 15) == 0 && !getenv("DDB_NO_TMA");
  {
    const char* env = getenv("DDB_TM_SPLIT");
    a.split = s.kind == 1 && (env ? atoi(env) != 0 : 1);
  }
  a.off = prob->path_offsets;
  a.pk = prob->path_k;
  a.pl = prob->path_l;
  a.ph = prob->path_gain;
  a.y = prob->y;
  a.lam = prob->lam;
  a.x = out->x;
  a.cnorm = out->c_norm;
  a.itdone = out->iterations_done;
  a.status = out->status;
  a.snaps = out->snapshots;
  a.bps = bps;
  a.labels = out->labels;
  a.llr = out->llr;
  a.nvar = out->noise_var;
  a.txl = out->tx_labels;
  a.txpk = out->tx_labels_packed ? 1 : 0;
  a.berr = out->bit_errors;
  a.prof = prof;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s.kind == 2) {
    const size_t need = ddb::sscga_global_workspace(prob->dtype == DDB_F64, a.B, a.M, a.N);
    if (!workspace || workspace_bytes < need)
      return fail(DDB_ERR_WORKSPACE, "grid (%d,%d) needs a %zu-byte workspace (ddb_sscga_workspace_bytes), got %zu",
                  a.M, a.N, need, workspace ? workspace_bytes : (size_t)0);
    if (prof) return fail(DDB_ERR_UNSUPPORTED, "phase profiling is a fused-kernel feature");
  }
  cudaError_t e = s.kind == 2                ? (prob->dtype == DDB_F64 ? ddb::launch_sscga_global<double>(a, workspace, st)
                                                                       : ddb::launch_sscga_global<float>(a, workspace, st))
                  : s.kind == 1              ? ddb::launch_sscga_tm(a, s, st)
                  : prob->dtype == DDB_F64 ? ddb::launch_sscga<double>(a, s, st)
                                           : ddb::launch_sscga<float>(a, s, st);
  if (e != cudaSuccess) return cuda_fail(e, "sscga launch");
  return ok();
}

int32_t ddb_sscga_solve(const ddb_sscga_problem* prob, const ddb_sscga_outputs* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return solve_impl(prob, out, nullptr, workspace, workspace_bytes, stream);
}

int32_t ddb_sscga_profile_phases(const ddb_sscga_problem* prob, const ddb_sscga_outputs* out,
                                 long long* phase_cycles, void* stream) {
  if (!phase_cycles) return fail(DDB_ERR_INVALID, "null phase buffer");
  return solve_impl(prob, out, phase_cycles, nullptr, 0, stream);
}

int32_t ddb_ss_apply(const ddb_sscga_problem* prob, void* outp, int32_t hermitian, void* stream) {
  if (!prob || !outp) return fail(DDB_ERR_INVALID, "null problem/output");
  if (prob->batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (prob->dtype != DDB_F32 && prob->dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", prob->dtype);
  int32_t r = check_grid(prob->M, prob->N);
  if (r) return r;
  if (prob->batch == 0) return ok();
  if (!prob->path_offsets || !prob->path_k || !prob->path_l || !prob->path_gain || !prob->y)
    return fail(DDB_ERR_INVALID, "null input pointer");
  if (prob->batch > 65535) return fail(DDB_ERR_UNSUPPORTED, "ss_apply batch > 65535");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = prob->dtype == DDB_F64
                      ? ddb::launch_ss_apply<double>(prob->batch, prob->M, prob->N, prob->path_offsets,
                                                     prob->path_k, prob->path_l, prob->path_gain, prob->y,
                                                     outp, hermitian != 0, st)
                      : ddb::launch_ss_apply<float>(prob->batch, prob->M, prob->N, prob->path_offsets,
                                                    prob->path_k, prob->path_l, prob->path_gain, prob->y,
                                                    outp, hermitian != 0, st);
  if (e != cudaSuccess) return cuda_fail(e, "ss_apply launch");
  return ok();
}

int32_t ddb_build_tables(int32_t M, int32_t N, int32_t n_paths, const int32_t* path_k, const int32_t* path_l,
                         const void* path_gain, void* fwd_coef, int32_t* fwd_col, void* herm_coef,
                         int32_t* herm_row, void* stream) {
  int32_t r = check_grid(M, N);
  if (r) return r;
  if (n_paths < 0) return fail(DDB_ERR_INVALID, "negative path count");
  if (n_paths == 0) return fail(DDB_ERR_INVALID, "no taps above threshold");  // EmptyChannel, sparse.py:126-127
  if (!path_k || !path_l || !path_gain || !fwd_coef || !fwd_col || !herm_coef || !herm_row)
    return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_build_tables(M, N, n_paths, path_k, path_l, path_gain, fwd_coef, fwd_col,
                                           herm_coef, herm_row, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "build_tables launch");
  return ok();
}

int32_t ddb_ss_mvm_tables(int32_t size, int32_t n_paths, const void* coef, const int32_t* index, const void* v,
                          void* u, void* stream) {
  if (size < 0 || n_paths < 0) return fail(DDB_ERR_INVALID, "negative size");
  if (!v || !u || (n_paths > 0 && (!coef || !index))) return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_mvm_tables(size, n_paths, coef, index, v, u, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mvm_tables launch");
  return ok();
}

int32_t ddb_hard_demod(int64_t count, int32_t dtype, const void* x, const void* points, int32_t n_points,
                       int32_t* labels, void* stream) {
  if (count < 0 || n_points < 1) return fail(DDB_ERR_INVALID, "bad count/n_points");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (count > 0 && (!x || !points || !labels)) return fail(DDB_ERR_INVALID, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = dtype == DDB_F64 ? ddb::launch_hard_demod<double>(count, x, points, n_points, labels, st)
                                   : ddb::launch_hard_demod<float>(count, x, points, n_points, labels, st);
  if (e != cudaSuccess) return cuda_fail(e, "hard_demod launch");
  return ok();
}

int32_t ddb_qam_demod(int64_t count, int32_t dtype, const void* x, int32_t bits_per_symbol, double noise_var,
                      uint8_t* labels, float* llr, void* stream) {
  if (count < 0) return fail(DDB_ERR_INVALID, "negative count");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (bits_per_symbol != 2 && bits_per_symbol != 4 && bits_per_symbol != 6)
    return fail(DDB_ERR_INVALID, "bits_per_symbol must be 2, 4 or 6, got %d", bits_per_symbol);
  if (count > 0 && !x) return fail(DDB_ERR_INVALID, "null input");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = dtype == DDB_F64
                      ? ddb::launch_qam_demod<double>(count, x, bits_per_symbol, noise_var, labels, llr, st)
                      : ddb::launch_qam_demod<float>(count, x, bits_per_symbol, noise_var, labels, llr, st);
  if (e != cudaSuccess) return cuda_fail(e, "qam_demod launch");
  return ok();
}

int32_t ddb_detect_paths(int32_t batch, int32_t M, int32_t N, const void* heff, double theta, int32_t max_paths,
                         int32_t* count, int32_t* path_k, int32_t* path_l, void* path_gain, void* stream) {
  if (batch < 0 || max_paths < 0) return fail(DDB_ERR_INVALID, "negative batch/max_paths");
  if (!(theta >= 0)) return fail(DDB_ERR_INVALID, "theta must be nonnegative");  // sparse.py:77-78
  int32_t r = check_grid(M, N);
  if (r) return r;
  if (batch == 0) return ok();
  if (!heff || !count || (max_paths > 0 && (!path_k || !path_l || !path_gain)))
    return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_detect_paths(batch, M, N, heff, theta, max_paths, count, path_k, path_l, path_gain,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "detect_paths launch");
  return ok();
}

int32_t ddb_paths_csr(int32_t batch, int32_t max_paths, const int32_t* count, const int32_t* path_k,
                      const int32_t* path_l, const void* path_gain, int32_t dtype, int32_t* path_offsets,
                      int32_t* csr_k, int32_t* csr_l, void* csr_gain, int32_t* stats, void* stream) {
  if (batch < 0 || max_paths < 0) return fail(DDB_ERR_INVALID, "negative batch/max_paths");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (batch == 0) return ok();
  if (!count || !path_offsets || !stats || (max_paths > 0 && (!path_k || !path_l || !path_gain || !csr_k ||
                                                               !csr_l || !csr_gain)))
    return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_paths_csr(batch, max_paths, count, path_k, path_l, path_gain, dtype == DDB_F64,
                                        path_offsets, csr_k, csr_l, csr_gain, stats,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "paths_csr launch");
  return ok();
}

int32_t ddb_dzt(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* y_time, const void* kernel,
                int32_t flags, double amplitude, void* out, void* stream) {
  if (batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (M < 1 || N < 1) return fail(DDB_ERR_SHAPE, "grid must be positive, got (%d,%d)", M, N);
  if ((long long)M * N >= (1LL << 29)) return fail(DDB_ERR_UNSUPPORTED, "grid too large");
  if (N > 256) return fail(DDB_ERR_UNSUPPORTED, "N=%d > 256 (kernel matrix exceeds shared memory)", N);
  if (flags & ~(DDB_DZT_COLMAJOR | DDB_DZT_PILOT | DDB_DZT_INPUT_F32 | DDB_DZT_INVERSE)) return fail(DDB_ERR_INVALID, "bad flags %d", flags);
  if ((flags & DDB_DZT_INVERSE) && (kernel || (flags & (DDB_DZT_PILOT | DDB_DZT_INPUT_F32)) || !(flags & DDB_DZT_COLMAJOR)))
    return fail(DDB_ERR_INVALID, "DDB_DZT_INVERSE takes the default kernel, DDB_DZT_COLMAJOR and no pilot / f32 input");
  if ((flags & DDB_DZT_INPUT_F32) && (dtype != DDB_F64 || kernel || N < 2 || (N & (N - 1))))
    return fail(DDB_ERR_UNSUPPORTED, "complex64 input needs dtype f64, the default kernel and a power-of-two N");
  if ((flags & DDB_DZT_PILOT) && !(amplitude > 0))
    return fail(DDB_ERR_INVALID, "pilot amplitude must be positive");  // pilot.py:45-46
  if ((flags & DDB_DZT_PILOT) && ((M & 1) || (N & 1)))
    return fail(DDB_ERR_SHAPE, "M and N must be even for the pilot estimate");  // grid.py:25-29
  if (batch == 0) return ok();
  if (!y_time || !out) return fail(DDB_ERR_INVALID, "null pointer");
  const double amp = (flags & DDB_DZT_PILOT) ? amplitude : 1.0;
  cudaError_t e = (flags & DDB_DZT_INPUT_F32)
                      ? ddb::launch_dzt_mixed(batch, M, N, y_time, flags & DDB_DZT_COLMAJOR, flags & DDB_DZT_PILOT, amp,
                                              out, static_cast<cudaStream_t>(stream))
                      : ddb::launch_dzt(dtype == DDB_F64, batch, M, N, y_time, kernel, flags & DDB_DZT_COLMAJOR,
                                        flags & DDB_DZT_PILOT, flags & DDB_DZT_INVERSE, amp, out,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dzt launch");
  return ok();
}

// ---- host round trips: a per-thread, per-device scratch and stream
namespace {
struct HostScratch {
  int dev = -1;
  cudaStream_t st = nullptr;
  void* buf = nullptr;
  size_t cap = 0;
};
thread_local HostScratch g_hs;

// Device scratch of at least `bytes` on the current device (grown, never shrunk).
cudaError_t host_scratch(size_t bytes, unsigned char** out, cudaStream_t* st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_hs.dev != dev) {  // a new device for this thread: the old scratch stays with its device
    g_hs = HostScratch{};
    g_hs.dev = dev;
    if ((e = cudaStreamCreateWithFlags(&g_hs.st, cudaStreamNonBlocking)) != cudaSuccess) return e;
  }
  if (g_hs.cap < bytes) {
    if (g_hs.buf) cudaFree(g_hs.buf);
    g_hs.buf = nullptr;
    g_hs.cap = 0;
    size_t cap = 1 << 16;
    while (cap < bytes) cap <<= 1;
    if ((e = cudaMalloc(&g_hs.buf, cap)) != cudaSuccess) return e;
    g_hs.cap = cap;
  }
  *out = static_cast<unsigned char*>(g_hs.buf);
  *st = g_hs.st;
  return cudaSuccess;
}
inline size_t al256(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace

int32_t ddb_host_dzt(int32_t M, int32_t N, const void* y_time, const void* kernel, void* out) {
  if (M < 1 || N < 1 || !y_time || !out) return fail(DDB_ERR_INVALID, "bad host dzt arguments");
  const size_t n = (size_t)M * N * 16, nk = kernel ? (size_t)N * N * 16 : 0;
  unsigned char* d;
  cudaStream_t st;
  cudaError_t e = host_scratch(2 * al256(n) + al256(nk), &d, &st);
  if (e != cudaSuccess) return cuda_fail(e, "host scratch");
  unsigned char *dy = d, *dout = d + al256(n), *dk = kernel ? d + 2 * al256(n) : nullptr;
  if ((e = cudaMemcpyAsync(dy, y_time, n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
  if (kernel && (e = cudaMemcpyAsync(dk, kernel, nk, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D");
  int32_t r = ddb_dzt(1, M, N, DDB_F64, dy, dk, 0, 1.0, dout, st);
  if (r) return r;
  if ((e = cudaMemcpyAsync(out, dout, n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, "D2H");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "host dzt");
  return ok();
}

int32_t ddb_host_estimate_heff(int64_t count, const void* y_dd, const void* twist, double amplitude, void* heff) {
  if (count < 0 || (count && (!y_dd || !twist || !heff))) return fail(DDB_ERR_INVALID, "bad host estimate arguments");
  if (!(amplitude > 0)) return fail(DDB_ERR_INVALID, "pilot amplitude must be positive");  // pilot.py:45-46
  if (count == 0) return ok();
  const size_t n = (size_t)count * 16;
  unsigned char* d;
  cudaStream_t st;
  cudaError_t e = host_scratch(3 * al256(n), &d, &st);
  if (e != cudaSuccess) return cuda_fail(e, "host scratch");
  unsigned char *dy = d, *dt = d + al256(n), *dh = d + 2 * al256(n);
  if ((e = cudaMemcpyAsync(dy, y_dd, n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
  if ((e = cudaMemcpyAsync(dt, twist, n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
  int32_t r = ddb_estimate_heff(count, DDB_F64, dy, dt, amplitude, dh, st);
  if (r) return r;
  if ((e = cudaMemcpyAsync(heff, dh, n, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, "D2H");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "host estimate_heff");
  return ok();
}

int32_t ddb_host_detect_paths(int32_t M, int32_t N, const void* heff, double theta, int32_t max_paths,
                              int32_t* count, int32_t* path_k, int32_t* path_l, void* path_gain) {
  if (max_paths < 0 || !heff || !count || (max_paths > 0 && (!path_k || !path_l || !path_gain)))
    return fail(DDB_ERR_INVALID, "bad host detect arguments");
  int32_t r = check_grid(M, N);
  if (r) return r;
  const size_t n = (size_t)M * N * 16, cap = (size_t)(max_paths > 0 ? max_paths : 1);
  // device layout [heff | gains 16 cap | k 4 cap | l 4 cap | count]: one D2H of the results
  const size_t og = al256(n), ok_ = og + 16 * cap, ol = ok_ + 4 * cap, oc = ol + 4 * cap;
  unsigned char* d;
  cudaStream_t st;
  cudaError_t e = host_scratch(oc + 16, &d, &st);
  if (e != cudaSuccess) return cuda_fail(e, "host scratch");
  if ((e = cudaMemcpyAsync(d, heff, n, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
  r = ddb_detect_paths(1, M, N, d, theta, max_paths, reinterpret_cast<int32_t*>(d + oc),
                       reinterpret_cast<int32_t*>(d + ok_), reinterpret_cast<int32_t*>(d + ol), d + og, st);
  if (r) return r;
  // count first (4 bytes), then only the rows that hold taps
  int32_t c = 0;
  if ((e = cudaMemcpyAsync(&c, d + oc, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, "D2H");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "host detect_paths");
  *count = c;
  const size_t rows = (size_t)(c < max_paths ? c : max_paths);
  if (rows > 0) {
    if ((e = cudaMemcpyAsync(path_gain, d + og, 16 * rows, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(path_k, d + ok_, 4 * rows, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(path_l, d + ol, 4 * rows, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return cuda_fail(e, "D2H");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "host detect_paths");
  }
  return ok();
}

int32_t ddb_estimate_heff(int64_t count, int32_t dtype, const void* y_dd, const void* twist, double amplitude,
                          void* heff, void* stream) {
  if (count < 0) return fail(DDB_ERR_INVALID, "negative count");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (!(amplitude > 0)) return fail(DDB_ERR_INVALID, "pilot amplitude must be positive");  // pilot.py:45-46
  if (count == 0) return ok();
  if (!y_dd || !twist || !heff) return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_estimate_heff(dtype == DDB_F64, count, y_dd, twist, amplitude, heff,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "estimate_heff launch");
  return ok();
}

int32_t ddb_modulate(int64_t count, int32_t dtype, const uint8_t* labels, int32_t bits_per_symbol, void* out,
                     void* stream) {
  if (count < 0) return fail(DDB_ERR_INVALID, "negative count");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (bits_per_symbol != 2 && bits_per_symbol != 4 && bits_per_symbol != 6)
    return fail(DDB_ERR_INVALID, "bits_per_symbol must be 2, 4 or 6, got %d", bits_per_symbol);
  if (count == 0) return ok();
  if (!labels || !out) return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_modulate(dtype == DDB_F64, count, labels, bits_per_symbol, out,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "modulate launch");
  return ok();
}

int32_t ddb_apply_channel(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* x,
                          const int32_t* path_offsets, const int32_t* delay_bin, const double* doppler_hz,
                          const double* delay_s, const void* gain, double bandwidth_hz, void* y, void* stream) {
  if (batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (M < 1 || N < 1) return fail(DDB_ERR_SHAPE, "grid must be positive, got (%d,%d)", M, N);
  if ((long long)M * N >= (1LL << 29)) return fail(DDB_ERR_UNSUPPORTED, "grid too large");
  if (!(bandwidth_hz > 0)) return fail(DDB_ERR_INVALID, "bandwidth must be positive");
  if (batch == 0) return ok();
  if (!x || !y || !path_offsets || !delay_bin || !doppler_hz || !delay_s || !gain)
    return fail(DDB_ERR_INVALID, "null pointer");
  if (x == y) return fail(DDB_ERR_INVALID, "apply_channel cannot run in place");
  cudaError_t e = ddb::launch_apply_channel(dtype == DDB_F64, batch, M * N, bandwidth_hz, x, path_offsets, delay_bin,
                                            doppler_hz, delay_s, gain, y, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "apply_channel launch");
  return ok();
}

int32_t ddb_add_awgn(int32_t batch, int64_t frame_len, int32_t dtype, const void* y, double snr_db, uint64_t seed,
                     double* frame_power, void* out, void* stream) {
  if (batch < 0 || frame_len < 0) return fail(DDB_ERR_INVALID, "negative batch/frame_len");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (snr_db != snr_db) return fail(DDB_ERR_INVALID, "snr_db is NaN");
  if (batch == 0 || frame_len == 0) return ok();
  if (!y || !out) return fail(DDB_ERR_INVALID, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (std::isinf(snr_db) && snr_db > 0) {  // noiseless sentinel (channel.py:112-113): a copy
    if (out == y) return ok();
    const size_t bytes = (size_t)batch * frame_len * (dtype == DDB_F64 ? 16 : 8);
    cudaError_t e = cudaMemcpyAsync(out, y, bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "awgn copy");
    return ok();
  }
  if (!frame_power) return fail(DDB_ERR_INVALID, "frame_power scratch [batch] is required");
  cudaError_t e = ddb::launch_add_awgn(dtype == DDB_F64, batch, frame_len, y, snr_db, seed, frame_power, out, st);
  if (e != cudaSuccess) return cuda_fail(e, "awgn launch");
  return ok();
}

int32_t ddb_threshold_frame(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* heff, double theta,
                            void* out, void* stream) {
  if (batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  if (M < 1 || N < 1) return fail(DDB_ERR_SHAPE, "grid must be positive, got (%d,%d)", M, N);
  if ((long long)M * N >= (1LL << 29)) return fail(DDB_ERR_UNSUPPORTED, "grid too large");
  if (batch == 0) return ok();
  if (!heff || !out) return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_threshold_frame(dtype == DDB_F64, batch, M * N, heff, theta, out,
                                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "threshold_frame launch");
  return ok();
}

int32_t ddb_build_dense_hdd(int32_t batch, int32_t M, int32_t N, int32_t dtype, const void* heff, void* H,
                            void* stream) {
  if (batch < 0) return fail(DDB_ERR_INVALID, "negative batch");
  if (dtype != DDB_F32 && dtype != DDB_F64) return fail(DDB_ERR_INVALID, "bad dtype %d", dtype);
  int32_t r = check_grid(M, N);
  if (r) return r;
  if (M * N > 4096) return fail(DDB_ERR_SHAPE, "dense channel matrix limited to MN <= 4096, got %d", M * N);
  if (batch == 0) return ok();
  if (!heff || !H) return fail(DDB_ERR_INVALID, "null pointer");
  cudaError_t e = ddb::launch_build_dense(dtype == DDB_F64, batch, M, N, heff, H, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "build_dense_hdd launch");
  return ok();
}

int32_t ddb_probe_fp32(int32_t mode, int32_t blocks, int32_t iters, float* scratch, void* stream) {
  if (mode < 0 || mode > 2 || blocks < 1 || iters < 1 || !scratch)
    return fail(DDB_ERR_INVALID, "bad probe arguments");
  cudaError_t e = ddb::launch_fp32_probe(mode, blocks, iters, scratch, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fp32 probe launch");
  return ok();
}

}  // extern "C"
