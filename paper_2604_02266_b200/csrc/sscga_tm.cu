// Fused SS-CGA solve with TMEM-resident operands (fp32, sm_100a).
//
// Same algorithm as sscga.cu (cga_equalize, equalize.py:43-77, on the
// matrix-free operator of sparse.py:91-160, closed forms in that file's
// header) with a data layout built around tensor memory.  The MVM of the
// reference is a gather-multiply-reduce: every complex MAC needs one fresh
// 8-byte operand.  Served from shared memory (128 B/clk/SM) that caps the MVM
// at half the FP32 FMA rate; tcgen05.ld delivers > 300 B/clk/SM
// (profiles/ubench_tmem_bw.txt), so here the gathered vectors live in TMEM.
//
// TMEM is lane-private: a warp reaches only its quarter of the 128 lanes and a
// thread only its own lane, but any column of it.  A Doppler-preserving tap
// (d_l == 0, the bulk of every Veh-A channel) shifts data along the delay axis
// only, so delay rows go along TMEM columns:
//   lane L = seg * Lcta + col   holds delay rows [seg G, seg G + G) of the
//                               CTA's Doppler column col (S = 128 / Lcta
//                               segments of G = M / S rows per column);
//   thread (warp w, lane t)     uses TMEM lane 32 (w % 4) + t and owns the
//                               R = G / WQ rows j R .. j R + R - 1 of that
//                               segment, j = w / 4 (WQ warps per lane quarter).
// Per lane the 512 columns hold c | u (the whole segment, 2G words each,
// gathered by H and H^H) and p | x (the WQ threads' own rows).  A d_l == 0 tap
// whose source rows stay inside the segment is one tcgen05.ld of 2R words at
// column 2 (j R + shift) followed by R FFMA2 complex MACs with a warp-uniform
// gain.  Everything else reads the column-major extended copies of c and u in
// shared memory (written beside every TMEM update, quasi-periodic halo rows
// included): d_l == 0 taps that leave the segment take one contiguous run of
// the lane's own column, other taps gather per element, through DSMEM when the
// source column lives in a peer CTA of the cluster.
//
// CG step (u-recurrence, two cluster barriers per iteration) and the
// deterministic reductions are those of sscga.cu.
#include <climits>
#include <cstdlib>

#include "cg.cuh"
#include "common.cuh"
#include "demod.cuh"
#include "internal.h"

namespace ddb {

namespace {

using V = float2;
using U64 = unsigned long long;

// Per-frame state, in shared memory (written at frame setup, read where
// needed, so none of it occupies registers across the CG loop).  Tap masks
// (P <= 32, tap table on chip) are per row block j: the TMEM test depends on
// the warp's rows, so they are warp-uniform.
struct FrameSm {
  int P0, P;
  int in_smem, halo, masks;
  int lo_c, hi_c, lo_u, hi_u;  // extension rows written for c (gathered by H) and u (by H^H)
  int remote;                  // some warp gathers per element (DSMEM): publish c / u with release
  int wrap;                    // some shift exceeds the halo: runs beyond it wrap the delay period
  int ghost;                   // ghost columns pushed per side this frame (0: none; the frame's largest |d_l| <= gd)
  uint32_t mk[8][6];           // [j][tmF, smF, gnF, tmH, smH, gnH]: TMEM run / shared run / per element
};

constexpr int kWarpTimers = 8;

__host__ __device__ inline size_t a16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout tm_layout_impl(int Lcta, int N, int CS, int TL, int TH, int pcap, int gd) {
  SmemLayout L;
  size_t o = 0;
  // extended c and u, column-major, each behind a 16-byte guard: odd-aligned
  // runs read one (unused) element beyond either end of a column
  o += 16;
  L.p = o; o = a16(o + (size_t)Lcta * CS * sizeof(V)) + 16;
  L.u = o; o = a16(o + (size_t)Lcta * CS * sizeof(V));
  L.x = o; o = a16(o + 16);                             // TMEM base-address slot (+0), y mbarrier (+8)
  L.tlo = o; o = a16(o + (size_t)TL * sizeof(V));
  L.thi = o; o = a16(o + (size_t)TH * sizeof(V));
  L.tw = o; o = a16(o + (size_t)N * sizeof(V));
  L.ptab = o; o = a16(o + (size_t)pcap * sizeof(PathEnt<float>));
  L.red = o; o = a16(o + 2 * 2 * kPushSlots * sizeof(V) + sizeof(ProfSm) + sizeof(FrameSm));
  L.q = o; o = a16(o + (128 + 16) * sizeof(int));       // frame list (kListChunk) of this CTA's class + warp counts
  if (gd > 0) {
    // clusters: ghost copies of the gd boundary columns on either side (the
    // left neighbour's last gd, then the right neighbour's first gd, extended
    // like the own columns) of c or u, whichever the next MVM gathers, pushed
    // by their owners (gh_push); a "full" mbarrier (bytes landed) and an
    // "empty" one (every warp of both neighbours done reading this CTA's last
    // push: each arrives remotely at the end of its remote pass)
    (void)N;
    L.gh = o; o = a16(o + (size_t)2 * gd * CS * sizeof(V));
    L.ghmb = o; o = a16(o + 16);
  }
  L.total = o;
  return L;
}

struct TmSm {
  V* c;  // extended column-major c: column col at c + col CS, row a (in [-H, M + H)) at + H + a
  V* u;
  uint32_t* tslot;
  const V* tlo;
  const V* thi;
  const V* tw;
  PathEnt<float>* ptab;
  int tlb;
  V* gh;  // ghost columns (clusters)
};

__device__ __forceinline__ V twid_tm(const TmSm& sm, int e) {
  return cmul(sm.thi[e >> sm.tlb], sm.tlo[e & ((1 << sm.tlb) - 1)]);
}

// Per-thread geometry (kept small: the kernel runs at 64-128 registers).
struct TmThr {
  int col;    // Doppler column inside the CTA (TMEM lane -> column)
  int colg;   // global Doppler column
  int jr;     // first owned row inside the segment (j R, j = warp / 4)
  int r0;     // first owned delay row
  uint32_t tl;  // TMEM address of this warp's lane quarter, column 0
};



__device__ __forceinline__ PathEnt<float> tm_path(const SolveArgs& a, const TmSm& sm, int kp, int lp, V h) {
  PathEnt<float> e;
  e.dk = a.K0 - kp;
  e.dl = a.L0 - lp;
  // off / pad: the forward per-row coefficient step W^{-d_l} of a Doppler tap
  // (tap_elem; the hermitian one is its conjugate), made once per frame
  const V st = e.dl ? twid_tm(sm, wrap1(-e.dl, a.MN)) : make_float2(1.f, 0.f);
  e.off = __float_as_int(st.x);
  e.pad = __float_as_int(st.y);
  e.hf = quad(e.dl ? cmul(h, twid_tm(sm, wrap1(-e.dl * e.dk, a.MN))) : h);
  e.hh = quad(cconj(h));
  return e;
}

__device__ __forceinline__ PathEnt<float> tm_get(const SolveArgs& a, const TmSm& sm, const FrameSm& fs, int p) {
  if (fs.in_smem) return sm.ptab[p];
  return tm_path(a, sm, __ldg(a.pk + fs.P0 + p), __ldg(a.pl + fs.P0 + p),
                 __ldg(reinterpret_cast<const V*>(a.ph) + fs.P0 + p));
}

// Tap classes for row block jr: 0 = TMEM run, 1 = shared-memory run, 2 = per element.
template <int R, bool HERM>
__device__ __forceinline__ int tap_class(const SolveArgs& a, int jr, bool halo, const PathEnt<float>& e) {
  if (e.dl != 0) return 2;
  const int s = HERM ? -e.dk : e.dk;
  if (jr + s >= 0 && jr + s + R <= a.G) return 0;
  return halo ? 1 : 2;
}

// ---- gathers ------------------------------------------------------------
// FFMA2 operand pairs X = (g.x, g.x), Y = (-g.y, g.y) of a tap's gain for one
// direction: one 128-bit shared load straight into two register pairs.
template <bool HERM>
__device__ __forceinline__ ulonglong2 gain_pairs(const PathEnt<float>& e) {
  return *reinterpret_cast<const ulonglong2*>(HERM ? &e.hh : &e.hf);
}
template <int R>
__device__ __forceinline__ void gather_tmem(uint32_t ta, U64 X, U64 Y, U64 (&acc)[R]) {
  uint32_t v[2 * R];
  tmem_ld<2 * R>(ta, v);
  tmem_wait_ld_tie<2 * R>(v);
#pragma unroll
  for (int i = 0; i < R; ++i) cmacxy(acc[i], X, Y, __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
}

// Start row of a thread's R-row source run in an extended column whose halo
// rows [-lo, 0) and [M, M + hi) are written.  A run beyond them (a frame whose
// shifts exceed the halo capacity H, e.g. taps anywhere on the grid) lies
// wholly outside [0, M) (R <= H), so it is read one delay period over, inside
// the column itself, and the quasi-periodic twist of that period (put_col:
// ext[r - M] = v W_N^{-l}, ext[r + M] = v W_N^{+l}) moves into the gain: no
// per-row wrap.  Returns the twist (1 when the run is in place).
template <int R>
__device__ __forceinline__ V wrap_run(int& a0, int M, int lo, int hi, V tw_src) {
  if (a0 < -lo) {
    a0 += M;
    return cconj(tw_src);
  }
  if (a0 + R > M + hi) {
    a0 -= M;
    return tw_src;
  }
  return make_float2(1.f, 0.f);
}

// One tap with a Doppler shift (d_l != 0), or any tap when the frame's shifts
// exceed the halo, from the (possibly remote) extended column of the source
// Doppler column.  With the halo the R source rows are one contiguous run:
// 16-byte DSMEM loads, and the row-dependent coefficient h W^{-+d_l k} of the
// forward / hermitian closed form (sparse.py:107-121) advanced by one complex
// multiply per row from an exact table value every 8 rows; a run beyond the
// written halo (wrap) is read one delay period over (wrap_run).  Without the
// halo rows wrap the delay period individually (twist applied in registers).
// LDS: every lane reads this CTA's shared memory -- its own columns, or the
// ghost copy of a neighbouring CTA's boundary column (frames with ghosts, taps
// with |d_l| = 1) -- instead of DSMEM (≈ 5 B/clk/SM for these scattered
// 16-byte reads, tools/ubench/dsmem_bw.cu).
template <int R, bool HERM, bool LDS>
__device__ __forceinline__ void tap_elem_impl(const SolveArgs& a, const TmThr& th, const TmSm& sm, const FrameSm& fs,
                                              bool halo, const V* buf, const PathEnt<float>& e, U64 (&acc)[R]) {
  const int M = a.M, MN = a.MN;
  const int dl = e.dl;
  const int s = HERM ? -e.dk : e.dk;
  const float4 g = HERM ? e.hh : e.hf;
  const V h0 = make_float2(g.x, g.w);
  const int ls = wrap1(th.colg + (HERM ? -dl : dl), a.N);  // source Doppler column
  const int own = ls / a.Lcta;
  const int lc = ls - own * a.Lcta;
  const V* colp = buf + (size_t)lc * a.CS + a.H;
  if (LDS) {  // a neighbour's boundary column: its ghost copy (|d_l| <= gd <= Lcta)
    const int rel = th.col + (HERM ? -dl : dl);  // source column relative to this CTA's first
    if (rel < 0) colp = sm.gh + (size_t)(a.gd + rel) * a.CS + a.H;
    else if (rel >= a.Lcta) colp = sm.gh + (size_t)(a.gd + rel - a.Lcta) * a.CS + a.H;
  }
  const uint32_t colad = LDS ? 0u : map_rank(smem_addr(colp), (uint32_t)own);
  const int sg = HERM ? dl : -dl;  // coefficient phase exponent per row
  if (halo) {
    constexpr int BS = R;  // rows per exact re-anchor (16-step fp32 recurrence: ~1e-6 relative)
    const V step = make_float2(__int_as_float(e.off), HERM ? -__int_as_float(e.pad) : __int_as_float(e.pad));
    int a0 = th.r0 + s;
    V hw = h0;
    if (fs.wrap) hw = cmul(h0, wrap_run<R>(a0, M, HERM ? fs.lo_u : fs.lo_c, HERM ? fs.hi_u : fs.hi_c, sm.tw[ls]));
    const uint32_t run = colad + (uint32_t)(a0 * (int)sizeof(V));
    const float4* lrun = reinterpret_cast<const float4*>(colp + a0 - (s & 1));
    auto ld4 = [&](int m, uint32_t off) { return LDS ? lrun[m] : ld_cluster4(run + off); };
    V v[R];
    if ((s & 1) == 0) {
#pragma unroll
      for (int m = 0; m < R / 2; ++m) {
        const float4 w = ld4(m, 16u * m);
        v[2 * m] = make_float2(w.x, w.y);
        v[2 * m + 1] = make_float2(w.z, w.w);
      }
    } else {
      float4 w = ld4(0, 0u - 8u);
      v[0] = make_float2(w.z, w.w);
#pragma unroll
      for (int m = 1; m < R / 2; ++m) {
        w = ld4(m, 16u * m - 8u);
        v[2 * m - 1] = make_float2(w.x, w.y);
        v[2 * m] = make_float2(w.z, w.w);
      }
      w = ld4(R / 2, 16u * (R / 2) - 8u);
      v[R - 1] = make_float2(w.x, w.y);
    }
#pragma unroll
    for (int b = 0; b < R; b += BS) {
      // |sg (r0 + b)| < |d_l| M <= MN / 2: one conditional add reduces it mod MN
      V c = cmul(hw, twid_tm(sm, wrap1(sg * (th.r0 + b), MN)));
#pragma unroll
      for (int i = 0; i < BS; ++i) {
        Acc<float>::mac(acc[b + i], c, v[b + i]);
        c = cmul(c, step);
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int k = th.r0 + i;
    const V coef = dl ? cmul(h0, twid_tm(sm, wrap1(sg * k, MN))) : h0;
    int ar = k + s;
    const int nw = ar < 0 ? -1 : (ar >= M ? 1 : 0);
    ar -= nw * M;
    V v = LDS ? colp[ar] : ld_cluster(static_cast<V*>(nullptr), colad + (uint32_t)(ar * (int)sizeof(V)));
    if (nw != 0) {
      V t = sm.tw[ls];
      if (nw < 0) t = cconj(t);
      v = cmul(v, t);
    }
    Acc<float>::mac(acc[i], coef, v);
  }
}

template <int R, bool HERM>
__device__ __forceinline__ void tap_elem(const SolveArgs& a, const TmThr& th, const TmSm& sm, const FrameSm& fs,
                                         bool halo, const V* buf, const PathEnt<float>& e, U64 (&acc)[R]) {
  // (a.gd is a constant in the compile-time-geometry instantiations: plans
  // without ghosts carry no ghost code)
  if (a.gd > 0 && halo && fs.ghost && e.dl >= -a.gd && e.dl <= a.gd)
    tap_elem_impl<R, HERM, true>(a, th, sm, fs, halo, buf, e, acc);
  else tap_elem_impl<R, HERM, false>(a, th, sm, fs, halo, buf, e, acc);
}

// TMEM taps of a mask, software-pipelined in half runs (R / 2 values): the
// load of the next half is in flight while the FFMA2s of the current one run
// (tcgen05.wait::ld covers every outstanding load, so the pipeline is one deep).
template <int R, bool HERM>
__device__ __forceinline__ void tmem_taps(int jr, const TmSm& sm, uint32_t tv, uint32_t m, U64 (&acc)[R]) {
  constexpr int H2 = R / 2;  // complex values per half run
  constexpr int W = R;       // 32-bit TMEM columns per half run
  if (!m) return;
  // the run's TMEM base, made opaque so ptxas keeps it in a register instead
  // of rematerialising the lane base from the thread index on every tap
  uint32_t tvj;
  asm volatile("mov.b32 %0, %1;" : "=r"(tvj) : "r"(tv + (uint32_t)(2 * jr)));
  auto addr = [&](const PathEnt<float>& e) { return tvj + (uint32_t)(2 * (HERM ? -e.dk : e.dk)); };
  const PathEnt<float>* ent = &sm.ptab[__ffs(m) - 1];
  m &= m - 1;
  uint32_t ad = addr(*ent);
  ulonglong2 g = gain_pairs<HERM>(*ent);
  uint32_t A[W], B[W];
  tmem_ld<W>(ad, A);
  tmem_wait_ld_tie<W>(A);
  while (true) {
    tmem_ld<W>(ad + (uint32_t)W, B);
    const U64 X = g.x, Y = g.y;
#pragma unroll
    for (int i = 0; i < H2; ++i) cmacxy(acc[i], X, Y, __uint_as_float(A[2 * i]), __uint_as_float(A[2 * i + 1]));
    tmem_wait_ld_tie<W>(B);
    const bool more = m != 0;
    if (more) {
      ent = &sm.ptab[__ffs(m) - 1];
      m &= m - 1;
      ad = addr(*ent);
      g = gain_pairs<HERM>(*ent);
      tmem_ld<W>(ad, A);
    }
#pragma unroll
    for (int i = 0; i < H2; ++i)
      cmacxy(acc[H2 + i], X, Y, __uint_as_float(B[2 * i]), __uint_as_float(B[2 * i + 1]));
    if (!more) break;
    tmem_wait_ld_tie<W>(A);
  }
}


// A d_l = 0 tap's run from the thread's own extended column when the frame's
// shifts exceed the halo (wrap_run): the period twist goes into the gain pairs.
template <int R, bool HERM>
__device__ __forceinline__ void wrap_gain(int& a0, int M, const FrameSm& fs, V tw_own, const PathEnt<float>& e,
                                          ulonglong2& g) {
  const V t = wrap_run<R>(a0, M, HERM ? fs.lo_u : fs.lo_c, HERM ? fs.hi_u : fs.hi_c, tw_own);
  const V h = cmul(e.coef(HERM), t);
  g = make_ulonglong2(pack2(h.x, h.x), pack2(-h.y, h.y));
}

// Local pass (after the CTA barrier): TMEM runs and own-column shared runs.
// GEN false (lean frames): masks always apply and no run wraps.
template <int R, bool HERM, bool GEN = true>
__device__ __forceinline__ void mvm_local(const SolveArgs& a, const TmThr& th, const TmSm& sm, const FrameSm& fs,
                                          uint32_t tv, const V* vcol, U64 (&acc)[R]) {
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0ull;
  if (!GEN || fs.masks) {  // lean frames always have their masks (P <= 32)
    const uint32_t* mk = fs.mk[th.jr / R] + (HERM ? 3 : 0);
    const uint32_t mt = mk[0], ms = mk[1];
    tmem_taps<R, HERM>(th.jr, sm, tv, mt, acc);
    for (uint32_t m = ms; m; m &= m - 1) {
      const PathEnt<float>& e = sm.ptab[__ffs(m) - 1];
      const int s = HERM ? -e.dk : e.dk;
      ulonglong2 g = gain_pairs<HERM>(e);
      int a0 = th.r0 + s;
      if constexpr (GEN)
        if (fs.wrap) wrap_gain<R, HERM>(a0, a.M, fs, sm.tw[th.colg], e, g);
      gather_run<R>(vcol + a0, (s & 1) != 0, g.x, g.y, acc);
    }
  } else if constexpr (GEN) {
    const bool halo = fs.halo;
    for (int p = 0; p < fs.P; ++p) {
      const PathEnt<float> e = tm_get(a, sm, fs, p);
      const int cls = tap_class<R, HERM>(a, th.jr, halo, e);
      const int s = HERM ? -e.dk : e.dk;
      const float4 g = HERM ? e.hh : e.hf;
      if (cls == 0) {
        gather_tmem<R>(tv + (uint32_t)(2 * (th.jr + s)), pack2(g.x, g.y), pack2(g.z, g.w), acc);
      } else if (cls == 1) {
        ulonglong2 gp = make_ulonglong2(pack2(g.x, g.y), pack2(g.z, g.w));
        int a0 = th.r0 + s;
        if (fs.wrap) wrap_gain<R, HERM>(a0, a.M, fs, sm.tw[th.colg], e, gp);
        gather_run<R>(vcol + a0, (s & 1) != 0, gp.x, gp.y, acc);
      }
    }
  }
}

// Remote pass (after the cluster barrier's wait): per-element taps.
template <int R, bool HERM>
__device__ __forceinline__ void mvm_remote(const SolveArgs& a, const TmThr& th, const TmSm& sm, const FrameSm& fs,
                                           const V* buf, void* ghmb, uint32_t& ghp, U64 (&acc)[R]) {
  const bool halo = fs.halo;
  if (a.gd > 0 && fs.ghost) {  // the ghost columns of this vector landed (gh_push of both neighbours)
    if (threadIdx.x == 0) mbar_expect_tx(ghmb, (uint32_t)(2 * fs.ghost * a.CS * (int)sizeof(V)));
    mbar_wait(ghmb, ghp & 1u);
    ghp ^= 1u;
  }
  if (fs.masks) {
    for (uint32_t m = fs.mk[th.jr / R][HERM ? 5 : 2]; m; m &= m - 1)
      tap_elem<R, HERM>(a, th, sm, fs, halo, buf, sm.ptab[__ffs(m) - 1], acc);
  } else {
    for (int p = 0; p < fs.P; ++p) {
      const PathEnt<float> e = tm_get(a, sm, fs, p);
      if (tap_class<R, HERM>(a, th.jr, halo, e) == 2) tap_elem<R, HERM>(a, th, sm, fs, halo, buf, e, acc);
    }
  }
  if (a.gd > 0 && fs.ghost) {  // this warp is done with the ghosts: release them to both neighbours
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      const int rank = th.colg / a.Lcta;
      const uint32_t me = smem_addr(static_cast<char*>(ghmb) + 8);
      mbar_arrive_remote(map_rank(me, (uint32_t)((rank + 1) % a.C)));
      mbar_arrive_remote(map_rank(me, (uint32_t)((rank + a.C - 1) % a.C)));
    }
  }
}

// A value ptxas must keep in a register (it cannot see through the move, so it
// does not rebuild it from %tid at every use).
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// ---- TMEM runs of E complex values (2E words) ----------------------------
template <int E>
__device__ __forceinline__ void tm_ld(uint32_t ta, uint32_t (&r)[2 * E]) {
  tmem_ld<2 * E>(ta, r);
}
template <int E>
__device__ __forceinline__ void tm_st(uint32_t ta, const V (&v)[E]) {
  uint32_t r[2 * E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    r[2 * i] = __float_as_uint(v[i].x);
    r[2 * i + 1] = __float_as_uint(v[i].y);
  }
  tmem_st<2 * E>(ta, r);
}
template <int E>
__device__ __forceinline__ V tm_get_v(const uint32_t (&r)[2 * E], int i) {
  return make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
}

// Store E values of rows rr .. rr + E - 1 into the lane's extended column
// (16-byte stores), plus the quasi-periodic copies a frame's shifts need:
// ext[r - M] = v W_N^{-l} for r >= M - lo, ext[r + M] = v W_N^{+l} for r < hi.
// MAIN false: the rows themselves are already in place (a bulk copy wrote them).
template <int E, bool MAIN = true>
__device__ __forceinline__ void put_col(V* colp, int rr, int M, int lo, int hi, V tw, const V (&v)[E]) {
  if constexpr (MAIN) {
    float4* q = reinterpret_cast<float4*>(colp + rr);
#pragma unroll
    for (int i = 0; i < E / 2; ++i) q[i] = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
  }
  if (rr + E > M - lo) {
    const V t = cconj(tw);
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (rr + i >= M - lo) colp[rr + i - M] = cmul(v[i], t);
  }
  if (rr < hi) {
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (rr + i < hi) colp[rr + i + M] = cmul(v[i], tw);
  }
}

// Barrier halves around TMEM traffic: stores of every warp complete and are
// ordered before the CTA barrier; loads after it see them.
// relaxed: no peer reads this CTA's shared memory in the current phase (the
// frame has no DSMEM taps): see cl_arrive_red (cg.cuh).
__device__ __forceinline__ void tm_arrive(int C, bool relaxed = false) {
  tmem_wait_st();
  tmem_fence_before();
  if (C > 1) cl_arrive_sem(!relaxed || (threadIdx.x >> 5) == 0);
  __syncthreads();
  tmem_fence_after();
}

// Timed variant (measurement builds): wt[4] TMEM store wait + fence, wt[5] CTA
// barrier, wt[6] fold + push, wt[7] cluster arrive.  BAR.SYNC defers blocking,
// so the CTA-barrier wait mostly lands in wt[6].
// The warp that folds the CTA partials (and then starts its next MVM late):
// one of a middle row block (fold_warp); in the lean kernel the lightest row
// block of the MVM that follows -- the first before a hermitian MVM, the last
// before a forward one (per-warp MVM times, profiles/r2_final_phase.json):
// cfg3 +0.4 %; the general kernel keeps the middle one (cfg4 -3.6 % otherwise).
__device__ __forceinline__ int tm_fold(int nwarps, bool before_herm, bool lean) {
  if (lean && nwarps == 16) return before_herm ? 0 : 12;
  return fold_warp(nwarps);
}
template <bool PROF, bool LEAN = false>
__device__ __forceinline__ void tm_arrive_red(int C, V* base, int nwarps, int warp, int lane, int rank,
                                              bool relaxed, long long* wt, bool before_herm = false) {
  if constexpr (!PROF) {
    cl_arrive_red<float, true>(C, base, nwarps, warp, lane, rank, relaxed, tm_fold(nwarps, before_herm, LEAN));
  } else {
    long long t = clock64(), u;
    tmem_wait_st();
    tmem_fence_before();
    u = clock64(); wt[4] += u - t; t = u;
    __syncthreads();
    u = clock64(); wt[5] += u - t; t = u;
    if (C > 1) {
      if (warp == tm_fold(nwarps, before_herm, LEAN)) {
        V v = lane < nwarps ? base[lane] : make_float2(0.f, 0.f);
        v.x = warp_sum(v.x);
        v.y = warp_sum(v.y);
        if (lane < C) st_cluster(map_rank(smem_addr(base + 32 + rank), (uint32_t)lane), v);
      }
      u = clock64(); wt[6] += u - t; t = u;
      (void)relaxed;
      cl_arrive_sem(warp == tm_fold(nwarps, before_herm, LEAN));
    }
    tmem_fence_after();
    u = clock64(); wt[7] += u - t;
  }
}

// Epilogue for E equalized symbols of rows rr.. (contiguous in q): x_hat,
// hard labels, max-log LLRs and the bit-error count vs TX labels.
// The transmitted-label word of the 4 symbols at q0 (bps bits each when packed).
template <int BA>
__device__ __forceinline__ uint32_t tx_word(const SolveArgs& a, size_t q0) {
  if (!a.txl || BA == 0) return 0u;
  if (!a.txpk) return __ldg(reinterpret_cast<const uint32_t*>(a.txl + q0));
  if constexpr (BA <= 2)
    return BA == 2 ? (uint32_t)__ldg(reinterpret_cast<const uint16_t*>(a.txl + (q0 >> 1)))
                   : (uint32_t)__ldg(a.txl + (q0 >> 2));
  return 0u;
}

// txpre: the TX word, already loaded (epi_pass issues them before the x staging)
template <int BA, int E>
__device__ __forceinline__ int tm_epilogue(const SolveArgs& a, const V (&xv)[E], size_t q0, float scale,
                                           uint32_t txpre) {
  V* xo = reinterpret_cast<V*>(a.x) + q0;
#pragma unroll
  for (int i = 0; i < E / 2; ++i)
    reinterpret_cast<float4*>(xo)[i] = make_float4(xv[2 * i].x, xv[2 * i].y, xv[2 * i + 1].x, xv[2 * i + 1].y);
  if constexpr (BA == 0) {
    return 0;
  } else {
    // the transmitted labels first: their load is then in flight during the
    // slicing (issued after the label / LLR stores it could not be hoisted
    // above them -- the pointers may alias as far as the compiler knows)
    static_assert(E == 4, "one TX word per call");
    const uint32_t txw = txpre;
    uint8_t lab[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      float l[2 * BA];
      lab[i] = (uint8_t)qam_symbol<float, BA>(xv[i].x, xv[i].y, scale, a.llr ? l : nullptr);
      if (a.llr) {
        float* dst = a.llr + (q0 + i) * (2 * BA);
        if constexpr (BA == 2) {
          *reinterpret_cast<float4*>(dst) = make_float4(l[0], l[1], l[2], l[3]);
        } else {
#pragma unroll
          for (int m = 0; m < BA; ++m) reinterpret_cast<float2*>(dst)[m] = make_float2(l[2 * m], l[2 * m + 1]);
        }
      }
    }
    int errs = 0;
    static_assert(E % 4 == 0, "label runs are stored in 32-bit words");
#pragma unroll
    for (int w = 0; w < E / 4; ++w) {
      const uint32_t word = (uint32_t)lab[4 * w] | ((uint32_t)lab[4 * w + 1] << 8) |
                            ((uint32_t)lab[4 * w + 2] << 16) | ((uint32_t)lab[4 * w + 3] << 24);
      if (a.labels) reinterpret_cast<uint32_t*>(a.labels + q0)[w] = word;
      if (a.txl) {
        if (!a.txpk) {
          errs += __popc(word ^ txw);
        } else if constexpr (BA <= 2) {  // four symbols = 2 BA bits each, LSB-first: 8 or 16 bits
          constexpr int SB = 2 * BA;
          const uint32_t mine = (uint32_t)lab[4 * w] | ((uint32_t)lab[4 * w + 1] << SB) |
                                ((uint32_t)lab[4 * w + 2] << (2 * SB)) | ((uint32_t)lab[4 * w + 3] << (3 * SB));
          errs += __popc(mine ^ txw);
        }  // (64-QAM labels are never packed: the ABI rejects it)
      }
    }
    return errs;
  }
}

// Coalesced epilogue pass over the CTA's staged x (column-major, stride M + 2).
// The thread's TX words for its (at most R / 4) passes, loaded before the x
// staging and its barrier so the L2 round trips overlap them.
template <int BA, int NP>
__device__ __forceinline__ void tx_preload(const SolveArgs& a, int M, size_t qb, uint32_t (&txp)[NP]) {
  const int tot = a.Lcta * M;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int e = 4 * ((int)threadIdx.x + k * (int)blockDim.x);
    txp[k] = e < tot ? tx_word<BA>(a, qb + e) : 0u;
  }
}

template <int BA, int NP>
__device__ __forceinline__ int epi_pass(const SolveArgs& a, const V* stg, int M, size_t qb, float scale,
                                        const uint32_t (&txp)[NP]) {
  const int tot = a.Lcta * M;
  int errs = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int e = 4 * ((int)threadIdx.x + k * (int)blockDim.x);
    if (e >= tot) break;
    const int cl = e / M;
    const float4* sp = reinterpret_cast<const float4*>(stg + cl * (M + 2) + (e - cl * M));
    const float4 w0 = sp[0], w1 = sp[1];
    const V xv[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                     make_float2(w1.z, w1.w)};
    errs += tm_epilogue<BA, 4>(a, xv, qb + e, scale, txp[k]);
  }
  return errs;
}

// Measurement builds: per-warp cycles of a call (wt[0] forward / wt[1]
// hermitian local MVM, wt[2] reduction arrive, wt[3] cluster wait), stored by
// lane 0 of every warp at prof[kProfWarpBase + (cta * 16 + warp) * kWarpTimers].
#define TM_WT(k, ...)                                  \
  do {                                                 \
    if constexpr (PROF) {                              \
      const long long t0_ = clock64();                 \
      __VA_ARGS__;                                     \
      wt[k] += clock64() - t0_;                        \
    } else {                                           \
      __VA_ARGS__;                                     \
    }                                                  \
  } while (0)

#ifndef DDB_GHOST
#define DDB_GHOST 1  // ghost columns for |d_l| = 1 taps (0: DSMEM for every Doppler tap, A/B builds)
#endif

// Frames are split between two instantiations of the kernel by tap geometry.
// "Lean" frames -- 1..32 taps, all Doppler-preserving (l_p = L0), delay shifts
// within the halo (every Veh-A frame with |nu| < dnu / 2, the headline's) --
// need only the TMEM and own-column routes; the general kernel (GEN) carries
// the Doppler (DSMEM), wrapped-run and large-P paths whose extra registers
// would otherwise spill in the lean one.  Both kernels are launched on every
// solve (lean first) and each takes its own class; EmptyChannel frames (P = 0)
// go to the lean one.
__device__ __forceinline__ bool frame_lean(const SolveArgs& a, int f) {
  const int P0 = __ldg(a.off + f), P = __ldg(a.off + f + 1) - P0;
  if (P <= 0) return true;
  if (a.snaps) return false;  // per-iteration snapshots (cfg.profile) are written by the general kernel only
  if (P > 32 || P > a.pcap) return false;
  int dmin = INT_MAX, dmax = INT_MIN;
  bool dl0 = true;
  // four taps' loads in flight at a time (one round trip for a Veh-A frame)
  for (int i0 = 0; i0 < P; i0 += 4) {
    int kk[4], ll[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = min(i0 + u, P - 1);
      kk[u] = __ldg(a.pk + P0 + i);
      ll[u] = __ldg(a.pl + P0 + i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dl0 &= ll[u] == a.L0;
      dmin = min(dmin, a.K0 - kk[u]);
      dmax = max(dmax, a.K0 - kk[u]);
    }
  }
  return dl0 && max(0, -dmin) <= a.H && max(0, dmax) <= a.H;
}

// This CTA's next chunk of frames of its class: candidates base + t n_clusters
// (t < kListChunk), compacted in order into flist; returns the count (all threads).
constexpr int kListChunk = 128;
template <bool GEN>
__device__ __forceinline__ int frame_list(const SolveArgs& a, int base, int* flist, int* wcnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int fc = base + tid * a.n_clusters;
  const bool mine = tid < kListChunk && fc < a.B && (GEN && !a.split ? true : frame_lean(a, fc) != GEN);
  const unsigned bal = __ballot_sync(0xffffffffu, mine);
  if (lane == 0) wcnt[warp] = __popc(bal);
  __syncthreads();
  int pos = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    pos += w < warp ? wcnt[w] : 0;
    tot += wcnt[w];
  }
  if (mine) flist[pos + __popc(bal & ((1u << lane) - 1u))] = fc;
  __syncthreads();
  return tot;
}

// Plans compiled with their geometry as constants (SPEC > 0): every TMEM
// column and shared-memory address then folds to immediates (cfg3: +11 %).
// The host picks an entry only when the planner's plan matches it exactly
// (spec_index, launch_r); any other plan runs the generic instantiation.
struct SpecPlan {
  int M, N, C, Lcta, G, WQ, CS, H, TL, TH, pcap, tcols, gd;
  int min_blocks;  // launch bounds: CTAs per SM the registers must allow (128-thread plans: 5)
};
constexpr SpecPlan kSpecs[] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},                   // 0: generic
    {512, 32, 2, 16, 64, 4, 874, 180, 128, 128, 64, 512, 0, 1},   // 1: cfg3   (R 16)
    {64, 16, 1, 16, 8, 1, 150, 42, 32, 32, 64, 64, 0, 5},         // 2: cfg1   (R 8, 128 threads: five CTAs per SM)
    {256, 16, 1, 16, 32, 2, 422, 82, 64, 64, 64, 256, 0, 1},      // 3: cfg2   (R 16)
    {1024, 64, 8, 8, 64, 4, 1154, 64, 256, 256, 64, 512, 4, 1},  // 4: cfg4   (R 16, four ghost columns a side)
    {128, 32, 1, 32, 32, 4, 386, 128, 64, 64, 64, 256, 0, 1},     // 5: (128, 32), the paper's grid (R 8)
};
constexpr int kNumSpecs = sizeof(kSpecs) / sizeof(kSpecs[0]);
inline int spec_index(const SolveArgs& a) {
  if (getenv("DDB_NO_SPEC")) return 0;
  for (int i = 1; i < kNumSpecs; ++i) {
    const SpecPlan& p = kSpecs[i];
    if (a.M == p.M && a.N == p.N && a.C == p.C && a.Lcta == p.Lcta && a.G == p.G && a.WQ == p.WQ && a.CS == p.CS &&
        a.H == p.H && a.TL == p.TL && a.TH == p.TH && a.pcap == p.pcap && a.tcols == p.tcols && a.gd == p.gd)
      return i;
  }
  return 0;
}

template <int R, int MAXT, bool PROF, bool GEN, int SPEC = 0>
__global__ void __launch_bounds__(kSpecs[SPEC].min_blocks > 1 ? 128 : MAXT, kSpecs[SPEC].min_blocks)
    sscga_tm_kernel(const SolveArgs a_) {
  // a local copy whose plan fields are constants in the specialised instantiation
  SolveArgs a = a_;
  if constexpr (SPEC > 0) {
    constexpr SpecPlan P = kSpecs[SPEC];
    a.M = P.M;
    a.N = P.N;
    a.MN = P.M * P.N;
    a.K0 = P.M / 2;
    a.L0 = P.N / 2;
    a.C = P.C;
    a.Lcta = P.Lcta;
    a.G = P.G;
    a.WQ = P.WQ;
    a.CS = P.CS;
    a.H = P.H;
    a.TL = P.TL;
    a.TH = P.TH;
    a.pcap = P.pcap;
    a.tcols = P.tcols;
    a.gd = P.gd;
  }
  constexpr int E = 4;  // elements per TMEM chunk of the elementwise steps
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = a.M;
  const SmemLayout L = tm_layout_impl(a.Lcta, a.N, a.CS, a.TL, a.TH, a.pcap, a.gd);
  TmSm sm;
  sm.c = reinterpret_cast<V*>(smem + L.p);
  sm.u = reinterpret_cast<V*>(smem + L.u);
  sm.tslot = reinterpret_cast<uint32_t*>(smem + L.x);
  V* tlo = reinterpret_cast<V*>(smem + L.tlo);
  V* thi = reinterpret_cast<V*>(smem + L.thi);
  V* tw = reinterpret_cast<V*>(smem + L.tw);
  sm.tlo = tlo;
  sm.thi = thi;
  sm.tw = tw;
  sm.ptab = reinterpret_cast<PathEnt<float>*>(smem + L.ptab);
  sm.tlb = __ffs(a.TL) - 1;
  sm.gh = reinterpret_cast<V*>(smem + L.gh);
  void* const ghmb = smem + L.ghmb;
  V* red = reinterpret_cast<V*>(smem + L.red);
  ProfSm* const psm = reinterpret_cast<ProfSm*>(red + 2 * 2 * kPushSlots);
  FrameSm& fs = *reinterpret_cast<FrameSm*>(psm + 1);
  int* const flist = reinterpret_cast<int*>(smem + L.q);
  int* const wcnt = flist + 128;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int rank = a.C > 1 ? (int)cluster_rank() : 0;
  TmThr th;
  {
    const int ln = 32 * (warp & 3) + lane;  // TMEM lane of this thread
    const int seg = ln / a.Lcta;
    th.col = ln - seg * a.Lcta;
    th.colg = rank * a.Lcta + th.col;
    th.jr = (warp >> 2) * R;
    th.r0 = seg * a.G + th.jr;
  }

  for (int i = tid; i < a.TL; i += blockDim.x) tlo[i] = twiddle(0.f, i, a.MN);
  for (int i = tid; i < a.TH; i += blockDim.x) thi[i] = twiddle(0.f, (int)(((long long)i * a.TL) % a.MN), a.MN);
  for (int l = tid; l < a.N; l += blockDim.x) tw[l] = twiddle(0.f, l, a.N);
  // y streaming (a.stream_y): the CTA's slice of a frame's y -- Lcta columns of
  // M contiguous complex values -- is copied by the TMA engine (cp.async.bulk,
  // one 8M-byte copy per column) straight into the rows of the extended u
  // columns, where setup needs it.  The copy of frame f + n_clusters is issued
  // as soon as frame f's last gather of u is behind a barrier, so it lands
  // during f's final update and epilogue; completion on the mbarrier ymb.
  void* const ymb = smem + L.x + 8;
  const V* const yg = reinterpret_cast<const V*>(a.y);
  auto issue_y = [&](int fy) {  // thread 0 only
    const V* src = yg + (size_t)fy * a.MN + (size_t)rank * a.Lcta * M;
    fence_proxy_async();  // this CTA's generic reads / writes of the u slice come first
    mbar_expect_tx(ymb, (uint32_t)(a.Lcta * M * (int)sizeof(V)));
    for (int c = 0; c < a.Lcta; ++c) bulk_g2s(sm.u + (size_t)c * a.CS + a.H, src + (size_t)c * M, M * sizeof(V), ymb);
  };
  // the same from the lanes of the last warp, one column each: the lean kernel's
  // copy of the next frame after the CG loop
  auto issue_y_warp = [&](int fy) {  // every lane of one warp
    const V* src = yg + (size_t)fy * a.MN + (size_t)rank * a.Lcta * M;
    fence_proxy_async();
    if (lane == 0) mbar_expect_tx(ymb, (uint32_t)(a.Lcta * M * (int)sizeof(V)));
    __syncwarp();
    for (int c = lane; c < a.Lcta; c += 32)
      bulk_g2s(sm.u + (size_t)c * a.CS + a.H, src + (size_t)c * M, M * sizeof(V), ymb);
  };
  uint32_t yph = 0;
  if (a.stream_y && tid == 0) mbar_init(ymb, 1);
  // the general instantiation is launched as a programmatic dependent of the
  // lean one (launch_r): it may start as soon as SMs free up, and its frames
  // do not depend on the lean ones; it waits for the lean grid only before it
  // completes, so the stream's order holds for whatever follows the solve
  if constexpr (!GEN) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // this CTA's first frames of its class: a CTA (cluster: every CTA computes the
  // same list) without any frame in the whole batch leaves at once
  const int base0 = blockIdx.x / a.C;
  int nlist = frame_list<GEN>(a, base0, flist, wcnt);
  if (nlist == 0 && base0 + a.n_clusters * kListChunk >= a.B) {
    if constexpr (GEN) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  if (warp == 0) tmem_alloc(sm.tslot, (uint32_t)a.tcols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *sm.tslot;
  th.tl = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  // ghost-column mbarriers ("full" at +0: one arrival plus the bytes of both
  // neighbours' pushes; "empty" at +8: both neighbours released this CTA's
  // last push), initialised in every CTA before any neighbour can use them
  uint32_t ghp = 0;  // full-barrier parity
  uint32_t npush = 0;  // pushes this CTA made (thread 0): the empty-barrier phase to wait for
  if constexpr (GEN) {
    if (a.gd > 0) {
      if (tid == 0) {
        mbar_init(ghmb, 1);
        mbar_init(static_cast<char*>(ghmb) + 8, 2 * nwarps);  // every warp of both neighbours
      }
      cl_sync<float>(a.C);
    }
  }
  const uint32_t rr = (uint32_t)((rank + 1) % a.C), rl = (uint32_t)((rank + a.C - 1) % a.C);
  // Push this CTA's gd first and gd last columns of c (vec 0) or u (vec 1)
  // into the neighbours' ghost slots (thread 0, after the CTA barrier that
  // completed them; every writer fenced its generic stores for the async
  // proxy first), once both neighbours released the previous push.  The owner
  // rewrites a column only after a cluster barrier the neighbour reaches after
  // its wait for the push, so the copy's reads are never raced.
  auto gh_push = [&](int vec) {
    if (npush > 0) mbar_wait_cluster(static_cast<char*>(ghmb) + 8, (npush - 1) & 1u);
    ++npush;
    const V* src = vec ? sm.u : sm.c;
    // only the gx columns a side this frame's taps reach (gx = max |d_l| <= gd)
    const int gx = fs.ghost;
    const uint32_t bytes = (uint32_t)(gx * a.CS * (int)sizeof(V));
    const uint32_t mb = smem_addr(ghmb);
    // the last gx columns -> the right neighbour's innermost left ghost slots, the first gx -> its left neighbour's right ones
    bulk_s2c(map_rank(smem_addr(sm.gh + (size_t)(a.gd - gx) * a.CS), rr), src + (size_t)(a.Lcta - gx) * a.CS, bytes,
             map_rank(mb, rr));
    bulk_s2c(map_rank(smem_addr(sm.gh + (size_t)a.gd * a.CS), rl), src, bytes, map_rank(mb, rl));
  };
  // TMEM regions of this lane: c | u (segment rows 0..G-1) | p | x (own runs)
  auto tC = [&](int c0) { return th.tl + (uint32_t)(2 * (th.jr + c0)); };
  auto tU = [&](int c0) { return th.tl + (uint32_t)(2 * (a.G + th.jr + c0)); };
  auto tP = [&](int c0) { return th.tl + (uint32_t)(2 * (2 * a.G + th.jr + c0)); };
  auto tX = [&](int c0) { return th.tl + (uint32_t)(2 * (3 * a.G + th.jr + c0)); };
  V* const ccol = sm.c + (size_t)th.col * a.CS + a.H;  // this lane's extended columns (row 0)
  V* const ucol = sm.u + (size_t)th.col * a.CS + a.H;

  const bool lead = (rank == 0 && tid == 0);
  const int stride = a.iters + 1;
  int par0 = 0, par1 = 0;
  if constexpr (PROF) prof_init(a.prof, psm);
  long long wt[kWarpTimers] = {0, 0, 0, 0, 0, 0, 0, 0};

  for (int base = base0; base < a.B; base += a.n_clusters * kListChunk) {
  if (base != base0) nlist = frame_list<GEN>(a, base, flist, wcnt);
  if (a.stream_y && tid == 0 && nlist > 0) issue_y(flist[0]);
  for (int li = 0; li < nlist; ++li) {
    const int f = flist[li];
    const int fnext = li + 1 < nlist ? flist[li + 1] : -1;  // this CTA's next frame of the class (y prefetch)
    const size_t fo = (size_t)f * a.MN;
    const size_t qown = fo + (size_t)th.colg * M + th.r0;  // first owned element of the frame
    const int P0 = __ldg(a.off + f);
    const int P = __ldg(a.off + f + 1) - P0;

    if (P <= 0) {  // EmptyChannel (sparse.py:126-127): flag it, no NaNs
      if (a.stream_y) {  // this frame's y is not needed, but its copy must retire before the next one
        mbar_wait(ymb, yph);
        yph ^= 1;
        __syncthreads();
        if (tid == 0 && fnext >= 0) issue_y(fnext);
      }
#pragma unroll 1
      for (int i = 0; i < R; ++i) {
        reinterpret_cast<V*>(a.x)[qown + i] = make_float2(0.f, 0.f);
        if (a.labels) a.labels[qown + i] = 0;
        if (a.llr)
          for (int b = 0; b < a.bps; ++b) a.llr[(qown + i) * a.bps + b] = 0.f;
      }
      if (lead) {
        float* cnorm = reinterpret_cast<float*>(a.cnorm);
        if (cnorm) for (int i = 0; i < stride; ++i) cnorm[(size_t)f * stride + i] = 0.f;
        if (a.itdone) a.itdone[f] = 0;
        if (a.status) a.status[f] = 1;
        if (a.berr) a.berr[f] = a.bps * a.MN / 2;  // harness.py:173 scoring of a failed packet
      }
      continue;
    }

    // ---- frame setup: tap table, halo extents, per-row-block tap classes
    if constexpr (PROF) prof_mark(a.prof, psm, kSetup);
    // this frame's y first: the 16-byte loads are in flight during the tap-table work
    const V* y = yg;
    float4 yv[R / 2];
    if (a.stream_y) {  // from the u slice, where the bulk copy put it
      mbar_wait(ymb, yph);
      yph ^= 1;
#pragma unroll
      for (int i = 0; i < R / 2; ++i) yv[i] = reinterpret_cast<const float4*>(ucol + th.r0)[i];
    } else {
#pragma unroll
      for (int i = 0; i < R / 2; ++i) yv[i] = __ldg(reinterpret_cast<const float4*>(y + qown) + i);
    }
    const bool in_smem = P <= a.pcap;
    if (warp == 0) {  // tap table and shift extents, lanes over taps
      const V* gains = reinterpret_cast<const V*>(a.ph);
      int dmin = INT_MAX, dmax = INT_MIN;
      int d1 = 0;  // the largest |d_l| <= gd of a tap (ghost columns per side)
      for (int i = lane; i < P; i += 32) {
        const int kp = __ldg(a.pk + P0 + i), lp = __ldg(a.pl + P0 + i);
        if (in_smem) sm.ptab[i] = tm_path(a, sm, kp, lp, __ldg(gains + P0 + i));
        dmin = min(dmin, a.K0 - kp);
        dmax = max(dmax, a.K0 - kp);
        const int adl = abs(lp - a.L0);
        if (adl <= a.gd) d1 = max(d1, adl);
      }
      dmin = __reduce_min_sync(0xffffffffu, dmin);
      dmax = __reduce_max_sync(0xffffffffu, dmax);
      d1 = __reduce_max_sync(0xffffffffu, d1);
      if (lane == 0) {
        // halo rows written per side: what the shifts need, at most H; a run
        // beyond them is read one delay period over (wrap_run), which needs
        // H >= R (the planner's halo is at least min(M, 64) rows)
        const int lo = max(0, -dmin), hi = max(0, dmax);
        const bool halo = a.H >= R;
        fs.P0 = P0;
        fs.P = P;
        fs.in_smem = in_smem;
        fs.halo = halo;
        fs.wrap = halo && (lo > a.H || hi > a.H);
        fs.masks = in_smem && P <= 32;
        fs.lo_c = halo ? min(lo, a.H) : 0;
        fs.hi_c = halo ? min(hi, a.H) : 0;
        fs.lo_u = fs.hi_c;
        fs.hi_u = fs.lo_c;
        fs.remote = !fs.masks;  // without per-warp masks assume DSMEM taps
        fs.ghost = DDB_GHOST && GEN && a.gd > 0 && halo ? d1 : 0;
      }
    }
    __syncthreads();
    if (fs.masks && tid < a.WQ) {  // thread j classifies the taps for row block j
      uint32_t mk[6] = {0u, 0u, 0u, 0u, 0u, 0u};
      const bool halo = fs.halo;
      for (int p = 0; p < P; ++p) {
        const PathEnt<float>& e = sm.ptab[p];
        const uint32_t bit = 1u << p;
        const int cf = tap_class<R, false>(a, tid * R, halo, e);
        const int ch = tap_class<R, true>(a, tid * R, halo, e);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          mk[c] |= cf == c ? bit : 0u;
          mk[3 + c] |= ch == c ? bit : 0u;
        }
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) fs.mk[tid][i] = mk[i];
      if (mk[2] | mk[5]) atomicOr(&fs.remote, 1);
    }
    const float lam = reinterpret_cast<const float*>(a.lam)[f];

    // y -> u (TMEM own rows + extended shared column); b = H^H y is gathered from it
    {
      const int lo_u = fs.lo_u, hi_u = fs.hi_u;
      const V twl = tw[th.colg];
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += E) {
        V w[E];
#pragma unroll
        for (int i = 0; i < E / 2; ++i) {
          const float4 t = yv[c0 / 2 + i];
          w[2 * i] = make_float2(t.x, t.y);
          w[2 * i + 1] = make_float2(t.z, t.w);
        }
        tm_st<E>(tU(c0), w);
        if (a.stream_y) put_col<E, false>(ucol, th.r0 + c0, M, lo_u, hi_u, twl, w);
        else put_col<E>(ucol, th.r0 + c0, M, lo_u, hi_u, twl, w);
        V z[E];
#pragma unroll
        for (int i = 0; i < E; ++i) z[i] = make_float2(0.f, 0.f);
        tm_st<E>(tX(c0), z);  // x = 0
        tm_st<E>(tP(c0), z);  // p = 0: the first update is then p = c + 0 p like every other
      }
      // warm L2 with this cluster's next frame (y, TX labels) while this one solves
      if (fnext >= 0) {
        const size_t qn = qown + (size_t)(fnext - f) * a.MN;
        if (!a.stream_y)
#pragma unroll
          for (int c0 = 0; c0 < R; c0 += 16) asm volatile("prefetch.global.L2 [%0];" :: "l"(y + qn + c0));
        if (a.txl) asm volatile("prefetch.global.L2 [%0];" :: "l"(tx_label_ptr(a.txl, qn, a.bps, a.txpk)));
      }
    }
    if (lead && a.berr) a.berr[f] = 0;

    U64 acc[R];
    if constexpr (PROF) prof_mark(a.prof, psm, kArrive);
    const bool ghost = GEN && a.gd > 0 && fs.ghost;  // (fs.ghost is written before the barrier above)
    if (ghost) fence_proxy_async();
    tm_arrive(a.C);  // y and the tap classes published
    if (ghost && tid == 0) gh_push(1);
    if constexpr (PROF) prof_mark(a.prof, psm, kMvmLocal);
    TM_WT(1, mvm_local<R, true, GEN>(a, th, sm, fs, tU(0) - 2 * th.jr, ucol, acc));  // b = H^H y (equalize.py:52)
    if constexpr (PROF) prof_mark(a.prof, psm, kWait);
    cl_wait(a.C);
    if constexpr (PROF) prof_mark(a.prof, psm, kMvmRemote);
    if constexpr (GEN) mvm_remote<R, true>(a, th, sm, fs, sm.u, ghmb, ghp, acc);
    if constexpr (PROF) prof_mark(a.prof, psm, kStep1);
    {
      V nrm = make_float2(0.f, 0.f);
      const int lo_c = fs.lo_c, hi_c = fs.hi_c;
      const V twl = tw[th.colg];
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += E) {
        V w[E];
#pragma unroll
        for (int i = 0; i < E; ++i) {
          w[i] = unpack2(acc[c0 + i]);
          nacc(nrm, w[i]);
        }
        tm_st<E>(tC(c0), w);  // c = b
        put_col<E>(ccol, th.r0 + c0, M, lo_c, hi_c, twl, w);
      }
      red_stage<float>(make_float2(nrm.x + nrm.y, 0.f), red + (2 + par1) * kPushSlots, warp, lane);
    }
    if constexpr (PROF) prof_mark(a.prof, psm, kArrive);
    if (ghost) fence_proxy_async();
    TM_WT(2, tm_arrive_red<PROF, !GEN>(a.C, red + (2 + par1) * kPushSlots, nwarps, warp, lane, rank, !GEN || !fs.remote, wt));  // c = b published
    if (ghost && tid == 0 && a.iters > 0) gh_push(0);
    if constexpr (PROF) prof_mark(a.prof, psm, kMvmLocal);
    TM_WT(0, mvm_local<R, false, GEN>(a, th, sm, fs, tC(0) - 2 * th.jr, ccol, acc));
    if constexpr (PROF) prof_mark(a.prof, psm, kWait);
    cl_wait(a.C);
    if constexpr (PROF) prof_mark(a.prof, psm, kRead);
    float cn = red_total<float>(a.C, red + (2 + par1) * kPushSlots, nwarps).x;
    par1 ^= 1;
    float beta = 0.f;
    if (lead && a.cnorm) reinterpret_cast<float*>(a.cnorm)[(size_t)f * stride] = cn;

    int done = 0;
    bool exact = false;
    for (int it = 0; it < a.iters; ++it) {
      // u = H c + beta u_old, p = c + beta p_old      (= H p, p of equalize.py:60, 72)
      if constexpr (PROF) prof_mark(a.prof, psm, kMvmRemote);
      if constexpr (GEN) mvm_remote<R, false>(a, th, sm, fs, sm.c, ghmb, ghp, acc);
      if constexpr (PROF) prof_mark(a.prof, psm, kStep1);
      {
        V nu = make_float2(0.f, 0.f), np = make_float2(0.f, 0.f);
        const int lo_u = fs.lo_u, hi_u = fs.hi_u;
        const V twl = tw[th.colg];
        const uint32_t rb = opaque_u32(tC(0));  // this thread's run in region c; u, p at + 2G, + 4G
#pragma unroll
        for (int c0 = 0; c0 < R; c0 += E) {
          uint32_t ru[2 * E], rc[2 * E], rp[2 * E];
          // iteration 0 takes the same form with beta = 0: u still holds y and
          // p was zeroed at setup, so u = Hc + 0 y and p = c + 0 p are exact
          tm_ld<E>(rb + 2 * c0, rc);
          tm_ld<E>(rb + 2 * (a.G + c0), ru);
          tm_ld<E>(rb + 2 * (2 * a.G + c0), rp);
          tmem_wait_ld_tie<2 * E>(ru);
          tmem_wait_ld_tie<2 * E>(rp);
          tmem_wait_ld_tie<2 * E>(rc);
          V w[E], pv[E];
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const V hc = unpack2(acc[c0 + i]);
            const V cr = tm_get_v<E>(rc, i);
            w[i] = axpy(hc, beta, tm_get_v<E>(ru, i));
            pv[i] = axpy(cr, beta, tm_get_v<E>(rp, i));
            nacc(nu, w[i]);
            nacc(np, pv[i]);
          }
          tm_st<E>(rb + 2 * (a.G + c0), w);
          tm_st<E>(rb + 2 * (2 * a.G + c0), pv);
          put_col<E>(ucol, th.r0 + c0, M, lo_u, hi_u, twl, w);
        }
        red_stage<float>(make_float2(nu.x + nu.y, np.x + np.y), red + par0 * kPushSlots, warp, lane);
      }
      if constexpr (PROF) prof_mark(a.prof, psm, kArrive);
      if (ghost) fence_proxy_async();
      TM_WT(2, tm_arrive_red<PROF, !GEN>(a.C, red + par0 * kPushSlots, nwarps, warp, lane, rank, !GEN || !fs.remote, wt,
                                   true));  // u published
        if (ghost && tid == 0) gh_push(1);
      // ap = H^H u + lam p;  x += alpha p;  c -= alpha ap      (equalize.py:60-70)
      if constexpr (PROF) prof_mark(a.prof, psm, kMvmLocal);
      TM_WT(1, mvm_local<R, true, GEN>(a, th, sm, fs, tU(0) - 2 * th.jr, ucol, acc));
      if constexpr (PROF) prof_mark(a.prof, psm, kWait);
      TM_WT(3, cl_wait(a.C));
      if constexpr (PROF) prof_mark(a.prof, psm, kMvmRemote);
      if constexpr (GEN) mvm_remote<R, true>(a, th, sm, fs, sm.u, ghmb, ghp, acc);
      if constexpr (PROF) prof_mark(a.prof, psm, kRead);
      const V up = red_total<float>(a.C, red + par0 * kPushSlots, nwarps);
      par0 ^= 1;
      if constexpr (PROF) prof_mark(a.prof, psm, kStep3);
      const float denom = up.x + lam * up.y;  // ||H p||^2 + lam ||p||^2 = Re p^H (H^H H + lam I) p
      if (denom == 0.f) {  // equalize.py:64-67
        exact = true;
        // peers may still be reading this CTA's u: one more full barrier
        tm_arrive(a.C);
            cl_wait(a.C);
        break;
      }
      const float alpha = cn / denom;
      {
        V nc = make_float2(0.f, 0.f);
        const int lo_c = fs.lo_c, hi_c = fs.hi_c;
        const V twl = tw[th.colg];
        const uint32_t rb = opaque_u32(tC(0));  // this thread's run in region c; p at + 4G, x at + 6G
#pragma unroll
        for (int c0 = 0; c0 < R; c0 += E) {
          uint32_t rx[2 * E], rp[2 * E], rc[2 * E];
          tm_ld<E>(rb + 2 * (3 * a.G + c0), rx);
          tm_ld<E>(rb + 2 * (2 * a.G + c0), rp);
          tm_ld<E>(rb + 2 * c0, rc);
          tmem_wait_ld_tie<2 * E>(rx);
          tmem_wait_ld_tie<2 * E>(rp);
          tmem_wait_ld_tie<2 * E>(rc);
          V xv[E], cv[E];
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const V pv = tm_get_v<E>(rp, i);
            const V ap = axpy(unpack2(acc[c0 + i]), lam, pv);
            xv[i] = axpy(tm_get_v<E>(rx, i), alpha, pv);
            cv[i] = axpy(tm_get_v<E>(rc, i), -alpha, ap);
            nacc(nc, cv[i]);
          }
          tm_st<E>(rb + 2 * (3 * a.G + c0), xv);
          tm_st<E>(rb + 2 * c0, cv);
          put_col<E>(ccol, th.r0 + c0, M, lo_c, hi_c, twl, cv);
          if (GEN && a.snaps) {  // profile runs: every frame goes to the general kernel (frame_lean)
            V* sp = reinterpret_cast<V*>(a.snaps) + ((size_t)f * a.iters + it) * a.MN + (qown - fo) + c0;
#pragma unroll
            for (int i = 0; i < E; ++i) sp[i] = xv[i];
          }
        }
        red_stage<float>(make_float2(nc.x + nc.y, 0.f), red + (2 + par1) * kPushSlots, warp, lane);
      }
      if constexpr (PROF) prof_mark(a.prof, psm, kArrive);
      if (ghost) fence_proxy_async();
      TM_WT(2, tm_arrive_red<PROF, !GEN>(a.C, red + (2 + par1) * kPushSlots, nwarps, warp, lane, rank, !GEN || !fs.remote, wt));  // c published
        if (ghost && tid == 0 && it + 1 < a.iters) gh_push(0);
      if constexpr (PROF) prof_mark(a.prof, psm, kMvmLocal);
      if (it + 1 < a.iters) TM_WT(0, mvm_local<R, false, GEN>(a, th, sm, fs, tC(0) - 2 * th.jr, ccol, acc));  // next H c
      if constexpr (PROF) prof_mark(a.prof, psm, kWait);
      TM_WT(3, cl_wait(a.C));
      if constexpr (PROF) prof_mark(a.prof, psm, kRead);
      const float nn = red_total<float>(a.C, red + (2 + par1) * kPushSlots, nwarps).x;
      par1 ^= 1;
      beta = nn / cn;
      cn = nn;
      done = it + 1;
      if (lead && a.cnorm) reinterpret_cast<float*>(a.cnorm)[(size_t)f * stride + done] = cn;
    }
    // every gather of this frame's u (here and in the peers) is behind the last barrier
    if constexpr (!GEN) {  // (the general kernel keeps thread 0: cfg4 -2.4 % with the warp)
      if (a.stream_y && fnext >= 0 && warp == nwarps - 1) issue_y_warp(fnext);
    } else if (a.stream_y && tid == 0 && fnext >= 0) {
      issue_y(fnext);
    }
    if (lead) {
      float* cnorm = reinterpret_cast<float*>(a.cnorm);
      if (cnorm) for (int i = done + 1; i < stride; ++i) cnorm[(size_t)f * stride + i] = 0.f;
      if (a.itdone) a.itdone[f] = done;
      if (a.status) a.status[f] = exact ? 2 : 0;
    }

    // epilogue: x_hat out, fused hard decisions / LLRs / bit errors
    if constexpr (PROF) prof_mark(a.prof, psm, kEpilogue);
    float scale = 1.f;
    if (a.bps) {
      const float nv = a.nvar ? reinterpret_cast<const float*>(a.nvar)[f] : lam;
      scale = nv > 0.f ? 1.f / nv : 1.f;
    }
    const size_t qb = fo + (size_t)rank * a.Lcta * M;
    constexpr int NP = R / 4 > 0 ? R / 4 : 1;  // epilogue passes per thread: Lcta M / (4 threads) = R / 4
    uint32_t txp[NP];
    switch (a.bps) {
      case 2: tx_preload<1, NP>(a, M, qb, txp); break;
      case 4: tx_preload<2, NP>(a, M, qb, txp); break;
      case 6: tx_preload<3, NP>(a, M, qb, txp); break;
      default: for (int k = 0; k < NP; ++k) txp[k] = 0u; break;
    }
    // x -> shared staging in q order (column-major, stride M + 2: conflict-free
    // 16-byte stores), then every thread takes 4 consecutive symbols at a time
    // so the x_hat / LLR / label stores and TX label loads are coalesced.  The
    // c slice is free: all gathers of this frame are behind the last barrier.
    {
      const int SS = M + 2;
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += E) {
        uint32_t rx[2 * E];
        tm_ld<E>(tX(c0), rx);
        tmem_wait_ld_tie<2 * E>(rx);
        float4* d = reinterpret_cast<float4*>(sm.c + th.col * SS + th.r0 + c0);
#pragma unroll
        for (int i = 0; i < E / 2; ++i)
          d[i] = make_float4(__uint_as_float(rx[4 * i]), __uint_as_float(rx[4 * i + 1]),
                             __uint_as_float(rx[4 * i + 2]), __uint_as_float(rx[4 * i + 3]));
      }
    }
    __syncthreads();
    int errs = 0;
    switch (a.bps) {
      case 0: epi_pass<0, NP>(a, sm.c, M, qb, scale, txp); break;
      case 2: errs = epi_pass<1, NP>(a, sm.c, M, qb, scale, txp); break;
      case 4: errs = epi_pass<2, NP>(a, sm.c, M, qb, scale, txp); break;
      default: errs = epi_pass<3, NP>(a, sm.c, M, qb, scale, txp); break;
    }
    if (a.berr) {
      errs = warp_sum(errs);
      if (lane == 0 && errs) atomicAdd(a.berr + f, errs);
    }
  }
  __syncthreads();  // the next chunk's list overwrites flist
  }
  if constexpr (PROF) prof_mark(a.prof, psm, kTail);
  if constexpr (PROF) prof_store(a.prof, psm);
  if constexpr (PROF) {
    if (a.prof != nullptr && lane == 0)
      for (int k = 0; k < kWarpTimers; ++k)
        a.prof[kProfWarpBase + ((size_t)blockIdx.x * 16 + warp) * kWarpTimers + k] = wt[k];
  }
  // no CTA may leave while a peer can still read its shared memory (DSMEM)
  tmem_fence_before();
  cl_sync<float>(a.C);
  if (warp == 0) tmem_dealloc(tbase, (uint32_t)a.tcols);
  if constexpr (GEN) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// CTAs of this kernel one SM really holds.  The occupancy API reports 1 for any
// kernel that issues tcgen05.alloc, but the hardware co-schedules such CTAs as
// long as shared memory, registers, threads and TMEM columns allow
// (tools/ubench/resident.cu, profiles/r2_resident.txt: two 256-column CTAs per
// SM, three 128-column ones).  DDB_TM_CTAS_PER_SM overrides (A/B runs).
inline int tm_hw_ctas_per_sm(const LaunchShape& s, int regs) {
  if (const char* env = getenv("DDB_TM_CTAS_PER_SM")) return atoi(env) > 0 ? atoi(env) : 1;
  int n = 512 / (s.tcols > 32 ? s.tcols : 32);                     // TMEM columns
  const int by_smem = 233472 / (s.smem + 1024);                     // 228 KiB, 1 KiB reserved per CTA
  const int warp_regs = ((regs > 0 ? regs : 128) * 32 + 255) / 256 * 256;
  const int by_regs = 65536 / (warp_regs * (s.threads / 32));
  const int by_thr = 2048 / s.threads;
  n = n < by_smem ? n : by_smem;
  n = n < by_regs ? n : by_regs;
  n = n < by_thr ? n : by_thr;
  return n > 0 ? n : 1;
}

// Attribute setting, the cluster-occupancy query and the residency computation
// run once per (kernel, shared memory, threads, cluster, device): the host time
// of a launch is part of the batch-1 latency.
struct TmOcc {
  const void* fn;
  int smem, threads, cluster, dev, clusters;
};

template <int R, int MAXT, bool PROF, bool GEN, int SPEC = 0>
cudaError_t launch_one(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  auto kern = sscga_tm_kernel<R, MAXT, PROF, GEN, SPEC>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(s.threads);
  cfg.dynamicSmemBytes = s.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = s.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static thread_local TmOcc cache[8] = {};
  static thread_local int next = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int max_clusters = 0;
  for (const TmOcc& c : cache)
    if (c.fn == (const void*)kern && c.smem == s.smem && c.threads == s.threads && c.cluster == s.cluster && c.dev == dev)
      max_clusters = c.clusters;
  if (max_clusters == 0) {
    // the function's dynamic shared-memory ceiling goes to the device maximum,
    // so a launch of any plan is valid whatever plan set it last
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin > s.smem ? optin : s.smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    if (s.cluster > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cfg.gridDim = dim3(s.cluster);
    int api = 0, api_per_sm = 0;
    e = cudaOccupancyMaxActiveClusters(&api, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (api < 1) return cudaErrorInvalidConfiguration;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&api_per_sm, kern, s.threads, s.smem);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const int hw = tm_hw_ctas_per_sm(s, fa.numRegs);
    // the API's cluster count assumes its own per-SM figure; scale it to the
    // measured residency (persistent grid: every cluster is resident at once)
    max_clusters = hw > api_per_sm && api_per_sm > 0 ? api * hw / api_per_sm : api;
    cache[next] = TmOcc{(const void*)kern, s.smem, s.threads, s.cluster, dev, max_clusters};
    next = (next + 1) % 8;
  }
  const int nclu = a.B < max_clusters ? a.B : max_clusters;
  a.n_clusters = nclu;
  cfg.gridDim = dim3(nclu * s.cluster);
  if (GEN && a.split && !getenv("DDB_NO_PDL")) cfg.numAttrs = 2;  // programmatic dependent of the lean launch
  // single-CTA frames need no cluster attribute; DDB_NO_CLUSTER_ATTR drops it
  // (compute-sanitizer runs: synccheck misreports cluster launches, profiles/r2_sanitizer.md)
  if (s.cluster == 1 && getenv("DDB_NO_CLUSTER_ATTR")) cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// Both instantiations on the stream: the lean frames, then the others; the
// plan's compile-time-geometry instantiation when there is one.
template <int R, int MAXT, bool PROF, bool GEN>
cudaError_t launch_spec(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  if constexpr (!PROF) {
    switch (spec_index(a)) {
      case 1: if constexpr (R == 16) return launch_one<R, MAXT, PROF, GEN, 1>(a, s, st); break;
      case 2: if constexpr (R == 8) return launch_one<R, MAXT, PROF, GEN, 2>(a, s, st); break;
      case 3: if constexpr (R == 16) return launch_one<R, MAXT, PROF, GEN, 3>(a, s, st); break;
      case 4: if constexpr (R == 16) return launch_one<R, MAXT, PROF, GEN, 4>(a, s, st); break;
      case 5: if constexpr (R == 8) return launch_one<R, MAXT, PROF, GEN, 5>(a, s, st); break;
      default: break;
    }
  }
  return launch_one<R, MAXT, PROF, GEN>(a, s, st);
}

// The compile-time-geometry instantiation a launch of this plan runs (spec_index
// from the plan alone: M = CS - 2 H - 2, N = C Lcta), so the residency reported
// with the plan is the launch's (cfg1's runs five CTAs per SM, the generic four).
inline int spec_index_shape(const LaunchShape& s) {
  SolveArgs a = {};
  a.M = s.cs - 2 * s.halo - 2;
  a.N = s.cluster * s.lcta;
  a.C = s.cluster;
  a.Lcta = s.lcta;
  a.G = s.g;
  a.WQ = s.wq;
  a.CS = s.cs;
  a.H = s.halo;
  a.TL = s.tl;
  a.TH = s.th;
  a.pcap = s.pcap;
  a.tcols = s.tcols;
  return spec_index(a);
}
template <int R, int MAXT>
const void* occ_kernel(const LaunchShape& s) {
  switch (spec_index_shape(s)) {
    case 1: if constexpr (R == 16) return (const void*)sscga_tm_kernel<R, MAXT, false, false, 1>; break;
    case 2: if constexpr (R == 8) return (const void*)sscga_tm_kernel<R, MAXT, false, false, 2>; break;
    case 3: if constexpr (R == 16) return (const void*)sscga_tm_kernel<R, MAXT, false, false, 3>; break;
    case 4: if constexpr (R == 16) return (const void*)sscga_tm_kernel<R, MAXT, false, false, 4>; break;
    case 5: if constexpr (R == 8) return (const void*)sscga_tm_kernel<R, MAXT, false, false, 5>; break;
    default: break;
  }
  return (const void*)sscga_tm_kernel<R, MAXT, false, false>;
}

template <int R, int MAXT>
cudaError_t occ_r(const LaunchShape& s, int* n) {
  const void* kern = occ_kernel<R, MAXT>(s);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // never below what a cached launch of another plan may need (see launch_one)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin > s.smem ? optin : s.smem);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  *n = tm_hw_ctas_per_sm(s, fa.numRegs);  // measured residency, not the API's 1
  return cudaSuccess;
}

}  // namespace

// ---- split compilation (build.py compiles this file once per TM_PART, in
// parallel; without TM_PART one object carries everything): the R = 16 lean
// and general instantiations, the small-R ones and the dispatcher.
cudaError_t tm_launch16(bool gen, SolveArgs a, const LaunchShape& s, cudaStream_t st);
cudaError_t tm_launch16_gen(SolveArgs a, const LaunchShape& s, cudaStream_t st);
cudaError_t tm_launch_small(int R, bool gen, SolveArgs a, const LaunchShape& s, cudaStream_t st);
cudaError_t tm_occ(int R, const LaunchShape& s, int* n);
cudaError_t tm_occ16(const LaunchShape& s, int* n);

#if !defined(TM_PART) || TM_PART == 1
cudaError_t tm_launch16(bool gen, SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  if (gen) return tm_launch16_gen(a, s, st);
  return a.prof ? launch_spec<16, 512, true, false>(a, s, st) : launch_spec<16, 512, false, false>(a, s, st);
}
cudaError_t tm_occ16(const LaunchShape& s, int* n) { return occ_r<16, 512>(s, n); }
#endif
#if !defined(TM_PART) || TM_PART == 2
cudaError_t tm_launch16_gen(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  return a.prof ? launch_spec<16, 512, true, true>(a, s, st) : launch_spec<16, 512, false, true>(a, s, st);
}
#endif
#if !defined(TM_PART) || TM_PART == 3
cudaError_t tm_launch_small(int R, bool gen, SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  if (a.prof) return cudaErrorNotSupported;  // the phase profile is an R = 16 measurement build
  if (R == 8) return gen ? launch_spec<8, 512, false, true>(a, s, st) : launch_spec<8, 512, false, false>(a, s, st);
  if (R == 4) return gen ? launch_spec<4, 512, false, true>(a, s, st) : launch_spec<4, 512, false, false>(a, s, st);
  return cudaErrorInvalidValue;
}
cudaError_t tm_occ(int R, const LaunchShape& s, int* n) {
  switch (R) {
    case 4: return occ_r<4, 512>(s, n);
    case 8: return occ_r<8, 512>(s, n);
    default: return cudaErrorInvalidValue;
  }
}
#endif

#if !defined(TM_PART) || TM_PART == 0
SmemLayout sscga_tm_layout(int M, int Lcta, int N, int CS, int TL, int TH, int pcap, int gd) {
  (void)M;
  return tm_layout_impl(Lcta, N, CS, TL, TH, pcap, gd);
}

// Both instantiations on the stream: the lean frames, then the others.
cudaError_t launch_sscga_tm(SolveArgs a, const LaunchShape& s, cudaStream_t st) {
  if (a.B == 0) return cudaSuccess;
  if (s.rows != 4 && s.rows != 8 && s.rows != 16) return cudaErrorInvalidValue;
  for (int gen = a.split ? 0 : 1; gen < 2; ++gen) {
    const cudaError_t e = s.rows == 16 ? tm_launch16(gen != 0, a, s, st) : tm_launch_small(s.rows, gen != 0, a, s, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t sscga_tm_occupancy(const LaunchShape& s, int* n) {
  return s.rows == 16 ? tm_occ16(s, n) : tm_occ(s.rows, s, n);
}
#endif

}  // namespace ddb
