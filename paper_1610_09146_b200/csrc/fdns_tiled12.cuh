// fdns_tiled12.cuh -- the 12-warp stage kernel (SN, RA; SS/RS on large planes).
//
// Same z-marching, TMA-fed scheme as fdns_tiled.cuh (read that first), laid
// out so that 12 warps fit on an SM instead of 8.  The 8-warp kernel is
// latency bound: its FP64 pipe is ~44% busy, and ncu's dominant stall is the
// fixed-latency dependency wait of the bitwise-fixed expression chains, which
// only more resident warps can hide.  What limits the warps is shared memory
// (a 6-slot ring of ten 36 x 12 field planes is 203 KB), so this kernel:
//
//  * uses a 32 x 12 column tile (384 threads, <= 168 registers each): the
//    staged box 36 x 16 carries 1.5x the tile's points instead of 1.69x;
//  * stores nine fields per plane slot, not ten: p is not staged but formed
//    at each tap as gm1 * (rho*e), the expression the arrival conversion
//    stored before (physics.py:195-202), so the bits are unchanged;
//  * runs a 5-slot ring (the stencil window itself) with no spare prefetch
//    slot: each step reads its column's nine values on the oldest plane
//    (axis-0 offset -2) into registers before the step barrier, after which
//    that slot is free and the producer streams the next plane into it, a
//    whole step ahead of its use;
//  * keeps the centre-plane buffers compact: D(u1,x1) over the tile's rows
//    only, D(u2,x2) over its columns only (pitch TK).
//
// 5 x 41.5 KB ring + 2 x 11.9 KB buffers = 231.7 KB of the 227 KB-per-CTA
// limit (232448 B).
//
// SS / RS (round 2) run on it from 384^2-point planes, where the round-robin
// split applies (see fdns_b200.cu:use_t12_ss): their buffer set is the three
// TMA boxes of the centre plane's stored diagonal gradients; the axis-0
// queues and the six off-diagonal gradients are per-thread loads, as in the
// 8-warp kernel.  Whole RK3 steps at 512^3 (interleaved A/B): SS +1.2-4.1%,
// RS -2..+1.7%; at 256^3 SS equal, RS -3%; without the round-robin split
// 6-11% slower (more DRAM traffic; profiles/r02_ss_t12_ab.txt).  There is no shared memory left
// to stage the off-diagonal gradients, so its load/store unit is busier
// than SN's (mio + lg throttle stalls ~0.8 vs ~0.4 cycles per instruction).
//
// Round-robin split in lockstep (end of round 2; SN from 512 planes, SS/RS
// from 256): 128-plane units dealt round-robin, the CTAs held within two
// step barriers of their tile-grid neighbours (tiled::ls_step) so the halo
// columns and rows neighbouring boxes share hit in L2 (ncu at 512^3: SN
// reads 25.5 -> 15.2 GB, SS 36.5 -> 26.7 GB per stage), and the partial
// last round cut into per-CTA plane ranges; whole RK3 steps SN +2.6%, SS
// +8.7%, RS +4.5% (profiles/r02_lockstep_ab.txt).  RA keeps the contiguous
// split (-1 to -3% with the units).
//
// RA (round 2) runs on the same layout.  It taps the oldest plane off its
// own column as well (the mixed terms re-expand D(u0,x0) at in-plane shifts
// and D(u1,x1), D(u2,x2) on plane i-2), so its buffer set holds, instead of
// SN's centre-plane derivatives, plane i-2's u0 box, u1 rows and u2 columns,
// copied before the step barrier (SAccRA12).  167 registers, no spills;
// whole RK3 steps +6.6% / +3.9% / +5.5-6.3% over the 8-warp RA kernel at
// 128^3 / 256^3 / 512^3.  (A 32 x 10 tile on a 6-slot ring of nine fields,
// 10 warps, was 7% slower than 8 warps: two of the four schedulers then
// carry three warps and the step barrier waits for them.)
#pragma once

#include "fdns_tiled.cuh"

namespace fdns {
namespace t12 {

using tiled::mbar_expect_tx;
using tiled::mbar_init;
using tiled::mbar_wait;
using tiled::Segments;
using tiled::tma_load_plane;
using tiled::tma_prefetch_l2;

constexpr int NSF = 9;                  // staged fields: rho, rhou0..2, rho*e, u0..2, T
constexpr int SF_T = 8;                 // slot index of T
constexpr int NLOAD = 8;                // TMA-loaded fields (rho..u2)
constexpr int NR = 5;                   // ring depth = the stencil window

// Tile layout: a 32 x TJ column tile, one thread per point.  TJ = 12: one
// 384-thread CTA per SM (the default SN kernel on grids whose rows fit).
// (TJ = 4 -- 128-thread CTAs, two per SM, their step barriers independent
// -- measured 2-3% slower than the 8-warp kernel at 64^3-256^3: the halo
// overhead of a 36 x 8 box outweighs the desynchronised warps.)
template <int TJ_>
struct Lay {
  static constexpr int TK = 32, TJ = TJ_, NT = TK * TJ;
  static constexpr int PK = TK + 4, PJ = TJ + 4;
  static constexpr int PLANE = PK * PJ;
  static constexpr int SLOT = NSF * PLANE;
  static constexpr uint32_t LOAD_BYTES = NLOAD * PLANE * 8;
  static constexpr int BU1_N = TJ * PK;   // D(u1,x1): tile rows, all box columns
  static constexpr int BU2_N = PJ * TK;   // D(u2,x2): all box rows, tile columns (pitch TK)
  static constexpr int BUFSET = PLANE + BU1_N + BU2_N;
  static constexpr int SMEM_BYTES = NR * SLOT * 8 + 2 * BUFSET * 8 + 64;
  static constexpr int MINB = TJ_ <= 4 ? 2 : 1;   // CTAs per SM
  static_assert(MINB * (SMEM_BYTES + 1024) <= 233472, "tile exceeds shared memory");
};
// the default (12-warp) layout's names, used by the host launcher
using L12 = Lay<12>;
constexpr int TK = L12::TK, TJ = L12::TJ, NT = L12::NT, PK = L12::PK, PJ = L12::PJ;
constexpr int SMEM_BYTES = L12::SMEM_BYTES;

__device__ __forceinline__ constexpr int sfield(int f) { return f == TF ? SF_T : f; }

// Accessor of the staged window.  Taps at axis-0 offset -2 come from the
// registers m2 (read before the step barrier: that slot is being refilled by
// then); the SN provider only taps the oldest plane at its own column.
#ifndef FDNS_SHFL_X
#define FDNS_SHFL_X 0
#endif
template <class L>
struct SAcc12 {
  static constexpr bool kInternalEnergy = true;
  static constexpr bool kMaskTaps = true;
  const double* p[5];   // p[0] unused (the -2 plane is in m2)
  double m2[NSF];
  double gm1;
  __device__ __forceinline__ double raw(int f, int di, int dj, int dk) const {
    const int sf = sfield(f);
    if (di == -2) return m2[sf];
#if FDNS_SHFL_X
    // A/B of the north star's "warp shuffles for the x-direction taps": a
    // warp is one 32-point row of the tile (axis 2), so a centre-plane tap
    // at dk comes from lane + dk's centre value (two 32-bit shuffles), the
    // edge lanes reading the box halo from shared memory.  Same bits.
    if (di == 0 && dj == 0 && dk != 0) {
      const double c = p[2][sf * L::PLANE];
      const int src = (int)(threadIdx.x & 31) + dk;
      double s = __shfl_sync(0xffffffffu, c, src & 31);
      if (src < 0 || src > 31) s = p[2][sf * L::PLANE + dk];
      return s;
    }
#endif
    return p[di + 2][sf * L::PLANE + dj * L::PK + dk];
  }
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    if (f == PF) return gm1 * raw(RHOE_F, di, dj, dk);   // p = gm1 * rho*e
    return raw(f, di, dj, dk);
  }
};

// RA accessor: RA also taps the oldest plane off its own column -- the mixed
// terms DD(u_J, x_O, x_J) with O or J = 0 re-expand D(u0,x0) at in-plane
// shifts and D(u1,x1), D(u2,x2) on plane i-2 -- so before the step barrier
// the kernel copies that plane's u0 box, u1 rows and u2 columns into the
// (double-buffered) buffer set, and the column's own nine values into m2.
template <class L>
struct SAccRA12 {
  static constexpr bool kInternalEnergy = true;
  static constexpr bool kMaskTaps = true;
  const double* p[5];   // p[0] unused
  const double* o0;     // u0 on plane i-2, box pitch PK, at this column
  const double* o1;     // u1 on plane i-2, pitch TK (box rows x tile columns)
  const double* o2;     // u2 on plane i-2, pitch PK (tile rows x box columns)
  double m2[NSF];
  double gm1;
  __device__ __forceinline__ double raw(int f, int di, int dj, int dk) const {
    const int sf = sfield(f);
    if (di == -2) {
      if (dj == 0 && dk == 0) return m2[sf];
      if (f == U0) return o0[dj * L::PK + dk];
      if (f == U1) return o1[dj * L::TK];
      return o2[dk];   // U2 (the only other off-column field tapped there)
    }
    return p[di + 2][sf * L::PLANE + dj * L::PK + dk];
  }
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    if (f == PF) return gm1 * raw(RHOE_F, di, dj, dk);   // p = gm1 * rho*e
    return raw(f, di, dj, dk);
  }
};

// Accessor over all five window planes in shared memory (the centre-plane
// buffers, before the step barrier).
template <class L>
struct SAccW {
  static constexpr bool kInternalEnergy = true;
  static constexpr bool kMaskTaps = true;
  const double* p[5];
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    return p[di + 2][sfield(f) * L::PLANE + dj * L::PK + dk];
  }
};

// Arrival conversion (fdns_tiled.cuh:stage_arrival without the p field).
template <class L>
__device__ __forceinline__ void stage_arrival(const Coef& k, double* slot, int tid) {
  constexpr int PLANE = L::PLANE;
#pragma unroll 1
  for (int x = tid; x < PLANE; x += L::NT) {
    const double rho = slot[RHO * PLANE + x];
    const double e = slot[RHOE_F * PLANE + x] -
                     0.5 * (slot[RU0 * PLANE + x] * slot[U0 * PLANE + x] +
                            slot[RU1 * PLANE + x] * slot[U1 * PLANE + x] +
                            slot[RU2 * PLANE + x] * slot[U2 * PLANE + x]);
    const double p = k.gm1 * e;
    slot[RHOE_F * PLANE + x] = e;
    slot[SF_T * PLANE + x] = k.gM2 * p / rho;
  }
}

// Staggered arrival conversion (round 2, RA: kStagger).  A box has 576
// points for 384 threads, so converting a whole plane per step gave half the
// warps two points and the other half one, and every step barrier waited
// for the first half.  But rho*e and T of a plane are only read at the
// thread's own column until the plane becomes the centre plane (the
// axis-0 taps), and in-plane around it then; so each step a thread converts
// its own point of the newest plane in full, and the 192 halo points are
// converted in two halves on the two following steps -- rho*e by threads
// 0..191 one step after arrival, T (from that rho*e) by threads 192..383 on
// the step the plane becomes the centre, before its barrier.  Same
// expressions on the same values, so the same bits; every thread now does
// one conversion plus half a halo conversion per step.
// Measured (profiles/r02_stagger_ab.txt): RA +0.7%; SN 1.3-2.8% slower (one
// more live register tips it into spills; its buffer computation already
// evens the warps out), SS unchanged -- so RA only.
template <class L>
__device__ __forceinline__ int halo_pos(int h) {   // h in [0, 4 * (PK + TJ))
  constexpr int PK = L::PK, PJ = L::PJ;
  if (h < 2 * PK) return h;                          // rows 0, 1
  h -= 2 * PK;
  if (h < 2 * PK) return (PJ - 2) * PK + h;          // rows PJ-2, PJ-1
  h -= 2 * PK;
  const int row = 2 + h / 4, c = h % 4;              // columns 0, 1, PK-2, PK-1
  return row * PK + (c < 2 ? c : PK - 4 + c);
}
template <class L>
__device__ __forceinline__ void conv_e(const Coef& k, double* slot, int x) {
  constexpr int PLANE = L::PLANE;
  (void)k;
  slot[RHOE_F * PLANE + x] = slot[RHOE_F * PLANE + x] -
                             0.5 * (slot[RU0 * PLANE + x] * slot[U0 * PLANE + x] +
                                    slot[RU1 * PLANE + x] * slot[U1 * PLANE + x] +
                                    slot[RU2 * PLANE + x] * slot[U2 * PLANE + x]);
}
template <class L>
__device__ __forceinline__ void conv_T(const Coef& k, double* slot, int x) {
  constexpr int PLANE = L::PLANE;
  const double p = k.gm1 * slot[RHOE_F * PLANE + x];
  slot[SF_T * PLANE + x] = k.gM2 * p / slot[RHO * PLANE + x];
}
template <class L>
__device__ __forceinline__ void conv_full(const Coef& k, double* slot, int x) {
  conv_e<L>(k, slot, x);
  conv_T<L>(k, slot, x);
}

// SS / RS: the three TMA boxes of the centre plane's stored diagonal
// gradients, laid out like SN's buffer set: D(u0,x0) over the whole box,
// D(u1,x1) over the tile rows (pitch PK), D(u2,x2) over the tile columns
// (pitch TK).  tg[0..2] are their tensor maps, tg[3] the L2-prefetch box of
// all nine stored gradients of a plane's tile columns.
struct GradMaps {
  CUtensorMap tg[4];
};

template <int V, int MODE, int TJ_ = 12, bool RR = false>
__global__ void __launch_bounds__(Lay<TJ_>::NT, Lay<TJ_>::MINB)
    k_stage_t12(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tsv,
                const __grid_constant__ GradMaps gm, const double* __restrict__ work,
                const double* saved, double* out, Coef k, Geom g, double coef, int ntk,
                int64_t total_steps, int wrap_mask, int i_lo, int nplanes, int split,
                int pf_saved, const int64_t* __restrict__ cuts) {
  static_assert(V == FDNS_SN || V == FDNS_RA || V == FDNS_SS || V == FDNS_RS,
                "12-warp kernel variant");
  constexpr bool kGB = (V == FDNS_SS || V == FDNS_RS);
  constexpr bool kStagger = (V == FDNS_RA && TJ_ == 12);   // staggered arrival conversion
  using L = Lay<TJ_>;
  constexpr int TK = L::TK, TJ = L::TJ, NT = L::NT, PK = L::PK, PLANE = L::PLANE;
  constexpr int SLOT = L::SLOT, BU1_N = L::BU1_N, BU2_N = L::BU2_N, BUFSET = L::BUFSET;
  constexpr uint32_t LOAD_BYTES = L::LOAD_BYTES;
  using SAcc12 = t12::SAcc12<L>;
  using SAccW = t12::SAccW<L>;
  extern __shared__ __align__(128) double sm[];
  double* bufs0 = sm + NR * SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NR * SLOT + 2 * BUFSET);
  uint64_t* gbars = bars + NR;   // SS/RS: the gradient boxes of the two buffer sets
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  Segments S = Segments::partition(blockIdx.x, gridDim.x, total_steps, nplanes, split, cuts);
  if constexpr (RR) S.tiles = (int64_t)ntk * ((g.n1 + TJ - 1) / TJ);
  volatile int64_t* s_tail = nullptr;
  if constexpr (RR) {
    s_tail = tiled::tail_slot<64 + V * 2 + MODE>();
    if (threadIdx.x == 0) { s_tail[0] = S.main_end; s_tail[1] = S.tbeg; s_tail[2] = S.tend; }
  }
  // segment walk: contiguous tile-major ranges, or (RR) round-robin units
  auto seg_next = [&](int64_t x) -> int64_t {
    if constexpr (RR) return S.next_rr(x, s_tail[0], s_tail[1], s_tail[2]);
    else return S.seg_end(x);
  };
  auto seg_end = [&](int64_t x) -> int64_t {
    if constexpr (RR) return S.seg_end_rr(x, s_tail[0], s_tail[2]);
    else return S.seg_end(x);
  };
  auto tile_at = [&](int64_t x) -> int64_t {
    if constexpr (RR) return S.tile_of(x);
    else return x / nplanes;
  };
  auto plane_at = [&](int64_t x) -> int {
    if constexpr (RR) return S.plane_of(x);
    else return (int)(x % nplanes);
  };
  // lockstep (RR only): K = pf_saved bits 8..15, 0 = off
  constexpr int LS_TID = tiled::LS_TID;   // the thread that publishes and waits
  int ls_k = 0;
  if constexpr (RR) ls_k = tiled::ls_slack(pf_saved);
  if (S.beg >= S.end) {
    if (RR && ls_k && tid == LS_TID) tiled::ls_publish(tiled::PROG_DONE);
    return;
  }
  tiled::trace(0);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    if constexpr (kGB) { mbar_init(&gbars[0], 1); mbar_init(&gbars[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tiled::trace(1);
  // (after the wait: the previous stage's CTAs no longer publish)
  if (RR && ls_k && tid == LS_TID) tiled::ls_publish(0);

  // SS/RS: the stored-gradient boxes of the centre plane of step gs
  auto issue_gb_tile = [&](int gs_, int k0, int j0, int plane) {
    double* dst = bufs0 + (gs_ & 1) * BUFSET;
    uint64_t* bar = &gbars[gs_ & 1];
    mbar_expect_tx(bar, BUFSET * 8);
    tma_load_plane(dst, &gm.tg[0], bar, k0 + g.h - 2, j0 + g.h - 2, plane + g.h);
    tma_load_plane(dst + PLANE, &gm.tg[1], bar, k0 + g.h - 2, j0 + g.h, plane + g.h);
    tma_load_plane(dst + PLANE + BU1_N, &gm.tg[2], bar, k0 + g.h, j0 + g.h - 2, plane + g.h);
  };
  auto issue_gb = [&](int gs_, int64_t x) {
    const int64_t tile = tile_at(x);
    issue_gb_tile(gs_, (int)(tile % ntk) * TK, (int)(tile / ntk) * TJ, i_lo + plane_at(x));
  };
  if constexpr (kGB)
    if (tid == 0) issue_gb(0, S.beg);
  int gs = 0;   // steps of this CTA: buffer-set parity

  // producer cursor (thread 0), as in k_stage_tiled
  int64_t p_seg = S.beg;
  int p_r = 0, issued = 0;
  int p_len = 0, p_c0 = 0, p_c1 = 0, p_plane = 0, p_slot = 0;
  auto enter_segment = [&]() {
    const int64_t tile = tile_at(p_seg);
    p_len = (int)(seg_end(p_seg) - p_seg) + 4;
    p_c0 = (int)(tile % ntk) * TK + g.h - 2;
    p_c1 = (int)(tile / ntk) * TJ + g.h - 2;
    p_plane = i_lo + plane_at(p_seg) - 2 + g.h;
  };
  if (tid == 0) enter_segment();
  auto issue_next = [&]() {
    mbar_expect_tx(&bars[p_slot], LOAD_BYTES);
#if FDNS_TMA_EL
    tiled::tma_load_plane_el(sm + p_slot * SLOT, &tin, &bars[p_slot], p_c0, p_c1, p_plane + p_r);
#else
    tma_load_plane(sm + p_slot * SLOT, &tin, &bars[p_slot], p_c0, p_c1, p_plane + p_r);
#endif
    if (MODE == 1 && (pf_saved & tiled::PF_SAVED) && p_r >= 2 && p_r < p_len - 2)
      tma_prefetch_l2(&tsv, p_c0 + 2, p_c1 + 2, p_plane + p_r);
    // SS/RS: the nine stored gradients of this plane's tile columns into L2
    if constexpr (kGB)
      if (pf_saved & tiled::PF_GRAD) tma_prefetch_l2(&gm.tg[3], p_c0 + 2, p_c1 + 2, p_plane + p_r);
    ++issued;
    p_slot = p_slot + 1 == NR ? 0 : p_slot + 1;
    if (++p_r == p_len) {
      p_r = 0;
      p_seg = seg_next(p_seg);
      if (p_seg < S.end) enter_segment();
    }
  };
  int total_pos = 0;
  for (int64_t x = S.beg; x < S.end; x = seg_next(x)) total_pos += (int)(seg_end(x) - x) + 4;
  if (tid == 0)
    while (issued < total_pos && issued < NR) issue_next();

  int w = 0, wsl = 0;
  auto slot_of = [&](int d) {
    const int x = wsl + d;
    return x >= NR ? x - NR : x;
  };
  for (int64_t x = S.beg; x < S.end; x = seg_next(x)) {
    const int64_t se = seg_end(x);
    const int64_t tile = tile_at(x);
    const int k0 = (int)(tile % ntk) * TK, j0 = (int)(tile / ntk) * TJ;
    const int jj = j0 + tj, kk = k0 + tk;
    const bool active = jj < g.n1 && kk < g.n2;
    const int toff = (tj + 2) * PK + (tk + 2);
    const int hx = halo_pos<L>(tid < NT / 2 ? tid : tid - NT / 2);   // staggered halo item
    const int nsteps = (int)(se - x);
    const int i_seg = i_lo + plane_at(x);
    if constexpr (RR) {
      // the last round's plane ranges differ per CTA: free running from here
      if (ls_k && x >= s_tail[0]) {
        if (tid == LS_TID) tiled::ls_publish(tiled::PROG_DONE);
        ls_k = 0;
      }
    }
    double q1[5], q2[5];
    for (int t = 0; t < nsteps; ++t, ++w, ++gs, wsl = (wsl + 1 == NR ? 0 : wsl + 1)) {
      if (t == 0 && w > 0) {
        // segment change: the new window's five planes; the ring slots of
        // the previous segment are free once every thread is past it
        __syncthreads();
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          while (issued < total_pos && issued < w + NR) issue_next();
        }
      }
      const int i = i_seg + t;
      const int64_t cl = (int64_t)(i + g.h) * g.s0 + (int64_t)(min(jj, g.n1 - 1) + g.h) * g.s1 +
                         (min(kk, g.n2 - 1) + g.h);
      double sv[5];
      if constexpr (MODE == 1) {
#pragma unroll
        for (int f = 0; f < 5; ++f) sv[f] = tiled::ld_stream(saved + f * g.fs + cl);
      }
      // SS/RS: the stored gradients this point FETCHes (plan.py:176-179):
      // the axis-0 queues of D(u1,x1), D(u2,x2) at this column and the six
      // off-diagonal D(u_q,x_a) at the point, issued early so their latency
      // runs under the arrival conversion and the barrier
      double gv[9];
      if constexpr (kGB) {
        const double* w11 = work + 4 * g.fs + cl;
        const double* w22 = work + 8 * g.fs + cl;
        if (t == 0) {
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            q1[d] = __ldg(w11 + (d - 2) * g.s0);
            q2[d] = __ldg(w22 + (d - 2) * g.s0);
          }
        } else {
#pragma unroll
          for (int d = 0; d < 4; ++d) { q1[d] = q1[d + 1]; q2[d] = q2[d + 1]; }
          q1[4] = __ldg(w11 + 2 * g.s0);
          q2[4] = __ldg(w22 + 2 * g.s0);
        }
      }
      if constexpr (kGB) {
        gv[0 * 3 + 1] = tiled::ldg_stream(work + 1 * g.fs + cl);
        gv[0 * 3 + 2] = tiled::ldg_stream(work + 2 * g.fs + cl);
        gv[1 * 3 + 0] = tiled::ldg_stream(work + 3 * g.fs + cl);
        gv[1 * 3 + 2] = tiled::ldg_stream(work + 5 * g.fs + cl);
        gv[2 * 3 + 0] = tiled::ldg_stream(work + 6 * g.fs + cl);
        gv[2 * 3 + 1] = tiled::ldg_stream(work + 7 * g.fs + cl);
      }
      int ls_v[4] = {tiled::PROG_DONE, tiled::PROG_DONE, tiled::PROG_DONE, tiled::PROG_DONE};
      if constexpr (RR) {
        if (ls_k && tid == LS_TID) {   // issued early: the latency runs under the conversion
#pragma unroll
          for (int j = 0; j < 4; ++j) ls_v[j] = tiled::ls_neighbour(j, ntk);
        }
      }
      if constexpr (kStagger) {
        static_assert(4 * (PK + TJ) == NT / 2, "halo points = half the threads");
        if (t == 0) {
          // a new window: own points of all five planes, the centre plane's
          // halo in full (threads 0..191), the next plane's halo rho*e
          // (threads 192..383); its T follows on the next step
          for (int d = 0; d < 5; ++d) {
            mbar_wait(&bars[slot_of(d)], ((w + d) / NR) & 1);
            conv_full<L>(k, sm + slot_of(d) * SLOT, toff);
          }
          if (tid < NT / 2) conv_full<L>(k, sm + slot_of(2) * SLOT, hx);
          else conv_e<L>(k, sm + slot_of(3) * SLOT, hx);
          __syncthreads();   // halo values written by other threads
        } else {
          mbar_wait(&bars[slot_of(4)], ((w + 4) / NR) & 1);
          conv_full<L>(k, sm + slot_of(4) * SLOT, toff);
          if (tid < NT / 2) conv_e<L>(k, sm + slot_of(3) * SLOT, hx);
          else conv_T<L>(k, sm + slot_of(2) * SLOT, hx);
        }
      } else if (t == 0) {
        for (int d = 0; d < 5; ++d) {
          mbar_wait(&bars[slot_of(d)], ((w + d) / NR) & 1);
          stage_arrival<L>(k, sm + slot_of(d) * SLOT, tid);
        }
        // the oldest plane's rho*e and T, read into m2 below (before the
        // step barrier), were just converted by other threads: make those
        // stores visible first (later steps read m2 from a plane converted
        // four step barriers earlier)
        __syncthreads();
      } else {
        mbar_wait(&bars[slot_of(4)], ((w + 4) / NR) & 1);
        stage_arrival<L>(k, sm + slot_of(4) * SLOT, tid);
      }
      double* bufs = bufs0 + (gs & 1) * BUFSET;
      double* bu1 = bufs + PLANE - 2 * PK;   // row 2 of the box at offset PLANE
      double* bu2 = bufs + PLANE + BU1_N;    // (row, column - 2), pitch TK
      if constexpr (V == FDNS_RA) {
        // plane i-2's u0 box, u1 (box rows x tile columns, pitch TK) and u2
        // (tile rows x box columns, pitch PK), before its slot is reused
        const double* old = sm + slot_of(0) * SLOT;
        double* r1 = bufs + PLANE;             // u1, PJ x TK
        double* r2 = bufs + PLANE + BU2_N;     // u2, TJ x PK
        static_assert(BU2_N == L::PJ * TK && BU1_N == TJ * PK, "RA buffer shapes");
        // each buffer's items past the first NT go to the highest thread
        // ids: the arrival conversion gave its extra points to the lowest
        // ones, so the pre-barrier work evens out across the warps
        auto cp0 = [&](int x0) { bufs[x0] = old[U0 * PLANE + x0]; };
        auto cp1 = [&](int y) { r1[y] = old[U1 * PLANE + (y / TK) * PK + 2 + y % TK]; };
        auto cp2 = [&](int y) { r2[y] = old[U2 * PLANE + 2 * PK + y]; };
        static_assert(PLANE <= 2 * NT && BU2_N <= 2 * NT && BU1_N <= 2 * NT, "two items at most");
        cp0(tid);
        cp1(tid);
        cp2(tid);
        if constexpr (kStagger) {
          // the conversion work is even across threads: deal the 368 extra
          // items one per thread (u0 to 0..191, u1 to 192..319, u2 after)
          if (tid < PLANE - NT) cp0(NT + tid);
          else if (tid - (PLANE - NT) < BU2_N - NT) cp1(NT + tid - (PLANE - NT));
          else if (tid - (PLANE - NT) - (BU2_N - NT) < BU1_N - NT)
            cp2(NT + tid - (PLANE - NT) - (BU2_N - NT));
        } else {
          // extra items to the highest thread ids: the whole-plane arrival
          // conversion gave its extra points to the lowest ones
          auto extra = [&](int n, auto&& item) {
            const int x = tid + n - 2 * NT;   // items NT..n-1 -> tids 2NT-n..NT-1
            if (x >= 0 && n > NT) item(x + NT);
          };
          extra(PLANE, cp0);
          extra(BU2_N, cp1);
          extra(BU1_N, cp2);
        }
      } else if constexpr (kGB) {
        // stored gradient boxes: TMA (issue_gb_tile)
      } else {
        const double* base[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) base[d] = sm + slot_of(d) * SLOT;
        if constexpr (TJ == 12) {
        // items past the first NT of each buffer: D(u1,x1)'s and D(u2,x2)'s
        // to threads 192..367; D(u0,x0)'s to threads 0..191 (staggered
        // conversion) or also to 192..383 (whole-plane conversion, whose
        // extra points sit on 0..191), so no warp carries much more than
        // the average
        static_assert(PLANE - NT == 192 && BU1_N - NT == 48 && BU2_N - NT == 128,
                      "item split below assumes the 32 x 12 tile");
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          // D(u0,x0), whole box; with the staggered conversion (even work
          // per thread) its extra items go to threads 0..191, which take
          // none of the other buffers' extras
          const int x0 = m == 0 ? tid : (kStagger ? tid + 384 : tid + 192);
          if (m == 0 || (kStagger ? tid < 192 : (tid >= 192 && x0 < PLANE))) {
            SAccW b;
#pragma unroll
            for (int d = 0; d < 5; ++d) b.p[d] = base[d] + x0;
            bufs[x0] = d1<0, E_FIELD, U0, 0>(k, b);
          }
          const int y1 = m == 0 ? tid : tid + 192;   // D(u1,x1), rows 2..TJ+1
          if (m == 0 || (tid >= 192 && y1 < BU1_N)) {
            const int pos = 2 * PK + y1;
            SAccW b;
            b.p[2] = base[2] + pos;
            bu1[pos] = d1<1, E_FIELD, U1, 0>(k, b);
          }
          const int y2 = m == 0 ? tid : tid + 144;   // D(u2,x2), cols 2..TK+1
          if (m == 0 || (tid >= 240 && y2 < BU2_N)) {
            const int row = y2 / TK, col = y2 % TK;
            SAccW b;
            b.p[2] = base[2] + row * PK + 2 + col;
            bu2[y2] = d1<2, E_FIELD, U2, 0>(k, b);
          }
        }
        } else {
#pragma unroll 1
          for (int x0 = tid; x0 < PLANE; x0 += NT) {   // D(u0,x0), whole box
            SAccW b;
#pragma unroll
            for (int d = 0; d < 5; ++d) b.p[d] = base[d] + x0;
            bufs[x0] = d1<0, E_FIELD, U0, 0>(k, b);
          }
#pragma unroll 1
          for (int y1 = tid; y1 < BU1_N; y1 += NT) {   // D(u1,x1), rows 2..TJ+1
            const int pos = 2 * PK + y1;
            SAccW b;
            b.p[2] = base[2] + pos;
            bu1[pos] = d1<1, E_FIELD, U1, 0>(k, b);
          }
#pragma unroll 1
          for (int y2 = tid; y2 < BU2_N; y2 += NT) {   // D(u2,x2), cols 2..TK+1
            const int row = y2 / TK, col = y2 % TK;
            SAccW b;
            b.p[2] = base[2] + row * PK + 2 + col;
            bu2[y2] = d1<2, E_FIELD, U2, 0>(k, b);
          }
        }
      }
      // axis-0 queues of D(u1,x1), D(u2,x2) at this column (before the
      // barrier: at a segment start they read the oldest slot too)
      if constexpr (V != FDNS_SN) {
      } else if (t == 0) {
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          SAccW b;
          b.p[2] = sm + slot_of(d) * SLOT + toff;
          q1[d] = d1<1, E_FIELD, U1, 0>(k, b);
          q2[d] = d1<2, E_FIELD, U2, 0>(k, b);
        }
      } else {
#pragma unroll
        for (int d = 0; d < 4; ++d) { q1[d] = q1[d + 1]; q2[d] = q2[d + 1]; }
        SAccW b;
        b.p[2] = sm + slot_of(4) * SLOT + toff;
        q1[4] = d1<1, E_FIELD, U1, 0>(k, b);
        q2[4] = d1<2, E_FIELD, U2, 0>(k, b);
      }

      // this column's values on the oldest plane, before its slot is reused
      using Acc = std::conditional_t<V == FDNS_RA, SAccRA12<L>, SAcc12>;
      Acc a;
      a.gm1 = k.gm1;
      {
        const double* old = sm + slot_of(0) * SLOT + toff;
#pragma unroll
        for (int f = 0; f < NSF; ++f) a.m2[f] = old[f * PLANE];
      }
      if constexpr (V == FDNS_RA) {
        a.o0 = bufs + toff;
        a.o1 = bufs + PLANE + (tj + 2) * TK + tk;
        a.o2 = bufs + PLANE + BU2_N + tj * PK + tk + 2;
      }
      __syncthreads();
      if (w == 0) tiled::trace(2);
      if constexpr (RR) {
        if (ls_k && tid == LS_TID) tiled::ls_step(ls_k, w, ls_v, ntk);
      }
      if (tid == 0) {
        if (issued < total_pos && issued < w + NR + 1) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_next();   // the next plane, into the oldest slot
        }
        if constexpr (kGB) {   // the next step's gradient boxes, other buffer set
          if (t + 1 < nsteps) issue_gb_tile(gs + 1, k0, j0, i + 1);
          else if (seg_next(x) < S.end) issue_gb(gs + 1, seg_next(x));
        }
      }
#pragma unroll
      for (int d = 0; d < 5; ++d) a.p[d] = sm + slot_of(d) * SLOT + toff;
      a.p[0] = nullptr;

      double r[NFIELDS];
#pragma unroll
      for (int f = 0; f < NFIELDS; ++f) r[f] = a.v(f, 0, 0, 0);   // r[RHOE_F] = rho*e
      double R[5];
      if constexpr (V == FDNS_RA) {
        InlineProvider<Acc> P(k, a);
        residual_point<true>(k, P, r, R);
      } else if constexpr (kGB) {
        mbar_wait(&gbars[gs & 1], (gs >> 1) & 1);
        const tiled::TiledSSProviderT<V == FDNS_RS, Acc, TK> P{
            k, a, q1, q2, bufs + toff, bu1 + toff, bu2 + (tj + 2) * TK + tk, gv};
        residual_point<true>(k, P, r, R);
      } else {
        const tiled::TiledLazyProviderT<SAcc12, TK> P{
            k, a, q1, q2, bufs + toff, bu1 + toff, bu2 + (tj + 2) * TK + tk};
        residual_point<true, true>(k, P, r, R);
      }
      if (active) {
        if constexpr (MODE == 0) {
          tiled::emit<5>(out, g, i, jj, kk, R, 0);
        } else {
          double q[NFIELDS];
          tiled::stage_update(sv, R, coef, q);
          tiled::emit<tiled::NOUT_STAGE>(out, g, i, jj, kk, q, wrap_mask);
        }
      }
    }
    w += 4;
    wsl = w % NR;
  }
  if (RR && tid == LS_TID && tiled::ls_slack(pf_saved)) tiled::ls_publish(tiled::PROG_DONE);
  tiled::trace(3);
}

}  // namespace t12
}  // namespace fdns
