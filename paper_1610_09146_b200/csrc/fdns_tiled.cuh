// fdns_tiled.cuh -- the z-marching, TMA-fed stage kernel for the register/
// recompute variants (SN, RA, RS, SS).
//
// Work decomposition: a CTA owns a TK x TJ column tile of the (axis-2,
// axis-1) plane (axis 2 contiguous) and marches along axis 0 over a chunk of
// planes.  All ten fields of every plane of the stencil window live in a
// ring of NR shared-memory plane slots, each slot one 4-D TMA box
// (TK+4) x (TJ+4) x 1 x 10 fields, loaded by cp.async.bulk.tensor one plane
// ahead and completed on an mbarrier.  When a plane lands, rhoE is replaced
// in shared memory by the internal energy rho*e = rhoE - 0.5*(rhou.u)
// (terms.py:39): every stencil tap of the energy terms then reads it instead
// of recomputing it (same per-point expression, so the bits are unchanged).
// Each thread computes one point per plane step; all stencil taps are LDS
// with compile-time offsets from five per-step plane base pointers.
//
// Epilogue: either the residual (MODE 0) or the fused RK update
// q = q_saved + coef*R plus the primitives of q (MODE 1), written to the
// interior AND to the point's periodic ghost images on the axes in
// wrap_mask, so no separate halo-fill pass is needed on one GPU.
#pragma once
#include <cuda.h>

#include "fdns_math.cuh"

namespace fdns {
namespace tiled {

constexpr int TK = 32, TJ = 8, NT = TK * TJ;

// Optional per-CTA timeline (debug): %globaltimer stamps at kernel entry,
// after the prologue, when the first window is ready, and at exit.
constexpr int TRACE_CTAS = 1024, TRACE_PTS = 4;
__device__ unsigned long long g_trace[TRACE_CTAS * TRACE_PTS];
__constant__ int g_trace_on;
// Log mode (g_trace_on == 2): every CTA of every launch also appends its
// four stamps plus (blockIdx | smid << 16) to g_trace_log, so a sequence of
// launches (a whole RK step) can be reconstructed.
constexpr int TRACE_LOG_N = 8192, TRACE_LOG_W = 5;
__device__ unsigned long long g_trace_log[TRACE_LOG_N * TRACE_LOG_W];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(int pt) {
  if (g_trace_on && threadIdx.x == 0 && blockIdx.x < TRACE_CTAS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (pt == 0)   // entry stamp carries the SM id in its top bits
      t = (t & 0x0000FFFFFFFFFFFFull) | ((unsigned long long)smid << 48);
    g_trace[blockIdx.x * TRACE_PTS + pt] = t;
    if (pt == TRACE_PTS - 1 && g_trace_on == 2) {
      const unsigned idx = atomicAdd(&g_trace_n, 1u);
      if (idx < TRACE_LOG_N) {
        unsigned long long* r = g_trace_log + (size_t)idx * TRACE_LOG_W;
        for (int q = 0; q < TRACE_PTS; ++q)
          r[q] = g_trace[blockIdx.x * TRACE_PTS + q] & 0x0000FFFFFFFFFFFFull;
        r[TRACE_PTS] = blockIdx.x | ((unsigned long long)smid << 16);
      }
    }
  }
}
constexpr int PK = TK + 4, PJ = TJ + 4;
constexpr int PLANE = PK * PJ;          // doubles per field per plane slot
constexpr int SLOT = NFIELDS * PLANE;   // doubles per plane slot
constexpr int NLOAD = 8;                // fields TMA-staged per plane (rho..u2);
                                        // p, T are derived on arrival
constexpr uint32_t LOAD_BYTES = NLOAD * PLANE * 8;
constexpr int NOUT_STAGE = 8;           // fields a fused stage writes (cons + u)
constexpr int NR = 6;                   // ring depth: 5-plane window + 1 prefetch
// pf_saved bits of the stage kernels: L2 prefetch of the saved state / of
// SS/RS's nine stored gradients (host kill switches, fdns_set_prefetch)
constexpr int PF_SAVED = 1, PF_GRAD = 2;
constexpr int SMEM_BYTES = NR * SLOT * 8 + 128;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.b32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(saddr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a producer/consumer bug must surface as a kernel error, not
// as a hung GPU.  ~4e9 cycles is seconds; a healthy wait is microseconds.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > 4000000000LL) __trap();
  }
}
#ifndef FDNS_ST_CS
#define FDNS_ST_CS 0
#endif
#ifndef FDNS_LD_CS
#define FDNS_LD_CS 0
#endif
#ifndef FDNS_TMA_EL
#define FDNS_TMA_EL 0
#endif
// streaming (evict-first) load of a value read once per stage
__device__ __forceinline__ double ld_stream(const double* p) {
#if FDNS_LD_CS
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ double ldg_stream(const double* p) {
#if FDNS_LD_CS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}
// state boxes with an L2 evict-last hint (their halo columns are re-read by
// the neighbouring tiles' CTAs)
__device__ __forceinline__ void tma_load_plane_el(double* dst, const CUtensorMap* map,
                                                  uint64_t* bar, int c0, int c1, int c2) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(saddr(bar)),
      "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_plane(double* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(saddr(bar))
      : "memory");
}

// L2 prefetch of a tensor box (no shared memory, no barrier): used for the
// saved-state tile of a plane a few steps before its epilogue reads it.
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(0)
      : "memory");
}

// Shared-memory accessor: p[d] is the plane slot for axis-0 offset d-2,
// already offset to this thread's (j, k) column and field 0.
struct SAcc {
  static constexpr bool kInternalEnergy = true;   // field RHOE_F holds rho*e
  static constexpr bool kMaskTaps = true;         // INLINE occurrences mask taps
  const double* p[5];
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    return p[di + 2][f * PLANE + dj * PK + dk];
  }
  __device__ __forceinline__ SAcc rebased(int z) const {
    SAcc r;
#pragma unroll
    for (int d = 0; d < 5; ++d) r.p[d] = p[d] + z;
    return r;
  }
};

// Write the NOUT output values of interior point (i, j, k) to its location
// and to every periodic ghost image on the axes of wrap_mask (mesh.py:118-139
// semantics: ghost = value at the wrapped coordinates).  When every wrapped
// axis has n >= 2h a coordinate has at most one image, and the (up to 7)
// image stores are explicit predicated stores -- no dynamically indexed
// arrays, so no local memory on the edge warps.  Tiny axes (n < 2h, where a
// point can have an image on both sides) take the general loop.
template <int NOUT>
__device__ __forceinline__ void emit_general(double* out, const Geom& g, int i, int j, int k,
                                          const double* val, int wrap_mask) {
  const int h = g.h;
  int ci[3], cj[3], ck[3], ni = 1, nj = 1, nk = 1;
  ci[0] = i + h; cj[0] = j + h; ck[0] = k + h;
  if (wrap_mask & 1) {
    if (i < h) ci[ni++] = i + h + g.n0;
    if (i >= g.n0 - h) ci[ni++] = i + h - g.n0;
  }
  if (wrap_mask & 2) {
    if (j < h) cj[nj++] = j + h + g.n1;
    if (j >= g.n1 - h) cj[nj++] = j + h - g.n1;
  }
  if (wrap_mask & 4) {
    if (k < h) ck[nk++] = k + h + g.n2;
    if (k >= g.n2 - h) ck[nk++] = k + h - g.n2;
  }
  for (int a = 0; a < ni; ++a)
    for (int b = 0; b < nj; ++b)
      for (int d = 0; d < nk; ++d) {
        const int64_t c = ci[a] * g.s0 + cj[b] * g.s1 + ck[d];
        for (int f = 0; f < NOUT; ++f) out[f * g.fs + c] = val[f];
      }
}

template <int NOUT>
__device__ __forceinline__ void emit_at(double* out, const Geom& g, int64_t c, const double* val) {
#pragma unroll
  for (int f = 0; f < NOUT; ++f) {
#if FDNS_ST_CS
    __stcs(out + f * g.fs + c, val[f]);
#else
    out[f * g.fs + c] = val[f];
#endif
  }
}

template <int NOUT>
__device__ __forceinline__ void emit(double* out, const Geom& g, int i, int j, int k,
                                     const double* val, int wrap_mask) {
  const int h = g.h;
  const int64_t ci = i + h, cj = j + h, ck = k + h;
  emit_at<NOUT>(out, g, ci * g.s0 + cj * g.s1 + ck, val);
  if (wrap_mask == 0) return;
  const bool small = ((wrap_mask & 1) && g.n0 < 2 * h) || ((wrap_mask & 2) && g.n1 < 2 * h) ||
                     ((wrap_mask & 4) && g.n2 < 2 * h);
  if (small) {
    // the general path rewrites the interior value too (same bits)
    double v[NOUT];
#pragma unroll
    for (int f = 0; f < NOUT; ++f) v[f] = val[f];
    emit_general<NOUT>(out, g, i, j, k, v, wrap_mask);
    return;
  }
  // at most one image per axis: its padded coordinate, or -1
  const int64_t gi = !(wrap_mask & 1) ? -1 : (i < h ? ci + g.n0 : (i >= g.n0 - h ? ci - g.n0 : -1));
  const int64_t gj = !(wrap_mask & 2) ? -1 : (j < h ? cj + g.n1 : (j >= g.n1 - h ? cj - g.n1 : -1));
  const int64_t gk = !(wrap_mask & 4) ? -1 : (k < h ? ck + g.n2 : (k >= g.n2 - h ? ck - g.n2 : -1));
  if (gi < 0 && gj < 0 && gk < 0) return;
  if (gi >= 0) emit_at<NOUT>(out, g, gi * g.s0 + cj * g.s1 + ck, val);
  if (gj >= 0) emit_at<NOUT>(out, g, ci * g.s0 + gj * g.s1 + ck, val);
  if (gk >= 0) emit_at<NOUT>(out, g, ci * g.s0 + cj * g.s1 + gk, val);
  if (gi >= 0 && gj >= 0) emit_at<NOUT>(out, g, gi * g.s0 + gj * g.s1 + ck, val);
  if (gi >= 0 && gk >= 0) emit_at<NOUT>(out, g, gi * g.s0 + cj * g.s1 + gk, val);
  if (gj >= 0 && gk >= 0) emit_at<NOUT>(out, g, ci * g.s0 + gj * g.s1 + gk, val);
  if (gi >= 0 && gj >= 0 && gk >= 0) emit_at<NOUT>(out, g, gi * g.s0 + gj * g.s1 + gk, val);
}

// Arrival conversion of one staged plane slot (all PLANE points of the box):
// rhoE -> rho*e = rhoE - 0.5*(rhou.u) (terms.py:39), then the primitive
// expressions of the reference (physics.py:195-202): p = gm1*rho*e (the same
// intermediate the reference forms), T = (gM2*p)/rho.  Bitwise the values
// the primitives pass would have stored.
__device__ __forceinline__ void stage_arrival(const Coef& k, double* slot, int tid, int nthreads) {
#pragma unroll 1
  for (int x = tid; x < PLANE; x += nthreads) {
    const double rho = slot[RHO * PLANE + x];
    const double e = slot[RHOE_F * PLANE + x] -
                     0.5 * (slot[RU0 * PLANE + x] * slot[U0 * PLANE + x] +
                            slot[RU1 * PLANE + x] * slot[U1 * PLANE + x] +
                            slot[RU2 * PLANE + x] * slot[U2 * PLANE + x]);
    const double p = k.gm1 * e;
    slot[RHOE_F * PLANE + x] = e;
    slot[PF * PLANE + x] = p;
    slot[TF * PLANE + x] = k.gM2 * p / rho;
  }
}

// Epilogue of a fused stage: q = q_saved + coef*R and u = rhou/rho
// (physics.py:192-194); p and T are left to the next stage's arrival
// conversion (or a final primitives pass).
__device__ __forceinline__ void stage_update(const double* sv, const double* R, double coef,
                                             double* q) {
#pragma unroll
  for (int f = 0; f < 5; ++f) q[f] = sv[f] + coef * R[f];
  q[U0] = q[RU0] / q[RHO];
  q[U1] = q[RU1] / q[RHO];
  q[U2] = q[RU2] / q[RHO];
}

// Centre-plane inner-derivative buffers (SN): D(u0,x0), D(u1,x1), D(u2,x2)
// over the staged box, so the in-plane mixed terms read 4 values each
// instead of re-expanding 4 inner stencils (same stencil shape at every
// point: bitwise equal to the reference's re-expansion, codegen.py:97-102).
// Double-buffered (step parity), so the buffers of step t are written while
// slower threads may still read those of step t-1: one barrier per step.
constexpr int NBUF = 3;
constexpr int BU1_N = TJ * PK;          // D(u1,x1): interior rows, all columns
constexpr int BU2_N = PJ * TK;          // D(u2,x2): all rows, interior columns
constexpr int BUF_WORK = PLANE + BU1_N + BU2_N;
constexpr int SMEM_BYTES_SN = NR * SLOT * 8 + 2 * NBUF * PLANE * 8 + 128;
static_assert(SMEM_BYTES_SN <= 232448, "SN tile exceeds the 227 KB shared-memory limit");
// SS / RS: the three stored diagonal gradients of the centre plane, one TMA
// box (PK x PJ x 1 x 3 fields of the work bundle), double-buffered by step.
constexpr int NGB = 3;
constexpr uint32_t GB_BYTES = NGB * PLANE * 8;
constexpr int SMEM_BYTES_SS = NR * SLOT * 8 + 2 * NGB * PLANE * 8 + 128;
static_assert(SMEM_BYTES_SS <= 232448, "SS tile exceeds the 227 KB shared-memory limit");
static_assert(PLANE <= 2 * NT && BU1_N <= 2 * NT && BU2_N <= 2 * NT,
              "centre-plane buffer items: at most two per thread");

// SN provider over the staged tile: every distinct derivative once (LOCAL),
// diagonal velocity gradients and the six mixed terms from the axis-0
// register queues (q1, q2: D(u1,x1), D(u2,x2) at this column on planes
// i-2..i+2) and the centre-plane buffers.
struct TiledLocalProvider {
  double v[N_SLOTS];
  template <int A_, int L>
  __device__ __forceinline__ void fill1(const Coef& k, const SAcc& a) {
    if constexpr (!(L >= S_U && L < S_U + 3 && (L - S_U) == A_)) v[slot(A_, L)] = eval_slot<A_, L>(k, a);
    if constexpr (L + 1 < S_PER_AXIS) fill1<A_, L + 1>(k, a);
  }
  __device__ __forceinline__ TiledLocalProvider(const Coef& k, const SAcc& a, const double* q1,
                                                const double* q2, const double* bu0,
                                                const double* bu1, const double* bu2) {
    fill1<0, 0>(k, a);
    fill1<1, 0>(k, a);
    fill1<2, 0>(k, a);
    v[slot(0, S_U + 0)] = bu0[0];
    v[slot(1, S_U + 1)] = q1[2];
    v[slot(2, S_U + 2)] = q2[2];
    // DD(u1,x0,x1), DD(u2,x0,x2): outer axis 0 over the queues
    v[S_DD + dd_index(1, 0)] = k.w1[0] * (q1[3] - q1[1]) + k.w2[0] * (q1[4] - q1[0]);
    v[S_DD + dd_index(2, 0)] = k.w1[0] * (q2[3] - q2[1]) + k.w2[0] * (q2[4] - q2[0]);
    // DD(u0,x1,x0), DD(u0,x2,x0): outer axes 1, 2 over D(u0,x0)
    v[S_DD + dd_index(0, 1)] = k.w1[1] * (bu0[PK] - bu0[-PK]) + k.w2[1] * (bu0[2 * PK] - bu0[-2 * PK]);
    v[S_DD + dd_index(0, 2)] = k.w1[2] * (bu0[1] - bu0[-1]) + k.w2[2] * (bu0[2] - bu0[-2]);
    // DD(u2,x1,x2): outer axis 1 over D(u2,x2); DD(u1,x2,x1): outer axis 2 over D(u1,x1)
    v[S_DD + dd_index(2, 1)] = k.w1[1] * (bu2[PK] - bu2[-PK]) + k.w2[1] * (bu2[2 * PK] - bu2[-2 * PK]);
    v[S_DD + dd_index(1, 2)] = k.w1[2] * (bu1[1] - bu1[-1]) + k.w2[2] * (bu1[2] - bu1[-2]);
  }
  template <int A_, int L, int OCC = 0, bool DES = false> __device__ __forceinline__ double g() const { return v[slot(A_, L)]; }
  template <int J, int O, int OCC = 0, bool DES = false> __device__ __forceinline__ double x() const { return v[S_DD + dd_index(J, O)]; }
};

// Lazily evaluated SN provider over the staged tile: a derivative is
// evaluated where it is used (repeated uses merged by the compiler), the
// diagonal velocity gradients and mixed terms come from the buffers/queues.
template <class A, int B2P>
struct TiledLazyProviderT {
  const Coef& k;
  const A& a;
  const double* q1;   // D(u1,x1) at this column, planes i-2..i+2
  const double* q2;   // D(u2,x2)
  const double* b0;   // D(u0,x0) centre of the box buffer (pitch PK)
  const double* b1;   // D(u1,x1) centre (pitch PK)
  const double* b2;   // D(u2,x2) centre (pitch B2P)
  template <int A_, int L, int OCC = 0, bool DES = false>
  __device__ __forceinline__ double g() const {
    if constexpr (L == S_U + A_) {
      if constexpr (A_ == 0) return b0[0];
      else if constexpr (A_ == 1) return q1[2];
      else return q2[2];
    } else {
      return eval_slot<A_, L>(k, a);
    }
  }
  template <int J, int O, int OCC = 0, bool DES = false>
  __device__ __forceinline__ double x() const {
    if constexpr (O == 0) {
      const double* q = J == 1 ? q1 : q2;
      return k.w1[0] * (q[3] - q[1]) + k.w2[0] * (q[4] - q[0]);
    } else if constexpr (J == 0) {
      constexpr int s = O == 1 ? PK : 1;
      return k.w1[O] * (b0[s] - b0[-s]) + k.w2[O] * (b0[2 * s] - b0[-2 * s]);
    } else if constexpr (J == 2) {
      return k.w1[1] * (b2[B2P] - b2[-B2P]) + k.w2[1] * (b2[2 * B2P] - b2[-2 * B2P]);
    } else {
      return k.w1[2] * (b1[1] - b1[-1]) + k.w2[2] * (b1[2] - b1[-2]);
    }
  }
};
using TiledLazyProvider = TiledLazyProviderT<SAcc, PK>;

// SS / RS provider over the staged tile with FETCHed gradients staged too:
// the centre plane's stored D(u0,x0), D(u1,x1), D(u2,x2) are a TMA box in
// shared memory (gb*), the axis-0 neighbours of D(u1,x1), D(u2,x2) come from
// register queues filled from the stored arrays, and the six off-diagonal
// gradients at the point are loaded at step start.  Every value is read from
// the work arrays (FETCH, plan.py:176-179); mixed terms apply the outer
// stencil to the stored inner values exactly as codegen.py:111-113 does.
template <bool INLINE_REST, class A, int B2P>
struct TiledSSProviderT {
  const Coef& k;
  const A& a;
  const double* q1;   // stored D(u1,x1) at this column, planes i-2..i+2
  const double* q2;   // stored D(u2,x2)
  const double* gb0;  // stored D(u0,x0), centre of the box (pitch PK)
  const double* gb1;  // stored D(u1,x1)
  const double* gb2;  // stored D(u2,x2) (row pitch B2P)
  const double* gv;   // off-diagonal D(u_q,x_a) at the point, [q*3+a]
  template <int A_, int L, int OCC = 0, bool DES = false>
  __device__ __forceinline__ double g() const {
    if constexpr (L >= S_U && L < S_U + 3) {
      constexpr int q = L - S_U;
      if constexpr (q == A_) return A_ == 0 ? gb0[0] : (A_ == 1 ? q1[2] : q2[2]);
      else return gv[q * 3 + A_];
    } else if constexpr (INLINE_REST) {
      return eval_slot<A_, L>(k, occurrence_view<OCC>(a));
    } else {
      return eval_slot<A_, L>(k, a);
    }
  }
  template <int J, int O, int OCC = 0, bool DES = false>
  __device__ __forceinline__ double x() const {
    if constexpr (O == 0) {
      const double* q = J == 1 ? q1 : q2;
      return k.w1[0] * (q[3] - q[1]) + k.w2[0] * (q[4] - q[0]);
    } else if constexpr (J == 0) {
      constexpr int s = O == 1 ? PK : 1;
      return k.w1[O] * (gb0[s] - gb0[-s]) + k.w2[O] * (gb0[2 * s] - gb0[-2 * s]);
    } else if constexpr (J == 2) {
      return k.w1[1] * (gb2[B2P] - gb2[-B2P]) + k.w2[1] * (gb2[2 * B2P] - gb2[-2 * B2P]);
    } else {
      return k.w1[2] * (gb1[1] - gb1[-1]) + k.w2[2] * (gb1[2] - gb1[-2]);
    }
  }
};
template <bool INLINE_REST>
using TiledSSProvider = TiledSSProviderT<INLINE_REST, SAcc, PK>;

// Static, balanced work split of one stage: the (tile, plane) steps in
// tile-major order are cut into gridDim.x equal ranges; a CTA walks its
// range as <= a few segments (one per tile touched).  The TMA producer
// (thread 0) streams the planes of all segments back to back through the
// ring, prefetching across segment boundaries.
// Partition modes of the (tile, plane) steps of one launch over G CTAs.
enum SplitMode : int { SPLIT_CONTIGUOUS = 0, SPLIT_ALIGNED = 1, SPLIT_BALANCED = 2,
                       SPLIT_TABLE = 3, SPLIT_ROUNDS = 4 };
// Ramp of a segment that starts inside a CTA's range (ring refill, five
// planes converted, queues rebuilt), in quarter plane steps (measured
// ~3.3 us vs ~3.0 us per step at 64^3).
constexpr int RAMP_MID_Q = 5;

struct Segments {
  int64_t beg, end;   // [beg, end) in tile-major (tile * nplanes + plane) order
  int n0;             // planes per tile (SPLIT_ROUNDS: per unit) in this launch
  int64_t stride = 0; // SPLIT_ROUNDS: distance between this CTA's units (G * n0)
  int64_t tiles = 1;  // SPLIT_ROUNDS: column tiles per plane chunk
  // SPLIT_ROUNDS: the whole rounds end at main_end; the units left over (fewer
  // than G) are cut into G equal plane ranges [tbeg, tend) per CTA, so the
  // last round keeps every SM busy instead of `left` of them
  int64_t main_end = 0, tbeg = 0, tend = 0;
  __host__ __device__ __forceinline__ int64_t seg_end(int64_t x) const {
    const int64_t tile_end = (x / n0 + 1) * (int64_t)n0;
    return tile_end < end ? tile_end : end;
  }
  // SPLIT_ROUNDS walk.  The kernels pass the three tail values from shared
  // memory (tl = {main_end, tbeg, tend}, read only at segment changes):
  // held in registers through the plane loop they pushed the 12-warp
  // kernels over their 168-register budget (SN 14% slower with 52 B of
  // spills).
  // (32-bit arithmetic: a round-robin launch has < 2^31 steps, checked by
  // the host launcher)
  __host__ __device__ __forceinline__ int64_t seg_end_rr(int64_t x64, int64_t me, int64_t te) const {
    const int x = (int)x64;
    const int tile_end = (x / n0 + 1) * n0;
    const int lim = x >= (int)me ? (int)te : (int)end;
    return tile_end < lim ? tile_end : lim;
  }
  // start of the segment after the one holding x (>= end: none)
  __host__ __device__ __forceinline__ int64_t next_rr(int64_t x64, int64_t me64, int64_t tb64,
                                                      int64_t te64) const {
    const int x = (int)x64, me = (int)me64, tb = (int)tb64, te = (int)te64;
    if (x < me) {
      const int nx = x - x % n0 + (int)stride;
      if (nx < me) return nx;
      return tb < te ? tb64 : end;
    }
    const int e = (int)seg_end_rr(x64, me64, te64);
    return e < te ? (int64_t)e : end;
  }
  // column tile and axis-0 plane (relative to the launch's first plane) of x
  __host__ __device__ __forceinline__ int64_t tile_of(int64_t x) const {
    return stride ? (int64_t)(((int)x / n0) % (int)tiles) : x / n0;
  }
  __host__ __device__ __forceinline__ int plane_of(int64_t x) const {
    return stride ? ((int)x / n0) / (int)tiles * n0 + (int)x % n0 : (int)(x % n0);
  }
  // CTA b of G over `total` = tiles * planes steps.
  //  SPLIT_ALIGNED (needs G >= tiles): each tile gets floor or ceil of
  //    G/tiles CTAs, each CTA one contiguous plane range of one tile (one
  //    pipeline ramp per CTA, ranges quantised per tile);
  //  SPLIT_CONTIGUOUS: equal contiguous ranges in tile-major order (a CTA may
  //    span tiles and pays a ramp per tile);
  //  SPLIT_BALANCED: contiguous ranges of equal cost, a tile counting its
  //    planes plus one mid-range ramp (RAMP_MID_Q), so a CTA whose range
  //    contains a tile start gets correspondingly fewer planes.
  //  SPLIT_TABLE: host-computed cut points `cuts[0..G]` (edge-weighted
  //    costs, see fdns_b200.cu:table_cuts).
  static __host__ __device__ __forceinline__ Segments partition(int64_t b, int64_t G,
                                                                int64_t total, int planes,
                                                                int mode,
                                                                const int64_t* cuts = nullptr) {
    if (mode == SPLIT_TABLE) return Segments{cuts[b], cuts[b + 1], planes};
    if (mode == SPLIT_ROUNDS) {
      // units of `planes` consecutive planes of one tile, chunk-major
      // (unit u = chunk * tiles + tile), dealt round-robin: in every round
      // the G CTAs work on G consecutive units -- neighbouring tiles of the
      // same plane chunk at the same time, so the halo columns one CTA's
      // boxes read were just staged by its neighbours and hit in L2.
      // The caller sets `tiles` (column tiles per plane chunk).
      Segments r{b * (int64_t)planes, total, planes};
      r.stride = G * (int64_t)planes;
      const int64_t units = total / planes, rounds = units / G, left = units - rounds * G;
      r.main_end = rounds * r.stride;
      const int64_t tail = left * planes;   // steps of the last, partial round
      r.tbeg = r.main_end + b * tail / G;
      r.tend = r.main_end + (b + 1) * tail / G;
      if (rounds == 0) r.beg = r.tbeg < r.tend ? r.tbeg : total;
      return r;
    }
    const int64_t tiles = total / planes;
    if (mode == SPLIT_ALIGNED && G >= tiles) {
      const int64_t base = G / tiles, rem = G % tiles;
      int64_t t, r, m;
      if (b < rem * (base + 1)) {
        t = b / (base + 1); r = b % (base + 1); m = base + 1;
      } else {
        const int64_t b2 = b - rem * (base + 1);
        t = rem + b2 / base; r = b2 % base; m = base;
      }
      const int64_t p0 = r * planes / m, p1 = (r + 1) * planes / m;
      return Segments{t * planes + p0, t * planes + p1, planes};
    }
    if (mode == SPLIT_BALANCED) {
      const int64_t unit = 4 * (int64_t)planes + RAMP_MID_Q;   // quarter steps per tile
      const int64_t V = tiles * unit;
      auto cut = [&](int64_t bb) -> int64_t {
        if (bb >= G) return total;
        const int64_t v = bb * V / G;
        const int64_t t = v / unit;
        const int64_t off = v - t * unit - RAMP_MID_Q;
        int64_t p = off > 0 ? (off + 2) / 4 : 0;
        if (p > planes) p = planes;
        return t * planes + p;
      };
      return Segments{cut(b), cut(b + 1), planes};
    }
    return Segments{b * total / G, (b + 1) * total / G, planes};
  }
};

// Lockstep of the round-robin split (RR): CTAs that stage neighbouring tiles
// drift apart over the ~2500 steps of a 512^3 stage (there is no inter-CTA
// sync), so the halo columns and rows their boxes share were fetched from
// DRAM again by each of them (ncu at 512^3: SS stage kernel 36.5 GB of reads
// for 23.6 GB of inputs).  Each CTA publishes the number of step barriers it
// has passed; after a barrier one thread holds the CTA back while a
// neighbour in the tile grid (CTA b +- 1, b +- ntk: the same round deals
// them neighbouring tiles) is more than K steps behind.  The slowest CTA
// never waits and the static split ends with it anyway, so the wait is
// free; the halos now hit in L2 (SS 26.5 GB, 1.12x its inputs; stage kernel
// 10.6 -> 9.8 ms).  Each CTA's slot is its own 128 B line: with the slots
// packed, every publish invalidated the line its neighbours poll and a step
// took twice as long.  The spin is bounded: a stale or foreign value can
// only end the lockstep, never hang the GPU.
constexpr int PROG_DONE = 0x7fffffff;
constexpr int PROG_SLOTS = 1024;
constexpr int PROG_STRIDE = 32;   // ints per slot
constexpr int LS_TID = 5 * 32;    // the thread that publishes and waits
__device__ int g_prog[PROG_SLOTS * PROG_STRIDE];
__device__ __forceinline__ int ld_prog(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_prog(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// K = pf_saved bits 8..15 (0 = free running)
__device__ __forceinline__ int ls_slack(int pf_saved) {
  return gridDim.x <= PROG_SLOTS ? (pf_saved >> 8) & 0xff : 0;
}
__device__ __forceinline__ void ls_publish(int v) {
  st_prog(&g_prog[blockIdx.x * PROG_STRIDE], v);
}
// progress of tile-grid neighbour j (0: b-1, 1: b+1, 2: b-ntk, 3: b+ntk)
__device__ __forceinline__ int ls_neighbour(int j, int ntk) {
  const int b = (int)blockIdx.x, G = (int)gridDim.x;
  const int n = j == 0 ? b - 1 : (j == 1 ? b + 1 : (j == 2 ? b - ntk : b + ntk));
  return n >= 0 && n < G ? ld_prog(&g_prog[n * PROG_STRIDE]) : PROG_DONE;
}
// after the barrier of step w: publish, then wait for the neighbours (v: their
// progress as loaded before the barrier)
__device__ __forceinline__ void ls_step(int& ls_k, int w, const int* v, int ntk) {
  ls_publish(w + 1);
  const int need = w + 1 - ls_k;
  int m = min(min(v[0], v[1]), min(v[2], v[3]));
  if (m >= need) return;
  const long long t0 = clock64();
  do {
    m = min(min(ls_neighbour(0, ntk), ls_neighbour(1, ntk)),
            min(ls_neighbour(2, ntk), ls_neighbour(3, ntk)));
    if (clock64() - t0 > 400000LL) {   // ~200 us: leave the lockstep
      ls_k = 0;
      ls_publish(PROG_DONE);
      return;
    }
  } while (m < need);
}

// the round-robin kernels' tail values {main_end, tbeg, tend} (see
// Segments::next_rr); one instance per kernel instantiation that calls it
template <int TAG>
__device__ __forceinline__ volatile int64_t* tail_slot() {
  __shared__ int64_t s[3];
  return s;
}

#ifndef FDNS_EARLY_GV
#define FDNS_EARLY_GV 1
#endif

template <int V, int MODE, bool LAZY = true, bool RR = false>
__global__ void __launch_bounds__(NT, 1)
    k_stage_tiled(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tgw,
                  const __grid_constant__ CUtensorMap tsv, const __grid_constant__ CUtensorMap tgp,
                  const double* __restrict__ work,
                  const double* saved, double* out, Coef k, Geom g, double coef, int ntk,
                  int64_t total_steps, int wrap_mask, int i_lo, int nplanes, int split,
                  int pf_saved, const int64_t* __restrict__ cuts) {
  extern __shared__ __align__(128) double sm[];
  constexpr bool kBuf = (V == FDNS_SN);
  constexpr bool kGB = (V == FDNS_SS || V == FDNS_RS);
  double* bufs0 = sm + NR * SLOT;   // SN: 2 x NBUF buffer planes; SS/RS: 2 x NGB staged
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      sm + NR * SLOT + (kBuf ? 2 * NBUF * PLANE : (kGB ? 2 * NGB * PLANE : 0)));
  uint64_t* gbars = bars + NR;      // SS/RS: the two gradient-box barriers
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  Segments S = Segments::partition(blockIdx.x, gridDim.x, total_steps, nplanes, split, cuts);
  if constexpr (RR) S.tiles = (int64_t)ntk * ((g.n1 + TJ - 1) / TJ);
  volatile int64_t* s_tail = nullptr;
  if constexpr (RR) {
    s_tail = tail_slot<V * 4 + MODE * 2 + (LAZY ? 1 : 0)>();
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
  if (S.beg >= S.end) {
    if (RR && ls_slack(pf_saved) && threadIdx.x == LS_TID) ls_publish(PROG_DONE);
    return;
  }
  trace(0);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    if constexpr (kGB) { mbar_init(&gbars[0], 1); mbar_init(&gbars[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Programmatic dependent launch: let the next stage's grid launch now (its
  // CTAs take SMs as ours retire and run their prologue), and wait for the
  // previous stage's writes before touching global memory.
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  trace(1);
  // lockstep of the round-robin CTAs (after the wait: the previous stage's
  // CTAs no longer publish)
  int ls_k = 0;
  if constexpr (RR) ls_k = ls_slack(pf_saved);
  if (RR && ls_k && tid == LS_TID) ls_publish(0);
  const CUtensorMap* tmap = &tin;
  double* outp = out;
  const double coefp = coef;
  const int pfp = pf_saved;

  // SS/RS: staged gradient box of the centre plane of step `gs`
  auto issue_gb_tile = [&](int gs, int k0, int j0, int plane) {
    double* dst = bufs0 + (gs & 1) * NGB * PLANE;
    mbar_expect_tx(&gbars[gs & 1], GB_BYTES);
    tma_load_plane(dst, &tgw, &gbars[gs & 1], k0 + g.h - 2, j0 + g.h - 2, plane + g.h);
  };
  auto issue_gb = [&](int gs, int64_t tile, int plane) {
    issue_gb_tile(gs, (int)(tile % ntk) * TK, (int)(tile / ntk) * TJ, plane);
  };
  if constexpr (kGB) {
    if (tid == 0) issue_gb(0, tile_at(S.beg), i_lo + plane_at(S.beg));
  }
  int gs = 0;   // step counter of this CTA (gradient-box parity)

  // producer cursor (thread 0): stream position, current segment, position
  // within it
  // (box coordinates are recomputed only when the cursor enters a segment:
  // no 64-bit division per issued plane)
  int64_t p_seg = S.beg;
  int p_r = 0;
  int issued = 0;
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
    tma_load_plane(sm + p_slot * SLOT, tmap, &bars[p_slot], p_c0, p_c1, p_plane + p_r);
    // saved state of this plane (a centre plane of the segment) into L2,
    // ~NR steps before the epilogue loads it: when it is not the stage
    // input it would otherwise come from DRAM at full latency
    if (MODE == 1 && (pfp & PF_SAVED) && p_r >= 2 && p_r < p_len - 2)
      tma_prefetch_l2(&tsv, p_c0 + 2, p_c1 + 2, p_plane + p_r);
    // SS/RS: the nine stored gradients of this plane's tile columns (the
    // off-diagonal loads at the centre and the axis-0 queue loads) into L2
    if constexpr (kGB)
      if (pfp & PF_GRAD) tma_prefetch_l2(&tgp, p_c0 + 2, p_c1 + 2, p_plane + p_r);
    ++issued;
    p_slot = p_slot + 1 == NR ? 0 : p_slot + 1;
    if (++p_r == p_len) {
      p_r = 0;
      p_seg = seg_next(p_seg);
      if (p_seg < S.end) enter_segment();
    }
  };
  int stage_pos = 0;   // stream positions of one stage (steps + 4 per segment)
  for (int64_t x = S.beg; x < S.end; x = seg_next(x)) stage_pos += (int)(seg_end(x) - x) + 4;
  int total_pos = stage_pos;   // issue limit: end of the current stage
  if (tid == 0)
    while (issued < total_pos && issued < NR) issue_next();

  int w = 0;    // stream position of the current window start
  int wsl = 0;  // w % NR, maintained incrementally (no per-step modulo)
  auto slot_of = [&](int d) {  // ring slot of window position d (0..5)
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
    const int nsteps = (int)(se - x);
    const int i_seg = i_lo + plane_at(x);   // axis-0 index of step 0
    if constexpr (RR) {
      // the last round's plane ranges differ per CTA: free running from here
      if (ls_k && x >= s_tail[0]) {
        if (tid == LS_TID) ls_publish(PROG_DONE);
        ls_k = 0;
      }
    }
    double q1[5], q2[5];   // SN axis-0 queues
    for (int t = 0; t < nsteps; ++t, ++w, ++gs, wsl = (wsl + 1 == NR ? 0 : wsl + 1)) {
      if (t == 0 && w > 0) {
        // segment change: the new window needs 5 fresh planes; refill the
        // ring once every thread is done with the previous segment's slots
        __syncthreads();
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          while (issued < total_pos && issued < w + NR) issue_next();
        }
      }
      const int i = i_seg + t;
      // this step's global loads are issued first, so their latency runs
      // under the plane's arrival conversion and the barrier: the saved
      // state (MODE 1) and, for SS/RS, the stored gradients (the axis-0
      // queue heads and the six off-diagonal values at the point);
      // inactive (edge) threads read a valid clamped column, never written
      const int64_t cl = (int64_t)(i + g.h) * g.s0 + (int64_t)(min(jj, g.n1 - 1) + g.h) * g.s1 +
                         (min(kk, g.n2 - 1) + g.h);
      double sv[5];
      if constexpr (MODE == 1) {
#pragma unroll
        for (int f = 0; f < 5; ++f) sv[f] = saved[f * g.fs + cl];
      }
      int ls_v[4] = {PROG_DONE, PROG_DONE, PROG_DONE, PROG_DONE};
      if constexpr (RR) {
        if (ls_k && tid == LS_TID) {   // consumed after the step barrier
#pragma unroll
          for (int j = 0; j < 4; ++j) ls_v[j] = ls_neighbour(j, ntk);
        }
      }
      double gv[9];
      if constexpr (kGB && FDNS_EARLY_GV) {
        const double* w11 = work + 4 * g.fs + cl;   // stored D(u1,x1)
        const double* w22 = work + 8 * g.fs + cl;   // stored D(u2,x2)
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
        gv[0 * 3 + 1] = __ldg(work + 1 * g.fs + cl);
        gv[0 * 3 + 2] = __ldg(work + 2 * g.fs + cl);
        gv[1 * 3 + 0] = __ldg(work + 3 * g.fs + cl);
        gv[1 * 3 + 2] = __ldg(work + 5 * g.fs + cl);
        gv[2 * 3 + 0] = __ldg(work + 6 * g.fs + cl);
        gv[2 * 3 + 1] = __ldg(work + 7 * g.fs + cl);
      }
      if (t == 0) {
        for (int d = 0; d < 5; ++d) {
          const int pp = w + d;
          mbar_wait(&bars[slot_of(d)], (pp / NR) & 1);
          stage_arrival(k, sm + slot_of(d) * SLOT, tid, NT);
        }
      } else {
        mbar_wait(&bars[slot_of(4)], ((w + 4) / NR) & 1);
        stage_arrival(k, sm + slot_of(4) * SLOT, tid, NT);
      }
      double* bufs = bufs0 + (w & 1) * NBUF * PLANE;
      if constexpr (kBuf) {
        // centre-plane buffers over the staged box (u0..u2 are untouched by
        // the energy conversion, so no barrier is needed before this).
        // Fixed per-thread items (no index math or branching per step): box
        // positions tid and tid+NT of each buffer, predicated.
        const double* base[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) base[d] = sm + slot_of(d) * SLOT;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int x0 = tid + m * NT;                       // D(u0,x0), whole box
          if (m == 0 || x0 < PLANE) {
            SAcc b;
#pragma unroll
            for (int d = 0; d < 5; ++d) b.p[d] = base[d] + x0;
            bufs[x0] = d1<0, E_FIELD, U0, 0>(k, b);
          }
          const int y1 = tid + m * NT;                       // D(u1,x1), rows 2..TJ+1
          if (y1 < BU1_N) {
            const int pos = 2 * PK + y1;
            SAcc b;
            b.p[2] = base[2] + pos;
            bufs[PLANE + pos] = d1<1, E_FIELD, U1, 0>(k, b);
          }
          const int y2 = tid + m * NT;                       // D(u2,x2), cols 2..TK+1
          if (y2 < BU2_N) {
            const int pos = (y2 / TK) * PK + 2 + y2 % TK;
            SAcc b;
            b.p[2] = base[2] + pos;
            bufs[2 * PLANE + pos] = d1<2, E_FIELD, U2, 0>(k, b);
          }
        }
      }
      __syncthreads();
      if (w == 0) trace(2);
      if constexpr (RR) {
        if (ls_k && tid == LS_TID) ls_step(ls_k, w, ls_v, ntk);
      }
      if (tid == 0) {
        if (issued < total_pos && issued < w + NR) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          while (issued < total_pos && issued < w + NR) issue_next();
        }
        if constexpr (kGB) {   // next step's centre gradient box
          if (t + 1 < nsteps) {
            issue_gb_tile(gs + 1, k0, j0, i_seg + t + 1);
          } else if (seg_next(x) < S.end) {
            issue_gb(gs + 1, tile_at(seg_next(x)), i_lo + plane_at(seg_next(x)));
          }
        }
      }
      SAcc a;
#pragma unroll
      for (int d = 0; d < 5; ++d) a.p[d] = sm + slot_of(d) * SLOT + toff;

      if constexpr (kBuf) {
        // axis-0 queues of D(u1,x1), D(u2,x2) at this column
        if (t == 0) {
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            SAcc b;
            b.p[2] = a.p[d];
            q1[d] = d1<1, E_FIELD, U1, 0>(k, b);
            q2[d] = d1<2, E_FIELD, U2, 0>(k, b);
          }
        } else {
#pragma unroll
          for (int d = 0; d < 4; ++d) { q1[d] = q1[d + 1]; q2[d] = q2[d + 1]; }
          SAcc b;
          b.p[2] = a.p[4];
          q1[4] = d1<1, E_FIELD, U1, 0>(k, b);
          q2[4] = d1<2, E_FIELD, U2, 0>(k, b);
        }
      }

      double r[NFIELDS];
#pragma unroll
      for (int f = 0; f < NFIELDS; ++f) r[f] = a.v(f, 0, 0, 0);   // r[RHOE_F] = rho*e
      double R[5];
      if constexpr (V == FDNS_SN) {
        if constexpr (LAZY) {
          const TiledLazyProvider P{k, a, q1, q2, bufs + toff, bufs + PLANE + toff,
                                    bufs + 2 * PLANE + toff};
          residual_point<true>(k, P, r, R);
        } else {
          TiledLocalProvider P(k, a, q1, q2, bufs + toff, bufs + PLANE + toff,
                               bufs + 2 * PLANE + toff);
          residual_point<true>(k, P, r, R);
        }
      } else if constexpr (V == FDNS_RA) {
        InlineProvider<SAcc> P(k, a);
        residual_point<true>(k, P, r, R);
      } else {  // SS / RS: stored velocity gradients from the work arrays
        if constexpr (!FDNS_EARLY_GV) {
          const double* w11 = work + 4 * g.fs + cl;   // stored D(u1,x1)
          const double* w22 = work + 8 * g.fs + cl;   // stored D(u2,x2)
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
          gv[0 * 3 + 1] = __ldg(work + 1 * g.fs + cl);
          gv[0 * 3 + 2] = __ldg(work + 2 * g.fs + cl);
          gv[1 * 3 + 0] = __ldg(work + 3 * g.fs + cl);
          gv[1 * 3 + 2] = __ldg(work + 5 * g.fs + cl);
          gv[2 * 3 + 0] = __ldg(work + 6 * g.fs + cl);
          gv[2 * 3 + 1] = __ldg(work + 7 * g.fs + cl);
        }
        mbar_wait(&gbars[gs & 1], (gs >> 1) & 1);
        const double* gb = bufs0 + (gs & 1) * NGB * PLANE + toff;
        const TiledSSProvider<V == FDNS_RS> P{k, a, q1, q2, gb, gb + PLANE, gb + 2 * PLANE, gv};
        residual_point<true>(k, P, r, R);
      }
      if (active) {
        if constexpr (MODE == 0) {
          emit<5>(out, g, i, jj, kk, R, 0);
        } else {
          const int64_t c = (int64_t)(i + g.h) * g.s0 + (int64_t)(jj + g.h) * g.s1 + (kk + g.h);
          double q[NFIELDS];
          (void)c;
          stage_update(sv, R, coefp, q);
          emit<NOUT_STAGE>(outp, g, i, jj, kk, q, wrap_mask);
        }
      }
    }
    w += 4;   // the segment's trailing positions
    wsl = w % NR;
  }
  if (RR && tid == LS_TID && ls_slack(pf_saved)) ls_publish(PROG_DONE);
  trace(3);
}

}  // namespace tiled
}  // namespace fdns
