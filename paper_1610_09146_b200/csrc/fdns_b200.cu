// fdns_b200.cu -- sm_100a kernels and the C ABI (include/fdns_b200.h).
//
// Built with -fmad=false (no FMA contraction) and IEEE division so every
// kernel reproduces the reference's bits (see fdns_math.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fdns_b200.h"
#include "fdns_math.cuh"
#include "fdns_tiled.cuh"
#include "fdns_tiled12.cuh"

#include <cudaTypedefs.h>


using namespace fdns;

namespace {

thread_local std::string g_err;
int g_kernel_path = 0;        // test hook: 0 default, 1 point kernels, 2 8-warp tiled
                              // (SN, RA), 4 eager-local SN, 5 12-warp (SN, RA)
int g_tiled_ctas = 0;         // test hook: force the tiled grid size (0 = one per SM)
std::atomic<long long> g_launches{0};
inline void count(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int fail(const char* what, cudaError_t e) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return 1;
}
int fail(const std::string& what) {
  g_err = what;
  return 2;
}
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(what, e);
  return 0;
}

Coef make_coef(const fdns_problem* pb) {
  Coef k;
  for (int a = 0; a < 3; ++a) {
    k.w1[a] = pb->w[5 * a + 0];
    k.w2[a] = pb->w[5 * a + 1];
    k.s0[a] = pb->w[5 * a + 2];
    k.s1[a] = pb->w[5 * a + 3];
    k.s2[a] = pb->w[5 * a + 4];
  }
  k.inv_Re = pb->kc[0];
  k.c13 = pb->kc[1];
  k.c43 = pb->kc[2];
  k.c23 = pb->kc[3];
  k.heat = pb->kc[4];
  k.gm1 = pb->gm1;
  k.gM2 = pb->gM2;
  return k;
}

Geom make_geom(const fdns_problem* pb) {
  Geom g;
  g.n0 = pb->n[0];
  g.n1 = pb->n[1];
  g.n2 = pb->n[2];
  g.h = pb->h;
  const int64_t P1 = g.n1 + 2 * g.h, P2 = g.n2 + 2 * g.h;
  g.s1 = P2;
  g.s0 = P1 * P2;
  g.fs = (int64_t)(g.n0 + 2 * g.h) * g.s0;
  return g;
}

// Whether two bundles of na / nb padded fields overlap in memory.
bool overlaps(const double* a, int na, const double* b, int nb, const Geom& g) {
  if (!a || !b) return false;
  const double *ae = a + na * g.fs, *be = b + nb * g.fs;
  return a < be && b < ae;
}

int validate(const fdns_problem* pb) {
  if (!pb) return fail("null problem");
  if (pb->h < 2) return fail("halo width must be >= 2");
  for (int a = 0; a < 3; ++a)
    if (pb->n[a] < 1) return fail("interior extent must be positive");
  if (pb->n[1] < pb->h || pb->n[2] < pb->h) return fail("axes 1/2 need at least h points");
  return 0;
}

// ---------------------------------------------------------------------------
// Primitives over the full padded bundle
// ---------------------------------------------------------------------------
// Entry of a kernel launched with programmatic dependent launch: wait for
// the preceding kernel's writes before any global access, then let the
// next kernel in the stream be scheduled as this grid's CTAs retire.  (A
// no-op pair when launched without the attribute.)
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void k_primitives(double* __restrict__ F, Coef k, int64_t fs, int64_t c0,
                             int64_t c1) {
  for (int64_t c = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < c1;
       c += (int64_t)gridDim.x * blockDim.x) {
    double q[5], pr[5];
#pragma unroll
    for (int f = 0; f < 5; ++f) q[f] = F[f * fs + c];
    primitives_point(k, q, pr);
#pragma unroll
    for (int f = 0; f < 5; ++f) F[(5 + f) * fs + c] = pr[f];
  }
}

// ---------------------------------------------------------------------------
// Periodic ghost fill (mesh.py:118-139).  After the reference's axis-ordered
// full-slab copies every ghost holds the interior value at the coordinates
// wrapped on each exchanged axis; this kernel writes exactly that, visiting
// only ghost points (three disjoint regions).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int wrap(int x, int n, int h) {
  return x < h ? x + n : (x >= n + h ? x - n : x);
}

__global__ void k_halo_wrap(double* __restrict__ F, int nf, int mask, Geom g, int64_t r0,
                            int64_t r1, int64_t r2) {
  const int h = g.h;
  const int P0 = g.n0 + 2 * h, P1 = g.n1 + 2 * h, P2 = g.n2 + 2 * h;
  const bool m0 = mask & 1, m1 = mask & 2, m2 = mask & 4;
  const int64_t total = r0 + r1 + r2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i, j, k;
    if (t < r0) {  // axis-0 ghost planes, all j, k
      int64_t u = t;
      k = u % P2; u /= P2;
      j = u % P1; u /= P1;
      i = (int)u;  // 0 .. 2h-1
      i = i < h ? i : g.n0 + i;
    } else if (t < r0 + r1) {  // axis-1 ghosts
      int64_t u = t - r0;
      const int ni = m0 ? g.n0 : P0;
      k = u % P2; u /= P2;
      j = u % (2 * h); u /= (2 * h);
      i = (int)u + (m0 ? h : 0);
      (void)ni;
      j = j < h ? j : g.n1 + j;
    } else {  // axis-2 ghosts
      int64_t u = t - r0 - r1;
      const int nj = m1 ? g.n1 : P1;
      k = u % (2 * h); u /= (2 * h);
      j = (int)(u % nj) + (m1 ? h : 0); u /= nj;
      i = (int)u + (m0 ? h : 0);
      k = k < h ? k : g.n2 + k;
    }
    const int si = m0 ? wrap(i, g.n0, h) : i;
    const int sj = m1 ? wrap(j, g.n1, h) : j;
    const int sk = m2 ? wrap(k, g.n2, h) : k;
    const int64_t dst = i * g.s0 + j * g.s1 + k;
    const int64_t src = si * g.s0 + sj * g.s1 + sk;
    for (int f = 0; f < nf; ++f) F[f * g.fs + dst] = F[f * g.fs + src];
  }
}

// ---------------------------------------------------------------------------
// Point-kernel residual (one thread per interior point), all variants.
// Mode: 0 = write residual, 1 = fused RK update + primitives.
// ---------------------------------------------------------------------------
// Axis-2 index of a point-kernel thread, shifted so that a warp's 32
// consecutive points start on a 32-byte sector of the padded row (interior
// column 0 sits h doubles into the row): full-sector stores, no
// read-modify-write of half-written sectors in L2/DRAM, and 8 instead of 9
// sectors per warp load (BL steps +5% at 256^3).  Needs rows that are a
// whole number of sectors; costs one extra, mostly idle block column per
// row, so it is used from n2 >= 128 on (at 64^3 it measured -3%).
__host__ __device__ __forceinline__ int ksector_shift(const Geom& g) {
  return (((g.n2 + 2 * g.h) & 3) == 0 && g.n2 >= 128) ? (g.h & 3) : 0;
}
__device__ __forceinline__ int point_k(const Geom& g) {
  return (int)(blockIdx.x * blockDim.x + threadIdx.x) - ksector_shift(g);
}

template <int V, int MODE>
__global__ void __launch_bounds__(256) k_residual(const double* __restrict__ in,
                                                  const double* saved, double* out,
                                                  const double* __restrict__ work, Coef k,
                                                  Geom g, double coef, int wrap_mask,
                                                  int i_lo) {
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  // BL walks its planes backwards: the fill just wrote them forwards, so
  // the most recently written (still L2-resident) planes of the 60 work
  // arrays are read first, and the next stage's forward fill starts on the
  // planes this kernel wrote last (BL 64^3 steps +6.7%, where the 151 MB
  // of work arrays just exceed L2; neutral from 128^3)
  const int ii = V == FDNS_BL ? i_lo + (int)(gridDim.z - 1 - blockIdx.z) : blockIdx.z + i_lo;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
  double r[NFIELDS];
#pragma unroll
  for (int f = 0; f < NFIELDS; ++f) r[f] = __ldg(in + f * g.fs + c);
  double R[5];
  if constexpr (V == FDNS_SN) {
    GAcc a{in, c, g.s0, g.s1, g.fs};
    LocalProvider<GAcc> P(k, a);
    residual_point(k, P, r, R);
  } else if constexpr (V == FDNS_RA) {
    GAcc a{in, c, g.s0, g.s1, g.fs};
    InlineProvider<GAcc> P(k, a);
    residual_point(k, P, r, R);
  } else if constexpr (V == FDNS_BL) {
    FetchProvider P{work, c, g.fs};
    residual_point(k, P, r, R);
  } else if constexpr (V == FDNS_SS) {
    GAcc a{in, c, g.s0, g.s1, g.fs};
    SSProvider<GAcc> P(k, a, work, c, g.fs, g.s0, g.s1);
    residual_point(k, P, r, R);
  } else {  // RS: stored velocity gradients, everything else inline
    GAcc a{in, c, g.s0, g.s1, g.fs};
    SSProvider<GAcc, true> P(k, a, work, c, g.fs, g.s0, g.s1);
    residual_point(k, P, r, R);
  }
  if constexpr (MODE == 0) {
    tiled::emit<5>(out, g, ii, jj, kk, R, 0);
  } else {
    double q[NFIELDS];
#pragma unroll
    for (int f = 0; f < 5; ++f) q[f] = saved[f * g.fs + c] + coef * R[f];
    primitives_point(k, q, q + 5);
    tiled::emit<NFIELDS>(out, g, ii, jj, kk, q, wrap_mask);
  }
}

template <int A_, int L>
__device__ __forceinline__ void fill_axis_all(const Coef& k, const GAcc& a,
                                              double* __restrict__ wa, int64_t fs) {
  wa[slot(A_, L) * fs + a.c] = eval_slot<A_, L>(k, a);
  if constexpr (L + 1 < S_PER_AXIS) fill_axis_all<A_, L + 1>(k, a, wa, fs);
}

// All 54 plain/product derivatives of an interior point in one pass over the
// fields (the reference's separate fill loops, plan.py:369-392, fused; each
// value is the same expression, so bitwise equal).
// AXES: bit a = fill the 18 slots of axis a (7 = all 54; 6 = the in-plane
// 36, beside the axis-0-marching k_fill_bl_ax0).
template <int AXES = 7>
__global__ void __launch_bounds__(256) k_fill_bl_all(const double* __restrict__ in,
                                                     double* __restrict__ wa, Coef k, Geom g) {
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
  GAcc a{in, c, g.s0, g.s1, g.fs};
  if constexpr (AXES & 1) fill_axis_all<0, 0>(k, a, wa, g.fs);
  if constexpr (AXES & 2) fill_axis_all<1, 0>(k, a, wa, g.fs);
  if constexpr (AXES & 4) fill_axis_all<2, 0>(k, a, wa, g.fs);
}

// ---------------------------------------------------------------------------
// Axis-0-marching fills.  A thread owns one (axis-1, axis-2) column and walks
// NPL consecutive planes, keeping the five-plane axis-0 stencil window of the
// fields it differentiates along axis 0 in registers (QAcc): each input
// value comes from DRAM about once (plus 4/NPL halo planes per chunk)
// instead of once per axis-0 tap -- with 54 output streams flowing through
// L2, the one-thread-per-point fill re-read every input ~5x (ncu at 512^3:
// 55 GB of reads for 10.7 GB of inputs).  In-plane taps still come through
// the read-only path (L1/L2 hits: the CTA's neighbouring columns loaded
// them).  Same expressions through the same eval_slot/d1 templates, so the
// bits are the point kernel's.
// ---------------------------------------------------------------------------
template <int NQ>
struct QAcc {
  static constexpr bool kInternalEnergy = false;
  const double (&q)[NQ][5];   // q[f][d]: field f at axis-0 offset d-2
  const double* __restrict__ b;
  int64_t c, s0, s1, fs;
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    if (dj == 0 && dk == 0) return q[f][di + 2];
    return __ldg(b + f * fs + c + di * s0 + dj * s1 + dk);
  }
};

template <int NQ>
__device__ __forceinline__ void load_plane(double (&dst)[NQ], const double* __restrict__ in,
                                           int64_t c, int64_t fs, const int (&fld)[NQ]) {
#pragma unroll
  for (int f = 0; f < NQ; ++f) dst[f] = __ldg(in + fld[f] * fs + c);
}

template <int A_, int L, int NQ>
__device__ __forceinline__ void fill_axis_q(const Coef& k, const QAcc<NQ>& a,
                                            double* __restrict__ wa, int64_t fs) {
  wa[slot(A_, L) * fs + a.c] = eval_slot<A_, L>(k, a);
  if constexpr (L + 1 < S_PER_AXIS) fill_axis_q<A_, L + 1>(k, a, wa, fs);
}

// BL: all 54 plain/product derivatives (the 10 point fields queued).
constexpr int MARCH_BX = 32, MARCH_BY = 4;
#ifndef FDNS_MARCH_MINB
#define FDNS_MARCH_MINB 1
#endif
template <int NPL, int AXES = 7>
__global__ void __launch_bounds__(MARCH_BX * MARCH_BY, FDNS_MARCH_MINB) k_fill_bl_march(
    const double* __restrict__ in, double* __restrict__ wa, Coef k, Geom g) {
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int i0 = blockIdx.z * NPL, i1 = min(i0 + NPL, g.n0);
  const int64_t col = (int64_t)(jj + g.h) * g.s1 + (kk + g.h);
  constexpr int fld[NFIELDS] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9};
  double q[NFIELDS][5], nx[NFIELDS];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    double t[NFIELDS];
    load_plane<NFIELDS>(t, in, (int64_t)(i0 - 2 + d + g.h) * g.s0 + col, g.fs, fld);
#pragma unroll
    for (int f = 0; f < NFIELDS; ++f) q[f][d] = t[f];
  }
  load_plane<NFIELDS>(nx, in, (int64_t)(i0 + 2 + g.h) * g.s0 + col, g.fs, fld);
#pragma unroll 1
  for (int i = i0; i < i1; ++i) {
#pragma unroll
    for (int f = 0; f < NFIELDS; ++f) q[f][4] = nx[f];
    if (i + 1 < i1)   // next step's new plane, loaded under this step's work
      load_plane<NFIELDS>(nx, in, (int64_t)(i + 3 + g.h) * g.s0 + col, g.fs, fld);
    const QAcc<NFIELDS> a{q, in, (int64_t)(i + g.h) * g.s0 + col, g.s0, g.s1, g.fs};
    if constexpr (AXES & 1) fill_axis_q<0, 0>(k, a, wa, g.fs);
    if constexpr (AXES & 2) fill_axis_q<1, 0>(k, a, wa, g.fs);
    if constexpr (AXES & 4) fill_axis_q<2, 0>(k, a, wa, g.fs);
#pragma unroll
    for (int f = 0; f < NFIELDS; ++f)
#pragma unroll
      for (int d = 0; d < 4; ++d) q[f][d] = q[f][d + 1];
  }
}

// The same with the axis-0 window in shared memory instead of registers:
// each thread keeps its own column's ten fields on five planes in a ring
// (slot = plane mod 5, [slot][field][thread]: consecutive threads hit
// consecutive words), so no barrier is needed and the registers are left to
// the in-plane taps -- four 128-thread CTAs per SM instead of the two the
// 255-register queue allowed (ncu at 512^3: 12% warps active, long-
// scoreboard bound, 4.2 TB/s).
struct SQAcc {
  static constexpr bool kInternalEnergy = false;
  const double* p[5];          // plane slots of axis-0 offsets -2..+2 (this thread)
  const double* __restrict__ b;
  int64_t c, s0, s1, fs;
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    if (dj == 0 && dk == 0) return p[di + 2][f * (MARCH_BX * MARCH_BY)];
    return __ldg(b + f * fs + c + di * s0 + dj * s1 + dk);
  }
};

// Work-array stores of the fills: written once, read by a later kernel long
// after they have left L2 -- evict-first (st.global.cs) keeps the 9 or 54
// output streams from pushing the fills' own input planes (re-read by the
// next planes' blocks) out of L2.  FDNS_FILL_CS=0: plain stores (A/B).
#ifndef FDNS_FILL_CS
#define FDNS_FILL_CS 1
#endif
__device__ __forceinline__ void st_fill(double* p, double v) {
#if FDNS_FILL_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}
template <bool CS>
__device__ __forceinline__ void st_fill2(double* p, double2 v) {
  if constexpr (CS && FDNS_FILL_CS) __stcs(reinterpret_cast<double2*>(p), v);
  else *reinterpret_cast<double2*>(p) = v;
}
// Measured whole RK3 steps (profiles/r02_fill_cs_ab.txt): at 512^3 SS +0.4%,
// RS +0.5%, BL +1.5-2.5% (BL fill reads 18.5 -> 14.7 GB); at 256^3 and
// 128^3 SS/RS lose 1.5% (the stage kernel then finds fewer of the freshly
// written gradients in L2), so the paired kernels take it from 64M points.
inline bool fill_cs(const Geom& g) { return (int64_t)g.n0 * g.n1 * g.n2 >= (64ll << 20); }

template <int A_, int L>
__device__ __forceinline__ void fill_axis_sq(const Coef& k, const SQAcc& a,
                                             double* __restrict__ wa, int64_t fs) {
  st_fill(&wa[slot(A_, L) * fs + a.c], eval_slot<A_, L>(k, a));
  if constexpr (L + 1 < S_PER_AXIS) fill_axis_sq<A_, L + 1>(k, a, wa, fs);
}

#ifndef FDNS_MARCH_SMEM_MINB
#define FDNS_MARCH_SMEM_MINB 3
#endif
constexpr int MARCH_NT = MARCH_BX * MARCH_BY;
constexpr int MARCH_SMEM = 5 * NFIELDS * MARCH_NT * 8;   // 51200 B
template <int NPL>
__global__ void __launch_bounds__(MARCH_NT, FDNS_MARCH_SMEM_MINB) k_fill_bl_march_s(
    const double* __restrict__ in, double* __restrict__ wa, Coef k, Geom g) {
  extern __shared__ __align__(16) double qs[];
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int tid = threadIdx.y * MARCH_BX + threadIdx.x;
  double* mine = qs + tid;
  auto slot_ptr = [&](int plane) { return mine + (plane % 5) * NFIELDS * MARCH_NT; };
  const int i0 = blockIdx.z * NPL, i1 = min(i0 + NPL, g.n0);
  const int64_t col = (int64_t)(jj + g.h) * g.s1 + (kk + g.h);
  // planes i0-2 .. i0+1 (index shifted by +2 so it stays non-negative)
#pragma unroll 1
  for (int d = 0; d < 4; ++d) {
    double* sp = slot_ptr(i0 + d);
    const int64_t c = (int64_t)(i0 - 2 + d + g.h) * g.s0 + col;
#pragma unroll
    for (int f = 0; f < NFIELDS; ++f) sp[f * MARCH_NT] = __ldg(in + f * g.fs + c);
  }
  double nx[NFIELDS];
#pragma unroll
  for (int f = 0; f < NFIELDS; ++f)
    nx[f] = __ldg(in + f * g.fs + (int64_t)(i0 + 2 + g.h) * g.s0 + col);
#pragma unroll 1
  for (int i = i0; i < i1; ++i) {
    {
      double* sp = slot_ptr(i + 4);   // plane i+2 (offset +2)
#pragma unroll
      for (int f = 0; f < NFIELDS; ++f) sp[f * MARCH_NT] = nx[f];
    }
    if (i + 1 < i1) {
#pragma unroll
      for (int f = 0; f < NFIELDS; ++f)
        nx[f] = __ldg(in + f * g.fs + (int64_t)(i + 3 + g.h) * g.s0 + col);
    }
    SQAcc a;
#pragma unroll
    for (int d = 0; d < 5; ++d) a.p[d] = slot_ptr(i + d);
    a.b = in;
    a.c = (int64_t)(i + g.h) * g.s0 + col;
    a.s0 = g.s0; a.s1 = g.s1; a.fs = g.fs;
    fill_axis_sq<0, 0>(k, a, wa, g.fs);
    fill_axis_sq<1, 0>(k, a, wa, g.fs);
    fill_axis_sq<2, 0>(k, a, wa, g.fs);
  }
}


// D(u_Q, x_Q) on the ghost frame only: points whose axis-Q coordinate is
// interior while another coordinate lies in the halo (the interior values
// come from the fill kernels).  Together they hold exactly what the
// reference's halo-exchanged inner arrays hold (plan.py:378-379).
template <int Q>
__device__ __forceinline__ void diag_ghost_point(const double* __restrict__ in,
                                                 double* __restrict__ dst, const Coef& k,
                                                 const Geom& g, int64_t t) {
  const int h = g.h;
  const int n[3] = {g.n0, g.n1, g.n2};
  constexpr int A = Q == 0 ? 1 : 0;   // the two other axes, A < B
  constexpr int B = Q == 2 ? 1 : 2;
  const int PB = n[B] + 2 * h;
  const int64_t frame = (int64_t)2 * h * PB + (int64_t)n[A] * 2 * h;
  const int q = (int)(t / frame) + h;
  int64_t f = t % frame;
  int ca, cb;
  if (f < (int64_t)2 * h * PB) {            // ghost rows of axis A, all of B
    ca = (int)(f / PB); cb = (int)(f % PB);
    ca = ca < h ? ca : n[A] + ca;
  } else {                                   // interior A, ghost columns of B
    f -= (int64_t)2 * h * PB;
    ca = (int)(f / (2 * h)) + h; cb = (int)(f % (2 * h));
    cb = cb < h ? cb : n[B] + cb;
  }
  int idx[3];
  idx[Q] = q; idx[A] = ca; idx[B] = cb;
  const int64_t c = idx[0] * g.s0 + idx[1] * g.s1 + idx[2];
  GAcc a{in, c, g.s0, g.s1, g.fs};
  dst[c] = d1<Q, E_FIELD, U0 + Q, 0>(k, a);
}

// D(u_q, x_q) on the ghost frames of all three diagonal arrays in one
// launch: points whose axis-q coordinate is interior while another
// coordinate lies in the halo (the interior values come from the fill
// kernels).  Together they hold exactly what the reference's halo-exchanged
// inner arrays hold (plan.py:378-379).
__global__ void k_diag_ghost(const double* __restrict__ in, double* __restrict__ d0,
                             double* __restrict__ d1p, double* __restrict__ d2p, Coef k, Geom g,
                             int64_t f0, int64_t f1, int64_t f2) {
  pdl_entry();
  const int64_t total = f0 + f1 + f2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < f0) diag_ghost_point<0>(in, d0, k, g, t);
    else if (t < f0 + f1) diag_ghost_point<1>(in, d1p, k, g, t - f0);
    else diag_ghost_point<2>(in, d2p, k, g, t - f0 - f1);
  }
}

// BL mixed fills: outer derivative of the stored inner arrays (plan.py:380-382).
__global__ void __launch_bounds__(256, 4) k_fill_cross(double* __restrict__ wa, Coef k, Geom g) {
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
  const int64_t st[3] = {g.s0, g.s1, 1};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double* inner = wa + slot(j, S_U + j) * g.fs;
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      if (o == j) continue;
      wa[(S_DD + dd_index(j, o)) * g.fs + c] = d1_stored(k, o, inner, c, st[o]);
    }
  }
}

// The same for two axis-2 neighbours per thread through 16-byte accesses
// (k_grad_ss_pair's layout): 22 loads + 6 stores per pair instead of 48 + 12.
template <bool CS>
__global__ void __launch_bounds__(256, 3) k_fill_cross_pair(double* __restrict__ wa, Coef k,
                                                            Geom g) {
  pdl_entry();
  const int pk = (int)(blockIdx.x * 64 + 2 * threadIdx.x);   // padded column of the pair
  const int kk = pk - g.h;
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + pk;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double* inner = wa + slot(j, S_U + j) * g.fs + c;
    auto ld2 = [&](int64_t off) { return __ldg(reinterpret_cast<const double2*>(inner + off)); };
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      if (o == j) continue;
      double2 d;
      if (o < 2) {
        const int64_t st = o == 0 ? g.s0 : g.s1;
        const double2 p1 = ld2(st), m1 = ld2(-st), p2 = ld2(2 * st), m2 = ld2(-2 * st);
        d.x = k.w1[o] * (p1.x - m1.x) + k.w2[o] * (p2.x - m2.x);
        d.y = k.w1[o] * (p1.y - m1.y) + k.w2[o] * (p2.y - m2.y);
      } else {
        const double2 a = ld2(-2), b = ld2(0), e = ld2(2);
        d.x = k.w1[2] * (b.y - a.y) + k.w2[2] * (e.x - a.x);
        d.y = k.w1[2] * (e.x - b.x) + k.w2[2] * (e.y - a.y);
      }
      st_fill2<CS>(wa + (S_DD + dd_index(j, o)) * g.fs + c, d);
    }
  }
}

// SS/RS fill in one launch: the nine velocity gradients ws[q*3+a] =
// D(u_q, x_a) on the interior, then the ghost frames of the three diagonal
// ones (k_diag_ghost semantics).
__global__ void __launch_bounds__(256) k_grad_ss_all(const double* __restrict__ in,
                                                     double* __restrict__ ws, Coef k, Geom g,
                                                     int64_t nint, int64_t f0, int64_t f1,
                                                     int64_t f2) {
  pdl_entry();
  const int64_t total = nint + f0 + f1 + f2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nint) {
      const int kk = (int)(t % g.n2);
      const int64_t u = t / g.n2;
      const int jj = (int)(u % g.n1);
      const int ii = (int)(u / g.n1);
      const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
      GAcc a{in, c, g.s0, g.s1, g.fs};
      ws[(0 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U0, 0>(k, a);
      ws[(0 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U0, 0>(k, a);
      ws[(0 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U0, 0>(k, a);
      ws[(1 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U1, 0>(k, a);
      ws[(1 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U1, 0>(k, a);
      ws[(1 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U1, 0>(k, a);
      ws[(2 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U2, 0>(k, a);
      ws[(2 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U2, 0>(k, a);
      ws[(2 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U2, 0>(k, a);
    } else {
      const int64_t x = t - nint;
      if (x < f0) diag_ghost_point<0>(in, ws + 0 * g.fs, k, g, x);
      else if (x < f0 + f1) diag_ghost_point<1>(in, ws + 4 * g.fs, k, g, x - f0);
      else diag_ghost_point<2>(in, ws + 8 * g.fs, k, g, x - f0 - f1);
    }
  }
}

// One stencil applied to one padded field, interior points only
// (stencil.py:71-102): first derivative along `op` (0-2) or second
// derivative along `op - 3`.  Same expression shapes as the residual's.
template <int OP>
__global__ void __launch_bounds__(256) k_derivative(const double* __restrict__ f,
                                                    double* __restrict__ out, Coef k, Geom g) {
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
  const GAcc a{f, c, g.s0, g.s1, 0};
  if constexpr (OP < 3) out[c] = d1<OP, E_FIELD, 0, 0>(k, a);
  else out[c] = d2<OP - 3, 0>(k, a);
}

// SS/RS interior fill as a 3-D grid of 32x8 point blocks (plane per
// blockIdx.z, sector-aligned columns): the nine velocity gradients
// ws[q*3+a] = D(u_q, x_a); the diagonal ghost frames follow in k_diag_ghost.
__global__ void __launch_bounds__(256) k_grad_ss_interior(const double* __restrict__ in,
                                                          double* __restrict__ ws, Coef k,
                                                          Geom g) {
  pdl_entry();
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
  const GAcc a{in, c, g.s0, g.s1, g.fs};
  ws[(0 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U0, 0>(k, a);
  ws[(0 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U0, 0>(k, a);
  ws[(0 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U0, 0>(k, a);
  ws[(1 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U1, 0>(k, a);
  ws[(1 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U1, 0>(k, a);
  ws[(1 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U1, 0>(k, a);
  ws[(2 * 3 + 0) * g.fs + c] = d1<0, E_FIELD, U2, 0>(k, a);
  ws[(2 * 3 + 1) * g.fs + c] = d1<1, E_FIELD, U2, 0>(k, a);
  ws[(2 * 3 + 2) * g.fs + c] = d1<2, E_FIELD, U2, 0>(k, a);
}

// The same fill, two axis-2 neighbours per thread through 16-byte accesses:
// a thread owns the padded columns (2t, 2t+1) of a 64-column block, so its
// pair is 16-byte aligned (even halo, even row pitch) and lies wholly inside
// or outside the interior.  Per velocity field the axis-2 taps of both points
// are three vector loads, the axis-1 and axis-0 taps four each: 33 loads + 9
// stores per pair instead of 72 + 18 -- the one-point kernel is bound by its
// load/store instruction queue (ncu: lg throttle 8.9, long scoreboard 27
// cycles per issue).  Same expressions per point (d1: stencil.py:80-84), so
// the bits are unchanged.
// Blocks past the interior planes (blockIdx.z >= n0) compute the diagonal
// arrays' ghost frames (k_diag_ghost semantics, f0 + f1 + f2 points; they
// read only the state): dispatched last, they fill the launch's tail
// instead of a separate, latency-bound 87 us kernel.
template <bool CS>
__global__ void __launch_bounds__(256) k_grad_ss_pair(const double* __restrict__ in,
                                                      double* __restrict__ ws, Coef k, Geom g,
                                                      int64_t f0, int64_t f1, int64_t f2) {
  pdl_entry();
  if ((int)blockIdx.z >= g.n0) {
    const int64_t blk = ((int64_t)(blockIdx.z - g.n0) * gridDim.y + blockIdx.y) * gridDim.x +
                        blockIdx.x;
    const int64_t t = blk * 256 + threadIdx.y * 32 + threadIdx.x;
    if (t < f0) diag_ghost_point<0>(in, ws + 0 * g.fs, k, g, t);
    else if (t < f0 + f1) diag_ghost_point<1>(in, ws + 4 * g.fs, k, g, t - f0);
    else if (t < f0 + f1 + f2) diag_ghost_point<2>(in, ws + 8 * g.fs, k, g, t - f0 - f1);
    return;
  }
  const int pk = (int)(blockIdx.x * 64 + 2 * threadIdx.x);   // padded column of the pair
  const int kk = pk - g.h;
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + pk;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double* u = in + (U0 + q) * g.fs + c;
    auto ld2 = [&](int64_t off) { return __ldg(reinterpret_cast<const double2*>(u + off)); };
    // axis 0 and axis 1: the pair's taps sit in the same 16 bytes
    double2 d[2];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const int64_t st = ax == 0 ? g.s0 : g.s1;
      const double2 p1 = ld2(st), m1 = ld2(-st), p2 = ld2(2 * st), m2 = ld2(-2 * st);
      d[ax].x = k.w1[ax] * (p1.x - m1.x) + k.w2[ax] * (p2.x - m2.x);
      d[ax].y = k.w1[ax] * (p1.y - m1.y) + k.w2[ax] * (p2.y - m2.y);
    }
    // axis 2: columns pk-2 .. pk+3
    const double2 a = ld2(-2), b = ld2(0), e = ld2(2);
    double2 d2v;
    d2v.x = k.w1[2] * (b.y - a.y) + k.w2[2] * (e.x - a.x);
    d2v.y = k.w1[2] * (e.x - b.x) + k.w2[2] * (e.y - a.y);
    double* w = ws + (q * 3) * g.fs + c;
    st_fill2<CS>(w, d[0]);
    st_fill2<CS>(w + g.fs, d[1]);
    st_fill2<CS>(w + 2 * g.fs, d2v);
  }
}
// whether k_grad_ss_pair applies: 16-byte aligned pairs that never straddle
// the interior's edge
inline bool ss_pair_ok(const Geom& g, const double* in, const double* ws) {
  return g.h == 2 && (g.n2 & 1) == 0 && (g.s1 & 1) == 0 && (g.s0 & 1) == 0 && (g.fs & 1) == 0 &&
         ((uintptr_t)in & 15) == 0 && ((uintptr_t)ws & 15) == 0;
}

// RK update on the interior of 5 fields (timeloop.py:80-85).
__global__ void k_rk_update(double* cons, const double* saved, const double* __restrict__ res,
                            double coef, Geom g) {
  const int kk = point_k(g);
  const int jj = blockIdx.y * blockDim.y + threadIdx.y;
  const int ii = blockIdx.z;
  if (kk < 0 || kk >= g.n2 || jj >= g.n1) return;
  const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
#pragma unroll
  for (int f = 0; f < 5; ++f) cons[f * g.fs + c] = saved[f * g.fs + c] + coef * res[f * g.fs + c];
}

// ---------------------------------------------------------------------------
// Diagnostics reduction (diagnostics.py:89-146, physics.py:121-129).
// Deterministic: fixed grid, fixed per-thread order, fixed tree.
// ---------------------------------------------------------------------------
constexpr int DIAG_Q = 9;
constexpr int DIAG_THREADS = 256;
constexpr int DIAG_BLOCKS = 148 * 4;

__global__ void __launch_bounds__(DIAG_THREADS) k_diag(const double* __restrict__ in,
                                                        const double* __restrict__ prim,
                                                        double* __restrict__ partials, Coef k,
                                                        Geom g) {
  double acc[DIAG_Q];
#pragma unroll
  for (int q = 0; q < DIAG_Q; ++q) acc[q] = 0.0;
  const int64_t npts = (int64_t)g.n0 * g.n1 * g.n2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npts;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int kk = t % g.n2;
    const int jj = (t / g.n2) % g.n1;
    const int ii = t / ((int64_t)g.n1 * g.n2);
    const int64_t c = (ii + g.h) * g.s0 + (jj + g.h) * g.s1 + (kk + g.h);
    GAcc a{in, c, g.s0, g.s1, g.fs};
    GAcc pa{prim, c, g.s0, g.s1, g.fs};   // velocities (may be another bundle)
    const double rho = a.v(RHO, 0, 0, 0);
    const double u0 = pa.v(U0, 0, 0, 0), u1 = pa.v(U1, 0, 0, 0), u2 = pa.v(U2, 0, 0, 0);
    acc[0] += 0.5 * rho * (u0 * u0 + u1 * u1 + u2 * u2);
    const double w0 = d1<1, E_FIELD, U2, 0>(k, pa) - d1<2, E_FIELD, U1, 0>(k, pa);
    const double w1 = d1<2, E_FIELD, U0, 0>(k, pa) - d1<0, E_FIELD, U2, 0>(k, pa);
    const double w2 = d1<0, E_FIELD, U1, 0>(k, pa) - d1<1, E_FIELD, U0, 0>(k, pa);
    acc[1] += 0.5 * rho * (w0 * w0 + w1 * w1 + w2 * w2);
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      const double v = a.v(f, 0, 0, 0);
      acc[2 + f] += v;
      if (!isfinite(v)) acc[7] += 1.0;
    }
    if (!(rho > 0.0)) acc[8] += 1.0;
  }
  __shared__ double sh[DIAG_Q][DIAG_THREADS];
#pragma unroll
  for (int q = 0; q < DIAG_Q; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = DIAG_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int q = 0; q < DIAG_Q; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < DIAG_Q) partials[blockIdx.x * DIAG_Q + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_diag_final(const double* __restrict__ partials, int nblocks, double* out) {
  __shared__ double sh[DIAG_Q][256];
  double acc[DIAG_Q];
  for (int q = 0; q < DIAG_Q; ++q) acc[q] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    for (int q = 0; q < DIAG_Q; ++q) acc[q] += partials[b * DIAG_Q + q];
  for (int q = 0; q < DIAG_Q; ++q) sh[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < DIAG_Q; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < DIAG_Q) out[threadIdx.x] = sh[threadIdx.x][0];
}

// FP64 issue-rate probe: 8 independent DADD chains per thread.
constexpr int PROBE_BLOCKS = 148 * 8, PROBE_THREADS = 256, PROBE_CHAINS = 8;
__global__ void __launch_bounds__(PROBE_THREADS) k_fp64_probe(double* out, int iters, double y) {
  double x[PROBE_CHAINS];
#pragma unroll
  for (int c = 0; c < PROBE_CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < PROBE_CHAINS; ++c) x[c] = x[c] + y;
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < PROBE_CHAINS; ++c) s += x[c];
  if (s == 123.456) out[0] = s;  // keep the chains live
}

__global__ void k_l2_flush(uint4* buf, int64_t n, uint32_t v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    buf[t] = make_uint4(v, v + 1, v + 2, v + 3);
}

// SM-driven copy between any two UVA addresses (device memory or pinned,
// mapped host memory): many 16-byte requests in flight from every SM.
__global__ void k_copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t];
}

inline dim3 point_grid(const Geom& g, dim3 blk) {
  const int ks = ksector_shift(g);
  return dim3((g.n2 + ks + blk.x - 1) / blk.x, (g.n1 + blk.y - 1) / blk.y, g.n0);
}

// ---------------------------------------------------------------------------
// TMA tensor map of a state bundle viewed as 4-D (k, j, i, field), box = one
// staged plane (TK+4, TJ+4, 1, 10).  Needs an even padded row (16-byte row
// pitch); otherwise the point kernels run.
// ---------------------------------------------------------------------------
// L2 sector promotion of every TMA box load: 64 B (round 2).  A box row is
// 36 or 32 doubles starting 16 B past a 32 B boundary (the padded row pitch
// is (n2 + 4) * 8 B), so 256 B promotion pulled up to 2.7x each row's bytes
// from DRAM: SN's stage reads 31.4 GB at 512^3 with 256 B, 28.4 with none,
// 25.5 with 64 B; whole steps SN +1.7%, SS +0.5%, RA equal
// (profiles/r02_l2_promotion_ab.txt).  A/B: FDNS_L2_PROMO = 0, 64, 128, 256.
inline CUtensorMapL2promotion l2_promotion() {
  static const int v = std::getenv("FDNS_L2_PROMO") ? std::atoi(std::getenv("FDNS_L2_PROMO")) : 64;
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// The three diagonal velocity gradients of an SS/RS work bundle (fields 0,
// 4, 8: D(u_q, x_q)) as a 4-D tensor with a field stride of 4 fields.
bool grad_map(CUtensorMap* m, const double* work, const Geom& g) {
  const int64_t P2 = g.n2 + 2 * g.h, P1 = g.n1 + 2 * g.h, P0 = g.n0 + 2 * g.h;
  if (P2 % 2 != 0 || g.h % 2 != 0) return false;
  if (reinterpret_cast<uintptr_t>(work) % 16 != 0) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)P1, (cuuint64_t)P0, 3};
  cuuint64_t strides[3] = {(cuuint64_t)(P2 * 8), (cuuint64_t)(P1 * P2 * 8),
                           (cuuint64_t)(4 * g.fs * 8)};
  cuuint32_t box[4] = {tiled::PK, tiled::PJ, 1, tiled::NGB};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(work), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The nine stored gradients of one plane's tile columns (TK x TJ x 1 x 9),
// the box the SS/RS stage kernel prefetches into L2.
bool grad_prefetch_map(CUtensorMap* m, const double* work, const Geom& g) {
  const int64_t P2 = g.n2 + 2 * g.h, P1 = g.n1 + 2 * g.h, P0 = g.n0 + 2 * g.h;
  if (P2 % 2 != 0 || g.h % 2 != 0) return false;
  if (reinterpret_cast<uintptr_t>(work) % 16 != 0) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)P1, (cuuint64_t)P0, 9};
  cuuint64_t strides[3] = {(cuuint64_t)(P2 * 8), (cuuint64_t)(P1 * P2 * 8),
                           (cuuint64_t)(g.fs * 8)};
  cuuint32_t box[4] = {tiled::TK, tiled::TJ, 1, 9};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(work), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool plane_map(CUtensorMap* m, const double* base, const Geom& g, int box_j = tiled::PJ) {
  const int64_t P2 = g.n2 + 2 * g.h, P1 = g.n1 + 2 * g.h, P0 = g.n0 + 2 * g.h;
  // 16-byte rows, and an even innermost box start (k0 + h - 2): an odd one
  // (odd h) is only 8-byte aligned and the bulk tensor copy faults on it
  if (P2 % 2 != 0 || g.h % 2 != 0) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)P1, (cuuint64_t)P0, (cuuint64_t)NFIELDS};
  cuuint64_t strides[3] = {(cuuint64_t)(P2 * 8), (cuuint64_t)(P1 * P2 * 8),
                           (cuuint64_t)(g.fs * 8)};
  cuuint32_t box[4] = {tiled::PK, (cuuint32_t)box_j, 1, tiled::NLOAD};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Saved-state tile of one plane (TK x TJ x 1 x 5 conservative fields), the
// box the stage kernel's L2 prefetch requests.
bool saved_map(CUtensorMap* m, const double* saved, const Geom& g, int box_j = tiled::TJ) {
  const int64_t P2 = g.n2 + 2 * g.h, P1 = g.n1 + 2 * g.h, P0 = g.n0 + 2 * g.h;
  if (P2 % 2 != 0 || g.h % 2 != 0) return false;
  if (reinterpret_cast<uintptr_t>(saved) % 16 != 0) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)P1, (cuuint64_t)P0, 5};
  cuuint64_t strides[3] = {(cuuint64_t)(P2 * 8), (cuuint64_t)(P1 * P2 * 8),
                           (cuuint64_t)(g.fs * 8)};
  cuuint32_t box[4] = {tiled::TK, (cuuint32_t)box_j, 1, 5};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(saved), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// General 4-D box map over `nf` fields of a padded bundle (field stride
// `fstride` elements), box (bk, bj, 1, bf).
bool box_map(CUtensorMap* m, const double* base, const Geom& g, int nf, int64_t fstride, int bk,
             int bj, int bf) {
  const int64_t P2 = g.n2 + 2 * g.h, P1 = g.n1 + 2 * g.h, P0 = g.n0 + 2 * g.h;
  if (P2 % 2 != 0 || g.h % 2 != 0) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)P2, (cuuint64_t)P1, (cuuint64_t)P0, (cuuint64_t)nf};
  cuuint64_t strides[3] = {(cuuint64_t)(P2 * 8), (cuuint64_t)(P1 * P2 * 8),
                           (cuuint64_t)(fstride * 8)};
  cuuint32_t box[4] = {(cuuint32_t)bk, (cuuint32_t)bj, 1, (cuuint32_t)bf};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Per-device state: a process may drive several GPUs (one per thread or
// in turn), so every cache below is keyed by the current device.
constexpr int MAX_DEVICES = 64;
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= MAX_DEVICES ? 0 : dev;
}
int num_sms() {
  static std::atomic<int> sms[MAX_DEVICES];
  const int dev = current_device();
  int n = sms[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
// Run `set` (a kernel's function attributes) once per device for the
// instantiation that owns `flags`.
template <class F>
void once_per_device(std::atomic<uint64_t>& flags, F set) {
  const uint64_t bit = 1ull << current_device();
  if (flags.load(std::memory_order_acquire) & bit) return;
  set();
  flags.fetch_or(bit, std::memory_order_acq_rel);
}

// Persistent grid: one CTA per SM with at least ~4 plane steps each, split
// contiguous, tile-aligned or balanced (Segments::partition).  Pick the split
// and CTA count minimising the longest CTA, in plane steps plus ~1.25 steps
// per extra segment (mid-range ramp; measured ~3.3 us vs ~3.0 us per step at
// 64^3), evaluated exactly over the CTAs of each candidate and cached.
// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor in the stream drains; it executes
// griddepcontrol.wait before any global memory access.
bool g_pdl = true;
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
// Cost model of a CTA's range: plane steps weighted by the tile's periodic
// image writes (edge tiles store each point's images too and finish later:
// measured +9% per step for a tile on a k edge, +8% on a j edge, at
// 256^3), plus the mid-range ramp of every extra segment.
// The image stores cost about the same time per point in every variant, so
// the relative weight shrinks with the variant's time per point (SS/RS
// ~1.05-1.1x SN).  For RA (1.45x) the weighted split measured no better
// than the uniform ones (-0.7% at 256^3 and 512^3), so RA keeps weight 1.
struct TileCost {
  int ntk, ntj;
  bool kw, jw;   // images written along axis 2 / axis 1
  double scale;  // SN = 1
  double weight(int64_t tile) const {
    const int kt = (int)(tile % ntk), jt = (int)(tile / ntk);
    return 1.0 + ((kw && (kt == 0 || kt == ntk - 1)) ? 0.09 * scale : 0.0) +
           ((jw && (jt == 0 || jt == ntj - 1)) ? 0.08 * scale : 0.0);
  }
};
#ifndef FDNS_EDGE_SCALE
#define FDNS_EDGE_SCALE 1.0
#endif
inline double edge_scale(int variant) {
  switch (variant & 0xff) {   // (launch keys carry the kernel family above bit 8)
    case FDNS_RA: return 0.0;
    case FDNS_SS: return FDNS_EDGE_SCALE / 1.05;
    case FDNS_RS: return FDNS_EDGE_SCALE / 1.1;
    default: return FDNS_EDGE_SCALE;
  }
}

double split_cost(int64_t G, const TileCost& tc, int planes, int mode,
                  const int64_t* cuts = nullptr) {
  const int64_t total = (int64_t)tc.ntk * tc.ntj * planes;
  const double Rm = tiled::RAMP_MID_Q / 4.0;
  double worst = 0;
  for (int64_t b = 0; b < G; ++b) {
    const tiled::Segments S = tiled::Segments::partition(b, G, total, planes, mode, cuts);
    if (S.beg >= S.end) continue;
    double c = -Rm;
    for (int64_t x = S.beg; x < S.end; x = S.seg_end(x))
      c += (double)(S.seg_end(x) - x) * tc.weight(x / planes) + Rm;
    worst = std::max(worst, c);
  }
  return worst;
}

// Cut points of G contiguous ranges in tile-major order minimising the
// largest range cost (plane steps times the tile's weight, plus a mid-range
// ramp for every tile a range enters after its first): binary search on
// that cost, each candidate checked by a greedy fill.  (Cutting at equal
// fractions of the total cost instead rounds each cut on its own and left
// some CTAs a whole step more than needed: 8 instead of 7 plane steps at
// 64^3, those CTAs ending ~3 us after the median.)
std::vector<int64_t> table_cuts(int64_t G, const TileCost& tc, int planes) {
  const int64_t tiles = (int64_t)tc.ntk * tc.ntj;
  const int64_t total = tiles * planes;
  const double Rm = tiled::RAMP_MID_Q / 4.0;
  // CTAs the greedy fill needs at max cost C (cut points into *cuts)
  auto fill = [&](double C, std::vector<int64_t>* cuts) -> int64_t {
    int64_t ctas = 1;
    double cur = 0;
    bool fresh = true;   // the current CTA has no segment yet
    if (cuts) cuts->assign(1, 0);
    for (int64_t t = 0; t < tiles; ++t) {
      const double wt = tc.weight(t);
      int64_t left = planes;
      while (left > 0) {
        const double extra = fresh ? 0.0 : Rm;
        int64_t fit = (int64_t)std::floor((C - cur - extra) / wt + 1e-9);
        if (fit <= 0 && fresh) fit = 1;   // C below one step: never stall
        if (fit <= 0) {
          ++ctas; cur = 0; fresh = true;
          if (cuts) cuts->push_back(t * planes + (planes - left));
          continue;
        }
        const int64_t take = std::min(fit, left);
        cur += extra + take * wt;
        fresh = false;
        left -= take;
        if (left > 0) {
          ++ctas; cur = 0; fresh = true;
          if (cuts) cuts->push_back(t * planes + (planes - left));
        }
      }
    }
    return ctas;
  };
  double wmax = 0, V = 0;
  for (int64_t t = 0; t < tiles; ++t) {
    wmax = std::max(wmax, tc.weight(t));
    V += planes * tc.weight(t);
  }
  double lo = std::max(V / (double)G, wmax), hi = lo + 2 * wmax + Rm;
  while (fill(hi, nullptr) > G) hi = 2 * hi;
  for (int it = 0; it < 60 && hi - lo > 1e-6; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (fill(mid, nullptr) <= G) hi = mid; else lo = mid;
  }
  std::vector<int64_t> cuts;
  fill(hi, &cuts);
  cuts.resize(G + 1, total);   // unused CTAs get empty ranges
  cuts[G] = total;
  for (int64_t b = 1; b <= G; ++b) cuts[b] = std::max(cuts[b], cuts[b - 1]);
  return cuts;
}

struct Launch { int64_t ctas; int aligned; const int64_t* cuts; };

// Round-robin units (tiled::SPLIT_ROUNDS): units of c planes of one tile,
// dealt chunk-major, so neighbouring tiles are staged at the same time and
// their shared halo columns and rows (state boxes, stored gradient boxes)
// can hit in L2.  Round 1 (SS/RS, 64-plane units): whole RK3 steps at 256^3
// SS +6.4%, RS +1.8%; at 128^3 the extra ramps cost more than the L2 hits
// win, so it is on from 256 planes.
// Round 2: free-running CTAs drift apart, so most of those halos still came
// from DRAM (ncu at 512^3: SS stage kernel 36.5 GB of reads for 23.6 GB of
// inputs).  With the CTAs held in lockstep (fdns_tiled.cuh:ls_step, K = 2
// steps of slack) the reads are 26.5 GB (1.12x) and SN's 15.2 GB (1.08x,
// 25.5 GB with the contiguous split); with the last, partial round cut into
// equal plane ranges (Segments::partition) no SM idles through it.  Whole
// RK3 steps at 512^3, interleaved A/B (profiles/r02_lockstep_ab.txt):
// SS +6%, RS +7%, SN +2-3% (128-plane units); RA -3% (FP64-bound and the
// least power-capped variant: it keeps the contiguous split).
// FDNS_ROUNDS=c overrides the unit (0 = off), FDNS_ROUNDS_ALL=1 adds RA,
// FDNS_LOCKSTEP=K sets the slack (0 = free running).
int g_rounds_env = std::getenv("FDNS_ROUNDS") ? std::atoi(std::getenv("FDNS_ROUNDS")) : -1;
int g_rounds_all = std::getenv("FDNS_ROUNDS_ALL") ? std::atoi(std::getenv("FDNS_ROUNDS_ALL")) : 0;
int g_lockstep = std::getenv("FDNS_LOCKSTEP") ? std::atoi(std::getenv("FDNS_LOCKSTEP")) : 2;
inline int rounds_planes(int variant, int nplanes) {
  const bool gb = variant == FDNS_SS || variant == FDNS_RS;
  if (!gb && variant != FDNS_SN && !(variant == FDNS_RA && g_rounds_all)) return 0;
  if (g_rounds_env >= 0) {
    const int c = g_rounds_env;
    return (c <= 0 || nplanes % c != 0 || nplanes < 2 * c) ? 0 : c;
  }
  // defaults: SS/RS from 256 planes, SN from 512; 128-plane units where
  // they divide the planes, else 64
  if (nplanes < (gb ? 256 : 512)) return 0;
  if (nplanes % 128 == 0) return 128;
  return nplanes % 64 == 0 ? 64 : 0;
}
// CTAs of a round-robin launch over `units` units
inline unsigned rounds_ctas(int64_t units) {
  const int64_t cap = g_tiled_ctas > 0 ? g_tiled_ctas : num_sms();
  return (unsigned)std::min<int64_t>(cap, units);
}

Launch pick_launch(int ntk, int ntj, int planes, int wrap, int variant, cudaStream_t s,
                   bool allow_table = true, int ctas_per_sm = 1) {
  const int64_t tiles = (int64_t)ntk * ntj;
  const int64_t total = tiles * planes;
  if (g_tiled_ctas > 0)
    return {std::min<int64_t>(g_tiled_ctas, total), tiled::SPLIT_ALIGNED, nullptr};
  const TileCost tc{ntk, ntj, (wrap & 4) != 0, (wrap & 2) != 0, edge_scale(variant)};
  using Key = std::tuple<int, int, int, int, int, int>;
  static std::map<Key, Launch> cache;
  static std::mutex mu;   // ctypes releases the GIL: calls may be concurrent
  std::lock_guard<std::mutex> lock(mu);
  // per device: the cut table is a device allocation of that GPU
  const Key key{ntk, ntj, planes, (wrap & 6) | (allow_table ? 8 : 0), variant,
                current_device()};
  const auto hit = cache.find(key);
  if (hit != cache.end()) return hit->second;
  const int64_t sms = (int64_t)num_sms() * ctas_per_sm;
  const int64_t G0 = std::max<int64_t>(1, std::min<int64_t>(sms, total / 4));
  Launch best{G0, tiled::SPLIT_CONTIGUOUS, nullptr};
  double best_cost = split_cost(G0, tc, planes, tiled::SPLIT_CONTIGUOUS);
  const double cb = split_cost(G0, tc, planes, tiled::SPLIT_BALANCED);
  if (cb < best_cost - 1e-9) { best_cost = cb; best = {G0, tiled::SPLIT_BALANCED, nullptr}; }
  // tile-aligned splits: one segment (one ramp) per CTA.  Small launches
  // (few planes, e.g. a slab's boundary planes) may use up to one CTA per
  // plane step: with G0 = total/4 their CTAs would each walk several short
  // segments, a ramp apiece (the boundary-first split cost +87% over one
  // launch at 64^3; tools/split_cost.py)
  const int64_t Gmax = std::max<int64_t>(G0, std::min<int64_t>(sms, total));
  for (int64_t G = tiles; G <= Gmax; ++G) {
    const double c = split_cost(G, tc, planes, tiled::SPLIT_ALIGNED);
    if (c < best_cost - 1e-9) { best_cost = c; best = {G, tiled::SPLIT_ALIGNED, nullptr}; }
  }
  // the edge-weighted table needs a device copy of the cuts: made once per
  // geometry, never while the stream is being captured into a graph
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusNone && allow_table) {
    const std::vector<int64_t> cuts = table_cuts(G0, tc, planes);
    const double ct = split_cost(G0, tc, planes, tiled::SPLIT_TABLE, cuts.data());
    if (ct < best_cost - 1e-9) {
      int64_t* d = nullptr;
      if (cudaMalloc(&d, cuts.size() * sizeof(int64_t)) == cudaSuccess &&
          cudaMemcpy(d, cuts.data(), cuts.size() * sizeof(int64_t), cudaMemcpyHostToDevice) ==
              cudaSuccess) {
        best_cost = ct;
        best = {G0, tiled::SPLIT_TABLE, d};
      } else {
        cudaGetLastError();
        if (d) cudaFree(d);
      }
    }
  }
  if (cs == cudaStreamCaptureStatusNone || !allow_table)
    cache[key] = best;   // (not cached while capturing: decided again later)
  return best;
}

// Kill switches of the L2 prefetches the producer thread issues (also A/B
// switches for experiments): FDNS_NO_SAVED_PREFETCH=1 disables the prefetch
// of the saved state, FDNS_NO_GRAD_PREFETCH=1 that of SS/RS's nine stored
// gradients (fdns_set_prefetch overrides both at run time).
bool g_prefetch_saved = std::getenv("FDNS_NO_SAVED_PREFETCH") == nullptr;
bool g_prefetch_grad = std::getenv("FDNS_NO_GRAD_PREFETCH") == nullptr;

template <int V, int MODE, bool LAZY = true>
int launch_tiled_v(const CUtensorMap& m, const double* in, const double* saved, double* out,
                   const double* work,
                   const Coef& k, const Geom& g, double coef, int wrap, int i_lo, int i_hi,
                   cudaStream_t s) {
  constexpr bool gb = (V == FDNS_SS || V == FDNS_RS);
  constexpr int smem = V == FDNS_SN ? tiled::SMEM_BYTES_SN
                                    : (gb ? tiled::SMEM_BYTES_SS : tiled::SMEM_BYTES);
  CUtensorMap mg = m, ms = m, mp = m;
  if constexpr (gb)
    if (!grad_map(&mg, work, g) || !grad_prefetch_map(&mp, work, g))
      return fail("gradient tensor map");
  // saved state != stage input (RK stages 2 and 3): prefetch it into L2
  int pf = 0;
  if constexpr (MODE == 1)
    pf = (g_prefetch_saved && saved != in && saved_map(&ms, saved, g)) ? tiled::PF_SAVED : 0;
  if constexpr (gb) pf |= g_prefetch_grad ? tiled::PF_GRAD : 0;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(tiled::k_stage_tiled<V, MODE, LAZY>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const int ntk = (g.n2 + tiled::TK - 1) / tiled::TK;
  const int ntj = (g.n1 + tiled::TJ - 1) / tiled::TJ;
  const int nplanes = i_hi - i_lo;
  const int64_t total = (int64_t)ntk * ntj * nplanes;
  if constexpr (V == FDNS_SS || V == FDNS_RS) {
    if (const int c = total < (1ll << 31) ? rounds_planes(V, nplanes) : 0) {
      pf |= (g_lockstep & 0xff) << 8;
      static std::atomic<uint64_t> attr_rr{0};
      once_per_device(attr_rr, [] {
        cudaFuncSetAttribute(tiled::k_stage_tiled<V, MODE, LAZY, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      });
      launch_pdl(tiled::k_stage_tiled<V, MODE, LAZY, true>,
                 dim3(rounds_ctas(total / c)), dim3(tiled::NT), smem,
                 s, m, mg, ms, mp, work, saved, out, k, g, coef, ntk, total, wrap, i_lo, c,
                 (int)tiled::SPLIT_ROUNDS, pf, (const int64_t*)nullptr);
      return 0;
    }
  }
  const Launch L = pick_launch(ntk, ntj, nplanes, wrap, V, s);
  launch_pdl(tiled::k_stage_tiled<V, MODE, LAZY>, dim3((unsigned)L.ctas), dim3(tiled::NT), smem, s,
             m, mg, ms, mp, work, saved, out, k, g, coef, ntk, total, wrap, i_lo, nplanes,
             L.aligned, pf, L.cuts);
  return 0;
}

// SN / RA kernel choice: the 12-warp kernel where its 12-row tiles waste few
// rows (measured whole RK3 steps, SN: +8% at 256^3, +5.5% at 128^3; at 64^3,
// where the last tile row holds 4 of 12 rows, -6%, so the 8-warp kernel
// stays; RA: +6.6% at 128^3, +3.9% at 256^3, +6.3% at 512^3).
inline bool use_t12(const Geom& g) {
  const int rows = (g.n1 + t12::TJ - 1) / t12::TJ * t12::TJ;
  return g.n1 >= 96 && 20 * (rows - g.n1) <= g.n1;
}

// SS / RS on the 12-warp kernel where the round-robin split applies and the
// planes are large (whole RK3 steps at 512^3: SS +1.8-2.6%, RS +0.2-1.7%;
// 256^3: SS equal, RS -3%); FDNS_SS_T12=0 keeps the 8-warp kernel (A/B).
const bool g_ss_t12 = !(std::getenv("FDNS_SS_T12") && std::atoi(std::getenv("FDNS_SS_T12")) == 0);
inline bool use_t12_ss(int variant, const Geom& g, int nplanes) {
  return g_ss_t12 && use_t12(g) && (int64_t)g.n1 * g.n2 >= 384 * 384 &&
         rounds_planes(variant, nplanes) > 0;
}

// The 12-warp stage kernel (fdns_tiled12.cuh): its own 36 x 16 plane box;
// SS/RS also the three stored-gradient boxes of the centre plane.
template <int MODE, int TJ_ = 12, int V = FDNS_SN>
int launch_t12(const double* in, const double* saved, double* out, const double* work,
               const Coef& k, const Geom& g, double coef, int wrap, int i_lo, int i_hi,
               cudaStream_t s) {
  using L = t12::Lay<TJ_>;
  constexpr bool gb = (V == FDNS_SS || V == FDNS_RS);
  CUtensorMap m, ms;
  if (!plane_map(&m, in, g, L::PJ)) return fail("plane tensor map");
  ms = m;
  t12::GradMaps gm;
  for (auto& t : gm.tg) t = m;
  if constexpr (gb) {
    if (!box_map(&gm.tg[0], work + 0 * g.fs, g, 1, g.fs, L::PK, L::PJ, 1) ||   // D(u0,x0)
        !box_map(&gm.tg[1], work + 4 * g.fs, g, 1, g.fs, L::PK, L::TJ, 1) ||   // D(u1,x1)
        !box_map(&gm.tg[2], work + 8 * g.fs, g, 1, g.fs, L::TK, L::PJ, 1) ||   // D(u2,x2)
        !box_map(&gm.tg[3], work, g, 9, g.fs, L::TK, L::TJ, 9))
      return fail("gradient tensor map");
  }
  int pf = 0;
  if constexpr (MODE == 1)
    pf = (g_prefetch_saved && saved != in && saved_map(&ms, saved, g, L::TJ)) ? tiled::PF_SAVED : 0;
  if constexpr (gb) pf |= g_prefetch_grad ? tiled::PF_GRAD : 0;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(t12::k_stage_t12<V, MODE, TJ_>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM_BYTES);
    if (L::MINB > 1)
      cudaFuncSetAttribute(t12::k_stage_t12<V, MODE, TJ_>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  });
  const int ntk = (g.n2 + L::TK - 1) / L::TK;
  const int ntj = (g.n1 + L::TJ - 1) / L::TJ;
  const int nplanes = i_hi - i_lo;
  const int64_t total = (int64_t)ntk * ntj * nplanes;
  {
    if (const int c = total < (1ll << 31) ? rounds_planes(V, nplanes) : 0) {   // round-robin units (SS/RS)
      pf |= (g_lockstep & 0xff) << 8;
      static std::atomic<uint64_t> attr_rr{0};
      once_per_device(attr_rr, [] {
        cudaFuncSetAttribute(t12::k_stage_t12<V, MODE, TJ_, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM_BYTES);
      });
      launch_pdl(t12::k_stage_t12<V, MODE, TJ_, true>,
                 dim3(rounds_ctas(total / c)), dim3(L::NT),
                 L::SMEM_BYTES, s, m, ms, gm, work, saved, out, k, g, coef, ntk, total, wrap,
                 i_lo, c, (int)tiled::SPLIT_ROUNDS, pf, (const int64_t*)nullptr);
      return 0;
    }
  }
  const Launch Lc = pick_launch(ntk, ntj, nplanes, wrap, V | 0x100 | (TJ_ << 12), s, true,
                                L::MINB);
  launch_pdl(t12::k_stage_t12<V, MODE, TJ_>, dim3((unsigned)Lc.ctas), dim3(L::NT),
             L::SMEM_BYTES, s, m, ms, gm, work, saved, out, k, g, coef, ntk, total, wrap, i_lo,
             nplanes, Lc.aligned, pf, Lc.cuts);
  return 0;
}

template <int MODE>
int launch_residual(int variant, const double* in, const double* saved, double* out,
                    double* work, const Coef& k, const Geom& g, double coef, int wrap,
                    int i_lo, int i_hi, cudaStream_t s) {
  if (i_hi <= i_lo) return 0;
  CUtensorMap m;
  if (variant != FDNS_BL && g_kernel_path != 1 && plane_map(&m, in, g)) {
    int rc = 0;
    switch (variant) {
      case FDNS_RA:
        if (g_kernel_path == 5 || (g_kernel_path == 0 && use_t12(g)))
          rc = launch_t12<MODE, 12, FDNS_RA>(in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        else rc = launch_tiled_v<FDNS_RA, MODE>(m, in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        break;
      case FDNS_RS:
        if (g_kernel_path == 5 || (g_kernel_path == 0 && use_t12_ss(FDNS_RS, g, i_hi - i_lo)))
          rc = launch_t12<MODE, 12, FDNS_RS>(in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        else rc = launch_tiled_v<FDNS_RS, MODE>(m, in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        break;
      case FDNS_SN:
        if (g_kernel_path == 5 || (g_kernel_path == 0 && use_t12(g)))
          rc = launch_t12<MODE>(in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        else if (g_kernel_path == 4)
          rc = launch_tiled_v<FDNS_SN, MODE, false>(m, in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        else rc = launch_tiled_v<FDNS_SN, MODE>(m, in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        break;
      case FDNS_SS:
        if (g_kernel_path == 5 || (g_kernel_path == 0 && use_t12_ss(FDNS_SS, g, i_hi - i_lo)))
          rc = launch_t12<MODE, 12, FDNS_SS>(in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        else rc = launch_tiled_v<FDNS_SS, MODE>(m, in, saved, out, work, k, g, coef, wrap, i_lo, i_hi, s);
        break;
      default: return fail("unknown variant");
    }
    if (rc) return rc;   // e.g. a tensor map that could not be encoded
    count();
    return check_launch("tiled stage kernel");
  }
  const dim3 blk(32, 8, 1);
  dim3 grd = point_grid(g, blk);
  grd.z = i_hi - i_lo;
  switch (variant) {
    case FDNS_BL: launch_pdl(k_residual<FDNS_BL, MODE>, grd, blk, 0, s, in, saved, out, work, k, g, coef, wrap, i_lo); break;
    case FDNS_RA: launch_pdl(k_residual<FDNS_RA, MODE>, grd, blk, 0, s, in, saved, out, work, k, g, coef, wrap, i_lo); break;
    case FDNS_RS: launch_pdl(k_residual<FDNS_RS, MODE>, grd, blk, 0, s, in, saved, out, work, k, g, coef, wrap, i_lo); break;
    case FDNS_SN: launch_pdl(k_residual<FDNS_SN, MODE>, grd, blk, 0, s, in, saved, out, work, k, g, coef, wrap, i_lo); break;
    case FDNS_SS: launch_pdl(k_residual<FDNS_SS, MODE>, grd, blk, 0, s, in, saved, out, work, k, g, coef, wrap, i_lo); break;
    default: return fail("unknown variant");
  }
  count();
  return check_launch("residual kernel");
}

// Planes per thread of the axis-0-marching fills; FDNS_MARCH_FILL=0 turns
// them off (A/B).
#ifndef FDNS_MARCH_NPL
#define FDNS_MARCH_NPL 32
#endif
constexpr int MARCH_NPL = FDNS_MARCH_NPL;
// BL fill: 0 = point kernel, 1 = register-queue march, 2 = shared-memory
// queue march, 3 = axis-0 march + in-plane point kernel; -1 (default) = 2
// on large planes, else 0.  Whole BL RK3 steps (tools/step_timing.py,
// profiles/r02_bl_fill_ab.txt): 512^3 point 109.2 ms, 1: 102.6, 2: 100.6,
// 3: 102.4; 256^3 point 12.8 ms, 2: 13.1.  The write-dominated fill runs
// at ~4.2-4.8 TB/s whichever way (HBM read/write turnaround: the read-heavy
// BL residual streams 6.4 TB/s); the marching fills cut its reads from 55
// to 15 GB per launch at 512^3.
const int g_march_fill = std::getenv("FDNS_MARCH_FILL") ? std::atoi(std::getenv("FDNS_MARCH_FILL")) : -1;
inline int march_fill_mode(const Geom& g) {
  if (g_march_fill >= 0) return g_march_fill;
  return (int64_t)g.n1 * g.n2 >= 384 * 384 ? 2 : 0;
}
// A/B switch: FDNS_SS_FILL_1D=1 selects the one-launch grid-stride SS fill.
const bool g_ss_fill_3d = std::getenv("FDNS_SS_FILL_1D") == nullptr;
// FDNS_SS_FILL_PAIR=0: the one-point-per-thread interior fill (A/B)
const bool g_ss_fill_pair =
    !(std::getenv("FDNS_SS_FILL_PAIR") && std::atoi(std::getenv("FDNS_SS_FILL_PAIR")) == 0);

// Work-array fills that precede the residual kernel (BL, RS, SS).
int launch_fills(int variant, const double* in, double* work, const Coef& k, const Geom& g,
                 cudaStream_t s) {
  const dim3 blk(32, 8, 1);
  const dim3 grd = point_grid(g, blk);
  // programmatic dependent launch for the fills: BL's chain and the one-
  // launch SS/RS fill (+1.4-1.8% BL/SS/RS steps at 64^3); the 3-D SS/RS
  // fill path keeps plain launches (with PDL its steps were 5-8% slower at
  // 128^3-256^3)
  auto ghosts = [&](double* d0, double* d1p, double* d2p, bool pdl) {
    const int h = g.h;
    const int64_t f0 = (int64_t)g.n0 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n1 * 2 * h);
    const int64_t f1 = (int64_t)g.n1 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n0 * 2 * h);
    const int64_t f2 = (int64_t)g.n2 * (2 * h * (g.n1 + 2 * h) + (int64_t)g.n0 * 2 * h);
    const int nb = (int)std::min<int64_t>((f0 + f1 + f2 + 255) / 256, 148 * 8);
    if (pdl) launch_pdl(k_diag_ghost, dim3(nb), dim3(256), 0, s, in, d0, d1p, d2p, k, g, f0, f1, f2);
    else k_diag_ghost<<<nb, 256, 0, s>>>(in, d0, d1p, d2p, k, g, f0, f1, f2);
  };
  // axis-0-marching fills (FDNS_MARCH_FILL=0 restores the point fills)
  const dim3 mblk(MARCH_BX, MARCH_BY, 1);
  auto march_grid = [&](int npl) {
    dim3 m = point_grid(g, mblk);
    m.z = (g.n0 + npl - 1) / npl;
    return m;
  };
  if (variant == FDNS_BL) {
    const int mode = march_fill_mode(g);
    if (mode == 2 && g.n0 >= 2 * MARCH_NPL) {
      static std::atomic<uint64_t> attr{0};
      once_per_device(attr, [] {
        cudaFuncSetAttribute(k_fill_bl_march_s<MARCH_NPL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, MARCH_SMEM);
      });
      launch_pdl(k_fill_bl_march_s<MARCH_NPL>, march_grid(MARCH_NPL), mblk, MARCH_SMEM, s, in,
                 work, k, g);
    } else if (mode == 3 && g.n0 >= 2 * MARCH_NPL) {
      // axis 0 by the marching kernel, axes 1-2 by the point kernel
      launch_pdl(k_fill_bl_march<MARCH_NPL, 1>, march_grid(MARCH_NPL), mblk, 0, s, in, work, k, g);
      launch_pdl(k_fill_bl_all<6>, grd, blk, 0, s, in, work, k, g);
      count();
    } else if (mode == 1 && g.n0 >= 2 * MARCH_NPL)
      launch_pdl(k_fill_bl_march<MARCH_NPL>, march_grid(MARCH_NPL), mblk, 0, s, in, work, k, g);
    else
      launch_pdl(k_fill_bl_all<7>, grd, blk, 0, s, in, work, k, g);
    ghosts(work + slot(0, S_U + 0) * g.fs, work + slot(1, S_U + 1) * g.fs,
           work + slot(2, S_U + 2) * g.fs, true);
    if (g_ss_fill_pair && ss_pair_ok(g, in, work))
      launch_pdl(fill_cs(g) ? k_fill_cross_pair<true> : k_fill_cross_pair<false>,
                 dim3((unsigned)((g.n2 + 2 * g.h + 63) / 64), grd.y, grd.z), blk, 0, s, work, k, g);
    else
      launch_pdl(k_fill_cross, grd, blk, 0, s, work, k, g);
    count(3);
    return check_launch("BL fills");
  }
  // SS/RS fill: from n2 >= 128 on the 3-D point-block kernel + the ghost
  // frames (+6% SS/RS steps at 256^3); below, one grid-stride launch
  // (its single launch wins at 64^3: -4% otherwise)
  if ((variant == FDNS_SS || variant == FDNS_RS) && g_ss_fill_3d && g.n2 >= 128) {
    if (g_ss_fill_pair && ss_pair_ok(g, in, work)) {
      // interior planes + the z layers of blocks that cover the ghost frames
      const int h = g.h;
      const int64_t f0 = (int64_t)g.n0 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n1 * 2 * h);
      const int64_t f1 = (int64_t)g.n1 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n0 * 2 * h);
      const int64_t f2 = (int64_t)g.n2 * (2 * h * (g.n1 + 2 * h) + (int64_t)g.n0 * 2 * h);
      dim3 pgrd((unsigned)((g.n2 + 2 * g.h + 63) / 64), grd.y, grd.z);
      const int64_t per_layer = (int64_t)256 * pgrd.x * pgrd.y;
      pgrd.z += (unsigned)((f0 + f1 + f2 + per_layer - 1) / per_layer);
      if (fill_cs(g)) k_grad_ss_pair<true><<<pgrd, blk, 0, s>>>(in, work, k, g, f0, f1, f2);
      else k_grad_ss_pair<false><<<pgrd, blk, 0, s>>>(in, work, k, g, f0, f1, f2);
      count(1);
    } else {
      k_grad_ss_interior<<<grd, blk, 0, s>>>(in, work, k, g);
      ghosts(work + 0 * g.fs, work + 4 * g.fs, work + 8 * g.fs, false);
      count(2);
    }
    return check_launch("SS fills");
  }
  if (variant == FDNS_SS || variant == FDNS_RS) {
    {   // 9 gradients on the interior + the diagonal ghost frames, one launch
      const int h = g.h;
      const int64_t nint = (int64_t)g.n0 * g.n1 * g.n2;
      const int64_t f0 = (int64_t)g.n0 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n1 * 2 * h);
      const int64_t f1 = (int64_t)g.n1 * (2 * h * (g.n2 + 2 * h) + (int64_t)g.n0 * 2 * h);
      const int64_t f2 = (int64_t)g.n2 * (2 * h * (g.n1 + 2 * h) + (int64_t)g.n0 * 2 * h);
      const int nb = (int)std::min<int64_t>((nint + f0 + f1 + f2 + 255) / 256, 148 * 16);
      launch_pdl(k_grad_ss_all, dim3(nb), dim3(256), 0, s, in, work, k, g, nint, f0, f1, f2);
    }
    count(1);
    return check_launch("SS fills");
  }
  return 0;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* fdns_last_error(void) { return g_err.c_str(); }

int32_t fdns_abi_version(void) { return 1; }

int64_t fdns_launch_count(void) { return g_launches.load(); }

void fdns_set_kernel_path(int32_t path) { g_kernel_path = path; }

void fdns_set_tiled_grid(int32_t ctas) { g_tiled_ctas = ctas; }

void fdns_set_pdl(int32_t enabled) { g_pdl = enabled != 0; }

void fdns_set_rounds(int32_t planes) { g_rounds_env = planes; }

void fdns_set_lockstep(int32_t slack) { g_lockstep = slack < 0 ? 2 : std::min(slack, 255); }

void fdns_set_prefetch(int32_t mask) {
  g_prefetch_saved = (mask & 1) != 0;
  g_prefetch_grad = (mask & 2) != 0;
}

int32_t fdns_debug_rounds_walk(int64_t tiles, int32_t planes, int32_t unit, int32_t ctas,
                               int32_t* cover, int32_t* steps, int32_t* segs) {
  if (tiles <= 0 || planes <= 0 || unit <= 0 || planes % unit != 0 || ctas <= 0 || !cover)
    return -1;
  const int64_t total = tiles * planes;
  if (total >= (1ll << 31)) return -1;
  const int64_t G = std::min<int64_t>(ctas, total / unit);
  for (int64_t b = 0; b < G; ++b) {
    tiled::Segments S = tiled::Segments::partition(b, G, total, unit, tiled::SPLIT_ROUNDS);
    S.tiles = tiles;
    int32_t nst = 0, nsg = 0;
    for (int64_t x = S.beg; x < S.end; x = S.next_rr(x, S.main_end, S.tbeg, S.tend)) {
      const int64_t e = S.seg_end_rr(x, S.main_end, S.tend);
      if (e <= x) return -1;   // a walk that does not advance
      const int64_t tile = S.tile_of(x);
      for (int64_t y = x; y < e; ++y) ++cover[tile * planes + S.plane_of(x) + (y - x)];
      nst += (int32_t)(e - x);
      ++nsg;
    }
    if (steps) steps[b] = nst;
    if (segs) segs[b] = nsg;
  }
  return (int32_t)G;
}

int32_t fdns_debug_trace(int32_t enable, uint64_t* out, int32_t n) {
  int on = enable;
  if (cudaMemcpyToSymbol(tiled::g_trace_on, &on, sizeof(int)) != cudaSuccess)
    return fail("trace flag", cudaGetLastError());
  if (enable == 2) {   // log mode: start a fresh launch log
    unsigned zero = 0;
    if (cudaMemcpyToSymbol(tiled::g_trace_n, &zero, sizeof(zero)) != cudaSuccess)
      return fail("trace log reset", cudaGetLastError());
  }
  if (out && n > 0 && enable == 3) {   // read the launch log: [count, records...]
    unsigned cnt = 0;
    if (cudaMemcpyFromSymbol(&cnt, tiled::g_trace_n, sizeof(cnt)) != cudaSuccess)
      return fail("trace log count", cudaGetLastError());
    cnt = std::min<unsigned>(cnt, tiled::TRACE_LOG_N);
    out[0] = cnt;
    const int m = std::min<int64_t>(n - 1, (int64_t)cnt * tiled::TRACE_LOG_W);
    if (m > 0 && cudaMemcpyFromSymbol(out + 1, tiled::g_trace_log, m * sizeof(uint64_t)) !=
                     cudaSuccess)
      return fail("trace log copy", cudaGetLastError());
    on = 0;
    cudaMemcpyToSymbol(tiled::g_trace_on, &on, sizeof(int));
    return 0;
  }
  if (out && n > 0) {
    const int m = std::min(n, tiled::TRACE_CTAS * tiled::TRACE_PTS);
    if (cudaMemcpyFromSymbol(out, tiled::g_trace, m * sizeof(uint64_t)) != cudaSuccess)
      return fail("trace copy", cudaGetLastError());
  }
  return 0;
}

int32_t fdns_workarray_count(int32_t variant) {
  switch (variant) {
    case FDNS_BL: return N_SLOTS;
    case FDNS_RS:
    case FDNS_SS: return 9;
    case FDNS_RA:
    case FDNS_SN: return 0;
    default: return -1;
  }
}

int32_t fdns_primitives(double* state, const fdns_problem* pb, void* stream) {
  if (int e = validate(pb)) return e;
  const Geom g = make_geom(pb);
  const Coef k = make_coef(pb);
  const int blocks = (int)std::min<int64_t>((g.fs + 255) / 256, 148 * 16);
  k_primitives<<<blocks, 256, 0, (cudaStream_t)stream>>>(state, k, g.fs, 0, g.fs);
  count();
  return check_launch("primitives kernel");
}

int32_t fdns_primitives_planes(double* state, int32_t p_lo, int32_t p_hi, const fdns_problem* pb,
                               void* stream) {
  if (int e = validate(pb)) return e;
  const Geom g = make_geom(pb);
  if (p_lo < 0 || p_hi > g.n0 + 2 * g.h || p_lo > p_hi)
    return fail("fdns_primitives_planes: plane range outside the padded bundle");
  if (p_lo == p_hi) return 0;
  const Coef k = make_coef(pb);
  const int64_t c0 = p_lo * g.s0, c1 = p_hi * g.s0;
  const int blocks = (int)std::min<int64_t>((c1 - c0 + 255) / 256, 148 * 16);
  k_primitives<<<blocks, 256, 0, (cudaStream_t)stream>>>(state, k, g.fs, c0, c1);
  count();
  return check_launch("primitives kernel");
}

int32_t fdns_derivative(const double* f, double* out, int32_t op, const fdns_problem* pb,
                        void* stream) {
  if (int e = validate(pb)) return e;
  if (op < 0 || op > 5) return fail("fdns_derivative: op must be 0-2 (first) or 3-5 (second)");
  if (f == out) return fail("fdns_derivative: output must not alias the input");
  const Geom g = make_geom(pb);
  const Coef k = make_coef(pb);
  const dim3 blk(32, 8, 1);
  const dim3 grd = point_grid(g, blk);
  cudaStream_t s = (cudaStream_t)stream;
  switch (op) {
    case 0: k_derivative<0><<<grd, blk, 0, s>>>(f, out, k, g); break;
    case 1: k_derivative<1><<<grd, blk, 0, s>>>(f, out, k, g); break;
    case 2: k_derivative<2><<<grd, blk, 0, s>>>(f, out, k, g); break;
    case 3: k_derivative<3><<<grd, blk, 0, s>>>(f, out, k, g); break;
    case 4: k_derivative<4><<<grd, blk, 0, s>>>(f, out, k, g); break;
    default: k_derivative<5><<<grd, blk, 0, s>>>(f, out, k, g); break;
  }
  count();
  return check_launch("derivative kernel");
}

int32_t fdns_halo_wrap(double* fields, int32_t nf, int32_t axes_mask, const fdns_problem* pb,
                       void* stream) {
  if (int e = validate(pb)) return e;
  const Geom g = make_geom(pb);
  const int h = g.h;
  const int64_t P0 = g.n0 + 2 * h, P1 = g.n1 + 2 * h, P2 = g.n2 + 2 * h;
  const bool m0 = axes_mask & 1, m1 = axes_mask & 2, m2 = axes_mask & 4;
  if (m0 && g.n0 < h) return fail("axis 0 needs at least h points to wrap");
  const int64_t r0 = m0 ? 2 * h * P1 * P2 : 0;
  const int64_t r1 = m1 ? (m0 ? g.n0 : P0) * 2 * h * P2 : 0;
  const int64_t r2 = m2 ? (m0 ? g.n0 : P0) * (m1 ? g.n1 : P1) * 2 * h : 0;
  const int64_t total = r0 + r1 + r2;
  if (total == 0 || nf == 0) return 0;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_halo_wrap<<<blocks, 256, 0, (cudaStream_t)stream>>>(fields, nf, axes_mask, g, r0, r1, r2);
  count();
  return check_launch("halo wrap kernel");
}

int32_t fdns_residual(int32_t variant, const double* state, double* work, double* out,
                      const fdns_problem* pb, void* stream) {
  if (int e = validate(pb)) return e;
  const int nw = fdns_workarray_count(variant);
  if (nw < 0) return fail("unknown variant");
  if (nw > 0 && !work) return fail("variant needs work arrays");
  const Geom g = make_geom(pb);
  if (overlaps(out, 5, state, NFIELDS, g) || (nw > 0 && (overlaps(work, nw, state, NFIELDS, g) ||
                                                         overlaps(work, nw, out, 5, g))))
    return fail("fdns_residual: out, state and work must not overlap");
  const Coef k = make_coef(pb);
  cudaStream_t s = (cudaStream_t)stream;
  if (int e = launch_fills(variant, state, work, k, g, s)) return e;
  return launch_residual<0>(variant, state, nullptr, out, work, k, g, 0.0, 0, 0, g.n0, s);
}

int32_t fdns_rk_update(double* cons, const double* saved, const double* res, double coef,
                       const fdns_problem* pb, void* stream) {
  if (int e = validate(pb)) return e;
  const Geom g = make_geom(pb);
  const dim3 blk(32, 8, 1);
  k_rk_update<<<point_grid(g, blk), blk, 0, (cudaStream_t)stream>>>(cons, saved, res, coef, g);
  count();
  return check_launch("rk update kernel");
}

int32_t fdns_stage_planes(int32_t variant, const double* in, const double* saved, double* out,
                          double* work, double coef, int32_t wrap_mask, int32_t i_lo,
                          int32_t i_hi, int32_t with_fills, const fdns_problem* pb,
                          void* stream) {
  if (int e = validate(pb)) return e;
  const int nw = fdns_workarray_count(variant);
  if (nw < 0) return fail("unknown variant");
  if (nw > 0 && !work) return fail("variant needs work arrays");
  if (in == out) return fail("fused stage needs distinct in/out bundles");
  {
    const Geom gg = make_geom(pb);
    if (overlaps(out, NFIELDS, in, NFIELDS, gg) ||
        (nw > 0 && (overlaps(work, nw, in, NFIELDS, gg) || overlaps(work, nw, out, NFIELDS, gg) ||
                    overlaps(work, nw, saved, 5, gg))))
      return fail("fused stage: in, out and work must not overlap (saved may alias out)");
  }
  if (i_lo < 0 || i_hi > pb->n[0] || i_lo > i_hi) return fail("plane range outside the slab");
  const Geom g = make_geom(pb);
  const Coef k = make_coef(pb);
  cudaStream_t s = (cudaStream_t)stream;
  if (with_fills)
    if (int e = launch_fills(variant, in, work, k, g, s)) return e;
  return launch_residual<1>(variant, in, saved, out, work, k, g, coef, wrap_mask, i_lo, i_hi, s);
}

int32_t fdns_stage(int32_t variant, const double* in, const double* saved, double* out,
                   double* work, double coef, int32_t wrap_mask, const fdns_problem* pb,
                   void* stream) {
  if (int e = validate(pb)) return e;
  return fdns_stage_planes(variant, in, saved, out, work, coef, wrap_mask, 0, pb->n[0], 1, pb,
                           stream);
}

int32_t fdns_diag_partials_size(const fdns_problem*) { return DIAG_BLOCKS * DIAG_Q; }

int32_t fdns_reduce_diag(const double* state, const double* prim_state, double* partials,
                         double* out9, const fdns_problem* pb, void* stream) {
  if (int e = validate(pb)) return e;
  const Geom g = make_geom(pb);
  const Coef k = make_coef(pb);
  cudaStream_t s = (cudaStream_t)stream;
  k_diag<<<DIAG_BLOCKS, DIAG_THREADS, 0, s>>>(state, prim_state ? prim_state : state, partials, k, g);
  k_diag_final<<<1, 256, 0, s>>>(partials, DIAG_BLOCKS, out9);
  count(2);
  return check_launch("diagnostics kernels");
}

int32_t fdns_fp64_probe(double* scratch, int32_t iters, double* out_count, void* stream) {
  k_fp64_probe<<<PROBE_BLOCKS, PROBE_THREADS, 0, (cudaStream_t)stream>>>(scratch, iters, 1e-9);
  if (out_count)
    *out_count = (double)PROBE_BLOCKS * PROBE_THREADS * (double)iters * PROBE_CHAINS;
  return check_launch("fp64 probe");
}

int32_t fdns_l2_flush(void* buf, int64_t bytes, void* stream) {
  const int64_t n = bytes / 16;
  static uint32_t v = 1;
  k_l2_flush<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((uint4*)buf, n, v++);
  return check_launch("l2 flush");
}

int32_t fdns_copy_rows(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                       int64_t row_bytes, int64_t rows, void* stream) {
  if (rows <= 0 || row_bytes <= 0) return 0;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch,
                                          (size_t)row_bytes, (size_t)rows, cudaMemcpyDefault,
                                          (cudaStream_t)stream);
  if (e != cudaSuccess) return fail("fdns_copy_rows", e);
  return 0;
}

int32_t fdns_copy_sm(void* dst, const void* src, int64_t bytes, int32_t ctas, void* stream) {
  if (((uintptr_t)dst | (uintptr_t)src | (uintptr_t)bytes) & 15)
    return fail("fdns_copy_sm: pointers and size must be 16-byte aligned");
  if (bytes <= 0) return 0;
  const int64_t n = bytes / 16;
  const int grid = ctas > 0 ? ctas : 148 * 4;
  k_copy16<<<grid, 256, 0, (cudaStream_t)stream>>>((uint4*)dst, (const uint4*)src, n);
  count();
  return check_launch("sm copy");
}

}  // extern "C"
