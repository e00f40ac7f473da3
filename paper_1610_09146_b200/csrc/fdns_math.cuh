// fdns_math.cuh -- per-point arithmetic of the 4th-order compressible
// Navier-Stokes residual, shared by every variant kernel.
//
// The arithmetic contract is the reference term list
// (pkg/src/fdns/terms.py:135-200) with the stencil shapes of
// pkg/src/fdns/stencil.py:71-102 / codegen.py:81-102.  Every expression below
// keeps the reference's left-to-right association, and the library is built
// with -fmad=false and IEEE division, so each variant reproduces the
// reference bits exactly (parity gate: tests/test_gpu_parity.py).
//
// The derivative *provider* decides where a derivative value comes from,
// which is exactly what distinguishes the paper's variants:
//   LocalProvider   (SN)  every distinct derivative evaluated once, kept live
//                         (point kernels; the tiled kernels use the lazily
//                         evaluated TiledLazyProvider, fdns_tiled.cuh)
//   InlineProvider  (RA)  re-expanded from the stencil at every occurrence
//   FetchProvider   (BL)  read from a stored work array
//   SSProvider      (SS)  9 velocity gradients stored, the rest local
//                   (RS)  the same with the rest re-expanded (INLINE)
// The residual body (residual_point) is written once over the provider API.
#pragma once
#include <cstdint>

namespace fdns {

enum Fld : int { RHO = 0, RU0, RU1, RU2, RHOE_F, U0, U1, U2, PF, TF, NFIELDS };

// Stencil weights per axis, pre-divided by the spacing (stencil.py:45-51),
// plus the five kernel constants (physics.py:78-81) and gm1/gM2.
struct Coef {
  double w1[3], w2[3], s0[3], s1[3], s2[3];
  double inv_Re, c13, c43, c23, heat;
  double gm1, gM2;
};

// Geometry of one padded bundle: field stride fs and axis strides.
struct Geom {
  int n0, n1, n2, h;   // interior points per axis (n0 = local slab planes)
  int64_t s0, s1, fs;  // strides (elements) of axis 0, axis 1, field
};

// ---------------------------------------------------------------------------
// Point accessors: value of field f at the centre point shifted by (di,dj,dk)
// ---------------------------------------------------------------------------

// Global-memory accessor through the read-only path.  Loads may be merged by
// the compiler (used by LOCAL/FETCH providers).
struct GAcc {
  static constexpr bool kInternalEnergy = false;
  static constexpr bool kMaskTaps = false;   // INLINE occurrences rebase (L1 hits)
  const double* __restrict__ b;
  int64_t c, s0, s1, fs;
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    return __ldg(b + f * fs + c + di * s0 + dj * s1 + dk);
  }
  __device__ __forceinline__ GAcc rebased(int z) const { return GAcc{b, c + z, s0, s1, fs}; }
};

// Occurrence-distinct zero offsets (RA semantics, plan.py:172-173).  The
// INLINE provider rebases every derivative occurrence's tap addresses by
// g_zero_offset[occurrence]: all entries are 0 at run time, but the compiler
// cannot prove two entries equal, so it can merge neither the loads nor the
// arithmetic built on them -- each occurrence is genuinely recomputed, as
// in the reference's generated RA kernel.  Integer offsets keep the bits
// exact (a floating-point +0.0 would not: it flips -0.0).
constexpr int N_ZERO_OFFSETS = 4096;
__constant__ int g_zero_offset[N_ZERO_OFFSETS];

template <int OCC>
__device__ __forceinline__ int zero_offset() {
  return g_zero_offset[OCC % N_ZERO_OFFSETS];
}

// Register-level variant (shared-memory accessors with FDNS_RA_OPAQUE=1, the
// default; global-memory point kernels keep the rebased addresses, which
// measured faster there -- the shared loads spill): taps are loaded
// once (the compiler may share loads between occurrences), and each
// occurrence XORs the high word of selected taps with its own
// constant-bank zero.  The result is bit-identical to the tap, yet opaque to the
// compiler, so every occurrence's arithmetic is still recomputed -- at the
// cost of about one integer instruction per tap instead of one
// shared-memory load.
#ifndef FDNS_RA_OPAQUE
#define FDNS_RA_OPAQUE 1
#endif
__constant__ int g_zero_word[N_ZERO_OFFSETS];

template <int OCC>
__device__ __forceinline__ double opaque(double x) {
  return __hiloint2double(__double2hiint(x) ^ g_zero_word[OCC % N_ZERO_OFFSETS],
                          __double2loint(x));
}

// Accessor of one INLINE occurrence: `v` reads a tap plainly, `m` reads it
// masked.  The stencils mask one operand of every first-level operation
// (ep1, ep2 of a first derivative; the centre, +1, +2 taps of a second
// derivative; the first factor of every product and of rho*e), which
// already makes every value of the occurrence distinct to the compiler.
template <class Acc, int OCC>
struct OpaqueAcc {
  static constexpr bool kInternalEnergy = Acc::kInternalEnergy;
  const Acc& a;
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    return a.v(f, di, dj, dk);
  }
  __device__ __forceinline__ double m(int f, int di, int dj, int dk) const {
    return opaque<OCC>(a.v(f, di, dj, dk));
  }
};

template <class A> struct is_opaque { static constexpr bool value = false; };
template <class A, int O> struct is_opaque<OpaqueAcc<A, O>> { static constexpr bool value = true; };

// A tap read, masked when M and the accessor is an occurrence view.
template <bool M, class A>
__device__ __forceinline__ double tap(const A& a, int f, int di, int dj, int dk) {
  if constexpr (M && is_opaque<A>::value) return a.m(f, di, dj, dk);
  else return a.v(f, di, dj, dk);
}

// The accessor one INLINE occurrence evaluates through.
template <int OCC, class Acc>
__device__ __forceinline__ auto occurrence_view(const Acc& a) {
  if constexpr (FDNS_RA_OPAQUE && Acc::kMaskTaps) return OpaqueAcc<Acc, OCC>{a};
  else return a.rebased(zero_offset<OCC>());
}

// ---------------------------------------------------------------------------
// Point expressions of the term list (terms.py:39, :158-174)
// ---------------------------------------------------------------------------
template <int AX> struct Off {
  static __device__ __forceinline__ void at(int o, int& di, int& dj, int& dk) {
    di = AX == 0 ? o : 0; dj = AX == 1 ? o : 0; dk = AX == 2 ? o : 0;
  }
};

// Internal energy rho*e at a point (terms.py:39).  Accessors over staged
// tiles hold it precomputed in place of rhoE (kInternalEnergy): the same
// per-point expression, evaluated once per staged point instead of once per
// stencil tap, so the bits are identical.
template <bool M = false, class A>
__device__ __forceinline__ double rhoe_at(const A& a, int di, int dj, int dk) {
  if constexpr (A::kInternalEnergy) {
    return tap<M>(a, RHOE_F, di, dj, dk);
  } else {   // arithmetic: every product masked, so no occurrence shares
             // any part of it
    return a.v(RHOE_F, di, dj, dk) -
           0.5 * (tap<true>(a, RU0, di, dj, dk) * a.v(U0, di, dj, dk) +
                  tap<true>(a, RU1, di, dj, dk) * a.v(U1, di, dj, dk) +
                  tap<true>(a, RU2, di, dj, dk) * a.v(U2, di, dj, dk));
  }
}

// Expression kinds differentiated by the stencils.
enum Ex : int { E_FIELD = 0, E_PROD, E_RHOE, E_RHOEU };

template <int EX, int F, int G, bool M = false, class A>
__device__ __forceinline__ double ex_at(const A& a, int di, int dj, int dk) {
  if constexpr (EX == E_FIELD) return tap<M>(a, F, di, dj, dk);
  else if constexpr (EX == E_PROD) return tap<true>(a, F, di, dj, dk) * a.v(G, di, dj, dk);
  else if constexpr (EX == E_RHOE) return rhoe_at<M>(a, di, dj, dk);
  else return rhoe_at<true>(a, di, dj, dk) * a.v(G, di, dj, dk);
}

// First derivative along AX of expression EX at centre+(bi,bj,bk):
//   fw1*((e(+1)) - (e(-1))) + fw2*((e(+2)) - (e(-2)))   (stencil.py:80-84)
template <int AX, int EX, int F, int G, class A>
__device__ __forceinline__ double d1(const Coef& k, const A& a, int bi = 0,
                                     int bj = 0, int bk = 0) {
  int i1, j1, k1;
  Off<AX>::at(1, i1, j1, k1);
  const double ep1 = ex_at<EX, F, G, true>(a, bi + i1, bj + j1, bk + k1);
  const double em1 = ex_at<EX, F, G>(a, bi - i1, bj - j1, bk - k1);
  const double ep2 = ex_at<EX, F, G, true>(a, bi + 2 * i1, bj + 2 * j1, bk + 2 * k1);
  const double em2 = ex_at<EX, F, G>(a, bi - 2 * i1, bj - 2 * j1, bk - 2 * k1);
  return k.w1[AX] * (ep1 - em1) + k.w2[AX] * (ep2 - em2);
}

// Second derivative along AX of field F (stencil.py:97-101).
template <int AX, int F, class A>
__device__ __forceinline__ double d2(const Coef& k, const A& a) {
  int i1, j1, k1;
  Off<AX>::at(1, i1, j1, k1);
  return k.s0[AX] * tap<true>(a, F, 0, 0, 0) +
         k.s1[AX] * (tap<true>(a, F, i1, j1, k1) + a.v(F, -i1, -j1, -k1)) +
         k.s2[AX] * (tap<true>(a, F, 2 * i1, 2 * j1, 2 * k1) + a.v(F, -2 * i1, -2 * j1, -2 * k1));
}

// Mixed DD(u_J, x_O, x_J): outer first derivative along O of the inner first
// derivative D(u_J, x_J) re-expanded at the four shifted points
// (codegen.py:97-102).
template <int O, int J, class A>
__device__ __forceinline__ double dd(const Coef& k, const A& a) {
  int i1, j1, k1;
  Off<O>::at(1, i1, j1, k1);
  const double ip1 = d1<J, E_FIELD, U0 + J, 0>(k, a, i1, j1, k1);
  const double im1 = d1<J, E_FIELD, U0 + J, 0>(k, a, -i1, -j1, -k1);
  const double ip2 = d1<J, E_FIELD, U0 + J, 0>(k, a, 2 * i1, 2 * j1, 2 * k1);
  const double im2 = d1<J, E_FIELD, U0 + J, 0>(k, a, -2 * i1, -2 * j1, -2 * k1);
  return k.w1[O] * (ip1 - im1) + k.w2[O] * (ip2 - im2);
}

// Outer first derivative along O of a stored inner-derivative array (the
// reference's FETCH inner read, codegen.py:111-113).
__device__ __forceinline__ double d1_stored(const Coef& k, int O,
                                            const double* __restrict__ wa,
                                            int64_t c, int64_t s) {
  return k.w1[O] * (__ldg(wa + c + s) - __ldg(wa + c - s)) +
         k.w2[O] * (__ldg(wa + c + 2 * s) - __ldg(wa + c - 2 * s));
}

// ---------------------------------------------------------------------------
// Derivative slots (60 distinct derivatives, terms.py:135-200)
// per axis a: 18 slots at a*18 + ...; then 6 mixed at 54 + ...
// ---------------------------------------------------------------------------
enum Slot : int {
  S_RHO = 0, S_P, S_RHOE, S_RHOEU, S_UP, S_T2,
  S_RU = 6,    // + q        D(rhou_q, x_a)
  S_U = 9,     // + q        D(u_q, x_a)
  S_RUU = 12,  // + q        D(rhou_q * u_a, x_a)
  S_U2 = 15,   // + q        D2(u_q, x_a)
  S_PER_AXIS = 18,
  S_DD = 54,   // + dd_index(j, o)   DD(u_j, x_o, x_j)
  N_SLOTS = 60
};
__host__ __device__ constexpr int slot(int a, int local) { return a * S_PER_AXIS + local; }
// mixed index for (inner field j, outer axis o), o != j
__host__ __device__ constexpr int dd_index(int j, int o) { return j * 2 + (o < j ? o : o - 1); }

// Evaluate one derivative slot from point data (used by LOCAL/INLINE
// providers and by the BL fill kernels).
template <int A_, int L, class Acc>
__device__ __forceinline__ double eval_slot(const Coef& k, const Acc& a) {
  if constexpr (L == S_RHO) return d1<A_, E_FIELD, RHO, 0>(k, a);
  else if constexpr (L == S_P) return d1<A_, E_FIELD, PF, 0>(k, a);
  else if constexpr (L == S_RHOE) return d1<A_, E_RHOE, 0, 0>(k, a);
  else if constexpr (L == S_RHOEU) return d1<A_, E_RHOEU, 0, U0 + A_>(k, a);
  else if constexpr (L == S_UP) return d1<A_, E_PROD, U0 + A_, PF>(k, a);
  else if constexpr (L == S_T2) return d2<A_, TF>(k, a);
  else if constexpr (L >= S_RU && L < S_RU + 3) return d1<A_, E_FIELD, RU0 + (L - S_RU), 0>(k, a);
  else if constexpr (L >= S_U && L < S_U + 3) return d1<A_, E_FIELD, U0 + (L - S_U), 0>(k, a);
  else if constexpr (L >= S_RUU && L < S_RUU + 3) return d1<A_, E_PROD, RU0 + (L - S_RUU), U0 + A_>(k, a);
  else return d2<A_, U0 + (L - S_U2)>(k, a);
}

// ---------------------------------------------------------------------------
// Providers
// ---------------------------------------------------------------------------

// INLINE (RA): every occurrence re-expands the stencil from rebased taps.
template <class Acc>
struct InlineProvider {
  const Coef& k;
  const Acc& a;
  __device__ InlineProvider(const Coef& k_, const Acc& a_) : k(k_), a(a_) {}
  template <int A_, int L, int OCC = 0, bool DES = false> __device__ __forceinline__ double g() const {
    if constexpr (DES && Acc::kMaskTaps) return eval_slot<A_, L>(k, a);   // designated
    else return eval_slot<A_, L>(k, occurrence_view<OCC>(a));
  }
  template <int J, int O, int OCC = 0, bool DES = false> __device__ __forceinline__ double x() const {
    if constexpr (DES && Acc::kMaskTaps) return dd<O, J>(k, a);
    else return dd<O, J>(k, occurrence_view<OCC>(a));
  }
};

// LOCAL (SN): each distinct derivative evaluated once into a local.
template <class Acc>
struct LocalProvider {
  double v[N_SLOTS];
  template <int A_, int L> __device__ __forceinline__ void fill1(const Coef& k, const Acc& a) {
    v[slot(A_, L)] = eval_slot<A_, L>(k, a);
    if constexpr (L + 1 < S_PER_AXIS) fill1<A_, L + 1>(k, a);
  }
  __device__ __forceinline__ LocalProvider(const Coef& k, const Acc& a) {
    fill1<0, 0>(k, a);
    fill1<1, 0>(k, a);
    fill1<2, 0>(k, a);
    v[S_DD + dd_index(1, 0)] = dd<0, 1>(k, a);
    v[S_DD + dd_index(2, 0)] = dd<0, 2>(k, a);
    v[S_DD + dd_index(0, 1)] = dd<1, 0>(k, a);
    v[S_DD + dd_index(2, 1)] = dd<1, 2>(k, a);
    v[S_DD + dd_index(0, 2)] = dd<2, 0>(k, a);
    v[S_DD + dd_index(1, 2)] = dd<2, 1>(k, a);
  }
  template <int A_, int L, int OCC = 0, bool DES = false> __device__ __forceinline__ double g() const { return v[slot(A_, L)]; }
  template <int J, int O, int OCC = 0, bool DES = false> __device__ __forceinline__ double x() const { return v[S_DD + dd_index(J, O)]; }
};

// FETCH (BL): every derivative read from its work array at the point.
struct FetchProvider {
  const double* __restrict__ wa;
  int64_t c, fs;
  template <int A_, int L, int OCC = 0, bool DES = false> __device__ __forceinline__ double g() const {
    return __ldg(wa + slot(A_, L) * fs + c);
  }
  template <int J, int O, int OCC = 0, bool DES = false> __device__ __forceinline__ double x() const {
    return __ldg(wa + (S_DD + dd_index(J, O)) * fs + c);
  }
};

// SS / RS: the nine velocity gradients D(u_q, x_a) are FETCHed from work
// arrays (ws[q*3+a]); mixed terms read the stored inner D(u_J, x_J) at
// outer-shifted points; everything else is LOCAL (SS, plan.py:178-179) or
// re-expanded at every occurrence (RS, INLINE, plan.py:176-177).
template <class Acc, bool INLINE_REST = false>
struct SSProvider {
  const Coef& k;
  const Acc& a;
  const double* __restrict__ ws;
  int64_t c, fs, st[3];
  __device__ SSProvider(const Coef& k_, const Acc& a_, const double* ws_, int64_t c_, int64_t fs_,
                        int64_t s0, int64_t s1)
      : k(k_), a(a_), ws(ws_), c(c_), fs(fs_) { st[0] = s0; st[1] = s1; st[2] = 1; }
  template <int A_, int L, int OCC = 0, bool DES = false> __device__ __forceinline__ double g() const {
    if constexpr (L >= S_U && L < S_U + 3) return __ldg(ws + ((L - S_U) * 3 + A_) * fs + c);
    else if constexpr (INLINE_REST) return eval_slot<A_, L>(k, occurrence_view<OCC>(a));
    else return eval_slot<A_, L>(k, a);
  }
  template <int J, int O, int OCC = 0, bool DES = false> __device__ __forceinline__ double x() const {
    return d1_stored(k, O, ws + (J * 3 + J) * fs, c, st[O]);
  }
};

// ---------------------------------------------------------------------------
// The five residual expressions (terms.py:151-183), left-to-right.
// Point values: r[10] = rho, rhou0..2, rhoE, u0..2, p, T at the centre.
// ---------------------------------------------------------------------------
// Occurrence ids of the INLINE providers (RA, RS).  By default every G/X
// call site gets its own id (__COUNTER__, salted by the helper's template
// arguments, so e.g. the three div(u) sums inside tau<0,0>, tau<1,1>,
// tau<2,2> stay distinct): every source occurrence is recomputed.  The id is
// SALT * 64 + counter (60 call sites), so the zero words of neighbouring
// call sites are adjacent in the constant bank and ptxas loads them as
// vectors (static LDCU count 221 -> 179 in the 12-warp RA kernel, whole
// steps +0.6%; the counter * 16 + salt form spread them 64 B apart).
//
// That is more recompute than the reference *executes*: its RA kernel has one
// numba statement per residual, each ending in a store to an output array
// that may alias the inputs, so LLVM merges identical loads and operations
// within a residual statement and never across statements.
// tools/ref_cse_count.py counts the reference's generated kernels under that
// rule -- RA 1074, RS 729, SN 774, SS 609, BL 198 FP ops per point -- against
// the disassembly counts of SURVEY.md 2.1 (RA 1065, SN 750, SS 585, BL 189).
// FDNS_RA_PER_EQUATION=1 reproduces it (every occurrence carries the id of
// its residual equation, EQ: 0 mass, 1-3 momentum, 4 energy), but the merged
// values stay live across the long energy equation: the RA stage kernel
// then needs 255 registers plus 476 B of spills and ran 1.5x slower at
// 256^3-512^3 (RS +3-6%), so the per-occurrence form stays the default.
#ifndef FDNS_RA_PER_EQUATION
#define FDNS_RA_PER_EQUATION 0
#endif
//
// Designated occurrences (round 2): an opaque mask is only needed to keep
// an occurrence apart from the *other* occurrences of the same derivative,
// so each of the 60 derivatives has exactly one call site evaluated from
// the plain accessor (GD / XD with the designation condition and group)
// and every other one masked.  All 117 occurrences are still evaluated
// separately -- every first-level operation of a masked occurrence has a
// masked operand, so none can merge with the designated one; the static
// FP64 count of the RA stage kernel is unchanged (1324) -- but only 57 of
// them are masked.  Groups (bits of FDNS_RA_DESIGNATED, default 27 = 0, 1,
// 3, 4): 0 the only occurrence of its derivative (D(rho), D(p), the
// convective products, D(rhoE), D(rhoE u), D(u p), D2(T), D(rhou_i, x_a)
// for a != i); 1 mass's D(rhou_a, x_a) and D(u_a, x_a); 3 the energy's
// off-diagonal D(u_i, x_j) stress-work multipliers; 4 the energy's viscous
// D2 and mixed terms (group 2 designates momentum's instead: 2.2 KB of
// spills in the 12-warp kernel).  12-warp RA kernel: 6248 -> 5912 static
// instructions, whole RK3 steps +6.4% (256^3) / +5.8% (512^3), RS
// unaffected (its providers ignore the designation;
// profiles/r02_ra_designated_ab.txt).
#ifndef FDNS_RA_DESIGNATED
#define FDNS_RA_DESIGNATED 27   // bit mask of the designated groups below
#endif
#if FDNS_RA_PER_EQUATION
#define G(a, L) P.template g<a, L, EQ>()
#define X(j, o) P.template x<j, o, EQ>()
#define GD(grp, c, a, L) G(a, L)
#define XD(grp, j, o) X(j, o)
#else
#define G(a, L) P.template g<a, L, SALT * 64 + __COUNTER__>()
#define X(j, o) P.template x<j, o, SALT * 64 + __COUNTER__>()
// designated when `c` holds and group `grp` is enabled: 0 = the only
// occurrence of its derivative; 1 = mass; 2 = momentum's viscous terms;
// 3 = the energy's stress-work multipliers
#define GD(grp, c, a, L) \
  P.template g<a, L, SALT * 64 + __COUNTER__, bool((c) && ((FDNS_RA_DESIGNATED >> (grp)) & 1))>()
#define XD(grp, j, o) \
  P.template x<j, o, SALT * 64 + __COUNTER__, bool((FDNS_RA_DESIGNATED >> (grp)) & 1)>()
#endif

template <int I, class Pv>
__device__ __forceinline__ double viscous(const Coef& k, const Pv& P) {
  [[maybe_unused]] constexpr int SALT = 1 + I, EQ = 4;   // used by the energy equation
  // c43*D2(u_i,x_i) + [j != i, ascending: inv_Re*D2(u_i,x_j) + c13*DD(u_j,x_i,x_j)]
  // (terms.py:113-123)
  constexpr int J1 = I == 0 ? 1 : 0;
  constexpr int J2 = I == 2 ? 1 : 2;
  return k.c43 * GD(4, true, I, S_U2 + I) + k.inv_Re * GD(4, true, J1, S_U2 + I) +
         k.c13 * XD(4, J1, I) + k.inv_Re * GD(4, true, J2, S_U2 + I) + k.c13 * XD(4, J2, I);
}

// Momentum i, split into the chain prefix -(0.5*(conv)) - D(p,x_i) and the
// viscous suffix (terms.py:164-165, one flat left-to-right chain; splitting
// a chain after a term keeps every rounding step, so prefix + suffix is
// bitwise the full chain).
template <int I, class Pv>
__device__ __forceinline__ double momentum_prefix(const Coef& k, const Pv& P, const double* r) {
  [[maybe_unused]] constexpr int SALT = 4 + I, EQ = 1 + I;
  const double rui = r[RU0 + I];
  const double conv = GD(0, true, 0, S_RUU + I) + r[U0] * GD(0, I != 0, 0, S_RU + I) + rui * G(0, S_U + 0) +
                      GD(0, true, 1, S_RUU + I) + r[U1] * GD(0, I != 1, 1, S_RU + I) + rui * G(1, S_U + 1) +
                      GD(0, true, 2, S_RUU + I) + r[U2] * GD(0, I != 2, 2, S_RU + I) + rui * G(2, S_U + 2);
  return -(0.5 * conv) - GD(0, true, I, S_P);
}

template <int I, class Pv>
__device__ __forceinline__ double momentum_suffix(const Coef& k, const Pv& P, double pre) {
  [[maybe_unused]] constexpr int SALT = 10 + I, EQ = 1 + I;
  constexpr int J1 = I == 0 ? 1 : 0;
  constexpr int J2 = I == 2 ? 1 : 2;
  return pre + k.c43 * GD(2, true, I, S_U2 + I) + k.inv_Re * GD(2, true, J1, S_U2 + I) + k.c13 * XD(2, J1, I) +
         k.inv_Re * GD(2, true, J2, S_U2 + I) + k.c13 * XD(2, J2, I);
}

template <int I, class Pv>
__device__ __forceinline__ double momentum(const Coef& k, const Pv& P, const double* r) {
  return momentum_suffix<I>(k, P, momentum_prefix<I>(k, P, r));
}

template <int I, int J, class Pv>
__device__ __forceinline__ double tau(const Coef& k, const Pv& P) {
  [[maybe_unused]] constexpr int SALT = 7 + I * 3 + J - (I * 3 + J > 8 ? 9 : 0), EQ = 4;
  // terms.py:126-132
  if constexpr (I == J)
    return 2.0 * k.inv_Re * G(I, S_U + I) - k.c23 * (G(0, S_U + 0) + G(1, S_U + 1) + G(2, S_U + 2));
  else
    return k.inv_Re * (G(J, S_U + I) + G(I, S_U + J));
}

// mass (terms.py:151-156)
template <class Pv>
__device__ __forceinline__ double mass_residual(const Coef& k, const Pv& P, const double* r) {
  [[maybe_unused]] constexpr int SALT = 13, EQ = 0;
  const double acc = GD(1, true, 0, S_RU + 0) + r[U0] * GD(0, true, 0, S_RHO) + r[RHO] * GD(1, true, 0, S_U + 0) +
                     GD(1, true, 1, S_RU + 1) + r[U1] * GD(0, true, 1, S_RHO) + r[RHO] * GD(1, true, 1, S_U + 1) +
                     GD(1, true, 2, S_RU + 2) + r[U2] * GD(0, true, 2, S_RHO) + r[RHO] * GD(1, true, 2, S_U + 2);
  return -(0.5 * acc);
}

// energy (terms.py:167-183), split after the nine stress-work terms
template <bool RHOE_INTERNAL, class Pv>
__device__ __forceinline__ double energy_prefix(const Coef& k, const Pv& P, const double* r) {
  [[maybe_unused]] constexpr int SALT = 14, EQ = 4;
  const double rhoe = RHOE_INTERNAL ? r[RHOE_F]
                                    : r[RHOE_F] - 0.5 * (r[RU0] * r[U0] + r[RU1] * r[U1] +
                                                         r[RU2] * r[U2]);
  const double conv = GD(0, true, 0, S_RHOEU) + r[U0] * GD(0, true, 0, S_RHOE) + rhoe * G(0, S_U + 0) +
                      GD(0, true, 1, S_RHOEU) + r[U1] * GD(0, true, 1, S_RHOE) + rhoe * G(1, S_U + 1) +
                      GD(0, true, 2, S_RHOEU) + r[U2] * GD(0, true, 2, S_RHOE) + rhoe * G(2, S_U + 2);
  const double pwork = GD(0, true, 0, S_UP) + GD(0, true, 1, S_UP) + GD(0, true, 2, S_UP);
  const double heat = k.heat * (GD(0, true, 0, S_T2) + GD(0, true, 1, S_T2) + GD(0, true, 2, S_T2));
  return -(0.5 * conv) - (pwork) + heat +
         tau<0, 0>(k, P) * G(0, S_U + 0) + tau<0, 1>(k, P) * GD(3, true, 1, S_U + 0) +
         tau<0, 2>(k, P) * GD(3, true, 2, S_U + 0) + tau<1, 0>(k, P) * GD(3, true, 0, S_U + 1) +
         tau<1, 1>(k, P) * G(1, S_U + 1) + tau<1, 2>(k, P) * GD(3, true, 2, S_U + 1) +
         tau<2, 0>(k, P) * GD(3, true, 0, S_U + 2) + tau<2, 1>(k, P) * GD(3, true, 1, S_U + 2) +
         tau<2, 2>(k, P) * G(2, S_U + 2);
}

template <class Pv>
__device__ __forceinline__ double energy_suffix(const Coef& k, const Pv& P, const double* r,
                                                double pre) {
  return pre + r[U0] * (viscous<0>(k, P)) + r[U1] * (viscous<1>(k, P)) +
         r[U2] * (viscous<2>(k, P));
}

// RHOE_INTERNAL: r[RHOE_F] already holds rho*e (staged-tile accessors).
// MOMENTUM_FIRST: evaluate the momentum equations before mass and energy
// (each equation's own association is unchanged, so the bits are too); the
// 12-warp SN kernel schedules ~1% faster that way at 512^3, the other
// variants do not gain (profiles/r02_residual_order_ab.txt).
template <bool RHOE_INTERNAL = false, bool MOMENTUM_FIRST = false, class Pv>
__device__ __forceinline__ void residual_point(const Coef& k, const Pv& P, const double* r,
                                               double* out) {
  if constexpr (MOMENTUM_FIRST) {
    out[1] = momentum<0>(k, P, r);
    out[2] = momentum<1>(k, P, r);
    out[3] = momentum<2>(k, P, r);
    out[0] = mass_residual(k, P, r);
  } else {
    out[0] = mass_residual(k, P, r);
    out[1] = momentum<0>(k, P, r);
    out[2] = momentum<1>(k, P, r);
    out[3] = momentum<2>(k, P, r);
  }
  out[4] = energy_suffix(k, P, r, energy_prefix<RHOE_INTERNAL>(k, P, r));
}
#undef G
#undef X
#undef GD
#undef XD

// Fused primitive recovery of one point (physics.py:185-202).
__device__ __forceinline__ void primitives_point(const Coef& k, const double* q, double* prim) {
  const double u0 = q[1] / q[0], u1 = q[2] / q[0], u2 = q[3] / q[0];
  const double p = k.gm1 * (q[4] - 0.5 * (q[1] * u0 + q[2] * u1 + q[3] * u2));
  prim[0] = u0; prim[1] = u1; prim[2] = u2; prim[3] = p;
  prim[4] = k.gM2 * p / q[0];
}

}  // namespace fdns
