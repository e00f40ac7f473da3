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
constexpr int PK = TK + 4, PJ = TJ + 4;
constexpr int PLANE = PK * PJ;          // doubles per field per plane slot
constexpr int SLOT = NFIELDS * PLANE;   // doubles per plane slot
constexpr int NR = 6;                   // ring depth: 5-plane window + 1 prefetch
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_plane(double* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(saddr(bar))
      : "memory");
}

// Shared-memory accessor: p[d] is the plane slot for axis-0 offset d-2,
// already offset to this thread's (j, k) column and field 0.
struct SAcc {
  static constexpr bool kInternalEnergy = true;   // field RHOE_F holds rho*e
  const double* p[5];
  __device__ __forceinline__ double v(int f, int di, int dj, int dk) const {
    return p[di + 2][f * PLANE + dj * PK + dk];
  }
};

// Write the 10 (MODE 1) or 5 (MODE 0) output values of interior point
// (i, j, k) to its location and to every periodic ghost image on the axes
// of wrap_mask (mesh.py:118-139 semantics: ghost = value at the wrapped
// coordinates).
template <int NOUT>
__device__ __forceinline__ void emit(double* out, const Geom& g, int i, int j, int k,
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
  {
    const int64_t c = ci[0] * g.s0 + cj[0] * g.s1 + ck[0];
#pragma unroll
    for (int f = 0; f < NOUT; ++f) out[f * g.fs + c] = val[f];
  }
  if (ni * nj * nk > 1) {
    for (int a = 0; a < ni; ++a)
      for (int b = 0; b < nj; ++b)
        for (int d = 0; d < nk; ++d) {
          if ((a | b | d) == 0) continue;
          const int64_t c = ci[a] * g.s0 + cj[b] * g.s1 + ck[d];
#pragma unroll
          for (int f = 0; f < NOUT; ++f) out[f * g.fs + c] = val[f];
        }
  }
}

// rhoE -> rho*e in one staged plane slot (all PLANE points of the box).
__device__ __forceinline__ void to_internal_energy(double* slot) {
  for (int x = threadIdx.x; x < PLANE; x += NT) {
    const double e = slot[RHOE_F * PLANE + x] -
                     0.5 * (slot[RU0 * PLANE + x] * slot[U0 * PLANE + x] +
                            slot[RU1 * PLANE + x] * slot[U1 * PLANE + x] +
                            slot[RU2 * PLANE + x] * slot[U2 * PLANE + x]);
    slot[RHOE_F * PLANE + x] = e;
  }
}

template <int V, int MODE>
__global__ void __launch_bounds__(NT, 1)
    k_stage_tiled(const __grid_constant__ CUtensorMap tin, const double* __restrict__ work,
                  const double* saved, double* out, Coef k, Geom g, double coef, int chunk,
                  int wrap_mask) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NR * SLOT);
  const int tid = threadIdx.x;
  const int tk = tid % TK, tj = tid / TK;
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * TJ;
  const int i0 = blockIdx.z * chunk;
  const int i1 = min(i0 + chunk, g.n0);
  if (i0 >= i1) return;
  const int nsteps = i1 - i0;
  const int nseq = nsteps + 4;   // planes i0-2 .. i1+1

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int s) {
    const int slot = s % NR;
    mbar_expect_tx(&bars[slot], SLOT * 8);
    tma_load_plane(sm + slot * SLOT, &tin, &bars[slot], k0 + g.h - 2, j0 + g.h - 2,
                   i0 - 2 + s + g.h);
  };
  if (tid == 0)
    for (int s = 0; s < min(NR - 1, nseq); ++s) issue(s);

  const int jj = j0 + tj, kk = k0 + tk;
  const bool active = jj < g.n1 && kk < g.n2;
  const int toff = (tj + 2) * PK + (tk + 2);

  for (int t = 0; t < nsteps; ++t) {
    if (t == 0) {
      for (int s = 0; s < 5; ++s) {
        mbar_wait(&bars[s % NR], (s / NR) & 1);
        to_internal_energy(sm + (s % NR) * SLOT);
      }
    } else {
      const int s = t + 4;
      mbar_wait(&bars[s % NR], (s / NR) & 1);
      to_internal_energy(sm + (s % NR) * SLOT);
    }
    __syncthreads();
    if (tid == 0 && t + 5 < nseq) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + 5);
    }

    SAcc a;
#pragma unroll
    for (int d = 0; d < 5; ++d) a.p[d] = sm + ((t + d) % NR) * SLOT + toff;
    double r[NFIELDS];
#pragma unroll
    for (int f = 0; f < NFIELDS; ++f) r[f] = a.v(f, 0, 0, 0);   // r[RHOE_F] = rho*e

    const int i = i0 + t;
    double R[5];
    if constexpr (V == FDNS_SN) {
      LocalProvider<SAcc> P(k, a);
      residual_point<true>(k, P, r, R);
    } else if constexpr (V == FDNS_RA) {
      InlineProvider<SAcc> P(k, a);
      residual_point<true>(k, P, r, R);
    } else {  // SS / RS: stored velocity gradients from the work arrays
      // inactive (edge) threads read a valid clamped column; never written
      const int64_t c = (int64_t)(i + g.h) * g.s0 + (int64_t)(min(jj, g.n1 - 1) + g.h) * g.s1 +
                        (min(kk, g.n2 - 1) + g.h);
      SSProvider<SAcc> P(k, a, work, c, g.fs, g.s0, g.s1);
      residual_point<true>(k, P, r, R);
    }
    if (active) {
      if constexpr (MODE == 0) {
        emit<5>(out, g, i, jj, kk, R, 0);
      } else {
        const int64_t c = (int64_t)(i + g.h) * g.s0 + (int64_t)(jj + g.h) * g.s1 + (kk + g.h);
        double q[NFIELDS];
#pragma unroll
        for (int f = 0; f < 5; ++f) q[f] = saved[f * g.fs + c] + coef * R[f];
        primitives_point(k, q, q + 5);
        emit<NFIELDS>(out, g, i, jj, kk, q, wrap_mask);
      }
    }
  }
}

}  // namespace tiled
}  // namespace fdns
