// fdns_sn2.cuh -- SN stage kernel with two warp groups per point.
//
// Same staging as k_stage_tiled (persistent CTAs, 32x8 column tiles marching
// along axis 0, a 6-slot TMA ring of whole planes, rhoE -> rho*e on arrival,
// SN centre-plane buffers), but 512 threads: 16 warps per SM instead of 8,
// which is what an FP64-latency-bound kernel needs and what shared memory
// (a 6-plane ring of 10 fields fills ~200 KB) otherwise forbids.
//
// Each point is owned by a thread in warp group A (warps 0-7) and one in
// group B (warps 8-15); groups are whole warps, so nothing diverges.
//   A: mass and the three momentum residuals, their RK update and u = rhou/rho
//   B: the energy residual and its RK update
// The two groups are independent within a step (the energy residual needs
// the viscous terms too, so B evaluates them itself); p and T are derived on
// arrival of each staged plane instead of being written by the epilogue.
// Each group evaluates every derivative it uses once (SN, LOCAL semantics
// per thread; the compiler CSEs repeated uses); the diagonal velocity
// gradients and mixed terms come from the shared centre-plane buffers and
// the axis-0 queues.
#pragma once
#include "fdns_tiled.cuh"

namespace fdns {
namespace sn2 {

using tiled::NR;
using tiled::PJ;
using tiled::PK;
using tiled::PLANE;
using tiled::SAcc;
using tiled::SLOT;
using tiled::TJ;
using tiled::TK;

constexpr int NPT = TK * TJ;     // points per plane step (256)
constexpr int NT = 2 * NPT;      // threads (512)
// packed centre-plane buffers: D(u0,x0) on the whole box (pitch PK),
// D(u1,x1) on interior rows (pitch PK), D(u2,x2) on interior columns
// (pitch TK); double-buffered by step parity
constexpr int B0_N = PLANE, B1_N = TJ * PK, B2_N = PJ * TK;
constexpr int BSET = B0_N + B1_N + B2_N;
constexpr int NXCH = 0;
constexpr int SMEM_BYTES = NR * SLOT * 8 + 2 * BSET * 8 + NXCH * NPT * 8 + 64;
static_assert(SMEM_BYTES <= 232448, "sn2 tile exceeds the 227 KB shared-memory limit");

// Lazily evaluated LOCAL provider over the staged tile: a derivative is
// evaluated where it is used; repeated uses are merged by the compiler.
// Diagonal velocity gradients and mixed terms come from the buffers/queues.
struct LazyProvider {
  const Coef& k;
  const SAcc& a;
  const double* q1;   // D(u1,x1) at this column, planes i-2..i+2 (group A)
  const double* q2;   // D(u2,x2)
  const double* b0;   // D(u0,x0) centre (pitch PK)
  const double* b1;   // D(u1,x1) centre (pitch PK, row stride PK)
  const double* b2;   // D(u2,x2) centre (pitch TK)
  template <int A_, int L, int OCC = 0>
  __device__ __forceinline__ double g() const {
    if constexpr (L == S_U + A_) {
      if constexpr (A_ == 0) return b0[0];
      else if constexpr (A_ == 1) return b1[0];
      else return b2[0];
    } else {
      return eval_slot<A_, L>(k, a);
    }
  }
  template <int J, int O, int OCC = 0>
  __device__ __forceinline__ double x() const {
    if constexpr (O == 0) {   // DD(u1,x0,x1), DD(u2,x0,x2): queues
      const double* q = J == 1 ? q1 : q2;
      return k.w1[0] * (q[3] - q[1]) + k.w2[0] * (q[4] - q[0]);
    } else if constexpr (J == 0) {   // DD(u0,x1,x0) / DD(u0,x2,x0)
      constexpr int s = O == 1 ? PK : 1;
      return k.w1[O] * (b0[s] - b0[-s]) + k.w2[O] * (b0[2 * s] - b0[-2 * s]);
    } else if constexpr (J == 2) {   // DD(u2,x1,x2): outer axis 1 over D(u2,x2)
      return k.w1[1] * (b2[TK] - b2[-TK]) + k.w2[1] * (b2[2 * TK] - b2[-2 * TK]);
    } else {                          // DD(u1,x2,x1): outer axis 2 over D(u1,x1)
      return k.w1[2] * (b1[1] - b1[-1]) + k.w2[2] * (b1[2] - b1[-2]);
    }
  }
};

template <int MODE>
__global__ void __launch_bounds__(NT, 1)
    k_stage_sn2(const __grid_constant__ CUtensorMap tin, const double* saved, double* out,
                Coef k, Geom g, double coef, int ntk, int64_t total_steps, int wrap_mask,
                int i_lo, int nplanes, int aligned) {
  extern __shared__ __align__(128) double sm[];
  double* bset0 = sm + NR * SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bset0 + 2 * BSET);
  const int tid = threadIdx.x;
  const bool groupB = tid >= NPT;
  const int pt = groupB ? tid - NPT : tid;
  const int tk = pt % TK, tj = pt / TK;
  tiled::Segments S = tiled::Segments::partition(blockIdx.x, gridDim.x, total_steps, nplanes,
                                                   aligned);
  if (S.beg >= S.end) return;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) tiled::mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  int64_t p_seg = S.beg;
  int p_r = 0, issued = 0;
  auto issue_next = [&]() {
    const int64_t se = S.seg_end(p_seg);
    const int len = (int)(se - p_seg) + 4;
    const int64_t tile = p_seg / nplanes;
    const int plane = i_lo + (int)(p_seg % nplanes) - 2 + p_r;
    const int slot = issued % NR;
    tiled::mbar_expect_tx(&bars[slot], tiled::LOAD_BYTES);
    tiled::tma_load_plane(sm + slot * SLOT, &tin, &bars[slot], (int)(tile % ntk) * TK + g.h - 2,
                          (int)(tile / ntk) * TJ + g.h - 2, plane + g.h);
    ++issued;
    if (++p_r == len) { p_r = 0; p_seg = se; }
  };
  int total_pos = 0;
  for (int64_t x = S.beg; x < S.end; x = S.seg_end(x)) total_pos += (int)(S.seg_end(x) - x) + 4;
  if (tid == 0)
    while (issued < total_pos && issued < NR) issue_next();

  int w = 0;
  for (int64_t x = S.beg; x < S.end; x = S.seg_end(x)) {
    const int64_t se = S.seg_end(x);
    const int64_t tile = x / nplanes;
    const int k0 = (int)(tile % ntk) * TK, j0 = (int)(tile / ntk) * TJ;
    const int jj = j0 + tj, kk = k0 + tk;
    const bool active = jj < g.n1 && kk < g.n2;
    const int toff = (tj + 2) * PK + (tk + 2);
    const int nsteps = (int)(se - x);
    double q1[5], q2[5];   // group A axis-0 queues
    for (int t = 0; t < nsteps; ++t, ++w) {
      if (t == 0 && w > 0) {
        __syncthreads();
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          while (issued < total_pos && issued < w + NR) issue_next();
        }
      }
      const int first = t == 0 ? w : w + 4;
      for (int pp = first; pp <= w + 4; ++pp) {
        tiled::mbar_wait(&bars[pp % NR], (pp / NR) & 1);
        tiled::stage_arrival(k, sm + (pp % NR) * SLOT, tid, NT);
      }
      double* bs = bset0 + (w & 1) * BSET;
      for (int xx = tid; xx < BSET; xx += NT) {      // centre-plane buffers
        int pos, which;
        if (xx < B0_N) { pos = xx; which = 0; }
        else if (xx < B0_N + B1_N) { pos = 2 * PK + (xx - B0_N); which = 1; }
        else { const int y = xx - B0_N - B1_N; pos = (y / TK) * PK + 2 + y % TK; which = 2; }
        SAcc b;
#pragma unroll
        for (int d = 0; d < 5; ++d) b.p[d] = sm + ((w + d) % NR) * SLOT + pos;
        if (which == 0) bs[xx] = d1<0, E_FIELD, U0, 0>(k, b);
        else if (which == 1) bs[xx] = d1<1, E_FIELD, U1, 0>(k, b);
        else bs[xx] = d1<2, E_FIELD, U2, 0>(k, b);
      }
      SAcc a;
#pragma unroll
      for (int d = 0; d < 5; ++d) a.p[d] = sm + ((w + d) % NR) * SLOT + toff;
      {   // axis-0 queues of D(u1,x1), D(u2,x2) (both groups use the mixed terms)
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
      __syncthreads();
      if (tid == 0 && issued < total_pos && issued < w + NR) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        while (issued < total_pos && issued < w + NR) issue_next();
      }

      double r[NFIELDS];
#pragma unroll
      for (int f = 0; f < NFIELDS; ++f) r[f] = a.v(f, 0, 0, 0);   // r[RHOE_F] = rho*e
      const int i = i_lo + (int)(x % nplanes) + t;
      const LazyProvider P{k, a, q1, q2, bs + toff, bs + B0_N + tj * PK + tk + 2,
                           bs + B0_N + B1_N + (tj + 2) * TK + tk};
      const int64_t c = (int64_t)(i + g.h) * g.s0 + (int64_t)(min(jj, g.n1 - 1) + g.h) * g.s1 +
                        (min(kk, g.n2 - 1) + g.h);
      if (groupB) {
        double sv = 0.0;
        if constexpr (MODE == 1) sv = saved[RHOE_F * g.fs + c];
        const double RE = energy_suffix(k, P, r, energy_prefix<true>(k, P, r));
        if (active) {
          if constexpr (MODE == 0) {
            tiled::emit<1>(out + RHOE_F * g.fs, g, i, jj, kk, &RE, 0);
          } else {
            const double qe = sv + coef * RE;
            tiled::emit<1>(out + RHOE_F * g.fs, g, i, jj, kk, &qe, wrap_mask);
          }
        }
      } else {
        double sv[4];
        if constexpr (MODE == 1) {
#pragma unroll
          for (int f = 0; f < 4; ++f) sv[f] = saved[f * g.fs + c];
        }
        double R[4];
        R[0] = mass_residual(k, P, r);
        R[1] = momentum<0>(k, P, r);
        R[2] = momentum<1>(k, P, r);
        R[3] = momentum<2>(k, P, r);
        if (active) {
          if constexpr (MODE == 0) {
            tiled::emit<4>(out, g, i, jj, kk, R, 0);
          } else {
            double q[8];
#pragma unroll
            for (int f = 0; f < 4; ++f) q[f] = sv[f] + coef * R[f];
            const double u[3] = {q[RU0] / q[RHO], q[RU1] / q[RHO], q[RU2] / q[RHO]};
            tiled::emit<4>(out, g, i, jj, kk, q, wrap_mask);
            tiled::emit<3>(out + U0 * g.fs, g, i, jj, kk, u, wrap_mask);
          }
        }
      }
    }
    w += 4;
  }
}

}  // namespace sn2
}  // namespace fdns
