/*
 * fdns_b200.h -- C ABI of the B200-native fdns hot path.
 *
 * Plain C: raw device pointers, sizes, a cudaStream_t passed as void*, and an
 * int status (0 = ok; otherwise fdns_last_error() describes the failure).
 * No torch types cross this boundary; the Python host layer
 * (paper_1610_09146_b200/_lib.py) binds it with ctypes and torch only owns
 * the buffers.
 *
 * Storage: every field is a float64 array C-ordered (n0+2h, n1+2h, n2+2h),
 * axis 2 contiguous -- byte-identical to the reference's padded numpy arrays
 * (pkg/src/fdns/mesh.py:3-6).  A "bundle" is `nf` such fields back to back at
 * a field stride of (n0+2h)(n1+2h)(n2+2h) elements; the state bundle holds
 * rho, rhou0, rhou1, rhou2, rhoE, u0, u1, u2, p, T in the reference's kernel
 * argument order (pkg/src/fdns/physics.py:115-119).  For a z-slab rank, n0 is
 * the number of local planes along axis 0.
 *
 * Reference interfaces each entry point replaces are cited per function
 * (paths relative to /root/reference/pkg/src/fdns/).
 */
#ifndef FDNS_B200_H
#define FDNS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variant ids: the reference's PLAN_NAMES (plan.py:33). */
enum fdns_variant { FDNS_BL = 0, FDNS_RA = 1, FDNS_RS = 2, FDNS_SN = 3, FDNS_SS = 4 };

/* Problem description shared by every call. */
typedef struct fdns_problem {
  int32_t n[3];      /* interior points per axis (n[0] = local planes) */
  int32_t h;         /* halo width (>= 2; mesh.py:17,82) */
  double w[15];      /* (fw1, fw2, s0, s1, s2) per axis (plan.py:339-344) */
  double kc[5];      /* inv_Re, c13, c43, c23, heat_coeff (physics.py:78-81) */
  double gm1, gM2;   /* gamma-1, gamma*M*M (physics.py:53-58) */
} fdns_problem;

/* Text of the last failure on this thread ("" if none). */
const char* fdns_last_error(void);

/* ABI version, for the host loader's sanity check. */
int32_t fdns_abi_version(void);

/* Number of hot-path kernels this library has launched so far (all
 * threads); the bench reports the delta over its timed region. */
int64_t fdns_launch_count(void);

/* Number of work arrays a variant allocates (plan.py:220-227: BL 60 (+0
 * scratch -- products are formed in registers), RA/SN 0, RS/SS 9). */
int32_t fdns_workarray_count(int32_t variant);

/* Primitive recovery u, p, T from the conservative fields of a state bundle,
 * over the full padded arrays -- replaces eval_primitives_fused /
 * eval_primitives_grouped (physics.py:169-202). */
int32_t fdns_primitives(double* state, const fdns_problem* pb, void* stream);

/* The same on padded axis-0 planes [p_lo, p_hi) only (0 <= p_lo <= p_hi <=
 * n0+2h): a z-slab rank forms u, p, T of its ghost planes after receiving
 * their conservative fields (decomp.py), the values the sending rank's
 * stage kernel computed with the same expressions. */
int32_t fdns_primitives_planes(double* state, int32_t p_lo, int32_t p_hi,
                               const fdns_problem* pb, void* stream);

/* Periodic ghost fill of nf consecutive fields along the axes in axes_mask
 * (bit a = axis a) -- replaces mesh.halo_exchange (mesh.py:118-139). */
int32_t fdns_halo_wrap(double* fields, int32_t nf, int32_t axes_mask,
                       const fdns_problem* pb, void* stream);

/* One 4th-order stencil applied to one padded field `f` (halo current),
 * written to the interior of `out` (not aliasing f): op 0-2 = first
 * derivative along that axis, 3-5 = second derivative along axis op-3 --
 * replaces stencil.first_derivative / second_derivative
 * (stencil.py:71-102). */
int32_t fdns_derivative(const double* f, double* out, int32_t op,
                        const fdns_problem* pb, void* stream);

/* Residual of a state bundle (primitives and halos current) under a variant;
 * writes the interior of the 5 residual fields -- replaces
 * ResidualEvaluator.evaluate (plan.py:394-416) and the generated kernel
 * (codegen.py:156-179).  `work` holds fdns_workarray_count(variant) padded
 * fields (may be NULL when the count is 0).  `out`, `state` and `work` must
 * not overlap (the kernels read the state's stencil while writing `out`);
 * an overlapping call fails. */
int32_t fdns_residual(int32_t variant, const double* state, double* work,
                      double* out, const fdns_problem* pb, void* stream);

/* RK stage update cons = saved + coef*res on the interior of 5 fields --
 * replaces the update loop of rk_substep (timeloop.py:80-85). */
int32_t fdns_rk_update(double* cons, const double* saved, const double* res,
                       double coef, const fdns_problem* pb, void* stream);

/* One fused RK stage: residual of `in` (a state bundle with current halos)
 * under the variant, q = saved + coef*R, primitives of q, all written to the
 * interior of the `out` state bundle AND to each point's periodic ghost
 * images on the axes in wrap_mask (0b111 on one GPU; 0b110 for a z-slab
 * rank, whose axis-0 ghosts come from the slab exchange).  `saved` is 5
 * conservative fields and may alias `out` (pointwise update).  Bitwise equal
 * to fdns_residual + fdns_rk_update + fdns_halo_wrap + fdns_primitives --
 * replaces rk_substep (timeloop.py:75-85). */
int32_t fdns_stage(int32_t variant, const double* in, const double* saved,
                   double* out, double* work, double coef, int32_t wrap_mask,
                   const fdns_problem* pb, void* stream);

/* The fused stage restricted to local axis-0 planes [i_lo, i_hi) (interior
 * indices); work-array fills over the whole slab first when with_fills.  A
 * z-slab rank updates its 2h boundary planes, starts the halo exchange on a
 * communication stream, and updates the interior planes meanwhile
 * (decomp.py); the union of the ranges is bitwise fdns_stage. */
int32_t fdns_stage_planes(int32_t variant, const double* in,
                          const double* saved, double* out, double* work,
                          double coef, int32_t wrap_mask, int32_t i_lo,
                          int32_t i_hi, int32_t with_fills,
                          const fdns_problem* pb, void* stream);

/* Test hook selecting the kernel family: 0 = default (TMA-staged tiled
 * kernels where the row pitch allows), 1 = one-thread-per-point kernels (global-memory
 * taps) for every variant; 2 = the 8-warp tiled kernel (SN, RA, SS, RS),
 * 5 = the 12-warp kernel (the default for SN and RA where its tile rows fit
 * the grid, for SS and RS on large planes with the round-robin split);
 * SN only: 4 = eagerly evaluated derivatives.  All paths are
 * parity-tested. */
void fdns_set_kernel_path(int32_t path);

/* Test hook: force the persistent tiled kernels onto `ctas` CTAs (0 =
 * default, one per SM) -- small grids then cross many tile/segment
 * boundaries inside one CTA. */
void fdns_set_tiled_grid(int32_t ctas);

/* Programmatic dependent launch of the tiled stage kernels (default on):
 * a stage's CTAs are dispatched as the previous stage's retire and wait in
 * griddepcontrol.wait before any global access. */
void fdns_set_pdl(int32_t enabled);

/* L2 prefetches issued by the stage kernels' producer thread (default: both
 * on; env FDNS_NO_SAVED_PREFETCH / FDNS_NO_GRAD_PREFETCH turn them off at
 * load): bit 0 = the saved state of RK stages 2/3, bit 1 = SS/RS's nine
 * stored gradients.  A kill switch and an A/B hook. */
void fdns_set_prefetch(int32_t mask);

/* Test hook: unit size (planes) of the round-robin split of the SS, RS and
 * SN stage kernels (-1 = default: SS/RS 64-plane units from 256 planes, SS/RS
 * and SN 128-plane units from 512; 0 = off; c > 0 = c-plane units wherever
 * the plane count is a multiple of c and at least 2c). */
void fdns_set_rounds(int32_t planes);

/* Lockstep of the round-robin CTAs: a CTA waits while a tile-grid neighbour
 * is more than `slack` step barriers behind, so the halos they share hit in
 * L2 (-1 = default, 2; 0 = free running).  A kill switch and an A/B hook;
 * results do not depend on it. */
void fdns_set_lockstep(int32_t slack);

/* Debug timeline of the tiled stage kernels: enable (1) / disable (0) the
 * per-CTA %globaltimer stamps (entry, prologue done, first window ready,
 * exit; 4 per CTA) and copy up to n of them to host memory `out`.
 * enable = 2 starts a launch log (every CTA of every launch appends its four
 * stamps and blockIdx | smid << 16); enable = 3 stops it and copies
 * [count, count x 5 words] to `out`. */
int32_t fdns_debug_trace(int32_t enable, uint64_t* out, int32_t n);

/* Host-side walk of the round-robin split (no GPU needed; a test hook for
 * the partition the stage kernels use, fdns_tiled.cuh:Segments): `tiles`
 * column tiles x `planes` planes in `unit`-plane units on `ctas` CTAs.
 * cover[tile * planes + plane] is incremented once per visit (the caller
 * zeroes it; every entry must end at 1), steps[b] receives CTA b's plane
 * steps and segs[b] its segment count (either may be NULL).  Returns the
 * number of CTAs launched (min(ctas, units)) or -1 on bad arguments. */
int32_t fdns_debug_rounds_walk(int64_t tiles, int32_t planes, int32_t unit, int32_t ctas,
                               int32_t* cover, int32_t* steps, int32_t* segs);

/* Device reduction of the diagnostics of a state bundle (halos current):
 * out[0] = sum 0.5*rho*|u|^2, out[1] = sum 0.5*rho*|omega|^2, with rho from
 * `state` and the velocities (fields 5-7) from `prim_state` (NULL = state;
 * the time loop passes the bundle whose primitives the reference's
 * ConservativeState would be holding, see timeloop.py),
 * out[2..6] = interior sums of rho, rhou0..2, rhoE, out[7] = count of
 * non-finite conservative values, out[8] = count of rho <= 0.
 * `partials` is scratch of fdns_diag_partials_size() doubles.  Replaces
 * kinetic_energy_integral / enstrophy_integral / conservation_sums /
 * check_physical (diagnostics.py:94-146, physics.py:121-129). */
int32_t fdns_diag_partials_size(const fdns_problem* pb);
int32_t fdns_reduce_diag(const double* state, const double* prim_state,
                         double* partials, double* out9,
                         const fdns_problem* pb, void* stream);

/* FP64 issue-rate probe: runs a DADD-only kernel for `iters` iterations and
 * returns (via out[0]) the number of FP64 instructions it executed; time it
 * with events on `stream` to get the in-run FP64 peak for the roofline. */
int32_t fdns_fp64_probe(double* scratch, int32_t iters, double* out_count,
                        void* stream);

/* L2 flush helper for timing hygiene: writes `bytes` of `buf`. */
int32_t fdns_l2_flush(void* buf, int64_t bytes, void* stream);

/* Copy `bytes` between two UVA addresses with an SM kernel (`ctas` CTAs,
 * <= 0: 4 per SM): device memory or pinned (mapped) host memory on either
 * side, 16-byte aligned.  The host-buffer stepping path (hostio.py) uses it
 * for the upload of the reference-layout host fields (the role of the
 * numpy arrays the reference passes to ResidualEvaluator.evaluate,
 * plan.py:394-416). */
int32_t fdns_copy_sm(void* dst, const void* src, int64_t bytes, int32_t ctas, void* stream);

/* `rows` runs of `row_bytes` each, `src_pitch` / `dst_pitch` bytes apart,
 * copied by a copy engine (cudaMemcpy2DAsync, direction inferred from the
 * pointers): one DMA operation for the same plane range of several fields
 * of a bundle (hostio.py's chunk uploads and downloads). */
int32_t fdns_copy_rows(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                       int64_t row_bytes, int64_t rows, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDNS_B200_H */
