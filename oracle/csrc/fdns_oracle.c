/*
 * C99 + OpenMP restatement of the reference hot path -- TEST INFRASTRUCTURE
 * ONLY (the checker and the CPU baseline; never linked into the product).
 *
 * Restates, per interior point, the reference's "SN" route: every distinct
 * derivative of the term list (pkg/src/fdns/terms.py:135-200) is evaluated
 * once into a local with the stencil shapes of stencil.py:71-102 /
 * codegen.py:81-102, then the five residual expressions are evaluated with
 * the reference's left-to-right association (codegen.py:138-149).  Compile
 * with -ffp-contract=off and without -ffast-math: no FMA contraction and no
 * reassociation, so results are bitwise identical to the reference (pinned
 * by tests/test_oracle_golden.py).
 *
 * Layout: a bundle of 10 padded fields, field-major, each C-ordered
 * (n0+2h, n1+2h, n2+2h) with axis 2 contiguous (mesh.py:3-6), in the order
 * rho, rhou0, rhou1, rhou2, rhoE, u0, u1, u2, p, T (physics.py:115-119).
 */
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    ptrdiff_t s[3];      /* element strides of axes 0, 1, 2 */
    ptrdiff_t fs;        /* field stride (elements per padded field) */
    int n[3], h;
} geom_t;

static geom_t mkgeom(int n0, int n1, int n2, int h)
{
    geom_t g;
    g.n[0] = n0; g.n[1] = n1; g.n[2] = n2; g.h = h;
    g.s[2] = 1;
    g.s[1] = n2 + 2 * h;
    g.s[0] = (ptrdiff_t)(n1 + 2 * h) * (n2 + 2 * h);
    g.fs = (ptrdiff_t)(n0 + 2 * h) * g.s[0];
    return g;
}

/* point expressions -- terms.py:39 and the product targets of :158-174 */
typedef struct {
    const double *rho, *ru0, *ru1, *ru2, *rE, *u0, *u1, *u2, *p, *T;
} flds_t;

static inline double rhoe_at(const flds_t *f, ptrdiff_t c)
{
    return f->rE[c] - 0.5 * (f->ru0[c] * f->u0[c] + f->ru1[c] * f->u1[c]
                             + f->ru2[c] * f->u2[c]);
}

/* first derivative of a stored field -- stencil.py:80-84 */
static inline double d1f(const double *a, ptrdiff_t c, ptrdiff_t s,
                         double w1, double w2)
{
    return w1 * (a[c + s] - a[c - s]) + w2 * (a[c + 2 * s] - a[c - 2 * s]);
}

/* first derivative of the product a*b -- products are formed per point and
 * then differentiated (plan.py:383-392, codegen.py:84-89) */
static inline double d1p(const double *a, const double *b, ptrdiff_t c,
                         ptrdiff_t s, double w1, double w2)
{
    return w1 * ((a[c + s] * b[c + s]) - (a[c - s] * b[c - s]))
         + w2 * ((a[c + 2 * s] * b[c + 2 * s]) - (a[c - 2 * s] * b[c - 2 * s]));
}

static inline double d1rhoe(const flds_t *f, ptrdiff_t c, ptrdiff_t s,
                            double w1, double w2)
{
    return w1 * (rhoe_at(f, c + s) - rhoe_at(f, c - s))
         + w2 * (rhoe_at(f, c + 2 * s) - rhoe_at(f, c - 2 * s));
}

static inline double d1rhoeu(const flds_t *f, const double *u, ptrdiff_t c,
                             ptrdiff_t s, double w1, double w2)
{
    return w1 * ((rhoe_at(f, c + s) * u[c + s]) - (rhoe_at(f, c - s) * u[c - s]))
         + w2 * ((rhoe_at(f, c + 2 * s) * u[c + 2 * s])
                 - (rhoe_at(f, c - 2 * s) * u[c - 2 * s]));
}

/* second derivative -- stencil.py:97-101 */
static inline double d2f(const double *a, ptrdiff_t c, ptrdiff_t s,
                         double s0, double s1, double s2)
{
    return s0 * a[c] + s1 * (a[c + s] + a[c - s])
         + s2 * (a[c + 2 * s] + a[c - 2 * s]);
}

/* mixed: outer first derivative (axis so) of the inner first derivative
 * (axis si) re-expanded at the shifted points -- codegen.py:97-102 */
static inline double ddf(const double *a, ptrdiff_t c, ptrdiff_t so,
                         double wo1, double wo2, ptrdiff_t si, double wi1,
                         double wi2)
{
    return wo1 * (d1f(a, c + so, si, wi1, wi2) - d1f(a, c - so, si, wi1, wi2))
         + wo2 * (d1f(a, c + 2 * so, si, wi1, wi2)
                  - d1f(a, c - 2 * so, si, wi1, wi2));
}

/*
 * Residual at every interior point.  w[15] = (fw1, fw2, s0, s1, s2) per axis
 * (plan.py:339-344); kc[5] = inv_Re, c13, c43, c23, heat_coeff
 * (physics.py:78-81).  Writes interior points of out (5 padded fields).
 */
int oracle_residual(const double *F, double *out, int n0, int n1, int n2,
                    int h, const double *w, const double *kc, int nthreads)
{
    geom_t g = mkgeom(n0, n1, n2, h);
    flds_t f;
    const double *fp[10];
    for (int q = 0; q < 10; ++q) fp[q] = F + q * g.fs;
    f.rho = fp[0]; f.ru0 = fp[1]; f.ru1 = fp[2]; f.ru2 = fp[3]; f.rE = fp[4];
    f.u0 = fp[5]; f.u1 = fp[6]; f.u2 = fp[7]; f.p = fp[8]; f.T = fp[9];
    const double inv_Re = kc[0], c13 = kc[1], c43 = kc[2], c23 = kc[3],
                 heat = kc[4];
    double *o_rho = out, *o_r0 = out + g.fs, *o_r1 = out + 2 * g.fs,
           *o_r2 = out + 3 * g.fs, *o_E = out + 4 * g.fs;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel for collapse(2) schedule(static)
    for (int i = h; i < n0 + h; ++i) {
        for (int j = h; j < n1 + h; ++j) {
            for (int k = h; k < n2 + h; ++k) {
                const ptrdiff_t c = i * g.s[0] + j * g.s[1] + k;
                const double *u[3] = {f.u0, f.u1, f.u2};
                const double *ru[3] = {f.ru0, f.ru1, f.ru2};
                double D_rho[3], D_p[3], D_rhoe[3], D_rhoeu[3], D_up[3],
                       D2_T[3], D_ru[3][3], D_u[3][3], D_ruu[3][3],
                       D2_u[3][3], DD_u[3][3];
                for (int a = 0; a < 3; ++a) {
                    const ptrdiff_t s = g.s[a];
                    const double w1 = w[5 * a], w2 = w[5 * a + 1];
                    const double s0 = w[5 * a + 2], s1 = w[5 * a + 3],
                                 s2 = w[5 * a + 4];
                    D_rho[a] = d1f(f.rho, c, s, w1, w2);
                    D_p[a] = d1f(f.p, c, s, w1, w2);
                    D_rhoe[a] = d1rhoe(&f, c, s, w1, w2);
                    D_rhoeu[a] = d1rhoeu(&f, u[a], c, s, w1, w2);
                    D_up[a] = d1p(u[a], f.p, c, s, w1, w2);
                    D2_T[a] = d2f(f.T, c, s, s0, s1, s2);
                    for (int q = 0; q < 3; ++q) {
                        D_ru[q][a] = d1f(ru[q], c, s, w1, w2);
                        D_u[q][a] = d1f(u[q], c, s, w1, w2);
                        D_ruu[q][a] = d1p(ru[q], u[a], c, s, w1, w2);
                        D2_u[q][a] = d2f(u[q], c, s, s0, s1, s2);
                    }
                }
                /* DD_u[j][o] = DD(u_j, x_o, x_j) for o != j */
                for (int jj = 0; jj < 3; ++jj)
                    for (int o = 0; o < 3; ++o)
                        DD_u[jj][o] = (o == jj) ? 0.0 :
                            ddf(u[jj], c, g.s[o], w[5 * o], w[5 * o + 1],
                                g.s[jj], w[5 * jj], w[5 * jj + 1]);

                const double rho = f.rho[c], rE = f.rE[c];
                const double uc[3] = {f.u0[c], f.u1[c], f.u2[c]};
                const double ruc[3] = {f.ru0[c], f.ru1[c], f.ru2[c]};

                /* mass -- terms.py:151-156 */
                double acc = D_ru[0][0] + uc[0] * D_rho[0] + rho * D_u[0][0]
                           + D_ru[1][1] + uc[1] * D_rho[1] + rho * D_u[1][1]
                           + D_ru[2][2] + uc[2] * D_rho[2] + rho * D_u[2][2];
                o_rho[c] = -(0.5 * acc);

                /* momentum -- terms.py:158-165 with _viscous :113-123 */
                double *o_ru[3] = {o_r0, o_r1, o_r2};
                double visc[3];
                for (int q = 0; q < 3; ++q) {
                    acc = D_ruu[q][0] + uc[0] * D_ru[q][0] + ruc[q] * D_u[0][0]
                        + D_ruu[q][1] + uc[1] * D_ru[q][1] + ruc[q] * D_u[1][1]
                        + D_ruu[q][2] + uc[2] * D_ru[q][2] + ruc[q] * D_u[2][2];
                    double r = -(0.5 * acc) - D_p[q];
                    double v = c43 * D2_u[q][q];
                    r = r + c43 * D2_u[q][q];
                    for (int jj = 0; jj < 3; ++jj) {
                        if (jj == q) continue;
                        r = r + inv_Re * D2_u[q][jj];
                        r = r + c13 * DD_u[jj][q];
                        v = v + inv_Re * D2_u[q][jj];
                        v = v + c13 * DD_u[jj][q];
                    }
                    o_ru[q][c] = r;
                    visc[q] = v;
                }

                /* energy -- terms.py:167-183, _tau :126-132 */
                const double rhoe = rE - 0.5 * (ruc[0] * uc[0] + ruc[1] * uc[1]
                                                + ruc[2] * uc[2]);
                acc = D_rhoeu[0] + uc[0] * D_rhoe[0] + rhoe * D_u[0][0]
                    + D_rhoeu[1] + uc[1] * D_rhoe[1] + rhoe * D_u[1][1]
                    + D_rhoeu[2] + uc[2] * D_rhoe[2] + rhoe * D_u[2][2];
                double r = -(0.5 * acc) - (D_up[0] + D_up[1] + D_up[2])
                         + heat * (D2_T[0] + D2_T[1] + D2_T[2]);
                for (int q = 0; q < 3; ++q) {
                    for (int jj = 0; jj < 3; ++jj) {
                        double tau;
                        if (q == jj)
                            tau = 2.0 * inv_Re * D_u[q][q]
                                - c23 * (D_u[0][0] + D_u[1][1] + D_u[2][2]);
                        else
                            tau = inv_Re * (D_u[q][jj] + D_u[jj][q]);
                        r = r + tau * D_u[q][jj];
                    }
                }
                for (int q = 0; q < 3; ++q) r = r + uc[q] * visc[q];
                o_E[c] = r;
            }
        }
    }
    return 0;
}

/* fused primitive recovery over the padded arrays -- physics.py:185-202 */
int oracle_primitives(double *F, int n0, int n1, int n2, int h, double gm1,
                      double gM2, int nthreads)
{
    geom_t g = mkgeom(n0, n1, n2, h);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    double *rho = F, *ru0 = F + g.fs, *ru1 = F + 2 * g.fs, *ru2 = F + 3 * g.fs,
           *rE = F + 4 * g.fs, *u0 = F + 5 * g.fs, *u1 = F + 6 * g.fs,
           *u2 = F + 7 * g.fs, *p = F + 8 * g.fs, *T = F + 9 * g.fs;
#pragma omp parallel for schedule(static)
    for (ptrdiff_t c = 0; c < g.fs; ++c) {
        const double a0 = ru0[c] / rho[c], a1 = ru1[c] / rho[c],
                     a2 = ru2[c] / rho[c];
        u0[c] = a0; u1[c] = a1; u2[c] = a2;
        const double pp = gm1 * (rE[c] - 0.5 * (ru0[c] * a0 + ru1[c] * a1
                                                + ru2[c] * a2));
        p[c] = pp;
        T[c] = gM2 * pp / rho[c];
    }
    return 0;
}

/* periodic ghost fill of nf consecutive padded fields -- mesh.py:118-139 */
int oracle_halo(double *F, int nf, int n0, int n1, int n2, int h)
{
    geom_t g = mkgeom(n0, n1, n2, h);
    const int P[3] = {n0 + 2 * h, n1 + 2 * h, n2 + 2 * h};
    for (int q = 0; q < nf; ++q) {
        double *a = F + q * g.fs;
        for (int ax = 0; ax < 3; ++ax) {
            const int n = g.n[ax];
            for (int i = 0; i < P[0]; ++i)
                for (int j = 0; j < P[1]; ++j)
                    for (int k = 0; k < P[2]; ++k) {
                        int idx[3] = {i, j, k};
                        int x = idx[ax];
                        if (x >= h && x < n + h) continue;
                        idx[ax] = x < h ? x + n : x - n;
                        a[i * g.s[0] + j * g.s[1] + k] =
                            a[idx[0] * g.s[0] + idx[1] * g.s[1] + idx[2]];
                    }
        }
    }
    return 0;
}

/*
 * niter save-state RK3 iterations in place on F (timeloop.py:75-94).
 * saved/res are caller-provided scratch of 5 padded fields each.
 */
int oracle_run(double *F, double *saved, double *res, int n0, int n1, int n2,
               int h, const double *w, const double *kc, double gm1,
               double gM2, double dt, int niter, int nthreads)
{
    static const double alpha[3] = {1.0 / 3.0, 1.0 / 2.0, 1.0};
    geom_t g = mkgeom(n0, n1, n2, h);
    for (int it = 0; it < niter; ++it) {
        memcpy(saved, F, (size_t)5 * g.fs * sizeof(double));
        for (int st = 0; st < 3; ++st) {
            oracle_primitives(F, n0, n1, n2, h, gm1, gM2, nthreads);
            oracle_residual(F, res, n0, n1, n2, h, w, kc, nthreads);
            const double coef = alpha[st] * dt;
            for (int q = 0; q < 5; ++q) {
                double *cq = F + q * g.fs;
                const double *sq = saved + q * g.fs, *rq = res + q * g.fs;
#pragma omp parallel for collapse(2) schedule(static)
                for (int i = h; i < n0 + h; ++i)
                    for (int j = h; j < n1 + h; ++j)
                        for (int k = h; k < n2 + h; ++k) {
                            const ptrdiff_t c = i * g.s[0] + j * g.s[1] + k;
                            cq[c] = sq[c] + coef * rq[c];
                        }
            }
            oracle_halo(F, 5, n0, n1, n2, h);
        }
    }
    return 0;
}
