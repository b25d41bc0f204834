/*
 * direct.c -- oracle direct modal sum (eq. "analysis:sum"):
 *   Phi^(n)(r_j, z_j) = sum_i S_i^(n) G^(n)(r_j, r_i, z_j - z_i),  n = 0..N.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Pairs with bitwise-equal (r, z) are skipped when
 * exclude_coincident is set (the self term, reading R#15).  Sum over i in input order.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "oracle.h"

int64_t or_direct(const double *sr, const double *sz, const double *S, int64_t ns,
                  const double *fr, const double *fz, int64_t nf, int nmodes, int miller,
                  int exclude_coincident, double *Phi, int nthreads)
{
    if (nmodes < 1) return -1;
    int64_t skipped = 0;
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel reduction(+ : skipped) reduction(| : err)
    {
        double *G = (double *)malloc(sizeof(double) * nmodes);
#pragma omp for schedule(dynamic, 16)
        for (int64_t j = 0; j < nf; ++j) {
            double *out = Phi + 2 * (size_t)j * nmodes;
            memset(out, 0, sizeof(double) * 2 * nmodes);
            for (int64_t i = 0; i < ns; ++i) {
                if (sr[i] == fr[j] && sz[i] == fz[j]) {
                    if (exclude_coincident) {
                        ++skipped;
                        continue;
                    }
                    err = 1;
                    continue;
                }
                if (or_greens(fr[j], sr[i], fz[j] - sz[i], nmodes - 1, miller, G) != 0) {
                    err = 1;
                    continue;
                }
                const double *Si = S + 2 * (size_t)i * nmodes;
                for (int n = 0; n < nmodes; ++n) {
                    out[2 * n] += Si[2 * n] * G[n];
                    out[2 * n + 1] += Si[2 * n + 1] * G[n];
                }
            }
        }
        free(G);
    }
    return err ? -1 : skipped;
}

/* Gradient of G^(n) with respect to the field point (r, x = z - z1) from the paper's first-order
 * derivative relations (potential gradients):
 *   dG^n/dx = (n - 1/2) [ (G^n + G^{n-1}) x / rho_+^2 + (G^n - G^{n-1}) x / rho_-^2 ]
 *   dG^n/dr = -G^n/(2r) + (n - 1/2) (r^2 - r1^2 - x^2)/(2r)
 *             [ (G^n + G^{n-1}) / rho_+^2 + (G^n - G^{n-1}) / rho_-^2 ]
 * with G^{-1} == G^{1}. */
int or_greens_grad(double r, double r1, double x, int nmax, int miller, double *G, double *dGr,
                   double *dGx)
{
    int Ni = nmax > 1 ? nmax : 1;
    double *Gi = (double *)malloc(sizeof(double) * (Ni + 1));
    if (!Gi) return -1;
    if (or_greens(r, r1, x, Ni, miller, Gi) != 0) {
        free(Gi);
        return -1;
    }
    double rp2 = (r + r1) * (r + r1) + x * x, rm2 = (r - r1) * (r - r1) + x * x;
    double u = (r * r - r1 * r1 - x * x) / (2.0 * r);
    for (int n = 0; n <= nmax; ++n) {
        double gn = Gi[n], gm = Gi[n == 0 ? 1 : n - 1];
        double sp = (gn + gm) / rp2, sm = (gn - gm) / rm2;
        G[n] = gn;
        dGx[n] = (n - 0.5) * x * (sp + sm);
        dGr[n] = -gn / (2.0 * r) + (n - 0.5) * u * (sp + sm);
    }
    free(Gi);
    return 0;
}

/* Direct sum with the field gradients dPhi/dr, dPhi/dz (each [nf][nmodes] complex). */
int64_t or_direct_grad(const double *sr, const double *sz, const double *S, int64_t ns,
                       const double *fr, const double *fz, int64_t nf, int nmodes, int miller,
                       int exclude_coincident, double *Phi, double *dPr, double *dPz,
                       int nthreads)
{
    if (nmodes < 1) return -1;
    int64_t skipped = 0;
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel reduction(+ : skipped) reduction(| : err)
    {
        double *G = (double *)malloc(sizeof(double) * 3 * nmodes);
        double *Gr = G + nmodes, *Gx = Gr + nmodes;
#pragma omp for schedule(dynamic, 16)
        for (int64_t j = 0; j < nf; ++j) {
            double *o = Phi + 2 * (size_t)j * nmodes, *orr = dPr + 2 * (size_t)j * nmodes;
            double *oz = dPz + 2 * (size_t)j * nmodes;
            memset(o, 0, sizeof(double) * 2 * nmodes);
            memset(orr, 0, sizeof(double) * 2 * nmodes);
            memset(oz, 0, sizeof(double) * 2 * nmodes);
            for (int64_t i = 0; i < ns; ++i) {
                if (sr[i] == fr[j] && sz[i] == fz[j]) {
                    if (exclude_coincident) {
                        ++skipped;
                        continue;
                    }
                    err = 1;
                    continue;
                }
                if (or_greens_grad(fr[j], sr[i], fz[j] - sz[i], nmodes - 1, miller, G, Gr, Gx) != 0) {
                    err = 1;
                    continue;
                }
                const double *Si = S + 2 * (size_t)i * nmodes;
                for (int n = 0; n < nmodes; ++n) {
                    o[2 * n] += Si[2 * n] * G[n];
                    o[2 * n + 1] += Si[2 * n + 1] * G[n];
                    orr[2 * n] += Si[2 * n] * Gr[n];
                    orr[2 * n + 1] += Si[2 * n + 1] * Gr[n];
                    oz[2 * n] += Si[2 * n] * Gx[n];
                    oz[2 * n + 1] += Si[2 * n + 1] * Gx[n];
                }
            }
        }
        free(G);
    }
    return err ? -1 : skipped;
}
