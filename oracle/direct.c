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
