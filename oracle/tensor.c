/*
 * tensor.c -- oracle derivative tensor Gbar^n_{abc} = 1/(a! b! c!) d^{a+b+c} G^(n) / dr^a dr1^b dx^c
 * (P:876-902).  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Steps, in the paper's order (Appendix A):
 *   1. G^(n), n = 0..max(N,1)  (G^(-1) == G^(1) for n = 0).
 *   2. x-derivatives Gbar_{00,c}, c <= 2p (reading R#22):
 *      a. modes n = 0, 1 by the paper's x-recursion from (Gbar^n +- Gbar^{n-1}) d^q/dx^q
 *         (x/rho_+-^2) (G^(-1) == G^(1));
 *      b. modes n >= 2 by the three-term recursion applied to the Taylor series in
 *         Delta x: chi(x + Delta) = chi + (x/(r r1)) Delta + Delta^2/(2 r r1) exactly, so
 *         (2n-1) g_n = 4(n-1) chi(Delta) g_{n-1} - (2n-3) g_{n-2} holds coefficient-wise
 *         (truncated series products).  Forward from g_0, g_1 on the paper's forward branch
 *         (R#3); on the backward branch Miller's algorithm in ratio form
 *         rho_n = g_n / g_{n-1}: rho_S = 0, rho_{n-1} = (2n-3) / (4(n-1) chi(Delta) - (2n-1) rho_n)
 *         (series reciprocal), then g_n = g_{n-1} rho_n.  Start S = N + e with e from R#4
 *         applied to the worst point of the unit disk in Delta (the Taylor coefficients must be
 *         converged over the S2L offsets |Delta| <= 1, not only at Delta = 0).
 *      The paper's cross-mode x-recursion for all n multiplies rounding errors by about
 *      (n - 1/2)/(k+1) per order when n > k (measured: relative error 4e1 at n = 64, p = 16),
 *      while the series recursion is as stable as the recursion for G itself.
 *   3. r-derivatives Gbar_{10k}.
 *   4. r1-derivatives Gbar_{01k} by exchanging r and r1.
 *   5. mixed Gbar_{11k}.
 *   6. Gbar_{a+2,b,c} for b in {0,1} from the cylindrical Laplace equation in (r, x)
 *      (P:1027-1065), then Gbar_{a,b+2,c} from the same equation in (r1, x) ("switching r and
 *      r1").  The printed recursion P:1046-1061 omits the axial term; we use the
 *      Laplace equation itself, multiplied by r^2 and expanded in Taylor coefficients (R#6):
 *        r^2 (a+1)(a+2) G_{a+2} + r (a+1)(2a+1) G_{a+1} + (a^2 - n^2) G_a
 *          + (c+1)(c+2) [ r^2 G_{a,c+2} + 2 r G_{a-1,c+2} + G_{a-2,c+2} ] = 0.
 * The Taylor coefficients of the rational kernels, which the paper uses but does not give, are
 * written from z_+- = 1/(x - i a_+-), a_+- = r +- r1 (R#7):
 *   x/rho^2 = Re z,  (r^2-r1^2-x^2)/rho^2 = -1 + 2 r Im z,  d/dr1 of the latter = +-2 r Re z^2,
 *   and the q-th Taylor coefficient of z^m in x is (-1)^q C(q+m-1, q) z^{m+q}.
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

/* Taylor coefficients (1/q!) d^q/dx^q of the kernels, q = 0..qmax. */
void or_rational_tables(double r, double r1, double x, int qmax, double *out)
{
    int Q = qmax + 1;
    double *tp = out, *tm = out + Q, *up = out + 2 * Q, *um = out + 3 * Q;
    double *vp = out + 4 * Q, *vm = out + 5 * Q, *sp = out + 6 * Q, *sm = out + 7 * Q;
    double a[2] = {r + r1, r - r1};    /* a_+, a_- */
    double as[2] = {r1 + r, r1 - r};   /* exchanged r <-> r1 */
    for (int s = 0; s < 2; ++s) {
        double complex z = 1.0 / (x - I * a[s]);
        double complex zs = 1.0 / (x - I * as[s]);
        double complex w = z;   /* (-1)^q z^{q+1} */
        double complex ws = zs;
        for (int q = 0; q <= qmax; ++q) {
            double complex w2 = w * z; /* (-1)^q z^{q+2} */
            double *t = s ? tm : tp, *u = s ? um : up, *v = s ? vm : vp, *us = s ? sm : sp;
            t[q] = creal(w);
            u[q] = (q == 0 ? -1.0 : 0.0) + 2.0 * r * cimag(w);
            v[q] = (s ? -1.0 : 1.0) * 2.0 * r * (q + 1) * creal(w2);
            us[q] = (q == 0 ? -1.0 : 0.0) + 2.0 * r1 * cimag(ws);
            w = -w * z;
            ws = -ws * zs;
        }
    }
}

#define T4(n, a, b, c) out[(((size_t)(n) * (p + 1) + (a)) * (p + 1) + (b)) * (2 * p + 1) + (c)]

int or_tensor(double r, double r1, double x, int nmax, int p, int miller, double *out)
{
    if (nmax < 0 || p < 1) return -1;
    int Ni = nmax > 1 ? nmax : 1; /* internal modes 0..Ni (mode 1 needed for n = 0) */
    int C = 2 * p;                /* maximum x order */
    int Q = C + 2;
    double *G = (double *)malloc(sizeof(double) * (Ni + 1));
    double *tab = (double *)malloc(sizeof(double) * 8 * Q);
    double *g00 = (double *)calloc((size_t)(Ni + 1) * (C + 1), sizeof(double));
    double *g10 = (double *)calloc((size_t)(Ni + 1) * (C + 1), sizeof(double));
    double *g01 = (double *)calloc((size_t)(Ni + 1) * (C + 1), sizeof(double));
    double *g11 = (double *)calloc((size_t)(Ni + 1) * (C + 1), sizeof(double));
    int rc = -1;
    if (!G || !tab || !g00 || !g10 || !g01 || !g11) goto done;
    if (or_greens(r, r1, x, Ni, miller, G) != 0) goto done;
    or_rational_tables(r, r1, x, Q - 1, tab);
    const double *tp = tab, *tm = tab + Q, *up = tab + 2 * Q, *um = tab + 3 * Q;
    const double *vp = tab + 4 * Q, *vm = tab + 5 * Q, *sp = tab + 6 * Q, *sm = tab + 7 * Q;
#define A(arr, n, c) arr[(size_t)(n) * (C + 1) + (c)]
    /* step 2a: x-derivatives of modes 0 and 1, order by order */
    A(g00, 0, 0) = G[0];
    A(g00, 1, 0) = G[1];
    for (int k = 0; k < C; ++k) {
        for (int n = 0; n <= 1; ++n) {
            int m = 1 - n; /* n = 0: G^(-1) == G^(1); n = 1: mode 0 */
            double s = 0.0;
            for (int q = 0; q <= k; ++q) {
                double gp = A(g00, n, k - q) + A(g00, m, k - q);
                double gm = A(g00, n, k - q) - A(g00, m, k - q);
                s += gp * tp[q] + gm * tm[q];
            }
            A(g00, n, k + 1) = (n - 0.5) * s / (k + 1);
        }
    }
    /* step 2b: modes n >= 2 by the three-term recursion on Taylor series in Delta x (R#22) */
    if (Ni >= 2) {
        const double chi = (r * r + r1 * r1 + x * x) / (2.0 * r * r1);
        double chis[3] = {chi, x / (r * r1), 1.0 / (2.0 * r * r1)}; /* chi(x + Delta) */
        double rho_m2 = (r - r1) * (r - r1) + x * x;
        int forward = rho_m2 < or_forward_coef(Ni, miller) * (r * r1); /* as in or_greens */
        if (forward) {
            for (int n = 2; n <= Ni; ++n)
                for (int c = 0; c <= C; ++c) {
                    double chig = 0.0; /* [chi(Delta) g_{n-1}]_c */
                    for (int j = 0; j <= 2 && j <= c; ++j) chig += chis[j] * A(g00, n - 1, c - j);
                    A(g00, n, c) = (4.0 * (n - 1) * chig - (2.0 * n - 3.0) * A(g00, n - 2, c)) /
                                   (2.0 * n - 1.0);
                }
        } else {
            /* start: the contamination lambda^{-2(S-n)} must be small over the whole disk
             * |Delta| <= rho_-/2 whose Taylor coefficients the S2L offsets use (|Delta| <= h and
             * rho_- >= 2h for every S2L pair), not just at Delta = 0 (R#22):
             * e = max(80, ceil(20 / m)), m = min over |Delta| = rho_-/2 of ln|lambda(chi(x + Delta))|
             * (harmonic, so the minimum is on the circle; 256 points) */
            int e = or_miller_extra(chi, miller);
            if (miller != OR_MILLER_PAPER) {
                double m = HUGE_VAL, R = 0.5 * sqrt(rho_m2);
                for (int k = 0; k < 256; ++k) {
                    double complex d = R * cexp(I * (2.0 * M_PI * k / 256.0));
                    double complex z = (r * r + r1 * r1 + (x + d) * (x + d)) / (2.0 * r * r1);
                    double v = fabs(log(cabs(z + csqrt(z * z - 1.0))));
                    if (v < m) m = v;
                }
                double es = ceil(20.0 / m);
                if (es > e) e = (int)es;
            }
            int S = Ni + e;
            double *rho = (double *)calloc((size_t)(C + 1), sizeof(double)); /* rho_S = 0 */
            double *den = (double *)calloc((size_t)(C + 1), sizeof(double));
            double *rat = (double *)calloc((size_t)(Ni + 1) * (C + 1), sizeof(double));
            if (!rho || !den || !rat) {
                free(rho);
                free(den);
                free(rat);
                goto done;
            }
            for (int n = S; n >= 2; --n) {
                /* den = 4(n-1) chi(Delta) - (2n-1) rho_n ; rho_{n-1} = (2n-3) / den */
                for (int c = 0; c <= C; ++c)
                    den[c] = (c <= 2 ? 4.0 * (n - 1) * chis[c] : 0.0) - (2.0 * n - 1.0) * rho[c];
                for (int c = 0; c <= C; ++c) { /* series reciprocal, triangular */
                    double s = (c == 0) ? (2.0 * n - 3.0) : 0.0;
                    for (int j = 0; j < c; ++j) s -= rho[j] * den[c - j];
                    rho[c] = s / den[0];
                }
                if (n - 1 <= Ni)
                    for (int c = 0; c <= C; ++c) A(rat, n - 1, c) = rho[c];
            }
            for (int n = 2; n <= Ni; ++n) /* g_n = g_{n-1} rho_n */
                for (int c = 0; c <= C; ++c) {
                    double s = 0.0;
                    for (int j = 0; j <= c; ++j) s += A(g00, n - 1, j) * A(rat, n, c - j);
                    A(g00, n, c) = s;
                }
            free(rho);
            free(den);
            free(rat);
        }
    }
    /* steps 3, 4: r- and r1-derivatives */
    for (int n = 0; n <= Ni; ++n) {
        int m = n == 0 ? 1 : n - 1;
        for (int k = 0; k < C; ++k) {
            double s1 = 0.0, s2 = 0.0;
            for (int q = 0; q <= k; ++q) {
                double gp = A(g00, n, k - q) + A(g00, m, k - q);
                double gm = A(g00, n, k - q) - A(g00, m, k - q);
                s1 += gp * up[q] + gm * um[q];
                s2 += gp * sp[q] + gm * sm[q];
            }
            A(g10, n, k) = -A(g00, n, k) / (2.0 * r) + (n - 0.5) / (2.0 * r) * s1;
            A(g01, n, k) = -A(g00, n, k) / (2.0 * r1) + (n - 0.5) / (2.0 * r1) * s2;
        }
    }
    /* step 5: mixed derivative */
    for (int n = 0; n <= Ni; ++n) {
        int m = n == 0 ? 1 : n - 1;
        for (int k = 0; k < C - 1; ++k) {
            double s = 0.0;
            for (int q = 0; q <= k; ++q) {
                double gp = A(g00, n, k - q) + A(g00, m, k - q);
                double gm = A(g00, n, k - q) - A(g00, m, k - q);
                double hp = A(g01, n, k - q) + A(g01, m, k - q);
                double hm = A(g01, n, k - q) - A(g01, m, k - q);
                s += gp * vp[q] + hp * up[q] + gm * vm[q] + hm * um[q];
            }
            A(g11, n, k) = -A(g01, n, k) / (2.0 * r) + (n - 0.5) / (2.0 * r) * s;
        }
    }
    /* step 6: seeds into the dense tensor, then the Laplace recursions */
    memset(out, 0, sizeof(double) * (size_t)(nmax + 1) * (p + 1) * (p + 1) * (2 * p + 1));
    for (int n = 0; n <= nmax; ++n) {
        for (int c = 0; c <= C; ++c) T4(n, 0, 0, c) = A(g00, n, c);
        for (int c = 0; c <= C - 1; ++c) {
            T4(n, 1, 0, c) = A(g10, n, c);
            T4(n, 0, 1, c) = A(g01, n, c);
        }
        for (int c = 0; c <= C - 2; ++c) T4(n, 1, 1, c) = A(g11, n, c);
        double n2 = (double)n * n;
        for (int b = 0; b <= 1; ++b)
            for (int a = 0; a + 2 <= p; ++a)
                for (int c = 0; a + 2 + b + c <= C; ++c) {
                    double lap = r * r * T4(n, a, b, c + 2);
                    if (a >= 1) lap += 2.0 * r * T4(n, a - 1, b, c + 2);
                    if (a >= 2) lap += T4(n, a - 2, b, c + 2);
                    double num = r * (a + 1) * (2.0 * a + 1) * T4(n, a + 1, b, c)
                                 + (a * (double)a - n2) * T4(n, a, b, c) + (c + 1.0) * (c + 2.0) * lap;
                    T4(n, a + 2, b, c) = -num / (r * r * (a + 1.0) * (a + 2.0));
                }
        for (int b = 0; b + 2 <= p; ++b)
            for (int a = 0; a <= p; ++a)
                for (int c = 0; a + b + 2 + c <= C; ++c) {
                    double lap = r1 * r1 * T4(n, a, b, c + 2);
                    if (b >= 1) lap += 2.0 * r1 * T4(n, a, b - 1, c + 2);
                    if (b >= 2) lap += T4(n, a, b - 2, c + 2);
                    double num = r1 * (b + 1) * (2.0 * b + 1) * T4(n, a, b + 1, c)
                                 + (b * (double)b - n2) * T4(n, a, b, c) + (c + 1.0) * (c + 2.0) * lap;
                    T4(n, a, b + 2, c) = -num / (r1 * r1 * (b + 1.0) * (b + 2.0));
                }
    }
#undef A
    rc = 0;
done:
    free(G);
    free(tab);
    free(g00);
    free(g10);
    free(g01);
    free(g11);
    return rc;
}
