/*
 * specfun.c -- oracle special functions: Carlson R_F/R_D, K/E, Q_{n-1/2}, G^(n).
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain FP64 C, no fast-math, no FMA contraction.
 *
 *  - K, E "computed using the method of Carlson": K = R_F(0,k'^2,1),
 *    E = R_F(0,k'^2,1) - (k^2/3) R_D(0,k'^2,1), written from Carlson's duplication algorithm
 *    (Carlson 1995, the paper's ref. carlson95) in its own notation.
 *  - Seeds Q_{-1/2} = mu K(mu), Q_{1/2} = chi mu K(mu) - (1+chi) mu E(mu), mu = sqrt(2/(1+chi)),
 *    with mu the MODULUS (reading R#1) and K, E fed the complementary parameter
 *    k'^2 = rho_-^2/rho_+^2 directly (R#2).
 *  - Three-term recursion (2n-3)G^(n-2) = 4(n-1) chi G^(n-1) - (2n-1) G^(n):
 *    forward for chi < 1.008, Miller backward otherwise, start index per R#4,
 *    exact power-of-two rescaling against overflow (R#5).
 *  - G^(n) = Q_{n-1/2}(chi) / (2 pi sqrt(r r1)).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

static double dmax3(double a, double b, double c)
{
    double m = a > b ? a : b;
    return m > c ? m : c;
}

/* Carlson 1995, Algorithm 1: R_F(x,y,z) = 1/2 int_0^inf dt / sqrt((t+x)(t+y)(t+z)). */
double or_carlson_rf(double x, double y, double z)
{
    const double r = ldexp(1.0, -53);
    double A0 = (x + y + z) / 3.0;
    double Q = pow(3.0 * r, -1.0 / 6.0) * dmax3(fabs(A0 - x), fabs(A0 - y), fabs(A0 - z));
    double xm = x, ym = y, zm = z, Am = A0, four_n = 1.0;
    while (four_n * fabs(Am) <= Q) { /* iterate while 4^-m Q > |A_m| */
        double sx = sqrt(xm), sy = sqrt(ym), sz = sqrt(zm);
        double lam = sx * sy + sx * sz + sy * sz;
        Am = (Am + lam) / 4.0;
        xm = (xm + lam) / 4.0;
        ym = (ym + lam) / 4.0;
        zm = (zm + lam) / 4.0;
        four_n *= 4.0;
    }
    double X = (A0 - x) / (four_n * Am);
    double Y = (A0 - y) / (four_n * Am);
    double Z = -(X + Y);
    double E2 = X * Y - Z * Z;
    double E3 = X * Y * Z;
    return (1.0 - E2 / 10.0 + E3 / 14.0 + E2 * E2 / 24.0 - 3.0 * E2 * E3 / 44.0) / sqrt(Am);
}

/* Carlson 1995, Algorithm 4: R_D(x,y,z) = 3/2 int_0^inf dt / ((t+z) sqrt((t+x)(t+y)(t+z))). */
double or_carlson_rd(double x, double y, double z)
{
    const double r = ldexp(1.0, -53);
    double A0 = (x + y + 3.0 * z) / 5.0;
    double Q = pow(r / 4.0, -1.0 / 6.0) * dmax3(fabs(A0 - x), fabs(A0 - y), fabs(A0 - z));
    double xm = x, ym = y, zm = z, Am = A0, four_n = 1.0, sum = 0.0;
    while (four_n * fabs(Am) <= Q) {
        double sx = sqrt(xm), sy = sqrt(ym), sz = sqrt(zm);
        double lam = sx * sy + sx * sz + sy * sz;
        sum += 1.0 / (four_n * sz * (zm + lam));
        Am = (Am + lam) / 4.0;
        xm = (xm + lam) / 4.0;
        ym = (ym + lam) / 4.0;
        zm = (zm + lam) / 4.0;
        four_n *= 4.0;
    }
    double X = (A0 - x) / (four_n * Am);
    double Y = (A0 - y) / (four_n * Am);
    double Z = -(X + Y) / 3.0;
    double E2 = X * Y - 6.0 * Z * Z;
    double E3 = (3.0 * X * Y - 8.0 * Z * Z) * Z;
    double E4 = 3.0 * (X * Y - Z * Z) * Z * Z;
    double E5 = X * Y * Z * Z * Z;
    double series = 1.0 - 3.0 * E2 / 14.0 + E3 / 6.0 + 9.0 * E2 * E2 / 88.0 - 3.0 * E4 / 22.0
                    - 9.0 * E2 * E3 / 52.0 + 3.0 * E5 / 26.0;
    return series / (four_n * Am * sqrt(Am)) + 3.0 * sum;
}

void or_ellip_ke(double kp2, double *K, double *E)
{
    double k2 = 1.0 - kp2;
    double rf = or_carlson_rf(0.0, kp2, 1.0);
    double rd = or_carlson_rd(0.0, kp2, 1.0);
    *K = rf;
    *E = rf - k2 / 3.0 * rd;
}

/* Miller extra steps e in the accurate mode (R#4): the backward recursion started at n = N+e
 * contaminates Q_{n-1/2} by ~lambda^{-2(N+e-n)}, lambda = chi + sqrt(chi^2 - 1); we take
 * e = max(80, ceil(20 / ln lambda)) so that the contamination is below e^-40 ~ 4e-18. */
int or_miller_extra(double chi, int miller)
{
    if (miller == OR_MILLER_PAPER) return 80;
    double lam = chi + sqrt((chi - 1.0) * (chi + 1.0));
    double e = ceil(20.0 / log(lam));
    return e > 80.0 ? (int)e : 80;
}

int or_legendre_q(double chi, double kp2, int forward, int nmax, int miller, double *Q)
{
    if (!(chi > 1.0) || nmax < 0) return -1;
    double K, E;
    or_ellip_ke(kp2, &K, &E);
    double mu = sqrt(2.0 / (1.0 + chi));
    double q0 = mu * K; /* Q_{-1/2} */
    if (forward) {
        /* (2n-1) Q_n = 4(n-1) chi Q_{n-1} - (2n-3) Q_{n-2} with chi = 1 + delta,
         * delta = chi - 1 = 2 k'^2 / (1 - k'^2) from the accurate k'^2 (R#2, R#24): on this branch
         * delta < 0.008 and a rounded chi carries delta to only ~1e-16 / delta relative
         * precision, which cost 4e-13 of Q_{63.5} at delta = 6e-9. */
        const double delta = 2.0 * kp2 / (1.0 - kp2);
        Q[0] = q0;
        if (nmax >= 1) Q[1] = chi * mu * K - (1.0 + chi) * mu * E; /* Q_{1/2} */
        for (int n = 2; n <= nmax; ++n)
            Q[n] = (4.0 * (n - 1) * Q[n - 1] - (2.0 * n - 3.0) * Q[n - 2] +
                    4.0 * (n - 1) * delta * Q[n - 1]) / (2.0 * n - 1.0);
        return 0;
    }
    /* Miller: arbitrary seeds Qt[S] = 0, Qt[S-1] = 1 (R#4), recur down to n = 0. */
    int S = nmax + or_miller_extra(chi, miller);
    double *Qt = (double *)calloc((size_t)S + 1, sizeof(double));
    if (!Qt) return -1;
    Qt[S] = 0.0;
    Qt[S - 1] = 1.0;
    const double big = ldexp(1.0, 600), shrink = ldexp(1.0, -600);
    for (int n = S; n >= 2; --n) {
        Qt[n - 2] = (4.0 * (n - 1) * chi * Qt[n - 1] - (2.0 * n - 1.0) * Qt[n]) / (2.0 * n - 3.0);
        if (fabs(Qt[n - 2]) > big) /* exact rescale of everything computed so far (R#5) */
            for (int m = n - 2; m <= S; ++m) Qt[m] *= shrink;
    }
    double scale = q0 / Qt[0]; /* normalise by the known Q_{-1/2} */
    for (int n = 0; n <= nmax; ++n) Q[n] = Qt[n] * scale;
    free(Qt);
    return 0;
}

/* Forward/backward switch (R#3): the paper's chi < 1.008.  In the accurate mode the
 * forward branch is narrowed for large N so that its rounding growth lambda^{2N} stays below
 * 2^6 (the paper ran N <= 17; for N <= 16 the rule is the paper's): chi - 1 < t_N with
 * t_N = min(0.008, cosh(ln(64) / (2N)) - 1).  Returned as 2 t_N, compared as
 * rho_-^2 < 2 t_N r r1 (chi - 1 = rho_-^2 / (2 r r1)). */
double or_forward_coef(int nmax, int miller)
{
    double t = 0.008;
    if (miller != OR_MILLER_PAPER && nmax > 0) {
        double c = cosh(log(64.0) / (2.0 * nmax)) - 1.0;
        if (c < t) t = c;
    }
    return 2.0 * t;
}

int or_greens(double r, double r1, double x, int nmax, int miller, double *G)
{
    if (!(r > 0.0) || !(r1 > 0.0)) return -1;
    double dm = r - r1, dp = r + r1;
    double rho_m2 = dm * dm + x * x;
    double rho_p2 = dp * dp + x * x;
    if (!(rho_m2 > 0.0)) return -1; /* coincident rings: log singularity */
    double chi = (r * r + r1 * r1 + x * x) / (2.0 * r * r1);
    double kp2 = rho_m2 / rho_p2;
    int forward = rho_m2 < or_forward_coef(nmax, miller) * (r * r1); /* chi - 1 < t_N (R#3) */
    if (or_legendre_q(chi, kp2, forward, nmax, miller, G) != 0) return -1;
    double inv = 1.0 / (2.0 * M_PI * sqrt(r * r1));
    for (int n = 0; n <= nmax; ++n) G[n] *= inv;
    return 0;
}
