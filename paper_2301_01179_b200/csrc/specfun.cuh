// specfun.cuh -- device FP64 modal ring Green's function G^(n) = Q_{n-1/2}(chi)/(2 pi sqrt(r r1))
// for n = 0..N, written for sm_100a.  Product code: shares nothing with oracle/.
//
// Method (the paper's, App. A), re-arranged for the GPU:
//  * K, E of modulus k = mu (R#1) from the complementary modulus k' = rho_- / rho_+ (R#2): on the
//    forward branch (k'^2 <= 0.004) by the small-k' series of DLMF 19.12.1-2 (ke_small), on the
//    Miller branch by the arithmetic-geometric mean (the oracle uses Carlson's R_F/R_D instead:
//    independent code):
//      K = pi / (2 AGM(1, k')),  E = K (1 - sum_{m>=0} 2^{m-1} c_m^2),  c_0^2 = k^2 = 4 r r1/rho_+^2.
//    With mu/(2 pi sqrt(r r1)) = 1/(pi rho_+):  G^(0) = 1/(2 a_inf rho_+),
//    G^(1) = G^(0) ((1+chi) s - 1)   (from Q_{1/2} = chi mu K - (1+chi) mu E).
//  * chi - 1 < t_N (tested as rho_-^2 < 2 t_N r r1; the paper's t = 0.008 for N <= 16 and in the
//    paper mode, narrowed for larger N so the forward rounding growth lambda^2N <= 2^6, R#3):
//    forward three-term recursion
//    (2n-1) G_n = 4(n-1) chi G_{n-1} - (2n-3) G_{n-2}, run on u_n = G_n / R_n with
//    R_n = prod_{k<=n} 4(k-1)/(2k-1): u_n = chi u_{n-1} - eps_n u_{n-2}, evaluated as
//    u_{n-1} - eps_n u_{n-2} + (chi - 1) u_{n-1} with chi - 1 = rho_-^2 / (2 r r1) (two DFMA;
//    R#24: on this branch chi - 1 < 0.008 and a rounded chi loses its low bits, which cost 7e-13
//    of G^(64) at chi - 1 = 6e-9; this form keeps 3e-14).
//  * chi >= 1.008: Miller's backward recursion from seeds (0, 1) at (S, S-1), run on
//    the rescaled minimal solution y_n = Q~_n (2 chi)^n, which changes by at most a factor 2 per
//    step (no overflow for any chi, unlike Q~_n itself, R#5), and w_n = y_n / P_n with
//    P_{n-2} = alpha_n P_{n-1}: w_{n-2} = w_{n-1} - delta_n q w_n, q = 1/(4 chi^2).  Then
//    G_n = G_0 * (w_n P_n (2 chi)^-n) / w_0.  Start index: paper mode S = N + 80; accurate mode
//    S = N + ceil(20 / ln lambda) + 4, lambda = chi + sqrt(chi^2 - 1) (contamination
//    lambda^{-2(S-n)} < e^-40), taken as the max over the Miller lanes of a warp so the loop is
//    warp-uniform and the coefficient tables are read by uniform index.  Long recurrences
//    (chi -> 1) are renormalised by a power of two every 64 steps (exact; y_n shrinks by at
//    most 2 per step).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cyl {

constexpr int kMaxModes = 256;   // CYLFMM_MAX_MODES
constexpr int kMaxSteps = 4096;  // Miller start index bound
constexpr double kPi = 3.141592653589793238462643383279502884;

constexpr int kKESeries = 8;      // terms of the small-k' series of K and E (forward branch)

struct RecTables {
    double delta[kMaxSteps + 2];   // Miller: delta_n = beta_n / (alpha_n alpha_{n+1}), n >= 2
    double Pn[kMaxModes + 2];      // Miller: P_n
    double eps[kMaxModes + 2];     // forward: eps_n = b_n R_{n-2} / R_n, n >= 2
    double Rn[kMaxModes + 2];      // forward: R_n
    // K = L P1(k'^2) + P2(k'^2),  E = 1 + k'^2 (L P3(k'^2) + P4(k'^2)),  L = ln(1/k')
    double ke[4][kKESeries];
    // far branch (chi >= kFarChi): A_n = Gamma(n+1/2)/(2 sqrt(pi) Gamma(n+1)) and the term ratios
    // of 2F1((2n+1)/4, (2n+3)/4; n+1; 1/chi^2)
    double farA[kMaxModes + 2];
    double farT[kMaxModes + 2][4];
    // the near-field kernel accumulates every branch in forward units u_n = G_n / R_n and
    // multiplies by R_n once per (target, mode) at the end: the far and Miller factors carry
    // the 1 / R_n (one multiply fewer per forward pair and mode)
    double farAR[kMaxModes + 2];   // farA_n / R_n
    double PnR[kMaxModes + 2];     // P_n / R_n
};
constexpr double kFarChi = 1.0e3;        // far branch from chi = 1000 (4 hypergeometric terms)
__constant__ RecTables c_rec;

// Host-side construction of the recursion constants (exact rationals rounded once).
inline void build_rec_tables(RecTables *t)
{
    auto alpha = [](int n) { return 2.0 * (n - 1) / (2.0 * n - 3.0); };  // n >= 2
    auto beta = [](int n) { return (2.0 * n - 1.0) / (2.0 * n - 3.0); };
    for (int n = 0; n < kMaxSteps + 2; ++n)
        t->delta[n] = n >= 2 ? beta(n) / (alpha(n) * alpha(n + 1)) : 0.0;
    t->Pn[0] = 1.0;
    for (int m = 0; m + 1 < kMaxModes + 2; ++m) t->Pn[m + 1] = t->Pn[m] / alpha(m + 2);
    auto a = [](int n) { return 4.0 * (n - 1) / (2.0 * n - 1.0); };       // n >= 2
    auto b = [](int n) { return (2.0 * n - 3.0) / (2.0 * n - 1.0); };
    t->Rn[0] = 1.0;
    t->Rn[1] = 1.0;
    for (int n = 2; n < kMaxModes + 2; ++n) t->Rn[n] = a(n) * t->Rn[n - 1];
    t->eps[0] = t->eps[1] = 0.0;
    for (int n = 2; n < kMaxModes + 2; ++n) t->eps[n] = b(n) * t->Rn[n - 2] / t->Rn[n];
    // small-k' expansions of the complete elliptic integrals (DLMF 19.12.1-2):
    //   K = sum_m [(1/2)_m / m!]^2 k'^{2m} (L + d_m),
    //   E = 1 + 1/2 sum_m (1/2)_m (3/2)_m / ((2)_m m!) k'^{2m+2} (L + d_m - 1/((2m+1)(2m+2))),
    //   d_0 = 2 ln 2, d_{m+1} = d_m - 1/((m+1)(2m+1))   (long double, rounded once)
    long double am = 1.0L, bm = 1.0L, dm = 2.0L * logl(2.0L);
    for (int m = 0; m < kKESeries; ++m) {
        t->ke[0][m] = (double)(am * am);
        t->ke[1][m] = (double)(am * am * dm);
        t->ke[2][m] = (double)(0.5L * am * bm);
        t->ke[3][m] = (double)(0.5L * am * bm * (dm - 1.0L / ((2.0L * m + 1.0L) * (2.0L * m + 2.0L))));
        am *= (m + 0.5L) / (m + 1.0L);
        bm *= (m + 1.5L) / (m + 2.0L);
        dm -= 1.0L / ((m + 1.0L) * (2.0L * m + 1.0L));
    }
    long double A = 0.5L;
    for (int n = 0; n < kMaxModes + 2; ++n) {
        if (n > 0) A *= (n - 0.5L) / n;
        t->farA[n] = (double)A;
        const long double a = (2.0L * n + 1.0L) / 4.0L, b = (2.0L * n + 3.0L) / 4.0L, c = n + 1.0L;
        for (int k = 0; k < 4; ++k)
            t->farT[n][k] = (double)((a + k) * (b + k) / ((c + k) * (k + 1.0L)));
    }
    for (int n = 0; n < kMaxModes + 2; ++n) {
        t->farAR[n] = t->farA[n] / t->Rn[n];
        t->PnR[n] = t->Pn[n] / t->Rn[n];
    }
}

// Reciprocal and (reciprocal) square root of a positive normal double: the SFU's approximation
// (rcp/rsqrt.approx.f64, ~2^-23 relative) refined by two Newton steps in FMA form (each squares
// the relative error), so the result is within an ulp or two of the correctly rounded value.
// Unlike the IEEE-conforming operators these have no special-case branches; the near-field
// kernel uses them for values that are positive and finite by construction.
__device__ __forceinline__ double rcp_nr(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x)
{
    double y;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    double e = fma(-h * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-h * y, y, 0.5);
    return fma(y, e, y);
}
__device__ __forceinline__ double sqrt_nr(double x)
{
    const double y = rsqrt_nr(x);
    const double s = x * y;
    return fma(fma(-s, s, x), 0.5 * y, s);
}

// ln x for positive normal finite x (the near field's forward pairs: k'^2 in (0, 0.004]):
// x = 2^e m with m in [1/sqrt 2, sqrt 2), ln m = 2 atanh(s) = 2 s sum_k s^2k / (2k+1),
// s = (m - 1)/(m + 1), |s| <= 0.1716 (13 terms: truncation < 1e-18); e ln 2 in two parts.
// Within 3.3e-16 relative of the exact log over (1e-30, 2) (25k points against 40-digit
// values); about half the instructions of the library log, which took 9% of the first
// near-field window's stall samples at C5.
__device__ __forceinline__ double log_pos(double x)
{
    const int hi = __double2hiint(x), lo = __double2loint(x);
    int ex = ((hi >> 20) & 0x7ff) - 1023;
    double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);   // [1, 2)
    const bool big = m > 1.4142135623730951;
    m = big ? 0.5 * m : m;
    ex += big ? 1 : 0;
    const double s = (m - 1.0) * rcp_nr(m + 1.0), s2 = s * s;
    double q = 1.0 / 25.0;
#pragma unroll
    for (int k = 11; k >= 0; --k) q = fma(q, s2, 1.0 / (2 * k + 1));
    const double e = (double)ex;
    return fma(e, 0x1.62e42fefa3800p-1, fma(e, 5.497923018708371e-14, 2.0 * s * q));
}

// K(k) and E(k) for small k'^2 = 1 - k^2 (forward branch: k'^2 <= t/(2+t) <= 0.004, truncation
// after kKESeries terms < 4e-20 relative); replaces the AGM there (one log, 4 short Horner sums).
__device__ __forceinline__ void ke_small(double kp2, double &K, double &E)
{
    const double L = -0.5 * log_pos(kp2);
    double p1 = c_rec.ke[0][kKESeries - 1], p2 = c_rec.ke[1][kKESeries - 1];
    double p3 = c_rec.ke[2][kKESeries - 1], p4 = c_rec.ke[3][kKESeries - 1];
#pragma unroll
    for (int m = kKESeries - 2; m >= 0; --m) {
        p1 = fma(p1, kp2, c_rec.ke[0][m]);
        p2 = fma(p2, kp2, c_rec.ke[1][m]);
        p3 = fma(p3, kp2, c_rec.ke[2][m]);
        p4 = fma(p4, kp2, c_rec.ke[3][m]);
    }
    K = fma(L, p1, p2);
    E = fma(kp2, fma(L, p3, p4), 1.0);
}

// Pair geometry shared by both branches.
struct PairGeo {
    double rp2, rm2;   // rho_+^2, rho_-^2
    double rr1;        // r * r1
    bool forward;      // chi < 1.008
    bool far;          // chi >= kFarChi: hypergeometric series in 1/chi^2 (greens_far)
    bool coincident;   // rho_-^2 == 0 (bitwise-equal rings)
};

// Host: the 2 t_N of the forward/backward switch (R#3), see the header comment.
inline double forward_coef(int nmax, int miller)
{
    double t = 0.008;
    if (miller != 1 && nmax > 0) {
        double c = cosh(log(64.0) / (2.0 * nmax)) - 1.0;
        if (c < t) t = c;
    }
    return 2.0 * t;
}

__device__ __forceinline__ PairGeo pair_geo(double r, double r1, double x, double fwd2)
{
    PairGeo g;
    double dp = r + r1, dm = r - r1;
    g.rp2 = fma(dp, dp, x * x);
    g.rm2 = fma(dm, dm, x * x);
    g.rr1 = r * r1;
    g.forward = g.rm2 < fwd2 * g.rr1;    // chi - 1 < t_N, tie goes backward (R#3)
    g.far = g.rm2 >= 2.0 * (kFarChi - 1.0) * g.rr1;
    g.coincident = !(g.rm2 > 0.0);
    return g;
}

// Accurate-mode Miller start offset e(chi) (evaluated in FP32 with a margin: it only has to be
// large enough).  chi - 1 = rho_-^2 / (2 r r1).
__device__ __forceinline__ int miller_extra(const PairGeo &g, int miller_mode)
{
    if (miller_mode == 1) return 80;
    float cm1 = (float)(g.rm2 / (2.0 * g.rr1));
    float lam_m1 = cm1 + sqrtf(cm1 * (cm1 + 2.0f));     // lambda - 1
    float lnl = log1pf(lam_m1);
    int e = (int)ceilf(20.0f / lnl) + 4;
    return min(e, kMaxSteps - kMaxModes - 4);
}

// AGM(1, k') with the E sum.  Returns a_inf; s = sum_{m>=0} 2^{m-1} c_m^2 when need_e.
__device__ __forceinline__ double agm(double kp, double k2, bool need_e, double &s)
{
    double a = 1.0, b = kp, pw = 0.5;
    s = 0.5 * k2;
#pragma unroll 1
    for (int it = 0; it < 40; ++it) {
        double c = 0.5 * (a - b);
        if (!(fabs(c) > 2.0e-16 * a)) break;
        double an = 0.5 * (a + b);
        b = sqrt(a * b);
        a = an;
        if (need_e) {
            pw *= 2.0;
            s = fma(pw * c, c, s);
        }
    }
    return a;
}

// Far pairs (chi >= 1000, e.g. a ring near the axis seen from a neighbouring ring): the
// hypergeometric form of Q_nu (DLMF 14.3.7) with nu = n - 1/2,
//   G^(n) = A_n q^n F_n(4 q^2) / sqrt(r^2 + r1^2 + x^2),  q = 1/(2 chi) = r r1 / (r^2 + r1^2 + x^2),
//   F_n(z) = 2F1((2n+1)/4, (2n+3)/4; n+1; z), four terms (relative truncation < 2e-17 for
//   z <= 4e-6, n <= 256); the same function the Miller recursion evaluates, without
//   its loop.  q^n underflows to 0 for the highest modes of very distant pairs (correct).
__device__ __forceinline__ void greens_far(const PairGeo &g, int m0, int m1, double *out, int ostride)
{
    const double sum2 = 0.5 * (g.rp2 + g.rm2);
    const double q = g.rr1 / sum2, z = 4.0 * q * q;
    double qn = 1.0 / sqrt(sum2);
    for (int n = 0; n < m1; ++n) {
        if (n > 0) qn *= q;
        if (n >= m0) {
            double t = z * c_rec.farT[n][3];
            t = z * c_rec.farT[n][2] * (1.0 + t);
            t = z * c_rec.farT[n][1] * (1.0 + t);
            t = z * c_rec.farT[n][0] * (1.0 + t);
            out[(n - m0) * ostride] = c_rec.farA[n] * qn * (1.0 + t);
        }
    }
}

// G^(n)(r, r1, x) for n = 0..m1-1, stored to out[(n - m0) * ostride] for n in [m0, m1).
// S_warp: Miller start index (only used on the backward branch; must be > m1 and >= 2).
// The pair must not be coincident.  Out may point to shared or global memory.
__device__ __forceinline__ void greens_pair(const PairGeo &g, int m0, int m1, int S_warp,
                                            double *out, int ostride)
{
    if (g.far) {
        greens_far(g, m0, m1, out, ostride);
        return;
    }
    double rho_p = sqrt(g.rp2);
    double inv_rho_p = 1.0 / rho_p;
    double sum2 = 0.5 * (g.rp2 + g.rm2);                    // r^2 + r1^2 + x^2 = 2 chi r r1
    if (g.forward) {
        // K, E from the small-k' series (k'^2 = rho_-^2 / rho_+^2 <= 0.004 here)
        double Kk, Ek;
        ke_small(g.rm2 * inv_rho_p * inv_rho_p, Kk, Ek);
        const double G0 = Kk * inv_rho_p * (1.0 / kPi);     // K / (pi rho_+)
        double chi = 0.5 * sum2 / g.rr1;
        const double dchi = 0.5 * g.rm2 / g.rr1;             // chi - 1 (R#24)
        // G^(1) / G^(0) = Q_{1/2}/Q_{-1/2} = chi - (1 + chi) E/K
        double u0 = G0, u1 = G0 * fma(-(1.0 + chi), Ek / Kk, chi);
        if (m0 == 0 && m1 > 0) out[0] = u0;
        if (m0 <= 1 && m1 > 1) out[(1 - m0) * ostride] = u1;
#pragma unroll 4
        for (int n = 2; n < m1; ++n) {
            double u2 = fma(dchi, u1, fma(-c_rec.eps[n], u0, u1));
            if (n >= m0) out[(n - m0) * ostride] = u2 * c_rec.Rn[n];
            u0 = u1;
            u1 = u2;
        }
        return;
    }
    double kp = sqrt(g.rm2) * inv_rho_p;                   // k'
    double k2 = 4.0 * g.rr1 * inv_rho_p * inv_rho_p;       // k^2 = 1 - k'^2 (no cancellation)
    double s;
    double a = agm(kp, k2, false, s);
    double G0 = 0.5 * inv_rho_p / a;                        // K / (pi rho_+)
    // Miller, on w_n (see header).  wn = w_n, wl = w_{n-1}; step produces w_{n-2}.
    double inv2chi = g.rr1 / sum2;
    double q = inv2chi * inv2chi;
    double wn = 0.0, wl = 1.0;
    int n = S_warp;
    // phase A: indices S-2 .. m1 (no store), renormalised every 64 steps
    while (n > m1 + 1) {
        const int nstop = max(m1 + 1, n - 64);
#pragma unroll 4
        for (; n > nstop; --n) {
            double w = fma(-c_rec.delta[n] * q, wn, wl);
            wn = wl;
            wl = w;
        }
        int ex;
        frexp(wl, &ex);
        wn = ldexp(wn, -ex);
        wl = ldexp(wl, -ex);
    }
    // here wl = w_{n-1} with n-1 = m1-1 (or the seed if S-1 == m1-1); store window values
    if (n - 1 >= m0 && n - 1 < m1) out[(n - 1 - m0) * ostride] = wl;
#pragma unroll 4
    for (; n >= 2; --n) {
        double w = fma(-c_rec.delta[n] * q, wn, wl);
        wn = wl;
        wl = w;
        if (n - 2 >= m0) out[(n - 2 - m0) * ostride] = w;
    }
    // wl = w_0.  Normalise and apply P_n (2 chi)^-n upward (v underflows to 0 correctly).
    double c = G0 / wl;
    double v = 1.0;
    for (int k = 0; k < m1; ++k) {
        if (k >= m0) {
            double *o = out + (k - m0) * ostride;
            *o = (*o) * c_rec.Pn[k] * c * v;
        }
        v *= inv2chi;
    }
}

}  // namespace cyl
