// tensor.cuh -- the Green-derivative tensor Gbar^n_{abc} = 1/(a!b!c!) d^{a+b+c}G^(n)/dr^a dr1^b dx^c
// at a geometry (r, r1, x), for a, b <= p and a+b+c <= 2p ("double truncation", R#8).
// Product code (sm_100a); independent of oracle/.
//
// Two kernels:
//  tensor_seed_kernel  (one CTA per geometry): G^(n), n = 0..max(N,1) (specfun.cuh); the Taylor
//     tables of the rational kernels from z_+- = 1/(x - i a_+-) (R#7); the x-derivatives
//     Gbar_{00,c}: modes 0, 1 by the paper's x-recursion (G^(-1) == G^(1)), modes
//     n >= 2 by the three-term recursion on Taylor series in Delta x, forward or Miller-ratio
//     (reading R#22); Gbar_{10k}, Gbar_{01k} and the mixed Gbar_{11k}
//     (P:993-1025).  Output: seeds[geom][4][Ni+1][2p+1].
//  tensor_fill_kernel  (one warp per (geometry, mode), registers and shuffles only): the tensor
//     of one mode from the seeds by the cylindrical Laplace equation in r (b in {0,1}) and in r1
//     (P:1027-1065), with the axial term the printed recursion omits restored (R#6):
//       r^2 (a+1)(a+2) G_{a+2} + r (a+1)(2a+1) G_{a+1} + (a^2 - n^2) G_a
//         + (c+1)(c+2) [ r^2 G_{a,c+2} + 2 r G_{a-1,c+2} + G_{a-2,c+2} ] = 0,
//     parallel over (b, c) per radial step.  Written out dense ([a][b][c], c <= 2p) or packed
//     (c <= 2p-a-b, (p+1)^3 entries: the entries the S2L operator reads, scaled by c!).
#pragma once
#include "specfun.cuh"

namespace cyl {

struct TensorGeomArgs {
    const double *r, *r1, *x;    // explicit geometries (test entry), or nullptr for stations
    int64_t n;                   // number of geometries
    int station_mode;            // 1: geometry g = (i_in, cls) normalised station (see below)
    int n_stations;              // stations: g = i_in * 12 + cls
    int K;                       // modes computed/written: 0..K-1 (window [m0, m1) for fill)
    int m0, m1;
    int p;
    int miller;
    double fwd2;                 // forward switch for N = max(K-1, 1) (R#3)
    double *seeds;               // [n][4][Ni+1][2p+1]
    int seed_m1;                 // fill: modes the seeds were computed for (0: m1)
    double *out;                 // dense [n][m1-m0][p+1][p+1][2p+1] or packed [n][m1-m0][(p+1)^3]
    int packed;
    int *err;
    const int *glist;            // nullable: CTA b works on geometry glist[b] (used stations)
    int64_t nwork;               // fill: (geometry, mode) items
};

// The 12 Green's-expansion classes per radial station: (dI, dJ) in {0..3}^2 with
// max(dI, dJ) >= 2; dI = outer column - inner column, dJ = |z offset| in boxes.
__host__ __device__ inline void station_class(int cls, int &dI, int &dJ)
{
    // order: dI-major over the 16 cells skipping the 4 near ones
    const int tab[12][2] = {{0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 0}, {2, 1},
                            {2, 2}, {2, 3}, {3, 0}, {3, 1}, {3, 2}, {3, 3}};
    dI = tab[cls][0];
    dJ = tab[cls][1];
}
__host__ __device__ inline int class_of(int dI, int dJ)
{
    // inverse of station_class; -1 for the near cells
    if (dI < 2 && dJ < 2) return -1;
    if (dI < 2) return dI * 2 + (dJ - 2);
    return 4 + (dI - 2) * 4 + dJ;
}

__device__ inline void geometry_of(const TensorGeomArgs &a, int64_t g, double &r, double &r1,
                                   double &x)
{
    if (a.station_mode) {
        int i_in = (int)(g / 12), cls = (int)(g % 12), dI, dJ;
        station_class(cls, dI, dJ);
        r1 = i_in + 0.5;          // inner column centre, in units of the box size h
        r = i_in + dI + 0.5;      // outer column centre
        x = (double)dJ;
    } else {
        r = a.r[g];
        r1 = a.r1[g];
        x = a.x[g];
    }
}

// Miller ratio-series recursion with the series in registers (one thread; D = 2p + 1 terms):
// rho_{n-1} = (2n-3) / (4(n-1) chi(Delta) - (2n-1) rho_n), rat[n-1] = rho_{n-1} for n-1 <= Ni.
template <int D>
__device__ __noinline__ void miller_series_regs(int S, int Ni, double chi0, double ch1, double ch2,
                                                double *rat)
{
    double rho[D], den[D];
#pragma unroll
    for (int c = 0; c < D; ++c) rho[c] = 0.0;
    for (int n = S; n >= 2; --n) {
        const double a4 = 4.0 * (n - 1), b2 = 2.0 * n - 1.0;
#pragma unroll
        for (int c = 0; c < D; ++c) den[c] = -b2 * rho[c];
        den[0] = fma(a4, chi0, den[0]);
        den[1] = fma(a4, ch1, den[1]);
        den[2] = fma(a4, ch2, den[2]);
        const double inv = 1.0 / den[0];
        // series reciprocal, right-looking: as soon as rho_j is known its terms go into every
        // later coefficient's sum, so the dependency chain is one FMA and one product per
        // coefficient (the left-looking dot products made it ~c/2 FMAs deep: 4x longer)
        double sacc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) sacc[c] = 0.0;
        rho[0] = (2.0 * n - 3.0) * inv;
#pragma unroll
        for (int j = 0; j + 1 < D; ++j) {
#pragma unroll
            for (int c = j + 1; c < D; ++c) sacc[c] = fma(rho[j], den[c - j], sacc[c]);
            rho[j + 1] = -sacc[j + 1] * inv;
        }
        if (n - 1 <= Ni) {
#pragma unroll
            for (int c = 0; c < D; ++c) rat[(n - 1) * D + c] = rho[c];
        }
    }
}

// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) tensor_seed_kernel(TensorGeomArgs a)
{
    extern __shared__ double sm[];
    const int p = a.p, C = 2 * p, Q = C + 2, D = C + 1;
    const int Nw = a.m1 - 1;                 // highest mode needed
    const int Ni = Nw > 1 ? Nw : 1;          // + mode 1 for n = 0
    const int NM = Ni + 1;
    // shared: G, the tables, g00 and g01 (read by later steps); g10 and g11 go straight to the
    // output (54 KB at p = 16, K = 65: four CTAs per SM instead of two)
    double *G = sm;                          // [NM]
    double *tab = G + NM;                    // 8 tables x Q: tsum tdif usum udif ssum sdif vp vm
    double *g00 = tab + 8 * Q;               // [NM][D]
    double *g01 = g00 + NM * D;
    double *rat = g01 + NM * D;              // [NM][D] Miller ratio series; first the raw tables
    double *raw = rat;                       // [2][4][Q] (consumed before the Miller step)
    double *rho = rat + (NM * D > 8 * Q ? NM * D : 8 * Q);   // [D]
    double *den = rho + D;                                   // [D + 4]
    int *sS = reinterpret_cast<int *>(den + D + 4);          // [2]
    const int64_t gi = a.glist ? a.glist[blockIdx.x] : blockIdx.x;
    double r, r1, x;
    geometry_of(a, gi, r, r1, x);
    const int tid = threadIdx.x;
    if (!(r > 0.0) || !(r1 > 0.0)) {
        if (tid == 0) atomicOr(a.err, 2);
        return;
    }
    PairGeo geo = pair_geo(r, r1, x, a.fwd2);
    if (geo.coincident) {
        if (tid == 0) atomicOr(a.err, 1);
        return;
    }
    if (tid < 32) {
        int S_lane = geo.forward ? 0 : (a.K - 1 > Ni ? a.K - 1 : Ni) + miller_extra(geo, a.miller);
        if (tid == 0) greens_pair(geo, 0, NM, S_lane, G, 1);
    } else if (tid < 34) {
        // Taylor coefficients in x of the rational kernels (R#7), sign s: a_s = r +- r1.
        int s = tid - 32;
        double as = s == 0 ? r + r1 : r - r1;     // a_+-
        double bs = s == 0 ? r1 + r : r1 - r;     // exchanged r <-> r1
        double den = x * x + as * as, dens = x * x + bs * bs;
        double zr = x / den, zi = as / den;       // z = 1/(x - i a) = (x + i a)/(x^2 + a^2)
        double yr = x / dens, yi = bs / dens;
        double wr = zr, wi = zi;                  // w_q = (-1)^q z^{q+1}
        double vr = yr, vi = yi;
        double sg = s == 0 ? 1.0 : -1.0;
        for (int q = 0; q < Q; ++q) {
            double t = wr;
            double u = (q == 0 ? -1.0 : 0.0) + 2.0 * r * wi;
            double us = (q == 0 ? -1.0 : 0.0) + 2.0 * r1 * vi;
            double w2r = wr * zr - wi * zi;       // (-1)^q z^{q+2}
            double v = sg * 2.0 * r * (q + 1) * w2r;
            // store raw per sign in scratch: [s][4][Q] (the Miller series area, reused later)
            raw[(s * 4 + 0) * Q + q] = t;
            raw[(s * 4 + 1) * Q + q] = u;
            raw[(s * 4 + 2) * Q + q] = us;
            raw[(s * 4 + 3) * Q + q] = v;
            double nwr = -(wr * zr - wi * zi), nwi = -(wr * zi + wi * zr);
            wr = nwr;
            wi = nwi;
            double nvr = -(vr * yr - vi * yi), nvi = -(vr * yi + vi * yr);
            vr = nvr;
            vi = nvi;
        }
    }
    __syncthreads();
    // raw tables per sign: t+- u+- us+- v+-
    for (int q = tid; q < Q; q += blockDim.x) {
        tab[0 * Q + q] = raw[0 * Q + q];  // t+
        tab[1 * Q + q] = raw[4 * Q + q];  // t-
        tab[2 * Q + q] = raw[1 * Q + q];  // u+
        tab[3 * Q + q] = raw[5 * Q + q];  // u-
        tab[4 * Q + q] = raw[2 * Q + q];  // us+
        tab[5 * Q + q] = raw[6 * Q + q];  // us-
        tab[6 * Q + q] = raw[3 * Q + q];  // v+
        tab[7 * Q + q] = raw[7 * Q + q];  // v-
    }
    for (int n = tid; n < NM; n += blockDim.x) g00[n * D] = G[n];
    __syncthreads();
    const double *tp = tab, *tm = tab + Q, *up = tab + 2 * Q, *um = tab + 3 * Q;
    const double *sp = tab + 4 * Q, *smn = tab + 5 * Q, *vp = tab + 6 * Q, *vm = tab + 7 * Q;
    // x-derivatives (reading R#22).  Modes 0 and 1: the paper's x-recursion with
    // (Gbar^n +- Gbar^{n-1}) formed first, G^(-1) == G^(1):
    //   Gbar_{00,k+1}^n = (n - 1/2)/(k+1) sum_q [(g_n + g_m)[k-q] t+_q + (g_n - g_m)[k-q] t-_q]
    if (tid < 2) {
        const int n = tid, m = 1 - tid;
        for (int k = 0; k < C; ++k) {
            double s = 0.0;
            for (int q = 0; q <= k; ++q) {
                double gn = g00[n * D + k - q], gm = g00[m * D + k - q];
                s = fma(gn + gm, tp[q], fma(gn - gm, tm[q], s));
            }
            __syncwarp(0x3u);
            g00[n * D + k + 1] = (n - 0.5) * s / (k + 1);
            __syncwarp(0x3u);
        }
    }
    __syncthreads();
    // Modes n >= 2: the three-term recursion on the Taylor series in Delta x, with
    // chi(x + Delta) = chi + (x / (r r1)) Delta + Delta^2 / (2 r r1) exactly; the x-recursion
    // for all modes amplifies rounding by ~(n - 1/2)/(k+1) per order when n > k.
    if (Ni >= 2) {
        const double chi0 = 0.5 * (geo.rp2 + geo.rm2) / (2.0 * geo.rr1);
        const double ch1 = x / geo.rr1, ch2 = 0.5 / geo.rr1;
        if (geo.forward) {
            // forward from g_0, g_1: lane c owns coefficient c
            for (int n = 2; n <= Ni; ++n) {
                if (tid < D) {
                    const double *g1 = g00 + (n - 1) * D, *g2 = g00 + (n - 2) * D;
                    double cg = chi0 * g1[tid];
                    if (tid >= 1) cg = fma(ch1, g1[tid - 1], cg);
                    if (tid >= 2) cg = fma(ch2, g1[tid - 2], cg);
                    g00[n * D + tid] = (4.0 * (n - 1) * cg - (2.0 * n - 3.0) * g2[tid]) / (2.0 * n - 1.0);
                }
                __syncthreads();
            }
        } else {
            // Miller in ratio form: rho_S = 0,
            //   rho_{n-1} = (2n-3) / (4(n-1) chi(Delta) - (2n-1) rho_n)   (series reciprocal),
            // S = N + e(chi) as for G (R#4); then g_n = g_{n-1} rho_n.
            // start: the contamination lambda^{-2(S-n)} must be small on the whole disk
            // |Delta| <= rho_-/2 whose Taylor coefficients the S2L offsets use (|Delta| <= h,
            // rho_- >= 2h), so e follows from the minimum of ln|lambda(chi(x + Delta))| on the
            // circle |Delta| = rho_-/2 (harmonic)
            double mloc = 1e300;
            const double Rd = 0.5 * sqrt(geo.rm2);
            for (int k = tid; k < 256; k += blockDim.x) {
                double sn, cs;
                sincospi(k / 128.0, &sn, &cs);
                const double xr = fma(Rd, cs, x), xi = Rd * sn;   // x + Delta
                const double inv2 = 0.5 / geo.rr1;
                const double zr = (r * r + r1 * r1 + xr * xr - xi * xi) * inv2, zi = 2.0 * xr * xi * inv2;
                // w = z + sqrt(z^2 - 1), |ln|w|| (either root gives the same modulus of the log)
                const double ar = zr * zr - zi * zi - 1.0, ai = 2.0 * zr * zi;
                const double md = hypot(ar, ai);
                double sr_ = sqrt(0.5 * (md + fabs(ar))), si_ = ai / (2.0 * (sr_ > 0.0 ? sr_ : 1.0));
                if (ar < 0.0) {
                    const double t = fabs(si_);
                    si_ = ai >= 0.0 ? sr_ : -sr_;
                    sr_ = t;
                }
                const double v = fabs(log(hypot(zr + sr_, zi + si_)));
                mloc = fmin(mloc, v);
            }
            for (int o = 16; o > 0; o >>= 1) mloc = fmin(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
            if ((tid & 31) == 0) den[tid >> 5] = mloc;
            __syncthreads();
            if (tid == 0) {
                double m = den[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, den[w]);
                int e = miller_extra(geo, a.miller);
                if (a.miller != 1) {
                    const double es = ceil(20.0 / (0.97 * m)) + 4.0;
                    const double cap = (double)(kMaxSteps - kMaxModes - 4);
                    e = max(e, (int)fmin(es, cap));
                }
                sS[0] = (a.K - 1 > Ni ? a.K - 1 : Ni) + e;
            }
            __syncthreads();
            const int S = sS[0];
            // Miller in ratio form on the Taylor series in Delta x (R#22):
            //   rho_S = 0,  rho_{n-1} = (2n-3) / (4(n-1) chi(Delta) - (2n-1) rho_n)
            // (series reciprocal), then g_n = g_{n-1} rho_n.  The recursion is sequential in n;
            // for the BASELINE orders it runs in one thread on register-resident series
            // (D = 17, 25, 33), otherwise on shared memory.
            {
                if (tid == 0 && D == 17) miller_series_regs<17>(S, Ni, chi0, ch1, ch2, rat);
                else if (tid == 0 && D == 25) miller_series_regs<25>(S, Ni, chi0, ch1, ch2, rat);
                else if (tid == 0 && D == 33) miller_series_regs<33>(S, Ni, chi0, ch1, ch2, rat);
                else if (tid == 0) {
                    for (int c = 0; c < D; ++c) rho[c] = 0.0;
                    for (int n = S; n >= 2; --n) {
                        const double a4 = 4.0 * (n - 1), b2 = 2.0 * n - 1.0;
                        den[0] = fma(a4, chi0, -b2 * rho[0]);
                        if (D > 1) den[1] = fma(a4, ch1, -b2 * rho[1]);
                        if (D > 2) den[2] = fma(a4, ch2, -b2 * rho[2]);
                        for (int c = 3; c < D; ++c) den[c] = -b2 * rho[c];
                        const double inv = 1.0 / den[0];
                        rho[0] = (2.0 * n - 3.0) * inv;
                        for (int c = 1; c < D; ++c) {
                            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                            int j2 = 0;
                            for (; j2 + 3 < c; j2 += 4) {
                                s0 = fma(rho[j2], den[c - j2], s0);
                                s1 = fma(rho[j2 + 1], den[c - j2 - 1], s1);
                                s2 = fma(rho[j2 + 2], den[c - j2 - 2], s2);
                                s3 = fma(rho[j2 + 3], den[c - j2 - 3], s3);
                            }
                            for (; j2 < c; ++j2) s0 = fma(rho[j2], den[c - j2], s0);
                            rho[c] = -((s0 + s1) + (s2 + s3)) * inv;
                        }
                        if (n - 1 <= Ni)
                            for (int c = 0; c < D; ++c) rat[(n - 1) * D + c] = rho[c];
                    }
                }
                __syncthreads();
                for (int n = 2; n <= Ni; ++n) {
                    if (tid < D) {
                        const double *g1 = g00 + (n - 1) * D, *rn = rat + n * D;
                        double acc = 0.0;
                        for (int j2 = 0; j2 <= tid; ++j2) acc = fma(g1[j2], rn[tid - j2], acc);
                        g00[n * D + tid] = acc;
                    }
                    __syncthreads();
                }
            }
        }
    }
    // seeds out: [4][NM][D]
    double *so = a.seeds + gi * 4 * (int64_t)NM * D;
    // r and r1 derivatives
    for (int e = tid; e < NM * C; e += blockDim.x) {
        int n = e / C, k = e % C, m = n == 0 ? 1 : n - 1;
        double s1 = 0.0, s2 = 0.0;
        for (int q = 0; q <= k; ++q) {
            double gn = g00[n * D + k - q], gm = g00[m * D + k - q];
            double gp = gn + gm, gd = gn - gm;
            s1 = fma(gp, up[q], fma(gd, um[q], s1));
            s2 = fma(gp, sp[q], fma(gd, smn[q], s2));
        }
        so[NM * D + n * D + k] = (-g00[n * D + k] + (n - 0.5) * s1) / (2.0 * r);
        g01[n * D + k] = (-g00[n * D + k] + (n - 0.5) * s2) / (2.0 * r1);
    }
    __syncthreads();
    // mixed: sum_q [(g+)v+ + (h+)u+ + (g-)v- + (h-)u-] with g = g00, h = g01
    for (int e = tid; e < NM * (C - 1); e += blockDim.x) {
        int n = e / (C - 1), k = e % (C - 1), m = n == 0 ? 1 : n - 1;
        double s = 0.0;
        for (int q = 0; q <= k; ++q) {
            double gn = g00[n * D + k - q], gm = g00[m * D + k - q];
            double hn = g01[n * D + k - q], hm = g01[m * D + k - q];
            s = fma(gn + gm, vp[q], fma(hn + hm, up[q], fma(gn - gm, vm[q], fma(hn - hm, um[q], s))));
        }
        so[3 * NM * D + n * D + k] = (-g01[n * D + k] + (n - 0.5) * s) / (2.0 * r);
    }
    for (int e = tid; e < NM * D; e += blockDim.x) {
        const int c = e % D;
        so[e] = g00[e];
        so[2 * NM * D + e] = c < C ? g01[e] : 0.0;
        if (c == C) so[NM * D + e] = 0.0;               // (g10, g11 beyond their last column)
        if (c >= C - 1) so[3 * NM * D + e] = 0.0;
    }
}

inline size_t tensor_seed_smem(int K, int m1, int p)
{
    int Nw = m1 - 1, Ni = Nw > 1 ? Nw : 1, NM = Ni + 1, Q = 2 * p + 2, D = 2 * p + 1;
    size_t ratsz = (size_t)NM * D;
    if (ratsz < (size_t)8 * Q) ratsz = 8 * Q;
    (void)K;
    return sizeof(double) * (NM + 8 * Q + 2 * (size_t)NM * D + ratsz + 2 * D + 6);
}

// closed form of packed_off
__host__ __device__ inline int packed_row_t(int a, int b, int p)
{
    return a * ((p + 1) * (2 * p + 1) - p * (p + 1) / 2) - (p + 1) * (a * (a - 1) / 2) +
           b * (2 * p + 1 - a) - b * (b - 1) / 2;
}
// 1 / ((k + 1)(k + 2)) for the Laplace steps (k <= 2 CYLFMM_MAX_ORDER)
__constant__ double c_lapinv[40] = {
#define LI(k) 1.0 / (((k) + 1.0) * ((k) + 2.0))
    LI(0), LI(1), LI(2), LI(3), LI(4), LI(5), LI(6), LI(7), LI(8), LI(9), LI(10), LI(11), LI(12),
    LI(13), LI(14), LI(15), LI(16), LI(17), LI(18), LI(19), LI(20), LI(21), LI(22), LI(23), LI(24),
    LI(25), LI(26), LI(27), LI(28), LI(29), LI(30), LI(31), LI(32), LI(33), LI(34), LI(35), LI(36),
    LI(37), LI(38), LI(39)
#undef LI
};
// packed offset of (a, b) for order p (host/device helper used by S2L)
__host__ __device__ inline int packed_off(int aa, int b, int p)
{
    // rows a' < aa contribute sum_{b'=0..p} (2p+1-a'-b') = (p+1)(2p+1-a') - p(p+1)/2
    int off = 0;
    for (int a2 = 0; a2 < aa; ++a2) off += (p + 1) * (2 * p + 1 - a2) - p * (p + 1) / 2;
    for (int b2 = 0; b2 < b; ++b2) off += 2 * p + 1 - aa - b2;
    return off;
}

// ---------------------------------------------------------------------------------------------
// Warp per (geometry, mode), no shared memory and no barriers.  Lane c holds column c of the
// current rows (c = lane, and c = lane + 32 in a second register: only column 2p = 32 of row
// (0, 0) at p = 16 needs it).  The Laplace recursion in r (b in {0, 1}, advancing a) and, for
// every a as soon as its b = 0, 1 rows exist, the recursion in r1 (advancing b) keep the three
// previous rows in registers; the (c + 2) terms come from lane c + 2 by shuffles.  Each row is
// written out as soon as it is formed (one coalesced store per row).  Entries with a + b + c > 2p
// are never read by a valid entry, so lanes past the end of a row carry don't-care values.
struct Row {                 // column c (lo) and c + 32 (hi) of one tensor row
    double lo, hi;
};
// column c + 2 of a row from lane c + 2; the one entry past lane 31 any valid entry reads is
// (0, 0, 2p = 32) at p = 16 (by lane 30 when forming rows (2, 0) and (0, 2)): hi00, a register
__device__ __forceinline__ double col_plus2(const Row &v, int lane, bool row00, double hi00)
{
    const double a = __shfl_down_sync(0xffffffffu, v.lo, 2);
    return (row00 && lane == 30) ? hi00 : a;
}

// PT > 0: the order as a compile-time constant (the BASELINE orders 8, 12, 16): every loop below
// unrolls, so the packed row offsets, the per-step coefficients' rational factors and the
// k >= 1 / k >= 2 cases become constants (the runtime-order loop spent ~100 instructions per
// row on index arithmetic, integer -> FP64 conversions and branches; now ~15).  PT = 0: any p.
//
// One Laplace step, written so that the newest row enters last through ONE FMA (the row-to-row
// dependency chain is a single DFMA; everything else is formed off the chain):
//   new = A_k cur + B_k prv + L_k(c) (s^2 prv[c+2] + 2 s pm1[c+2] + pm2[c+2]),
//   A_k = -(2k+1) / ((k+2) s),  B_k = (n^2 - k^2) / (s^2 (k+1)(k+2)),
//   L_k(c) = -(c+1)(c+2) / (s^2 (k+1)(k+2))
// (the same recursion as  s^2 (k+1)(k+2) new + s (k+1)(2k+1) cur + (k^2 - n^2) prv + ... = 0).
template <int PT>
__global__ void __launch_bounds__(128, PT ? 4 : 1) tensor_fill_kernel(TensorGeomArgs a)
{
    const int p = PT ? PT : a.p, C = 2 * p, D = C + 1, P1 = p + 1;
    const int KW = a.m1 - a.m0;
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= a.nwork) return;
    const int64_t gi = a.glist ? a.glist[w / KW] : w / KW;
    const int n = a.m0 + (int)(w % KW);
    const int Nw = (a.seed_m1 ? a.seed_m1 : a.m1) - 1, Ni = Nw > 1 ? Nw : 1, NM = Ni + 1;
    double r, r1, x;
    geometry_of(a, gi, r, r1, x);
    if (!(r > 0.0) || !(r1 > 0.0) || (r == r1 && x == 0.0)) return;   // flagged by seed kernel
    const double *sd = a.seeds + gi * 4 * (int64_t)NM * D;
    const double n2 = (double)n * n;
    const int c0 = lane, c1 = lane + 32;
    // packed (FMM) layout stores H_ab(c) = c! Gbar_abc (the S2L Hankel form); dense: Gbar_abc
    double f0 = 1.0, f1 = 1.0;
    if (a.packed) {
        for (int t = 2; t <= c0; ++t) f0 *= t;
        f1 = f0;
        for (int t = c0 + 1; t <= c1; ++t) f1 *= t;
    }
    const int64_t TP = (int64_t)P1 * P1 * P1, TPp = TP + (TP & 1);   // packed: padded 16-B blocks
    double *o = a.out + (gi * KW + (n - a.m0)) * (a.packed ? TPp : (int64_t)P1 * P1 * D);
    auto store = [&](int aa, int b, const Row &v) {
        const int cmax = C - aa - b;
        if (a.packed) {
            double *q = o + packed_row_t(aa, b, p);
            if (c0 <= cmax) q[c0] = v.lo * f0;
            if (c1 <= cmax) q[c1] = v.hi * f1;
        } else {
            double *q = o + ((int64_t)aa * P1 + b) * D;
            if (c0 < D) q[c0] = c0 <= cmax ? v.lo : 0.0;
            if (c1 < D) q[c1] = c1 <= cmax ? v.hi : 0.0;
        }
    };
    auto seed = [&](int k, int cmax) {
        Row v;
        v.lo = c0 <= cmax ? sd[(k * NM + n) * D + c0] : 0.0;
        v.hi = c1 <= cmax ? sd[(k * NM + n) * D + c1] : 0.0;
        return v;
    };
    double hi00 = 0.0;   // (0, 0, 32) at p = 16, set from the seeds below
    const double cc = -(c0 + 1.0) * (c0 + 2.0);
    // per direction (r: s = r; r1: s = r1): 1/s, 1/s^2, s^2, 2 s
    struct Dir {
        double is, is2, s2, s2x;
    };
    auto mkdir = [](double sc) {
        Dir d;
        d.is = 1.0 / sc;
        d.is2 = d.is * d.is;
        d.s2 = sc * sc;
        d.s2x = 2.0 * sc;
        return d;
    };
    const Dir dr = mkdir(r), dr1 = mkdir(r1);
    auto lap_step = [&](const Dir &d, int k, const Row &cur, const Row &prv, const Row &pm1,
                        const Row &pm2, bool prv00) {
        const double li = c_lapinv[k] * d.is2;                 // 1 / (s^2 (k+1)(k+2))
        const double A = (-(2.0 * k + 1.0) / (k + 2.0)) * d.is;
        const double B = (n2 - (double)(k * k)) * li;
        const double t0 = col_plus2(prv, lane, prv00, hi00);
        double lap = d.s2 * t0;
        if (k >= 1) lap = fma(d.s2x, col_plus2(pm1, lane, false, 0.0), lap);
        if (k >= 2) lap += col_plus2(pm2, lane, false, 0.0);
        Row nw;
        nw.lo = fma(A, cur.lo, fma(B, prv.lo, (cc * li) * lap));
        // column c + 32 (only c = 32 at p = 16, row (0, 0), never recursed into): not needed
        nw.hi = 0.0;
        return nw;
    };
    // b = 0, 1 rows of a = 0, 1 from the seeds
    Row ra0[4] = {}, ra1[4] = {};   // rows a-4 .. a-1 of the b = 0 (ra0) and b = 1 (ra1) planes
    Row b0 = seed(0, C), b1 = p >= 1 ? seed(2, C - 1) : Row{};
    hi00 = __shfl_sync(0xffffffffu, b0.hi, 0);
    Row a1b0 = p >= 1 ? seed(1, C - 1) : Row{}, a1b1 = p >= 1 ? seed(3, C - 2) : Row{};
#pragma unroll
    for (int aa = 0; aa <= p; ++aa) {
        Row rb0, rb1;   // rows (aa, 0) and (aa, 1)
        if (aa == 0) {
            rb0 = b0;
            rb1 = b1;
        } else if (aa == 1) {
            rb0 = a1b0;
            rb1 = a1b1;
        } else {   // Laplace in r (k = aa - 2): rows k+1, k, k-1, k-2 = aa-1 .. aa-4
            const int k = aa - 2;
            rb0 = lap_step(dr, k, ra0[3], ra0[2], ra0[1], ra0[0], aa == 2);
            rb1 = lap_step(dr, k, ra1[3], ra1[2], ra1[1], ra1[0], false);
        }
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            ra0[h] = ra0[h + 1];
            ra1[h] = ra1[h + 1];
        }
        ra0[3] = rb0;
        ra1[3] = rb1;
        store(aa, 0, rb0);
        if (p >= 1) store(aa, 1, rb1);
        // Laplace in r1 for this a: rows b + 2 from b + 1, b, b - 1, b - 2
        Row hb[4] = {Row{}, Row{}, rb0, rb1};   // rows b-2, b-1, b, b+1 (b = 0)
#pragma unroll
        for (int bb = 0; bb + 2 <= p && aa + bb + 2 <= C; ++bb) {
            const Row nb = lap_step(dr1, bb, hb[3], hb[2], hb[1], hb[0], aa == 0 && bb == 0);
            hb[0] = hb[1];
            hb[1] = hb[2];
            hb[2] = hb[3];
            hb[3] = nb;
            store(aa, bb + 2, nb);
        }
    }
}

}  // namespace cyl
