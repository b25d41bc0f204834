// fmm_ops.cuh -- the FMM expansion passes of Algorithm 1 on sm_100a, FP64.
//
// Units.  Every box quantity is stored normalised by its box size h = L / 2^l (reading of the
// paper's scaling relation G(s r, s r1, s x) = G / s, applied to the derivatives:
// Gbar_{abc}(h g) = h^{-(1+a+b+c)} Gbar_{abc}(g)):
//     moments  M^_ij = S_ij / h^{i+j}                  (S_ij = sum_q S_q dr^i dz^j)
//     locals   L^_kl = h^{1+k+l} Phi_kl                (Phi = sum Phi_kl dr^k dz^l)
// so that S2L is the same operator at every level,
//     L^_kl += sum_{i+j<=p} sigma C(j+l, j) M^_ij Gbar^_{A,B,j+l}(station),
// with the tensor evaluated once per normalised station geometry (r^, r1^, x^) =
// (i_in + dI + 1/2, i_in + 1/2, dJ), and M2M / L2L become constant
// binomial re-centrings (child - parent = +-h_parent/4 per axis, R#9):
//     M2M: M^_ij(parent) = sum C(i,q) C(j,u) s_r^q s_z^u 2^{-(i+j+q+u)} M^'_{i-q,j-u}
//     L2L: L^_ij(child)  = sum C(i+q,q) C(j+u,u) s_r^q s_z^u 2^{-(1+i+j+2q+2u)} L^'_{i+q,j+u}
// Coefficient (i, j), i + j <= p, sits at tri(i, j) = i (p+1) - i (i-1)/2 + j.
#pragma once
#include "tensor.cuh"
#include "p2p.cuh"

namespace cyl {

constexpr int kMaxLevels = 12;

struct FarArgs {
    int depth, p, P, K, m0, m1;
    double L, z0;
    int truncation;
    // per level l (2..depth): compact box lists
    const int *smap[kMaxLevels], *skeys[kMaxLevels];
    const int *tmap[kMaxLevels], *tkeys[kMaxLevels];
    int scount[kMaxLevels], tcount[kMaxLevels];
    int64_t soff[kMaxLevels], toff[kMaxLevels];  // box offsets into M / Lc
    double2 *M;          // moments  [box][KW][P]
    double2 *Lc;         // locals   [box][KW][P]
    const int *slstart, *flstart;
    const double *sr, *sz;
    const double2 *S;    // sorted sources [ns][K]
    const double *fr, *fz;
    const int *fperm;
    double2 *out;        // [nf][K], input field order
    const double *tens;  // [12 * 2^d][KW][(p+1)^3] packed
    unsigned long long *s2l_pairs;  // counter of (source box, target box) applications
};

__device__ __forceinline__ int tri(int i, int j, int p) { return i * (p + 1) - i * (i - 1) / 2 + j; }

__device__ __forceinline__ void box_centre(uint32_t key, int level, double L, double z0,
                                           double &rc, double &zc, double &h)
{
    h = L / (double)(1u << level);
    rc = ((double)compact1(key) + 0.5) * h;
    zc = z0 + ((double)compact1(key >> 1) + 0.5) * h;
}

// ---------------------------------------------------------------------------------------------
// P2M at the leaves: CTA per non-empty source leaf.  Outputs (n, ij) spread over threads, sources
// streamed through smem in chunks of 32 with their monomials.
constexpr int kP2MThreads = 256;
constexpr int kP2MChunk = 32;
constexpr int kP2MOut = 4;

__global__ void __launch_bounds__(kP2MThreads) p2m_kernel(FarArgs a)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0, d = a.depth;
    double *mono = sm;                                           // [chunk][P]
    double2 *Sx = reinterpret_cast<double2 *>(mono + kP2MChunk * P);  // [chunk][KW]
    const int slot = blockIdx.x;
    const uint32_t key = (uint32_t)a.skeys[d][slot];
    double rc, zc, h;
    box_centre(key, d, a.L, a.z0, rc, zc, h);
    const int q0 = a.slstart[key], q1 = a.slstart[key + 1];
    double2 *Mo = a.M + (a.soff[d] + slot) * (int64_t)KW * P;
    const int nout = KW * P;
    for (int g0 = 0; g0 < nout; g0 += kP2MThreads * kP2MOut) {
        double2 acc[kP2MOut];
#pragma unroll
        for (int k = 0; k < kP2MOut; ++k) acc[k] = make_double2(0.0, 0.0);
        for (int c0 = q0; c0 < q1; c0 += kP2MChunk) {
            const int nc = min(kP2MChunk, q1 - c0);
            __syncthreads();
            if (threadIdx.x < nc) {
                int q = c0 + threadIdx.x;
                double dr = (a.sr[q] - rc) / h, dz = (a.sz[q] - zc) / h;
                double pr = 1.0;
                for (int i = 0; i <= p; ++i) {
                    double pz = pr;
                    for (int j = 0; i + j <= p; ++j) {
                        mono[threadIdx.x * P + tri(i, j, p)] = pz;
                        pz *= dz;
                    }
                    pr *= dr;
                }
            }
            for (int e = threadIdx.x; e < nc * KW; e += kP2MThreads) {
                int q = e / KW, n = e % KW;
                Sx[e] = a.S[(int64_t)(c0 + q) * a.K + a.m0 + n];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kP2MOut; ++k) {
                int o = g0 + threadIdx.x + k * kP2MThreads;
                if (o < nout) {
                    int n = o / P, ij = o % P;
                    double2 s = acc[k];
                    for (int q = 0; q < nc; ++q) {
                        double m = mono[q * P + ij];
                        double2 sv = Sx[q * KW + n];
                        s.x = fma(sv.x, m, s.x);
                        s.y = fma(sv.y, m, s.y);
                    }
                    acc[k] = s;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kP2MOut; ++k) {
            int o = g0 + threadIdx.x + k * kP2MThreads;
            if (o < nout) Mo[o] = acc[k];
        }
    }
}

// binomial C(n, k) for n <= 2 * 20 (exact in FP64)
__device__ __forceinline__ double binom_d(int n, int k)
{
    if (k < 0 || k > n) return 0.0;
    double b = 1.0;
    for (int i = 1; i <= k; ++i) b = b * (n - k + i) / i;
    return b;
}

// ---------------------------------------------------------------------------------------------
// M2M, level l from l+1: CTA per (parent box, mode).
__global__ void __launch_bounds__(256) m2m_kernel(FarArgs a, int level)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0;
    const int slot = blockIdx.x / KW, n = blockIdx.x % KW;
    double2 *ch = reinterpret_cast<double2 *>(sm);   // [4][P]
    double *bin = reinterpret_cast<double *>(ch + 4 * P);   // [(p+1)^2]
    const uint32_t key = (uint32_t)a.skeys[level][slot];
    int cs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) cs[c] = a.smap[level + 1][4 * key + c];
    for (int e = threadIdx.x; e < (p + 1) * (p + 1); e += blockDim.x)
        bin[e] = binom_d(e / (p + 1), e % (p + 1));
    for (int e = threadIdx.x; e < 4 * P; e += blockDim.x) {
        int c = e / P, ij = e % P;
        ch[e] = cs[c] >= 0 ? a.M[((a.soff[level + 1] + cs[c]) * (int64_t)KW + n) * P + ij]
                           : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int ij = threadIdx.x; ij < P; ij += blockDim.x) {
        // decode (i, j)
        int i = 0;
        while (tri(i + 1, 0, p) <= ij && i < p) ++i;
        int j = ij - tri(i, 0, p);
        double2 s = make_double2(0.0, 0.0);
        for (int c = 0; c < 4; ++c) {
            if (cs[c] < 0) continue;
            double sr = (c & 1) ? 1.0 : -1.0, sz = (c & 2) ? 1.0 : -1.0;
            const double2 *C = ch + c * P;
            double pq = 1.0;
            for (int q = 0; q <= i; ++q) {
                double pu = pq * bin[i * (p + 1) + q];
                for (int u = 0; u <= j; ++u) {
                    double coef = ldexp(pu * bin[j * (p + 1) + u], -(i + j + q + u));
                    double2 v = C[tri(i - q, j - u, p)];
                    s.x = fma(coef, v.x, s.x);
                    s.y = fma(coef, v.y, s.y);
                    pu *= sz;
                }
                pq *= sr;
            }
        }
        a.M[((a.soff[level] + slot) * (int64_t)KW + n) * P + ij] = s;
    }
}

// ---------------------------------------------------------------------------------------------
// L2L, level l from l-1 (overwrites the level-l locals): CTA per (child box, mode).
__global__ void __launch_bounds__(256) l2l_kernel(FarArgs a, int level)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0;
    const int slot = blockIdx.x / KW, n = blockIdx.x % KW;
    double2 *par = reinterpret_cast<double2 *>(sm);  // [P]
    double *bin = reinterpret_cast<double *>(par + P);
    const uint32_t key = (uint32_t)a.tkeys[level][slot];
    const int ps = a.tmap[level - 1][key >> 2];
    const int c = key & 3;
    for (int e = threadIdx.x; e < (p + 1) * (p + 1); e += blockDim.x)
        bin[e] = binom_d(e / (p + 1), e % (p + 1));
    for (int e = threadIdx.x; e < P; e += blockDim.x)
        par[e] = a.Lc[((a.toff[level - 1] + ps) * (int64_t)KW + n) * P + e];
    __syncthreads();
    const double sr = (c & 1) ? 1.0 : -1.0, sz = (c & 2) ? 1.0 : -1.0;
    for (int ij = threadIdx.x; ij < P; ij += blockDim.x) {
        int i = 0;
        while (tri(i + 1, 0, p) <= ij && i < p) ++i;
        int j = ij - tri(i, 0, p);
        double2 s = make_double2(0.0, 0.0);
        double pq = 1.0;
        for (int q = 0; i + j + q <= p; ++q) {
            double pu = pq * bin[(i + q) * (p + 1) + q];
            for (int u = 0; i + j + q + u <= p; ++u) {
                double coef = ldexp(pu * bin[(j + u) * (p + 1) + u], -(1 + i + j + 2 * q + 2 * u));
                double2 v = par[tri(i + q, j + u, p)];
                s.x = fma(coef, v.x, s.x);
                s.y = fma(coef, v.y, s.y);
                pu *= sz;
            }
            pq *= sr;
        }
        a.Lc[((a.toff[level] + slot) * (int64_t)KW + n) * P + ij] = s;
    }
}

// ---------------------------------------------------------------------------------------------
// L2P at the leaves: CTA per (target leaf, mode group of <= 16); writes out rows (input order).
constexpr int kL2PModes = 16;
constexpr int kL2PPts = 16;

__global__ void __launch_bounds__(256) l2p_kernel(FarArgs a)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0, d = a.depth;
    const int ngrp = (KW + kL2PModes - 1) / kL2PModes;
    const int slot = blockIdx.x / ngrp, g = blockIdx.x % ngrp;
    const int n0 = g * kL2PModes, nm = min(kL2PModes, KW - n0);
    double2 *loc = reinterpret_cast<double2 *>(sm);     // [nm][P]
    double *mono = reinterpret_cast<double *>(loc + kL2PModes * P);  // [pts][P]
    const uint32_t key = (uint32_t)a.tkeys[d][slot];
    double rc, zc, h;
    box_centre(key, d, a.L, a.z0, rc, zc, h);
    const double inv_h = 1.0 / h;
    const int t0 = a.flstart[key], t1 = a.flstart[key + 1];
    for (int e = threadIdx.x; e < nm * P; e += blockDim.x)
        loc[e] = a.Lc[((a.toff[d] + slot) * (int64_t)KW + n0) * P + e];
    for (int c0 = t0; c0 < t1; c0 += kL2PPts) {
        const int nc = min(kL2PPts, t1 - c0);
        __syncthreads();
        if (threadIdx.x < nc) {
            int t = c0 + threadIdx.x;
            double dr = (a.fr[t] - rc) / h, dz = (a.fz[t] - zc) / h;
            double pr = 1.0;
            for (int i = 0; i <= p; ++i) {
                double pz = pr;
                for (int j = 0; i + j <= p; ++j) {
                    mono[threadIdx.x * P + tri(i, j, p)] = pz;
                    pz *= dz;
                }
                pr *= dr;
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nc * nm; e += blockDim.x) {
            int t = e / nm, n = e % nm;
            const double *mo = mono + t * P;
            const double2 *lo = loc + n * P;
            double sx = 0.0, sy = 0.0;
            for (int kl = 0; kl < P; ++kl) {
                sx = fma(lo[kl].x, mo[kl], sx);
                sy = fma(lo[kl].y, mo[kl], sy);
            }
            int64_t row = a.fperm[c0 + t];
            a.out[row * a.K + a.m0 + n0 + n] = make_double2(sx * inv_h, sy * inv_h);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// S2L, batched per target column: CTA per (level, target column i_t,
// parity of j_t, tile of JT target boxes of that parity, mode n).  For each of the <= 27 offsets
// (dI, dJ) of the interaction list (children of the parent's neighbours that are not neighbours,
// P:246-252, 539-559) the P x P operator
//     A[(k,l), (i,j)] = sigma C(j+l, j) Gbar^_{A,B, j+l}
// (FO: sigma = (-1)^j, (A,B) = (k,i); BO: (-1)^l, (k,i); FI: (-1)^j, (i,k); BI: (-1)^l, (i,k))
// is gathered from the station tensor into smem (k-chunked) and applied to the moments of the
// JT source boxes (2 JT real columns) by a register-tiled FP64 GEMM on the CUDA cores.
// Locals accumulate in registers over all offsets in a fixed order (deterministic).
template <int NT, int TM, int RM, int RN, int KC>
struct S2LCfg {
    static constexpr int TN = NT / TM;
    static constexpr int MP = TM * RM;          // padded rows (>= P)
    static constexpr int NC = TN * RN;          // columns = 2 JT
    static constexpr int JT = NC / 2;
};

template <int NT, int TM, int RM, int RN, int KC>
__global__ void __launch_bounds__(NT) s2l_kernel(FarArgs a, int level, int jtiles)
{
    using Cfg = S2LCfg<NT, TM, RM, RN, KC>;
    constexpr int TN = Cfg::TN, MP = Cfg::MP, NC = Cfg::NC, JT = Cfg::JT;
    extern __shared__ double sm[];
    double *As = sm;                               // [KC][MP]
    double *Bs = As + KC * MP;                     // [KC][NC]
    double *bin = Bs + KC * NC;                    // [(2p+1)][(p+1)]
    int *tri_i = reinterpret_cast<int *>(bin + (2 * a.p + 1) * (a.p + 1));  // [P]
    int *tri_j = tri_i + a.P;
    int *poff = tri_j + a.P;                       // [(p+1)^2]
    int *tsl = poff + (a.p + 1) * (a.p + 1);       // [JT]
    int *ssl = tsl + JT;                           // [JT]

    const int p = a.p, P = a.P, KW = a.m1 - a.m0;
    const int nb = 1 << level;
    int bid = blockIdx.x;
    const int nloc = bid % KW;
    bid /= KW;
    const int jt = bid % jtiles;
    bid /= jtiles;
    const int jpar = bid & 1;
    const int it = bid >> 1;
    const int n = a.m0 + nloc;
    const int tid = threadIdx.x;
    const int tm = tid % TM, tn = tid / TM;

    // target boxes of this tile
    int anyt = 0;
    if (tid < JT) {
        int jtb = jpar + 2 * (jt * JT + tid);
        int s = -1;
        if (jtb < nb) s = a.tmap[level][morton2((uint32_t)it, (uint32_t)jtb)];
        tsl[tid] = s;
        anyt = s >= 0;
    }
    if (!__syncthreads_or(anyt)) return;
    for (int e = tid; e < (2 * p + 1) * (p + 1); e += NT) bin[e] = binom_d(e / (p + 1), e % (p + 1));
    for (int i = 0, ij = 0; i <= p; ++i)
        for (int j = 0; i + j <= p; ++j, ++ij)
            if (ij % NT == tid) {
                tri_i[ij] = i;
                tri_j[ij] = j;
            }
    for (int e = tid; e < (p + 1) * (p + 1); e += NT) poff[e] = packed_off(e / (p + 1), e % (p + 1), p);

    // accumulators: rows m = 2 (tm + TM u) + {0,1}, cols c = tn + TN v
    double acc[RM][RN];
    const int64_t TP = (int64_t)(p + 1) * (p + 1) * (p + 1);
    __syncthreads();
#pragma unroll
    for (int v = 0; v < RN; ++v) {
        int col = tn + TN * v, box = col >> 1, im = col & 1;
        int s = tsl[box];
#pragma unroll
        for (int u = 0; u < RM; ++u) {
            int m = 2 * (tm + TM * (u >> 1)) + (u & 1);
            double x = 0.0;
            if (s >= 0 && m < P) {
                double2 L = a.Lc[((a.toff[level] + s) * (int64_t)KW + nloc) * P + m];
                x = im ? L.y : L.x;
            }
            acc[u][v] = x;
        }
    }
    const int di0 = (it & 1) ? -3 : -2, dj0 = jpar ? -3 : -2;
    for (int di = di0; di <= di0 + 5; ++di) {
        const int is = it + di;
        if (is < 0 || is >= nb) continue;
        for (int dj = dj0; dj <= dj0 + 5; ++dj) {
            if (di >= -1 && di <= 1 && dj >= -1 && dj <= 1) continue;
            __syncthreads();
            int anys = 0;
            if (tid < JT) {
                int jtb = jpar + 2 * (jt * JT + tid), js = jtb + dj;
                int s = -1;
                if (tsl[tid] >= 0 && js >= 0 && js < nb)
                    s = a.smap[level][morton2((uint32_t)is, (uint32_t)js)];
                ssl[tid] = s;
                anys = s >= 0;
            }
            const int npair = __syncthreads_count(anys);
            if (npair == 0) continue;
            if (tid == 0 && nloc == 0 && a.m0 == 0 && a.s2l_pairs) atomicAdd(a.s2l_pairs, (unsigned long long)npair);
            const bool outward = di <= 0, fwd = dj <= 0;
            const int iin = min(it, is), dI = di < 0 ? -di : di, dJ = dj < 0 ? -dj : dj;
            const double *Tn = a.tens + ((int64_t)(iin * 12 + class_of(dI, dJ)) * KW + nloc) * TP;
            for (int k0 = 0; k0 < P; k0 += KC) {
                const int kc = min(KC, P - k0);
                __syncthreads();
                // A[kk][m]: kk = source coefficient (i, j) = k0 + kk, m = local (k, l)
                for (int e = tid; e < KC * MP; e += NT) {
                    int kk = e / MP, m = e % MP;
                    double val = 0.0;
                    if (kk < kc && m < P) {
                        int ij = k0 + kk;
                        int i = tri_i[ij], j = tri_j[ij], k = tri_i[m], l = tri_j[m];
                        if (a.truncation == 0 || i + j + k + l <= p) {
                            int A = outward ? k : i, B = outward ? i : k;
                            double sg = fwd ? ((j & 1) ? -1.0 : 1.0) : ((l & 1) ? -1.0 : 1.0);
                            val = sg * bin[(j + l) * (p + 1) + j] * __ldg(Tn + poff[A * (p + 1) + B] + j + l);
                        }
                    }
                    As[e] = val;
                }
                for (int e = tid; e < KC * NC; e += NT) {
                    int kk = e / NC, col = e % NC;
                    int s = ssl[col >> 1];
                    double val = 0.0;
                    if (kk < kc && s >= 0) {
                        double2 M = a.M[((a.soff[level] + s) * (int64_t)KW + nloc) * P + k0 + kk];
                        val = (col & 1) ? M.y : M.x;
                    }
                    Bs[e] = val;
                }
                __syncthreads();
#pragma unroll 2
                for (int kk = 0; kk < kc; ++kk) {
                    double av[RM], bv[RN];
#pragma unroll
                    for (int u = 0; u < RM / 2; ++u) {
                        double2 t = *reinterpret_cast<const double2 *>(As + kk * MP + 2 * (tm + TM * u));
                        av[2 * u] = t.x;
                        av[2 * u + 1] = t.y;
                    }
#pragma unroll
                    for (int v = 0; v < RN; ++v) bv[v] = Bs[kk * NC + tn + TN * v];
#pragma unroll
                    for (int u = 0; u < RM; ++u)
#pragma unroll
                        for (int v = 0; v < RN; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
                }
            }
        }
    }
    // write back
#pragma unroll
    for (int v = 0; v < RN; ++v) {
        int col = tn + TN * v, box = col >> 1, im = col & 1;
        int s = tsl[box];
        if (s < 0) continue;
        double *dst = reinterpret_cast<double *>(a.Lc + ((a.toff[level] + s) * (int64_t)KW + nloc) * P);
#pragma unroll
        for (int u = 0; u < RM; ++u) {
            int m = 2 * (tm + TM * (u >> 1)) + (u & 1);
            if (m < P) dst[2 * m + im] = acc[u][v];
        }
    }
}

template <int NT, int TM, int RM, int RN, int KC>
inline size_t s2l_smem_bytes(int p)
{
    using Cfg = S2LCfg<NT, TM, RM, RN, KC>;
    int P = (p + 1) * (p + 2) / 2;
    return sizeof(double) * ((size_t)KC * Cfg::MP + (size_t)KC * Cfg::NC + (2 * p + 1) * (p + 1)) +
           sizeof(int) * (2 * P + (p + 1) * (p + 1) + 2 * Cfg::JT);
}

// Near-field task list: one task per tile of <= TT field points of a non-empty target leaf.
__global__ void near_tasks_count_kernel(const int *tkeys, int nleaf, const int *flstart, int TT,
                                        int *cnt)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nleaf) return;
    int key = tkeys[s];
    int nt = flstart[key + 1] - flstart[key];
    cnt[s] = (nt + TT - 1) / TT;
}
__global__ void near_tasks_emit_kernel(const int *tkeys, int nleaf, const int *flstart, int TT,
                                       const int *off, int4 *tasks, int *ntasks)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nleaf) return;
    int key = tkeys[s];
    int t0 = flstart[key], t1 = flstart[key + 1];
    int o = off[s];
    for (int t = t0; t < t1; t += TT) tasks[o++] = make_int4(t, min(t + TT, t1), key, 0);
    if (s == nleaf - 1) *ntasks = o;
}

}  // namespace cyl
