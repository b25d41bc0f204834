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

#include <cmath>
#include <vector>

namespace cyl {

constexpr int kMaxLevels = 12;

struct FarArgs {
    int depth, p, P, K, m0, m1;   // p, P: source (moment) order and size
    int pl, Pl, pt;               // local order and size; tensor order max(p, pl)
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
    const int *s2l_idx;  // [4][P][MP] operator gather table (build_s2l_index)
    const int *s2l_tiles;               // compact list of S2L tiles with >= 1 interaction
    const unsigned char *s2l_written;   // dense per level [lvoff[l] + key]: local written by S2L
    int64_t lvoff[kMaxLevels];          // dense per-level offsets (level maps, s2l_written)
    const unsigned char *need;          // dense per level: local materialised (see need_kernel)
    int l2p_accumulate;                 // L2P adds onto out (the near field wrote it first)
    int l2p_lc;                         // L2P: consecutive target leaves per CTA (>= 1)
    // recentring tables (host-built once per plan, recentre_tables_host): [cm | cl] 4 (p+1)^2
    // doubles and [tri_i | tri_j] 2 P ints, for the source order (M2M) and the local order (L2L)
    const double *rtab_m, *rtab_l;
    const int *tritab_m, *tritab_l;
    const double *pscale;               // [P] (-1)^j / j! per source coefficient (S2L prescale)
    double2 *outr, *outz;               // gradient rows (nullable): dPhi/dr, dPhi/dz
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
// P2M at the leaves, as a small complex-by-real GEMM per leaf:
//   M^(n)_ij = sum_q S_q^(n) mono_q[ij],  mono_q[ij] = ((r_q - r_c)/h)^i ((z_q - z_c)/h)^j.
// CTA per (source leaf, block of kP2MModes modes); sources streamed through shared memory in
// chunks of kP2MSrc (monomials computed once per chunk); thread tile = 2 modes x kP2MRC
// coefficients in registers (20 DFMA per 7 shared loads per source).
constexpr int kP2MThreads = 256;
constexpr int kP2MSrc = 32;
constexpr int kP2MModes = 16;
constexpr int kP2MRC = 5;

// 16-byte asynchronous global -> shared copy (zero fill when !valid)
__device__ __forceinline__ void p2m_async16(void *smem, const void *gmem, bool valid)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid ? 16 : 0));
}

__global__ void __launch_bounds__(kP2MThreads) p2m_kernel(FarArgs a)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0, d = a.depth;
    const int nmb = (KW + kP2MModes - 1) / kP2MModes;
    const int slot = blockIdx.x / nmb, n0 = (blockIdx.x % nmb) * kP2MModes;
    const int nm = min(kP2MModes, KW - n0);
    double *mono = sm;                                                  // [kP2MSrc][P]
    double2 *Sx = reinterpret_cast<double2 *>(mono + kP2MSrc * P);      // [kP2MSrc][kP2MModes]
    const uint32_t key = (uint32_t)a.skeys[d][slot];
    double rc, zc, h;
    box_centre(key, d, a.L, a.z0, rc, zc, h);
    const double inv_h = 1.0 / h;
    const int q0 = a.slstart[key], q1 = a.slstart[key + 1];
    const int tn = threadIdx.x % (kP2MModes / 2), tc = threadIdx.x / (kP2MModes / 2);
    const int c0 = tc * kP2MRC;
    const bool active = c0 < P;
    double2 acc[2][kP2MRC];
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int u = 0; u < kP2MRC; ++u) acc[v][u] = make_double2(0.0, 0.0);
    for (int s0 = q0; s0 < q1; s0 += kP2MSrc) {
        const int nc = min(kP2MSrc, q1 - s0);
        __syncthreads();
        if (threadIdx.x < nc) {
            const int q = s0 + threadIdx.x;
            const double dr = (a.sr[q] - rc) * inv_h, dz = (a.sz[q] - zc) * inv_h;
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
        // coefficient rows by asynchronous copies (in flight while the monomials are formed)
        for (int e = threadIdx.x; e < nc * kP2MModes; e += kP2MThreads) {
            const int q = e / kP2MModes, n = e % kP2MModes;
            const bool v = n < nm;
            p2m_async16(Sx + e, v ? a.S + (int64_t)(s0 + q) * a.K + a.m0 + n0 + n : a.S, v);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        if (active) {
            for (int q = 0; q < nc; ++q) {
                const double2 sa = Sx[q * kP2MModes + 2 * tn], sb = Sx[q * kP2MModes + 2 * tn + 1];
                const double *mq = mono + q * P + c0;
#pragma unroll
                for (int u = 0; u < kP2MRC; ++u) {
                    const double m = c0 + u < P ? mq[u] : 0.0;
                    acc[0][u].x = fma(sa.x, m, acc[0][u].x);
                    acc[0][u].y = fma(sa.y, m, acc[0][u].y);
                    acc[1][u].x = fma(sb.x, m, acc[1][u].x);
                    acc[1][u].y = fma(sb.y, m, acc[1][u].y);
                }
            }
        }
    }
    if (active) {
        double2 *Mo = a.M + (a.soff[d] + slot) * (int64_t)KW * P;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int n = n0 + 2 * tn + v;
            if (2 * tn + v >= nm) continue;
#pragma unroll
            for (int u = 0; u < kP2MRC; ++u)
                if (c0 + u < P) Mo[(int64_t)n * P + c0 + u] = acc[v][u];
        }
    }
}

inline size_t p2m_smem(int P)
{
    return sizeof(double) * kP2MSrc * P + sizeof(double2) * kP2MSrc * kP2MModes;
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
// M2M and L2L: constant binomial recentrings in normalised units, applied separably (r, then z).
//   M2M (child c -> parent, d = child - parent = (s_r, s_z) h_parent / 4):
//     T_c[i][j]  = sum_{q<=i} C(i,q) s_r^q 2^-(i+q) M'_c[i-q][j]
//     M^[i][j]   = sum_c sum_{u<=j} C(j,u) s_z^u 2^-(j+u) T_c[i][j-u]
//   L2L (parent -> child c), added to the child's S2L contribution:
//     T[i][m]    = sum_{q: i+q+m<=p} C(i+q,q) s_r^q 2^-(i+2q) L'[i+q][m]
//     L^[i][j]  += 1/2 sum_{u: i+j+u<=p} C(j+u,u) s_z^u 2^-(j+2u) T[i][j+u]
// CTA per (box, group of kMMG modes); coefficient tables built in smem.
constexpr int kMMG = 4;

// Recentring tables, built once per plan on the host (exact binomials times powers of two):
//   cm[s][i][q] = C(i,q) s^q 2^-(i+q);  cl[s][i][q] = C(i+q,q) s^q 2^-(i+2q)   (s = -1, +1)
// out = [cm | cl] (4 (p+1)^2), tri = [tri_i | tri_j] (2 P).
inline void recentre_tables_host(int p, std::vector<double> &out, std::vector<int> &tri)
{
    const int P1 = p + 1, P = (p + 1) * (p + 2) / 2;
    out.assign((size_t)4 * P1 * P1, 0.0);
    for (int e = 0; e < 2 * P1 * P1; ++e) {
        int sgn = e / (P1 * P1), i = (e / P1) % P1, q = e % P1;
        double s = sgn ? 1.0 : -1.0;
        double bm = 0.0, bl = 0.0;
        if (q <= i) {
            double c = 1.0;
            for (int t = 1; t <= q; ++t) c = c * (i - q + t) / t;
            bm = c;
        }
        if (i + q <= p) {
            double c = 1.0;
            for (int t = 1; t <= q; ++t) c = c * (i + t) / t;
            bl = c;
        }
        double sq = (q & 1) ? s : 1.0;
        out[e] = bm * sq * std::ldexp(1.0, -(i + q));
        out[2 * P1 * P1 + e] = bl * sq * std::ldexp(1.0, -(i + 2 * q));
    }
    tri.assign((size_t)2 * P, 0);
    for (int i = 0, q = 0; i <= p; ++i)
        for (int j = 0; i + j <= p; ++j, ++q) {
            tri[q] = i;
            tri[P + q] = j;
        }
}
__device__ __forceinline__ void load_recentre_tables(int p, const double *rtab, const int *tritab,
                                                     double *cm, int *tri_i, int *tri_j)
{
    const int P1 = p + 1, P = (p + 1) * (p + 2) / 2;
    for (int e = threadIdx.x; e < 4 * P1 * P1; e += blockDim.x) cm[e] = __ldg(rtab + e);   // cm, cl
    for (int q = threadIdx.x; q < P; q += blockDim.x) {
        tri_i[q] = __ldg(tritab + q);
        tri_j[q] = __ldg(tritab + P + q);
    }
}


__global__ void __launch_bounds__(256) m2m_kernel(FarArgs a, int level)
{
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0, P1 = p + 1;
    const int ngrp = (KW + kMMG - 1) / kMMG;
    const int slot = blockIdx.x / ngrp, n0 = (blockIdx.x % ngrp) * kMMG;
    const int nm = min(kMMG, KW - n0);
    double *cm = sm, *cl = cm + 2 * P1 * P1;
    double2 *ch = reinterpret_cast<double2 *>(cl + 2 * P1 * P1);   // [4][nm][P]
    double2 *T = ch + 4 * kMMG * P;                                  // [4][nm][P]
    int *tri_i = reinterpret_cast<int *>(T + 4 * kMMG * P);
    int *tri_j = tri_i + P;
    const uint32_t key = (uint32_t)a.skeys[level][slot];
    int cs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) cs[c] = a.smap[level + 1][4 * key + c];
    load_recentre_tables(p, a.rtab_m, a.tritab_m, cm, tri_i, tri_j);   // cl = cm + 2 (p+1)^2
    for (int e = threadIdx.x; e < 4 * nm * P; e += blockDim.x) {
        int c = e / (nm * P), r = e % (nm * P);
        ch[e] = cs[c] >= 0 ? a.M[((a.soff[level + 1] + cs[c]) * (int64_t)KW + n0) * P + r]
                           : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * nm * P; e += blockDim.x) {
        int c = e / (nm * P), r = e % (nm * P), n = r / P, ij = r % P;
        double2 acc = make_double2(0.0, 0.0);
        if (cs[c] >= 0) {
            int i = tri_i[ij], j = tri_j[ij];
            const double *co = cm + ((c & 1) * P1 + i) * P1;
            const double2 *src = ch + (c * nm + n) * P;
            for (int q = 0; q <= i; ++q) {
                double2 v = src[tri(i - q, j, p)];
                acc.x = fma(co[q], v.x, acc.x);
                acc.y = fma(co[q], v.y, acc.y);
            }
        }
        T[e] = acc;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nm * P; r += blockDim.x) {
        int n = r / P, ij = r % P, i = tri_i[ij], j = tri_j[ij];
        double2 acc = make_double2(0.0, 0.0);
        for (int c = 0; c < 4; ++c) {
            if (cs[c] < 0) continue;
            const double *co = cm + (((c >> 1) & 1) * P1 + j) * P1;
            const double2 *src = T + (c * nm + n) * P;
            for (int u = 0; u <= j; ++u) {
                double2 v = src[tri(i, j - u, p)];
                acc.x = fma(co[u], v.x, acc.x);
                acc.y = fma(co[u], v.y, acc.y);
            }
        }
        a.M[((a.soff[level] + slot) * (int64_t)KW + n0) * P + r] = acc;
    }
}

// Lazy downward pass.  A target box's local is materialised only if it, or a target box below
// it, receives an S2L contribution (need = written || any child needs); otherwise it equals the
// re-centred local of its nearest materialised ancestor (L2L is an exact re-centring of a
// degree-p polynomial), and L2P evaluates that ancestor's local directly.  Uniform
// inputs (C2, C3) need every box; surface inputs (C5) skip L2L for most of the 700k boxes.
__global__ void need_kernel(FarArgs a, int level, unsigned char *need)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.tcount[level]) return;
    const uint32_t key = (uint32_t)a.tkeys[level][s];
    bool nd = a.s2l_written[a.lvoff[level] + key] != 0;
    if (level < a.depth)
        for (int c = 0; c < 4 && !nd; ++c) {
            const uint32_t ck = 4 * key + c;
            nd = a.tmap[level + 1][ck] >= 0 && need[a.lvoff[level + 1] + ck] != 0;
        }
    need[a.lvoff[level] + key] = nd ? 1 : 0;
}

// L2L, one warp per (child box, mode), grid-stride over the level's target boxes; separable
// (r then z) binomial re-centring in normalised units with the tables in shared memory.
constexpr int kL2LWarps = 8;
__global__ void __launch_bounds__(32 * kL2LWarps) l2l_kernel(FarArgs a, int level)
{
    extern __shared__ double sm[];
    const int p = a.pl, P = a.Pl, KW = a.m1 - a.m0, P1 = p + 1;   // local order
    double *cm = sm, *cl = cm + 2 * P1 * P1;
    int *tri_i = reinterpret_cast<int *>(cl + 2 * P1 * P1);
    int *tri_j = tri_i + P;
    double2 *wbuf = reinterpret_cast<double2 *>(tri_j + P + 2 * (P & 1));   // 16-B aligned
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2 *par = wbuf + warp * 2 * P, *T = par + P;
    load_recentre_tables(p, a.rtab_l, a.tritab_l, cm, tri_i, tri_j);   // local order
    __syncthreads();
    const int64_t items = (int64_t)a.tcount[level] * KW;
    for (int64_t it = (int64_t)blockIdx.x * kL2LWarps + warp; it < items;
         it += (int64_t)gridDim.x * kL2LWarps) {
        const int slot = (int)(it / KW), n = (int)(it % KW);
        const uint32_t key = (uint32_t)a.tkeys[level][slot];
        if (!a.need[a.lvoff[level] + key]) continue;
        const int ps = a.tmap[level - 1][key >> 2];
        const int sr = key & 1, sz = (key >> 1) & 1;
        const bool child_w = a.s2l_written[a.lvoff[level] + key] != 0;
        const bool par_ok = level - 1 > 2 || a.s2l_written[a.lvoff[level - 1] + (key >> 2)] != 0;
        const double2 *pg = a.Lc + ((a.toff[level - 1] + ps) * (int64_t)KW + n) * P;
        for (int e = lane; e < P; e += 32) par[e] = par_ok ? pg[e] : make_double2(0.0, 0.0);
        __syncwarp();
        for (int e = lane; e < P; e += 32) {
            const int i = tri_i[e], m = tri_j[e];
            const double *co = cl + (sr * P1 + i) * P1;
            double2 acc = make_double2(0.0, 0.0);
            for (int q = 0; i + q + m <= p; ++q) {
                const double2 v = par[tri(i + q, m, p)];
                acc.x = fma(co[q], v.x, acc.x);
                acc.y = fma(co[q], v.y, acc.y);
            }
            T[e] = acc;
        }
        __syncwarp();
        double2 *o = a.Lc + ((a.toff[level] + slot) * (int64_t)KW + n) * P;
        for (int e = lane; e < P; e += 32) {
            const int i = tri_i[e], j = tri_j[e];
            const double *co = cl + (sz * P1 + j) * P1;
            double2 acc = make_double2(0.0, 0.0);
            for (int u = 0; i + j + u <= p; ++u) {
                const double2 v = T[tri(i, j + u, p)];
                acc.x = fma(co[u], v.x, acc.x);
                acc.y = fma(co[u], v.y, acc.y);
            }
            const double2 cur = child_w ? o[e] : make_double2(0.0, 0.0);
            o[e] = make_double2(fma(0.5, acc.x, cur.x), fma(0.5, acc.y, cur.y));
        }
        __syncwarp();
    }
}

inline size_t l2l_smem(int p)
{
    int P = (p + 1) * (p + 2) / 2;
    return sizeof(double) * 4 * (p + 1) * (p + 1) + sizeof(int) * (2 * P + 2) +
           sizeof(double2) * 2 * P * kL2LWarps;
}

inline size_t m2m_smem(int p)
{
    int P = (p + 1) * (p + 2) / 2;
    return sizeof(double) * 4 * (p + 1) * (p + 1) + sizeof(double2) * 8 * kMMG * P + sizeof(int) * 2 * P;
}

// ---------------------------------------------------------------------------------------------
// L2P at the leaves: CTA per (target leaf, mode group of <= 16); writes out rows (input order).
constexpr int kL2PModes = 16;
constexpr int kL2PPts = 16;

// GRAD: also d/dr and d/dz of the local polynomial from the derivative
// monomials k dr^(k-1) dz^l and l dr^k dz^(l-1) (normalised units: an extra 1/h).
template <bool GRAD>
__global__ void __launch_bounds__(256) l2p_kernel(FarArgs a)
{
    extern __shared__ double sm[];
    const int p = a.pl, P = a.Pl, KW = a.m1 - a.m0, d = a.depth;   // local order
    const int ngrp = (KW + kL2PModes - 1) / kL2PModes;
    const int chunk = blockIdx.x / ngrp, g = blockIdx.x % ngrp;
    const int n0 = g * kL2PModes, nm = min(kL2PModes, KW - n0);
    double2 *loc = reinterpret_cast<double2 *>(sm);     // [nm][P]
    double *mono = reinterpret_cast<double *>(loc + kL2PModes * P);  // [pts][P]
    double *monr = mono + kL2PPts * P, *monz = monr + kL2PPts * P;   // GRAD: derivative monomials
    // a CTA takes l2p_lc consecutive target leaves (Morton order, so their field points are one
    // contiguous sorted range) and walks them in runs that share the evaluating box: the local is
    // loaded once per run (C5: leaves of 4 points under coarse boxes)
    const int nleaf = a.tcount[d];
    const int l0 = chunk * a.l2p_lc, l1 = min(nleaf, l0 + a.l2p_lc);
    // the deepest ancestor (or the leaf) that received an S2L contribution: below it the chain
    // adds nothing, so the leaf's local is that box's local re-centred (exact) and is
    // evaluated directly.  Written boxes are always materialised (need_kernel), and the choice
    // depends only on the leaf's own chain, so results do not depend on the other field points
    // (a field-partitioned multi-GPU solve is bitwise identical to the 1-GPU one).  None: zero.
    auto owner = [&](int leaf, int &la, uint32_t &ka) {
        la = d;
        ka = (uint32_t)a.tkeys[d][leaf];
        while (la >= 2 && !a.s2l_written[a.lvoff[la] + ka]) {
            --la;
            ka >>= 2;
        }
        if (la < 2) la = -1;                            // nothing written: zero local
    };
    for (int li = l0; li < l1;) {
    int la;
    uint32_t ka;
    owner(li, la, ka);
    int lj = li + 1;
    for (; lj < l1; ++lj) {
        int lb;
        uint32_t kb;
        owner(lj, lb, kb);
        if (lb != la || (la >= 2 && kb != ka)) break;
    }
    const uint32_t key = (uint32_t)a.tkeys[d][li], keyl = (uint32_t)a.tkeys[d][lj - 1];
    const int t0 = a.flstart[key], t1 = a.flstart[keyl + 1];
    const bool ok = la >= 2;
    if (!ok) {
        la = 2;
        ka = key >> (2 * (d - 2));
    }
    double rc, zc, h;
    box_centre(ka, la, a.L, a.z0, rc, zc, h);
    const double inv_h = 1.0 / h;
    const int64_t aslot = ok ? a.tmap[la][ka] : 0;
    __syncthreads();                                    // the previous run is done with loc
    for (int e = threadIdx.x; e < nm * P; e += blockDim.x)
        loc[e] = ok ? a.Lc[((a.toff[la] + aslot) * (int64_t)KW + n0) * P + e] : make_double2(0.0, 0.0);
    for (int c0 = t0; c0 < t1; c0 += kL2PPts) {
        const int nc = min(kL2PPts, t1 - c0);
        __syncthreads();
        if (threadIdx.x < nc) {
            int t = c0 + threadIdx.x;
            double dr = (a.fr[t] - rc) / h, dz = (a.fz[t] - zc) / h;
            double pr = 1.0, prm = 0.0;   // dr^i and i dr^(i-1)
            for (int i = 0; i <= p; ++i) {
                double pz = pr, pzm = 0.0, pzr = prm;   // dr^i dz^j, j dr^i dz^(j-1), i dr^(i-1) dz^j
                for (int j = 0; i + j <= p; ++j) {
                    mono[threadIdx.x * P + tri(i, j, p)] = pz;
                    if (GRAD) {
                        monr[threadIdx.x * P + tri(i, j, p)] = pzr;
                        monz[threadIdx.x * P + tri(i, j, p)] = pzm;
                    }
                    pzm = (j + 1) * pz;
                    pz *= dz;
                    pzr *= dz;
                }
                prm = (i + 1) * pr;
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
            if (GRAD) {
                const double *mr = monr + t * P, *mz = monz + t * P;
                double rx = 0.0, ry = 0.0, zx = 0.0, zy = 0.0;
                for (int kl = 0; kl < P; ++kl) {
                    rx = fma(lo[kl].x, mr[kl], rx);
                    ry = fma(lo[kl].y, mr[kl], ry);
                    zx = fma(lo[kl].x, mz[kl], zx);
                    zy = fma(lo[kl].y, mz[kl], zy);
                }
                const double s2 = inv_h * inv_h;
                double2 *orr = a.outr + row * a.K + a.m0 + n0 + n, *oz = a.outz + row * a.K + a.m0 + n0 + n;
                if (a.l2p_accumulate) {
                    const double2 cr = *orr, cz = *oz;
                    *orr = make_double2(fma(rx, s2, cr.x), fma(ry, s2, cr.y));
                    *oz = make_double2(fma(zx, s2, cz.x), fma(zy, s2, cz.y));
                } else {
                    *orr = make_double2(rx * s2, ry * s2);
                    *oz = make_double2(zx * s2, zy * s2);
                }
            }
            double2 *o = a.out + row * a.K + a.m0 + n0 + n;
            if (a.l2p_accumulate) {
                const double2 cur = *o;
                *o = make_double2(fma(sx, inv_h, cur.x), fma(sy, inv_h, cur.y));
            } else {
                *o = make_double2(sx * inv_h, sy * inv_h);
            }
        }
    }
    li = lj;
    }   // runs
}

// ---------------------------------------------------------------------------------------------
// S2L, all levels in ONE launch.  CTA per (level, target column i_t, parity
// of j_t, tile of JT target boxes of that parity, mode n); it writes the level's S2L contribution
// only (the L2L chain adds the parents afterwards, top-down; L2L is linear so the sum is the
// paper's L(l) = L2L(L(l-1)) + S2L(l)).  For each of the <= 27 offsets (dI, dJ) of the
// interaction list (children of the parent's neighbours that are not neighbours, P:246-252,
// 539-559) the P x P operator
//     A[(k,l), (i,j)] = sigma C(j+l, j) Gbar^_{A,B, j+l}
// (FO: sigma = (-1)^j, (A,B) = (k,i); BO: (-1)^l, (k,i); FI: (-1)^j, (i,k); BI: (-1)^l, (i,k))
// is factored as A = diag(1/l!) A' diag((-1)^j / j!) with A'[(k,l),(i,j)] = s H_{A,B}(j+l),
// H_{ab}(m) = m! Gbar^_{abm} (stored so by the tensor kernel), s = 1 (FO/FI) or (-1)^{j+l}
// (BO/BI): a pure gather from the station's tensor block, which is copied to smem contiguously.
// The JT source boxes' moments (2 JT real columns, pre-scaled by (-1)^j/j!) are multiplied on
// the CUDA cores by a register-tiled FP64 GEMM; outputs accumulate in registers over the offsets
// in a fixed order (deterministic) and are post-scaled by 1/l! on the write.
template <int NT, int TM, int RM, int RN, int KC, int ST = 2, int PF = 0, int PC = 0>
struct S2LCfg {
    static constexpr int TN = NT / TM;
    static constexpr int MP = TM * RM;          // padded rows (>= P)
    static constexpr int NC = TN * RN;          // columns = 2 JT (even-j boxes, then odd-j boxes)
    static constexpr int NCP = NC + 2;          // smem row stride of B (breaks 512-B bank aliasing)
    static constexpr int JT = NC / 2;           // target boxes per CTA (JT/2 of each parity)
    static constexpr int JH = JT / 2;
    static constexpr int NOFF = 33;             // (dI, dJ) in [6] x [-3..3] minus the 9 near
    static constexpr int STAGES = ST;           // 2: next offset staged behind the GEMM; 1: not
};

struct S2LGrid {
    int nlev;                       // levels 2..depth
    int level[kMaxLevels];
    int jtiles[kMaxLevels];
    int64_t start[kMaxLevels + 1];  // tile prefix per level entry; tile = (column it, row tile jt)
};

// Tile activity for S2L: one warp per tile (level, target column it, row tile jt of JT = 2 JH
// target boxes, JH of each parity).  A tile is active iff some target box in it has a non-empty
// source box in its interaction list (children of the parent's neighbours that are not
// neighbours); every target box of an active tile is written by S2L, the
// others are marked unwritten (their S2L contribution is zero).
struct TileArgs {
    const int *smap[kMaxLevels], *tmap[kMaxLevels];
    int64_t lvoff[kMaxLevels];
};
__global__ void s2l_tile_flags_kernel(TileArgs ta, S2LGrid gr, int JH, int *active,
                                      unsigned char *written)
{
    const int lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= gr.start[gr.nlev]) return;
    int e = 0;
    while (e + 1 < gr.nlev && t >= gr.start[e + 1]) ++e;
    const int level = gr.level[e], jtiles = gr.jtiles[e];
    const int64_t tl = t - gr.start[e];
    const int jt = (int)(tl % jtiles), it = (int)(tl / jtiles);
    const int nb = 1 << level, JT = 2 * JH;
    const int di0 = (it & 1) ? -3 : -2;
    const int *tmap = ta.tmap[level], *smap = ta.smap[level];
    bool any = false;
    // no early exit: the unrolled loop keeps several map lookups in flight per lane
#pragma unroll 6
    for (int q = lane; q < 42 * JT; q += 32) {
        const int o = q / JT, b = q % JT;
        const int di = di0 + o / 7, dj = o % 7 - 3;
        if (di >= -1 && di <= 1 && dj >= -1 && dj <= 1) continue;
        const int par = b / JH, jtb = 2 * (jt * JH + (b % JH)) + par;
        const int is = it + di, js = jtb + dj;
        if (jtb >= nb || is < 0 || is >= nb || js < 0 || js >= nb) continue;
        if ((dj == 3 && par == 1) || (dj == -3 && par == 0)) continue;
        if (tmap[morton2((uint32_t)it, (uint32_t)jtb)] < 0) continue;
        if (smap[morton2((uint32_t)is, (uint32_t)js)] >= 0) any = true;
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) active[t] = any ? 1 : 0;
    for (int b = lane; b < JT; b += 32) {
        const int jtb = 2 * (jt * JH + (b % JH)) + b / JH;
        if (jtb < nb) {
            const uint32_t key = morton2((uint32_t)it, (uint32_t)jtb);
            if (tmap[key] >= 0) written[ta.lvoff[level] + key] = any ? 1 : 0;
        }
    }
}

// compact list of active tiles (pos = exclusive scan of active)
__global__ void s2l_tile_emit_kernel(const int *active, const int *pos, int64_t ntiles, int *tiles,
                                     int *count)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    if (active[t]) tiles[pos[t]] = (int)t;
    if (t == ntiles - 1) *count = pos[t] + active[t];
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;   // src-size 0: zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// Bulk (TMA, 1-D) global -> shared copies completing on an mbarrier (sm_90+/sm_100a).
__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int RM, int RN, int TM, int TN, int MP, int NC, int MASK, int PF>
__device__ __forceinline__ void s2l_gemm(const double *As, const double *Bs, int kc, int tm,
                                         int tn, double (&acc)[RM][RN])
{
    if constexpr (PF) {
        // register double buffer: fragments of kk + 1 are loaded before the FMAs of kk
        double av[2][RM], bv[2][RN];
        auto load = [&](int kk, int b) {
#pragma unroll
            for (int u = 0; u < RM / 2; ++u) {
                double2 t = *reinterpret_cast<const double2 *>(As + kk * MP + 2 * (tm + TM * u));
                av[b][2 * u] = t.x;
                av[b][2 * u + 1] = t.y;
            }
#pragma unroll
            for (int v = 0; v < RN; ++v)
                if (MASK & (1 << v)) bv[b][v] = Bs[kk * NC + tn + TN * v];
        };
        load(0, 0);
        int kk = 0;
        for (; kk + 1 < kc; kk += 2) {
            load(kk + 1, 1);
#pragma unroll
            for (int u = 0; u < RM; ++u)
#pragma unroll
                for (int v = 0; v < RN; ++v)
                    if (MASK & (1 << v)) acc[u][v] = fma(av[0][u], bv[0][v], acc[u][v]);
            if (kk + 2 < kc) load(kk + 2, 0);
#pragma unroll
            for (int u = 0; u < RM; ++u)
#pragma unroll
                for (int v = 0; v < RN; ++v)
                    if (MASK & (1 << v)) acc[u][v] = fma(av[1][u], bv[1][v], acc[u][v]);
        }
        if (kk < kc) {
#pragma unroll
            for (int u = 0; u < RM; ++u)
#pragma unroll
                for (int v = 0; v < RN; ++v)
                    if (MASK & (1 << v)) acc[u][v] = fma(av[0][u], bv[0][v], acc[u][v]);
        }
        return;
    }
#pragma unroll 3
    for (int kk = 0; kk < kc; ++kk) {
        double av[RM], bv[RN];
#pragma unroll
        for (int u = 0; u < RM / 2; ++u) {
            double2 t = *reinterpret_cast<const double2 *>(As + kk * MP + 2 * (tm + TM * u));
            av[2 * u] = t.x;
            av[2 * u + 1] = t.y;
        }
#pragma unroll
        for (int v = 0; v < RN; ++v)
            if (MASK & (1 << v)) bv[v] = Bs[kk * NC + tn + TN * v];
#pragma unroll
        for (int u = 0; u < RM; ++u)
#pragma unroll
            for (int v = 0; v < RN; ++v)
                if (MASK & (1 << v)) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
}

template <int RM, int RN, int TM, int TN, int MP, int NC, int M, int PF>
__device__ __forceinline__ void s2l_gemm_dispatch(int mask, const double *As, const double *Bs,
                                                  int kc, int tm, int tn, double (&acc)[RM][RN])
{
    if constexpr (M > 0) {
        if (mask == M) {
            s2l_gemm<RM, RN, TM, TN, MP, NC, M, PF>(As, Bs, kc, tm, tn, acc);
            return;
        }
        s2l_gemm_dispatch<RM, RN, TM, TN, MP, NC, M - 1, PF>(mask, As, Bs, kc, tm, tn, acc);
    }
}

// Blocked-column GEMM (PF == 2): thread tn owns the RN consecutive columns tn*RN.. (RN/2 whole
// boxes), so B fragments load as 16-byte vectors and a whole warp can skip an offset none of its
// boxes interacts with (warp-uniform branch, no mask instantiations).
template <int RM, int RN, int TM, int MP, int NC>
__device__ __forceinline__ void s2l_gemm_blk(const double *As, const double *Bs, int kc, int tm,
                                             int tn, double (&acc)[RM][RN])
{
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
        for (int v = 0; v < RN / 2; ++v) {
            double2 t = *reinterpret_cast<const double2 *>(Bs + kk * NC + tn * RN + 2 * v);
            bv[2 * v] = t.x;
            bv[2 * v + 1] = t.y;
        }
#pragma unroll
        for (int u = 0; u < RM; ++u)
#pragma unroll
            for (int v = 0; v < RN; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
}

// Box-major GEMM (PF == 3): B staged by bulk copies as [box][BPS] complex rows (BPS odd: the
// four boxes a warp reads per step fall in distinct bank groups); thread tn owns boxes
// tn*RN/2 .. +RN/2-1 (both re and im columns of each).
template <int RM, int RN, int TM, int MP>
__device__ __forceinline__ void s2l_gemm_box(const double *As, const double2 *Bs, int BPS, int kc,
                                             int tm, int tn, double (&acc)[RM][RN])
{
    const double2 *Bt = Bs + (tn * RN / 2) * BPS;
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
        for (int v = 0; v < RN / 2; ++v) {
            double2 t = Bt[v * BPS + kk];
            bv[2 * v] = t.x;
            bv[2 * v + 1] = t.y;
        }
#pragma unroll
        for (int u = 0; u < RM; ++u)
#pragma unroll
            for (int v = 0; v < RN; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
}

template <int NT, int TM, int RM, int RN, int KC, int ST, int PF, int PC>
__global__ void __launch_bounds__(NT, (RM * RN >= 40 ? 256 : 512) / NT) s2l_kernel(FarArgs a, S2LGrid gr)
{
    using Cfg = S2LCfg<NT, TM, RM, RN, KC, ST, PF, PC>;
    constexpr int TN = Cfg::TN, MP = Cfg::MP, NC = Cfg::NCP, JT = Cfg::JT, JH = Cfg::JH;
    constexpr int NOFF = Cfg::NOFF;
    constexpr int BOXV = TN / 2;                   // boxes per column block v
    extern __shared__ double sm[];
    // PC > 0: the expansion order is a compile-time constant (BASELINE orders 8, 12, 16), so
    // every index division below is by a constant
    // p, P: source order and size (GEMM depth); pl, Pl: local order and size (GEMM rows, <= MP);
    // pt = max(p, pl): tensor order.  PC > 0 implies p = pl = PC.
    const int p = PC ? PC : a.p, P = PC ? (PC + 1) * (PC + 2) / 2 : a.P, KW = a.m1 - a.m0;
    const int pl = PC ? PC : a.pl, Pl = PC ? P : a.Pl, pt = PC ? PC : a.pt;
    const int TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1), HST = TPp + 2;
    constexpr bool TMA = PF == 3;                  // box-major B staged by bulk copies
    const int BPS = P | 1;                         // TMA: complex row stride per box (odd)
    double *As = sm;                               // [KC][MP]
    double *Bs0 = As + KC * MP;                    // ST x [P][NC] (TMA: [JT][BPS] complex)
    double *Hs0 = Bs0 + (TMA ? ST * 2 * JT * BPS : ST * P * NC);   // ST x [HST], Hs[TPp] = 0
    uint64_t *bar = reinterpret_cast<uint64_t *>(Hs0 + ST * HST);   // TMA barriers, one per stage
    double *post = reinterpret_cast<double *>(bar + 2);            // [Pl] 1 / l!
    int *tsl = reinterpret_cast<int *>(post + Pl); // [JT]  (box b: parity b / JH, index b % JH)
    int *ssl = tsl + JT;                           // [NOFF][JT]
    int *olist = ssl + NOFF * JT;                  // [NOFF] active offsets
    int *nact = olist + NOFF;
    unsigned *omask = reinterpret_cast<unsigned *>(nact + 1);   // [NOFF] boxes with a source
    constexpr bool BLK = PF >= 2;                  // blocked columns (box-aligned per thread)
    static_assert(!BLK || JT <= 32, "box bit masks are 32-bit");

    const int nloc = (int)(blockIdx.x % KW);
    int64_t bid = a.s2l_tiles[blockIdx.x / KW];      // active tile (s2l_tile_flags_kernel)
    int e = 0;
    while (e + 1 < gr.nlev && bid >= gr.start[e + 1]) ++e;
    const int level = gr.level[e], jtiles = gr.jtiles[e];
    bid -= gr.start[e];
    const int jt = (int)(bid % jtiles);
    const int it = (int)(bid / jtiles);
    const int nb = 1 << level;
    const int tid = threadIdx.x;
    const int tm = tid % TM, tn = tid / TM;
    const int di0 = (it & 1) ? -3 : -2;
    auto jt_of = [&](int b) { return 2 * (jt * JH + (b % JH)) + b / JH; };  // target j of box b

    int anyt = 0;
    if (tid < JT) {
        int jtb = jt_of(tid);
        int s = -1;
        if (jtb < nb) s = a.tmap[level][morton2((uint32_t)it, (uint32_t)jtb)];
        tsl[tid] = s;
        anyt = s >= 0;
    }
    if (!__syncthreads_or(anyt)) return;
    // the 33 offsets in a fixed order, then the source slots of every (offset, box) in one pass
    // (dj = 0, -1, +1, -2, +2, -3, +3 per column: the forward / backward partners of a column
    // are adjacent, so the backward one can reuse the gathered operator, see below)
    if (tid == 0) {
        int k = 0;
        for (int di = di0; di <= di0 + 5; ++di)
            for (int t = 0; t < 7; ++t) {
                const int dj = (t & 1) ? -((t + 1) >> 1) : (t >> 1);
                if (di >= -1 && di <= 1 && dj >= -1 && dj <= 1) continue;
                olist[k++] = ((di + 3) << 4) | (dj + 3);
            }
    }
    for (int q = tid; q < Pl; q += NT) {   // target coefficient (k, l), local order pl
        int i = 0;
        while (i < pl && q >= (i + 1) * (pl + 1) - (i + 1) * i / 2) ++i;
        int l = q - (i * (pl + 1) - i * (i - 1) / 2);
        double f = 1.0;
        for (int t = 2; t <= l; ++t) f *= t;
        post[q] = 1.0 / f;
    }
    if (tid < ST) Hs0[tid * HST + TPp] = 0.0;
    if (TMA && tid == 0) {
        for (int b = 0; b < ST; ++b) mbar_init(bar + b, 1);
        fence_mbar_init();
    }
    __syncthreads();
    for (int q = tid; q < NOFF * JT; q += NT) {
        int o = q / JT, b = q % JT;
        int code = olist[o];
        int di = (code >> 4) - 3, dj = (code & 15) - 3;
        int is = it + di, jtb = jt_of(b), js = jtb + dj;
        int par = b / JH;
        bool ok = tsl[b] >= 0 && is >= 0 && is < nb && js >= 0 && js < nb &&
                  !(dj == 3 && par == 1) && !(dj == -3 && par == 0);
        ssl[q] = ok ? a.smap[level][morton2((uint32_t)is, (uint32_t)js)] : -1;
    }
    __syncthreads();
    // compact the active offsets (fixed order) with their column-block masks
    if (BLK && tid < 32) {
        // warp 0: one ballot per offset over the (<= 32) boxes
        int k = 0;
        unsigned long long npairs = 0;
        for (int o = 0; o < NOFF; ++o) {
            // TMA path: (di, -3) reaches only odd target boxes and (di, +3) only even ones
            // (parity rule of the interaction list), so the pair is one merged offset: the odd
            // boxes' sources from (di, -3), the even boxes' from (di, +3) (signs: see `mg`)
            const int oc = olist[o];
            const bool mrg = TMA && (oc & 15) == 0;
            bool has = tid < JT && ssl[o * JT + tid] >= 0;
            if (mrg && tid < JT) {
                const int sp = ssl[(o + 1) * JT + tid];
                if (sp >= 0) {
                    ssl[o * JT + tid] = sp;
                    has = true;
                }
            }
            const unsigned bm = __ballot_sync(0xffffffffu, has);
            if (bm) {
                npairs += __popc(bm);
                if (tid == 0) {
                    omask[k] = bm;
                    olist[k] = (oc & 0xff) | (o << 8) | (mrg ? 1 << 24 : 0);
                }
                ++k;
            }
            if (mrg) ++o;
        }
        if (tid == 0) {
            *nact = k;
            if (nloc == 0 && a.m0 == 0 && a.s2l_pairs && npairs) atomicAdd(a.s2l_pairs, npairs);
        }
    } else if (!BLK && tid == 0) {
        int k = 0;
        unsigned long long npairs = 0;
        for (int o = 0; o < NOFF; ++o) {
            int mask = 0, cnt = 0;
            unsigned bm = 0;
            for (int b = 0; b < JT; ++b)
                if (ssl[o * JT + b] >= 0) {
                    ++cnt;
                    mask |= 1 << ((2 * b) / TN);   // column block of box b (strided layout)
                    bm |= 1u << b;                  // box bit (blocked layout)
                }
            if (!cnt) continue;
            npairs += cnt;
            omask[k] = bm;
            olist[k++] = (olist[o] & 0xff) | (o << 8) | (mask << 16);
        }
        *nact = k;
        if (nloc == 0 && a.m0 == 0 && a.s2l_pairs && npairs) atomicAdd(a.s2l_pairs, npairs);
    }
    __syncthreads();
    const int na = *nact;

    double acc[RM][RN];
#pragma unroll
    for (int u = 0; u < RM; ++u)
#pragma unroll
        for (int v = 0; v < RN; ++v) acc[u][v] = 0.0;
    // boxes covered by this warp (blocked layout: thread tn owns boxes tn*RN/2 .. +RN/2-1)
    unsigned wbox = 0;
    if constexpr (BLK) {
        unsigned mine = 0;
#pragma unroll
        for (int v = 0; v < RN; v += 2) mine |= 1u << ((tn * RN + v) >> 1);
        wbox = __reduce_or_sync(0xffffffffu, mine);
    }

    // reuse masks: moment coefficients kk with odd j; this thread's accumulator rows with odd l
    unsigned long long oddj = 0;
    unsigned oddl = 0;
    if (PF == 3) {
        for (int i = 0, q = 0; i <= p; ++i)
            for (int j = 0; i + j <= p; ++j, ++q)
                if ((j & 1) && q < 64) oddj |= 1ull << q;   // used only when P <= 64 (reuse)
#pragma unroll
        for (int r = 0; r < RM; ++r) {
            const int m = 2 * (tm + TM * (r >> 1)) + (r & 1);
            if (m < Pl) {
                int kq = 0;
                while (kq < pl && m >= (kq + 1) * (pl + 1) - (kq + 1) * kq / 2) ++kq;
                if ((m - (kq * (pl + 1) - kq * (kq - 1) / 2)) & 1) oddl |= 1u << r;
            }
        }
    }
    auto negate_oddl = [&]() {
#pragma unroll
        for (int r = 0; r < RM; ++r)
            if ((oddl >> r) & 1u) {
#pragma unroll
                for (int v = 0; v < RN; ++v) acc[r][v] = -acc[r][v];
            }
    };
    // async stage of offset k into buffer (k % ST): tensor block + (pre-scaled) moments
    auto stage = [&](int k) {
        const int code = olist[k];
        const int di = ((code >> 4) & 15) - 3, dj = (code & 15) - 3, o = (code >> 8) & 0xff;
        const int is = it + di;
        const int iin = min(it, is), dI = di < 0 ? -di : di, dJ = dj < 0 ? -dj : dj;
        const double *Tn = a.tens + ((int64_t)(iin * 12 + class_of(dI, dJ)) * KW + nloc) * TPp;
        double *Hs = Hs0 + (k % ST) * HST;
        double *Bs = Bs0 + (k % ST) * P * NC;
        for (int q = tid; q < TPp / 2; q += NT) cp_async16(Hs + 2 * q, Tn + 2 * q, true);
        for (int q = tid; q < P * JT; q += NT) {
            int b = q / P, kk = q % P;
            int s = ssl[o * JT + b];
            const double2 *src = a.M + ((a.soff[level] + (s >= 0 ? s : 0)) * (int64_t)KW + nloc) * P + kk;
            cp_async16(Bs + kk * NC + 2 * b, src, s >= 0);
        }
        cp_async_commit();
    };
    // TMA stage of offset k into buffer bf: the station's tensor block and one bulk copy per
    // source box; rows of boxes without a source at this offset are zeroed by plain stores.
    // The caller guarantees no thread still reads buffer bf (a block barrier precedes).
    // Operator reuse (single-stage TMA path, whole operator in As): a backward offset (di, +a)
    // right after its forward partner (di, -a) has the same station tensor and the same gathered
    // A' up to the sign (-1)^{j+l} = (-1)^j (-1)^l: it negates the odd-j moment
    // coefficients and the odd-l accumulator rows around its GEMM instead of re-gathering.
    auto reuse_of = [&](int k) -> bool {
        if (!(PF == 3 && ST == 1) || P > KC || P > 64 || k == 0) return false;   // oddj: 64 bits
        const int c = olist[k], cq = olist[k - 1];
        const int dj = (c & 15) - 3, djq = (cq & 15) - 3;
        return ((c >> 4) & 15) == ((cq >> 4) & 15) && dj > 0 && dj == -djq;
    };
    auto tma_issue = [&](int k, int bf) {
        const int code = olist[k];
        const int di = ((code >> 4) & 15) - 3, dj = (code & 15) - 3, o = (code >> 8) & 0xff;
        const int is = it + di;
        const int iin = min(it, is), dI = di < 0 ? -di : di, dJ = dj < 0 ? -dj : dj;
        const double *Tn = a.tens + ((int64_t)(iin * 12 + class_of(dI, dJ)) * KW + nloc) * TPp;
        double2 *Bs = reinterpret_cast<double2 *>(Bs0) + (size_t)bf * JT * BPS;
        const unsigned bm = omask[k];
        const bool ru = reuse_of(k);
        if (tid < 32) {
            if (tid == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(bar + bf, (unsigned)((ru ? 0 : TPp * 8) + __popc(bm) * P * 16));
                if (!ru) bulk_g2s(Hs0 + bf * HST, Tn, (unsigned)(TPp * 8), bar + bf);
            }
            __syncwarp();
            if (tid < JT && ((bm >> tid) & 1u)) {
                const int sl = ssl[o * JT + tid];
                bulk_g2s(Bs + tid * BPS, a.M + ((a.soff[level] + sl) * (int64_t)KW + nloc) * P,
                         (unsigned)(P * 16), bar + bf);
            }
        }
        for (int b = tid >> 5; b < JT; b += NT / 32)
            if (!((bm >> b) & 1u))
                for (int kk = tid & 31; kk < P; kk += 32) Bs[b * BPS + kk] = make_double2(0.0, 0.0);
    };
    if (TMA && na > 0) tma_issue(0, 0);
    if (!TMA && ST == 2 && na > 0) stage(0);
    for (int k = 0; k < na; ++k) {
        const int buf = ST == 2 ? (k & 1) : 0;
        if (TMA) {
            if (ST == 1 && k > 0) {
                __syncthreads();              // GEMM k-1 done with the single buffer and As
                tma_issue(k, 0);
            }
            mbar_wait(bar + buf, (unsigned)((ST == 2 ? (k >> 1) : k) & 1));
        } else {
            if (ST == 1) {
                if (k > 0) __syncthreads();   // GEMM k-1 done with the single buffer
                stage(k);
            }
            cp_async_wait_all();
        }
        // buffer k ready (zero rows visible); As free.  Single-stage TMA: As is free since the
        // barrier before tma_issue, the bulk copies are visible after mbar_wait, and the zero
        // rows (stored by tma_issue) become visible at the barrier after the gather / negation
        // below, before any GEMM reads them (negations touch only TMA-written rows)
        if (!(TMA && ST == 1)) __syncthreads();
        if (!TMA && ST == 2 && k + 1 < na) stage(k + 1);   // overlaps the build and GEMM below
        const int code = olist[k];
        const int di = ((code >> 4) & 15) - 3, dj = (code & 15) - 3;
        const int mask = (code >> 16) & 0xff;
        const int variant = (di <= 0 ? 0 : 2) + (dj <= 0 ? 0 : 1);   // FO, BO, FI, BI
        const int *itab = a.s2l_idx + (size_t)variant * P * MP;
        const double *Hs = Hs0 + buf * HST;
        const double *Bs = Bs0 + buf * P * NC;
        const double2 *Bt = reinterpret_cast<const double2 *>(Bs0) + (size_t)buf * JT * BPS;
        const bool ru = reuse_of(k);
        // merged (di, -3) / (di, +3) offset: the operator is the forward one; the even boxes'
        // (+3) part is its backward partner, (-1)^j on their moments and (-1)^l on their
        // accumulator rows around the GEMM, as for the operator reuse below
        const bool mg = TMA && ((code >> 24) & 1);
        const bool evenT = (tn * RN / 2) < JH;
        if (mg) {
            double2 *Bw = reinterpret_cast<double2 *>(Bs0) + (size_t)buf * JT * BPS;
            const unsigned bmk = omask[k];
            for (int q = tid; q < JH * (p + 1); q += NT) {
                const int b = q / (p + 1), i = q - b * (p + 1);
                if (!((bmk >> b) & 1u)) continue;
                const int q0 = i * (p + 1) - i * (i - 1) / 2;
                for (int j = 1; i + j <= p; j += 2) {
                    const double2 v = Bw[b * BPS + q0 + j];
                    Bw[b * BPS + q0 + j] = make_double2(-v.x, -v.y);
                }
            }
            __syncthreads();
            if (evenT) negate_oddl();
        }
        if (ru) {                             // A' of the forward partner stays in As
            double2 *Bw = reinterpret_cast<double2 *>(Bs0) + (size_t)buf * JT * BPS;
            const unsigned bmk = omask[k];
            for (int q = tid; q < JT * P; q += NT) {
                const int b = q / P, kk = q - b * P;
                if (((oddj >> kk) & 1ull) && ((bmk >> b) & 1u)) {
                    const double2 v = Bw[b * BPS + kk];
                    Bw[b * BPS + kk] = make_double2(-v.x, -v.y);
                }
            }
            __syncthreads();
            negate_oddl();
        }
        for (int k0 = 0; k0 < P; k0 += KC) {
            const int kc = min(KC, P - k0);
            if (k0 > 0) __syncthreads();
            // A'[kk][m] = +-H_{A,B}(j+l): gather through the precomputed (index, sign) table
            if (!ru) {
            for (int q = tid; q < kc * MP; q += NT) {
                int c = __ldg(itab + k0 * MP + q);
                double v = Hs[c >> 1];
                As[q] = (c & 1) ? -v : v;
            }
            __syncthreads();
            }
            // double-buffered TMA: the next offset's copies start now (every thread is past the
            // GEMM that read buffer (k+1) & 1) and land behind this GEMM
            if (TMA && ST == 2 && k0 == 0 && k + 1 < na) tma_issue(k + 1, (k + 1) & 1);
            if constexpr (TMA) {
                if (omask[k] & wbox)
                    s2l_gemm_box<RM, RN, TM, MP>(As, Bt + k0, BPS, kc, tm, tn, acc);
            } else if constexpr (BLK) {
                if (omask[k] & wbox) s2l_gemm_blk<RM, RN, TM, MP, NC>(As, Bs + k0 * NC, kc, tm, tn, acc);
            } else {
                s2l_gemm_dispatch<RM, RN, TM, TN, MP, NC, (1 << RN) - 1, PF>(mask, As, Bs + k0 * NC,
                                                                            kc, tm, tn, acc);
            }
        }
        if (ru || (mg && evenT)) negate_oddl();   // back to the forward sign
        if (TMA && ST == 2) __syncthreads();  // As is rebuilt for the next offset
    }
    (void)BOXV;
    // write the level's S2L contribution (post-scaled by 1/l!); every target of the tile is
    // written, zeros included, so the locals need no initialisation
#pragma unroll
    for (int v = 0; v < RN; ++v) {
        int col = BLK ? tn * RN + v : tn + TN * v, b = col >> 1, im = col & 1;
        int s = tsl[b];
        if (s < 0) continue;
        double *dst = reinterpret_cast<double *>(a.Lc + ((a.toff[level] + s) * (int64_t)KW + nloc) * Pl);
#pragma unroll
        for (int u = 0; u < RM; ++u) {
            int m = 2 * (tm + TM * (u >> 1)) + (u & 1);
            if (m < Pl) dst[2 * m + im] = acc[u][v] * post[m];
        }
    }
}

// Host: (index << 1 | negate) gather table of A'[kk][m] for the 4 variants (FO, BO, FI, BI),
// rows padded to MP; masked / padded entries point at the zero slot TPp.
inline void build_s2l_index(int p, int pl, int MP, int truncation, std::vector<int> &tab)
{
    // rows kk = (i, j): source coefficients of order p; columns m = (k, l): local order pl;
    // entries H_{A,B}(j + l) of the tensor of order pt = max(p, pl) (packed layout)
    const int pt = p > pl ? p : pl;
    const int P = (p + 1) * (p + 2) / 2, Pl = (pl + 1) * (pl + 2) / 2;
    const int TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1);
    std::vector<int> ti(P), tj(P), tk(Pl), tl(Pl);
    for (int i = 0, q = 0; i <= p; ++i)
        for (int j = 0; i + j <= p; ++j, ++q) {
            ti[q] = i;
            tj[q] = j;
        }
    for (int k = 0, q = 0; k <= pl; ++k)
        for (int l = 0; k + l <= pl; ++l, ++q) {
            tk[q] = k;
            tl[q] = l;
        }
    tab.assign((size_t)4 * P * MP, TPp << 1);
    for (int var = 0; var < 4; ++var) {
        const bool outward = var < 2, fwd = (var & 1) == 0;
        for (int kk = 0; kk < P; ++kk)
            for (int m = 0; m < Pl; ++m) {
                int i = ti[kk], j = tj[kk], k = tk[m], l = tl[m];
                if (truncation == 1 && i + j + k + l > p) continue;
                int A = outward ? k : i, B = outward ? i : k;
                int idx = packed_off(A, B, pt) + j + l;
                int neg = (!fwd && ((j + l) & 1)) ? 1 : 0;
                tab[((size_t)var * P + kk) * MP + m] = (idx << 1) | neg;
            }
    }
}

// Source moments pre-scaled once for S2L: M'_ij = (-1)^j M^_ij / j! (all levels, after M2M).
__global__ void prescale_moments_kernel(double2 *M, int64_t nrows, int P, const double *pscale)
{
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nrows * P) return;
    const double f = __ldg(pscale + (int)(e % P));   // (-1)^j / j! of coefficient (i, j)
    double2 v = M[e];
    M[e] = make_double2(v.x * f, v.y * f);
}

template <int NT, int TM, int RM, int RN, int KC, int ST, int PF, int PC>
inline size_t s2l_smem_bytes(int p, int pl)
{
    using Cfg = S2LCfg<NT, TM, RM, RN, KC, ST, PF, PC>;
    const int pt = p > pl ? p : pl;
    int P = (p + 1) * (p + 2) / 2, TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1);
    P = P > (pl + 1) * (pl + 2) / 2 ? P : (pl + 1) * (pl + 2) / 2;   // post[] of Pl, B rows of P
    const size_t bsz = PF == 3 ? (size_t)ST * 2 * Cfg::JT * (P | 1) : ST * (size_t)P * Cfg::NCP;
    return sizeof(double) * ((size_t)KC * Cfg::MP + bsz + ST * (TPp + 2) + 2 + P) +
           sizeof(int) * (Cfg::JT + Cfg::NOFF * Cfg::JT + 2 * Cfg::NOFF + 1);
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
