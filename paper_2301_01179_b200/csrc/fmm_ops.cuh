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
    double2 *Lc;         // locals   [materialised box (lrow)][KW][Pl]
    const int *slstart, *flstart;
    const double *sr, *sz;
    const double2 *S;    // sorted sources [ns][K]
    const double *fr, *fz;
    const int *fperm;
    double2 *out;        // [nf][K], input field order
    const double *tens;  // [12 * 2^d][KW][(p+1)^3] packed
    const unsigned char *s2l_written;   // dense per level [lvoff[l] + key]: local written by S2L
    int64_t lvoff[kMaxLevels];          // dense per-level offsets (level maps, s2l_written)
    const unsigned char *need;          // dense per level: local materialised (see need_kernel)
    const int *lrow;                    // dense per level: Lc row of a materialised local
    const int64_t *rowkey;              // Lc row -> dense position (lvoff[l] + key)
    int lrow_lev[kMaxLevels + 1];       // first Lc row of each level (rows are level-major)
    int l2p_accumulate;                 // L2P adds onto out (the near field wrote it first)
    int64_t tfield;                     // field points (L2P)
    int l2p_tp;                         // L2P threads per task
    int l2p_run;                        // L2P task size (points): l2p_tp x points per thread
    int p2m_slot0;                      // P2M: first leaf slot (multi-device split)
    int p2m_level;                      // P2M: level of the boxes (0: the leaf level d)
    int sigma;                          // adaptive source tree leaf size (R#26), 0 = uniform
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
// CTA per (source leaf, block of <= kP2MModes modes); sources streamed through shared memory in
// chunks of kP2MSrc (monomials computed once per chunk).  Warp w owns nv_w of the block's modes
// (the nm modes dealt as evenly as 4 warps allow: 13 = 4 + 3 + 3 + 3, a compile-time count per
// warp: no mode slot multiplies zeros), lane = RC coefficients: thread tile nv x RC in registers,
// the coefficient row read as warp broadcasts, the monomials from a lane-major layout
// (slot(c) = (c % RC) * 32 + c / RC: conflict-free).  (Before: every warp held 4 x 4 mode slots,
// 16 for K = 65's blocks of 13, 19% of the FP64 issue on zero rows; ncu FP64 pipe 50%.)
constexpr int kP2MSrc = 32;
constexpr int kP2MModes = 16;
constexpr int kP2MTM = 4;                                    // modes per thread (at most)
constexpr int kP2MThreads = (kP2MModes / kP2MTM) * 32;
// coefficients per lane RC = 2 / 3 / 5 by order (32 RC >= P: p <= 9 / 12 / 16), so that most
// lanes hold coefficients at every order (RC = 5 at p = 8 left 23 of 32 lanes idle)
__host__ __device__ constexpr int p2m_rc(int P) { return P <= 64 ? 2 : (P <= 96 ? 3 : 5); }

// 16-byte asynchronous global -> shared copy (zero fill when !valid)
__device__ __forceinline__ void p2m_async16(void *smem, const void *gmem, bool valid)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid ? 16 : 0));
}

template <int NV, int kP2MRC>
__device__ __forceinline__ void p2m_chunk(const double2 *Sx, const double *mono, int nc, int lane,
                                          double2 (&acc)[kP2MTM][kP2MRC])
{
    constexpr int kP2MRow = 32 * kP2MRC;
    for (int q = 0; q < nc; ++q) {
        double2 sv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sv[v] = Sx[q * kP2MModes + v];
        const double *mq = mono + q * kP2MRow + lane;
#pragma unroll
        for (int u = 0; u < kP2MRC; ++u) {
            const double m = mq[u * 32];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                acc[v][u].x = fma(sv[v].x, m, acc[v][u].x);
                acc[v][u].y = fma(sv[v].y, m, acc[v][u].y);
            }
        }
    }
}

template <int kP2MRC>
__global__ void __launch_bounds__(kP2MThreads, 4) p2m_kernel(FarArgs a)
{
    constexpr int kP2MRow = 32 * kP2MRC, NE = (kP2MRow + kP2MThreads - 1) / kP2MThreads;
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, KW = a.m1 - a.m0, d = a.depth;
    // balanced mode blocks of <= kP2MModes (K = 65: 5 x 13, not 4 x 16 + 1)
    const int nmb = (KW + kP2MModes - 1) / kP2MModes;
    const int mb = blockIdx.x % nmb;
    const int slot = a.p2m_slot0 + blockIdx.x / nmb, n0 = (KW * mb) / nmb;
    const int nm = (KW * (mb + 1)) / nmb - n0;
    double *mono = sm;                                                  // [kP2MSrc][kP2MRow]
    double2 *Sx = reinterpret_cast<double2 *>(mono + kP2MSrc * kP2MRow);   // [kP2MSrc][kP2MModes]
    double *pw = reinterpret_cast<double *>(Sx + kP2MSrc * kP2MModes);  // [kP2MSrc][2][p+1]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // this thread's monomial slots s = tid, tid + 128 (coefficient c = RC (s % 32) + s / 32)
    int ci[NE], cj[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const int sl = threadIdx.x + e * kP2MThreads;
        const int c = kP2MRC * (sl % 32) + sl / 32;
        ci[e] = cj[e] = -1;
        if (sl < kP2MRow && c < P) {
            int i = 0;
            while (i < p && c >= (i + 1) * (p + 1) - (i + 1) * i / 2) ++i;
            ci[e] = i;
            cj[e] = c - (i * (p + 1) - i * (i - 1) / 2);
        } else if (sl < kP2MRow) {
            for (int qq = 0; qq < kP2MSrc; ++qq) mono[qq * kP2MRow + sl] = 0.0;   // slots past P
        }
    }
    // level lv (adaptive source tree: every level, leaves only; uniform: the leaf level d)
    const int lv = a.p2m_level ? a.p2m_level : d, sh = 2 * (d - lv);
    const uint32_t key = (uint32_t)a.skeys[lv][slot];
    const int q0 = a.slstart[(int64_t)key << sh], q1 = a.slstart[(int64_t)(key + 1) << sh];
    if (lv < d && q1 - q0 > a.sigma) return;   // above the source leaves: M2M forms it (uniform CTA)
    double rc, zc, h;
    box_centre(key, lv, a.L, a.z0, rc, zc, h);
    const double inv_h = 1.0 / h;
    // the warp's modes [w0, w0 + nv) of the block
    const int nv = nm / 4 + (warp < nm % 4 ? 1 : 0);
    const int w0 = warp * (nm / 4) + min(warp, nm % 4);
    const int c0 = lane * kP2MRC;
    double2 acc[kP2MTM][kP2MRC];
#pragma unroll
    for (int v = 0; v < kP2MTM; ++v)
#pragma unroll
        for (int u = 0; u < kP2MRC; ++u) acc[v][u] = make_double2(0.0, 0.0);
    for (int s0 = q0; s0 < q1; s0 += kP2MSrc) {
        const int nc = min(kP2MSrc, q1 - s0);
        __syncthreads();
        // powers dr^i, dz^j of every source of the chunk, one thread per (source, axis)
        if (threadIdx.x < 2 * kP2MSrc) {
            const int qq = threadIdx.x >> 1, ax = threadIdx.x & 1;
            if (qq < nc) {
                const int q = s0 + qq;
                const double v = ax ? (a.sz[q] - zc) * inv_h : (a.sr[q] - rc) * inv_h;
                double pv = 1.0;
                for (int i = 0; i <= p; ++i) {
                    pw[(qq * 2 + ax) * (p + 1) + i] = pv;
                    pv *= v;
                }
            }
        }
        // coefficient rows by asynchronous copies (in flight while the monomials are formed)
        for (int e = threadIdx.x; e < nc * kP2MModes; e += kP2MThreads) {
            const int q = e / kP2MModes, n = e % kP2MModes;
            const bool v = n < nm;
            p2m_async16(Sx + q * kP2MModes + n, v ? a.S + (int64_t)(s0 + q) * a.K + a.m0 + n0 + n : a.S, v);
        }
        __syncthreads();
        // monomials dr^i dz^j: thread per slot (its (i, j) in registers), all sources
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            if (ci[e] < 0) continue;
            const int sl = threadIdx.x + e * kP2MThreads;
            for (int qq = 0; qq < nc; ++qq)
                mono[qq * kP2MRow + sl] = pw[(qq * 2) * (p + 1) + ci[e]] * pw[(qq * 2 + 1) * (p + 1) + cj[e]];
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        const double2 *Sw = Sx + w0;
        switch (nv) {   // warp-uniform
        case 4: p2m_chunk<4, kP2MRC>(Sw, mono, nc, lane, acc); break;
        case 3: p2m_chunk<3, kP2MRC>(Sw, mono, nc, lane, acc); break;
        case 2: p2m_chunk<2, kP2MRC>(Sw, mono, nc, lane, acc); break;
        case 1: p2m_chunk<1, kP2MRC>(Sw, mono, nc, lane, acc); break;
        default: break;
        }
    }
    double2 *Mo = a.M + (a.soff[lv] + slot) * (int64_t)KW * P;
#pragma unroll
    for (int v = 0; v < kP2MTM; ++v) {
        if (v >= nv) break;
        const int n = n0 + w0 + v;
#pragma unroll
        for (int u = 0; u < kP2MRC; ++u)
            if (c0 + u < P) Mo[(int64_t)n * P + c0 + u] = acc[v][u];
    }
}

inline size_t p2m_smem(int P, int p)
{
    return sizeof(double) * kP2MSrc * 32 * p2m_rc(P) + sizeof(double2) * kP2MSrc * kP2MModes +
           sizeof(double) * kP2MSrc * 2 * (p + 1);
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
    if (a.sigma > 0) {   // an adaptive source leaf: P2M formed its moments (CTA-uniform)
        const int sh = 2 * (a.depth - level);
        if (a.slstart[(int64_t)(key + 1) << sh] - a.slstart[(int64_t)key << sh] <= a.sigma) return;
    }
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
// Dense form (thread per position of the level, before the host knows the level counts):
// need[g] for g = lvoff[l] + key, and needi[g] = need as int (scanned into the compact Lc row).
// Lc row -> dense position, and the first row of every level (lrow is an exclusive scan of the
// dense need flags, so the rows of a level are contiguous)
__global__ void need_rows_kernel(const int *lrow, const unsigned char *need, int64_t n, int64_t *rowkey)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && need[g]) rowkey[lrow[g]] = g;
}
struct LevelOffsets {
    int64_t v[kMaxLevels + 2];
};
__global__ void level_rows_kernel(const int *lrow, const unsigned char *need, LevelOffsets lo,
                                  int depth, int *out)
{
    const int64_t *lvoff = lo.v;
    // out[l] = first row of level l (l = 2..depth), out[depth + 1] = total rows
    const int l = threadIdx.x + 2;
    if (l > depth + 1) return;
    if (l <= depth) out[l] = lrow[lvoff[l]];
    else out[l] = lrow[lvoff[l] - 1] + (need[lvoff[l] - 1] ? 1 : 0);
}

struct NeedArgs {
    int depth;
    const int *tmap[kMaxLevels];
    int64_t lvoff[kMaxLevels + 1];
    const unsigned char *written;
    unsigned char *need;
    int *needi;
};
__global__ void need_kernel(NeedArgs a, int level)
{
    const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (key >= ((int64_t)1 << (2 * level))) return;
    const int64_t g = a.lvoff[level] + key;
    bool nd = false;
    if (a.tmap[level][key] >= 0) {
        nd = a.written[g] != 0;
        if (level < a.depth)
            for (int c = 0; c < 4 && !nd; ++c) nd = a.need[a.lvoff[level + 1] + 4 * key + c] != 0;
    }
    a.need[g] = nd ? 1 : 0;
    a.needi[g] = nd ? 1 : 0;
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
    // the level's materialised boxes only: local rows [row0, row1), row -> dense position
    const int row0 = a.lrow_lev[level], row1 = a.lrow_lev[level + 1];
    const int64_t items = (int64_t)(row1 - row0) * KW;
    for (int64_t it = (int64_t)blockIdx.x * kL2LWarps + warp; it < items;
         it += (int64_t)gridDim.x * kL2LWarps) {
        const int row = row0 + (int)(it / KW), n = (int)(it % KW);
        const uint32_t key = (uint32_t)(a.rowkey[row] - a.lvoff[level]);
        const int sr = key & 1, sz = (key >> 1) & 1;
        const bool child_w = a.s2l_written[a.lvoff[level] + key] != 0;
        const bool par_ok = level - 1 > 2 || a.s2l_written[a.lvoff[level - 1] + (key >> 2)] != 0;
        const double2 *pg = a.Lc + ((int64_t)a.lrow[a.lvoff[level - 1] + (key >> 2)] * KW + n) * P;
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
        double2 *o = a.Lc + ((int64_t)row * KW + n) * P;
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

// one-shot TMA bulk copy on an mbarrier (L2P local staging)
__device__ __forceinline__ void l2p_mbar_init(uint64_t *bar)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// generic-proxy reads of a buffer (previous item) before an async-proxy (TMA) write to it
__device__ __forceinline__ void l2p_fence_proxy()
{
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void l2p_bulk(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void l2p_mbar_wait(uint64_t *bar, unsigned phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase)
        : "memory");
}

// ---------------------------------------------------------------------------------------------
// L2P at the leaves: Phi^(n)(r, z) += sum_{k+l<=p} Phi_kl (r - r_c)^k (z - z_c)^l.
// The local evaluated is that of the deepest ancestor (or the leaf itself) whose local was
// written by S2L: below it the chain adds nothing, so the leaf's local is that box's local
// re-centred (exact) and is evaluated directly.  Written boxes are always
// materialised (need_kernel), and the choice depends only on the leaf's own chain, so results
// do not depend on the other field points.  None written: the far field is zero.
// owner[s] for target leaf slot s: (level << 24) | Lc row of the evaluating box, or -1.
__global__ void l2p_owner_kernel(FarArgs a, int *owner)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = a.depth;
    if (s >= a.tcount[d]) return;
    int la = d;
    uint32_t ka = (uint32_t)a.tkeys[d][s];
    while (la >= 2 && !a.s2l_written[a.lvoff[la] + ka]) {
        --la;
        ka >>= 2;
    }
    owner[s] = la < 2 ? -1 : (la << 24) | a.lrow[a.lvoff[la] + ka];
}

// L2P tasks: runs of <= TP consecutive sorted field points with the same evaluating box (a task
// starts where the owner changes or at a multiple of TP; TP = a.l2p_tp in {16, 32, 64, 128}).
// C5: 4M points in ~15k runs, most of them hundreds of points under a coarse written box;
// C2 / C3: leaves of ~16 points, each its own evaluating box.
constexpr int kL2PThreads = 128;
__device__ __forceinline__ int point_owner(const FarArgs &a, const uint32_t *fkey, const int *owner,
                                           int64_t t)
{
    return owner[a.tmap[a.depth][fkey[t]]];
}
__global__ void l2p_task_flags_kernel(FarArgs a, const uint32_t *fkey, const int *owner, int *flag)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.tfield) return;
    flag[t] = (t % a.l2p_run == 0 || point_owner(a, fkey, owner, t) != point_owner(a, fkey, owner, t - 1)) ? 1 : 0;
}
__global__ void l2p_task_emit_kernel(int64_t nf, const int *flag, const int *pos, int *tstart)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nf && flag[t]) tstart[pos[t]] = (int)t;
}

// NP points of one thread against the MB modes of a staged local (potential only): a coefficient
// broadcast feeds 2 NP DFMA.  dr, dz: the points' normalised offsets (absent points: zeros).
template <int MB, int NP, bool EXACT, int NPA>
__device__ __forceinline__ void l2p_points(const double2 *lg, int P, int p, int nm,
                                           const double (&dr)[NPA], const double (&dz)[NPA],
                                           double2 (&acc)[NPA][MB])
{
    double pr[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) pr[j] = 1.0;
    int q = 0;
    for (int k = 0; k <= p; ++k) {
        double pz[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) pz[j] = pr[j];
        for (int l = 0; k + l <= p; ++l, ++q) {
#pragma unroll
            for (int m = 0; m < MB; ++m) {
                if (EXACT || m < nm) {
                    const double2 c = lg[m * P + q];
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        acc[j][m].x = fma(c.x, pz[j], acc[j][m].x);
                        acc[j][m].y = fma(c.y, pz[j], acc[j][m].y);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NP; ++j) pz[j] *= dz[j];
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) pr[j] *= dr[j];
    }
}

// CTA item = (task, gpc = 128 / TP consecutive groups of <= MB modes): the evaluating box's
// local (the groups' modes, one contiguous block of the compact local storage) arrives by one TMA
// bulk copy; thread = (field point, mode group), monomials (r - r_c)^k (z - z_c)^l / h^(k+l)
// generated in registers in the coefficient order (k-major), the local's coefficients read as
// shared-memory broadcasts (the points of a task evaluate the same box): MB vector loads for
// 2 MB DFMA per coefficient.  GRAD: also d/dr and d/dz of the local polynomial (SURVEY 8(f)
// item 3), from k dr^(k-1) dz^l and l dr^k dz^(l-1).
// PT = 2, 4 (tasks of PT TP points, thread = points ip + j TP): the inner loop is bound by the
// shared-memory pipe (a 16-byte coefficient broadcast is 2 wavefronts of the SM's one per clock,
// 2 DFMA are 4 clocks of one of its four FP64 pipes: ncu lsu wavefronts 83%, FP64 pipe 43% at C5
// with one point per thread, 65% / 52% with two), so a coefficient read serves PT points; warps
// with fewer points run the loop for 2 or 1.
// PL > 0: compile-time local order (the row stride P becomes an immediate: one address register
// for the MB coefficient loads of a step, which the compiler then issues as a batch); EXACT:
// every mode group holds exactly MB modes (no per-mode predicates).
template <int MB, bool GRAD, int PT = 1, int PL = 0, bool EXACT = false>
__global__ void __launch_bounds__(kL2PThreads, PT >= 2 ? 3 : 1) l2p_kernel(FarArgs a, const uint32_t *fkey, const int *owner,
                                                          const int *tstart, const int *ntasks, int ngrp)
{
    static_assert(PT == 1 || !GRAD, "several points per thread: potential only");
    static_assert(PT == 1 || PT == 2 || PT == 4, "points per thread");
    extern __shared__ double sm[];
    const int p = PL ? PL : a.pl, P = PL ? (PL + 1) * (PL + 2) / 2 : a.Pl;   // local order
    const int KW = a.m1 - a.m0, d = a.depth;
    const int TP = a.l2p_tp, gpc = kL2PThreads / TP;
    const int ngi = (ngrp + gpc - 1) / gpc;                          // CTA items per task
    double2 *loc = reinterpret_cast<double2 *>(sm);                 // [staged modes][Pl]
    uint64_t *bar = reinterpret_cast<uint64_t *>(loc + (size_t)min(KW, gpc * MB) * P);
    const int nt = *ntasks;
    if (threadIdx.x == 0) l2p_mbar_init(bar);
    __syncthreads();
    unsigned phase = 0;
    const int ip = threadIdx.x % TP, jg = threadIdx.x / TP;
    // persistent CTAs over (task, group block) items
    for (int64_t item = blockIdx.x; item < (int64_t)nt * ngi; item += gridDim.x) {
    const int task = (int)(item / ngi), G0 = (int)(item - (int64_t)task * ngi) * gpc;
    const int nG = min(gpc, ngrp - G0);
    const int64_t t0 = tstart[task], t1 = task + 1 < nt ? tstart[task + 1] : a.tfield;
    const int nA = (KW * G0) / ngrp, nB = (KW * (G0 + nG)) / ngrp;    // staged modes [nA, nB)
    const int g = G0 + jg;
    const int n0 = (KW * g) / ngrp, nm = jg < nG ? (KW * (g + 1)) / ngrp - n0 : 0;   // <= MB
    const int own = point_owner(a, fkey, owner, t0);
    const int64_t t = t0 + ip;
    double inv_h = 0.0, dr = 0.0, dz = 0.0;
    double drs[PT], dzs[PT];   // points t + j TP (PT > 1)
#pragma unroll
    for (int j = 0; j < PT; ++j) drs[j] = dzs[j] = 0.0;
    // points per thread this warp needs (warp-uniform): 1 runs the one-point loop below
    int np = 1;
    if (PT > 1) {
        np = __any_sync(0xffffffffu, t + TP < t1) ? 2 : 1;
        if (PT > 2 && __any_sync(0xffffffffu, t + 2 * TP < t1)) np = 4;
    }
    if (own >= 0) {
        if (threadIdx.x == 0) {
            l2p_fence_proxy();
            l2p_bulk(loc, a.Lc + ((int64_t)(own & 0xffffff) * KW + nA) * P, (unsigned)((nB - nA) * P * 16), bar);
        }
        const int la = own >> 24;
        double rc, zc, h;
        box_centre(fkey[t0] >> (2 * (d - la)), la, a.L, a.z0, rc, zc, h);
        inv_h = 1.0 / h;
        if (t < t1) {
            dr = (a.fr[t] - rc) * inv_h;
            dz = (a.fz[t] - zc) * inv_h;
        }
        if (PT > 1) {
#pragma unroll
            for (int j = 0; j < PT; ++j) {
                if (t + j * TP < t1) {
                    drs[j] = (a.fr[t + j * TP] - rc) * inv_h;
                    dzs[j] = (a.fz[t + j * TP] - zc) * inv_h;
                }
            }
        }
        l2p_mbar_wait(bar, phase);
        phase ^= 1u;
    }
    const double2 *lg = loc + (size_t)(n0 - nA) * P;
    if (PT > 1 && np > 1) {
    if (nm > 0) {   // (a warp with a second point: every lane has its first)
    double2 acc[PT][MB];
#pragma unroll
    for (int j = 0; j < PT; ++j)
#pragma unroll
        for (int m = 0; m < MB; ++m) acc[j][m] = make_double2(0.0, 0.0);
    if (own >= 0) {
        if (PT > 2 && np > 2) l2p_points<MB, PT, EXACT, PT>(lg, P, p, nm, drs, dzs, acc);
        else l2p_points<MB, 2, EXACT, PT>(lg, P, p, nm, drs, dzs, acc);
    }
#pragma unroll
    for (int j = 0; j < PT; ++j) {
        if (j >= np || t + j * TP >= t1) break;
        double2 *o = a.out + a.fperm[t + j * TP] * a.K + a.m0 + n0;
#pragma unroll
        for (int m = 0; m < MB; ++m) {
            if (m >= nm) break;
            const double2 sv = acc[j][m];
            double2 v = make_double2(sv.x * inv_h, sv.y * inv_h);
            if (a.l2p_accumulate) {
                const double2 cur = o[m];
                v = make_double2(fma(sv.x, inv_h, cur.x), fma(sv.y, inv_h, cur.y));
            }
            o[m] = v;
        }
    }
    }
    } else if (t < t1 && nm > 0) {
    const int64_t row = a.fperm[t];
    double2 acc[MB], accr[GRAD ? MB : 1], accz[GRAD ? MB : 1];
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[m] = make_double2(0.0, 0.0);
    if (GRAD) {
#pragma unroll
        for (int m = 0; m < MB; ++m) accr[GRAD ? m : 0] = accz[GRAD ? m : 0] = make_double2(0.0, 0.0);
    }
    if (own >= 0) {
        double pr = 1.0, prm = 0.0;   // dr^k and k dr^(k-1)
        int q = 0;
        for (int k = 0; k <= p; ++k) {
            double pz = pr, pzr = prm, pzm = 0.0;   // dr^k dz^l, k dr^(k-1) dz^l, l dr^k dz^(l-1)
            for (int l = 0; k + l <= p; ++l, ++q) {
#pragma unroll
                for (int m = 0; m < MB; ++m) {
                    if (m < nm) {
                        const double2 c = lg[m * P + q];
                        acc[m].x = fma(c.x, pz, acc[m].x);
                        acc[m].y = fma(c.y, pz, acc[m].y);
                        if (GRAD) {
                            accr[GRAD ? m : 0].x = fma(c.x, pzr, accr[GRAD ? m : 0].x);
                            accr[GRAD ? m : 0].y = fma(c.y, pzr, accr[GRAD ? m : 0].y);
                            accz[GRAD ? m : 0].x = fma(c.x, pzm, accz[GRAD ? m : 0].x);
                            accz[GRAD ? m : 0].y = fma(c.y, pzm, accz[GRAD ? m : 0].y);
                        }
                    }
                }
                if (GRAD) {
                    pzm = (l + 1) * pz;
                    pzr *= dz;
                }
                pz *= dz;
            }
            if (GRAD) prm = (k + 1) * pr;
            pr *= dr;
        }
    }
    // (the normalised local is h^(1+k+l) Phi_kl: divide by h once; gradients by h^2)
    double2 *o = a.out + row * a.K + a.m0 + n0;
#pragma unroll
    for (int m = 0; m < MB; ++m) {
        if (m >= nm) break;
        double2 v = make_double2(acc[m].x * inv_h, acc[m].y * inv_h);
        if (a.l2p_accumulate) {
            const double2 cur = o[m];
            v = make_double2(fma(acc[m].x, inv_h, cur.x), fma(acc[m].y, inv_h, cur.y));
        }
        o[m] = v;
    }
    if (GRAD) {
        const double s2 = inv_h * inv_h;
        double2 *orr = a.outr + row * a.K + a.m0 + n0, *oz = a.outz + row * a.K + a.m0 + n0;
#pragma unroll
        for (int m = 0; m < MB; ++m) {
            if (m >= nm) break;
            const double2 ar = accr[GRAD ? m : 0], az = accz[GRAD ? m : 0];
            if (a.l2p_accumulate) {
                const double2 cr = orr[m], cz = oz[m];
                orr[m] = make_double2(fma(ar.x, s2, cr.x), fma(ar.y, s2, cr.y));
                oz[m] = make_double2(fma(az.x, s2, cz.x), fma(az.y, s2, cz.y));
            } else {
                orr[m] = make_double2(ar.x * s2, ar.y * s2);
                oz[m] = make_double2(az.x * s2, az.y * s2);
            }
        }
    }
    }
    __syncthreads();   // every thread is done with loc before the next item's copy
    }
}
template <int MB>
inline size_t l2p_smem(int Pl, int KW, int TP)
{
    const int gpc = kL2PThreads / TP;
    return sizeof(double2) * (size_t)std::min(KW, gpc * MB) * Pl + 2 * sizeof(uint64_t);
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
