// p2p.cuh -- pairwise modal sums Phi_t^(n) += sum_s S_s^(n) G^(n)(r_t, r_s, z_t - z_s)
// (P:195-201): the direct sum (C1) and the FMM near field over the 9 neighbour leaves
// (P:647-651).  This is the paper's bottleneck.
//
// CTA design (sm_100a, FP64 CUDA cores; no tensor cores: special-function arithmetic):
//   a CTA owns a tile of TT target points and streams its source list through shared memory in
//   chunks of SC sources.  Per chunk, the NT = TT*SC pairs are
//     1. classified (forward chi < 1.008 / Miller / skipped) and compacted with warp ballots so
//        that each warp runs one branch (warp-uniform loops, uniform constant-bank reads);
//     2. evaluated one pair per thread: G^(n) for the mode window [m0, m1) written to smem;
//     3. contracted with lane = (target, mode): acc(t, n) += S_s^(n) G_ts^(n) over the chunk,
//        with the accumulators distributed over the CTA (register use independent of K).
//   Summation order is fixed (source list order, chunk by chunk): results are bitwise
//   reproducible and independent of the compaction.
#pragma once
#include "specfun.cuh"

namespace cyl {

struct P2PArgs {
    const double *sr, *sz;      // sources (sorted order for the near field)
    const double2 *S;           // [ns][K] complex
    const double *fr, *fz;      // targets (sorted order for the near field)
    int64_t ns, nf;
    int K;                      // total modes (N = K - 1 sets the Miller start)
    int m0, m1;                 // mode window
    int miller;                 // 0 accurate, 1 paper
    double fwd2;                // forward switch 2 t_N (R#3)
    int exclude;                // skip coincident pairs
    // output
    double2 *out;               // rows [*][K]
    double2 *outr, *outz;       // gradient rows dPhi/dr, dPhi/dz (GRAD kernels only)
    const int *out_row;         // target t -> output row (nullptr: row = t)
    int accumulate;             // load initial value from out
    int64_t part_stride;        // direct: out += blockIdx.y * part_stride (complex elements)
    // direct mode: sources [y * src_per_part, ...) ; near mode: tasks
    int64_t src_per_part;
    const int4 *tasks;          // near: {t0, t1, leafkey, 0}
    const int *ntasks;          // near: device count
    int *task_ctr;              // near, warp-task kernel: dynamic task counter (zeroed)
    const int *leafstart;       // near: dense source leaf starts [4^d + 1]
    int depth;
    int level;                  // near: level of the task boxes (0: the leaf level d)
    int adaptive_leaf;          // near: adaptive source tree sigma (R#26), 0 = uniform
    unsigned long long *n_skipped;
    unsigned long long *n_pairs;
    unsigned long long *n_branch;   // nullable: [0] forward, [1] far, [2] Miller pairs, [3] sum S - N
    // window state (K in (33, 66]: two mode windows): save = 1 in the first window writes, per
    // pair, the forward chain state (u_31, u_32) or the Miller state (w_66, w_65, c (2 chi)^-64)
    // in the final scaling; save = 2 in the second window reads it instead of re-running the
    // setup and the chain below / above the window.  Pair slot = pbase[leaf slot] + (target index
    // in its leaf) * (sources of the leaf's 9 neighbours) + (source index in that list).
    int save;
    double2 *sv2;
    double *sv1;
    const int64_t *pbase;
    const int *tmap_leaf;         // target leaf key -> slot
    const int *fleafstart;        // dense target leaf starts
    int *err_flag;
};

__device__ __forceinline__ uint32_t morton2(uint32_t ix, uint32_t iz)
{
    auto spread = [](uint32_t v) {
        v &= 0xffffu;
        v = (v | (v << 8)) & 0x00ff00ffu;
        v = (v | (v << 4)) & 0x0f0f0f0fu;
        v = (v | (v << 2)) & 0x33333333u;
        v = (v | (v << 1)) & 0x55555555u;
        return v;
    };
    return spread(ix) | (spread(iz) << 1);
}
__device__ __forceinline__ uint32_t compact1(uint32_t v)
{
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0f0f0f0fu;
    v = (v | (v >> 4)) & 0x00ff00ffu;
    v = (v | (v >> 8)) & 0x0000ffffu;
    return v;
}

// Sources of neighbour k (0..8, (dx, dz) = (k / 3 - 1, k % 3 - 1)) of the level-lv box `key` that
// the near field sums directly: (first sorted source, count).  Every box at every
// level owns the contiguous sorted range [slstart[b 4^(d-lv)], slstart[(b+1) 4^(d-lv)]).
// Uniform tree (sigma = 0): the whole neighbour (lv = d).  Adaptive source tree (sigma > 0, R#26):
// the pair (box, neighbour S) is evaluated directly at level lv iff it was descended into (lv = 2
// or S's parent holds > sigma sources) and stops here (S holds <= sigma sources, or lv = d).
__device__ __forceinline__ int2 near_segment(const int *slstart, int depth, int lv, int sigma,
                                             uint32_t key, int k)
{
    const int x = (int)compact1(key) + k / 3 - 1, z = (int)compact1(key >> 1) + k % 3 - 1;
    const int nb = 1 << lv;
    if (x < 0 || z < 0 || x >= nb || z >= nb) return make_int2(0, 0);
    const int sh = 2 * (depth - lv);
    const uint32_t m = morton2((uint32_t)x, (uint32_t)z);
    const int s0 = slstart[(int64_t)m << sh], len = slstart[(int64_t)(m + 1) << sh] - s0;
    if (sigma > 0 && len > 0) {
        if (lv < depth && len > sigma) return make_int2(s0, 0);   // S is descended into
        if (lv > 2) {
            const int64_t pm = m >> 2;
            if (slstart[(pm + 1) << (sh + 2)] - slstart[pm << (sh + 2)] <= sigma)
                return make_int2(s0, 0);                            // the parent pair stopped
        }
    }
    return make_int2(s0, len);
}

// GRAD (near field, one mode window from mode 0): also the field gradients, from the paper's
// first-order derivative relations (P:917-923 in x, P:958-966 in r; G^(-1) == G^(1)):
//   dG^n/dx = (n - 1/2) x q_n,   dG^n/dr = -G^n/(2r) + (n - 1/2) u q_n,
//   q_n = (G^n + G^{n-1}) / rho_+^2 + (G^n - G^{n-1}) / rho_-^2,   u = (r^2 - r1^2 - x^2)/(2r).
template <int TT, int SC, int MAXT, bool NEAR, bool GRAD = false>
__global__ void __launch_bounds__(TT *SC, (MAXT > 6 ? 4 : 8)) p2p_kernel(P2PArgs a)
{
    constexpr int NT = TT * SC;
    constexpr int NW = NT / 32;
    const int KW = a.m1 - a.m0;
    const int KG = GRAD && KW < 2 ? 2 : KW;              // GRAD needs G^1 for mode 0
    extern __shared__ double smem[];
    double *Gs = smem;                                  // [KG][TT][SC]
    double2 *Ss = reinterpret_cast<double2 *>(Gs + (size_t)KG * NT);  // [SC][KW]
    double *src_r = reinterpret_cast<double *>(Ss + (size_t)SC * KW);
    double *src_z = src_r + SC;
    double *tg_r = src_z + SC;
    double *tg_z = tg_r + TT;
    double *pf = tg_z + TT;                             // GRAD: [4][NT] 1/rho+^2, 1/rho-^2, x, u
    int *sidx = reinterpret_cast<int *>(pf + (GRAD ? 4 * NT : 0));     // [SC]
    int *order = sidx + SC;                             // [NT]
    int *wcnt = order + NT;                             // [3 NW]
    int *seg = wcnt + 3 * NW;                           // [9][2] + prefix [10]
    int *segpre = seg + 18;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int t0, nt, nseg;
    if (NEAR) {
        if ((int)blockIdx.x >= *a.ntasks) return;
        int4 tk = a.tasks[blockIdx.x];
        t0 = tk.x;
        nt = tk.y - tk.x;
        if (tid == 0) {
            uint32_t key = (uint32_t)tk.z;
            int ix = (int)compact1(key), iz = (int)compact1(key >> 1);
            int nb = 1 << a.depth, k = 0, acc = 0;
            for (int da = -1; da <= 1; ++da)
                for (int dc = -1; dc <= 1; ++dc) {
                    int x = ix + da, z = iz + dc;
                    if (x < 0 || z < 0 || x >= nb || z >= nb) continue;
                    uint32_t m = morton2((uint32_t)x, (uint32_t)z);
                    int s0 = a.leafstart[m], s1 = a.leafstart[m + 1];
                    if (s1 <= s0) continue;
                    seg[2 * k] = s0;
                    seg[2 * k + 1] = s1;
                    segpre[k] = acc;
                    acc += s1 - s0;
                    ++k;
                }
            segpre[k] = acc;
            wcnt[0] = k;  // temp
        }
        __syncthreads();
        nseg = wcnt[0];
        __syncthreads();
    } else {
        t0 = blockIdx.x * TT;
        nt = (int)min((int64_t)TT, a.nf - t0);
        if (tid == 0) {
            int64_t s0 = (int64_t)blockIdx.y * a.src_per_part;
            int64_t s1 = min(a.ns, s0 + a.src_per_part);
            seg[0] = (int)s0;
            seg[1] = (int)max(s0, s1);
            segpre[0] = 0;
            segpre[1] = seg[1] - seg[0];
        }
        nseg = 1;
    }
    if (tid < TT) {
        int t = t0 + min(tid, nt - 1);
        tg_r[tid] = a.fr[t];
        tg_z[tid] = a.fz[t];
    }
    __syncthreads();
    const int total = segpre[nseg];
    double2 *out = a.out + (NEAR ? 0 : (int64_t)blockIdx.y * a.part_stride);

    double2 acc[MAXT], accr[GRAD ? MAXT : 1], accz[GRAD ? MAXT : 1];
#pragma unroll
    for (int k = 0; k < MAXT; ++k) {
        acc[k] = make_double2(0.0, 0.0);
        if constexpr (GRAD) {
            accr[k] = make_double2(0.0, 0.0);
            accz[k] = make_double2(0.0, 0.0);
        }
        int id = tid + k * NT;
        if (a.accumulate && id < TT * KW) {
            int t = id % TT, n = id / TT;
            if (t < nt) {
                int64_t row = a.out_row ? a.out_row[t0 + t] : (t0 + t);
                acc[k] = out[row * a.K + a.m0 + n];
                if constexpr (GRAD) {
                    accr[k] = a.outr[row * a.K + a.m0 + n];
                    accz[k] = a.outz[row * a.K + a.m0 + n];
                }
            }
        }
    }
    unsigned long long my_skipped = 0, my_pairs = 0;
    const int Nglob = a.K - 1;

    for (int v0 = 0; v0 < total; v0 += SC) {
        __syncthreads();
        if (tid < SC) {
            int v = v0 + tid, gi = -1;
            if (v < total) {
                int k = 0;
                while (k + 1 < nseg && v >= segpre[k + 1]) ++k;
                gi = seg[2 * k] + (v - segpre[k]);
                src_r[tid] = a.sr[gi];
                src_z[tid] = a.sz[gi];
            }
            sidx[tid] = gi;
        }
        __syncthreads();
        for (int e = tid; e < SC * KW; e += NT) {
            int s = e / KW, n = e - s * KW;
            int gi = sidx[s];
            Ss[e] = gi >= 0 ? a.S[(int64_t)gi * a.K + a.m0 + n] : make_double2(0.0, 0.0);
        }
        // classify pair slot p = tid (t = p % TT, s = p / TT)
        int cls;
        {
            int t = tid % TT, s = tid / TT;
            bool valid = t < nt && sidx[s] >= 0;
            cls = 2;
            if (valid) {
                double r = tg_r[t], r1 = src_r[s];
                double z = tg_z[t], z1 = src_z[s];
                if (r == r1 && z == z1) {
                    if (a.exclude) ++my_skipped;
                    else atomicOr(a.err_flag, 1);
                } else {
                    PairGeo g = pair_geo(r, r1, z - z1, a.fwd2);
                    cls = g.forward ? 0 : (g.far ? 3 : 1);   // forward / Miller / far
                    ++my_pairs;
                }
            }
        }
        // order: forward, far, Miller, skipped (warps then run one evaluation path each)
        unsigned bF = __ballot_sync(0xffffffffu, cls == 0);
        unsigned bX = __ballot_sync(0xffffffffu, cls == 3);
        unsigned bM = __ballot_sync(0xffffffffu, cls == 1);
        if (lane == 0) {
            wcnt[warp] = __popc(bF);
            wcnt[NW + warp] = __popc(bX);
            wcnt[2 * NW + warp] = __popc(bM);
        }
        __syncthreads();
        {
            int preF = 0, preX = 0, preM = 0, totF = 0, totX = 0, totM = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                int cF = wcnt[w], cX = wcnt[NW + w], cM = wcnt[2 * NW + w];
                if (w < warp) {
                    preF += cF;
                    preX += cX;
                    preM += cM;
                }
                totF += cF;
                totX += cX;
                totM += cM;
            }
            unsigned lt = (1u << lane) - 1u;
            int bf = __popc(bF & lt), bx = __popc(bX & lt), bm = __popc(bM & lt);
            int pos;
            if (cls == 0) pos = preF + bf;
            else if (cls == 3) pos = totF + preX + bx;
            else if (cls == 1) pos = totF + totX + preM + bm;
            else pos = totF + totX + totM + (warp * 32 - preF - preX - preM) + (lane - bf - bx - bm);
            order[pos] = tid | (cls << 16);
        }
        __syncthreads();
        {
            int my = order[tid];
            int p = my & 0xffff, c = my >> 16;
            int t = p % TT, s = p / TT;
            double *g = Gs + t * SC + s;
            bool miller = (c == 1);
            int S_lane = 0;
            PairGeo geo;
            if (c != 2) {
                geo = pair_geo(tg_r[t], src_r[s], tg_z[t] - src_z[s], a.fwd2);
                if (miller) S_lane = Nglob + miller_extra(geo, a.miller);
            }
            int S_warp = __reduce_max_sync(0xffffffffu, S_lane);
            if (c == 2) {
                for (int n = 0; n < KG; ++n) g[n * NT] = 0.0;
            } else {
                greens_pair(geo, a.m0, a.m0 + KG, S_warp, g, NT);
            }
            if constexpr (GRAD) {
                const int q = t * SC + s;
                if (c == 2) {
                    pf[q] = pf[NT + q] = pf[2 * NT + q] = pf[3 * NT + q] = 0.0;
                } else {
                    const double r = tg_r[t], r1 = src_r[s], x = tg_z[t] - src_z[s];
                    pf[q] = 1.0 / geo.rp2;
                    pf[NT + q] = 1.0 / geo.rm2;
                    pf[2 * NT + q] = x;
                    pf[3 * NT + q] = (r * r - r1 * r1 - x * x) / (2.0 * r);
                }
            }
        }
        __syncthreads();
        // contraction: lane = (t, n)
#pragma unroll
        for (int k = 0; k < MAXT; ++k) {
            int id = tid + k * NT;
            if (id < TT * KW) {
                int t = id % TT, n = id / TT;
                const double *g = Gs + (n * TT + t) * SC;
                double2 sum = acc[k];
                if constexpr (GRAD) {
                    const int nm1 = a.m0 + n == 0 ? 1 : n - 1;     // G^(-1) == G^(1)
                    const double *gm = Gs + (nm1 * TT + t) * SC;
                    const double hn = a.m0 + n - 0.5, inv2r = 0.5 / tg_r[t];
                    double2 sr_ = accr[k], sz_ = accz[k];
#pragma unroll
                    for (int s = 0; s < SC; ++s) {
                        const int q = t * SC + s;
                        const double G = g[s], Gm = gm[s];
                        const double qn = hn * fma(G + Gm, pf[q], (G - Gm) * pf[NT + q]);
                        const double dz = qn * pf[2 * NT + q];
                        const double dr = fma(qn, pf[3 * NT + q], -G * inv2r);
                        double2 sv = Ss[s * KW + n];
                        sum.x = fma(sv.x, G, sum.x);
                        sum.y = fma(sv.y, G, sum.y);
                        sr_.x = fma(sv.x, dr, sr_.x);
                        sr_.y = fma(sv.y, dr, sr_.y);
                        sz_.x = fma(sv.x, dz, sz_.x);
                        sz_.y = fma(sv.y, dz, sz_.y);
                    }
                    accr[k] = sr_;
                    accz[k] = sz_;
                } else {
#pragma unroll
                    for (int s = 0; s < SC; ++s) {
                        double2 sv = Ss[s * KW + n];
                        sum.x = fma(sv.x, g[s], sum.x);
                        sum.y = fma(sv.y, g[s], sum.y);
                    }
                }
                acc[k] = sum;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < MAXT; ++k) {
        int id = tid + k * NT;
        if (id < TT * KW) {
            int t = id % TT, n = id / TT;
            if (t < nt) {
                int64_t row = a.out_row ? a.out_row[t0 + t] : (t0 + t);
                out[row * a.K + a.m0 + n] = acc[k];
                if constexpr (GRAD) {
                    a.outr[row * a.K + a.m0 + n] = accr[k];
                    a.outz[row * a.K + a.m0 + n] = accz[k];
                }
            }
        }
    }
    // counters (integers: deterministic)
    my_skipped = __reduce_add_sync(0xffffffffu, (unsigned)my_skipped);
    my_pairs = __reduce_add_sync(0xffffffffu, (unsigned)my_pairs);
    if (lane == 0 && a.n_skipped && my_skipped && a.m0 == 0) atomicAdd(a.n_skipped, my_skipped);
    if (lane == 0 && a.n_pairs && my_pairs && a.m0 == 0) atomicAdd(a.n_pairs, my_pairs);
}

template <int TT, int SC, bool GRAD = false>
inline size_t p2p_smem_bytes(int KW)
{
    constexpr int NT = TT * SC;
    const int KG = GRAD && KW < 2 ? 2 : KW;
    return sizeof(double) * ((size_t)KG * NT + 2 * (size_t)SC * KW + 2 * SC + 2 * TT +
                             (GRAD ? 4 * NT : 0)) +
           sizeof(int) * (SC + NT + 3 * (NT / 32) + 18 + 10);
}

// Deterministic reduction of direct-sum partial results: out[t][n] = sum_part ws[part][t][n].
__global__ void reduce_parts_kernel(const double2 *ws, int64_t nelem, int nparts, double2 *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nelem) return;
    double2 s = ws[i];
    for (int p = 1; p < nparts; ++p) {
        double2 v = ws[(int64_t)p * nelem + i];
        s.x += v.x;
        s.y += v.y;
    }
    out[i] = s;
}

// Test entry kernel: one thread per (r, r1, x) triple, all modes to global memory.
__global__ void greens_batch_kernel(const double *r, const double *r1, const double *x,
                                    int64_t n, int K, int miller, double fwd2, double *out,
                                    int *err)
{
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = q < n;
    PairGeo g;
    int S_lane = 0;
    if (ok) {
        double rr = r[q], rr1 = r1[q];
        if (!(rr > 0.0) || !(rr1 > 0.0)) {
            atomicOr(err, 2);
            ok = false;
        } else {
            g = pair_geo(rr, rr1, x[q], fwd2);
            if (g.coincident) {
                atomicOr(err, 1);
                ok = false;
            } else if (!g.forward) {
                S_lane = (K - 1) + miller_extra(g, miller);
            }
        }
    }
    int S_warp = __reduce_max_sync(0xffffffffu, S_lane);
    if (ok) greens_pair(g, 0, K, S_warp, out + q * K, 1);
}

}  // namespace cyl
