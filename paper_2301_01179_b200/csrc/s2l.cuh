// s2l.cuh -- S2L, the far-field interactions of Algorithm 1, on
// sm_100a in FP64, organised by STATION instead of by target box.
//
// The operator of an S2L interaction depends only on the normalised station geometry
// (r^, r1^, x^) = (i_in + dI + 1/2, i_in + 1/2, dJ) -- i_in = min(target column, source column),
// (dI, dJ) = |offset| one of the 12 classes of P:561-568 -- on whether the target lies outside
// (FO/BO: (A,B) = (k,i)) or inside (FI/BI: (A,B) = (i,k)) the source's radius, and on the sign of
// the z offset (forward / backward), where backward = forward with (-1)^{j+l}.  With
// moments and locals in box-normalised units (fmm_ops.cuh) the same operator serves every level
// (scaling relation).  So every (source box, target box) pair of every level is
// enumerated once (target-major, offsets in a fixed order), bucketed by the station key
//     key = ((i_in * 12 + class) << 1) | inward,
// and each bucket is cut into batches of JT pairs: one CTA applies ONE staged operator to JT
// pairs (a full register-tiled FP64 GEMM, however sparse the inputs are: C5's sources lie on two
// curves, so a target column sees ~2 of them per offset).  Backward pairs read a moment copy
// with their odd-j sign flip folded in and negate their odd-l result rows (exact).  Each pair's contribution
// goes to its own slot of a pair buffer (target-major), and a reduction sums every target box's
// slots in the fixed offset order: results are bitwise reproducible, independent of how pairs are
// batched and of which other target boxes exist (a field-partitioned solve equals the full one).
#pragma once
#include "fmm_ops.cuh"

namespace cyl {

// ---------------------------------------------------------------------------------------------
// Interaction lists: the children of the parent's neighbours that are not
// neighbours of the target box (it, jt) at level l: di in [di0, di0 + 5], dj in [dj0, dj0 + 5]
// with di0 = -2 (it even) or -3 (it odd), likewise dj0, minus the 3 x 3 near cells.  Order:
// di-major, dj ascending (the summation order of a target's contributions).  Targets are indexed
// densely, g = lvoff[l] + key, so the lists are built on the device before the host knows the
// level counts.
struct S2LListArgs {
    int depth;
    const int *smap[kMaxLevels], *tmap[kMaxLevels];
    int64_t lvoff[kMaxLevels + 1];   // dense per-level offsets, lvoff[depth + 1] = total
    int nkeys;               // 2 * 12 * 2^depth station keys
    int JT;                  // pairs per batch
    int *pcnt, *poff;        // [ltot] pairs per target, exclusive prefix (pair slots)
    int *khist, *kstart, *kcur, *bstart;   // [nkeys]
    int4 *pairs;             // station-major (source slot, pair slot, backward, level)
    int4 *batches;           // (first pair, count, key, 0)
    unsigned char *written;  // dense [lvoff[l] + key]: S2L wrote this box's local
    int *wlist, *wcount;     // targets (dense index) with >= 1 pair
    int *totals;             // [0] pairs, [1] batches (s2l_totals_kernel)
};

template <typename F>
__device__ __forceinline__ void for_each_s2l(const S2LListArgs &a, int l, uint32_t key, F &&f)
{
    const int it = (int)compact1(key), jt = (int)compact1(key >> 1), nb = 1 << l;
    const int di0 = (it & 1) ? -3 : -2, dj0 = (jt & 1) ? -3 : -2;
    const int *smap = a.smap[l];
    for (int di = di0; di <= di0 + 5; ++di) {
        const int is = it + di;
        if (is < 0 || is >= nb) continue;
        for (int dj = dj0; dj <= dj0 + 5; ++dj) {
            if (di >= -1 && di <= 1 && dj >= -1 && dj <= 1) continue;
            const int js = jt + dj;
            if (js < 0 || js >= nb) continue;
            const int s = smap[morton2((uint32_t)is, (uint32_t)js)];
            if (s < 0) continue;   // empty, or below an adaptive source leaf (R#26)
            const int iin = min(it, is), dI = di < 0 ? -di : di, dJ = dj < 0 ? -dj : dj;
            f(s, ((iin * 12 + class_of(dI, dJ)) << 1) | (di > 0 ? 1 : 0), dj > 0 ? 1 : 0);
        }
    }
}

__device__ __forceinline__ int dense_level(const int64_t *lvoff, int depth, int64_t g)
{
    int l = 2;
    while (l < depth && g >= lvoff[l + 1]) ++l;
    return l;
}

// thread per dense target position g: pair count, station histogram, written flag, written list
__global__ void s2l_count_kernel(S2LListArgs a)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.lvoff[a.depth + 1]) return;
    const int l = dense_level(a.lvoff, a.depth, g);
    const uint32_t key = (uint32_t)(g - a.lvoff[l]);
    int cnt = 0;
    if (a.tmap[l][key] >= 0)
        for_each_s2l(a, l, key, [&](int, int skey, int) {
            atomicAdd(a.khist + skey, 1);
            ++cnt;
        });
    a.pcnt[g] = cnt;
    a.written[g] = cnt > 0 ? 1 : 0;
    if (cnt) a.wlist[atomicAdd(a.wcount, 1)] = (int)g;
}

// thread per station key: number of batches
__global__ void s2l_nbatch_kernel(S2LListArgs a)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < a.nkeys) a.bstart[k] = (a.khist[k] + a.JT - 1) / a.JT;
}

// thread per dense target g: its pairs into their station buckets (slot = target-major index).
// The order inside a bucket is arbitrary (atomics): a pair's result does not depend on its batch.
__global__ void s2l_emit_kernel(S2LListArgs a)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.lvoff[a.depth + 1] || a.pcnt[g] == 0) return;
    const int l = dense_level(a.lvoff, a.depth, g);
    const uint32_t key = (uint32_t)(g - a.lvoff[l]);
    int slot = a.poff[g];
    for_each_s2l(a, l, key, [&](int s, int skey, int bwd) {
        const int pos = a.kstart[skey] + atomicAdd(a.kcur + skey, 1);
        a.pairs[pos] = make_int4(s, slot++, bwd, l);
    });
}

// thread per station key: its batches of <= JT pairs (bstart = exclusive scan of batch counts)
__global__ void s2l_batch_emit_kernel(S2LListArgs a)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.nkeys) return;
    const int n = a.khist[k], s0 = a.kstart[k];
    int b = a.bstart[k];
    for (int q = 0; q < n; q += a.JT) a.batches[b++] = make_int4(s0 + q, min(a.JT, n - q), k, 0);
}

// stations (i_in, class) with at least one pair (either in/out key): the only tensors S2L reads
__global__ void s2l_station_flags_kernel(const int *khist, int nstat, int *flag)
{
    const int st = blockIdx.x * blockDim.x + threadIdx.x;
    if (st < nstat) flag[st] = (khist[2 * st] + khist[2 * st + 1]) > 0 ? 1 : 0;
}
__global__ void s2l_station_emit_kernel(const int *flag, const int *pos, int nstat, int *list)
{
    const int st = blockIdx.x * blockDim.x + threadIdx.x;
    if (st < nstat && flag[st]) list[pos[st]] = st;
}

// totals of the scanned counts (one thread): pairs, batches
__global__ void s2l_totals_kernel(S2LListArgs a)
{
    if (threadIdx.x) return;
    const int k = a.nkeys - 1;
    a.totals[0] = a.kstart[k] + a.khist[k];
    a.totals[1] = a.bstart[k] + (a.khist[k] + a.JT - 1) / a.JT;
}

// ---------------------------------------------------------------------------------------------
// The batched S2L product.  CTA per (batch, mode): the station's tensor block (packed Hankel
// form H_ab(c) = c! Gbar_abc, tensor.cuh) and the JT source moment rows (pre-scaled by
// (-1)^j / j!) arrive by TMA bulk copies on one mbarrier.  The operator is never materialised:
//     Phi'_(k,l) = sum_i sum_j H_{A,B}(j + l) M'_(i,j),  (A,B) = (k,i) outward, (i,k) inward,
// is, for fixed (k, i), a Hankel product in (l, j).  A thread owns R consecutive rows
// (k, l0 .. l0+R-1) of one k (a "unit") and C pairs: for each i it walks j = 0 .. p-i with a
// ring of R tensor values in registers, H[T(k,i) + j + l0 + r], loading ONE new value per step
// (the window slides by one), so a step is 1 scalar + C vector shared loads for 2 R C DFMA.
// Results are post-scaled by 1/l! (and (-1)^l for backward pairs) and written as contiguous runs
// of the pair's row in the pair buffer.  Backward pairs read moments pre-scaled without the
// (-1)^j (their sign flip on j is folded into the second copy).  Single truncation (i+j+k+l <= p, R#8) zeroes the tensor
// entries with a + b + c > p in shared memory first.
template <int R, int C, int NU, int CG>
struct S2LCfg {
    static constexpr int NT = NU * CG;   // threads: NU units x CG column groups
    static constexpr int JT = CG * C;    // pairs per batch
    static constexpr int MP = 0;         // (no gathered operator)
};

struct S2LArgs {
    int p, P, pl, Pl, pt, K, m0, m1;
    int truncation;
    const double *tens;        // [stations][KW][TPp] packed
    const double2 *M;          // pre-scaled moments [row][KW][P]: (-1)^j / j! (forward pairs)
    const double2 *Mb;         // the same with 1 / j! (backward pairs: (-1)^j folded in)
    const int4 *pairs, *batches;
    int64_t soff[kMaxLevels];  // per level: first moment row
    double2 *pairbuf;          // [slot][KW][Pl]
};

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
// bulk (TMA, 1-D) global -> shared copy completing on an mbarrier
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
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// packed offset of the tensor row (a, b) at order pt (closed form of packed_off, tensor.cuh)
__device__ __forceinline__ int packed_row(int a, int b, int pt)
{
    return a * ((pt + 1) * (2 * pt + 1) - pt * (pt + 1) / 2) - (pt + 1) * (a * (a - 1) / 2) +
           b * (2 * pt + 1 - a) - b * (b - 1) / 2;
}

// resident CTAs per SM each shape is built for (<= 128 registers at 128 / 256 threads, 96 at
// 192: p = 16's three CTAs, whose shared memory is the tensor 39 KB + 12 moment rows; measured:
// the p <= 12 shape at 140 registers fit one CTA per SM, C3 S2L 29.0 vs 22.9 ms)
template <int NT>
__host__ __device__ constexpr int s2l_min_blocks() { return NT <= 128 ? 4 : (NT <= 192 ? 3 : 2); }

template <int R, int C, int NU, int CG>
__global__ void __launch_bounds__(NU * CG, s2l_min_blocks<NU * CG>()) s2l_batch_kernel(S2LArgs a)
{
    constexpr int NT = NU * CG, JT = CG * C;
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, pl = a.pl, Pl = a.Pl, pt = a.pt;
    const int KW = a.m1 - a.m0;
    const int TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1);
    const int BPS = P | 1;                            // moment row stride (complex, odd)
    double2 *Xs = reinterpret_cast<double2 *>(sm);   // [JT][BPS] moments
    double *Hs = reinterpret_cast<double *>(Xs + JT * BPS);   // [TPp + R + 2] (zero tail)
    uint64_t *bar = reinterpret_cast<uint64_t *>(Hs + TPp + R + 2 + ((R + 2) & 1));
    int4 *rec = reinterpret_cast<int4 *>(bar + 2);   // [JT]
    int *Tk = reinterpret_cast<int *>(rec + JT);     // [(pl+1) * (p+1)] row offsets T(k, i)
    int *ukl = Tk + 17 * 17;                         // [NU] units (k << 8 | l0), -1 = none

    const int nloc = (int)(blockIdx.x % KW);
    const int4 bt = a.batches[blockIdx.x / KW];
    const int cnt = bt.y, skey = bt.z, inward = skey & 1;
    const int64_t station = skey >> 1;
    const int tid = threadIdx.x;
    // warp 0 starts the copies at once (barrier, tensor block, one moment row per pair: backward
    // pairs read the copy with (-1)^j folded in) while the other warps build the index tables
    if (tid < 32) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(bar, (unsigned)(TPp * 8 + cnt * P * 16));
            bulk_g2s(Hs, a.tens + (station * KW + nloc) * (int64_t)TPp, (unsigned)(TPp * 8), bar);
        }
        __syncwarp();
        for (int b = tid; b < JT; b += 32) {
            const int4 pr = b < cnt ? a.pairs[bt.x + b] : make_int4(0, -1, 0, 0);
            rec[b] = pr;
            if (b < cnt)
                bulk_g2s(Xs + b * BPS, (pr.z ? a.Mb : a.M) + ((a.soff[pr.w] + pr.x) * KW + nloc) * P,
                         (unsigned)(P * 16), bar);
        }
    } else {
        for (int q = tid - 32; q < (pl + 1) * (p + 1); q += NT - 32) {
            const int k = q / (p + 1), i = q - k * (p + 1);
            Tk[q] = inward ? packed_row(i, k, pt) : packed_row(k, i, pt);
        }
        if (tid == 32) {
            int u = 0;
            for (int k = 0; k <= pl; ++k)
                for (int l0 = 0; l0 <= pl - k; l0 += R) ukl[u++] = (k << 8) | l0;
            for (; u < NU; ++u) ukl[u] = -1;
            for (int e = 0; e < R + 2; ++e) Hs[TPp + e] = 0.0;
        }
    }
    __syncthreads();   // tables, records and the initialised barrier
    mbar_wait(bar, 0);
    if (a.truncation == 1) {   // single truncation: H(a, b, c) = 0 for a + b + c > p
        for (int q = tid; q < (pt + 1) * (pt + 1); q += NT) {
            const int aa = q / (pt + 1), bb = q - aa * (pt + 1);
            const int o = packed_row(aa, bb, pt);
            for (int c = max(p - aa - bb + 1, 0); c <= 2 * pt - aa - bb; ++c) Hs[o + c] = 0.0;
        }
        __syncthreads();
    }

    const int u = tid % NU, cg = tid / NU;
    const int kl = ukl[u];
    if (kl < 0 || cg * C >= cnt) return;
    const int k = kl >> 8, l0 = kl & 0xff;
    double2 acc[R][C];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = make_double2(0.0, 0.0);
    const double2 *X0 = Xs + cg * C * BPS;
    // one step j of the Hankel product: rows r use H[T(k,i) + l0 + j + r] = w[(j + r) % R]
    // (ring slot of H[.. + s] is s % R); x holds M'_(i,j) of the C pairs, xn is prefetched
    auto step = [&](const double *h, const double2 *X, int j, int t, double (&w)[R],
                    double2 (&xn)[C]) {
        double2 x[C];
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = xn[c];
#pragma unroll
        for (int c = 0; c < C; ++c) xn[c] = X[c * BPS + j + 1];   // next step (may run one past)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double hv = w[(t + r) % R];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                acc[r][c].x = fma(hv, x[c].x, acc[r][c].x);
                acc[r][c].y = fma(hv, x[c].y, acc[r][c].y);
            }
        }
        w[t] = h[j + R];
    };
    for (int i = 0; i <= p; ++i) {
        const int jn = p + 1 - i;   // steps j = 0 .. p - i
        const double *h = Hs + Tk[k * (p + 1) + i] + l0;
        const double2 *X = X0 + i * (p + 1) - i * (i - 1) / 2;
        double w[R];
        double2 xn[C];
#pragma unroll
        for (int r = 0; r < R; ++r) w[r] = h[r];
#pragma unroll
        for (int c = 0; c < C; ++c) xn[c] = X[c * BPS];
        int j0 = 0;
        for (; j0 + R <= jn; j0 += R) {   // full blocks: straight-line, loads run ahead
#pragma unroll
            for (int t = 0; t < R; ++t) step(h, X, j0 + t, t, w, xn);
        }
#pragma unroll
        for (int t = 0; t < R - 1; ++t)   // remainder (warp-uniform)
            if (j0 + t < jn) step(h, X, j0 + t, t, w, xn);
    }
    // rows (k, l0 + r): post-scale 1/l! (and (-1)^l for backward pairs), contiguous runs
    const int m0 = k * (pl + 1) - k * (k - 1) / 2 + l0;
    double f[R];
    {
        double fl = 1.0;
        for (int t = 2; t <= l0; ++t) fl *= t;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r > 0) fl *= (l0 + r);
            f[r] = 1.0 / fl;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int b = cg * C + c;
        if (b >= cnt) break;
        const int4 rc = rec[b];
        double2 *dst = a.pairbuf + ((int64_t)rc.y * KW + nloc) * Pl + m0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (l0 + r > pl - k) break;
            const double s = (rc.z && ((l0 + r) & 1)) ? -f[r] : f[r];
            dst[r] = make_double2(acc[r][c].x * s, acc[r][c].y * s);
        }
    }
}

// s2l_batch_units_kernel, U = 2: the same batch with two units per thread (u and u + NUT) on the
// same C pairs (the one-unit kernel above is kept as it is: the generalised source compiled to a
// slower one-unit kernel, C5 S2L 38.6 vs 36.0 ms).  The loop is bound by the
// shared-memory pipe as much as by the FP64 pipe (per step C 16-byte moment loads, 2 clocks each
// of the SM's register write-back, and one tensor value for 2 R C DFMA = 4 R C clocks of one of
// four FP64 pipes: (2 C + 1) / (R C) = 0.75 at 3 x 4, plus bank conflicts on the tensor loads;
// ncu: FP64 pipe 58%, memory pipes 79%); two units share the moment loads, halving them, without
// the row-slot waste of longer units (units of 6 rows: 198 slots for p = 16's 153 rows).
template <int R, int C, int NU, int CG, int U>
__global__ void __launch_bounds__(((NU + U - 1) / U) * CG, 3)
    s2l_batch_units_kernel(S2LArgs a)
{
    constexpr int NUT = (NU + U - 1) / U;   // unit slots (threads per column group)
    constexpr int NT = NUT * CG, JT = CG * C;
    extern __shared__ double sm[];
    const int p = a.p, P = a.P, pl = a.pl, Pl = a.Pl, pt = a.pt;
    const int KW = a.m1 - a.m0;
    const int TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1);
    const int BPS = P | 1;                            // moment row stride (complex, odd)
    double2 *Xs = reinterpret_cast<double2 *>(sm);   // [JT][BPS] moments
    double *Hs = reinterpret_cast<double *>(Xs + JT * BPS);   // [TPp + R + 2] (zero tail)
    uint64_t *bar = reinterpret_cast<uint64_t *>(Hs + TPp + R + 2 + ((R + 2) & 1));
    int4 *rec = reinterpret_cast<int4 *>(bar + 2);   // [JT]
    int *Tk = reinterpret_cast<int *>(rec + JT);     // [(pl+1) * (p+1)] row offsets T(k, i)
    int *ukl = Tk + 17 * 17;                         // [NU] units (k << 8 | l0), -1 = none

    const int nloc = (int)(blockIdx.x % KW);
    const int4 bt = a.batches[blockIdx.x / KW];
    const int cnt = bt.y, skey = bt.z, inward = skey & 1;
    const int64_t station = skey >> 1;
    const int tid = threadIdx.x;
    // warp 0 starts the copies at once (barrier, tensor block, one moment row per pair: backward
    // pairs read the copy with (-1)^j folded in) while the other warps build the index tables
    if (tid < 32) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(bar, (unsigned)(TPp * 8 + cnt * P * 16));
            bulk_g2s(Hs, a.tens + (station * KW + nloc) * (int64_t)TPp, (unsigned)(TPp * 8), bar);
        }
        __syncwarp();
        for (int b = tid; b < JT; b += 32) {
            const int4 pr = b < cnt ? a.pairs[bt.x + b] : make_int4(0, -1, 0, 0);
            rec[b] = pr;
            if (b < cnt)
                bulk_g2s(Xs + b * BPS, (pr.z ? a.Mb : a.M) + ((a.soff[pr.w] + pr.x) * KW + nloc) * P,
                         (unsigned)(P * 16), bar);
        }
    } else {
        for (int q = tid - 32; q < (pl + 1) * (p + 1); q += NT - 32) {
            const int k = q / (p + 1), i = q - k * (p + 1);
            Tk[q] = inward ? packed_row(i, k, pt) : packed_row(k, i, pt);
        }
        if (tid == 32) {
            int u = 0;
            for (int k = 0; k <= pl; ++k)
                for (int l0 = 0; l0 <= pl - k; l0 += R) ukl[u++] = (k << 8) | l0;
            for (; u < NU; ++u) ukl[u] = -1;
            for (int e = 0; e < R + 2; ++e) Hs[TPp + e] = 0.0;
        }
    }
    __syncthreads();   // tables, records and the initialised barrier
    mbar_wait(bar, 0);
    if (a.truncation == 1) {   // single truncation: H(a, b, c) = 0 for a + b + c > p
        for (int q = tid; q < (pt + 1) * (pt + 1); q += NT) {
            const int aa = q / (pt + 1), bb = q - aa * (pt + 1);
            const int o = packed_row(aa, bb, pt);
            for (int c = max(p - aa - bb + 1, 0); c <= 2 * pt - aa - bb; ++c) Hs[o + c] = 0.0;
        }
        __syncthreads();
    }

    const int ut = tid % NUT, cg = tid / NUT;
    int uk[U], ul0[U];
    bool uv[U];
#pragma unroll
    for (int e = 0; e < U; ++e) {
        const int u = ut + e * NUT;
        const int kl = u < NU ? ukl[u] : -1;
        uv[e] = kl >= 0;
        uk[e] = uv[e] ? kl >> 8 : 0;      // (an absent second unit walks unit (0, 0): discarded)
        ul0[e] = uv[e] ? kl & 0xff : 0;
    }
    if (!uv[0] || cg * C >= cnt) return;
    double2 acc[U][R][C];
#pragma unroll
    for (int e = 0; e < U; ++e)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[e][r][c] = make_double2(0.0, 0.0);
    const double2 *X0 = Xs + cg * C * BPS;
    // one step j of the Hankel product: rows r use H[T(k,i) + l0 + j + r] = w[(j + r) % R]
    // (ring slot of H[.. + s] is s % R); x holds M'_(i,j) of the C pairs, xn is prefetched
    auto step = [&](const double *const (&h)[U], const double2 *X, int j, int t, double (&w)[U][R],
                    double2 (&xn)[C]) {
        double2 x[C];
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = xn[c];
#pragma unroll
        for (int c = 0; c < C; ++c) xn[c] = X[c * BPS + j + 1];   // next step (may run one past)
#pragma unroll
        for (int e = 0; e < U; ++e) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double hv = w[e][(t + r) % R];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    acc[e][r][c].x = fma(hv, x[c].x, acc[e][r][c].x);
                    acc[e][r][c].y = fma(hv, x[c].y, acc[e][r][c].y);
                }
            }
        }
#pragma unroll
        for (int e = 0; e < U; ++e) w[e][t] = h[e][j + R];
    };
    for (int i = 0; i <= p; ++i) {
        const int jn = p + 1 - i;   // steps j = 0 .. p - i
        const double *h[U];
#pragma unroll
        for (int e = 0; e < U; ++e) h[e] = Hs + Tk[uk[e] * (p + 1) + i] + ul0[e];
        const double2 *X = X0 + i * (p + 1) - i * (i - 1) / 2;
        double w[U][R];
        double2 xn[C];
#pragma unroll
        for (int e = 0; e < U; ++e)
#pragma unroll
            for (int r = 0; r < R; ++r) w[e][r] = h[e][r];
#pragma unroll
        for (int c = 0; c < C; ++c) xn[c] = X[c * BPS];
        int j0 = 0;
        for (; j0 + R <= jn; j0 += R) {   // full blocks: straight-line, loads run ahead
#pragma unroll
            for (int t = 0; t < R; ++t) step(h, X, j0 + t, t, w, xn);
        }
#pragma unroll
        for (int t = 0; t < R - 1; ++t)   // remainder (warp-uniform)
            if (j0 + t < jn) step(h, X, j0 + t, t, w, xn);
    }
    // rows (k, l0 + r): post-scale 1/l! (and (-1)^l for backward pairs), contiguous runs
#pragma unroll
    for (int e = 0; e < U; ++e) {
        if (!uv[e]) break;
        const int k = uk[e], l0 = ul0[e];
        const int m0 = k * (pl + 1) - k * (k - 1) / 2 + l0;
        double f[R];
        {
            double fl = 1.0;
            for (int t = 2; t <= l0; ++t) fl *= t;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r > 0) fl *= (l0 + r);
                f[r] = 1.0 / fl;
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int b = cg * C + c;
            if (b >= cnt) break;
            const int4 rc = rec[b];
            double2 *dst = a.pairbuf + ((int64_t)rc.y * KW + nloc) * Pl + m0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (l0 + r > pl - k) break;
                const double sgn = (rc.z && ((l0 + r) & 1)) ? -f[r] : f[r];
                dst[r] = make_double2(acc[e][r][c].x * sgn, acc[e][r][c].y * sgn);
            }
        }
    }
}

template <int R, int C, int NU, int CG>
inline size_t s2l_smem_bytes(int p, int pl)
{
    constexpr int JT = CG * C;
    const int pt = p > pl ? p : pl;
    const int P = (p + 1) * (p + 2) / 2;
    const int TP = (pt + 1) * (pt + 1) * (pt + 1), TPp = TP + (TP & 1);
    return sizeof(double2) * (size_t)JT * (P | 1) + sizeof(double) * (TPp + R + 2 + ((R + 2) & 1)) +
           2 * sizeof(uint64_t) + sizeof(int4) * JT + sizeof(int) * (17 * 17 + NU);
}

// warp per (target box with >= 1 pair, mode): Lc[row][n] = sum over the box's pairs, in the
// fixed offset order, of their pair-buffer rows
struct S2LReduceArgs {
    int depth, nw, KW, Pl;
    int64_t lvoff[kMaxLevels + 1];
    const int *lrow;   // dense: Lc row of a materialised local
    const int *wlist, *poff, *pcnt;
    const double2 *pairbuf;
    double2 *Lc;
};
__global__ void __launch_bounds__(256) s2l_reduce_kernel(S2LReduceArgs a)
{
    const int lane = threadIdx.x & 31, KW = a.KW, Pl = a.Pl;
    const int64_t items = (int64_t)a.nw * KW;
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int g = a.wlist[it / KW], n = (int)(it % KW);
        const int64_t row = a.lrow[g];
        const int o = a.poff[g], c = a.pcnt[g];
        for (int e = lane; e < Pl; e += 32) {
            double2 s = a.pairbuf[((int64_t)o * KW + n) * Pl + e];
            for (int k = 1; k < c; ++k) {
                const double2 v = a.pairbuf[((int64_t)(o + k) * KW + n) * Pl + e];
                s.x += v.x;
                s.y += v.y;
            }
            a.Lc[(row * KW + n) * Pl + e] = s;
        }
    }
}

// Source moments pre-scaled once for S2L: M'_ij = (-1)^j M^_ij / j! (all levels, after M2M),
// and Mb = M^_ij / j! for backward pairs (their (-1)^j, cancels the forward sign).
__global__ void prescale_moments_kernel(double2 *M, double2 *Mb, int64_t nrows, int P,
                                        const double *pscale)
{
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nrows * P) return;
    const double f = __ldg(pscale + (int)(e % P));   // (-1)^j / j! of coefficient (i, j)
    const double2 v = M[e];
    M[e] = make_double2(v.x * f, v.y * f);
    Mb[e] = make_double2(v.x * fabs(f), v.y * fabs(f));
}

}  // namespace cyl
