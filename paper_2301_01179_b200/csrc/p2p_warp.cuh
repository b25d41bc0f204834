// p2p_warp.cuh -- FMM near field with warp-autonomous tasks: the paper's bottleneck
// (P:582-584, 729-733, 799-802), Phi_t^(n) += sum_s S_s^(n) G^(n)(r_t, r_s, z_t - z_s) over the
// sources of the 9 neighbour leaves of t's leaf, bitwise-coincident pairs skipped (R#15).
//
// Design (sm_100a, FP64 CUDA cores).  The CTA-wide variant (p2p.cuh) classifies and compacts
// pairs across the CTA and therefore synchronises four times per 128 pairs; on C2 a third of its
// stall samples were barrier waits and most issue slots went to index arithmetic.  Here every
// warp owns one task (<= 32 targets of one leaf) and never waits for another warp:
//   * lanes = (target tl, source slot sl), TW x SL = 32, TW = the task's target count rounded up
//     to a power of two (tasks are emitted as power-of-two-sized pieces of a leaf);
//   * the task's source rows (r, z and the K-mode coefficient row) are staged by the warp into
//     its own shared-memory slice, 32 sources per stage (odd row stride: the SL rows read by one
//     LDS.128 fall into distinct bank quads), __syncwarp only;
//   * per stage each lane classifies its pairs (forward chi < 1.008 / Miller / far chi >= 1000 /
//     skipped, R#3) and walks them class by class (forward, far, then Miller: iteration i of
//     the warp runs the same branch on as many lanes as the per-lane class counts allow);
//   * G^(n) is produced in registers and contracted at once into the lane's register
//     accumulators acc[n] (forward and far upward in n; Miller downward into w[n], normalised
//     upward by G^(0) = K/(pi rho_+) from the AGM), all in the forward recursion's units
//     u_n = G^(n) / R_n: the forward pairs add S u_n with no per-pair scaling, the far and Miller
//     factors carry 1 / R_n, and each (target, mode) sum is multiplied by R_n once at the end;
//   * the SL partial sums of a target are combined by a fixed xor-shuffle tree, so results are
//     bitwise reproducible.
// Mode window: all K <= KT modes in one pass (KT compile-time: register arrays).
#pragma once
#include "p2p.cuh"

namespace cyl {

constexpr int kWarpCH = 32;   // sources per warp stage
constexpr int kWinStart = 33; // first mode of the second window of a K in (33, 66] solve
constexpr int kWarps = 4;     // warps per CTA (one task per CTA, the source list split in four)

template <int KT>
__host__ __device__ constexpr int p2pw_row() { return KT | 1; }   // odd double2 row stride

// WSM ("wide occupancy"): four resident CTAs per SM (register cap 128) instead of three
template <int KT, bool WSM>
inline size_t p2pw_smem_bytes()
{
    return 4 * sizeof(double) +                          // one mbarrier per warp
           (size_t)kWarps * (sizeof(double2) * kWarpCH * p2pw_row<KT>() + sizeof(double) * 2 * kWarpCH +
                             2 * sizeof(int) * kWarpCH) +
           sizeof(int) * 20;
}
template <int KT, bool WSM>
__host__ __device__ constexpr int p2pw_min_blocks()
{
    return KT <= 9 ? 4 : (KT <= 17 ? (WSM ? 4 : 3) : 2);
}

// asynchronous global -> shared copies (LDGSTS): a stage's loads are all in flight at once
__device__ __forceinline__ void pw_async8(void *smem, const void *gmem)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void pw_async_wait()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
// a stage's coefficient rows arrive by one TMA bulk copy per source row on the warp's mbarrier
// (one instruction per row instead of a 16-byte cp.async per element with its address arithmetic)
__device__ __forceinline__ void pw_mbar_init(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void pw_mbar_expect(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void pw_bulk(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("fence.proxy.async.shared::cta;\n"
                 "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void pw_mbar_wait(uint64_t *bar, unsigned phase)
{
    asm volatile("{\n.reg .pred p;\nPW_WAIT_%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra PW_WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(phase)
                 : "memory");
}

__device__ __forceinline__ double2 cfma(double2 s, double g, double2 acc)
{
    acc.x = fma(s.x, g, acc.x);
    acc.y = fma(s.y, g, acc.y);
    return acc;
}

// A CTA works on one task at a time (<= 32 targets of one leaf); warp w takes the w-th quarter
// of the task's source list; the four partial sums are added in warp order at the end
// (deterministic).  Persistent CTAs fetch tasks from *a.task_ctr (zeroed before the launch).
// EXACT: the mode count equals KT (no per-mode guards).
// WIN: a mode window [m0, m0 + KW) of a K > KT solve (the recursions start at mode 0, only the
// window's modes are accumulated; forward pairs run two per lane in lockstep; m0 = 0 works too).
// DIRECT: the direct sum: task = (tile of 32 targets, source partition), the
// partition's partial sums written to out + part * part_stride (reduced in fixed order after).
template <int KT, bool EXACT, bool WSM, bool WIN = false, bool DIRECT = false, bool SV = false>
__global__ void __launch_bounds__(128, (p2pw_min_blocks<KT, WSM>())) p2p_warp_kernel(P2PArgs a)
{
    constexpr int CH = kWarpCH, ROW = p2pw_row<KT>();
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // layout: mbarriers [4] | S rows [kWarps][CH][ROW] double2 | r, z [kWarps][2 CH] |
    //         source index [kWarps][CH] | segments: starts [9], prefixes [9], total
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem) + warp;
    double2 *stS0 = reinterpret_cast<double2 *>(smem + 4);
    double2 *stS = stS0 + (size_t)warp * CH * ROW;
    double *stR = reinterpret_cast<double *>(stS0 + (size_t)kWarps * CH * ROW) + warp * 2 * CH;
    double *stZ = stR + CH;
    double *wbase = reinterpret_cast<double *>(stS0 + (size_t)kWarps * CH * ROW) + kWarps * 2 * CH;
    int *segS0 = reinterpret_cast<int *>(wbase) + kWarps * CH;
    int *segPre = segS0 + 9;
    int *stV = segS0 + 20 + warp * CH;                   // source index in the task's list

    if (lane == 0) pw_mbar_init(bar);
    __syncwarp();
    unsigned ph = 0;                                     // the warp's mbarrier phase
    unsigned my_skipped = 0, my_pairs = 0, my_fwd = 0, my_far = 0, my_mil = 0;
    unsigned long long my_msteps = 0;
    const int nparts = DIRECT ? (int)((a.ns + a.src_per_part - 1) / a.src_per_part) : 1;
    const int ntasks = DIRECT ? (int)((a.nf + 31) / 32) * nparts : *a.ntasks;
    for (;;) {                                           // persistent: fetch tasks heaviest first
    if (threadIdx.x == 0) segS0[18] = atomicAdd(a.task_ctr, 1);
    __syncthreads();
    const int task = segS0[18];
    __syncthreads();
    if (task >= ntasks) break;                           // CTA-uniform
    int4 tk;
    if (DIRECT) {
        const int tile = task / nparts, part = task % nparts;
        tk = make_int4(tile * 32, (int)min(a.nf, (int64_t)tile * 32 + 32), part, 0);
    } else {
        tk = a.tasks[task];
    }
    const int t0 = tk.x, nt = tk.y - tk.x;
    const int TW = nt <= 1 ? 1 : 1 << (32 - __clz(nt - 1));   // next power of two >= nt
    const int lgTW = __ffs(TW) - 1;
    const int SL = 32 >> lgTW;
    const int tl = lane & (TW - 1), sl = lane >> lgTW;
    const bool tvalid = tl < nt;
    const int KW = EXACT ? KT : a.m1 - a.m0;
    // (the saved-state second window of a K in (33, 66] solve starts at mode KT = 33: a
    // compile-time window start turns the recursion and Miller constants into immediates)
    const int M0 = WIN ? (SV ? kWinStart : a.m0) : 0, M1 = M0 + KW;

    // neighbour source segments (warp 0, lane k < 9 = neighbour k), prefix by shuffles; the
    // direct sum has one segment, the partition
    if (DIRECT && warp == 0) {
        const int64_t s0 = (int64_t)tk.z * a.src_per_part, s1 = min(a.ns, s0 + a.src_per_part);
        if (lane < 9) {
            segS0[lane] = lane == 0 ? (int)s0 : 0;
            segPre[lane] = lane == 0 ? 0 : (int)(s1 - s0);
        }
        if (lane == 8) segS0[18] = (int)(s1 - s0);
    } else if (warp == 0) {
        int s0 = 0, len = 0;
        if (lane < 9) {
            const int2 sg = near_segment(a.leafstart, a.depth, a.level ? a.level : a.depth,
                                         a.adaptive_leaf, (uint32_t)tk.z, lane);
            s0 = sg.x;
            len = sg.y;
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane < 9) {
            segS0[lane] = s0;
            segPre[lane] = incl - len;
        }
        if (lane == 8) segS0[18] = incl;                 // total (after segS0[9], segPre[9])
    }
    __syncthreads();
    const int total = segS0[18];
    // the warps' shares of the source list interleave in chunks of 4 (chunk c goes to warp
    // c mod 4): every warp sees all neighbour leaves, so the Miller / forward mix, and with it
    // the warps' durations, are alike (contiguous quarters left warps waiting at the final
    // barrier).  Warp-local index u -> source v = (4 (u / 4) + warp) 4 + u % 4 (chunks of 1,
    // 2, 4, 8, 16 measured: 1-4 alike, 8 and 16 slower).
    constexpr int ICH = 4;
    const int rem = total % (kWarps * ICH);
    const int vb = 0, ve = ICH * (total / (kWarps * ICH)) + min(max(rem - ICH * warp, 0), ICH);

    const double tr = a.fr[t0 + min(tl, nt - 1)], tz = a.fz[t0 + min(tl, nt - 1)];
    // window-state slots of this lane's target (see P2PArgs::save)
    int64_t tslot = 0;
    if (SV && !DIRECT && a.save) {
        const int lkey = tk.z;
        tslot = a.pbase[a.tmap_leaf[lkey]] + (int64_t)(t0 + tl - a.fleafstart[lkey]) * total;
    }
    double2 acc[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) acc[j] = make_double2(0.0, 0.0);
    const int Nglob = a.K - 1;
    const double fwd2 = a.fwd2;

    for (int v0 = vb; v0 < ve; v0 += CH) {
        const int nch = min(CH, ve - v0);
        __syncwarp();
        if (lane == 0) pw_mbar_expect(bar, (unsigned)(nch * KW) * (unsigned)sizeof(double2));
        if (lane < nch) {
            const int uu = v0 + lane;
            const int v = (kWarps * (uu / ICH) + warp) * ICH + uu % ICH;
            int k = 0;
#pragma unroll
            for (int kk = 1; kk < 9; ++kk) k += (v >= segPre[kk]);
            const int gi = segS0[k] + (v - segPre[k]);
            if (SV) stV[lane] = v;
            pw_async8(stR + lane, a.sr + gi);
            pw_async8(stZ + lane, a.sz + gi);
            // the source's coefficient row (modes M0 .. M0 + KW - 1): one bulk copy
            pw_bulk(stS + lane * ROW, a.S + (int64_t)gi * a.K + M0, (unsigned)(KW * sizeof(double2)), bar);
        }
        pw_async_wait();
        pw_mbar_wait(bar, ph);
        ph ^= 1u;
        __syncwarp();
        // classify this lane's pairs c = sl + SL i
        unsigned mF = 0, mX = 0, mM = 0, mL = 0;     // forward, far, Miller short / long
        const int npl = (nch - sl + SL - 1) / SL;    // pairs of this lane (may be <= 0)
        if (tvalid) {
            for (int i = 0; i < npl; ++i) {
                const int c = sl + SL * i;
                const double r1 = stR[c], z1 = stZ[c];
                if (tr == r1 && tz == z1) {
                    if (a.exclude) ++my_skipped;
                    else atomicOr(a.err_flag, 1);
                    continue;
                }
                const PairGeo g = pair_geo(tr, r1, tz - z1, fwd2);
                if (g.forward) mF |= 1u << i;
                else if (g.far) mX |= 1u << i;
                else if (g.rm2 < 0.1122 * g.rr1) mL |= 1u << i;   // chi < 1.0561: e >= 64
                else mM |= 1u << i;
            }
        }
        const int nF = __popc(mF), nX = __popc(mX), nM = __popc(mM) + __popc(mL);
        my_pairs += nF + nX + nM;
        my_fwd += nF;
        my_far += nX;
        my_mil += nM;
        // forward pairs on u_n = G_n / R_n, K, E by the small-k' series.  The
        // recursion is a chain of dependent FMAs: in the windowed pass (K > KT, where the chain
        // also advances to the window) two pairs per lane run in lockstep to hide its latency;
        // a missing second pair runs with zero seeds (the recursion is linear: exact zeros).
        constexpr bool TWO = WIN || SV || (!DIRECT && KT <= 17);   // (SV: both windows of a K in (33, 66] solve)
        const bool load = SV && WIN && a.save == 2;   // (u_31, u_32) from the first window
        // load mode: the states of the next iteration's pairs are fetched one iteration ahead
        double2 pfA = make_double2(0.0, 0.0), pfB = make_double2(0.0, 0.0);
        auto prefetch = [&](unsigned m) {
            if (!m) return;
            pfA = a.sv2[tslot + stV[sl + SL * (__ffs(m) - 1)]];
            const unsigned m2 = m & (m - 1);
            if (TWO && m2) pfB = a.sv2[tslot + stV[sl + SL * (__ffs(m2) - 1)]];
        };
        if (load) prefetch(mF);
        const int itF = __reduce_max_sync(0xffffffffu, TWO ? (nF + 1) >> 1 : nF);
        for (int it = 0; it < itF; ++it) {
            int ia = -1, ib = -1;
            if (mF) { ia = __ffs(mF) - 1; mF &= mF - 1; }
            if (TWO && mF) { ib = __ffs(mF) - 1; mF &= mF - 1; }
            if (ia < 0) continue;
            const double2 sA = pfA, sBp = pfB;
            if (load) prefetch(mF);
            const int ca = sl + SL * ia, cb = ib >= 0 ? sl + SL * ib : ca;
            const double wb = ib >= 0 ? 1.0 : 0.0;
            const PairGeo gA = pair_geo(tr, stR[ca], tz - stZ[ca], fwd2);
            const double2 *SA = stS + ca * ROW, *SB = stS + cb * ROW;
            const double irA = rcp_nr(gA.rr1);
            const double dA = 0.5 * gA.rm2 * irA;   // chi - 1, exact to rounding (R#24)
            double u0A, u1A, u0B = 0.0, u1B = 0.0, dB = 0.0;
            if (load) {
                u0A = sA.x;
                u1A = sA.y;
            } else {
                const double ipA = rsqrt_nr(gA.rp2);
                double KA, EA;
                ke_small(gA.rm2 * ipA * ipA, KA, EA);
                const double G0A = KA * ipA * (1.0 / kPi);
                const double chA = 0.25 * (gA.rp2 + gA.rm2) * irA;
                u0A = G0A;
                u1A = G0A * fma(-(1.0 + chA), EA * rcp_nr(KA), chA);
            }
            if constexpr (TWO) {
                const PairGeo gB = pair_geo(tr, stR[cb], tz - stZ[cb], fwd2);
                const double irB = rcp_nr(gB.rr1);
                dB = 0.5 * gB.rm2 * irB;
                if (load) {
                    const double2 sB = ib >= 0 ? sBp : make_double2(0.0, 0.0);
                    u0B = sB.x;
                    u1B = sB.y;
                } else {
                    const double ipB = rsqrt_nr(gB.rp2);
                    double KB, EB;
                    ke_small(gB.rm2 * ipB * ipB, KB, EB);
                    const double G0B = KB * ipB * (wb / kPi);
                    const double chB = 0.25 * (gB.rp2 + gB.rm2) * irB;
                    u0B = G0B;
                    u1B = G0B * fma(-(1.0 + chB), EB * rcp_nr(KB), chB);
                }
            }
            if constexpr (WIN) {                        // advance to the window (M0 >= 2)
#pragma unroll 4
                for (int n = load ? M0 : 2; n < M0; ++n) {
                    const double e = c_rec.eps[n];
                    const double u2A = fma(dA, u1A, fma(-e, u0A, u1A));
                    u0A = u1A;
                    u1A = u2A;
                    if constexpr (TWO) {
                        const double u2B = fma(dB, u1B, fma(-e, u0B, u1B));
                        u0B = u1B;
                        u1B = u2B;
                    }
                }
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    if (j < KW) {
                        const int n = M0 + j;
                        if (n < 2) {                    // the first window: the seeds
                            const double gA = n == 0 ? u0A : u1A, gB = n == 0 ? u0B : u1B;
                            acc[j] = cfma(SA[j], gA, acc[j]);
                            if constexpr (TWO) acc[j] = cfma(SB[j], gB, acc[j]);
                            continue;
                        }
                        const double e = c_rec.eps[n];
                        const double u2A = fma(dA, u1A, fma(-e, u0A, u1A));
                        acc[j] = cfma(SA[j], u2A, acc[j]);
                        u0A = u1A;
                        u1A = u2A;
                        if constexpr (TWO) {
                            const double u2B = fma(dB, u1B, fma(-e, u0B, u1B));
                            acc[j] = cfma(SB[j], u2B, acc[j]);
                            u0B = u1B;
                            u1B = u2B;
                        }
                    }
                }
            } else {
                acc[0] = cfma(SA[0], u0A, acc[0]);
                if (KW > 1) acc[1] = cfma(SA[1], u1A, acc[1]);
                if constexpr (TWO) {
                    acc[0] = cfma(SB[0], u0B, acc[0]);
                    if (KW > 1) acc[1] = cfma(SB[1], u1B, acc[1]);
                }
#pragma unroll
                for (int n = 2; n < KT; ++n) {
                    if (n < KW) {
                        const double u2A = fma(dA, u1A, fma(-c_rec.eps[n], u0A, u1A));
                        acc[n] = cfma(SA[n], u2A, acc[n]);
                        u0A = u1A;
                        u1A = u2A;
                        if constexpr (TWO) {
                            const double u2B = fma(dB, u1B, fma(-c_rec.eps[n], u0B, u1B));
                            acc[n] = cfma(SB[n], u2B, acc[n]);
                            u0B = u1B;
                            u1B = u2B;
                        }
                    }
                }
                if (SV && a.save == 1) {   // (u_31, u_32) for the second window
                    a.sv2[tslot + stV[ca]] = make_double2(u0A, u1A);
                    if (TWO && ib >= 0) a.sv2[tslot + stV[cb]] = make_double2(u0B, u1B);
                }
            }
        }
        // far pairs (chi >= 1000), one per lane and iteration: hypergeometric form (DLMF
        // 14.3.7), see greens_far; every mode is independent (no chain)
        const int itX = __reduce_max_sync(0xffffffffu, nX);
        for (int it = 0; it < itX; ++it) {
            if (!mX) continue;
            const int idx = __ffs(mX) - 1;
            mX &= mX - 1;
            const int c = sl + SL * idx;
            const PairGeo g = pair_geo(tr, stR[c], tz - stZ[c], fwd2);
            const double2 *Srow = stS + c * ROW;
            const double sum2 = 0.5 * (g.rp2 + g.rm2);
            const double isum = rcp_nr(sum2);
            const double q = g.rr1 * isum, z = 4.0 * q * q;
            double qn = rsqrt_nr(sum2);
            if constexpr (WIN) {
                for (int n = 0; n < M0 - 1; ++n) qn *= q;   // q^(M0-1): the loop multiplies once more
            }
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                if (j < KW) {
                    const int n = M0 + j;
                    if (n > 0) qn *= q;
                    double t = z * c_rec.farT[n][3];
                    t = z * c_rec.farT[n][2] * (1.0 + t);
                    t = z * c_rec.farT[n][1] * (1.0 + t);
                    t = z * c_rec.farT[n][0] * (1.0 + t);
                    acc[j] = cfma(Srow[j], c_rec.farAR[n] * qn * (1.0 + t), acc[j]);
                }
            }
        }
        // Miller pairs, two per lane and iteration in lockstep (two independent
        // dependency chains per lane: the recursion is latency-bound).  w_n is recomputed in a
        // second pass over the last KW steps instead of being stored: pass 1 yields w_0 and the
        // normalisation c = G^(0) / w_0, pass 2 contracts G_n = w_n P_n c (2 chi)^-n downward.
        const int itM = __reduce_max_sync(0xffffffffu, (nM + 1) >> 1);
        for (int it = 0; it < itM; ++it) {
            int ia = -1, ib = -1;
            // long chains first, so that lanes run chains of similar length side by side
            if (mL) { ia = __ffs(mL) - 1; mL &= mL - 1; }
            else if (mM) { ia = __ffs(mM) - 1; mM &= mM - 1; }
            if (mL) { ib = __ffs(mL) - 1; mL &= mL - 1; }
            else if (mM) { ib = __ffs(mM) - 1; mM &= mM - 1; }
            const bool va = ia >= 0, vb = ib >= 0;
            const int ca = sl + SL * (va ? ia : 0), cb = vb ? sl + SL * ib : ca;
            const PairGeo gA = pair_geo(tr, stR[ca], tz - stZ[ca], fwd2);
            const PairGeo gB = pair_geo(tr, stR[cb], tz - stZ[cb], fwd2);
            const int eA = va ? miller_extra(gA, a.miller) : 0, eB = vb ? miller_extra(gB, a.miller) : 0;
            const int S_lane = va ? Nglob + max(eA, eB) : 0;
            my_msteps += (unsigned)(eA + eB);
            const int S_warp = __reduce_max_sync(0xffffffffu, S_lane);
            if (va) {
                const double sumA = 0.5 * (gA.rp2 + gA.rm2), sumB = 0.5 * (gB.rp2 + gB.rm2);
                const double i2A = gA.rr1 * rcp_nr(sumA), i2B = gB.rr1 * rcp_nr(sumB);   // 1/(2 chi)
                const double qA = i2A * i2A, qB = i2B * i2B;
                double wnA, wlA, wnB, wlB, cvA, cvB;
                if (SV && WIN && a.save == 2) {   // the first window's chain state (see P2PArgs::save)
                    const double2 sA = a.sv2[tslot + stV[ca]];
                    wnA = sA.x;
                    wlA = sA.y;
                    cvA = a.sv1[tslot + stV[ca]];
                    const double2 sB = vb ? a.sv2[tslot + stV[cb]] : make_double2(0.0, 0.0);
                    wnB = sB.x;
                    wlB = sB.y;
                    cvB = vb ? a.sv1[tslot + stV[cb]] : 0.0;
                } else {
                const double ipA = rsqrt_nr(gA.rp2), ipB = rsqrt_nr(gB.rp2);
                // AGM(1, k') of both pairs (K = pi / (2 AGM)); a converged pair is frozen
                double a1 = 1.0, b1 = sqrt_nr(gA.rm2) * ipA, a2 = 1.0, b2 = sqrt_nr(gB.rm2) * ipB;
#pragma unroll 1
                for (int k = 0; k < 40; ++k) {
                    const bool uA = fabs(0.5 * (a1 - b1)) > 2.0e-16 * a1;
                    const bool uB = fabs(0.5 * (a2 - b2)) > 2.0e-16 * a2;
                    if (!uA && !uB) break;
                    const double nA = 0.5 * (a1 + b1), nB = 0.5 * (a2 + b2);
                    const double sA = sqrt_nr(a1 * b1), sB = sqrt_nr(a2 * b2);
                    if (uA) { a1 = nA; b1 = sA; }
                    if (uB) { a2 = nB; b2 = sB; }
                }
                const double G0A = 0.5 * ipA * rcp_nr(a1), G0B = 0.5 * ipB * rcp_nr(a2);
                wnA = 0.0;
                wlA = 1.0;
                wnB = 0.0;
                wlB = 1.0;
                // first window of a two-window solve: the chain state at (K + 1, K), kept in the
                // final scaling, is what the second window's contraction restarts from (the
                // start S >= K - 1 + 7 lies above it)
                const int ncap = (SV && !WIN && a.save == 1) ? a.K + 1 : -1;
                double cnA = 0.0, clA = 0.0, cnB = 0.0, clB = 0.0;
                int n = S_warp;
                while (n > M1 + 1) {
                    int nstop = max(M1 + 1, n - 64);
                    if (ncap > nstop && n > ncap) nstop = ncap;
#pragma unroll 4
                    for (; n > nstop; --n) {
                        const double d = c_rec.delta[n];
                        const double wA = fma(-d * qA, wnA, wlA);
                        const double wB = fma(-d * qB, wnB, wlB);
                        wnA = wlA;
                        wlA = wA;
                        wnB = wlB;
                        wlB = wB;
                    }
                    int exA, exB;
                    frexp(wlA, &exA);
                    wnA = ldexp(wnA, -exA);
                    wlA = ldexp(wlA, -exA);
                    frexp(wlB, &exB);
                    wnB = ldexp(wnB, -exB);
                    wlB = ldexp(wlB, -exB);
                    if (ncap > 0) {
                        if (n == ncap) {               // captured after this block's rescaling
                            cnA = wnA;
                            clA = wlA;
                            cnB = wnB;
                            clB = wlB;
                        } else if (n < ncap) {         // later rescalings apply to the capture
                            cnA = ldexp(cnA, -exA);
                            clA = ldexp(clA, -exA);
                            cnB = ldexp(cnB, -exB);
                            clB = ldexp(clB, -exB);
                        }
                    }
                }
                // pass 1: w_0 of both chains (wl = w_M1, wn = w_{M1+1} here)
                double xnA = wnA, xlA = wlA, xnB = wnB, xlB = wlB;
                cvA = 1.0;
                cvB = 1.0;
                if constexpr (WIN) {                    // steps below the window (n = M0 + 1 .. 2)
                    for (int j = KW - 1; j >= 0; --j) {
                        const double d = c_rec.delta[M0 + j + 2];
                        const double wA = fma(-d * qA, xnA, xlA);
                        const double wB = fma(-d * qB, xnB, xlB);
                        xnA = xlA;
                        xlA = wA;
                        xnB = xlB;
                        xlB = wB;
                        if (M0 + j > 0) {               // w_{M0+j} produced: (2 chi)^-1 unless n = 0
                            cvA *= i2A;
                            cvB *= i2B;
                        }
                    }
                    for (int m = M0 + 1; m >= 2; --m) {
                        const double d = c_rec.delta[m];
                        const double wA = fma(-d * qA, xnA, xlA);
                        const double wB = fma(-d * qB, xnB, xlB);
                        xnA = xlA;
                        xlA = wA;
                        xnB = xlB;
                        xlB = wB;
                        if (m > 2) {
                            cvA *= i2A;
                            cvB *= i2B;
                        }
                    }
                }
#pragma unroll
                for (int j = KT - 1; j >= 0; --j) {
                    if (!WIN && j < KW) {
                        const double d = c_rec.delta[j + 2];
                        const double wA = fma(-d * qA, xnA, xlA);
                        const double wB = fma(-d * qB, xnB, xlB);
                        xnA = xlA;
                        xlA = wA;
                        xnB = xlB;
                        xlB = wB;
                        if (j > 0) {
                            cvA *= i2A;
                            cvB *= i2B;
                        }
                    }
                }
                cvA *= G0A * rcp_nr(xlA);                // c (2 chi)^-(M1-1)
                cvB = vb ? cvB * (G0B * rcp_nr(xlB)) : 0.0;
                if (ncap > 0) {   // second window's start: (w_{K+1}, w_K), c (2 chi)^-(K-1)
                    double pA = 1.0, pB = 1.0;        // (2 chi)^-((K - 1) - (M1 - 1))
                    for (int t = M1; t < a.K; ++t) {
                        pA *= i2A;
                        pB *= i2B;
                    }
                    a.sv2[tslot + stV[ca]] = make_double2(cnA, clA);
                    a.sv1[tslot + stV[ca]] = cvA * pA;
                    if (vb) {
                        a.sv2[tslot + stV[cb]] = make_double2(cnB, clB);
                        a.sv1[tslot + stV[cb]] = cvB * pB;
                    }
                }
                }
                const double tcA = sumA * rcp_nr(gA.rr1), tcB = sumB * rcp_nr(gB.rr1);   // 2 chi
                // pass 2: G_n = w_n P_n c (2 chi)^-n, n = M0 + j, j = KW-1 .. 0
#pragma unroll
                for (int j = KT - 1; j >= 0; --j) {
                    if (j < KW) {
                        const int nn = M0 + j;
                        const double d = c_rec.delta[nn + 2];
                        const double wA = fma(-d * qA, wnA, wlA);
                        const double wB = fma(-d * qB, wnB, wlB);
                        wnA = wlA;
                        wlA = wA;
                        wnB = wlB;
                        wlB = wB;
                        const double2 SA = stS[ca * ROW + j], SB = stS[cb * ROW + j];
                        acc[j] = cfma(SA, wA * c_rec.PnR[nn] * cvA, acc[j]);
                        acc[j] = cfma(SB, wB * c_rec.PnR[nn] * cvB, acc[j]);
                        cvA *= tcA;
                        cvB *= tcB;
                    }
                }
            }
        }
    }
    // combine the SL partial sums of each target (fixed xor tree), then the four warps in order
    for (int o = TW; o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            acc[j].x += __shfl_xor_sync(0xffffffffu, acc[j].x, o);
            acc[j].y += __shfl_xor_sync(0xffffffffu, acc[j].y, o);
        }
    }
    __syncthreads();                                     // staging buffers are free
    double2 *red = stS0;                                 // [kWarps][KT][32] <= [kWarps][CH][ROW]
    if (sl == 0) {
#pragma unroll
        for (int j = 0; j < KT; ++j)
            if (j < KW) red[(warp * KT + j) * 32 + tl] = acc[j];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nt * KW; e += 32 * kWarps) {
        const int t = e / KW, j = e - t * KW;
        double2 v = red[j * 32 + t];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) {
            const double2 p = red[(w * KT + j) * 32 + t];
            v.x += p.x;
            v.y += p.y;
        }
        const double Rn = c_rec.Rn[M0 + j];             // u units -> G (see RecTables::farAR)
        v.x *= Rn;
        v.y *= Rn;
        const int64_t row = a.out_row ? a.out_row[t0 + t] : (t0 + t);
        double2 *o = a.out + (DIRECT ? tk.z * a.part_stride : 0) + row * a.K + a.m0 + j;
        if (a.accumulate) {
            const double2 p = *o;
            v.x += p.x;
            v.y += p.y;
        }
        *o = v;
    }
    }   // task loop
    my_skipped = __reduce_add_sync(0xffffffffu, my_skipped);
    my_pairs = __reduce_add_sync(0xffffffffu, my_pairs);
    if (a.m0 > 0) my_skipped = my_pairs = 0;            // counted by the first window
    if (lane == 0 && a.n_skipped && my_skipped) atomicAdd(a.n_skipped, (unsigned long long)my_skipped);
    if (lane == 0 && a.n_pairs && my_pairs) atomicAdd(a.n_pairs, (unsigned long long)my_pairs);
    if (a.m0 == 0 && a.n_branch) {
        my_fwd = __reduce_add_sync(0xffffffffu, my_fwd);
        my_far = __reduce_add_sync(0xffffffffu, my_far);
        my_mil = __reduce_add_sync(0xffffffffu, my_mil);
        for (int o = 16; o > 0; o >>= 1) my_msteps += __shfl_xor_sync(0xffffffffu, my_msteps, o);
        if (lane == 0) {
            if (my_fwd) atomicAdd(a.n_branch + 0, (unsigned long long)my_fwd);
            if (my_far) atomicAdd(a.n_branch + 1, (unsigned long long)my_far);
            if (my_mil) atomicAdd(a.n_branch + 2, (unsigned long long)my_mil);
            if (my_msteps) atomicAdd(a.n_branch + 3, my_msteps);
        }
    }
}

// Near-field tasks for the warp kernel: each target leaf is cut into pieces of 32 targets, the
// remainder r < 32 into power-of-two pieces unless r fills >= 3/4 of the next power of two.
// Tasks are emitted heaviest first (32 buckets by log2 of lanes x sources; the task order
// does not affect any result: every task owns its output rows), so the persistent CTAs finish
// together.  ctr layout: [0] ntasks, [1] fetch counter, [2..33] bucket counts, [34..65] fill.
// size of the next piece of a leaf with nt >= 1 remaining targets
__device__ __forceinline__ int piece_size(int nt)
{
    if (nt >= 32) return 32;
    const int p = nt <= 1 ? 1 : 1 << (32 - __clz(nt - 1));
    return (4 * nt >= 3 * p) ? nt : p / 2;
}
constexpr int kTaskCtrInts = 66;
__device__ __forceinline__ int near_sources(int key, const int *slstart, int depth, int level = 0,
                                            int sigma = 0)
{
    int tot = 0;
    for (int k = 0; k < 9; ++k)
        tot += near_segment(slstart, depth, level ? level : depth, sigma, (uint32_t)key, k).y;
    return tot;
}
// window-state slots: pairs per target leaf (targets x sources of the 9 neighbours), by leaf slot
__global__ void near_leaf_pairs_kernel(const int *tmap_leaf, const int *flstart, const int *slstart,
                                       int depth, int64_t *cnt)
{
    const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (key >= ((int64_t)1 << (2 * depth))) return;
    const int s = tmap_leaf[key];
    if (s < 0) return;
    cnt[s] = (int64_t)(flstart[key + 1] - flstart[key]) * near_sources((int)key, slstart, depth);
}
__global__ void total64_kernel(const int64_t *scan, const int64_t *v, int64_t n, int64_t *out)
{
    if (threadIdx.x == 0) *out = n > 0 ? scan[n - 1] + v[n - 1] : 0;
}

__device__ __forceinline__ int task_bucket(int nt, int nsrc)
{
    const int tw = nt <= 1 ? 1 : 1 << (32 - __clz(nt - 1));
    const unsigned cost = (unsigned)tw * (unsigned)max(nsrc, 1);
    return 31 - __clz(cost);
}
// skip_empty: leaves without a source in their 9 neighbours get no task (the near field only
// adds onto rows the far field wrote: an empty task would add zeros)
// level, sigma: tasks for the target boxes of one level under the adaptive source tree (R#26;
// level 0 = the leaf level, sigma 0 = uniform)
__global__ void near_wtasks_count_kernel(const int *tkeys, int nleaf, const int *flstart,
                                         const int *slstart, int depth, int skip_empty, int level,
                                         int sigma, int *ctr)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nleaf) return;
    const int key = tkeys[s];
    const int nsrc = near_sources(key, slstart, depth, level, sigma);
    if (skip_empty && nsrc == 0) return;
    const int sh = 2 * (depth - (level ? level : depth));
    int nt = flstart[(int64_t)(key + 1) << sh] - flstart[(int64_t)key << sh];
    if (nt >= 32) {   // the run of full pieces: one update (see the emit kernel)
        atomicAdd(&ctr[2 + task_bucket(32, nsrc)], nt / 32);
        nt &= 31;
    }
    while (nt > 0) {
        const int take = piece_size(nt);
        atomicAdd(&ctr[2 + task_bucket(take, nsrc)], 1);
        nt -= take;
    }
}
__global__ void near_wtasks_emit_kernel(const int *tkeys, int nleaf, const int *flstart,
                                        const int *slstart, int depth, int skip_empty, int level,
                                        int sigma, int4 *tasks, int *ctr)
{
    __shared__ int off[32];
    if (threadIdx.x < 32) {
        int o = 0;                                       // buckets in descending order
        for (int b = 31; b > (int)threadIdx.x; --b) o += ctr[2 + b];
        off[threadIdx.x] = o;
        if (blockIdx.x == 0 && threadIdx.x == 0) ctr[0] = o + ctr[2];
    }
    __syncthreads();
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nleaf) return;
    const int key = tkeys[s];
    const int nsrc = near_sources(key, slstart, depth, level, sigma);
    if (skip_empty && nsrc == 0) return;
    const int sh = 2 * (depth - (level ? level : depth));
    int t = flstart[(int64_t)key << sh], nt = flstart[(int64_t)(key + 1) << sh] - t;
    if (nt >= 32) {
        // the full pieces of a box share a bucket: one returning atomic reserves their slots (a
        // coarse box of the adaptive tree holds up to ~10^5 targets, and a round trip per piece in
        // one thread made this kernel 0.5 ms per level at C4: 5.0 of the solve's 83 ms under ncu)
        const int nfull = nt / 32, b = task_bucket(32, nsrc);
        int4 *dst = tasks + off[b] + atomicAdd(&ctr[34 + b], nfull);
        for (int i = 0; i < nfull; ++i, t += 32) dst[i] = make_int4(t, t + 32, key, 0);
        nt &= 31;
    }
    while (nt > 0) {
        const int take = piece_size(nt);
        const int b = task_bucket(take, nsrc);
        tasks[off[b] + atomicAdd(&ctr[34 + b], 1)] = make_int4(t, t + take, key, 0);
        t += take;
        nt -= take;
    }
}

}  // namespace cyl
