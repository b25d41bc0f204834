// cylfmm.cu -- libcylfmm.so: the C-ABI of include/cylfmm.h and the single-GPU orchestration of
// the paper's Algorithm 1.  Product code for sm_100a; independent of oracle/.
#include "../../include/cylfmm.h"

#include <cuda_runtime.h>
#include <nccl.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "fmm_ops.cuh"
#include "s2l.cuh"
#include "p2p.cuh"
#include "p2p_warp.cuh"
#include "specfun.cuh"
#include "tensor.cuh"
#include "tree.cuh"

using namespace cyl;

// ------------------------------------------------------------------------------------------
// errors
static thread_local std::string g_last_error;
static void set_err(const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
}
#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_err("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));       \
            return e_ == cudaErrorMemoryAllocation ? CYLFMM_ENOMEM : CYLFMM_ECUDA;            \
        }                                                                                     \
    } while (0)
#define CKL()  CK(cudaGetLastError())
#define RET_IF(st)                                                                            \
    do {                                                                                      \
        cylfmm_status s_ = (st);                                                              \
        if (s_ != CYLFMM_OK) return s_;                                                       \
    } while (0)

// ------------------------------------------------------------------------------------------
// NCCL, loaded at run time (only the multi-device entry points need it): the process's
// libnccl.so.2 (PyTorch's when torch.distributed is up, else the system one).  Types from nccl.h.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char *(*GetErrorString)(ncclResult_t);
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;
static bool load_nccl()
{
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.ok) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
#define SYM(F) g_nccl.F = reinterpret_cast<decltype(g_nccl.F)>(dlsym(h, "nccl" #F))
    SYM(GetUniqueId);
    SYM(CommInitRank);
    SYM(CommDestroy);
    SYM(Broadcast);
    SYM(AllGather);
    SYM(GroupStart);
    SYM(GroupEnd);
    SYM(GetErrorString);
#undef SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.Broadcast &&
                g_nccl.AllGather && g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.GetErrorString;
    return g_nccl.ok;
}
#define NC(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            set_err("%s:%d %s: %s", __FILE__, __LINE__, #call, g_nccl.GetErrorString(r_));    \
            return CYLFMM_ENCCL;                                                              \
        }                                                                                     \
    } while (0)

extern "C" const char *cylfmm_status_string(cylfmm_status s)
{
    switch (s) {
    case CYLFMM_OK: return "ok";
    case CYLFMM_EINVAL: return "invalid argument";
    case CYLFMM_EDOMAIN: return "point outside the domain (r <= 0, non-finite, or outside [0,L]x[z0,z0+L])";
    case CYLFMM_ENUMERIC: return "numerical error (unexcluded coincident pair or non-finite value)";
    case CYLFMM_ECUDA: return "CUDA error";
    case CYLFMM_ENCCL: return "NCCL error";
    case CYLFMM_ENOMEM: return "out of device memory";
    }
    return "unknown status";
}
extern "C" const char *cylfmm_last_error(void) { return g_last_error.c_str(); }
extern "C" const char *cylfmm_version(void) { return "cylfmm-b200 0.1 (sm_100a, FP64)"; }

// ------------------------------------------------------------------------------------------
// per-device init: recursion tables into constant memory, smem opt-in for the kernels
static std::mutex g_init_mu;
static bool g_init_done[64];

template <typename F>
static cudaError_t allow_smem(F *kernel)
{
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

#define P2PW_INSTANCES(X) X(9, true, false, false, false, false) X(17, true, false, false, false, false) \
    X(33, true, false, false, false, false) X(9, false, false, false, false, false)                    \
    X(17, false, false, false, false, false) X(33, false, false, false, false, false)                  \
    X(33, false, false, true, false, false) X(9, true, false, false, true, false)                      \
    X(17, true, false, false, true, false) X(33, true, false, false, true, false)                      \
    X(9, false, false, false, true, false) X(17, false, false, false, true, false)                     \
    X(33, false, false, false, true, false) X(33, false, false, true, true, false)                     \
    X(33, true, false, false, false, true) X(33, false, false, true, false, true)                      \
    X(32, true, false, true, false, true)
#define P2P_INSTANCES(X)                                                                       \
    X(8, 16, 2) X(8, 16, 5) X(16, 8, 3) X(16, 8, 9) X(32, 4, 6) X(32, 4, 18)

// S2L batch shapes (R rows per unit, C pairs per thread, NU units >= units(pl, R), CG column
// groups) per local-order class; JT = CG C pairs per batch
#define S2L_P8 3, 4, 18, 8
#define S2L_P12 3, 4, 35, 8
#define S2L_P16 3, 4, 57, 3
#define S2L_ALL(X) X(S2L_P8) X(S2L_P12) X(S2L_P16)

// Stream-ordered scratch of the plan-less entry points (direct sum, test batches) comes from a
// library-owned pool that keeps up to 64 MB cached: the device's default pool returns its memory
// to the driver at every synchronisation, which made each small synchronising call re-map its
// scratch (9 ms per C1 direct sum against 0.12 ms of work).
static cudaMemPool_t g_pool[64];
static cylfmm_status scratch_alloc(void **ptr, size_t bytes, cudaStream_t st)
{
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 64 && g_pool[dev]) CK(cudaMallocFromPoolAsync(ptr, bytes, g_pool[dev], st));
    else CK(cudaMallocAsync(ptr, bytes, st));
    return CYLFMM_OK;
}

static cylfmm_status ensure_init()
{
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (dev < 64 && g_init_done[dev]) return CYLFMM_OK;
    RecTables *t = new RecTables;
    build_rec_tables(t);
    cudaError_t e = cudaMemcpyToSymbol(c_rec, t, sizeof(RecTables));
    delete t;
    CK(e);
#define X(KT, E, W, N, DR, SV) CK(allow_smem(p2p_warp_kernel<KT, E, W, N, DR, SV>));
    P2PW_INSTANCES(X)
#undef X
#define X(TT, SC, MT)                                                                          \
    CK(allow_smem(p2p_kernel<TT, SC, MT, true>));                                              \
    CK(allow_smem(p2p_kernel<TT, SC, MT, true, true>));                                        \
    CK(allow_smem(p2p_kernel<TT, SC, MT, false>));
    P2P_INSTANCES(X)
#undef X
    CK(allow_smem(tensor_seed_kernel));
    CK(allow_smem(p2m_kernel<2>));
    CK(allow_smem(p2m_kernel<3>));
    CK(allow_smem(p2m_kernel<5>));
    CK(allow_smem(m2m_kernel));
    CK(allow_smem(l2l_kernel));
    CK(allow_smem(l2p_kernel<4, false>));
    CK(allow_smem(l2p_kernel<9, false>));
    CK(allow_smem(l2p_kernel<13, false>));
    CK(allow_smem(l2p_kernel<16, false>));
    CK(allow_smem(l2p_kernel<4, false, 2>));
    CK(allow_smem(l2p_kernel<9, false, 2>));
    CK(allow_smem(l2p_kernel<13, false, 2>));
    CK((allow_smem(l2p_kernel<13, false, 2, 16, true>)));
    CK(allow_smem(l2p_kernel<16, false, 2>));
    CK(allow_smem(l2p_kernel<16, true>));
#define X(...) CK(allow_smem(s2l_batch_kernel<__VA_ARGS__>));
    S2L_ALL(X)
#undef X
    CK((allow_smem(s2l_batch_units_kernel<S2L_P16, 2>)));
    if (dev < 64) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        CK(cudaMemPoolCreate(&g_pool[dev], &props));
        uint64_t keep = 64ull << 20;
        CK(cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep));
        g_init_done[dev] = true;
    }
    return CYLFMM_OK;
}

static cylfmm_status launch_p2m(const FarArgs &fa, unsigned grid, int P, int pp, cudaStream_t st)
{
    switch (p2m_rc(P)) {
    case 2: p2m_kernel<2><<<grid, kP2MThreads, p2m_smem(P, pp), st>>>(fa); break;
    case 3: p2m_kernel<3><<<grid, kP2MThreads, p2m_smem(P, pp), st>>>(fa); break;
    default: p2m_kernel<5><<<grid, kP2MThreads, p2m_smem(P, pp), st>>>(fa); break;
    }
    return CYLFMM_OK;
}

static int s2l_jt(int pl)
{
    if (pl <= 8) return S2LCfg<S2L_P8>::JT;
    if (pl <= 12) return S2LCfg<S2L_P12>::JT;
    return S2LCfg<S2L_P16>::JT;
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------------------------------------
// P2P launcher (direct and near field)
template <int TT, int SC, int MT, bool NEAR, bool GRAD>
static cudaError_t launch_p2p_t(const P2PArgs &a, dim3 grid, cudaStream_t st)
{
    size_t sm = p2p_smem_bytes<TT, SC, GRAD>(a.m1 - a.m0);
    p2p_kernel<TT, SC, MT, NEAR, GRAD><<<grid, TT * SC, sm, st>>>(a);
    return cudaGetLastError();
}

// pick (TT, SC, MAXT) for a target tile size and mode window; grid.x must be set by caller
template <bool NEAR, bool GRAD = false>
static cudaError_t launch_p2p(int TT, const P2PArgs &a, dim3 grid, cudaStream_t st)
{
    int KW = a.m1 - a.m0;
    if (TT == 8) return KW <= 32 ? launch_p2p_t<8, 16, 2, NEAR, GRAD>(a, grid, st)
                                 : launch_p2p_t<8, 16, 5, NEAR, GRAD>(a, grid, st);
    if (TT == 16) return KW <= 24 ? launch_p2p_t<16, 8, 3, NEAR, GRAD>(a, grid, st)
                                  : launch_p2p_t<16, 8, 9, NEAR, GRAD>(a, grid, st);
    return KW <= 24 ? launch_p2p_t<32, 4, 6, NEAR, GRAD>(a, grid, st)
                    : launch_p2p_t<32, 4, 18, NEAR, GRAD>(a, grid, st);
}
static constexpr int kP2PWindow = 72;

// warp-task near field (p2p_warp.cuh): compile-time mode bound KT >= K
static constexpr int kP2PWWindow = 33;   // warp-task kernel: modes per pass for K > 33
static int p2pw_kt(int K)
{
    if (K <= 9) return 9;
    if (K <= 17) return 17;
    return 33;
}
// the warp-task kernel serves every potential solve; the CTA-wide kernel (p2p.cuh) the gradients
static bool p2pw_enabled(int K, bool grad) { return !grad && K <= kP2PWindow * 8; }
// one pass over the mode window [a.m0, a.m1) (m0 > 0 only for K > 33); direct: the direct sum
static cudaError_t launch_p2pw(const P2PArgs &a, cudaStream_t st, bool direct = false)
{
    const int KW = a.m1 - a.m0;
    int kt = p2pw_kt(a.m0 > 0 ? kP2PWWindow : a.K);
    const bool wsm = false;
    const bool win = a.m0 > 0;   // windows after the first (the first runs the exact-33 kernel:
                                 // measured C5 near field 48.2 ms vs 60.0 ms with the windowed one)
    bool exact = !win && KW == kt;
    if (win && a.save == 2 && KW == 32) {   // K = 65 (C5): the second window exactly 32 modes
        kt = 32;
        exact = true;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (win || direct) {       // the previous launch consumed the fetch counter
        cudaError_t err = cudaMemsetAsync(a.task_ctr, 0, sizeof(int), st);
        if (err != cudaSuccess) return err;
    }
    const bool sv = a.save != 0;   // window state saved / restored (K in (33, 66])
#define X(KT, E, W, N, DR, SV)                                                                 \
    if (kt == KT && exact == E && wsm == W && win == N && direct == DR && sv == SV) {          \
        p2p_warp_kernel<KT, E, W, N, DR, SV><<<nsm * p2pw_min_blocks<KT, W>(), 128,            \
                                               p2pw_smem_bytes<KT, W>(), st>>>(a);             \
        return cudaGetLastError();                                                             \
    }
    P2PW_INSTANCES(X)
#undef X
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// direct modal sum
// Direct sum: partition of the sources among the CTAs of one target tile, and the launches.
struct DirectShape {
    bool wk;          // warp-task kernel (p2p_warp.cuh)
    int nparts;       // source partitions per target tile (partial sums reduced afterwards)
    int64_t per;      // sources per partition
    int64_t tiles;    // 32-target tiles
};
static cylfmm_status direct_shape(int64_t n_src, int64_t n_fld, int K, DirectShape *sh)
{
    int dev = 0, nsm = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // warp-task kernel: tasks = (32-target tile, source partition of >= 32: 8 per warp), ~12
    // tasks per resident CTA slot (a lane walks its pairs one after another, so the C1-sized sum
    // is bound by that chain: more, shorter partitions); the CTA-wide kernel serves the mode
    // counts the warp kernel does not
    const bool wk = p2pw_enabled(K, false);
    const int TT = 32, SC = 4;
    int64_t tiles = (n_fld + TT - 1) / TT;
    int64_t want = (int64_t)nsm * (wk ? 12 * 3 : 4);
    int nparts = (int)std::max<int64_t>(1, std::min<int64_t>((want + tiles - 1) / tiles,
                                                             (n_src + (wk ? 31 : 63)) / (wk ? 32 : 64)));
    int64_t per = (n_src + nparts - 1) / nparts;
    per = (per + SC - 1) / SC * SC;
    nparts = (int)((n_src + per - 1) / per);
    *sh = {wk, nparts, per, tiles};
    return CYLFMM_OK;
}
// d_err: DEVICE int[2] (error flag, task counter), zeroed here; ws: DEVICE double2[nparts][n_fld][K]
// when sh.nparts > 1.  Launches only: no allocation, no synchronisation.
static cylfmm_status direct_launch(const DirectShape &sh, const double *src_r, const double *src_z,
                                   const double *src_S, int64_t n_src, const double *fld_r,
                                   const double *fld_z, int64_t n_fld, int K, int miller,
                                   int exclude_coincident, double *out_Phi, int *d_err, double2 *ws,
                                   cudaStream_t st)
{
    CK(cudaMemsetAsync(d_err, 0, 2 * sizeof(int), st));
    const int win = sh.wk ? kP2PWWindow : kP2PWindow;
    for (int m0 = 0; m0 < K; m0 += win) {
        P2PArgs a = {};
        a.sr = src_r;
        a.sz = src_z;
        a.S = reinterpret_cast<const double2 *>(src_S);
        a.fr = fld_r;
        a.fz = fld_z;
        a.ns = n_src;
        a.nf = n_fld;
        a.K = K;
        a.m0 = m0;
        a.m1 = std::min(K, m0 + win);
        a.miller = miller;
        a.fwd2 = forward_coef(K - 1, miller);
        a.exclude = exclude_coincident;
        a.out = sh.nparts > 1 ? ws : reinterpret_cast<double2 *>(out_Phi);
        a.out_row = nullptr;
        a.accumulate = 0;
        a.part_stride = n_fld * K;
        a.src_per_part = sh.per;
        a.err_flag = d_err;
        a.task_ctr = d_err + 1;
        if (sh.wk) CK(launch_p2pw(a, st, true));
        else CK(launch_p2p<false>(32, a, dim3((unsigned)sh.tiles, sh.nparts), st));
    }
    if (sh.nparts > 1) {
        int64_t ne = n_fld * K;
        reduce_parts_kernel<<<nblk(ne, 256), 256, 0, st>>>(ws, ne, sh.nparts,
                                                          reinterpret_cast<double2 *>(out_Phi));
        CKL();
    }
    return CYLFMM_OK;
}
static cylfmm_status direct_check_args(const char *who, const double *src_r, const double *src_z,
                                       const double *src_S, int64_t n_src, const double *fld_r,
                                       const double *fld_z, int64_t n_fld, int n_modes, int miller,
                                       const double *out_Phi)
{
    if (n_src < 0 || n_fld < 0 || n_modes < 1 || n_modes > CYLFMM_MAX_MODES ||
        (miller != 0 && miller != 1) || n_src > INT32_MAX || n_fld > INT32_MAX) {
        set_err("%s: bad sizes (n_src=%lld n_fld=%lld n_modes=%d miller=%d)", who,
                (long long)n_src, (long long)n_fld, n_modes, miller);
        return CYLFMM_EINVAL;
    }
    if ((n_src > 0 && (!src_r || !src_z || !src_S)) || (n_fld > 0 && (!fld_r || !fld_z || !out_Phi))) {
        set_err("%s: null pointer", who);
        return CYLFMM_EINVAL;
    }
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_direct(const double *src_r, const double *src_z,
                                       const double *src_S, int64_t n_src, const double *fld_r,
                                       const double *fld_z, int64_t n_fld, int n_modes,
                                       int miller, int exclude_coincident, double *out_Phi,
                                       cylfmm_stream_t stream)
{
    RET_IF(direct_check_args("cylfmm_direct", src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld,
                             n_modes, miller, out_Phi));
    RET_IF(ensure_init());
    cudaStream_t st = (cudaStream_t)stream;
    if (n_fld == 0) return CYLFMM_OK;
    const int K = n_modes;
    if (n_src == 0) {
        CK(cudaMemsetAsync(out_Phi, 0, sizeof(double) * 2 * K * n_fld, st));
        return CYLFMM_OK;
    }
    DirectShape sh;
    RET_IF(direct_shape(n_src, n_fld, K, &sh));
    int *d_err = nullptr;
    double2 *ws = nullptr;
    // stream-ordered frees on every return path (including CK failures below)
    struct AsyncFree {
        void **q;
        cudaStream_t s;
        ~AsyncFree()
        {
            if (*q) cudaFreeAsync(*q, s);
        }
    } free_err{(void **)&d_err, st}, free_ws{(void **)&ws, st};
    RET_IF(scratch_alloc((void **)&d_err, 2 * sizeof(int), st));
    if (sh.nparts > 1) RET_IF(scratch_alloc((void **)&ws, sizeof(double2) * (size_t)sh.nparts * n_fld * K, st));
    RET_IF(direct_launch(sh, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, K, miller,
                         exclude_coincident, out_Phi, d_err, ws, st));
    int h_err = 0;
    CK(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h_err) {
        set_err("cylfmm_direct: unexcluded coincident source/field pair");
        return CYLFMM_ENUMERIC;
    }
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_direct_workspace_bytes(int64_t n_src, int64_t n_fld, int n_modes,
                                                       int64_t *bytes)
{
    if (!bytes || n_src < 0 || n_fld < 0 || n_modes < 1 || n_modes > CYLFMM_MAX_MODES ||
        n_src > INT32_MAX || n_fld > INT32_MAX) {
        set_err("cylfmm_direct_workspace_bytes: bad arguments");
        return CYLFMM_EINVAL;
    }
    RET_IF(ensure_init());
    *bytes = 16;   // the two flag words, padded
    if (n_src == 0 || n_fld == 0) return CYLFMM_OK;
    DirectShape sh;
    RET_IF(direct_shape(n_src, n_fld, n_modes, &sh));
    if (sh.nparts > 1) *bytes += (int64_t)sizeof(double2) * sh.nparts * n_fld * n_modes;
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_direct_enqueue(const double *src_r, const double *src_z,
                                               const double *src_S, int64_t n_src,
                                               const double *fld_r, const double *fld_z,
                                               int64_t n_fld, int n_modes, int miller,
                                               int exclude_coincident, double *out_Phi,
                                               void *workspace, int64_t workspace_bytes,
                                               cylfmm_stream_t stream)
{
    RET_IF(direct_check_args("cylfmm_direct_enqueue", src_r, src_z, src_S, n_src, fld_r, fld_z,
                             n_fld, n_modes, miller, out_Phi));
    int64_t need = 0;
    RET_IF(cylfmm_direct_workspace_bytes(n_src, n_fld, n_modes, &need));
    if (!workspace || workspace_bytes < need || ((uintptr_t)workspace & 15)) {
        set_err("cylfmm_direct_enqueue: workspace of %lld bytes (16-byte aligned) needed, %lld given",
                (long long)need, (long long)workspace_bytes);
        return CYLFMM_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int *d_err = (int *)workspace;
    const int K = n_modes;
    if (n_fld == 0 || n_src == 0) {
        CK(cudaMemsetAsync(d_err, 0, 2 * sizeof(int), st));
        if (n_fld > 0) CK(cudaMemsetAsync(out_Phi, 0, sizeof(double) * 2 * K * n_fld, st));
        return CYLFMM_OK;
    }
    DirectShape sh;
    RET_IF(direct_shape(n_src, n_fld, K, &sh));
    return direct_launch(sh, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, K, miller,
                         exclude_coincident, out_Phi, d_err,
                         reinterpret_cast<double2 *>((char *)workspace + 16), st);
}

// ------------------------------------------------------------------------------------------
// Green's function and tensor test entry points
extern "C" cylfmm_status cylfmm_greens_batch(const double *r, const double *r1, const double *x,
                                             int64_t n, int n_modes, int miller, double *out_G,
                                             cylfmm_stream_t stream)
{
    if (n < 0 || n_modes < 1 || n_modes > CYLFMM_MAX_MODES || (miller != 0 && miller != 1) ||
        (n > 0 && (!r || !r1 || !x || !out_G))) {
        set_err("cylfmm_greens_batch: bad arguments");
        return CYLFMM_EINVAL;
    }
    RET_IF(ensure_init());
    if (n == 0) return CYLFMM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int *d_err;
    RET_IF(scratch_alloc((void **)&d_err, sizeof(int), st));
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), st));
    greens_batch_kernel<<<nblk(n, 128), 128, 0, st>>>(r, r1, x, n, n_modes, miller,
                                                      forward_coef(n_modes - 1, miller), out_G, d_err);
    CKL();
    int h = 0;
    CK(cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d_err, st));
    CK(cudaStreamSynchronize(st));
    if (h & 2) {
        set_err("cylfmm_greens_batch: r <= 0 or r1 <= 0");
        return CYLFMM_EDOMAIN;
    }
    if (h & 1) {
        set_err("cylfmm_greens_batch: coincident rings");
        return CYLFMM_ENUMERIC;
    }
    return CYLFMM_OK;
}

static cylfmm_status run_seeds(TensorGeomArgs ta, int64_t ngeom, cudaStream_t st)
{
    size_t sm_seed = tensor_seed_smem(ta.K, ta.m1, ta.p);
    // 64 threads: lanes over the 2p + 1 <= 33 series coefficients plus the two table threads
    tensor_seed_kernel<<<(unsigned)ngeom, 64, sm_seed, st>>>(ta);
    CKL();
    return CYLFMM_OK;
}
static cylfmm_status run_fill(TensorGeomArgs ta, int64_t ngeom, cudaStream_t st)
{
    // warp per (station, mode), 4 warps per CTA (tensor.cuh)
    ta.nwork = ngeom * (ta.m1 - ta.m0);
    switch (ta.p) {   // compile-time orders for the BASELINE configurations
    case 8: tensor_fill_kernel<8><<<nblk(ta.nwork, 4), 128, 0, st>>>(ta); break;
    case 12: tensor_fill_kernel<12><<<nblk(ta.nwork, 4), 128, 0, st>>>(ta); break;
    case 16: tensor_fill_kernel<16><<<nblk(ta.nwork, 4), 128, 0, st>>>(ta); break;
    default: tensor_fill_kernel<0><<<nblk(ta.nwork, 4), 128, 0, st>>>(ta); break;
    }
    CKL();
    return CYLFMM_OK;
}
static cylfmm_status run_tensors(TensorGeomArgs ta, int64_t ngeom, cudaStream_t st)
{
    RET_IF(run_seeds(ta, ngeom, st));
    return run_fill(ta, ngeom, st);
}

extern "C" cylfmm_status cylfmm_tensor_batch(const double *r, const double *r1, const double *x,
                                             int64_t n, int n_modes, int p, int miller,
                                             double *out, cylfmm_stream_t stream)
{
    if (n < 0 || n_modes < 1 || n_modes > CYLFMM_MAX_MODES || p < 1 || p > CYLFMM_MAX_ORDER ||
        (miller != 0 && miller != 1) || (n > 0 && (!r || !r1 || !x || !out))) {
        set_err("cylfmm_tensor_batch: bad arguments");
        return CYLFMM_EINVAL;
    }
    RET_IF(ensure_init());
    if (n == 0) return CYLFMM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int Ni = std::max(n_modes - 1, 1), NM = Ni + 1, D = 2 * p + 1;
    double *seeds;
    int *d_err;
    RET_IF(scratch_alloc((void **)&seeds, sizeof(double) * (size_t)n * 4 * NM * D, st));
    RET_IF(scratch_alloc((void **)&d_err, sizeof(int), st));
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), st));
    TensorGeomArgs ta = {};
    ta.r = r;
    ta.r1 = r1;
    ta.x = x;
    ta.n = n;
    ta.K = n_modes;
    ta.m0 = 0;
    ta.m1 = n_modes;
    ta.p = p;
    ta.miller = miller;
    ta.fwd2 = forward_coef(std::max(n_modes - 1, 1), miller);
    ta.seeds = seeds;
    ta.out = out;
    ta.packed = 0;
    ta.err = d_err;
    RET_IF(run_tensors(ta, n, st));
    int h = 0;
    CK(cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(seeds, st));
    CK(cudaFreeAsync(d_err, st));
    CK(cudaStreamSynchronize(st));
    if (h & 2) {
        set_err("cylfmm_tensor_batch: r <= 0 or r1 <= 0");
        return CYLFMM_EDOMAIN;
    }
    if (h & 1) {
        set_err("cylfmm_tensor_batch: coincident geometry");
        return CYLFMM_ENUMERIC;
    }
    return CYLFMM_OK;
}

// ------------------------------------------------------------------------------------------
// plan
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cylfmm_status need(size_t bytes)
    {
        if (bytes <= cap) return CYLFMM_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t b = std::max<size_t>(bytes, 256);
        CK(cudaMalloc(&p, b));
        cap = b;
        return CYLFMM_OK;
    }
    template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Phase timing: CUDA events recorded on the stream each phase runs on (no synchronisation),
// summed when the timings are read (after the solve has completed), plus NVTX ranges.
enum { PH_SORT, PH_LISTS, PH_TENSOR, PH_P2M, PH_M2M, PH_S2L, PH_L2L, PH_L2P, PH_P2P, PH_TOTAL, PH_ALLGATHER, PH_SEEDS, PH_N };
static const char *kPhaseName[PH_N] = {"cylfmm.sort", "cylfmm.lists", "cylfmm.tensor", "cylfmm.p2m",
                                       "cylfmm.m2m", "cylfmm.s2l", "cylfmm.l2l", "cylfmm.l2p",
                                       "cylfmm.near", "cylfmm.solve", "cylfmm.allgather",
                                       "cylfmm.tensor_seeds"};
struct PhaseMark {
    int ph;
    cudaEvent_t a, b;
};
struct Phases {
    cylfmm_plan p;
    bool on;
    int open[PH_N];
    void beg(int ph, cudaStream_t s);
    void end(int ph, cudaStream_t s);
};

// mailbox layout (ints): [0, 3 kMaxLevels + 8) level counts, [kMboxErr] error flag,
// [kMboxSlots, +2) the near-field window-slot count (int64)
constexpr int kMboxErr = 3 * kMaxLevels + 8, kMboxSlots = kMboxErr + 2, kMboxInts = kMboxSlots + 2;
__global__ void mailbox_kernel(const int *counts, int nc, const int *err, const int64_t *slots,
                               volatile int *out)
{
    for (int i = threadIdx.x; i < nc; i += blockDim.x) out[i] = counts[i];
    if (threadIdx.x == 0) {
        out[kMboxErr] = *err;
        if (slots) *reinterpret_cast<volatile int64_t *>(out + kMboxSlots) = *slots;
    }
}

struct cylfmm_plan_s {
    cylfmm_params prm;
    int device = 0;
    int nsm = 148;
    // tree buffers
    DevBuf skey, sidx, skey2, sidx2, fkey, fidx, fkey2, fidx2, hist, scan_tmp[4], scan_tmp_n[4];
    DevBuf sr_s, sz_s, S_s, fr_s, fz_s;
    DevBuf slstart, flstart, flags, smap, skeys, tmap, tkeys, counts;
    DevBuf M, Lc, tens, seeds;
    DevBuf tasks, ntasks, tcnt, toff;
    DevBuf written;                       // per-box 'local written by S2L' flags
    DevBuf pcnt, poff, khist, kstart, kcur, bstart, pairs, batches, wlist, pairbuf;   // S2L lists
    DevBuf need, lrow, rowkey;            // lazy L2L flags, compact local rows, row -> box
    DevBuf pbase, pcnt64, sv2, sv1;       // near-field window state (K in (33, 66])
    DevBuf stflag, stlist;                // stations with an S2L pair
    DevBuf l2pown, l2pflag, l2ppos, l2ptask, l2pntask;   // L2P evaluating boxes and tasks
    DevBuf err, ctr;
    DevBuf rtab;     // M2M / L2L recentring tables: [rtab(p) | rtab(pl)] doubles, then tri ints
    size_t rtab_nm = 0, rtab_nd = 0, rtab_ntm = 0;
    // host-API staging
    DevBuf h_sr, h_sz, h_S, h_fr, h_fz, h_out;
    cudaEvent_t ev[16] = {};
    bool ev_ok = false;
    int64_t launches = 0;
    int auto_kw = 0;   // last automatic mode chunk
    // concurrency: the data-independent tensors and the near field run on their own streams,
    // joined to the caller's stream by events (aev: start, tree, tensors, near, s2l)
    cudaStream_t aux[2] = {nullptr, nullptr};
    cudaEvent_t aev[5] = {};
    bool aux_ok = false;
    // host-buffer solves: the coefficient rows are copied on their own stream behind the tree
    // build (hev: previous work on the caller's stream done, coefficients resident)
    cudaStream_t hcp = nullptr;
    cudaEvent_t hev[2] = {};
    // pipelined host-buffer solves (cylfmm_fmm_solve_host_async): two device staging slots used
    // alternately; uploads on hcp, downloads on hdn; per slot: coordinates / coefficients
    // resident, solve done (inputs free, result ready), download done (result buffer free)
    struct HostSlot {
        DevBuf sr, sz, S, fr, fz, out;
        cudaEvent_t coords = nullptr, coef = nullptr, done = nullptr, down = nullptr;
    } hs[2];
    int hslot = 0;
    cudaStream_t hdn = nullptr;
    // mapped pinned mailbox: the mid-solve counts the host needs, written by mailbox_kernel
    int *mbox = nullptr, *mbox_dev = nullptr;
    // phase events (Phases): pool reused across solves, marks of the solves since the last read
    std::vector<cudaEvent_t> evpool;
    size_t evused = 0;
    std::vector<PhaseMark> marks;
    int prof_solves = 0;
    bool prof_on = false;
    int64_t last_npairs = 0, last_launches = 0;
    // geometry cache (cylfmm_plan_set_geometry_cache): the coordinate-only results of the last
    // solve (sorted orders, lists, tensors, task lists live in the plan's buffers)
    bool geo_cache = false;
    struct {
        bool valid = false, grad = false;
        const double *sr = nullptr, *sz = nullptr, *fr = nullptr, *fz = nullptr;
        int64_t ns = 0, nf = 0, nslots = 0;
        int *sperm = nullptr, *fperm = nullptr;
        uint32_t *skey_s = nullptr, *fkey_s = nullptr;
        int hcnt[3 * kMaxLevels + 8];
    } geo;
    // multi-device (cylfmm_plan_create_dist): the library-owned NCCL communicator
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    DevBuf g_r, g_z, g_S, g_cnt;          // gathered sources, shard counts
};

static cudaEvent_t pool_event(cylfmm_plan p)
{
    if (p->evused == p->evpool.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        p->evpool.push_back(e);
    }
    return p->evpool[p->evused++];
}
void Phases::beg(int ph, cudaStream_t s)
{
    nvtxRangePushA(kPhaseName[ph]);
    if (!on) return;
    PhaseMark m = {ph, pool_event(p), nullptr};
    if (m.a) cudaEventRecord(m.a, s);
    open[ph] = (int)p->marks.size();
    p->marks.push_back(m);
}
void Phases::end(int ph, cudaStream_t s)
{
    nvtxRangePop();
    if (!on) return;
    PhaseMark &m = p->marks[open[ph]];
    m.b = pool_event(p);
    if (m.b) cudaEventRecord(m.b, s);
}
// sum the phase marks of the solves since the last read into t (averaged per solve), then reset
static cylfmm_status read_phases(cylfmm_plan p, cylfmm_timings *t)
{
    double acc[PH_N] = {0};
    for (const PhaseMark &m : p->marks) {
        if (!m.a || !m.b) continue;
        CK(cudaEventSynchronize(m.b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, m.a, m.b));
        acc[m.ph] += ms;
    }
    const double n = std::max(p->prof_solves, 1);
    t->ms_sort = acc[PH_SORT] / n;
    t->ms_lists = acc[PH_LISTS] / n;
    t->ms_tree = t->ms_sort + t->ms_lists;
    t->ms_tensor = (acc[PH_TENSOR] + acc[PH_SEEDS]) / n;
    t->ms_seeds = acc[PH_SEEDS] / n;
    t->ms_p2m = acc[PH_P2M] / n;
    t->ms_m2m = acc[PH_M2M] / n;
    t->ms_s2l = acc[PH_S2L] / n;
    t->ms_l2l = acc[PH_L2L] / n;
    t->ms_l2p = acc[PH_L2P] / n;
    t->ms_p2p = acc[PH_P2P] / n;
    t->ms_total = acc[PH_TOTAL] / n;
    t->ms_unpermute = 0.0;   // fused into the L2P / near-field row writes (a13)
    t->ms_allgather = acc[PH_ALLGATHER] / n;
    t->n_solves = p->prof_solves;
    p->marks.clear();
    p->evused = 0;
    p->prof_solves = 0;
    return CYLFMM_OK;
}

static void free_plan_bufs(cylfmm_plan p)
{
    DevBuf *all[] = {&p->skey, &p->sidx, &p->skey2, &p->sidx2, &p->fkey, &p->fidx, &p->fkey2,
                     &p->fidx2, &p->hist, &p->scan_tmp[0], &p->scan_tmp[1], &p->scan_tmp[2],
                     &p->scan_tmp[3], &p->scan_tmp_n[0], &p->scan_tmp_n[1], &p->scan_tmp_n[2],
                     &p->scan_tmp_n[3], &p->sr_s, &p->sz_s, &p->S_s, &p->fr_s, &p->fz_s,
                     &p->slstart, &p->flstart, &p->flags, &p->smap, &p->skeys, &p->tmap,
                     &p->tkeys, &p->counts, &p->M, &p->Lc, &p->tens, &p->seeds, &p->tasks,
                     &p->ntasks, &p->tcnt, &p->toff, &p->written, &p->pcnt, &p->poff, &p->khist, &p->kstart, &p->kcur, &p->bstart, &p->pairs, &p->batches, &p->wlist, &p->pairbuf, &p->need, &p->lrow, &p->rowkey, &p->pbase, &p->pcnt64, &p->sv2, &p->sv1, &p->stflag, &p->stlist, &p->l2pown, &p->l2pflag, &p->l2ppos, &p->l2ptask, &p->l2pntask, &p->err, &p->ctr, &p->rtab, &p->h_sr, &p->h_sz,
                     &p->h_S, &p->h_fr, &p->h_fz, &p->h_out, &p->g_r, &p->g_z, &p->g_S, &p->g_cnt};
    for (DevBuf *b : all) b->release();
}

static cylfmm_status plan_init(cylfmm_plan p, const cylfmm_params &q);

extern "C" cylfmm_status cylfmm_plan_create(cylfmm_plan *plan, const cylfmm_params *prm)
{
    if (!plan || !prm) {
        set_err("cylfmm_plan_create: null pointer");
        return CYLFMM_EINVAL;
    }
    *plan = nullptr;
    const cylfmm_params &q = *prm;
    if (q.n_modes < 1 || q.n_modes > CYLFMM_MAX_MODES || q.order < 1 || q.order > CYLFMM_MAX_ORDER ||
        q.order_local < 0 || q.order_local > CYLFMM_MAX_ORDER ||
        q.depth < 2 || q.depth > CYLFMM_MAX_DEPTH || (q.truncation != 0 && q.truncation != 1) ||
        (q.miller != 0 && q.miller != 1) || !(q.domain_L > 0.0) || !(q.domain_z0 == q.domain_z0) ||
        q.mode_chunk < 0 || q.adaptive_leaf < 0 || (q.adaptive_leaf > 0 && q.n_modes > kP2PWWindow)) {
        set_err("cylfmm_plan_create: bad parameters (K=%d p=%d d=%d trunc=%d miller=%d L=%g)",
                q.n_modes, q.order, q.depth, q.truncation, q.miller, q.domain_L);
        return CYLFMM_EINVAL;
    }
    RET_IF(ensure_init());
    cylfmm_plan p = new cylfmm_plan_s;
    const cylfmm_status st = plan_init(p, q);
    if (st != CYLFMM_OK) {
        cylfmm_plan_destroy(p);   // releases whatever was created before the failure
        return st;
    }
    *plan = p;
    return CYLFMM_OK;
}

static cylfmm_status plan_init(cylfmm_plan p, const cylfmm_params &q)
{
    p->prm = q;
    CK(cudaGetDevice(&p->device));
    CK(cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, p->device));
    for (int i = 0; i < 16; ++i) CK(cudaEventCreate(&p->ev[i]));
    p->ev_ok = true;
    for (int i = 0; i < 2; ++i) CK(cudaStreamCreateWithFlags(&p->aux[i], cudaStreamNonBlocking));
    for (int i = 0; i < 5; ++i) CK(cudaEventCreateWithFlags(&p->aev[i], cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&p->hcp, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&p->hev[i], cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&p->hdn, cudaStreamNonBlocking));
    CK(cudaHostAlloc(reinterpret_cast<void **>(&p->mbox), sizeof(int) * kMboxInts, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&p->mbox_dev), p->mbox, 0));
    for (auto &h : p->hs)
        for (cudaEvent_t *e : {&h.coords, &h.coef, &h.done, &h.down})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    p->aux_ok = true;
    {
        const int pl = q.order_local > 0 ? q.order_local : q.order;
        // recentring tables for the source order (M2M) and the local order (L2L), once per plan
        std::vector<double> rm, rl;
        std::vector<int> tm_, tl_;
        recentre_tables_host(q.order, rm, tm_);
        recentre_tables_host(pl, rl, tl_);
        // S2L moment prescale (-1)^j / j! per source coefficient (i, j) (fmm_ops.cuh)
        const int Pm = (q.order + 1) * (q.order + 2) / 2;
        for (int qq = 0; qq < Pm; ++qq) {
            const int j = tm_[Pm + qq];
            double f = 1.0;
            for (int t = 2; t <= j; ++t) f *= t;
            rl.push_back(((j & 1) ? -1.0 : 1.0) / f);
        }
        const size_t nd = rm.size() + rl.size(), ni = tm_.size() + tl_.size();
        RET_IF(p->rtab.need(sizeof(double) * nd + sizeof(int) * ni));
        std::vector<char> blob(sizeof(double) * nd + sizeof(int) * ni);
        memcpy(blob.data(), rm.data(), sizeof(double) * rm.size());
        memcpy(blob.data() + sizeof(double) * rm.size(), rl.data(), sizeof(double) * rl.size());
        memcpy(blob.data() + sizeof(double) * nd, tm_.data(), sizeof(int) * tm_.size());
        memcpy(blob.data() + sizeof(double) * nd + sizeof(int) * tm_.size(), tl_.data(), sizeof(int) * tl_.size());
        CK(cudaMemcpy(p->rtab.p, blob.data(), blob.size(), cudaMemcpyHostToDevice));
        p->rtab_nm = rm.size();
        p->rtab_nd = nd;
        p->rtab_ntm = tm_.size();
    }
    return CYLFMM_OK;
}

extern "C" void cylfmm_plan_destroy(cylfmm_plan plan)
{
    if (!plan) return;
    cudaDeviceSynchronize();
    free_plan_bufs(plan);
    // every handle is null until created, so a partly built plan is released too
    for (cudaEvent_t e : plan->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : plan->evpool) cudaEventDestroy(e);
    for (cudaStream_t x : plan->aux)
        if (x) cudaStreamDestroy(x);
    for (cudaEvent_t e : plan->aev)
        if (e) cudaEventDestroy(e);
    if (plan->hcp) cudaStreamDestroy(plan->hcp);
    if (plan->comm && g_nccl.ok) g_nccl.CommDestroy(plan->comm);
    for (cudaEvent_t e : plan->hev)
        if (e) cudaEventDestroy(e);
    if (plan->hdn) cudaStreamDestroy(plan->hdn);
    if (plan->mbox) cudaFreeHost(plan->mbox);
    for (auto &h : plan->hs) {
        for (cudaEvent_t e : {h.coords, h.coef, h.done, h.down})
            if (e) cudaEventDestroy(e);
        for (DevBuf *b : {&h.sr, &h.sz, &h.S, &h.fr, &h.fz, &h.out}) b->release();
    }
    delete plan;
}

static cylfmm_status err_status(int h)
{
    if (h & 4) {
        set_err("cylfmm: point outside the domain [0,L]x[z0,z0+L] or r <= 0 / non-finite");
        return CYLFMM_EDOMAIN;
    }
    if (h & 3) {
        set_err("cylfmm: unexcluded coincident pair or degenerate geometry");
        return CYLFMM_ENUMERIC;
    }
    return CYLFMM_OK;
}
// the plan's error flag after the work queued on `st` (through the mapped mailbox: no copy
// engine, see mailbox_kernel)
static cylfmm_status check_err_flag(cylfmm_plan p, cudaStream_t st)
{
    if (!p->mbox) {   // a scratch plan without a mailbox (cylfmm_tree_sort)
        int h = 0;
        CK(cudaMemcpyAsync(&h, p->err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return err_status(h);
    }
    mailbox_kernel<<<1, 32, 0, st>>>(nullptr, 0, p->err.as<int>(), nullptr, p->mbox_dev);
    CKL();
    CK(cudaStreamSynchronize(st));
    return err_status(p->mbox[kMboxErr]);
}

extern "C" cylfmm_status cylfmm_plan_set_profiling(cylfmm_plan plan, int on)
{
    if (!plan) {
        set_err("cylfmm_plan_set_profiling: null plan");
        return CYLFMM_EINVAL;
    }
    plan->prof_on = on != 0;
    plan->marks.clear();
    plan->evused = 0;
    plan->prof_solves = 0;
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_plan_set_geometry_cache(cylfmm_plan plan, int on)
{
    if (!plan) {
        set_err("cylfmm_plan_set_geometry_cache: null plan");
        return CYLFMM_EINVAL;
    }
    plan->geo_cache = on != 0;
    plan->geo.valid = false;   // the next solve builds (and remembers) its geometry
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_plan_read_timings(cylfmm_plan plan, cylfmm_timings *t)
{
    if (!plan || !t) {
        set_err("cylfmm_plan_read_timings: null argument");
        return CYLFMM_EINVAL;
    }
    *t = cylfmm_timings{};
    t->n_s2l_pairs = plan->last_npairs;
    t->kernel_launches = plan->last_launches;
    return read_phases(plan, t);
}

extern "C" cylfmm_status cylfmm_plan_sync(cylfmm_plan plan)
{
    if (!plan) {
        set_err("cylfmm_plan_sync: null plan");
        return CYLFMM_EINVAL;
    }
    CK(cudaDeviceSynchronize());
    if (plan->err.p) return check_err_flag(plan, nullptr);
    return CYLFMM_OK;
}

// exclusive scan in place on d (n ints or int64s), scratch from plan->scan_tmp[depth] (set 0,
// the caller's stream) or plan->scan_tmp_n[depth] (set 1, the near-field stream)
template <typename T>
static cylfmm_status scan_excl(cylfmm_plan p, T *d, int64_t n, cudaStream_t st, int lvl = 0,
                               int set = 0)
{
    if (n <= 0) return CYLFMM_OK;
    int64_t nt = (n + kScanTile - 1) / kScanTile;
    if (lvl >= 4) {
        set_err("scan: too deep");
        return CYLFMM_EINVAL;
    }
    DevBuf &tmp = set ? p->scan_tmp_n[lvl] : p->scan_tmp[lvl];
    RET_IF(tmp.need(sizeof(T) * (size_t)std::max<int64_t>(nt, 1)));
    T *sums = tmp.as<T>();
    scan_tile_kernel<T><<<(unsigned)nt, kScanThreads, 0, st>>>(d, n, d, sums);
    CKL();
    p->launches++;
    if (nt > 1) {
        RET_IF(scan_excl(p, sums, nt, st, lvl + 1, set));
        scan_add_kernel<T><<<nblk(n, 256), 256, 0, st>>>(d, n, sums);
        CKL();
        p->launches++;
    }
    return CYLFMM_OK;
}

// stable radix sort of (key, idx) by the low `bits` bits; returns buffers holding the result
static cylfmm_status radix_sort(cylfmm_plan p, DevBuf &k1, DevBuf &v1, DevBuf &k2, DevBuf &v2,
                                int64_t n, int bits, cudaStream_t st, uint32_t **ko, int **vo)
{
    const int items = sort_items(n), tile = kSortThreads * items;
    int ntiles = (int)((n + tile - 1) / tile);
    if (n <= 0) {
        *ko = k1.as<uint32_t>();
        *vo = v1.as<int>();
        return CYLFMM_OK;
    }
    RET_IF(p->hist.need(sizeof(int) * 256 * (size_t)std::max(ntiles, 1)));
    uint32_t *ka = k1.as<uint32_t>(), *kb = k2.as<uint32_t>();
    int *va = v1.as<int>(), *vb = v2.as<int>();
    for (int sh = 0; sh < bits; sh += 8) {
        radix_hist_kernel<<<ntiles, kSortThreads, 0, st>>>(ka, n, sh, ntiles, p->hist.as<int>(), items);
        CKL();
        RET_IF(scan_excl(p, p->hist.as<int>(), 256LL * ntiles, st));
        radix_scatter_kernel<<<ntiles, kSortThreads, 0, st>>>(ka, va, n, sh, ntiles,
                                                              p->hist.as<int>(), kb, vb, items);
        CKL();
        p->launches += 2;
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    *ko = ka;
    *vo = va;
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_tree_sort(const double *r, const double *z, int64_t n, int depth,
                                          double L, double z0, uint32_t *key, int32_t *perm,
                                          cylfmm_stream_t stream)
{
    if (n < 0 || n > INT32_MAX || depth < 1 || depth > CYLFMM_MAX_DEPTH || !(L > 0.0) ||
        (n > 0 && (!r || !z || !key || !perm))) {
        set_err("cylfmm_tree_sort: bad arguments");
        return CYLFMM_EINVAL;
    }
    RET_IF(ensure_init());
    if (n == 0) return CYLFMM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cylfmm_plan_s tmp;
    DevBuf k1, v1, k2, v2;
    cylfmm_status s = CYLFMM_OK;
    do {
        if ((s = k1.need(4 * n)) || (s = v1.need(4 * n)) || (s = k2.need(4 * n)) ||
            (s = v2.need(4 * n)) || (s = tmp.err.need(4)))
            break;
        cudaMemsetAsync(tmp.err.p, 0, 4, st);
        keys_kernel<<<nblk(n, 256), 256, 0, st>>>(r, z, n, depth, L, z0, k1.as<uint32_t>(),
                                                  v1.as<int>(), tmp.err.as<int>());
        cudaMemcpyAsync(key, k1.p, 4 * n, cudaMemcpyDeviceToDevice, st);
        uint32_t *ko;
        int *vo;
        if ((s = radix_sort(&tmp, k1, v1, k2, v2, n, 2 * depth, st, &ko, &vo))) break;
        cudaMemcpyAsync(perm, vo, 4 * n, cudaMemcpyDeviceToDevice, st);
        s = check_err_flag(&tmp, st);
    } while (0);
    cudaStreamSynchronize(st);
    k1.release();
    v1.release();
    k2.release();
    v2.release();
    free_plan_bufs(&tmp);
    return s;
}

// ------------------------------------------------------------------------------------------
// FMM solve
static int64_t pow4(int l) { return (int64_t)1 << (2 * l); }

template <int R, int C, int NU, int CG, int U = 1>
static cudaError_t launch_s2l_t(const S2LArgs &sa, int64_t nbatches, cudaStream_t st)
{
    const int KW = sa.m1 - sa.m0;
    if (nbatches == 0) return cudaSuccess;
    size_t sm = s2l_smem_bytes<R, C, NU, CG>(sa.p, sa.pl);
    if (U > 1)
        s2l_batch_units_kernel<R, C, NU, CG, U><<<(unsigned)(nbatches * KW), ((NU + U - 1) / U) * CG, sm, st>>>(sa);
    else
        s2l_batch_kernel<R, C, NU, CG><<<(unsigned)(nbatches * KW), NU * CG, sm, st>>>(sa);
    return cudaGetLastError();
}
// class by the local order (units(pl, R) <= NU)
// p > 12 with well-filled batches (>= 90% of the JT pair slots, C4's clusters): two units per
// thread (C4 S2L 37.3 -> 35.9 ms).  Sparse stations (C5: 8.5 pairs per batch of 12, a third of
// the column groups idle) keep one unit per thread, whose CTAs hold twice the warps (C5 S2L 36.0
// vs 37.7 ms with two).  The p <= 12 shape with two units (144 threads, 136 registers): C3 S2L
// 34.0 vs 20.9 ms, not kept.
static cudaError_t launch_s2l(const S2LArgs &sa, int64_t nbatches, int64_t npairs, cudaStream_t st)
{
    if (sa.pl <= 8) return launch_s2l_t<S2L_P8>(sa, nbatches, st);
    if (sa.pl <= 12) return launch_s2l_t<S2L_P12>(sa, nbatches, st);
    if (10 * npairs >= 9 * nbatches * S2LCfg<S2L_P16>::JT) return launch_s2l_t<S2L_P16, 2>(sa, nbatches, st);
    return launch_s2l_t<S2L_P16>(sa, nbatches, st);
}

static cylfmm_status build_tree(cylfmm_plan p, const double *r, const double *z, int64_t n,
                                bool is_src, cudaStream_t st, int **perm_out, uint32_t **key_out)
{
    const cylfmm_params &q = p->prm;
    DevBuf &k1 = is_src ? p->skey : p->fkey, &v1 = is_src ? p->sidx : p->fidx;
    DevBuf &k2 = is_src ? p->skey2 : p->fkey2, &v2 = is_src ? p->sidx2 : p->fidx2;
    size_t nb = sizeof(int) * (size_t)std::max<int64_t>(n, 1);
    RET_IF(k1.need(nb));
    RET_IF(v1.need(nb));
    RET_IF(k2.need(nb));
    RET_IF(v2.need(nb));
    if (n > 0) {
        keys_kernel<<<nblk(n, 256), 256, 0, st>>>(r, z, n, q.depth, q.domain_L, q.domain_z0,
                                                  k1.as<uint32_t>(), v1.as<int>(), p->err.as<int>());
        CKL();
        p->launches++;
    }
    RET_IF(radix_sort(p, k1, v1, k2, v2, n, 2 * q.depth, st, key_out, perm_out));
    return CYLFMM_OK;
}

static cylfmm_status fmm_solve_impl(cylfmm_plan p, const double *src_r, const double *src_z,
                                    const double *src_S, int64_t ns, const double *fld_r,
                                    const double *fld_z, int64_t nf, double *out_Phi,
                                    cudaStream_t st, cylfmm_timings *tm,
                                    double *out_dr = nullptr, double *out_dz = nullptr,
                                    cudaEvent_t s_ready = nullptr, bool dist = false)
{
    const bool grad = out_dr != nullptr && out_dz != nullptr;
    // multi-device solve: the leaf moments are split across the ranks (P2M of a contiguous
    // range of source leaves each) and replicated by NCCL broadcasts (one per rank, grouped)
    // (the adaptive source tree computes its leaf moments on every rank)
    const bool split = dist && p->comm && p->nranks > 1 && p->prm.adaptive_leaf == 0;
    const cylfmm_params &q = p->prm;
    const int d = q.depth, K = q.n_modes, pp = q.order, P = (pp + 1) * (pp + 2) / 2;
    // local order (0 = the source order) and the tensor order max(p, pl)
    const int pl = q.order_local > 0 ? q.order_local : pp, Pl = (pl + 1) * (pl + 2) / 2;
    const int pt = std::max(pp, pl);
    int KW = q.mode_chunk > 0 ? std::min(q.mode_chunk, K) : K;
    p->launches = 0;
    // phase events: always in the synchronised timings path, on request (plan profiling) else
    if (tm && !dist) {
        p->marks.clear();
        p->evused = 0;
        p->prof_solves = 0;
    }
    if (tm && dist) p->prof_solves = 0;
    Phases T{p, tm != nullptr || p->prof_on, {}};
    if (T.on) p->prof_solves++;
    RET_IF(p->err.need(sizeof(int)));
    RET_IF(p->ctr.need(sizeof(unsigned long long) * 8));
    CK(cudaMemsetAsync(p->err.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(p->ctr.p, 0, sizeof(unsigned long long) * 8, st));
    T.beg(PH_TOTAL, st);
    if (nf == 0) {
        T.end(PH_TOTAL, st);
        return CYLFMM_OK;
    }
    // Streams: the timings path runs every phase on `st` (clean per-phase events).  Small
    // problems (launch-latency bound: C2, C3) run the tensors (independent of the data:
    // normalised stations) and the near field (independent of the far field) on the plan's
    // auxiliary streams, joined by events; large ones (C4, C5) keep every kernel on `st`, where
    // each already fills the GPU (measured: C5 162.6 ms overlapped vs 163.0 ms serialised) and
    // the per-phase events stay clean.
    // (the adaptive tree's near field runs one accumulating launch per level: serial)
    const bool overlap = tm == nullptr && p->aux_ok && ns + nf <= ((int64_t)1 << 20) && q.adaptive_leaf == 0;
    cudaStream_t st_t = overlap ? p->aux[0] : st, st_n = overlap ? p->aux[1] : st;
    // large solves: the tensor seeds alone on the auxiliary stream, overlapping P2M / M2M.  The
    // seed kernel's duration is set by its few longest Miller stations (a sequential series
    // recursion of up to ~10^3 steps in one thread; C5: 3.3 ms with most SMs idle at the end);
    // the fill follows behind M2M on `st`, joined by an event.
    const bool seeds_aside = !overlap && tm == nullptr && p->aux_ok;
    cudaStream_t st_s = (overlap || seeds_aside) ? p->aux[0] : st;
    const int64_t nstat = (int64_t)12 << d;
    const int NM = std::max(K - 1, 1) + 1, D = 2 * pt + 1;
    RET_IF(p->seeds.need(sizeof(double) * (size_t)nstat * 4 * NM * D));
    TensorGeomArgs ta = {};
    ta.station_mode = 1;
    ta.n = nstat;
    ta.K = K;
    ta.m0 = 0;
    ta.m1 = K;
    ta.p = pt;
    ta.miller = q.miller;
    ta.fwd2 = forward_coef(std::max(K - 1, 1), q.miller);
    ta.seeds = p->seeds.as<double>();
    ta.packed = 1;
    ta.err = p->err.as<int>();
    // ---- tree and lists (geometry).  With the plan's geometry cache on and the same coordinate
    // arrays as the previous solve (the caller guarantees unchanged coordinates), everything
    // below that depends only on the coordinates is reused: no sort, no lists, no tensors and no
    // host synchronisation, so the solve can be captured into a CUDA graph.
    const bool same = fld_r == src_r && fld_z == src_z && nf == ns;
    const bool reuse = p->geo_cache && p->geo.valid && p->geo.sr == src_r && p->geo.sz == src_z &&
                       p->geo.fr == fld_r && p->geo.fz == fld_z && p->geo.ns == ns &&
                       p->geo.nf == nf && p->geo.grad == grad && !dist;
    int *sperm = reuse ? p->geo.sperm : nullptr, *fperm = reuse ? p->geo.fperm : nullptr;
    uint32_t *skey_s = reuse ? p->geo.skey_s : nullptr, *fkey_s = reuse ? p->geo.fkey_s : nullptr;
    const int64_t nleaf = pow4(d);
    int64_t lvoff[kMaxLevels + 1];
    lvoff[0] = lvoff[1] = lvoff[2] = 0;
    for (int l = 2; l <= d; ++l) lvoff[l + 1] = lvoff[l] + pow4(l);
    const int64_t ltot = lvoff[d + 1];
    // buffer pointers: set after the buffers are sized (geometry pass) or taken as they are (reuse)
    const int *flstart = nullptr;
    int *tmap_b = nullptr, *tkeys_b = nullptr;
    // fields == sources: one sort and one set of leaf ranges; the level maps are shared too
    // unless the source tree is adaptive (its maps omit the boxes below source leaves)
    const int sigma = q.adaptive_leaf;
    const bool share = same && sigma == 0;
    auto set_ptrs = [&]() {
        flstart = same ? p->slstart.as<int>() : p->flstart.as<int>();
        tmap_b = share ? p->smap.as<int>() : p->tmap.as<int>();
        tkeys_b = share ? p->skeys.as<int>() : p->tkeys.as<int>();
    };
    if (reuse) set_ptrs();
    const int nkeys = 2 * 12 * (1 << d), JT = s2l_jt(pl);
    const bool wsave = ns > 0 && !grad && K > kP2PWWindow && K <= 2 * kP2PWWindow &&
                       p2pw_enabled(K, grad);
    int64_t nslots = reuse ? p->geo.nslots : 0;
    int hcnt[3 * kMaxLevels + 8] = {0};
    if (reuse) memcpy(hcnt, p->geo.hcnt, sizeof hcnt);
    S2LListArgs la = {};
    int *cnt_ex = nullptr;
    T.beg(PH_SORT, st);
    if (!reuse) {
    // fields == sources (C2-C4: "field points equal to source points"): one tree serves both
    RET_IF(build_tree(p, src_r, src_z, ns, true, st, &sperm, &skey_s));
    if (same) {
        fperm = sperm;
        fkey_s = skey_s;
    } else {
        RET_IF(build_tree(p, fld_r, fld_z, nf, false, st, &fperm, &fkey_s));
    }
    RET_IF(p->sr_s.need(8 * std::max<int64_t>(ns, 1)));
    RET_IF(p->sz_s.need(8 * std::max<int64_t>(ns, 1)));
    RET_IF(p->S_s.need(16 * (size_t)std::max<int64_t>(ns, 1) * K));
    RET_IF(p->fr_s.need(8 * nf));
    RET_IF(p->fz_s.need(8 * nf));
    if (!same) {
        gather_points_kernel<<<nblk(nf, 256), 256, 0, st>>>(fld_r, fld_z, nullptr, fperm, nf, 0,
                                                            p->fr_s.as<double>(), p->fz_s.as<double>(),
                                                            nullptr);
        CKL();
        p->launches++;
    }
    T.end(PH_SORT, st);
    T.beg(PH_LISTS, st);
    RET_IF(p->slstart.need(sizeof(int) * (nleaf + 1)));
    RET_IF(p->flstart.need(sizeof(int) * (nleaf + 1)));
    leaf_start_kernel<<<nblk(nleaf + 1, 256), 256, 0, st>>>(skey_s, ns, nleaf, p->slstart.as<int>());
    CKL();
    p->launches++;
    if (!same) {
        leaf_start_kernel<<<nblk(nleaf + 1, 256), 256, 0, st>>>(fkey_s, nf, nleaf, p->flstart.as<int>());
        CKL();
        p->launches++;
    }
    // level maps
    RET_IF(p->flags.need(sizeof(int) * ltot));
    RET_IF(p->smap.need(sizeof(int) * ltot));
    RET_IF(p->skeys.need(sizeof(int) * ltot));
    RET_IF(p->tmap.need(sizeof(int) * ltot));
    RET_IF(p->tkeys.need(sizeof(int) * ltot));
    RET_IF(p->counts.need(sizeof(int) * (3 * kMaxLevels + 8)));
    set_ptrs();
    const int nside = share ? 1 : 2;
    int lsmall = 1;   // levels 2..lsmall in one launch (4^l <= kSmallLevelBoxes)
    while (lsmall + 1 <= d && pow4(lsmall + 1) <= kSmallLevelBoxes) ++lsmall;
    if (lsmall >= 2) {
        SmallLevelArgs sa = {};
        for (int side = 0; side < nside; ++side) {
            sa.ls[side] = side == 0 ? p->slstart.as<int>() : flstart;
            sa.map[side] = side == 0 ? p->smap.as<int>() : p->tmap.as<int>();
            sa.keys[side] = side == 0 ? p->skeys.as<int>() : p->tkeys.as<int>();
            sa.count[side] = p->counts.as<int>() + side * kMaxLevels;
            sa.sigma[side] = side == 0 ? sigma : 0;
        }
        for (int l = 0; l <= d + 1 && l < 17; ++l) sa.lvoff[l] = lvoff[l];
        sa.depth = d;
        sa.lmin = 2;
        sa.nlev = lsmall - 1;
        level_maps_small_kernel<<<nside * sa.nlev, 1024, 0, st>>>(sa);
        CKL();
        p->launches++;
    }
    for (int side = 0; side < nside; ++side) {
        const int *ls = side == 0 ? p->slstart.as<int>() : flstart;
        int *map = side == 0 ? p->smap.as<int>() : p->tmap.as<int>();
        int *keys = side == 0 ? p->skeys.as<int>() : p->tkeys.as<int>();
        for (int l = lsmall + 1; l <= d; ++l) {
            int *fl = p->flags.as<int>() + lvoff[l];
            const int sg = side == 0 ? sigma : 0;
            level_flags_kernel<<<nblk(pow4(l), 256), 256, 0, st>>>(ls, d, l, sg, fl);
            CKL();
            RET_IF(scan_excl(p, fl, pow4(l), st));
            level_map_kernel<<<nblk(pow4(l), 256), 256, 0, st>>>(
                ls, d, l, sg, fl, map + lvoff[l], keys + lvoff[l], p->counts.as<int>() + side * kMaxLevels + l);
            CKL();
            p->launches += 2;
        }
    }
    // S2L interaction lists (s2l.cuh): every (target box, source box) pair of every level,
    // counted per target (dense index) and per station key; the per-box "written by S2L" flags
    // that L2L / L2P use instead of zero-initialised locals
    RET_IF(p->written.need(std::max<int64_t>(ltot, 1)));
    RET_IF(p->pcnt.need(sizeof(int) * std::max<int64_t>(ltot, 1)));
    RET_IF(p->poff.need(sizeof(int) * std::max<int64_t>(ltot, 1)));
    RET_IF(p->wlist.need(sizeof(int) * std::max<int64_t>(ltot, 1)));
    RET_IF(p->khist.need(sizeof(int) * nkeys));
    RET_IF(p->kstart.need(sizeof(int) * nkeys));
    RET_IF(p->kcur.need(sizeof(int) * nkeys));
    RET_IF(p->bstart.need(sizeof(int) * nkeys));
    cnt_ex = p->counts.as<int>() + 2 * kMaxLevels;   // [0] written targets, [1] max source
                                                          // column, [2] pairs, [3] batches,
                                                          // [4] materialised locals,
                                                          // [5] stations with a pair,
                                                          // [6 + l] first local row of level l
    CK(cudaMemsetAsync(cnt_ex, 0, 6 * sizeof(int), st));
    if (ns > 0) {   // the largest source column bounds the stations S2L reads: uniform tree,
                    // at the leaf level; adaptive source tree, over the levels (its leaves sit
                    // at every level)
        for (int l = sigma > 0 ? 2 : d; l <= d; ++l) {
            max_col_kernel<<<nblk(std::min<int64_t>(ns, pow4(l)), 256), 256, 0, st>>>(
                p->skeys.as<int>() + lvoff[l], p->counts.as<int>() + l, cnt_ex + 1);
            CKL();
            p->launches++;
        }
    }
    la.depth = d;
    for (int l = 2; l <= d; ++l) {
        la.smap[l] = p->smap.as<int>() + lvoff[l];
        la.tmap[l] = tmap_b + lvoff[l];
    }
    for (int l = 0; l <= d + 1; ++l) la.lvoff[l] = lvoff[l];
    la.nkeys = nkeys;
    la.JT = JT;
    la.pcnt = p->pcnt.as<int>();
    la.poff = p->poff.as<int>();
    la.khist = p->khist.as<int>();
    la.kstart = p->kstart.as<int>();
    la.kcur = p->kcur.as<int>();
    la.bstart = p->bstart.as<int>();
    la.written = p->written.as<unsigned char>();
    la.wlist = p->wlist.as<int>();
    la.wcount = cnt_ex;
    la.totals = cnt_ex + 2;
    CK(cudaMemsetAsync(la.khist, 0, sizeof(int) * nkeys, st));
    CK(cudaMemsetAsync(la.kcur, 0, sizeof(int) * nkeys, st));
    s2l_count_kernel<<<nblk(ltot, 256), 256, 0, st>>>(la);
    CKL();
    s2l_nbatch_kernel<<<nblk(nkeys, 256), 256, 0, st>>>(la);
    CKL();
    CK(cudaMemcpyAsync(la.poff, la.pcnt, sizeof(int) * ltot, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(la.kstart, la.khist, sizeof(int) * nkeys, cudaMemcpyDeviceToDevice, st));
    RET_IF(scan_excl(p, la.poff, ltot, st));
    RET_IF(scan_excl(p, la.kstart, nkeys, st));
    RET_IF(scan_excl(p, la.bstart, nkeys, st));
    s2l_totals_kernel<<<1, 32, 0, st>>>(la);
    CKL();
    p->launches += 3;
    // the stations S2L reads (a key with a pair), a compact list for the tensor kernels
    RET_IF(p->stflag.need(sizeof(int) * nstat));
    RET_IF(p->stlist.need(sizeof(int) * nstat));
    {
        int *fl = p->stflag.as<int>(), *ps = p->kcur.as<int>();   // kcur is free until the emit
        s2l_station_flags_kernel<<<nblk(nstat, 256), 256, 0, st>>>(la.khist, (int)nstat, fl);
        CKL();
        CK(cudaMemcpyAsync(ps, fl, sizeof(int) * nstat, cudaMemcpyDeviceToDevice, st));
        RET_IF(scan_excl(p, ps, nstat, st));
        s2l_station_emit_kernel<<<nblk(nstat, 256), 256, 0, st>>>(fl, ps, (int)nstat, p->stlist.as<int>());
        CKL();
        l2p_ntasks_kernel<<<1, 32, 0, st>>>(ps, fl, nstat, cnt_ex + 5);
        CKL();
        CK(cudaMemsetAsync(la.kcur, 0, sizeof(int) * nkeys, st));
        p->launches += 3;
    }
    // lazy downward pass: which target locals are materialised (need = written or a child
    // needs, bottom-up, fmm_ops.cuh); only those get a row of the local storage (compact lrow)
    RET_IF(p->need.need(std::max<int64_t>(ltot, 1)));
    RET_IF(p->lrow.need(sizeof(int) * std::max<int64_t>(ltot, 1)));
    {
        NeedArgs na = {};
        na.depth = d;
        for (int l = 2; l <= d; ++l) na.tmap[l] = tmap_b + lvoff[l];
        for (int l = 0; l <= d + 1; ++l) na.lvoff[l] = lvoff[l];
        na.written = la.written;
        na.need = p->need.as<unsigned char>();
        na.needi = p->lrow.as<int>();
        for (int l = d; l >= 2; --l) {
            need_kernel<<<nblk(pow4(l), 256), 256, 0, st>>>(na, l);
            CKL();
            p->launches++;
        }
        RET_IF(scan_excl(p, p->lrow.as<int>(), ltot, st));
        count_total_kernel<<<1, 32, 0, st>>>(p->lrow.as<int>(), p->need.as<unsigned char>(), ltot,
                                             cnt_ex + 4);
        CKL();
        // row -> dense position, first row of each level (L2L walks materialised boxes only)
        RET_IF(p->rowkey.need(sizeof(int64_t) * std::max<int64_t>(ltot, 1)));
        LevelOffsets lo = {};   // by value: no host-to-device copy on the solve's stream (it
                                // would queue behind a pipelined solve's upload)
        for (int l = 0; l <= d + 1; ++l) lo.v[l] = lvoff[l];
        need_rows_kernel<<<nblk(ltot, 256), 256, 0, st>>>(p->lrow.as<int>(), p->need.as<unsigned char>(),
                                                         ltot, p->rowkey.as<int64_t>());
        CKL();
        level_rows_kernel<<<1, 32, 0, st>>>(p->lrow.as<int>(), p->need.as<unsigned char>(), lo, d,
                                            cnt_ex + 6);
        CKL();
        p->launches += 3;
    }
    // near-field window state (K in (33, 66], two mode windows): pair slots by target leaf
    if (wsave) {
        const int64_t nl = pow4(d);
        RET_IF(p->pbase.need(sizeof(int64_t) * (nl + 2)));
        RET_IF(p->pcnt64.need(sizeof(int64_t) * nl));
        int64_t *pb = p->pbase.as<int64_t>(), *pc = p->pcnt64.as<int64_t>();
        CK(cudaMemsetAsync(pc, 0, sizeof(int64_t) * nl, st));
        near_leaf_pairs_kernel<<<nblk(nl, 256), 256, 0, st>>>(tmap_b + lvoff[d], flstart, p->slstart.as<int>(), d, pc);
        CKL();
        CK(cudaMemcpyAsync(pb, pc, sizeof(int64_t) * nl, cudaMemcpyDeviceToDevice, st));
        RET_IF(scan_excl(p, pb, nl, st));
        total64_kernel<<<1, 32, 0, st>>>(pb, pc, nl, pb + nl);
        CKL();
        p->launches += 3;
    }
    // the level counts, the error flag and the window-slot count reach the host through mapped
    // pinned memory written by a kernel (a device-to-host copy on this stream would queue behind
    // a pipelined solve's multi-GB download on the copy engine)
    mailbox_kernel<<<1, 64, 0, st>>>(p->counts.as<int>(), 3 * kMaxLevels + 8, p->err.as<int>(),
                                     wsave ? p->pbase.as<int64_t>() + pow4(d) : nullptr, p->mbox_dev);
    CKL();
    CK(cudaStreamSynchronize(st));
    memcpy(hcnt, p->mbox, sizeof(int) * (3 * kMaxLevels + 8));
    if (wsave) memcpy(&nslots, p->mbox + kMboxSlots, sizeof(int64_t));
    RET_IF(err_status(p->mbox[kMboxErr]));
        if (share)
            for (int l = 0; l < kMaxLevels; ++l) hcnt[kMaxLevels + l] = hcnt[l];
    } else {
        T.end(PH_SORT, st);
        T.beg(PH_LISTS, st);
    }
    if (ns > 0) {
        if (s_ready) CK(cudaStreamWaitEvent(st, s_ready, 0));   // host solve: S copied behind the sort
        gather_points_kernel<<<nblk(ns * std::max(K, 1), 256), 256, 0, st>>>(
            src_r, src_z, reinterpret_cast<const double2 *>(src_S), sperm, ns, K,
            p->sr_s.as<double>(), p->sz_s.as<double>(), p->S_s.as<double2>());
        CKL();
        p->launches++;
    }
    const double *fr_sorted = same ? p->sr_s.as<double>() : p->fr_s.as<double>();
    const double *fz_sorted = same ? p->sz_s.as<double>() : p->fz_s.as<double>();
    // the pair lists, now that their sizes are known
    const int64_t npairs = hcnt[2 * kMaxLevels + 2], nbatches = hcnt[2 * kMaxLevels + 3];
    const int nwritten = hcnt[2 * kMaxLevels];
    const int64_t nlc = hcnt[2 * kMaxLevels + 4];   // materialised locals (Lc rows)
    // stations i_in <= the largest source column (C5: 35% of them) are the only ones S2L reads
    const int64_t nstat_used = ns > 0 ? 12 * std::min<int64_t>(1 << d, hcnt[2 * kMaxLevels + 1] + 1) : 0;
    const int64_t nstu = hcnt[2 * kMaxLevels + 5];   // stations with a pair (<= nstat_used)
    ta.glist = p->stlist.as<int>();
    RET_IF(p->pairs.need(sizeof(int4) * std::max<int64_t>(npairs, 1)));
    RET_IF(p->batches.need(sizeof(int4) * std::max<int64_t>(nbatches, 1)));
    la.pairs = p->pairs.as<int4>();
    la.batches = p->batches.as<int4>();
    if (!reuse) {
    if (npairs > 0) {
        s2l_emit_kernel<<<nblk(ltot, 256), 256, 0, st>>>(la);
        CKL();
        s2l_batch_emit_kernel<<<nblk(nkeys, 256), 256, 0, st>>>(la);
        CKL();
        p->launches += 2;
    }
        // remember the geometry for the next solve with the same coordinate arrays
        p->geo.valid = true;
        p->geo.sr = src_r;
        p->geo.sz = src_z;
        p->geo.fr = fld_r;
        p->geo.fz = fld_z;
        p->geo.ns = ns;
        p->geo.nf = nf;
        p->geo.grad = grad;
        p->geo.sperm = sperm;
        p->geo.fperm = fperm;
        p->geo.skey_s = skey_s;
        p->geo.fkey_s = fkey_s;
        p->geo.nslots = nslots;
        memcpy(p->geo.hcnt, hcnt, sizeof hcnt);
    }
    T.end(PH_LISTS, st);
    // ---- far-field storage
    FarArgs fa = {};
    fa.depth = d;
    fa.p = pp;
    fa.P = P;
    fa.pl = pl;
    fa.Pl = Pl;
    fa.pt = pt;
    fa.K = K;
    fa.L = q.domain_L;
    fa.z0 = q.domain_z0;
    fa.truncation = q.truncation;
    int64_t stot = 0, ttot = 0;
    for (int l = 2; l <= d; ++l) {
        fa.smap[l] = p->smap.as<int>() + lvoff[l];
        fa.skeys[l] = p->skeys.as<int>() + lvoff[l];
        fa.tmap[l] = tmap_b + lvoff[l];
        fa.tkeys[l] = tkeys_b + lvoff[l];
        fa.scount[l] = ns > 0 ? hcnt[l] : 0;
        fa.tcount[l] = hcnt[kMaxLevels + l];
        fa.soff[l] = stot;
        fa.toff[l] = ttot;
        stot += fa.scount[l];
        ttot += fa.tcount[l];
    }
    const int64_t TP = (int64_t)(pt + 1) * (pt + 1) * (pt + 1) + ((pt + 1) & 1);  // padded
    if (q.mode_chunk == 0) {
        // automatic chunk: the far-field workspace (moments, locals, tensors per mode) of one
        // chunk must fit in a third of the free device memory (C5: 1.8 GB per mode).  The free
        // memory is queried only when the current allocations cannot hold all modes (the query
        // is slow; steady-state solves reuse the plan's workspace).
        size_t per_mode = sizeof(double2) * ((size_t)2 * stot * P + (size_t)(nlc + npairs) * Pl) +
                          sizeof(double) * nstat_used * TP;
        size_t have = p->M.cap + p->Lc.cap + p->tens.cap + p->pairbuf.cap;   // reusable allocations
        if (per_mode * (size_t)K > have) {
            size_t fmem = 0, tot = 0;
            CK(cudaMemGetInfo(&fmem, &tot));
            size_t budget = (fmem + have) / 3;
            int64_t kw = (int64_t)(budget / std::max<size_t>(per_mode, 1));
            KW = (int)std::max<int64_t>(1, std::min<int64_t>(K, kw));
            if (KW < K) KW = (K + (K + KW - 1) / KW - 1) / ((K + KW - 1) / KW);  // balanced chunks
            p->auto_kw = KW;
        } else {
            KW = p->auto_kw > 0 ? std::min(p->auto_kw, K) : K;
        }
    }
    if (split) {   // the moment broadcasts run per mode chunk: every rank takes the smallest chunk
        RET_IF(p->g_cnt.need(sizeof(int64_t) * (p->nranks + 1)));
        int64_t *dkw = p->g_cnt.as<int64_t>();
        const int64_t mine = KW;
        CK(cudaMemcpyAsync(dkw + p->nranks, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        NC(g_nccl.AllGather(dkw + p->nranks, dkw, 1, ncclInt64, p->comm, st));
        std::vector<int64_t> kws((size_t)p->nranks);
        CK(cudaMemcpyAsync(kws.data(), dkw, sizeof(int64_t) * p->nranks, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t v : kws) KW = (int)std::min<int64_t>(KW, v);
    }
    // moments, then their S2L copy for backward pairs (prescale_moments_kernel)
    RET_IF(p->M.need(sizeof(double2) * (size_t)std::max<int64_t>(stot, 1) * KW * P * 2));
    RET_IF(p->Lc.need(sizeof(double2) * (size_t)std::max<int64_t>(nlc, 1) * KW * Pl));
    RET_IF(p->tens.need(sizeof(double) * (size_t)std::max<int64_t>(nstat_used, 1) * KW * TP));
    RET_IF(p->pairbuf.need(sizeof(double2) * (size_t)std::max<int64_t>(npairs, 1) * KW * Pl));
    fa.M = p->M.as<double2>();
    fa.Lc = p->Lc.as<double2>();
    fa.tens = p->tens.as<double>();
    fa.slstart = p->slstart.as<int>();
    fa.sigma = sigma;
    fa.flstart = flstart;
    fa.sr = p->sr_s.as<double>();
    fa.sz = p->sz_s.as<double>();
    fa.S = p->S_s.as<double2>();
    fa.fr = fr_sorted;
    fa.fz = fz_sorted;
    fa.fperm = fperm;
    fa.out = reinterpret_cast<double2 *>(out_Phi);
    fa.rtab_m = p->rtab.as<double>();
    fa.rtab_l = p->rtab.as<double>() + p->rtab_nm;
    fa.tritab_m = reinterpret_cast<const int *>(p->rtab.as<double>() + p->rtab_nd);
    fa.tritab_l = fa.tritab_m + p->rtab_ntm;
    fa.pscale = p->rtab.as<double>() + p->rtab_nd - (pp + 1) * (pp + 2) / 2;
    fa.s2l_written = p->written.as<unsigned char>();
    for (int l = 2; l <= d; ++l) fa.lvoff[l] = lvoff[l];
    // S2L batch GEMM and reduction arguments (s2l.cuh)
    S2LArgs sa = {};
    sa.p = pp;
    sa.P = P;
    sa.pl = pl;
    sa.Pl = Pl;
    sa.pt = pt;
    sa.K = K;
    sa.tens = p->tens.as<double>();
    sa.M = p->M.as<double2>();
    sa.Mb = sa.M + (size_t)std::max<int64_t>(stot, 1) * KW * P;
    sa.pairs = p->pairs.as<int4>();
    sa.batches = p->batches.as<int4>();
    for (int l = 2; l <= d; ++l) sa.soff[l] = fa.soff[l];
    sa.truncation = q.truncation;
    sa.pairbuf = p->pairbuf.as<double2>();
    S2LReduceArgs ra = {};
    ra.depth = d;
    ra.nw = nwritten;
    ra.Pl = Pl;
    for (int l = 0; l <= d + 1; ++l) ra.lvoff[l] = lvoff[l];
    ra.lrow = p->lrow.as<int>();
    ra.wlist = p->wlist.as<int>();
    ra.poff = p->poff.as<int>();
    ra.pcnt = p->pcnt.as<int>();
    ra.pairbuf = sa.pairbuf;
    ra.Lc = fa.Lc;
    fa.l2p_accumulate = ns > 0 && overlap;   // L2P adds onto the near field's rows (overlapped)
    fa.tfield = nf;
    RET_IF(p->l2pown.need(sizeof(int) * std::max(hcnt[kMaxLevels + d], 1)));
    RET_IF(p->l2pflag.need(sizeof(int) * nf));
    RET_IF(p->l2ppos.need(sizeof(int) * nf));
    RET_IF(p->l2ptask.need(sizeof(int) * (nf / 16 + hcnt[kMaxLevels + d] + 1)));
    RET_IF(p->l2pntask.need(sizeof(int)));
    fa.outr = grad ? reinterpret_cast<double2 *>(out_dr) : nullptr;
    fa.outz = grad ? reinterpret_cast<double2 *>(out_dz) : nullptr;
    fa.need = p->need.as<unsigned char>();
    fa.lrow = p->lrow.as<int>();
    fa.rowkey = p->rowkey.as<int64_t>();
    for (int l = 2; l <= d + 1; ++l) fa.lrow_lev[l] = hcnt[2 * kMaxLevels + 6 + l];
    // tree done: the near field and the tensors start behind it on their own streams
    if (overlap || seeds_aside) {
        CK(cudaEventRecord(p->aev[1], st));
        CK(cudaStreamWaitEvent(st_s, p->aev[1], 0));
    }
    if (nstu > 0 && !(reuse && KW == K)) {   // seeds of all modes once, stations with a pair
        T.beg(PH_SEEDS, st_s);
        RET_IF(run_seeds(ta, nstu, st_s));
        p->launches++;
        T.end(PH_SEEDS, st_s);
    }
    if (seeds_aside) CK(cudaEventRecord(p->aev[2], st_s));
    // ---- near field.  Overlapped (small) solves: first, on its own stream, writing
    // every field row, and L2P adds the far field; serial (large) solves: after L2P, adding onto
    // the rows L2P wrote (the read-modify-write then sits at the end of long near-field tasks
    // instead of inside the short L2P items)
    const bool near_first = overlap;
    auto run_near = [&](int accumulate) -> cylfmm_status {
        if (ns > 0) {
            if (overlap) CK(cudaStreamWaitEvent(st_n, p->aev[1], 0));
            T.beg(PH_P2P, st_n);
            const int ntl = fa.tcount[d];
            double avg = (double)nf / std::max(ntl, 1);
            const int TT = avg <= 10.0 ? 8 : (avg <= 24.0 ? 16 : 32);
            const bool wk = p2pw_enabled(K, grad);
            const int sigma = q.adaptive_leaf;
            RET_IF(p->tcnt.need(sizeof(int) * (ntl + 1)));
            RET_IF(p->ntasks.need(kTaskCtrInts * sizeof(int)));
            // warp tasks: <= nf/32 full pieces + <= 5 power-of-two pieces per leaf (per box of a
            // level under the adaptive tree)
            int64_t maxtasks = wk ? nf / 32 + 6 * (int64_t)ntl + 1 : nf / TT + ntl + 1;
            if (sigma > 0)
                for (int l = 2; l < d; ++l) maxtasks = std::max<int64_t>(maxtasks, nf / 32 + 6 * (int64_t)fa.tcount[l] + 1);
            RET_IF(p->tasks.need(sizeof(int4) * maxtasks));
            if (sigma > 0) {
                // adaptive source tree (R#26): one accumulating launch per level, over the target
                // boxes with a neighbour pair that stops there (each launch owns its rows)
                unsigned long long *ctr = p->ctr.as<unsigned long long>();
                for (int l = 2; l <= d; ++l) {
                    const int nbx = fa.tcount[l];
                    if (nbx == 0) continue;
                    CK(cudaMemsetAsync(p->ntasks.as<int>(), 0, kTaskCtrInts * sizeof(int), st_n));
                    near_wtasks_count_kernel<<<nblk(nbx, 256), 256, 0, st_n>>>(fa.tkeys[l], nbx, fa.flstart,
                                                                            fa.slstart, d, 1, l, sigma,
                                                                            p->ntasks.as<int>());
                    CKL();
                    near_wtasks_emit_kernel<<<nblk(nbx, 256), 256, 0, st_n>>>(fa.tkeys[l], nbx, fa.flstart,
                                                                           fa.slstart, d, 1, l, sigma,
                                                                           p->tasks.as<int4>(),
                                                                           p->ntasks.as<int>());
                    CKL();
                    P2PArgs a = {};
                    a.sr = fa.sr;
                    a.sz = fa.sz;
                    a.S = fa.S;
                    a.fr = fa.fr;
                    a.fz = fa.fz;
                    a.ns = ns;
                    a.nf = nf;
                    a.K = K;
                    a.m0 = 0;
                    a.m1 = K;
                    a.miller = q.miller;
                    a.fwd2 = forward_coef(K - 1, q.miller);
                    a.exclude = q.exclude_coincident;
                    a.out = fa.out;
                    a.out_row = fperm;
                    a.accumulate = 1;
                    a.tasks = p->tasks.as<int4>();
                    a.ntasks = p->ntasks.as<int>();
                    a.task_ctr = p->ntasks.as<int>() + 1;
                    a.leafstart = fa.slstart;
                    a.depth = d;
                    a.level = l;
                    a.adaptive_leaf = sigma;
                    a.n_skipped = ctr + 0;
                    a.n_pairs = ctr + 1;
                    a.n_branch = ctr + 3;
                    a.err_flag = p->err.as<int>();
                    CK(launch_p2pw(a, st_n));
                    p->launches += 3;
                }
                T.end(PH_P2P, st_n);
                return CYLFMM_OK;
            }
            if (wk && reuse) {   // the task list is the previous solve's: rewind the fetch counter
                CK(cudaMemsetAsync(p->ntasks.as<int>() + 1, 0, sizeof(int), st_n));
            } else if (wk) {
                CK(cudaMemsetAsync(p->ntasks.as<int>(), 0, kTaskCtrInts * sizeof(int), st_n));
                near_wtasks_count_kernel<<<nblk(ntl, 256), 256, 0, st_n>>>(fa.tkeys[d], ntl, fa.flstart,
                                                                        fa.slstart, d, accumulate, 0, 0,
                                                                        p->ntasks.as<int>());
                CKL();
                near_wtasks_emit_kernel<<<nblk(ntl, 256), 256, 0, st_n>>>(fa.tkeys[d], ntl, fa.flstart,
                                                                       fa.slstart, d, accumulate, 0, 0,
                                                                       p->tasks.as<int4>(),
                                                                       p->ntasks.as<int>());
            } else {
                near_tasks_count_kernel<<<nblk(ntl, 256), 256, 0, st_n>>>(fa.tkeys[d], ntl, fa.flstart, TT,
                                                                       p->tcnt.as<int>());
                CKL();
                RET_IF(scan_excl(p, p->tcnt.as<int>(), ntl, st_n, 0, 1));
                near_tasks_emit_kernel<<<nblk(ntl, 256), 256, 0, st_n>>>(fa.tkeys[d], ntl, fa.flstart, TT,
                                                                      p->tcnt.as<int>(), p->tasks.as<int4>(),
                                                                      p->ntasks.as<int>());
            }
            CKL();
            p->launches += 2;
            unsigned long long *ctr = p->ctr.as<unsigned long long>();
            const int win = wk ? kP2PWWindow : kP2PWindow;
            if (wsave) {
                RET_IF(p->sv2.need(sizeof(double2) * (size_t)std::max<int64_t>(nslots, 1)));
                RET_IF(p->sv1.need(sizeof(double) * (size_t)std::max<int64_t>(nslots, 1)));
            }
            for (int m0 = 0; m0 < K; m0 += win) {
                P2PArgs a = {};
                a.sr = fa.sr;
                a.sz = fa.sz;
                a.S = fa.S;
                a.fr = fa.fr;
                a.fz = fa.fz;
                a.ns = ns;
                a.nf = nf;
                a.K = K;
                a.m0 = m0;
                a.m1 = std::min(K, m0 + win);
                a.miller = q.miller;
                a.fwd2 = forward_coef(K - 1, q.miller);
                a.exclude = q.exclude_coincident;
                a.out = fa.out;
                a.outr = fa.outr;
                a.outz = fa.outz;
                a.out_row = fperm;
                a.accumulate = accumulate;
                a.tasks = p->tasks.as<int4>();
                a.ntasks = p->ntasks.as<int>();
                a.leafstart = fa.slstart;
                a.depth = d;
                a.n_skipped = ctr + 0;
                a.n_pairs = ctr + 1;
                a.n_branch = ctr + 3;
                a.err_flag = p->err.as<int>();
                if (wsave) {   // first window saves the chain state, the second restarts from it
                    a.save = m0 == 0 ? 1 : 2;
                    a.sv2 = p->sv2.as<double2>();
                    a.sv1 = p->sv1.as<double>();
                    a.pbase = p->pbase.as<int64_t>();
                    a.tmap_leaf = fa.tmap[d];
                    a.fleafstart = fa.flstart;
                }
                const dim3 grid((unsigned)maxtasks);
                a.task_ctr = p->ntasks.as<int>() + 1;
                if (wk) CK(launch_p2pw(a, st_n));
                else if (grad) CK((launch_p2p<true, true>(TT, a, grid, st_n)));
                else CK(launch_p2p<true>(TT, a, grid, st_n));
                p->launches++;
            }
            T.end(PH_P2P, st_n);
            if (overlap) CK(cudaEventRecord(p->aev[3], st_n));
        }
        return CYLFMM_OK;
    };
    if (near_first) RET_IF(run_near(0));
    for (int m0 = 0; m0 < K; m0 += KW) {
        fa.m0 = m0;
        fa.m1 = std::min(K, m0 + KW);
        const int kw = fa.m1 - fa.m0;
        // tensors for the normalised stations (shared by all levels): seeds of all modes once,
        // the Laplace fill per mode chunk (behind M2M when the seeds run aside)
        auto run_fill_chunk = [&]() -> cylfmm_status {
            ta.out = p->tens.as<double>();
            ta.m0 = fa.m0;
            ta.m1 = fa.m1;
            ta.seed_m1 = K;
            if (overlap && m0 > 0) CK(cudaStreamWaitEvent(st_t, p->aev[4], 0));  // previous S2L done
            T.beg(PH_TENSOR, st_t);
            // the stations with a pair are the only ones S2L reads (dense layout, i_in <= the
            // largest source column)
            // (reused with the geometry when all modes fit one chunk: the tensors are still there)
            if (nstu > 0 && !(reuse && KW == K)) RET_IF(run_fill(ta, nstu, st_t));
            p->launches++;
            T.end(PH_TENSOR, st_t);
            if (overlap) CK(cudaEventRecord(p->aev[2], st_t));
            return CYLFMM_OK;
        };
        if (!seeds_aside) RET_IF(run_fill_chunk());
        if (ns > 0) {
        if (sigma > 0) {
            // adaptive source tree: P2M at every source leaf, whatever its level (the kernel
            // skips the boxes above the leaves: M2M forms them), then M2M over the boxes above
            T.beg(PH_P2M, st);
            const int nmb = (kw + kP2MModes - 1) / kP2MModes;
            fa.p2m_slot0 = 0;
            for (int l = 2; l <= d; ++l) {
                if (fa.scount[l] == 0) continue;
                fa.p2m_level = l;
                RET_IF(launch_p2m(fa, (unsigned)((int64_t)fa.scount[l] * nmb), P, pp, st));
                CKL();
                p->launches++;
            }
            fa.p2m_level = 0;
            T.end(PH_P2M, st);
        } else {
            T.beg(PH_P2M, st);
            const int nl = fa.scount[d];
            auto leaf0 = [&](int r) { return (int)((int64_t)nl * r / (split ? p->nranks : 1)); };
            const int a0 = split ? leaf0(p->rank) : 0, a1 = split ? leaf0(p->rank + 1) : nl;
            if (a1 > a0) {
                const int nmb = (kw + kP2MModes - 1) / kP2MModes;
                fa.p2m_slot0 = a0;
                RET_IF(launch_p2m(fa, (unsigned)((int64_t)(a1 - a0) * nmb), P, pp, st));
                CKL();
                p->launches++;
            }
            T.end(PH_P2M, st);
            if (split && nl > 0) {   // every rank's leaf moments to every rank
                T.beg(PH_ALLGATHER, st);
                NC(g_nccl.GroupStart());
                for (int r = 0; r < p->nranks; ++r) {
                    const int b0 = leaf0(r), b1 = leaf0(r + 1);
                    if (b1 <= b0) continue;
                    double *base = reinterpret_cast<double *>(fa.M + (fa.soff[d] + b0) * (int64_t)kw * P);
                    NC(g_nccl.Broadcast(base, base, (size_t)(b1 - b0) * kw * P * 2, ncclFloat64, r, p->comm, st));
                }
                NC(g_nccl.GroupEnd());
                T.end(PH_ALLGATHER, st);
            }
        }
            T.beg(PH_M2M, st);
            for (int l = d - 1; l >= 2; --l) {
                if (fa.scount[l] == 0) continue;
                unsigned g = (unsigned)((int64_t)fa.scount[l] * ((kw + kMMG - 1) / kMMG));
                m2m_kernel<<<g, 256, m2m_smem(pp), st>>>(fa, l);
                CKL();
                p->launches++;
            }
            // S2L consumes the moments pre-scaled by (-1)^j / j! (fmm_ops.cuh)
            prescale_moments_kernel<<<nblk(stot * kw * P, 256), 256, 0, st>>>(fa.M, const_cast<double2 *>(sa.Mb), stot * kw, P, fa.pscale);
            CKL();
            p->launches++;
            T.end(PH_M2M, st);
        }
        if (seeds_aside) {
            if (m0 == 0) CK(cudaStreamWaitEvent(st, p->aev[2], 0));   // seeds done
            RET_IF(run_fill_chunk());
        }
        // S2L of every level in one launch (each level's contribution), then the L2L chain
        if (overlap) CK(cudaStreamWaitEvent(st, p->aev[2], 0));   // tensors of this chunk ready
        T.beg(PH_S2L, st);
        if (ns > 0 && npairs > 0) {
            sa.m0 = fa.m0;
            sa.m1 = fa.m1;
            ra.KW = kw;
            CK(launch_s2l(sa, nbatches, npairs, st));
            const int64_t witems = (int64_t)nwritten * kw;
            s2l_reduce_kernel<<<(unsigned)std::min<int64_t>((witems + 7) / 8, (int64_t)p->nsm * 16), 256, 0, st>>>(ra);
            CKL();
            p->launches++;
            p->launches++;
        }
        T.end(PH_S2L, st);
        if (overlap) CK(cudaEventRecord(p->aev[4], st));
        T.beg(PH_L2L, st);
        for (int l = 3; l <= d; ++l) {
            const int64_t nrow = fa.lrow_lev[l + 1] - fa.lrow_lev[l];
            if (nrow == 0) continue;
            int64_t items = nrow * kw;
            unsigned g = (unsigned)std::min<int64_t>((items + kL2LWarps - 1) / kL2LWarps,
                                                     (int64_t)p->nsm * 8);
            l2l_kernel<<<g, 32 * kL2LWarps, l2l_smem(pl), st>>>(fa, l);
            CKL();
            p->launches++;
        }
        T.end(PH_L2L, st);
        if (near_first && ns > 0 && m0 == 0) CK(cudaStreamWaitEvent(st, p->aev[3], 0));  // near field
        T.beg(PH_L2P, st);
        {
            // tasks: runs of <= TP sorted field points sharing their evaluating box; TP from the
            // points per target leaf (C5's leaves hold 4 points but share coarse boxes: 128)
            const int ntl = fa.tcount[d];
            const int64_t ppl = nf / std::max(ntl, 1);
            fa.l2p_tp = ppl < 8 ? 128 : (int)std::min<int64_t>(128, std::max<int64_t>(16, (int64_t)1 << (63 - __builtin_clzll(ppl))));
            const int gpc = kL2PThreads / fa.l2p_tp;
            // CTA-wide tasks (coarse evaluating boxes, C5) take two points per thread (four points
            // on groups of 5 modes measured slower: C5 10.05 vs 9.73 ms)
            const bool two = !grad && fa.l2p_tp == kL2PThreads;
            fa.l2p_run = fa.l2p_tp * (two ? 2 : 1);
            const int64_t ub_tasks = nf / fa.l2p_run + ntl + 1;
            if (m0 == 0 && !reuse) {   // evaluating box of every target leaf and the L2P runs
                l2p_owner_kernel<<<nblk(ntl, 256), 256, 0, st>>>(fa, p->l2pown.as<int>());
                CKL();
                int *flag = p->l2pflag.as<int>(), *pos = p->l2ppos.as<int>();
                l2p_task_flags_kernel<<<nblk(nf, 256), 256, 0, st>>>(fa, fkey_s, p->l2pown.as<int>(), flag);
                CKL();
                CK(cudaMemcpyAsync(pos, flag, sizeof(int) * nf, cudaMemcpyDeviceToDevice, st));
                RET_IF(scan_excl(p, pos, nf, st));
                l2p_task_emit_kernel<<<nblk(nf, 256), 256, 0, st>>>(nf, flag, pos, p->l2ptask.as<int>());
                CKL();
                l2p_ntasks_kernel<<<1, 32, 0, st>>>(pos, flag, nf, p->l2pntask.as<int>());
                CKL();
                p->launches += 5;
            }
            // modes per thread: the groups of a task fill the CTA (gpc groups per item)
            int ngrp = (kw + 15) / 16;
            if (gpc > 1) ngrp = std::max(ngrp, std::min(kw, gpc * ((ngrp + gpc - 1) / gpc)));
            const int mb = (kw + ngrp - 1) / ngrp;
            const int64_t items = ub_tasks * ((ngrp + gpc - 1) / gpc);
            // persistent CTAs over the items (the task count stays on the device)
            const unsigned grid = (unsigned)std::min<int64_t>(items, (int64_t)p->nsm * 16);
            const uint32_t *fk = fkey_s;
            const int *own = p->l2pown.as<int>(), *tst = p->l2ptask.as<int>(), *ntk = p->l2pntask.as<int>();
            const int tp = fa.l2p_tp;
#define L2P_GO(MBV, GR, PTV) \
    l2p_kernel<MBV, GR, PTV><<<grid, kL2PThreads, l2p_smem<MBV>(Pl, kw, tp), st>>>(fa, fk, own, tst, ntk, ngrp)
            if (grad) L2P_GO(16, true, 1);
            else if (mb <= 4) { if (two) L2P_GO(4, false, 2); else L2P_GO(4, false, 1); }
            else if (mb <= 9) { if (two) L2P_GO(9, false, 2); else L2P_GO(9, false, 1); }
            else if (mb == 13 && two && Pl == 153 && kw % ngrp == 0)   // C5: order 16, 65 = 5 x 13
                l2p_kernel<13, false, 2, 16, true><<<grid, kL2PThreads, l2p_smem<13>(Pl, kw, tp), st>>>(fa, fk, own, tst, ntk, ngrp);
            else if (mb <= 13) { if (two) L2P_GO(13, false, 2); else L2P_GO(13, false, 1); }
            else { if (two) L2P_GO(16, false, 2); else L2P_GO(16, false, 1); }
#undef L2P_GO
            CKL();
            p->launches++;
        }
        T.end(PH_L2P, st);
    }
    if (!near_first) RET_IF(run_near(1));   // onto the far field L2P wrote
    T.end(PH_TOTAL, st);
    if (tm) {
        unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        CK(cudaMemcpyAsync(c, p->ctr.p, sizeof(c), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        RET_IF(read_phases(p, tm));
        tm->n_skipped = (int64_t)c[0];
        tm->n_near_pairs = (int64_t)c[1];
        tm->n_s2l_pairs = npairs;
        tm->kernel_launches = p->launches;
        tm->n_forward = (int64_t)c[3];
        tm->n_far = (int64_t)c[4];
        tm->n_miller = (int64_t)c[5];
        tm->miller_steps = (int64_t)c[6];
        RET_IF(check_err_flag(p, st));
    } else if (!q.exclude_coincident && ns > 0) {
        // coincident pairs are an error in this mode: the near-field flag is checked here
        // (one synchronisation), as cylfmm_direct does, not deferred to cylfmm_plan_sync
        RET_IF(check_err_flag(p, st));
    }
    if (!tm && p->prof_on) {
        p->last_npairs = npairs;
        p->last_launches = p->launches;
    }
    return CYLFMM_OK;
}

static cylfmm_status validate_solve(cylfmm_plan plan, const double *sr, const double *sz,
                                    const double *S, int64_t ns, const double *fr, const double *fz,
                                    int64_t nf, const double *out)
{
    if (!plan) {
        set_err("cylfmm_fmm_solve: null plan");
        return CYLFMM_EINVAL;
    }
    if (ns < 0 || nf < 0 || ns > INT32_MAX || nf > INT32_MAX ||
        (ns > 0 && (!sr || !sz || !S)) || (nf > 0 && (!fr || !fz || !out))) {
        set_err("cylfmm_fmm_solve: bad sizes or null pointer");
        return CYLFMM_EINVAL;
    }
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_fmm_solve(cylfmm_plan plan, const double *src_r,
                                          const double *src_z, const double *src_S, int64_t n_src,
                                          const double *fld_r, const double *fld_z, int64_t n_fld,
                                          double *out_Phi, cylfmm_stream_t stream,
                                          cylfmm_timings *timings)
{
    RET_IF(validate_solve(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi));
    CK(cudaSetDevice(plan->device));
    return fmm_solve_impl(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi,
                          (cudaStream_t)stream, timings);
}

extern "C" cylfmm_status cylfmm_fmm_solve_grad(cylfmm_plan plan, const double *src_r,
                                               const double *src_z, const double *src_S,
                                               int64_t n_src, const double *fld_r,
                                               const double *fld_z, int64_t n_fld,
                                               double *out_Phi, double *out_dPhi_dr,
                                               double *out_dPhi_dz, cylfmm_stream_t stream,
                                               cylfmm_timings *timings)
{
    RET_IF(validate_solve(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi));
    if (n_fld > 0 && (!out_dPhi_dr || !out_dPhi_dz)) {
        set_err("cylfmm_fmm_solve_grad: null gradient output");
        return CYLFMM_EINVAL;
    }
    if (plan->prm.n_modes > kP2PWindow) {
        set_err("cylfmm_fmm_solve_grad: gradients support n_modes <= %d", kP2PWindow);
        return CYLFMM_EINVAL;
    }
    if (plan->prm.adaptive_leaf > 0) {
        set_err("cylfmm_fmm_solve_grad: gradients use the uniform tree (adaptive_leaf = 0)");
        return CYLFMM_EINVAL;
    }
    CK(cudaSetDevice(plan->device));
    return fmm_solve_impl(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi,
                          (cudaStream_t)stream, timings, out_dPhi_dr, out_dPhi_dz);
}

extern "C" cylfmm_status cylfmm_fmm_solve_host(cylfmm_plan plan, const double *src_r,
                                               const double *src_z, const double *src_S,
                                               int64_t n_src, const double *fld_r,
                                               const double *fld_z, int64_t n_fld,
                                               double *out_Phi, cylfmm_stream_t stream,
                                               cylfmm_timings *timings)
{
    RET_IF(validate_solve(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi));
    CK(cudaSetDevice(plan->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int K = plan->prm.n_modes;
    size_t bs = 8 * (size_t)std::max<int64_t>(n_src, 1), bf = 8 * (size_t)std::max<int64_t>(n_fld, 1);
    RET_IF(plan->h_sr.need(bs));
    RET_IF(plan->h_sz.need(bs));
    RET_IF(plan->h_S.need(bs * 2 * K));
    RET_IF(plan->h_fr.need(bf));
    RET_IF(plan->h_fz.need(bf));
    RET_IF(plan->h_out.need(bf * 2 * K));
    if (n_src > 0) {
        CK(cudaMemcpyAsync(plan->h_sr.p, src_r, 8 * n_src, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(plan->h_sz.p, src_z, 8 * n_src, cudaMemcpyHostToDevice, st));
        // the K-mode coefficient rows (the bulk of the input) on their own stream: they are
        // first read by the gather after the Morton sort, so the copy overlaps the tree build
        CK(cudaEventRecord(plan->hev[0], st));
        CK(cudaStreamWaitEvent(plan->hcp, plan->hev[0], 0));
        CK(cudaMemcpyAsync(plan->h_S.p, src_S, 16 * (size_t)n_src * K, cudaMemcpyHostToDevice, plan->hcp));
        CK(cudaEventRecord(plan->hev[1], plan->hcp));
    }
    // fields == sources (same host arrays): copied once, one tree serves both
    const bool same = fld_r == src_r && fld_z == src_z && n_fld == n_src;
    if (n_fld > 0 && !same) {
        CK(cudaMemcpyAsync(plan->h_fr.p, fld_r, 8 * n_fld, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(plan->h_fz.p, fld_z, 8 * n_fld, cudaMemcpyHostToDevice, st));
    }
    const double *dfr = same ? plan->h_sr.as<double>() : plan->h_fr.as<double>();
    const double *dfz = same ? plan->h_sz.as<double>() : plan->h_fz.as<double>();
    RET_IF(fmm_solve_impl(plan, plan->h_sr.as<double>(), plan->h_sz.as<double>(),
                          plan->h_S.as<double>(), n_src, dfr, dfz, n_fld,
                          plan->h_out.as<double>(), st, timings, nullptr, nullptr,
                          n_src > 0 ? plan->hev[1] : nullptr));
    if (n_fld > 0)
        CK(cudaMemcpyAsync(out_Phi, plan->h_out.p, 16 * (size_t)n_fld * K, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return check_err_flag(plan, st);
}

extern "C" cylfmm_status cylfmm_fmm_solve_host_async(cylfmm_plan plan, const double *src_r,
                                                     const double *src_z, const double *src_S,
                                                     int64_t n_src, const double *fld_r,
                                                     const double *fld_z, int64_t n_fld,
                                                     double *out_Phi, cylfmm_stream_t stream)
{
    RET_IF(validate_solve(plan, src_r, src_z, src_S, n_src, fld_r, fld_z, n_fld, out_Phi));
    CK(cudaSetDevice(plan->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int K = plan->prm.n_modes;
    auto &h = plan->hs[plan->hslot];
    plan->hslot ^= 1;
    const bool same = fld_r == src_r && fld_z == src_z && n_fld == n_src;
    size_t bs = 8 * (size_t)std::max<int64_t>(n_src, 1), bf = 8 * (size_t)std::max<int64_t>(n_fld, 1);
    // the slot's previous solve has read its inputs and its download has left the result
    // buffer before either is overwritten (events never recorded: no wait).  (Growing a slot
    // reallocates: the host waits for that slot's previous work first.)
    if (h.sr.cap < bs || h.S.cap < bs * 2 * K || h.fr.cap < bf || h.out.cap < bf * 2 * K) {
        CK(cudaEventSynchronize(h.done));
        CK(cudaEventSynchronize(h.down));
    }
    RET_IF(h.sr.need(bs));
    RET_IF(h.sz.need(bs));
    RET_IF(h.S.need(bs * 2 * K));
    RET_IF(h.fr.need(bf));
    RET_IF(h.fz.need(bf));
    RET_IF(h.out.need(bf * 2 * K));
    CK(cudaStreamWaitEvent(plan->hcp, h.done, 0));
    if (n_src > 0) {
        CK(cudaMemcpyAsync(h.sr.p, src_r, 8 * n_src, cudaMemcpyHostToDevice, plan->hcp));
        CK(cudaMemcpyAsync(h.sz.p, src_z, 8 * n_src, cudaMemcpyHostToDevice, plan->hcp));
    }
    if (n_fld > 0 && !same) {
        CK(cudaMemcpyAsync(h.fr.p, fld_r, 8 * n_fld, cudaMemcpyHostToDevice, plan->hcp));
        CK(cudaMemcpyAsync(h.fz.p, fld_z, 8 * n_fld, cudaMemcpyHostToDevice, plan->hcp));
    }
    CK(cudaEventRecord(h.coords, plan->hcp));
    // the coefficient rows last: first read by the gather after the Morton sort
    if (n_src > 0) CK(cudaMemcpyAsync(h.S.p, src_S, 16 * (size_t)n_src * K, cudaMemcpyHostToDevice, plan->hcp));
    CK(cudaEventRecord(h.coef, plan->hcp));
    CK(cudaStreamWaitEvent(st, h.coords, 0));
    CK(cudaStreamWaitEvent(st, h.down, 0));
    const double *dfr = same ? h.sr.as<double>() : h.fr.as<double>();
    const double *dfz = same ? h.sz.as<double>() : h.fz.as<double>();
    RET_IF(fmm_solve_impl(plan, h.sr.as<double>(), h.sz.as<double>(), h.S.as<double>(), n_src,
                          dfr, dfz, n_fld, h.out.as<double>(), st, nullptr, nullptr, nullptr,
                          n_src > 0 ? h.coef : nullptr));
    CK(cudaEventRecord(h.done, st));
    CK(cudaStreamWaitEvent(plan->hdn, h.done, 0));
    if (n_fld > 0)
        CK(cudaMemcpyAsync(out_Phi, h.out.p, 16 * (size_t)n_fld * K, cudaMemcpyDeviceToHost, plan->hdn));
    CK(cudaEventRecord(h.down, plan->hdn));
    return CYLFMM_OK;
}

// ------------------------------------------------------------------------------------------
// multi-device solves (one process per GPU, a library-owned NCCL communicator)
extern "C" cylfmm_status cylfmm_comm_unique_id(void *unique_id)
{
    if (!unique_id) {
        set_err("cylfmm_comm_unique_id: null pointer");
        return CYLFMM_EINVAL;
    }
    if (!load_nccl()) {
        set_err("cylfmm_comm_unique_id: libnccl.so.2 not found");
        return CYLFMM_ENCCL;
    }
    ncclUniqueId id;
    NC(g_nccl.GetUniqueId(&id));
    memcpy(unique_id, &id, sizeof id);
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_plan_create_dist(cylfmm_plan *plan, const cylfmm_params *prm,
                                                 int nranks, int rank, const void *unique_id)
{
    if (!plan || !prm || !unique_id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_err("cylfmm_plan_create_dist: bad arguments (nranks=%d rank=%d)", nranks, rank);
        return CYLFMM_EINVAL;
    }
    if (!load_nccl()) {
        set_err("cylfmm_plan_create_dist: libnccl.so.2 not found");
        return CYLFMM_ENCCL;
    }
    RET_IF(cylfmm_plan_create(plan, prm));
    cylfmm_plan p = *plan;
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof id);
    const ncclResult_t r = g_nccl.CommInitRank(&p->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        set_err("cylfmm_plan_create_dist: ncclCommInitRank: %s", g_nccl.GetErrorString(r));
        p->comm = nullptr;
        cylfmm_plan_destroy(p);
        *plan = nullptr;
        return CYLFMM_ENCCL;
    }
    p->nranks = nranks;
    p->rank = rank;
    return CYLFMM_OK;
}

extern "C" cylfmm_status cylfmm_fmm_solve_dist(cylfmm_plan plan, const double *src_r,
                                               const double *src_z, const double *src_S,
                                               int64_t n_src_local, const double *fld_r,
                                               const double *fld_z, int64_t n_fld_local,
                                               double *out_Phi, cylfmm_stream_t stream,
                                               cylfmm_timings *timings)
{
    RET_IF(validate_solve(plan, src_r, src_z, src_S, n_src_local, fld_r, fld_z, n_fld_local, out_Phi));
    if (!plan->comm) {
        set_err("cylfmm_fmm_solve_dist: the plan has no communicator (cylfmm_plan_create_dist)");
        return CYLFMM_EINVAL;
    }
    CK(cudaSetDevice(plan->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int R = plan->nranks, K = plan->prm.n_modes;
    // shard sizes of every rank (all-gather), then the shards themselves: one broadcast per
    // rank, grouped (NCCL over NVLink / NVSwitch), into the plan's replicated source arrays
    RET_IF(plan->g_cnt.need(sizeof(int64_t) * (R + 1)));
    int64_t *dcnt = plan->g_cnt.as<int64_t>();
    CK(cudaMemcpyAsync(dcnt + R, &n_src_local, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    NC(g_nccl.AllGather(dcnt + R, dcnt, 1, ncclInt64, plan->comm, st));
    std::vector<int64_t> cnt((size_t)R), off((size_t)R + 1, 0);
    CK(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int r = 0; r < R; ++r) off[r + 1] = off[r] + cnt[r];
    const int64_t ns = off[R];
    if (ns > INT32_MAX) {
        set_err("cylfmm_fmm_solve_dist: %lld sources in total", (long long)ns);
        return CYLFMM_EINVAL;
    }
    RET_IF(plan->g_r.need(8 * (size_t)std::max<int64_t>(ns, 1)));
    RET_IF(plan->g_z.need(8 * (size_t)std::max<int64_t>(ns, 1)));
    RET_IF(plan->g_S.need(16 * (size_t)std::max<int64_t>(ns, 1) * K));
    double *gr = plan->g_r.as<double>(), *gz = plan->g_z.as<double>(), *gS = plan->g_S.as<double>();
    Phases T{plan, timings != nullptr || plan->prof_on, {}};
    if (timings) {
        plan->marks.clear();
        plan->evused = 0;
    }
    T.beg(PH_ALLGATHER, st);
    NC(g_nccl.GroupStart());
    for (int r = 0; r < R; ++r) {
        if (cnt[r] == 0) continue;
        const bool me = r == plan->rank;
        NC(g_nccl.Broadcast(me ? src_r : gr + off[r], gr + off[r], cnt[r], ncclFloat64, r, plan->comm, st));
        NC(g_nccl.Broadcast(me ? src_z : gz + off[r], gz + off[r], cnt[r], ncclFloat64, r, plan->comm, st));
        NC(g_nccl.Broadcast(me ? src_S : gS + 2 * off[r] * K, gS + 2 * off[r] * K, 2 * cnt[r] * K,
                            ncclFloat64, r, plan->comm, st));
    }
    NC(g_nccl.GroupEnd());
    T.end(PH_ALLGATHER, st);
    // the gathered-source marks stay in the plan's list: the solve adds its own (a timings
    // solve keeps them, see fmm_solve_impl) and the moment broadcasts
    return fmm_solve_impl(plan, gr, gz, gS, ns, fld_r, fld_z, n_fld_local, out_Phi, st, timings,
                          nullptr, nullptr, nullptr, true);
}

// ------------------------------------------------------------------------------------------
// host-side field partition for multi-GPU solves (include/cylfmm.h)
static inline uint32_t host_morton(uint32_t ix, uint32_t iz)
{
    uint32_t k = 0;
    for (int b = 0; b < 16; ++b) k |= ((ix >> b) & 1u) << (2 * b) | ((iz >> b) & 1u) << (2 * b + 1);
    return k;
}
static inline bool host_box(double r, double z, int d, double L, double z0, uint32_t &ix, uint32_t &iz)
{
    if (!(r > 0.0) || !(r <= L) || !(z >= z0) || !(z <= z0 + L)) return false;
    const double nb = (double)(1u << d);
    uint32_t i = (uint32_t)std::floor(r * nb / L), j = (uint32_t)std::floor((z - z0) * nb / L);
    const uint32_t m = (1u << d) - 1u;
    ix = std::min(i, m);
    iz = std::min(j, m);
    return true;
}

extern "C" cylfmm_status cylfmm_partition_fields(const double *src_r, const double *src_z,
                                                 int64_t n_src, const double *fld_r,
                                                 const double *fld_z, int64_t n_fld,
                                                 const cylfmm_params *prm, int n_parts,
                                                 int32_t *part, double *part_cost)
{
    if (!prm || n_parts < 1 || n_src < 0 || n_fld < 0 || (n_src > 0 && (!src_r || !src_z)) ||
        (n_fld > 0 && (!fld_r || !fld_z || !part)) || prm->depth < 2 ||
        prm->depth > CYLFMM_MAX_DEPTH || prm->order < 1 || prm->n_modes < 1 || !(prm->domain_L > 0.0)) {
        set_err("cylfmm_partition_fields: bad arguments");
        return CYLFMM_EINVAL;
    }
    const int d = prm->depth, nb = 1 << d, K = prm->n_modes, p = prm->order;
    const double L = prm->domain_L, z0 = prm->domain_z0, P = (p + 1) * (p + 2) / 2.0;
    const size_t nleaf = (size_t)nb * nb;
    std::vector<int64_t> ns(nleaf, 0), nt(nleaf, 0);
    std::vector<uint32_t> fkey((size_t)n_fld);
    for (int64_t i = 0; i < n_src; ++i) {
        uint32_t ix, iz;
        if (!host_box(src_r[i], src_z[i], d, L, z0, ix, iz)) {
            set_err("cylfmm_partition_fields: source %lld outside the domain", (long long)i);
            return CYLFMM_EDOMAIN;
        }
        ns[host_morton(ix, iz)]++;
    }
    for (int64_t j = 0; j < n_fld; ++j) {
        uint32_t ix, iz;
        if (!host_box(fld_r[j], fld_z[j], d, L, z0, ix, iz)) {
            set_err("cylfmm_partition_fields: field point %lld outside the domain", (long long)j);
            return CYLFMM_EDOMAIN;
        }
        fkey[j] = host_morton(ix, iz);
        nt[fkey[j]]++;
    }
    // cost per target leaf, in Morton order
    std::vector<double> cost(nleaf, 0.0);
    const double wpair = 200.0 + 9.0 * K, wl2p = 4.0 * P * K, ws2l = 4.0 * P * P * K;
    for (int ix = 0; ix < nb; ++ix)
        for (int iz = 0; iz < nb; ++iz) {
            const uint32_t k = host_morton((uint32_t)ix, (uint32_t)iz);
            if (!nt[k]) continue;
            double near = 0.0, far = 0.0;
            for (int a = -1; a <= 1; ++a)
                for (int c = -1; c <= 1; ++c) {
                    int x = ix + a, z = iz + c;
                    if (x >= 0 && z >= 0 && x < nb && z < nb)
                        near += (double)ns[host_morton((uint32_t)x, (uint32_t)z)];
                }
            // S2L list at the leaf level: children of the parent's neighbours, not neighbours
            const int px = ix >> 1, pz = iz >> 1;
            for (int x = 2 * px - 2; x <= 2 * px + 3; ++x)
                for (int z = 2 * pz - 2; z <= 2 * pz + 3; ++z) {
                    if (x < 0 || z < 0 || x >= nb || z >= nb) continue;
                    if (std::abs(x - ix) <= 1 && std::abs(z - iz) <= 1) continue;
                    if (ns[host_morton((uint32_t)x, (uint32_t)z)]) far += ws2l;
                }
            cost[k] = (double)nt[k] * (near * wpair + wl2p) + far;
        }
    // the ancestors' S2L (levels 2..d-1), shared among a box's target leaves by field count
    for (int l = 2; l < d; ++l) {
        const int nbl = 1 << l, sh = 2 * (d - l);
        std::vector<int64_t> nsl((size_t)nbl * nbl, 0), ntl((size_t)nbl * nbl, 0);
        for (size_t k = 0; k < nleaf; ++k) {
            nsl[k >> sh] += ns[k];
            ntl[k >> sh] += nt[k];
        }
        std::vector<double> share((size_t)nbl * nbl, 0.0);   // S2L flops per field point
        for (int ix = 0; ix < nbl; ++ix)
            for (int iz = 0; iz < nbl; ++iz) {
                const uint32_t k = host_morton((uint32_t)ix, (uint32_t)iz);
                if (!ntl[k]) continue;
                int pairs = 0;
                const int px = ix >> 1, pz = iz >> 1;
                for (int x = 2 * px - 2; x <= 2 * px + 3; ++x)
                    for (int z = 2 * pz - 2; z <= 2 * pz + 3; ++z) {
                        if (x < 0 || z < 0 || x >= nbl || z >= nbl) continue;
                        if (std::abs(x - ix) <= 1 && std::abs(z - iz) <= 1) continue;
                        if (nsl[host_morton((uint32_t)x, (uint32_t)z)]) ++pairs;
                    }
                share[k] = pairs * ws2l / (double)ntl[k];
            }
        for (size_t k = 0; k < nleaf; ++k)
            if (nt[k]) cost[k] += share[k >> sh] * (double)nt[k];
    }
    double total = 0.0;
    for (double c : cost) total += c;
    // contiguous Morton ranges: leaf k goes to part floor(n_parts * (prefix before k + c/2) / total)
    std::vector<int32_t> leaf_part(nleaf, 0);
    std::vector<double> pc((size_t)n_parts, 0.0);
    double acc = 0.0;
    for (size_t k = 0; k < nleaf; ++k) {
        int q = total > 0.0 ? (int)((acc + 0.5 * cost[k]) / total * n_parts) : 0;
        q = std::min(std::max(q, 0), n_parts - 1);
        leaf_part[k] = q;
        pc[(size_t)q] += cost[k];
        acc += cost[k];
    }
    for (int64_t j = 0; j < n_fld; ++j) part[j] = leaf_part[fkey[j]];
    if (part_cost)
        for (int q = 0; q < n_parts; ++q) part_cost[q] = pc[(size_t)q];
    return CYLFMM_OK;
}

// ------------------------------------------------------------------------------------------
// host-side error-driven order and depth selection (include/cylfmm.h, R#25)
namespace {
// round-1 measured fractions of the FP64 peak: near field ~0.12,
// S2L GEMM ~0.3, tensor seeds + fill ~0.05; F64 nominal 37.2 TF/s
constexpr double kEffNear = 0.12, kEffS2L = 0.30, kEffTens = 0.05, kF64 = 37.2e12;
}

extern "C" cylfmm_status cylfmm_select_params(const double *src_r, const double *src_z,
                                              int64_t n_src, const double *fld_r,
                                              const double *fld_z, int64_t n_fld, double tol,
                                              int depth_min, int depth_max, cylfmm_params *prm,
                                              int64_t *near_pairs, int64_t *s2l_pairs,
                                              double *est_ms, double *eps_model)
{
    if (!prm || !(tol > 0.0) || !std::isfinite(tol) || depth_min > depth_max || n_src < 0 ||
        n_fld < 0 || (n_src > 0 && (!src_r || !src_z)) || (n_fld > 0 && (!fld_r || !fld_z)) ||
        prm->n_modes < 1 || prm->n_modes > CYLFMM_MAX_MODES || !(prm->domain_L > 0.0) ||
        !std::isfinite(prm->domain_L) || !std::isfinite(prm->domain_z0)) {
        set_err("cylfmm_select_params: bad arguments");
        return CYLFMM_EINVAL;
    }
    const int K = prm->n_modes;
    const double L = prm->domain_L, z0 = prm->domain_z0;
    // order: smallest p with CYLFMM_EPS_C 10^(-0.4 p) <= tol
    int p = 1;
    while (p < CYLFMM_MAX_ORDER && CYLFMM_EPS_C * std::pow(10.0, -0.4 * p) > tol) ++p;
    const double P = (p + 1) * (p + 2) / 2.0;
    const int d0 = std::max(depth_min, 2), d1 = std::min(depth_max, CYLFMM_MAX_DEPTH);
    const int nd = depth_max - depth_min + 1;
    if (d0 > d1) {
        set_err("cylfmm_select_params: no depth in [%d, %d] within [2, %d]", depth_min, depth_max,
                CYLFMM_MAX_DEPTH);
        return CYLFMM_EINVAL;
    }
    // finest-level box of every point (Morton key at d1); coarser keys by shifting
    const int D = d1;
    std::vector<uint32_t> skey((size_t)n_src), fkey((size_t)n_fld);
    for (int64_t i = 0; i < n_src; ++i) {
        uint32_t ix, iz;
        if (!host_box(src_r[i], src_z[i], D, L, z0, ix, iz)) {
            set_err("cylfmm_select_params: source %lld outside the domain", (long long)i);
            return CYLFMM_EDOMAIN;
        }
        skey[i] = host_morton(ix, iz);
    }
    for (int64_t j = 0; j < n_fld; ++j) {
        uint32_t ix, iz;
        if (!host_box(fld_r[j], fld_z[j], D, L, z0, ix, iz)) {
            set_err("cylfmm_select_params: field point %lld outside the domain", (long long)j);
            return CYLFMM_EDOMAIN;
        }
        fkey[j] = host_morton(ix, iz);
    }
    // per level l = 2..D: source / target counts per box (dense, Morton-indexed), the level's
    // S2L pair count, and (l in [d0, d1]) the near-pair count with leaves at level l
    std::vector<int64_t> s2l_lev((size_t)D + 1, 0), near_lev((size_t)D + 1, 0);
    std::vector<int64_t> ns, nt;
    for (int l = 2; l <= D; ++l) {
        const int nb = 1 << l, sh = 2 * (D - l);
        ns.assign((size_t)nb * nb, 0);
        nt.assign((size_t)nb * nb, 0);
        for (uint32_t k : skey) ns[k >> sh]++;
        for (uint32_t k : fkey) nt[k >> sh]++;
        int64_t s2l = 0, near = 0;
        for (int ix = 0; ix < nb; ++ix)
            for (int iz = 0; iz < nb; ++iz) {
                const int64_t t = nt[host_morton((uint32_t)ix, (uint32_t)iz)];
                if (!t) continue;
                // interaction list: children of the parent's neighbours that are not neighbours
                const int px = ix >> 1, pz = iz >> 1;
                for (int x = 2 * px - 2; x <= 2 * px + 3; ++x)
                    for (int z = 2 * pz - 2; z <= 2 * pz + 3; ++z) {
                        if (x < 0 || z < 0 || x >= nb || z >= nb) continue;
                        if (std::abs(x - ix) <= 1 && std::abs(z - iz) <= 1) continue;
                        if (ns[host_morton((uint32_t)x, (uint32_t)z)]) ++s2l;
                    }
                if (l < d0) continue;
                int64_t s9 = 0;
                for (int a = -1; a <= 1; ++a)
                    for (int c = -1; c <= 1; ++c) {
                        const int x = ix + a, z = iz + c;
                        if (x >= 0 && z >= 0 && x < nb && z < nb)
                            s9 += ns[host_morton((uint32_t)x, (uint32_t)z)];
                    }
                near += t * s9;
            }
        s2l_lev[l] = s2l;
        near_lev[l] = near;
    }
    int best = -1;
    double best_ms = 0.0;
    const double wpair = (200.0 + 9.0 * K) / kEffNear, ws2l = 4.0 * P * P * K / kEffS2L;
    const double wtens = 12.0 * K * (12.0 * (2 * p + 1) * (2 * p + 1) + 12.0 * (p + 1) * (p + 1) * (p + 1)) / kEffTens;
    int64_t s2l_cum = 0;
    for (int d = 2; d <= D; ++d) {
        s2l_cum += s2l_lev[d];
        if (d < d0 || d > d1) continue;
        const double ms = 1e3 * ((double)near_lev[d] * wpair + (double)s2l_cum * ws2l +
                                 (double)(1 << d) * wtens) / kF64;
        const int q = d - depth_min;
        if (near_pairs) near_pairs[q] = near_lev[d];
        if (s2l_pairs) s2l_pairs[q] = s2l_cum;
        if (est_ms) est_ms[q] = ms;
        if (best < 0 || ms < best_ms) {
            best = d;
            best_ms = ms;
        }
    }
    for (int q = 0; q < nd; ++q) {
        const int d = depth_min + q;
        if (d >= d0 && d <= d1) continue;
        if (near_pairs) near_pairs[q] = -1;
        if (s2l_pairs) s2l_pairs[q] = -1;
        if (est_ms) est_ms[q] = -1.0;
    }
    prm->order = p;
    prm->order_local = 0;
    prm->depth = best;
    if (eps_model) *eps_model = CYLFMM_EPS_C * std::pow(10.0, -0.4 * p);
    return CYLFMM_OK;
}
