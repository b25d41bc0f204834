// tree.cuh -- uniform quadtree on [0, L] x [z0, z0 + L] (R#11).
//   leaf box (ix, iz) = (min(floor(r 2^d / L), 2^d - 1), min(floor((z - z0) 2^d / L), 2^d - 1)),
//   key = Morton interleave with the radial index in the even bits;
//   points sorted by a stable LSD radix sort (8-bit digits, 2048-key tiles, stable in-tile ranks
//   from warp match_any), so every level-l box owns a contiguous range of sorted points.
//   Dense leaf starts (lower_bound per leaf key) give every box range by index arithmetic;
//   per-level occupancy maps (dense key -> compact slot, -1 empty) come from an exclusive scan.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cyl {

__global__ void keys_kernel(const double *r, const double *z, int64_t n, int depth, double L,
                            double z0, uint32_t *key, int *idx, int *err)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double nb = (double)(1u << depth);
    double rr = r[i], zz = z[i];
    if (!(rr > 0.0) || !(rr <= L) || !(zz >= z0) || !(zz <= z0 + L)) atomicOr(err, 4);
    double fi = floor(rr * nb / L), fj = floor((zz - z0) * nb / L);
    fi = fmin(fmax(fi, 0.0), nb - 1.0);   // fmax maps NaN to 0 (flagged above)
    fj = fmin(fmax(fj, 0.0), nb - 1.0);
    uint32_t ix = (uint32_t)fi, iz = (uint32_t)fj;
    auto spread = [](uint32_t v) {
        v &= 0xffffu;
        v = (v | (v << 8)) & 0x00ff00ffu;
        v = (v | (v << 4)) & 0x0f0f0f0fu;
        v = (v | (v << 2)) & 0x33333333u;
        v = (v | (v << 1)) & 0x55555555u;
        return v;
    };
    key[i] = spread(ix) | (spread(iz) << 1);
    idx[i] = (int)i;
}

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                         // keys per thread for large inputs
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
// keys per thread: 4 for small inputs (16k keys: 16 CTAs of 4 serial rounds instead of 8 of 8;
// measured on the C2 step: 1 and 2 keys per thread are slower, the histogram scan grows), else 8
inline int sort_items(int64_t n) { return n <= 65536 ? 4 : kSortItems; }

__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint32_t *key, int64_t n,
                                                                  int shift, int ntiles,
                                                                  int *hist, int items)
{
    __shared__ int cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortThreads * items;
    for (int k = 0; k < items; ++k) {
        int64_t i = base + k * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(key[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const uint32_t *key_in, const int *val_in, int64_t n, int shift, int ntiles,
    const int *offsets, uint32_t *key_out, int *val_out, int items)
{
    __shared__ int wcount[kSortThreads / 32][257];
    __shared__ int running[256];
    __shared__ int base[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    running[tid] = 0;
    base[tid] = offsets[(int64_t)tid * ntiles + blockIdx.x];
    const int64_t tbase = (int64_t)blockIdx.x * kSortThreads * items;
    for (int rnd = 0; rnd < items; ++rnd) {
        for (int e = tid; e < (kSortThreads / 32) * 257; e += kSortThreads) (&wcount[0][0])[e] = 0;
        __syncthreads();
        int64_t i = tbase + rnd * kSortThreads + tid;
        bool valid = i < n;
        uint32_t k = valid ? key_in[i] : 0u;
        int v = valid ? val_in[i] : 0;
        int digit = valid ? (int)((k >> shift) & 255u) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, digit);
        int rank = __popc(peers & ((1u << lane) - 1u));
        if (rank == 0) wcount[warp][digit] = __popc(peers);
        __syncthreads();
        {
            int acc = running[tid];
            for (int w = 0; w < kSortThreads / 32; ++w) {
                int c = wcount[w][tid];
                wcount[w][tid] = acc;
                acc += c;
            }
            running[tid] = acc;
        }
        __syncthreads();
        if (valid) {
            int pos = base[digit] + wcount[warp][digit] + rank;
            key_out[pos] = k;
            val_out[pos] = v;
        }
        __syncthreads();
    }
}

// ---- exclusive scan of int arrays (3-phase, recursive on block sums) ----
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *sh, T &total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < (int)(blockDim.x / 32) ? sh[lane] : 0;
        T ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        sh[lane] = ws - w;
        if (lane == 31) sh[32] = ws;
    }
    __syncthreads();
    T res = sh[warp] + x - v;
    total = sh[32];
    __syncthreads();
    return res;
}

// out[i] = sum_{k<i} in[i]; sums[b] = tile total.  in may equal out.  T = int or int64_t.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(const T *in, int64_t n, T *out,
                                                                 T *sums)
{
    __shared__ T sh[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T v[kScanItems], s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    T total;
    T pre = block_excl_scan(s, sh, total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = pre;
        pre += v[k];
    }
    if (threadIdx.x == 0 && sums) sums[blockIdx.x] = total;
}

template <typename T>
__global__ void scan_add_kernel(T *out, int64_t n, const T *offs)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += offs[i / kScanTile];
}

// ---- leaf starts and level maps ----
// lstart[k] = first sorted index with key >= k, k = 0..nleaf (nleaf = 4^d).
__global__ void leaf_start_kernel(const uint32_t *skey, int64_t n, int64_t nleaf, int *lstart)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > nleaf) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)skey[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    lstart[k] = (int)lo;
}

// flags[b] = box b of level l non-empty (b in [0, 4^l))
// A box of the tree at `level`: non-empty and, for the adaptive source tree (sigma > 0, R#26),
// below no leaf (level 2, or the parent holds > sigma points).  Boxes below a source leaf take
// part in nothing (no moments, no S2L), so they get no slot.
__device__ __forceinline__ bool box_in_tree(const int *lstart, int depth, int level, int64_t b,
                                            int sigma)
{
    const int sh = 2 * (depth - level);
    if (lstart[(b + 1) << sh] <= lstart[b << sh]) return false;
    if (sigma > 0 && level > 2) {
        const int64_t pb = b >> 2;
        return lstart[(pb + 1) << (sh + 2)] - lstart[pb << (sh + 2)] > sigma;
    }
    return true;
}

__global__ void level_flags_kernel(const int *lstart, int depth, int level, int sigma, int *flags)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nbox = (int64_t)1 << (2 * level);
    if (b >= nbox) return;
    flags[b] = box_in_tree(lstart, depth, level, b, sigma) ? 1 : 0;
}

// map[b] = slot or -1; keys[slot] = b; count written by the last box.
__global__ void level_map_kernel(const int *lstart, int depth, int level, int sigma, const int *scan,
                                 int *map, int *keys, int *count)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nbox = (int64_t)1 << (2 * level);
    if (b >= nbox) return;
    bool ne = box_in_tree(lstart, depth, level, b, sigma);
    int s = scan[b];
    map[b] = ne ? s : -1;
    if (ne) keys[s] = (int)b;
    if (b == nbox - 1) *count = s + (ne ? 1 : 0);
}

// largest radial box index among the non-empty boxes of a level (stations beyond it are unused)
// out = scan[n-1] + flag[n-1] (the total of an exclusive scan of 0/1 flags)
__global__ void count_total_kernel(const int *scan, const unsigned char *flag, int64_t n, int *out)
{
    if (threadIdx.x == 0) *out = n > 0 ? scan[n - 1] + (flag[n - 1] ? 1 : 0) : 0;
}

// *out = scan[n-1] + flag[n-1] for int flags
__global__ void l2p_ntasks_kernel(const int *scan, const int *flag, int64_t n, int *out)
{
    if (threadIdx.x == 0) *out = n > 0 ? scan[n - 1] + flag[n - 1] : 0;
}

__global__ void max_col_kernel(const int *keys, const int *count, int *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *count) return;
    uint32_t v = (uint32_t)keys[i] & 0x55555555u;   // radial bits (even positions)
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0f0f0f0fu;
    v = (v | (v >> 4)) & 0x00ff00ffu;
    v = (v | (v >> 8)) & 0x0000ffffu;
    atomicMax(out, (int)v);
}

// Level maps of the small levels (4^l <= 4096) for both point sets in ONE launch: CTA per
// (side, level), flags + block-wide exclusive scan in shared memory (replaces the per-level
// flags / scan / map launches, which dominate the tree phase of small problems such as C2).
constexpr int kSmallLevelBoxes = 4096;
struct SmallLevelArgs {
    const int *ls[2];          // dense leaf starts per side
    int *map[2], *keys[2];     // dense level maps / compact key lists (level offsets below)
    int *count[2];             // per side: count[l]
    int64_t lvoff[17];
    int depth, lmin, nlev;     // levels lmin .. lmin + nlev - 1
    int sigma[2];              // per side: adaptive leaf size (box_in_tree), 0 = uniform
};
__global__ void __launch_bounds__(1024) level_maps_small_kernel(SmallLevelArgs a)
{
    __shared__ int wsum[32];
    const int side = blockIdx.x / a.nlev, level = a.lmin + blockIdx.x % a.nlev;
    const int nbox = 1 << (2 * level);
    const int *ls = a.ls[side];
    int *map = a.map[side] + a.lvoff[level], *keys = a.keys[side] + a.lvoff[level];
    constexpr int PER = kSmallLevelBoxes / 1024;
    const int b0 = threadIdx.x * PER;
    int f[PER], c = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = b0 + k;
        f[k] = b < nbox && box_in_tree(ls, a.depth, level, b, a.sigma[side]);
        c += f[k];
    }
    // block exclusive scan of c
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = c;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;   // inclusive per warp
    }
    __syncthreads();
    int pos = x - c + (w > 0 ? wsum[w - 1] : 0);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = b0 + k;
        if (b >= nbox) break;
        map[b] = f[k] ? pos : -1;
        if (f[k]) keys[pos++] = b;
    }
    if (threadIdx.x == 1023) a.count[side][level] = wsum[31];
}

template <typename T>
__global__ void gather_kernel(const T *in, const int *perm, int64_t n, T *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[perm[i]];
}

// rows of K complex values: out[i][:] = in[perm[i]][:]
__global__ void gather_rows_kernel(const double2 *in, const int *perm, int64_t n, int K,
                                   double2 *out)
{
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * K) return;
    int64_t i = e / K;
    int k = (int)(e - i * K);
    out[e] = in[(int64_t)perm[i] * K + k];
}

// sorted copies of a point set in one pass: r, z (and the coefficient rows when S != nullptr)
__global__ void gather_points_kernel(const double *r, const double *z, const double2 *S,
                                     const int *perm, int64_t n, int K, double *rs, double *zs,
                                     double2 *Ss)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) {
        const int pi = perm[e];
        rs[e] = r[pi];
        zs[e] = z[pi];
    }
    if (S && e < n * K) {
        const int64_t i = e / K;
        const int k = (int)(e - i * K);
        Ss[e] = S[(int64_t)perm[i] * K + k];
    }
}

}  // namespace cyl
