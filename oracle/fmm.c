/*
 * fmm.c -- oracle reference FMM, Algorithm 1 of the paper step by step.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 *   tree:      uniform quadtree on [0,L] x [z0,z0+L], 2^l x 2^l boxes at level l,
 *              box index min(floor(coord * 2^l / L), 2^l - 1) (R#11), Morton key with the
 *              radial index in the even bits.
 *   P2M:       S_ij = sum_q S_q (dr_q)^i (dz_q)^j about the leaf centre.
 *   M2M:       S_ij = sum C(i,q) C(j,u) D_r^q D_z^u S'_{i-q,j-u}, D = child - parent (R#9).
 *   S2L:       Phi_kl += sum_ij sigma C(j+l,j) S_ij Gbar_{A,B,j+l} with the FO/BO/FI/BI variant
 *              and the tensor at (outer centre, inner centre, |dz|) (R#8, R#10).
 *   L2L:       Phi_ij = sum C(i+q,q) C(j+u,u) D_r^q D_z^u Phi'_{i+q,j+u}, D = child - parent.
 *   L2P:       Phi(r,z) += sum Phi_kl (r-r_c)^k (z-z_c)^l.
 *   near:      direct sum over the 9 neighbour leaves, coincident pairs skipped.
 * Every ordered (source box, target box) pair computes its own tensor (no 12-class reuse).
 *
 * Adaptive source tree (reading R#26; leaf_src = sigma > 0): a source box with
 * <= sigma sources is a leaf, its subtree is not descended.  An ordered pair of adjacent boxes
 * (T, S) at level l whose parent pair was descended (l = 2, or S's parent holds > sigma sources)
 * is evaluated directly when S is a leaf or l = d: every target of T against every source of S
 * (P:647-651 applied at level l).  An S2L pair at level l > 2 exists only if S's
 * parent holds > sigma sources (otherwise the parent pair was evaluated directly).  Every
 * (target, source) pair is then covered exactly once, by the first level at which its boxes
 * separate or its source box becomes a leaf; sigma = 0 is the uniform tree above, operation for
 * operation.  Only the paper's operators are used (same-level S2L, M2M, L2L, L2P, direct sum).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "oracle.h"

static int tri_idx(int i, int j, int p) { return i * (p + 1) - i * (i - 1) / 2 + j; }
static int tri_size(int p) { return (p + 1) * (p + 2) / 2; }

static double binom(int n, int k)
{
    if (k < 0 || k > n) return 0.0;
    double b = 1.0;
    for (int i = 1; i <= k; ++i) b = b * (n - k + i) / i;
    return b;
}

static uint32_t morton(uint32_t ix, uint32_t iz)
{
    uint32_t key = 0;
    for (int b = 0; b < 16; ++b) {
        key |= ((ix >> b) & 1u) << (2 * b);
        key |= ((iz >> b) & 1u) << (2 * b + 1);
    }
    return key;
}

static void box_of(double r, double z, int level, double L, double z0, uint32_t *ix, uint32_t *iz)
{
    double nb = (double)(1u << level);
    double fi = floor(r * nb / L), fj = floor((z - z0) * nb / L);
    if (fi > nb - 1) fi = nb - 1;
    if (fj > nb - 1) fj = nb - 1;
    if (fi < 0) fi = 0;
    if (fj < 0) fj = 0;
    *ix = (uint32_t)fi;
    *iz = (uint32_t)fj;
}

typedef struct { uint32_t key; int64_t idx; } kv_t;
static int kv_cmp(const void *a, const void *b)
{
    const kv_t *x = (const kv_t *)a, *y = (const kv_t *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

void or_tree_keys(const double *r, const double *z, int64_t n, int depth, double L, double z0,
                  uint32_t *key, int64_t *perm)
{
    kv_t *kv = (kv_t *)malloc(sizeof(kv_t) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        uint32_t ix, iz;
        box_of(r[i], z[i], depth, L, z0, &ix, &iz);
        key[i] = morton(ix, iz);
        kv[i].key = key[i];
        kv[i].idx = i;
    }
    qsort(kv, (size_t)n, sizeof(kv_t), kv_cmp);
    for (int64_t i = 0; i < n; ++i) perm[i] = kv[i].idx;
    free(kv);
}

void or_p2m(const double *r, const double *z, const double *S, int64_t n, int nmodes, int p,
            double rc, double zc, double *M)
{
    int P = tri_size(p);
    for (int64_t q = 0; q < n; ++q) {
        double dr = r[q] - rc, dz = z[q] - zc;
        for (int i = 0; i <= p; ++i)
            for (int j = 0; i + j <= p; ++j) {
                double mono = pow(dr, i) * pow(dz, j);
                for (int m = 0; m < nmodes; ++m) {
                    M[2 * ((size_t)m * P + tri_idx(i, j, p))] += S[2 * (q * nmodes + m)] * mono;
                    M[2 * ((size_t)m * P + tri_idx(i, j, p)) + 1] += S[2 * (q * nmodes + m) + 1] * mono;
                }
            }
    }
}

void or_m2m(const double *Mc, int nmodes, int p, double dr, double dz, double *Mp)
{
    int P = tri_size(p);
    for (int m = 0; m < nmodes; ++m)
        for (int i = 0; i <= p; ++i)
            for (int j = 0; i + j <= p; ++j) {
                double re = 0.0, im = 0.0;
                for (int q = 0; q <= i; ++q)
                    for (int u = 0; u <= j; ++u) {
                        double c = binom(i, q) * binom(j, u) * pow(dr, q) * pow(dz, u);
                        const double *s = Mc + 2 * ((size_t)m * P + tri_idx(i - q, j - u, p));
                        re += c * s[0];
                        im += c * s[1];
                    }
                Mp[2 * ((size_t)m * P + tri_idx(i, j, p))] += re;
                Mp[2 * ((size_t)m * P + tri_idx(i, j, p)) + 1] += im;
            }
}

void or_l2l(const double *Lp, int nmodes, int p, double dr, double dz, double *Lc)
{
    int P = tri_size(p);
    for (int m = 0; m < nmodes; ++m)
        for (int i = 0; i <= p; ++i)
            for (int j = 0; i + j <= p; ++j) {
                double re = 0.0, im = 0.0;
                for (int q = 0; i + q + j <= p; ++q)
                    for (int u = 0; i + q + j + u <= p; ++u) {
                        double c = binom(i + q, q) * binom(j + u, u) * pow(dr, q) * pow(dz, u);
                        const double *s = Lp + 2 * ((size_t)m * P + tri_idx(i + q, j + u, p));
                        re += c * s[0];
                        im += c * s[1];
                    }
                Lc[2 * ((size_t)m * P + tri_idx(i, j, p))] += re;
                Lc[2 * ((size_t)m * P + tri_idx(i, j, p)) + 1] += im;
            }
}

/* gradient of the local expansion at (r, z): d/dr and d/dz of sum Phi_kl dr^k dz^l */
void or_l2p_grad(const double *Lc, int nmodes, int p, double rc, double zc, double r, double z,
                 double *gr, double *gz)
{
    int P = tri_size(p);
    double dr = r - rc, dz = z - zc;
    for (int m = 0; m < nmodes; ++m)
        for (int k = 0; k <= p; ++k)
            for (int l = 0; k + l <= p; ++l) {
                double mr = k > 0 ? k * pow(dr, k - 1) * pow(dz, l) : 0.0;
                double mz = l > 0 ? l * pow(dr, k) * pow(dz, l - 1) : 0.0;
                const double *c = Lc + 2 * ((size_t)m * P + tri_idx(k, l, p));
                gr[2 * m] += c[0] * mr;
                gr[2 * m + 1] += c[1] * mr;
                gz[2 * m] += c[0] * mz;
                gz[2 * m + 1] += c[1] * mz;
            }
}

void or_l2p(const double *Lc, int nmodes, int p, double rc, double zc, double r, double z,
            double *phi)
{
    int P = tri_size(p);
    double dr = r - rc, dz = z - zc;
    for (int m = 0; m < nmodes; ++m)
        for (int k = 0; k <= p; ++k)
            for (int l = 0; k + l <= p; ++l) {
                double mono = pow(dr, k) * pow(dz, l);
                phi[2 * m] += Lc[2 * ((size_t)m * P + tri_idx(k, l, p))] * mono;
                phi[2 * m + 1] += Lc[2 * ((size_t)m * P + tri_idx(k, l, p)) + 1] * mono;
            }
}

int or_s2l(const double *M, int nmodes, int p, int pl, double rs, double zs, double rt,
           double zt, int truncation, int miller, double *Lacc)
{
    /* p: source (moment) order, pl: local order (they may differ); the tensor is
     * computed to a, b <= max(p, pl), a + b + c <= 2 max(p, pl), which contains every entry
     * the double-truncated operator reads (A, B <= max, c = j + l <= p + pl - A - B) */
    int P = tri_size(p), Pl = tri_size(pl), pt = p > pl ? p : pl;
    int outward = rt >= rs;       /* target at equal or larger radius: FO/BO (R#10) */
    int forward = zt >= zs;       /* target at equal or larger z: FO/FI */
    double r = outward ? rt : rs; /* tensor at r >= r1, x >= 0 */
    double r1 = outward ? rs : rt;
    double x = fabs(zt - zs);
    int D = 2 * pt + 1;
    size_t tsz = (size_t)nmodes * (pt + 1) * (pt + 1) * D;
    double *T = (double *)malloc(sizeof(double) * tsz);
    if (!T) return -1;
    if (or_tensor(r, r1, x, nmodes - 1, pt, miller, T) != 0) {
        free(T);
        return -1;
    }
    for (int m = 0; m < nmodes; ++m)
        for (int k = 0; k <= pl; ++k)
            for (int l = 0; k + l <= pl; ++l) {
                double re = 0.0, im = 0.0;
                for (int i = 0; i <= p; ++i)
                    for (int j = 0; i + j <= p; ++j) {
                        if (truncation == OR_TRUNC_SINGLE && i + j + k + l > p) continue;
                        double sigma = forward ? ((j & 1) ? -1.0 : 1.0) : ((l & 1) ? -1.0 : 1.0);
                        int a = outward ? k : i, b = outward ? i : k;
                        double g = T[(((size_t)m * (pt + 1) + a) * (pt + 1) + b) * D + (j + l)];
                        double c = sigma * binom(j + l, j) * g;
                        const double *s = M + 2 * ((size_t)m * P + tri_idx(i, j, p));
                        re += c * s[0];
                        im += c * s[1];
                    }
                Lacc[2 * ((size_t)m * Pl + tri_idx(k, l, pl))] += re;
                Lacc[2 * ((size_t)m * Pl + tri_idx(k, l, pl)) + 1] += im;
            }
    free(T);
    return 0;
}

/* --------------------------------------------------------------------------------------- */

typedef struct {
    int level;
    int32_t *map;   /* dense Morton key -> compact slot, -1 = empty */
    int64_t count;
    uint32_t *keys; /* compact slot -> Morton key (ascending) */
    double *data;   /* [count][nmodes][P] complex */
} level_t;

static void level_free(level_t *lv)
{
    free(lv->map);
    free(lv->keys);
    free(lv->data);
}

/* Build the compact set of boxes at `level` from sorted leaf keys (ascending). */
static int level_from_leaf_keys(level_t *lv, int level, int depth, const uint32_t *sorted_keys,
                                int64_t n, size_t per_box)
{
    size_t nbox = (size_t)1 << (2 * level);
    lv->level = level;
    lv->map = (int32_t *)malloc(sizeof(int32_t) * nbox);
    if (!lv->map) return -1;
    for (size_t b = 0; b < nbox; ++b) lv->map[b] = -1;
    int shift = 2 * (depth - level);
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t k = sorted_keys[i] >> shift;
        if (lv->map[k] < 0) lv->map[k] = (int32_t)cnt++;
    }
    lv->count = cnt;
    lv->keys = (uint32_t *)malloc(sizeof(uint32_t) * (cnt > 0 ? cnt : 1));
    lv->data = (double *)calloc((size_t)(cnt > 0 ? cnt : 1) * per_box, sizeof(double));
    if (!lv->keys || !lv->data) return -1;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t k = sorted_keys[i] >> shift;
        lv->keys[lv->map[k]] = k;
    }
    return 0;
}

static void demorton(uint32_t key, uint32_t *ix, uint32_t *iz)
{
    uint32_t a = 0, b = 0;
    for (int bit = 0; bit < 16; ++bit) {
        a |= ((key >> (2 * bit)) & 1u) << bit;
        b |= ((key >> (2 * bit + 1)) & 1u) << bit;
    }
    *ix = a;
    *iz = b;
}

int64_t or_fmm(const double *sr, const double *sz, const double *S, int64_t ns,
               const double *fr, const double *fz, int64_t nf, int nmodes, int p, int pl,
               int depth, double L, double z0, int truncation, int miller, double *Phi,
               double *dPr, double *dPz, int nthreads, int64_t leaf_src)
{
    /* dPr, dPz (nullable, both or neither): the field gradients, from the gradient of the local
     * expansion at the point plus the near field with the derivative relations of G (or_greens_grad) */
    const int grad = dPr != NULL && dPz != NULL;
    if (pl <= 0) pl = p; /* local order defaults to the source order */
    if (depth < 2 || depth > 15 || p < 1 || nmodes < 1 || !(L > 0.0) || leaf_src < 0) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t i = 0; i < ns; ++i)
        if (!(sr[i] > 0.0) || !(sr[i] <= L) || !(sz[i] >= z0) || !(sz[i] <= z0 + L)) return -1;
    for (int64_t j = 0; j < nf; ++j)
        if (!(fr[j] > 0.0) || !(fr[j] <= L) || !(fz[j] >= z0) || !(fz[j] <= z0 + L)) return -1;

    int64_t *scnt[16] = {0}, *sfirst[16] = {0};   /* per level: sources per box, first source */
    int P = tri_size(p), Pl = tri_size(pl);
    size_t per_box = (size_t)2 * nmodes * P;     /* source boxes: moments of order p */
    size_t per_tbox = (size_t)2 * nmodes * Pl;   /* target boxes: locals of order pl */
    int64_t skipped = 0;
    int err = 0;

    /* sort sources and fields by leaf Morton key (Algorithm 1, line 2) */
    uint32_t *skey = (uint32_t *)malloc(sizeof(uint32_t) * (ns > 0 ? ns : 1));
    int64_t *sperm = (int64_t *)malloc(sizeof(int64_t) * (ns > 0 ? ns : 1));
    uint32_t *fkey = (uint32_t *)malloc(sizeof(uint32_t) * (nf > 0 ? nf : 1));
    int64_t *fperm = (int64_t *)malloc(sizeof(int64_t) * (nf > 0 ? nf : 1));
    uint32_t *skey_sorted = (uint32_t *)malloc(sizeof(uint32_t) * (ns > 0 ? ns : 1));
    uint32_t *fkey_sorted = (uint32_t *)malloc(sizeof(uint32_t) * (nf > 0 ? nf : 1));
    or_tree_keys(sr, sz, ns, depth, L, z0, skey, sperm);
    or_tree_keys(fr, fz, nf, depth, L, z0, fkey, fperm);
    for (int64_t i = 0; i < ns; ++i) skey_sorted[i] = skey[sperm[i]];
    for (int64_t j = 0; j < nf; ++j) fkey_sorted[j] = fkey[fperm[j]];

    level_t src[16], tgt[16];
    memset(src, 0, sizeof(src));
    memset(tgt, 0, sizeof(tgt));
    for (int l = 2; l <= depth; ++l) {
        if (level_from_leaf_keys(&src[l], l, depth, skey_sorted, ns, per_box) != 0) err = 1;
        if (level_from_leaf_keys(&tgt[l], l, depth, fkey_sorted, nf, per_tbox) != 0) err = 1;
    }
    /* leaf ranges of sorted sources: start[slot], end[slot] */
    int64_t nleaf = src[depth].count;
    int64_t *lstart = (int64_t *)malloc(sizeof(int64_t) * (nleaf + 1));
    {
        int64_t slot = -1;
        for (int64_t i = 0; i < ns; ++i) {
            int32_t s = src[depth].map[skey_sorted[i]];
            if (s != slot) {
                slot = s;
                lstart[s] = i;
            }
        }
        lstart[nleaf] = ns;
    }
    /* sources per box and first sorted source of each box, every level (a box's sources are
     * contiguous in Morton order) */
    for (int l = 2; l <= depth; ++l) {
        int64_t nb_ = src[l].count > 0 ? src[l].count : 1;
        scnt[l] = (int64_t *)calloc((size_t)nb_, sizeof(int64_t));
        sfirst[l] = (int64_t *)calloc((size_t)nb_, sizeof(int64_t));
        if (!scnt[l] || !sfirst[l]) err = 1;
    }
    if (!err)
        for (int64_t i = 0; i < ns; ++i)
            for (int l = 2; l <= depth; ++l) {
                int32_t s = src[l].map[skey_sorted[i] >> (2 * (depth - l))];
                if (scnt[l][s]++ == 0) sfirst[l][s] = i;
            }
    if (err) goto cleanup;

    double hd = L / (double)(1u << depth);
    /* leaf moments (Algorithm 1, line 3) */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t b = 0; b < nleaf; ++b) {
        uint32_t ix, iz;
        demorton(src[depth].keys[b], &ix, &iz);
        double rc = (ix + 0.5) * hd, zc = z0 + (iz + 0.5) * hd;
        for (int64_t q = lstart[b]; q < lstart[b + 1]; ++q) {
            int64_t i = sperm[q];
            or_p2m(&sr[i], &sz[i], &S[2 * (size_t)i * nmodes], 1, nmodes, p, rc, zc,
                   src[depth].data + (size_t)b * per_box);
        }
    }
    /* upward pass l = d-1..2 (Algorithm 1, lines 5-7): children in Morton order */
    for (int l = depth - 1; l >= 2; --l) {
        double h = L / (double)(1u << l), hc = h / 2.0;
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t b = 0; b < src[l].count; ++b) {
            uint32_t key = src[l].keys[b], ix, iz;
            demorton(key, &ix, &iz);
            double pr = (ix + 0.5) * h, pz = z0 + (iz + 0.5) * h;
            for (uint32_t c = 0; c < 4; ++c) {
                int32_t cs = src[l + 1].map[4 * key + c];
                if (cs < 0) continue;
                uint32_t cx, cz;
                demorton(4 * key + c, &cx, &cz);
                double cr = (cx + 0.5) * hc, czc = z0 + (cz + 0.5) * hc;
                or_m2m(src[l + 1].data + (size_t)cs * per_box, nmodes, p, cr - pr, czc - pz,
                       src[l].data + (size_t)b * per_box);
            }
        }
    }
    /* downward pass l = 2..d (Algorithm 1, lines 9-21) */
    for (int l = 2; l <= depth; ++l) {
        uint32_t nb = 1u << l;
        double h = L / (double)nb;
        int err_l = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err_l)
        for (int64_t b = 0; b < tgt[l].count; ++b) {
            uint32_t key = tgt[l].keys[b], ix, iz;
            demorton(key, &ix, &iz);
            double tr = (ix + 0.5) * h, tz = z0 + (iz + 0.5) * h;
            double *Lb = tgt[l].data + (size_t)b * per_tbox;
            if (l >= 3) { /* shift parent local expansion */
                uint32_t px, pz;
                demorton(key >> 2, &px, &pz);
                double hp = 2.0 * h;
                double pr = (px + 0.5) * hp, pzc = z0 + (pz + 0.5) * hp;
                int32_t ps = tgt[l - 1].map[key >> 2];
                or_l2l(tgt[l - 1].data + (size_t)ps * per_tbox, nmodes, pl, tr - pr, tz - pzc, Lb);
            }
            /* S2L list: children of the parent's neighbours that are not neighbours */
            int px = (int)(ix >> 1), pz = (int)(iz >> 1);
            for (int a = px - 1; a <= px + 1; ++a)
                for (int c = pz - 1; c <= pz + 1; ++c) {
                    if (a < 0 || c < 0 || a >= (int)(nb / 2) || c >= (int)(nb / 2)) continue;
                    for (int ci = 2 * a; ci <= 2 * a + 1; ++ci)
                        for (int cj = 2 * c; cj <= 2 * c + 1; ++cj) {
                            int di = ci - (int)ix, dj = cj - (int)iz;
                            if (abs(di) <= 1 && abs(dj) <= 1) continue;
                            int32_t ss = src[l].map[morton((uint32_t)ci, (uint32_t)cj)];
                            if (ss < 0) continue;
                            /* adaptive: the parent pair was evaluated directly (R#26) */
                            if (leaf_src > 0 && l > 2 &&
                                scnt[l - 1][src[l - 1].map[morton((uint32_t)a, (uint32_t)c)]] <= leaf_src)
                                continue;
                            double sr0 = (ci + 0.5) * h, sz0 = z0 + (cj + 0.5) * h;
                            if (or_s2l(src[l].data + (size_t)ss * per_box, nmodes, p, pl, sr0, sz0,
                                       tr, tz, truncation, miller, Lb) != 0)
                                err_l = 1;
                        }
                }
        }
        if (err_l) err = 1;
    }
    /* leaves: local expansion + direct sum over the 9 neighbour leaves (Algorithm 1, 22-24) */
    {
        uint32_t nb = 1u << depth;
#pragma omp parallel reduction(+ : skipped) reduction(| : err)
        {
            double *G = (double *)malloc(sizeof(double) * 3 * nmodes);
            double *Gr = G + nmodes, *Gx = Gr + nmodes;
#pragma omp for schedule(dynamic, 16)
            for (int64_t j = 0; j < nf; ++j) {
                double *out = Phi + 2 * (size_t)j * nmodes;
                double *outr = grad ? dPr + 2 * (size_t)j * nmodes : NULL;
                double *outz = grad ? dPz + 2 * (size_t)j * nmodes : NULL;
                memset(out, 0, sizeof(double) * 2 * nmodes);
                if (grad) {
                    memset(outr, 0, sizeof(double) * 2 * nmodes);
                    memset(outz, 0, sizeof(double) * 2 * nmodes);
                }
                uint32_t ix, iz;
                demorton(fkey[j], &ix, &iz);
                double rc = (ix + 0.5) * hd, zc = z0 + (iz + 0.5) * hd;
                int32_t ts = tgt[depth].map[fkey[j]];
                or_l2p(tgt[depth].data + (size_t)ts * per_tbox, nmodes, pl, rc, zc, fr[j], fz[j], out);
                if (grad)
                    or_l2p_grad(tgt[depth].data + (size_t)ts * per_tbox, nmodes, pl, rc, zc, fr[j],
                                fz[j], outr, outz);
                /* uniform: the 9 neighbour leaves; adaptive: at every level, the neighbours S of
                 * the target's box whose pair is evaluated directly (R#26) */
                for (int l = leaf_src > 0 ? 2 : depth; l <= depth; ++l) {
                    const int sh = depth - l, nbl = (int)(nb >> sh);
                    const int bx = (int)(ix >> sh), bz = (int)(iz >> sh);
                for (int a = bx - 1; a <= bx + 1; ++a)
                    for (int c = bz - 1; c <= bz + 1; ++c) {
                        if (a < 0 || c < 0 || a >= nbl || c >= nbl) continue;
                        int32_t ls = src[l].map[morton((uint32_t)a, (uint32_t)c)];
                        if (ls < 0) continue;
                        if (leaf_src > 0) {
                            const int active = l == 2 ||
                                scnt[l - 1][src[l - 1].map[morton((uint32_t)a >> 1, (uint32_t)c >> 1)]] > leaf_src;
                            const int direct = l == depth || scnt[l][ls] <= leaf_src;
                            if (!active || !direct) continue;
                        }
                        for (int64_t q = sfirst[l][ls]; q < sfirst[l][ls] + scnt[l][ls]; ++q) {
                            int64_t i = sperm[q];
                            if (sr[i] == fr[j] && sz[i] == fz[j]) {
                                ++skipped;
                                continue;
                            }
                            int rc2 = grad ? or_greens_grad(fr[j], sr[i], fz[j] - sz[i], nmodes - 1,
                                                            miller, G, Gr, Gx)
                                           : or_greens(fr[j], sr[i], fz[j] - sz[i], nmodes - 1, miller, G);
                            if (rc2 != 0) {
                                err = 1;
                                continue;
                            }
                            const double *Si = S + 2 * (size_t)i * nmodes;
                            for (int n = 0; n < nmodes; ++n) {
                                out[2 * n] += Si[2 * n] * G[n];
                                out[2 * n + 1] += Si[2 * n + 1] * G[n];
                                if (grad) {
                                    outr[2 * n] += Si[2 * n] * Gr[n];
                                    outr[2 * n + 1] += Si[2 * n + 1] * Gr[n];
                                    outz[2 * n] += Si[2 * n] * Gx[n];
                                    outz[2 * n + 1] += Si[2 * n + 1] * Gx[n];
                                }
                            }
                        }
                    }
                }
            }
            free(G);
        }
    }
cleanup:
    for (int l = 0; l < 16; ++l) {
        level_free(&src[l]);
        level_free(&tgt[l]);
        free(scnt[l]);
        free(sfirst[l]);
    }
    free(lstart);
    free(skey);
    free(sperm);
    free(fkey);
    free(fperm);
    free(skey_sorted);
    free(fkey_sorted);
    return err ? -1 : skipped;
}
