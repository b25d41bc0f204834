/*
 * oracle.h -- plain, slow, obviously-correct CPU reference for the hot path of
 * Carley, "A fast multipole method for ... cylindrical coordinates" (arXiv 2301.01179).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product path
 * (libcylfmm.so, paper_2301_01179_b200/) never links, imports or executes this code,
 * and the two share no source, header, table or constant generator.
 *
 * Citations "P:n" are line numbers of PAPER.md (the paper's LaTeX source); "R#k" are the
 * readings listed in DESIGN.md section 3 where the paper is silent or garbled.
 * All arithmetic is IEEE binary64; compiled without -ffast-math and with -ffp-contract=off.
 *
 * Layouts (shared convention with the C-ABI, not shared code):
 *   complex arrays are interleaved (re, im) doubles, row-major [point][mode].
 *   tensor output is dense [mode][a][b][c], a,b in 0..p, c in 0..2p, zero where a+b+c > 2p.
 */
#ifndef CYLFMM_ORACLE_H
#define CYLFMM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Miller start-index rule (R#4): 0 = accurate (contamination below 2^-53), 1 = paper (N+80). */
enum { OR_MILLER_ACCURATE = 0, OR_MILLER_PAPER = 1 };
/* S2L truncation (R#8): 0 = double (i+j<=p, k+l<=p), 1 = single (i+j+k+l<=p). */
enum { OR_TRUNC_DOUBLE = 0, OR_TRUNC_SINGLE = 1 };

/* Carlson symmetric integrals R_F, R_D ("method of Carlson"). */
double or_carlson_rf(double x, double y, double z);
double or_carlson_rd(double x, double y, double z);
/* K(k), E(k) of modulus k given the complementary parameter kp2 = 1 - k^2 (R#1, R#2). */
void or_ellip_ke(double kp2, double *K, double *E);

/* Q_{n-1/2}(chi), n = 0..nmax.  kp2 = rho_-^2/rho_+^2 (complementary parameter);
 * forward != 0 selects the forward branch (chi < 1.008, R#3).  Returns 0 on success. */
int or_legendre_q(double chi, double kp2, int forward, int nmax, int miller, double *Q);
/* 2 t_N of the forward/backward switch chi - 1 < t_N (R#3): 0.016 in the paper mode and for
 * nmax <= 16; 2 (cosh(ln 64 / (2 nmax)) - 1) beyond in the accurate mode. */
double or_forward_coef(int nmax, int miller);
/* Miller extra steps e(chi) beyond nmax (R#4); the backward recursion starts at nmax + e. */
int or_miller_extra(double chi, int miller);
/* G^(n)(r, r1, x), n = 0..nmax. Returns 0, or -1 if r<=0, r1<=0, coincident. */
int or_greens(double r, double r1, double x, int nmax, int miller, double *G);

/* Taylor coefficients in x of the rational kernels used by the derivative recursions (R#7):
 * out[0..qmax] per table, 8 tables in this order:
 *   t+ t-   (x/rho_+-^2), u+ u- ((r^2-r1^2-x^2)/rho_+-^2), v+ v- (d/dr1 of u+-),
 *   us+ us- (u+- with r and r1 exchanged).  out has 8*(qmax+1) doubles. */
void or_rational_tables(double r, double r1, double x, int qmax, double *out);

/* Derivative tensor Gbar^n_{abc} (Laplace recursion corrected per R#6), modes
 * 0..nmax, a,b <= p, a+b+c <= 2p; out dense [nmax+1][p+1][p+1][2p+1]. Returns 0 on success. */
int or_tensor(double r, double r1, double x, int nmax, int p, int miller, double *out);

/* Direct modal sum: Phi_j^(n) = sum_i S_i^(n) G^(n)(r_j, r_i, z_j - z_i),
 * pairs with bitwise-equal (r, z) skipped when exclude_coincident (R#15).
 * Returns number of skipped pairs, or -1 on a domain error. nthreads<=0: OpenMP default. */
int64_t or_direct(const double *sr, const double *sz, const double *S, int64_t ns,
                  const double *fr, const double *fz, int64_t nf, int nmodes, int miller,
                  int exclude_coincident, double *Phi, int nthreads);

/* Tree (R#11): leaf box of each point and the stable Morton-sorted
 * permutation.  key[i] = interleave(ix, iz) radial bits even; perm = argsort(key) stable. */
void or_tree_keys(const double *r, const double *z, int64_t n, int depth, double L, double z0,
                  uint32_t *key, int64_t *perm);

/* Single-box FMM operators on one mode-block: arrays [nmodes][P] complex,
 * coefficient (i,j) with i+j <= p stored at index i*(p+1) - i*(i-1)/2 + j (row-major triangle). */
void or_p2m(const double *r, const double *z, const double *S, int64_t n, int nmodes, int p,
            double rc, double zc, double *M);
void or_m2m(const double *Mc, int nmodes, int p, double dr, double dz, double *Mp_accum);
void or_l2l(const double *Lp, int nmodes, int p, double dr, double dz, double *Lc_accum);
void or_l2p(const double *Lc, int nmodes, int p, double rc, double zc, double r, double z,
            double *phi_accum);
/* S2L from source box centre (rs, zs) to target box centre (rt, zt): computes the tensor at
 * (outer centre, inner centre, |dz|) and applies the FO/BO/FI/BI variant. */
int or_s2l(const double *M, int nmodes, int p, int pl, double rs, double zs, double rt,
           double zt, int truncation, int miller, double *L_accum);

/* Reference FMM, Algorithm 1 step by step.  Domain [0,L] x [z0, z0+L].
 * Returns number of skipped coincident near-field pairs, or -1 on error. */
int64_t or_fmm(const double *sr, const double *sz, const double *S, int64_t ns,
               const double *fr, const double *fz, int64_t nf, int nmodes, int p, int pl,
               int depth, double L, double z0, int truncation, int miller, double *Phi,
               double *dPr, double *dPz, int nthreads, int64_t leaf_src);
/* potential gradients: G and its field-point derivatives d/dr, d/dx by the
 * paper's first-order relations; direct sum with gradients; local-expansion
 * gradient */
int or_greens_grad(double r, double r1, double x, int nmax, int miller, double *G, double *dGr,
                   double *dGx);
int64_t or_direct_grad(const double *sr, const double *sz, const double *S, int64_t ns,
                       const double *fr, const double *fz, int64_t nf, int nmodes, int miller,
                       int exclude_coincident, double *Phi, double *dPr, double *dPz,
                       int nthreads);
void or_l2p_grad(const double *Lc, int nmodes, int p, double rc, double zc, double r, double z,
                 double *gr, double *gz);

#ifdef __cplusplus
}
#endif
#endif
