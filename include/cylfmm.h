/*
 * cylfmm.h -- C-ABI of libcylfmm.so, the B200-native (sm_100a) FP64 hot path of
 * M. Carley, "A fast multipole method for ... ring sources in cylindrical coordinates"
 * (arXiv 2301.01179).  Citations "P:n" are line numbers of the paper text;
 * "R#k" are the readings of DESIGN.md section 3 where the paper is silent or garbled.
 *
 * Problem: ring sources at (r_i, z_i) carrying per-mode complex Fourier
 * coefficients S_i^(n), n = 0..N (K = N+1 modes).  Output: the modal potentials
 *     Phi^(n)(r_j, z_j) = sum_i S_i^(n) G^(n)(r_j, r_i, z_j - z_i)
 * with the modal ring Green's function G^(n) = Q_{n-1/2}(chi) / (2 pi sqrt(r r1)),
 * chi = (r^2 + r1^2 + x^2) / (2 r r1),
 * either summed directly or by the paper's uniform (r, z) quadtree FMM (Algorithm 1).
 *
 * Conventions for every entry point
 *  - Pointers marked DEVICE are device pointers on the current CUDA device; pointers marked
 *    HOST are ordinary host memory (pinned or pageable).  All arrays are C-contiguous.
 *  - Real arrays are IEEE binary64.  Complex arrays are interleaved (re, im) binary64 pairs,
 *    row-major [point][mode], i.e. element (j, n) at doubles 2*(j*K+n), 2*(j*K+n)+1.
 *  - The caller owns every buffer passed in; the library never frees or retains them beyond
 *    the call (device buffers must stay valid until work queued on `stream` completes).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Device-side work is queued
 *    asynchronously on it; the *_host entry points and cylfmm_plan_sync() synchronise.
 *  - Errors are returned as cylfmm_status codes; nothing throws across the ABI.  A detail
 *    message for the last failure on the calling thread is available from cylfmm_last_error().
 *    Argument errors (EINVAL / EDOMAIN) are detected before any work is queued and leave the
 *    outputs untouched.
 *  - Coincident pairs (bitwise-equal (r, z)) are the logarithmic singularity of the ring kernel;
 *    with exclude_coincident = 1 they are skipped (the "self term", R#15), otherwise they are
 *    reported as CYLFMM_ENUMERIC.
 */
#ifndef CYLFMM_H
#define CYLFMM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *cylfmm_stream_t; /* == cudaStream_t */

typedef enum {
    CYLFMM_OK = 0,
    CYLFMM_EINVAL = 1,   /* null pointer, bad size / order / depth / mode count */
    CYLFMM_EDOMAIN = 2,  /* r <= 0, non-finite coordinate, point outside the FMM domain */
    CYLFMM_ENUMERIC = 3, /* unexcluded coincident pair, non-finite result */
    CYLFMM_ECUDA = 4,    /* CUDA runtime error (message in cylfmm_last_error) */
    CYLFMM_ENCCL = 5,    /* NCCL missing or a collective failed (multi-device entry points) */
    CYLFMM_ENOMEM = 6    /* device allocation failed */
} cylfmm_status;

/* Miller start rule for the backward recursion (R#4). */
enum { CYLFMM_MILLER_ACCURATE = 0, /* contamination of Q_{n-1/2} below ~e^-40 */
       CYLFMM_MILLER_PAPER = 1 };  /* the paper's literal start index N + 80 */
/* S2L truncation (R#8). */
enum { CYLFMM_TRUNC_DOUBLE = 0,    /* source i+j <= p and local k+l <= p (default) */
       CYLFMM_TRUNC_SINGLE = 1 };  /* joint i+j+k+l <= p */

/* Limits of this build. */
#define CYLFMM_MAX_MODES 256   /* K <= 256 */
#define CYLFMM_MAX_ORDER 16    /* p <= 16 (the paper's highest order) */
#define CYLFMM_MAX_DEPTH 11    /* d <= 11 (leaf Morton keys fit 22 bits) */

typedef struct {
    int n_modes;            /* K = N+1 >= 1 */
    int order;              /* p >= 1, the paper's expansion order M */
    int depth;              /* d, 2 <= d <= CYLFMM_MAX_DEPTH */
    int truncation;         /* CYLFMM_TRUNC_* */
    int miller;             /* CYLFMM_MILLER_* */
    int exclude_coincident; /* 1: skip bitwise-coincident pairs (R#15) */
    double domain_z0;       /* the square domain is [0, L] x [z0, z0 + L] (R#11) */
    double domain_L;        /* L > 0; a power of two keeps box indices bit-exact */
    int mode_chunk;         /* far-field passes run over modes in chunks of this many; 0 = auto
                               (all modes if the workspace fits a third of free memory) */
    int order_local;        /* local-expansion order pl (the source and local orders
                               may differ); 0 = the source order `order`.  1 <= pl <= 16 */
    int adaptive_leaf;      /* adaptive source tree (DESIGN R#26): a source box
                               holding <= adaptive_leaf sources is a leaf; an adjacent box pair
                               stops there with a direct sum (P:647-651 at that level) and the
                               S2L pairs below it are dropped.  0 = the uniform tree of
                               Algorithm 1.  >= 0; > 0 needs n_modes <= 33 and is not available
                               to cylfmm_fmm_solve_grad (CYLFMM_EINVAL) */
} cylfmm_params;

/* Per-phase device times, milliseconds: CUDA events recorded on the stream each phase runs on
 * (the tensors and the near field run on the plan's auxiliary streams, concurrently with the
 * tree / far-field chain, so the phases may sum to more than ms_total).  Filled by a solve with
 * a non-null `timings` (that solve runs every phase on `stream`, serialised, and synchronises),
 * or averaged over the solves since profiling was switched on by cylfmm_plan_read_timings. */
typedef struct {
    double ms_tree;        /* ms_sort + ms_lists */
    double ms_p2m, ms_m2m, ms_tensor, ms_s2l, ms_l2l, ms_l2p, ms_p2p, ms_total;
    int64_t n_near_pairs;  /* near-field (source, field) pairs evaluated, coincident excluded */
    int64_t n_skipped;     /* coincident pairs skipped */
    int64_t n_s2l_pairs;   /* (source box, target box) S2L applications, all levels */
    int64_t kernel_launches;
    double ms_sort;        /* Morton keys, radix sorts, permuted coordinate / coefficient copies */
    double ms_lists;       /* leaf starts, level maps, S2L pair lists, lazy-L2L flags */
    double ms_unpermute;   /* 0: the un-permutation is fused into the output row writes (a13) */
    double ms_allgather;   /* collective time (multi-device solves; 0 on one device) */
    int64_t n_solves;      /* solves averaged */
    /* near-field branch counts (synchronised timings path only): pairs on the forward branch
     * (chi < 1.008), the far series (chi >= 1000) and Miller's backward recursion
     * (P:868-874), and the sum over Miller pairs of the start offset S - N (R#4) */
    int64_t n_forward, n_far, n_miller, miller_steps;
    /* the tensor seed kernel's span (included in ms_tensor).  Solves without `timings` on large
     * problems run it on the plan's auxiliary stream, overlapping P2M / M2M, so this is a span
     * shared with those phases, not an exclusive time */
    double ms_seeds;
} cylfmm_timings;

typedef struct cylfmm_plan_s *cylfmm_plan;

const char *cylfmm_status_string(cylfmm_status s);
/* Detail message of the last failing call on this thread ("" if none). */
const char *cylfmm_last_error(void);
/* Library version string and the SM architecture it was compiled for ("sm_100a"). */
const char *cylfmm_version(void);

/* ---------------------------------------------------------------------------------------
 * Direct modal sum: out_Phi[j][n] = sum_i S_i^(n) G^(n)(fld_r[j], src_r[i],
 * fld_z[j] - src_z[i]), n = 0..n_modes-1, coincident pairs skipped if exclude_coincident.
 *   src_r, src_z : DEVICE double[n_src]; src_r > 0, finite.
 *   src_S        : DEVICE complex128[n_src][n_modes].
 *   fld_r, fld_z : DEVICE double[n_fld];  fld_r > 0, finite.
 *   out_Phi      : DEVICE complex128[n_fld][n_modes], overwritten.
 *   miller       : CYLFMM_MILLER_*.
 * Summation over i is in a fixed order: results are bitwise reproducible.
 * Returns CYLFMM_ENUMERIC (after synchronising) if an unexcluded coincident pair was met.
 * --------------------------------------------------------------------------------------- */
cylfmm_status cylfmm_direct(const double *src_r, const double *src_z, const double *src_S,
                            int64_t n_src, const double *fld_r, const double *fld_z,
                            int64_t n_fld, int n_modes, int miller, int exclude_coincident,
                            double *out_Phi, cylfmm_stream_t stream);

/* The same direct sum as launches only: no allocation, no synchronisation and no
 * host read, so the call can be captured into a CUDA graph and replayed (the C1-sized sum is
 * launch-latency bound otherwise).  Arguments as for cylfmm_direct, plus
 *   workspace : DEVICE, 16-byte aligned, at least cylfmm_direct_workspace_bytes(...) bytes,
 *               owned by the caller and in use until the work queued here has completed.
 *               Its first int is the error flag, zeroed by the call: non-zero after completion
 *               iff an unexcluded coincident pair was met (what cylfmm_direct reports as
 *               CYLFMM_ENUMERIC); the rest holds per-partition partial sums.
 * Results are bitwise those of cylfmm_direct.  Errors: EINVAL (sizes, null pointers, workspace
 * too small or misaligned), ECUDA. */
cylfmm_status cylfmm_direct_workspace_bytes(int64_t n_src, int64_t n_fld, int n_modes,
                                            int64_t *bytes);
cylfmm_status cylfmm_direct_enqueue(const double *src_r, const double *src_z, const double *src_S,
                                    int64_t n_src, const double *fld_r, const double *fld_z,
                                    int64_t n_fld, int n_modes, int miller, int exclude_coincident,
                                    double *out_Phi, void *workspace, int64_t workspace_bytes,
                                    cylfmm_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * FMM plan.  The plan owns its device workspace (grown on demand, freed by destroy).
 * One plan serves one device and one solve at a time.
 * --------------------------------------------------------------------------------------- */
cylfmm_status cylfmm_plan_create(cylfmm_plan *plan, const cylfmm_params *prm);
void cylfmm_plan_destroy(cylfmm_plan plan);
cylfmm_status cylfmm_plan_sync(cylfmm_plan plan);

/* Profiling of asynchronous solves.  on != 0: every following solve records CUDA events around
 * its phases on the streams they run on (no synchronisation, no change to the launch sequence
 * or results); cylfmm_plan_read_timings then synchronises those events and returns the phase
 * times averaged over the solves since the last read (or since profiling was switched on), and
 * the S2L pair count / kernel launches of the last solve.  Errors: EINVAL (null argument),
 * ECUDA. */
cylfmm_status cylfmm_plan_set_profiling(cylfmm_plan plan, int on);

/* Geometry cache.  on != 0: a solve whose coordinate arrays (src_r, src_z, fld_r, fld_z pointers
 * and sizes) are those of the previous solve on this plan reuses everything that depends only on
 * the coordinates -- the Morton orders, leaf ranges and level maps, the S2L pair lists and
 * batches, the lazy-L2L rows, the near-field and L2P task lists, and (when all modes fit one
 * chunk) the derivative tensors -- and runs only the coefficient-dependent passes (gather of the
 * coefficient rows, P2M, M2M, S2L, L2L, L2P, near field).  Such a solve has NO host
 * synchronisation and allocates nothing, so it can be captured into a CUDA graph.  The caller
 * guarantees that the coordinates themselves did not change (the coefficients src_S may).
 * Switching the cache on (or off) invalidates the remembered geometry.  Results are bitwise those
 * of an uncached solve.  Errors: EINVAL (null plan). */
cylfmm_status cylfmm_plan_set_geometry_cache(cylfmm_plan plan, int on);
cylfmm_status cylfmm_plan_read_timings(cylfmm_plan plan, cylfmm_timings *timings);

/* FMM solve, Algorithm 1 of the paper:
 *   tree (Morton sort of sources and fields on the uniform depth-d quadtree)
 *   -> P2M -> M2M l = d-1..2
 *   -> for l = 2..d: L2L from l-1, S2L from the interaction list with the
 *      FO/BO/FI/BI variants of the tensor at (outer centre, inner centre, |dz|) (P:411-423,
 *      492-537, 561-568)
 *   -> leaves: L2P + direct sum over the 9 neighbour leaves.
 * Inputs as for cylfmm_direct (DEVICE); every point must lie in the plan's domain
 * (0 < r <= L, z0 <= z <= z0 + L), else CYLFMM_EDOMAIN.  out_Phi (DEVICE) is in input field
 * order.  Timings (HOST, nullable) are filled after an internal synchronisation when given.
 * The far field runs over modes in chunks of prm.mode_chunk (results identical). */
cylfmm_status cylfmm_fmm_solve(cylfmm_plan plan, const double *src_r, const double *src_z,
                               const double *src_S, int64_t n_src, const double *fld_r,
                               const double *fld_z, int64_t n_fld, double *out_Phi,
                               cylfmm_stream_t stream, cylfmm_timings *timings);

/* Same as cylfmm_fmm_solve with HOST input and output buffers: copies the inputs to the
 * device, solves, copies out_Phi back and synchronises `stream` before returning. */
cylfmm_status cylfmm_fmm_solve_host(cylfmm_plan plan, const double *src_r, const double *src_z,
                                    const double *src_S, int64_t n_src, const double *fld_r,
                                    const double *fld_z, int64_t n_fld, double *out_Phi,
                                    cylfmm_stream_t stream, cylfmm_timings *timings);

/* Pipelined variant of cylfmm_fmm_solve_host for a stream of solves: returns as soon as the
 * work is queued.  The inputs are uploaded into one of two plan-owned device staging slots
 * (alternating between calls) on a plan copy stream, the solve runs on `stream` behind them, and
 * out_Phi is downloaded on a second plan copy stream; so the next call's upload and the previous
 * call's download overlap the current solve (PCIe is full duplex).  Host buffers (HOST pointers,
 * same layouts as cylfmm_fmm_solve) should be pinned (cudaHostAlloc / cudaHostRegister) for the
 * copies to be asynchronous; the caller keeps them valid and the inputs unmodified, and reads
 * out_Phi, only after cylfmm_plan_sync() (which waits for every queued call).  Argument errors
 * (EINVAL / EDOMAIN) return before any work is queued; device-side errors (ENUMERIC, domain
 * flags) are reported by cylfmm_plan_sync().  The geometry cache does not apply (the staging
 * slots alternate).  Errors: as cylfmm_fmm_solve_host, ENOMEM for the staging slots. */
cylfmm_status cylfmm_fmm_solve_host_async(cylfmm_plan plan, const double *src_r,
                                          const double *src_z, const double *src_S,
                                          int64_t n_src, const double *fld_r,
                                          const double *fld_z, int64_t n_fld, double *out_Phi,
                                          cylfmm_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Test entry points (batched, DEVICE pointers, asynchronous on `stream`).
 * --------------------------------------------------------------------------------------- */

/* G^(n)(r[q], r1[q], x[q]), n = 0..n_modes-1: out_G DEVICE double[n][n_modes].
 * r, r1 > 0 and (r, x) != (r1, 0) required (else CYLFMM_EDOMAIN is flagged on sync). */
cylfmm_status cylfmm_greens_batch(const double *r, const double *r1, const double *x, int64_t n,
                                  int n_modes, int miller, double *out_G, cylfmm_stream_t stream);

/* Derivative tensor Gbar^n_{abc} = (1/(a!b!c!)) d^{a+b+c} G^(n)/dr^a dr1^b dx^c (P:876-1065,
 * Laplace recursion corrected per R#6), modes 0..n_modes-1, a, b <= p, a+b+c <= 2p.
 * out DEVICE double[n][n_modes][p+1][p+1][2p+1], zero where a+b+c > 2p. */
cylfmm_status cylfmm_tensor_batch(const double *r, const double *r1, const double *x, int64_t n,
                                  int n_modes, int p, int miller, double *out,
                                  cylfmm_stream_t stream);

/* Leaf keys and stable Morton sort (R#11): for points (r, z) DEVICE
 * double[n] at depth d on [0, L] x [z0, z0 + L]: key[i] = interleave(ix, iz) (radial index
 * in the even bits), perm = stable argsort(key) (DEVICE int32[n] each; key as uint32). */
cylfmm_status cylfmm_tree_sort(const double *r, const double *z, int64_t n, int depth,
                               double L, double z0, uint32_t *key, int32_t *perm,
                               cylfmm_stream_t stream);

/* FMM solve with the potential gradients (the paper's motivating
 * application): as cylfmm_fmm_solve, plus out_dPhi_dr and out_dPhi_dz (DEVICE,
 * complex128 [n_fld][n_modes], input field order), the derivatives of Phi^(n) with respect to
 * the field point's r and z.  Far field: derivative of the local expansion; near field: the
 * paper's first-order relations dG/dx and dG/dr, G^(-1) == G^(1).
 * Errors: as cylfmm_fmm_solve; EINVAL for null gradient outputs or n_modes > 72. */
cylfmm_status cylfmm_fmm_solve_grad(cylfmm_plan plan, const double *src_r, const double *src_z,
                                    const double *src_S, int64_t n_src, const double *fld_r,
                                    const double *fld_z, int64_t n_fld, double *out_Phi,
                                    double *out_dPhi_dr, double *out_dPhi_dz,
                                    cylfmm_stream_t stream, cylfmm_timings *timings);

/* ---------------------------------------------------------------------------------------
 * Multi-device solves (BASELINE north_star: "field points are partitioned across the GPUs of one
 * 8xB200 box, with sources and the upper tree replicated via NCCL all-gather over NVLink";
 * SURVEY 8(b), 8(e)).  One process per GPU; the library owns the NCCL communicator (NCCL is
 * loaded at run time: libnccl.so.2 of the process, else the system one).
 *
 * cylfmm_comm_unique_id: HOST out, CYLFMM_UNIQUE_ID_BYTES bytes; called on one rank, shared with
 *   the others by the caller (e.g. a torch.distributed broadcast).  Errors: EINVAL, ENCCL.
 * cylfmm_plan_create_dist: a plan (as cylfmm_plan_create, on the current device) with an NCCL
 *   communicator of nranks ranks; collective (every rank calls it with the same id).  Errors:
 *   EINVAL (bad rank/nranks/params), ENCCL (NCCL missing or init failed), as plan_create.
 * cylfmm_fmm_solve_dist: collective solve.  Rank r passes its shard of the sources (DEVICE,
 *   n_src_local rows; the shards in rank order form the global source set) and its own field
 *   points (DEVICE, typically its part of cylfmm_partition_fields); out_Phi (DEVICE) receives
 *   the potentials of ALL sources at its field points, in its input order.  Steps: shard sizes
 *   by ncclAllGather, the shards by grouped ncclBroadcast (one per rank) into plan-owned
 *   replicated arrays; every rank builds the identical source tree; P2M is split by contiguous
 *   source-leaf ranges across the ranks and the leaf moments are replicated by grouped
 *   ncclBroadcast before M2M; the rest runs for the rank's own field points.  Results equal the
 *   single-device solve of the same field points bit for bit.  Timings: ms_allgather is the
 *   collective time.  Errors: as cylfmm_fmm_solve, EINVAL (no communicator), ENCCL.
 * --------------------------------------------------------------------------------------- */
#define CYLFMM_UNIQUE_ID_BYTES 128
cylfmm_status cylfmm_comm_unique_id(void *unique_id);
cylfmm_status cylfmm_plan_create_dist(cylfmm_plan *plan, const cylfmm_params *prm, int nranks,
                                      int rank, const void *unique_id);
cylfmm_status cylfmm_fmm_solve_dist(cylfmm_plan plan, const double *src_r, const double *src_z,
                                    const double *src_S, int64_t n_src_local, const double *fld_r,
                                    const double *fld_z, int64_t n_fld_local, double *out_Phi,
                                    cylfmm_stream_t stream, cylfmm_timings *timings);

/* Field-point partition for a multi-GPU solve (BASELINE north_star: "field points are
 * partitioned across the GPUs ... sources and the upper tree replicated").
 * HOST-only (no device needed): every rank calls it with the same replicated inputs and gets
 * the same answer.  Target leaves of the depth-prm->depth tree (box rule R#11) are cut, in
 * Morton order, into n_parts contiguous ranges of equal estimated cost
 *     cost(leaf) = n_t * [ (sum over the 9 neighbour leaves of n_s) * (200 + 9 K)   near field
 *                          + 4 P K ]                                                L2P
 *                + (non-empty source boxes in the leaf's S2L list) * 4 P^2 K        S2L
 *                + sum over its ancestors A (levels 2..d-1) of the S2L work of A times
 *                  n_t / (field points in A)                          ancestors' S2L
 * (P = (p+1)(p+2)/2; SURVEY 8(d) work per unit), and every field point gets the part of its
 * leaf.  part (HOST, int32 [n_fld], out): part index in [0, n_parts) of each field point, input
 * order.  part_cost (HOST, double [n_parts], out, nullable): estimated flops per part.
 * Errors: EINVAL (null pointers, n_parts < 1, bad params), EDOMAIN (point outside the domain).
 * Because the FMM result at a field point depends only on the sources and on its own box
 * chain, solving each part separately gives bitwise the same values as one solve. */
cylfmm_status cylfmm_partition_fields(const double *src_r, const double *src_z, int64_t n_src,
                                      const double *fld_r, const double *fld_z, int64_t n_fld,
                                      const cylfmm_params *prm, int n_parts, int32_t *part,
                                      double *part_cost);

/* Error-driven choice of the expansion order and the tree depth (the paper
 * fixes neither: its error "scales approximately as C^{-0.4M} with weak dependence on tree
 * depth", read as eps(p) = CYLFMM_EPS_C * 10^(-0.4 p), R#25).  HOST-only.
 *  - order: the smallest p in [1, CYLFMM_MAX_ORDER] with eps(p) <= tol (CYLFMM_MAX_ORDER if
 *    none); order_local = 0 (equal orders, as in the paper's runs).
 *  - depth: the d in [depth_min, depth_max] (clamped to [2, CYLFMM_MAX_DEPTH]) minimising the
 *    modelled solve time
 *        T(d) = [ near(d) * (200 + 9 K) / e_near  +  s2l(d) * 4 P^2 K / e_s2l
 *               + 12 * 2^d * K * (12 (2p+1)^2 + 12 (p+1)^3) / e_tens ] / F64_peak
 *    (SURVEY 8(d) work per unit; e_* = round-1 measured fractions of the FP64 peak), where
 *    near(d) = sum over non-empty target leaves t of n_t * (sources in the 9 leaves around t)
 *    (coincident pairs included) and s2l(d) = sum over levels 2..d of (non-empty target box,
 *    non-empty source box in its interaction list) pairs: the exact counts a
 *    depth-d solve reports as n_near_pairs + n_skipped and n_s2l_pairs.
 * prm (in/out): n_modes, domain_L, domain_z0 read (checked as for plan_create); order, depth
 * and order_local written; other fields untouched.  tol > 0 (per-mode relative error).
 * near_pairs, s2l_pairs (HOST int64 [depth_max - depth_min + 1], nullable), est_ms (HOST double
 * [same], nullable): the per-depth counts and modelled times (-1 for depths outside [2, 11]).
 * eps_model (HOST, nullable): eps(order).
 * Errors: EINVAL (null prm, tol <= 0 or not finite, depth_min > depth_max, bad prm fields),
 * EDOMAIN (point outside the domain). */
#define CYLFMM_EPS_C 0.1
cylfmm_status cylfmm_select_params(const double *src_r, const double *src_z, int64_t n_src,
                                   const double *fld_r, const double *fld_z, int64_t n_fld,
                                   double tol, int depth_min, int depth_max, cylfmm_params *prm,
                                   int64_t *near_pairs, int64_t *s2l_pairs, double *est_ms,
                                   double *eps_model);

#ifdef __cplusplus
}
#endif
#endif
