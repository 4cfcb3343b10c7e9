/*
 * sfcdd_b200.h -- C ABI of the B200-native SFC two-level Schwarz PCG path.
 *
 * Drop-in boundary for the hot path of the reference package `sfcdd`
 * (arXiv 2110.11211; /root/reference/pkg/src/sfcdd/).  Every entry point
 * cites the reference interface it replaces (file:line).  The Python mirror
 * in paper_2110_11211_b200/ binds these with ctypes exactly as a maintainer
 * would from the reference side.
 *
 * Conventions
 *   - Every function returns int status: 0 = OK, negative = error; the
 *     message is available from sfcdd_last_error() (thread-local).
 *   - *_dev pointers are device pointers owned by the caller; *_host
 *     pointers are host memory.  Streams are cudaStream_t passed as void*.
 *   - Vectors are fp64 in SFC-rank order (grid.py:1-8), length N.
 *   - The operator never mutates caller inputs (schwarz.py:103-118).
 */
#ifndef SFCDD_B200_H
#define SFCDD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python shim maps them to the reference's exceptions */
#define SFCDD_OK 0
#define SFCDD_EVALUE (-1)      /* ValueError          (partition.py:66, coarse.py:39) */
#define SFCDD_EFACTOR (-2)     /* FactorizationError  (linalg.py:21)                 */
#define SFCDD_EBREAKDOWN (-3)  /* BreakdownError      (krylov.py:21)                 */
#define SFCDD_EOVERFLOW (-4)   /* OverflowError       (grid.py:55)                   */
#define SFCDD_ECUDA (-5)       /* CUDA runtime failure / no device                   */
#define SFCDD_EINTERNAL (-6)   /* internal invariant violated                        */

/* variants / weightings (schwarz.py:27-28) */
#define SFCDD_VARIANT_ONE_LEVEL 0
#define SFCDD_VARIANT_ADDITIVE 1
#define SFCDD_VARIANT_DEFLATED 2
#define SFCDD_VARIANT_BALANCED 3
#define SFCDD_WEIGHT_NONE 0
#define SFCDD_WEIGHT_OMEGA 1
#define SFCDD_WEIGHT_DMATRIX 2

const char* sfcdd_last_error(void);
int sfcdd_version(void);

/* ------------------------------------------------------------------ SFC --
 * Replaces sfc.encode (sfc.py:120-136) for a batch of n points.
 * coords_dev: n*dim uint64 words, point-major; keys as (hi, lo) uint64 words.
 * dim*bits <= 128 (sfc.py:36-39); coordinates must be < 2^bits.        */
int sfcdd_sfc_encode(int dim, int bits, const uint64_t* coords_dev, int64_t n,
                     uint64_t* keys_hi_dev, uint64_t* keys_lo_dev, void* stream);

/* Replaces sfc.decode (sfc.py:139-147) for a batch of n keys. */
int sfcdd_sfc_decode(int dim, int bits, const uint64_t* keys_hi_dev,
                     const uint64_t* keys_lo_dev, int64_t n, uint64_t* coords_dev,
                     void* stream);

/* Replaces grid.sfc_permutation (grid.py:60-77): perm[s] = lex index of the
 * interior point with the s-th smallest grid_point_key (sfc.py:150-169).
 * rank_dev (optional, may be NULL) receives the inverse permutation.
 * force_radix != 0 selects the general radix-sort path even when the dense
 * key-space bitmap path applies (test hook).                              */
int sfcdd_sfc_perm(int dim, const int32_t* levels_host, int64_t* perm_dev,
                   int64_t* rank_dev, int force_radix, void* stream);

/* Curve option (north star subsystem (1): Hilbert / Lebesgue keys).  The
 * three calls above are the Hilbert curve of the reference (curve 0); curve 1
 * is the Lebesgue (Morton, Z-order) curve: the same MSB-first interleaving
 * of the raw lattice coordinates, axis 0 first, without the Hilbert
 * transform.  No reference implementation exists for curve 1 (oracle
 * restatement only). */
#define SFCDD_CURVE_HILBERT 0
#define SFCDD_CURVE_LEBESGUE 1
int sfcdd_sfc_encode_curve(int curve, int dim, int bits, const uint64_t* coords_dev, int64_t n,
                           uint64_t* keys_hi_dev, uint64_t* keys_lo_dev, void* stream);
int sfcdd_sfc_decode_curve(int curve, int dim, int bits, const uint64_t* keys_hi_dev,
                           const uint64_t* keys_lo_dev, int64_t n, uint64_t* coords_dev, void* stream);
int sfcdd_sfc_perm_curve(int curve, int dim, const int32_t* levels_host, int64_t* perm_dev,
                         int64_t* rank_dev, int force_radix, void* stream);

/* -------------------------------------------------------------- operator --
 * One handle = one grid, partition, coarse space and Schwarz configuration,
 * bound to one CUDA device.  Replaces the composition
 *   grid.assemble_laplacian + symmetrize_diag   (grid.py:91-130)
 *   partition.build_partition/compute_weights   (partition.py:130-157)
 *   coarse.build_coarse + deflation_ops         (coarse.py:38-88)
 *   schwarz.setup / SchwarzOperator             (schwarz.py:48-130)     */
typedef struct sfcdd_op sfcdd_op;

typedef struct sfcdd_op_desc {
  int32_t dim;
  int32_t levels[8];
  int32_t p;                 /* number of subdomains                        */
  int32_t q;                 /* coarse dofs per subdomain (0 = none)        */
  int32_t variant;           /* SFCDD_VARIANT_*                             */
  int32_t weighting;         /* SFCDD_WEIGHT_*                              */
  int32_t device;            /* CUDA device ordinal                         */
  const int64_t* ov_start;   /* host, p entries: overlapped cyclic ranges,  */
  const int64_t* ov_len;     /*   or NULL: computed from gamma (sfcdd_partition) */
  const int64_t* dj_start;   /* host, p entries: disjoint ranges (NULL with ov_*) */
  const int64_t* dj_len;
  const double* omega;       /* host, p entries (partition.py:151-157), or NULL */
  int32_t host_threads;      /* setup threads (0 = hardware concurrency)    */
  int32_t shard_first;       /* shard mode: first owned subdomain           */
  int32_t shard_count;       /* shard mode: owned subdomains (0 = all)      */
  int32_t curve;             /* SFCDD_CURVE_HILBERT (0) | SFCDD_CURVE_LEBESGUE */
  int32_t raw_laplacian;     /* 0: scaled Â = T A T (grid.py:117-130); 1: the
                                unscaled A of assemble_laplacian (grid.py:91-114) */
  int64_t gamma_num;         /* overlap gamma = gamma_num / gamma_den, used    */
  int64_t gamma_den;         /*   when ov_start == NULL (partition.py:78-116)  */
  int32_t reserved[4];
} sfcdd_op_desc;

/* ------------------------------------------------------------ partition --
 * Replaces partition.disjoint_partition + enlarge (partition.py:64-116):
 * P disjoint ranges (first N mod P one longer) and the gamma-overlapped
 * cyclic ranges, gamma = gamma_num / gamma_den exactly (the caller applies
 * Fraction(gamma).limit_denominator(10**6), partition.py:78-81).  Errors
 * (ValueError) as the reference: P outside [1, N], gamma < 0, overlap with
 * P < 2, 2 gamma + 1 > P.  All outputs host arrays of P entries.          */
int sfcdd_partition(int64_t n, int32_t p, int64_t gamma_num, int64_t gamma_den, int64_t* dj_start,
                    int64_t* dj_len, int64_t* ov_start, int64_t* ov_len);
/* Replaces partition.compute_weights (partition.py:151-157): counts[N]
 * (nullable) = number of overlapped ranges covering each index, omega[P]
 * (nullable) = max over range i of 1/counts.                              */
int sfcdd_partition_weights(int64_t n, int32_t p, const int64_t* ov_start, const int64_t* ov_len,
                            int32_t* counts, double* omega);

typedef struct sfcdd_stats {
  int64_t n;                 /* fine dofs                                   */
  int64_t n0;                /* coarse dofs                                 */
  int64_t factor_nnz;        /* sum_i stored entries of the local factors   */
  int64_t factor_nnz_l;      /* sum_i nnz(L_i) (no amalgamation zeros)      */
  int64_t coarse_nnz;        /* stored entries of the coarse operator       */
  int64_t num_tasks;         /* DAG tasks per sweep                         */
  int64_t num_supernodes;
  double setup_seconds;      /* host+device setup wall time                 */
  double order_seconds;
  double factor_seconds;
  int64_t apply_calls;
  int64_t device_bytes;      /* device memory held by the handle            */
  double last_solve_ms;      /* DAG local-solve kernel time of last apply   */
  int64_t reserved[8];
} sfcdd_stats;

int sfcdd_op_create(const sfcdd_op_desc* desc, sfcdd_op** out);
/* factorizes all A_i and A_0 (schwarz.py:58-61, coarse.py:59-60) */
int sfcdd_op_setup(sfcdd_op* op, void* stream);
/* h = C^{-1} g (schwarz.py:103-118); g_dev, h_dev length N               */
int sfcdd_op_apply(sfcdd_op* op, const double* g_dev, double* h_dev, void* stream);
/* y = Â x, matrix-free scaled 2d+1-point stencil (linalg.py:31-34)        */
int sfcdd_op_matvec(sfcdd_op* op, const double* x_dev, double* y_dev, void* stream);
/* PCG (krylov.py:257-291) with relative-residual stopping on Â, b̂.
 * x_dev holds x0 on entry and the solution on exit; res_hist_host gets
 * max_iters+1 entries (first *iters+1 valid).  Returns SFCDD_EBREAKDOWN on
 * nonpositive curvature (krylov.py:278-279).                              */
int sfcdd_op_pcg(sfcdd_op* op, const double* b_dev, double* x_dev, double tol,
                 int32_t max_iters, double* res_hist_host, int32_t* iters,
                 int32_t* converged, void* stream);
/* PCG with the reference tracker's full semantics (krylov.py:171-200):
 * exact_dev (nullable) = the exact solution; when given, energy_hist_host
 * receives ||x_k - x*||_A = sqrt(max(e.(b - r - A x*), 0)) per iteration
 * (krylov.py:189-193).  tol_kind 0 = relative_residual, 1 =
 * energy_error_reduction (needs exact_dev; stopping metric <= tol * metric_0,
 * krylov.py:194-200).  sfcdd_op_pcg == sfcdd_op_pcg_ex(..., NULL, 0, NULL).  */
int sfcdd_op_pcg_ex(sfcdd_op* op, const double* b_dev, double* x_dev, const double* exact_dev,
                    int32_t tol_kind, double tol, int32_t max_iters, double* res_hist_host,
                    double* energy_hist_host, int32_t* iters, int32_t* converged, void* stream);
/* ------------------------------------------------------- vector kernels --
 * Deterministic fp64 BLAS-1 on device vectors for the non-PCG solvers
 * (Richardson + Lanczos, flexible CG: krylov.py:102-168, 219-254, 294-326);
 * the dot is summed in a fixed order (bitwise repeatable).                 */
int sfcdd_vec_dot(const double* x_dev, const double* y_dev, int64_t n, double* out_host, void* stream);
/* y = a x + b y */
int sfcdd_vec_axpby(double a, const double* x_dev, double b, double* y_dev, int64_t n, void* stream);
/* Config-4 fault mode: in apply call number apply_index the
 * local contributions of the listed subdomains are zeroed.  n = 0 clears. */
int sfcdd_op_set_fault(sfcdd_op* op, int64_t apply_index, const int32_t* ids_host, int32_t n);
int sfcdd_op_reset_calls(sfcdd_op* op);
/* Measurement hook for bench.py: average device time (CUDA events on the
 * launching stream) over `reps` launches of
 *   ms[0] the local-solve DAG kernel alone (input g_dev),
 *   ms[1] one full preconditioner apply,
 *   ms[2] one stencil matvec.
 * launches[0..2] = kernels launched per measured unit.                    */
int sfcdd_op_profile(sfcdd_op* op, const double* g_dev, double* scratch_dev, int32_t reps,
                     double* ms, int32_t* launches, void* stream);
/* Diagnostics: one traced local-solve DAG launch.  out_host receives 24
 * uint64 per task {sm, t_top, t_deps_ok, t_data_ok, t_end (globaltimer ns),
 * kind, copy_bytes, group, values, wait_idx, wait_target, signal_idx,
 * 12 reserved zeros}; *ntask gets the task count (call with out_host =
 * NULL first).                                                            */
int sfcdd_op_trace(sfcdd_op* op, const double* g_dev, uint64_t* out_host, int64_t* ntask);
int sfcdd_op_stats(sfcdd_op* op, sfcdd_stats* out);
/* diagnostics: Â's constants (diag, off per axis) and symmetric scaling t */
int sfcdd_op_stencil(sfcdd_op* op, double* diag, double* off /*dim*/, double* t);
/* diagnostics: coarse matrix A_0 as dense n0*n0 (host), n0 <= 8192         */
int sfcdd_op_coarse_dense(sfcdd_op* op, double* a0_host);
void sfcdd_op_destroy(sfcdd_op* op);

/* ---------------------------------------------------------- shard mode --
 * Multi-GPU: one handle per rank, created with
 * desc.shard_first/shard_count = the rank's contiguous block of subdomains
 * (an SFC segment).  Only those subdomains are factorized.  Vectors stay full
 * length N; every step below computes the owned segment / owned aggregates
 * only.  Partial scalars are written to device doubles for the caller's
 * allreduce; coarse restrictions are per owned aggregate for the caller's
 * allgather (Bank-Holst: every rank then solves the full coarse problem).
 * info = {g0, g1 (owned points), ch0, ch1 (owned chunks), a0, a1 (owned
 * aggregates), xy doubles, n0}; xy_off_host[P] = slot of every subdomain's
 * local solution in the xy buffer (-1: not needed on this rank).          */
int sfcdd_shard_info(sfcdd_op* op, int64_t* info, int64_t* xy_off_host);
/* host copy of the stencil neighbour table int32[2d][N] (-1 = boundary)  */
int sfcdd_op_neighbors(sfcdd_op* op, int32_t* nbr_host);
int sfcdd_shard_xy(sfcdd_op* op, double** xy_dev);
int sfcdd_shard_residual(sfcdd_op* op, const double* b, const double* x, double* r, double* rr_out,
                         double* cagg_out, void* stream);
int sfcdd_shard_pm(sfcdd_op* op, const double* z, const double* pold, double beta, double* pnew,
                   double* ap, double* pap_out, void* stream);
int sfcdd_shard_update(sfcdd_op* op, double* x, double* r, const double* p, const double* ap,
                       double alpha, double* rr_out, double* cagg_out, void* stream);
int sfcdd_shard_coarse(sfcdd_op* op, const double* c, double* y, void* stream);
int sfcdd_shard_tvec(sfcdd_op* op, const double* g, const double* y0, double* t, void* stream);
int sfcdd_shard_local_solve(sfcdd_op* op, const double* t, void* stream);
int sfcdd_shard_combine(sfcdd_op* op, double* w, void* stream);
int sfcdd_shard_stencil_restrict(sfcdd_op* op, const double* w, double* cagg_out, void* stream);
int sfcdd_shard_finalize(sfcdd_op* op, const double* w, const double* y0, const double* y0b, double* z,
                         const double* r, double* rz_out, void* stream);
/* Device-driven sharded PCG (one rank of G, one process per GPU): the whole
 * solve -- stencil halo, overlap extension, foreign local solutions, coarse
 * allgathers, CG scalars -- runs on the GPU as ONE CUDA graph whose
 * iteration loop is a conditional WHILE node; exchanges are NCCL
 * send / recv groups and allgathers on the handle's own communicator
 * (libnccl.so.2 loaded at run time).  Replaces the host-driven program of
 * distributed.pcg_program for production runs (krylov.py:257-291 over
 * schwarz.py:103-118, sharded as SURVEY §8(e)).
 *   sfcdd_nccl_unique_id: 128-byte ncclUniqueId for rank 0 to broadcast;
 *   sfcdd_shard_attach: communicator (nccl_id may be NULL when world == 1)
 *     and the allgather layout agg_counts[world] (owned aggregates per rank);
 *   sfcdd_shard_set_exchange: kind 0 halo, 1 overlap extension, 2 foreign
 *     solutions; per peer (ascending) the send / recv index lists;
 *   sfcdd_shard_pcg: x holds x0, receives the owned segment of the solution. */
int sfcdd_nccl_unique_id(void* id_out);
int sfcdd_shard_attach(sfcdd_op* op, const void* nccl_id, int32_t rank, int32_t world, const int64_t* agg_counts);
int sfcdd_shard_set_exchange(sfcdd_op* op, int32_t kind, int32_t npeer, const int32_t* peers, const int64_t* nsend,
                             const int64_t* send_idx, const int64_t* nrecv, const int64_t* recv_idx);
int sfcdd_shard_pcg(sfcdd_op* op, const double* b, double* x, double tol, int32_t max_iters, double* res_hist_host,
                    int32_t* iters, int32_t* converged, void* stream);
/* exchange packing: dst[i] = src[idx[i]] / dst[idx[i]] = src[i]           */
int sfcdd_pack(const double* src, const int64_t* idx, int64_t n, double* dst, void* stream);
int sfcdd_unpack(const double* src, const int64_t* idx, int64_t n, double* dst, void* stream);

/* ------------------------------------------------------- direct solver --
 * Replaces linalg.Factorization (linalg.py:37-72) for a general SPD CSR
 * matrix on the GPU: AMD ordering, supernodal Cholesky, block-inverse
 * factor applied by the same DAG kernel as the local solves.              */
typedef struct sfcdd_factor sfcdd_factor;
int sfcdd_factor_create(int64_t n, const int64_t* indptr_host, const int32_t* indices_host,
                        const double* data_host, int32_t device, sfcdd_factor** out);
int sfcdd_factor_solve(sfcdd_factor* f, const double* b_dev, double* x_dev, void* stream);
int sfcdd_factor_info(sfcdd_factor* f, int64_t* nnz_l, int64_t* stored, int64_t* nsuper);
void sfcdd_factor_destroy(sfcdd_factor* f);

/* --------------------------------------------------- general matrix --
 * y = A x for a CSR matrix on the device (the `A @ v` of krylov.py:257-291
 * when A is not a grid Laplacian, e.g. test_krylov.py:154-166); summed in
 * stored order with separate multiply/add roundings like scipy csr_matvec. */
typedef struct sfcdd_csr sfcdd_csr;
int sfcdd_csr_create(int64_t rows, int64_t cols, const int64_t* indptr_host, const int32_t* indices_host,
                     const double* data_host, int32_t device, sfcdd_csr** out);
int sfcdd_csr_matvec(sfcdd_csr* m, const double* x_dev, double* y_dev, void* stream);
void sfcdd_csr_destroy(sfcdd_csr* m);

/* --------------------------------------------------- host test hooks --
 * CPU-only checks of the host setup logic (no device needed): AMD ordering
 * and the block-inverse supernodal factor applied on the host.            */
int sfcdd_host_amd(int64_t n, const int64_t* indptr, const int32_t* indices, int32_t* perm_out);
int sfcdd_host_factor_solve(int64_t n, const int64_t* indptr, const int32_t* indices,
                            const double* data, const double* b, double* x,
                            int64_t* nnz_l, int64_t* stored);
/* Factor the principal sub-blocks of a global SPD CSR matrix on p cyclic
 * ranges (start, len), build the device execution plan and run it through
 * the host interpreter of the device blob format.  xy receives the p local
 * solutions A_i^{-1} rhs[range_i], concatenated in range order.  blob_max /
 * scratch_max override the plan budgets (0 = default).                    */
int sfcdd_host_plan_solve(int64_t n, const int64_t* indptr, const int32_t* indices,
                          const double* data, int32_t p, const int64_t* start,
                          const int64_t* len, const double* rhs, double* xy,
                          int32_t blob_max, int32_t scratch_max, int64_t* nfrag);

/* The deferred-value plan (metadata segments + value descriptors, used when
 * the factor values are produced on the device) rebuilds byte for byte the
 * blob image of the plan built from host values; *mismatch = differing bytes. */
int sfcdd_host_plan_deferred_check(int64_t n, const int64_t* indptr, const int32_t* indices,
                                   const double* data, int32_t p, const int64_t* start, const int64_t* len,
                                   int64_t* mismatch, int64_t* nseg, int64_t* nvd);
/* Diagnostics: wall seconds of the setup phases for one SPD block
 * (times[3]: ordering + symbolic, host numeric factorization, plan build)
 * and sizes[6]: nnz(L), stored, supernodes, update-matrix doubles, largest
 * front, factor flops.  numeric = 0 skips the numeric phase and the plan.  */
int sfcdd_host_setup_timing(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data,
                            int32_t numeric, double* times, int64_t* sizes);

#ifdef __cplusplus
}
#endif
#endif /* SFCDD_B200_H */
