/*
 * sexpm.h — C ABI of libsexpm: the filtered precise-integration (PIM)
 * scaling-and-squaring matrix exponential of arXiv 2110.04493 on B200 (sm_100a).
 *
 * PAPER.md citations are P:<line> (Wu, Zhang, Zhu, Hu, "High-performance
 * computation of large sparse matrix exponential").
 *
 * What the library computes (Algorithm 4.2):
 *   1. (M, N) from Eq. (4.20) with the plan norm (1-norm by default;
 *      Frobenius as in the paper's experiments);
 *   2. a = 1/(N+1) if H is normal else min(1, 1/||H||) (Eq. 4.19);
 *   3. filtered Taylor phase on H0 = H 2^-N: S^_1 = H0, S~_i = S^_{i-1} H0 / i,
 *      S^_i = Alg4.1(S~_i, eps_g^(0)), T^_0 = sum S^_i, eps_g^(0) = a r0/(M e^{2||H0||})
 *      (Eq. 4.10-4.14);
 *   4. N filtered squarings T~_i = 2 T^_{i-1} + T^_{i-1}^2, T^_i = Alg4.1(T~_i, eps_g^(i))
 *      (Eq. 2.7, Eq. 4.15), eps_g^(i) = a r_i ||I + T^_{i-1}||_F
 *      (reading R4 of DESIGN.md; option ABS gives a r_i as printed at P:422);
 *   5. e^H = I + T^_N.
 * Algorithm 4.1 is the adaptive drop filter of P:360-380 (strict '>' keep).
 * All arithmetic is IEEE fp64.
 *
 * Memory / ownership conventions
 *   - Every pointer inside sexpm_csr_in / sexpm_csr_out is a CUDA DEVICE pointer on the
 *     caller's current device, except in sexpm_plan_host (HOST pointers) and
 *     sexpm_result_copy (host or device pointers).
 *   - CSR: int64 rowptr (row_end - row_begin + 1 entries, rowptr[0] == 0), int32 column
 *     indices (global, strictly increasing within a row), fp64 values (finite, nonzero).
 *   - Inputs are borrowed: the library copies what it needs during sexpm_plan*; the caller
 *     may free them when the call returns.
 *   - Outputs (sexpm_csr_out) are owned by the plan and stay valid until the next
 *     sexpm_run on the same plan or sexpm_destroy.
 *   - A plan is bound to one device and one CUDA stream and is not thread-safe.
 *   - With world > 1 (an NCCL communicator in the options), sexpm_plan / sexpm_run are
 *     collective: every rank passes its own contiguous row block and gets its row block
 *     of e^H back.
 *
 * Errors: every entry point returns an sexpm_status; no exception crosses the ABI;
 * sexpm_last_error() returns a thread-local message for the last non-OK status.
 * Sticky CUDA errors map to SEXPM_ECUDA.
 *
 * Diagnostics (environment, read at call time; they change no result): SEXPM_PLAN_LOG
 * (host phase times of sexpm_plan, synchronising), SEXPM_STEP_LOG (per Taylor term /
 * squaring: nnz, passes, kernel times, accumulator sizing), SEXPM_CACHE_LOG (device-block
 * cache traffic), SEXPM_BSR_NATURAL (block kernel in index order instead of the locality
 * order; for measurements).
 */
#ifndef SEXPM_H
#define SEXPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SEXPM_OK = 0,
  SEXPM_EINVAL = 1,        /* bad argument / malformed CSR / n == 0 */
  SEXPM_ENONFINITE = 2,    /* H holds a NaN or Inf */
  SEXPM_ETOL = 3,          /* eps_tol below the unit roundoff reading (R13: eps_tol >= 1e-16) */
  SEXPM_EINFEASIBLE = 4,   /* Eq. (4.20) has no solution with M <= m_cap in the N window */
  SEXPM_ENOMEM = 5,        /* device allocation failed */
  SEXPM_ECUDA = 6,         /* CUDA runtime error */
  SEXPM_ENCCL = 7,         /* NCCL error / NCCL unavailable */
  SEXPM_ESTATE = 8,        /* call out of order (e.g. stats before run) */
  SEXPM_EINTERNAL = 9      /* invariant violated (e.g. Algorithm 4.1 pass cap) */
} sexpm_status;

typedef struct sexpm_plan_s *sexpm_plan_t;
typedef struct sexpm_copy_s *sexpm_copy_t; /* a result copy in flight (sexpm_result_copy_async) */

typedef struct {
  int64_t n;                  /* global dimension (n >= 1) */
  int64_t row_begin, row_end; /* rows held by this rank; [0, n) on one GPU */
  int64_t nnz;                /* entries in this row block */
  const int64_t *rowptr;      /* row_end - row_begin + 1 entries, rowptr[0] == 0 */
  const int32_t *colidx;      /* global columns, strictly increasing within a row */
  const double *vals;         /* finite; explicit zeros are allowed and ignored */
} sexpm_csr_in;

typedef struct {
  int64_t n, row_begin, row_end, nnz;
  const int64_t *rowptr; /* device, plan-owned */
  const int32_t *colidx;
  const double *vals;
} sexpm_csr_out;

typedef struct {
  uint32_t struct_size;   /* = sizeof(sexpm_options) (ABI check) */
  int32_t plan_norm;      /* 0 = 1-norm (default, BASELINE north star), 1 = Frobenius */
  int32_t normal;         /* -1 auto: bit-exact symmetric or skew-symmetric => normal; 0 no; 1 yes */
  int32_t threshold_mode; /* 0 = a r_i ||I+T^_{i-1}||_F (default, R4); 1 = a r_i (P:422 as printed) */
  int32_t filter;         /* 1 = paper's filter (default); 0 = unfiltered PIM (all eps_g = 0) */
  int32_t m_cap;          /* max Taylor order in Eq. (4.20) enumeration (default 120) */
  int32_t n_window;       /* N in [N0, N0 + n_window] (default 50) */
  int32_t force_M;        /* -1 = from Eq. (4.20) */
  int32_t force_N;        /* -1 = from Eq. (4.20) */
  int32_t output_T;       /* 0 = return E = I + T^_N (default); 1 = return T^_N */
  int32_t window_cols;    /* dense accumulator window of the block-window kernel (0 = 8192) */
  int32_t kernel;         /* K3 kernel: 0 auto (squarings: the block-sparse kernel on the BSR-8
                             view, 13 = fp64 tensor-core DMMA (default) or 11 = exact DMUL/DADD
                             per exact_products, on one GPU and on a rank's rows inside its halo;
                             Taylor terms: the offset-window kernel 8 when H0 has <= 16
                             distinct diagonal offsets whose Minkowski sums up to order M
                             fit its shared-memory rows (<= 4096 offsets: 1D / 2D
                             stencils), else the diagonal push kernel 7 when H0 has <= 16
                             offsets, else the pull over H0^T 6); 3 block
                             window, 5 k-synchronous paged, 6 Taylor pull (Taylor terms only;
                             else 5), 7 Taylor diagonal push (Taylor terms only; else as 0),
                             8 Taylor offset window (Taylor phase only; else as 0),
                             11 block-sparse exact, 13 block-sparse tensor core (squarings
                             only; else as 0).  All meet parity; 5, 6, 7, 8 and 11 reproduce the
                             oracle's C~ bit for bit.  Rows a kernel cannot hold fall through
                             11/13 -> 5 -> 3, 7 -> 7 at twice the accumulator slots -> 5 -> 3,
                             6 -> 5 -> 3. */
  int32_t ssat;           /* 0 = the paper's PIM (default); 1 = the SSAT baseline of Table 1
                             (SURVEY section 8(f) N2): the same Taylor phase
                             (filtered per `filter`), then E_0 = I + T^_0 and N plain
                             squarings E_i = E_{i-1}^2 without the incremental split and
                             without filtering.  Incompatible with output_T (SEXPM_EINVAL). */
  int32_t reorder;        /* 0 = none (default); 1 = reverse Cuthill-McKee on the device
                             (Def. 3.2a's real bandwidth):
                             the plan computes a permutation P of pattern(H + H^T), runs on
                             P H P^T and returns E = P^T E' P in the caller's order
                             (e^{PHP^T} = P e^H P^T).  Single GPU; nnz < 2^31. */
  int32_t sq_order;       /* 1 = (default) the squarings run on T^_0 relabelled into 8-row
                             aggregates of H's graph (fuller 8x8 blocks for K3b), E mapped
                             back; 0 = index order.  One GPU only; not with ssat.  Results
                             equal up to rounding order (north-star parity). */
  int32_t exact_products; /* 0 = (default) squarings on the fp64 tensor-core block kernel 13
                             (fused multiply-adds: C~ within rounding of the oracle's), Taylor
                             terms too once their rows outgrow the diagonal kernel;
                             1 = the bit-exact block kernel 11 (DMUL + DADD in the oracle's
                             order: C~ bit-identical to the oracle's).  Only with kernel = 0. */
  int32_t sym_squaring;   /* -1 = (default) auto: when H is bit-exactly symmetric, one GPU,
                             kernel 0 / 13, not exact_products / ssat, the squarings compute
                             only the output blocks J >= I of T~ = 2T + T^2 (symmetric for a
                             symmetric T) and read the others as transposes (K3c count, K3s
                             product, K3a row assembly; kernels.cuh SymOut), after making T^_0
                             exactly symmetric from its upper triangle (reading R21: changes
                             T^_0 by rounding only).  Falls back to the full product when a
                             block row does not fit.  0 = off (the full product). */
  double e_r;             /* Algorithm 4.1 tolerance e_r > 0 (default 0.1, R6) */
  void *stream;           /* cudaStream_t to run on (NULL = a stream created by the plan; to run
                             on the legacy default stream pass cudaStreamLegacy, as the Python
                             binding does for torch's default stream) */
  void *nccl_comm;        /* communicator handle from sexpm_nccl_comm_init (NCCL) or
                             sexpm_virtual_comm_create (virtual ranks), or NULL for one GPU */
} sexpm_options;

#define SEXPM_MAXSTEP 160

typedef struct {
  uint32_t struct_size;
  int32_t M, N, M_eff, normal, world, rank;
  double norm, a, r0, eps_g0;
  /* Taylor terms i = 2..M at index i */
  int64_t taylor_nnz_unf[SEXPM_MAXSTEP]; /* distinct nonzeros of S~_i */
  int64_t taylor_nnz[SEXPM_MAXSTEP];     /* nnz of S^_i after Algorithm 4.1 */
  int32_t taylor_passes[SEXPM_MAXSTEP];
  double taylor_tau[SEXPM_MAXSTEP];      /* final Algorithm 4.1 threshold */
  double taylor_ms[SEXPM_MAXSTEP];
  double taylor_numeric_ms[SEXPM_MAXSTEP];    /* device time of the term's SpGEMM kernel */
  double taylor_numeric_bytes[SEXPM_MAXSTEP]; /* its compulsory bytes: A + B + staged writes */
  double taylor_fmas_i[SEXPM_MAXSTEP];        /* its products */
  /* squarings i = 1..N at index i; index 0 describes T^_0 */
  int64_t sq_nnz_unf[SEXPM_MAXSTEP];
  int64_t sq_nnz[SEXPM_MAXSTEP];
  int64_t sq_staged[SEXPM_MAXSTEP];      /* entries above the floor eps_g/sqrt(K) */
  int32_t sq_passes[SEXPM_MAXSTEP];
  double sq_eps_g[SEXPM_MAXSTEP];
  double sq_tau[SEXPM_MAXSTEP];
  double sq_normIT[SEXPM_MAXSTEP];       /* ||I + T^_i||_F */
  int64_t sq_l1[SEXPM_MAXSTEP], sq_l2[SEXPM_MAXSTEP]; /* Eq. (3.1) bandwidths of T^_i */
  double sq_fmas[SEXPM_MAXSTEP];         /* sum_r sum_{k in row r} nnz(row k) (+ 2T adds) */
  double sq_ms[SEXPM_MAXSTEP];           /* device time of the whole step */
  double sq_numeric_ms[SEXPM_MAXSTEP];   /* device time of the SpGEMM kernel alone */
  double sq_bytes[SEXPM_MAXSTEP];        /* compulsory HBM bytes of the step: 12 nnz(T^_{i-1}) + 12 nnz(T^_i) + 16 rows */
  double sq_numeric_bytes[SEXPM_MAXSTEP];/* compulsory bytes of the SpGEMM kernel: A + B + staged writes */
  double ms_plan, ms_taylor, ms_squaring, ms_finalize, ms_total;
  double taylor_bytes, taylor_fmas;
  int64_t nnz_out;
  int32_t gpu_launches;                  /* kernels launched by the last sexpm_run */
  int32_t retries;                       /* steps re-run after a staging-pool overflow */
  int64_t taylor_fallback_rows[SEXPM_MAXSTEP]; /* rows the term's first kernel handed on */
  int64_t sq_fallback_rows[SEXPM_MAXSTEP];     /* rows the squaring's first kernel handed on */
  double sq_first_ms[SEXPM_MAXSTEP];           /* device time of the squaring's first stage */
  double sq_kernel_ms[SEXPM_MAXSTEP];          /* its product kernel alone (block kernel: without
                                                  building the BSR view) */
  int64_t sq_bsr_blocks[SEXPM_MAXSTEP];        /* 8x8 blocks of the BSR view (block kernel) */
  double sq_block_products[SEXPM_MAXSTEP];     /* 8x8 block products it executed (512 each) */
  /* the library's device-block cache during the last sexpm_plan + sexpm_run (process-wide) */
  int64_t cache_hits, cache_misses, cache_releases;
  double cache_bytes_cached, cache_bytes_allocated;
  int32_t sq_order_used;                       /* squarings ran in: 0 index order, 1 BFS
                                                  aggregates, 2 compact aggregates (host
                                                  thread), 3 diamond tiles of a 2D grid, 4
                                                  2x2x2 cubes of a 3D grid (device, one GPU)
                                                  (sq_order) */
  double sq_exchange_ms[SEXPM_MAXSTEP];        /* world > 1: halo exchange of the squaring
                                                  (host wall clock, incl. the peers' wait) */
  double ms_order_host;  /* the squarings' locality / aggregate order, computed on a host
                            thread from H's pattern while the Taylor phase runs (wall ms) */
  double ms_order_wait;  /* how long the first squaring waited for it (0 when hidden) */
  int32_t taylor_window; /* 1: the Taylor phase ran on the offset-window kernel K5w (dense
                            rows over the Minkowski sums of H0's diagonal offsets); 0: term
                            by term on the product kernels */
  int32_t sq_sym_used;   /* squarings that ran on the symmetric path (sym_squaring) */
  double sq_assemble_ms[SEXPM_MAXSTEP]; /* symmetric path: K3c count + K3a row assembly
                                           (sq_kernel_ms is the product kernel K3s alone) */
} sexpm_stats;

/* sizes[0..3] = sizeof(sexpm_options), sizeof(sexpm_stats), sizeof(sexpm_csr_in),
 * sizeof(sexpm_csr_out): lets bindings verify their struct layouts (host only). */
int sexpm_abi_sizes(uint32_t *sizes);

/* Kernels enqueued by this library since it was loaded (all plans, all threads). */
int sexpm_kernel_launches(int64_t *count);

/* fp64 throughput of the current device, measured (the squaring kernels' roofline
 * denominator): best of 5 timed launches of 8 independent DFMA chains per thread (TF/s, 2
 * flops per DFMA) and of 8 independent mma.sync.m8n8k4.f64 accumulators per warp (TF/s, 512
 * flops per DMMA), 8 CTAs x 256 threads per SM.  Either pointer may be NULL (not both).
 * Synchronous; allocates and frees its own scratch.  Errors: SEXPM_EINVAL, SEXPM_ECUDA. */
int sexpm_fp64_peak(double *dfma_tflops, double *dmma_tflops);

/* Fill defaults (see field comments). */
int sexpm_options_init(sexpm_options *o);

/* NCCL bootstrap: rank 0 calls sexpm_nccl_unique_id and ships the 128 bytes to all ranks
 * (e.g. torch.distributed broadcast); every rank then calls sexpm_nccl_comm_init with its
 * own CUDA device current.  The communicator is destroyed with sexpm_nccl_comm_destroy. */
int sexpm_nccl_unique_id(void *id128);
int sexpm_nccl_comm_init(int rank, int world, const void *id128, void **comm);
int sexpm_nccl_comm_destroy(void *comm);

/* Virtual ranks (testing the multi-rank path on one GPU): creates `world` communicator
 * handles comms[0..world) that connect `world` plans in ONE process on ONE device, each
 * driven by its own host thread (its own stream).  Every collective of the row-partitioned
 * path (scalar all-gathers, the all-gather of H, the halo exchange of every squaring) is a
 * host barrier, device-to-device copies from the peers' buffers on the caller's stream, and
 * a second barrier; no kernel waits on another rank.  A rank that does not arrive within
 * 300 s makes the others fail with SEXPM_ENCCL.  Pass comms[r] as options.nccl_comm of rank
 * r; destroy each with sexpm_nccl_comm_destroy.  world in [1, 64], else SEXPM_EINVAL. */
int sexpm_virtual_comm_create(int world, void **comms);

/* Step 1-3 set-up: validate H (device CSR), compute ||H|| on the device, solve Eq. (4.20),
 * choose a, r0, eps_g^(0), scale H0 = H 2^-N.  eps_tol: target relative error bound r_N. */
int sexpm_plan(const sexpm_csr_in *H, double eps_tol, const sexpm_options *o, sexpm_plan_t *out);

/* Same as sexpm_plan but H's arrays are HOST pointers; the library copies them in. */
int sexpm_plan_host(const sexpm_csr_in *H_host, double eps_tol, const sexpm_options *o,
                    sexpm_plan_t *out);

/* Steps 3-5: Taylor phase, N filtered squarings, E = I + T^_N.  Synchronises the plan's
 * stream before returning.  E (device, plan-owned) may be NULL. */
int sexpm_run(sexpm_plan_t p, sexpm_csr_out *E);

/* Copy the last result (rows+1 rowptr, nnz cols, nnz vals) into caller-owned arrays,
 * HOST (D2H, pinned or pageable) or DEVICE (D2D) pointers alike; synchronises the stream. */
int sexpm_result_copy(sexpm_plan_t p, int64_t *rowptr, int32_t *colidx, double *vals);

/* The same copy without waiting for it: E = I + T^_N (Algorithm 4.2 step 5) is DETACHED
 * from the plan (which then has no result: sexpm_apply / sexpm_result_copy return
 * SEXPM_ESTATE until the next sexpm_run) and copied on the library's own copy stream, ordered
 * after the plan's stream; returns at once with *ticket.  The plan may be destroyed and the
 * next plan created and run on any stream while the copy is in flight: with results larger
 * than the link can move in one e^H (config 5: 14.6 GB over PCIe), consecutive e^H overlap
 * their copy-out with the next computation.  The caller's arrays (HOST, pinned for overlap,
 * or DEVICE) must not be read before sexpm_result_wait(ticket) returns; every ticket must
 * be waited for exactly once (it frees the detached device blocks: they go back to the
 * library's cache for the next plan's result).  sexpm_result_wait(NULL) is a no-op.
 * Errors: SEXPM_ESTATE (no result), SEXPM_EINVAL (null arrays / ticket), SEXPM_ECUDA. */
int sexpm_result_copy_async(sexpm_plan_t p, int64_t *rowptr, int32_t *colidx, double *vals,
                            sexpm_copy_t *ticket);
int sexpm_result_wait(sexpm_copy_t ticket);

/* N1 apply: Y = R^steps X, R the last result (E = I + T^_N, or T^_N
 * with output_T), i.e. `steps` steps of the discretised system u_{k+1} = e^H u_k (Eq. 2.2,
 * P:54; the validation protocol of P:501-503).  X: DEVICE, row-major, n x m (row stride
 * ldx >= m doubles); Y: DEVICE, row-major, n x m (ldy >= m), caller-owned, must not overlap
 * X.  m >= 0, steps >= 1.  For m >= 32 every Y entry is the sum over the row's entries in
 * ascending column order with separately rounded products (bit-identical to the oracle's
 * or_spmm); for m < 32 the row's entries are split over lane groups and combined by a fixed
 * tree (deterministic).  steps > 1 uses two plan-owned n x m buffers.  With several ranks
 * (collective: every rank calls it with the same m and steps): X and Y hold this rank's rows
 * [row_begin, row_end); each step exchanges the rows of the current block within E's
 * bandwidth (Lemma 3.1) with the peers through the plan's communicator, then
 * multiplies the rank's rows of E.  SEXPM_ESTATE before sexpm_run.  Synchronises the stream. */
int sexpm_apply(sexpm_plan_t p, int64_t m, const double *X, int64_t ldx, double *Y, int64_t ldy,
                int32_t steps);

/* Plan scalars, per-step trace and CUDA-event timings of the last run. */
int sexpm_stats_get(sexpm_plan_t p, sexpm_stats *s);

int sexpm_destroy(sexpm_plan_t p);
/* Device blocks of destroyed plans stay cached in the library (process-wide, per device)
 * and are reused by later plans; this returns them to the CUDA memory pool.  Allocation
 * failures release the cache automatically before reporting SEXPM_ENOMEM. */
int sexpm_release_cache(void);

const char *sexpm_last_error(void);

/* ----- component entry points (used by the parity tests; same kernels as sexpm_run) ----- */

/* One filtered product on the plan's device/stream (single GPU):
 *   C~ = (self_coef * A + A * B) / divisor,  C^ = Alg4.1(C~, eps_g, e_r).
 * self_coef = 2, divisor = 1 is a squaring step (Eq. 4.15); self_coef = 0, divisor = i is
 * a Taylor term (Eq. 4.11).  A and B are device CSR over all n rows.  The result is
 * plan-owned (valid until the next call on the plan); *passes / *tau report Algorithm 4.1;
 * *nnz_unf the distinct nonzeros of C~. */
int sexpm_filtered_product(sexpm_plan_t p, const sexpm_csr_in *A, const sexpm_csr_in *B,
                           double self_coef, double divisor, double eps_g, sexpm_csr_out *C,
                           int32_t *passes, double *tau, int64_t *nnz_unf);

/* Algorithm 4.1 over a device array of cnt values: returns the number of passes, the final
 * threshold tau (entries kept are exactly |x| > tau; the first pass always runs (reading R1); 0 when
 * eps_g == 0) and the dropped Frobenius norm. */
int sexpm_alg41(sexpm_plan_t p, const double *x, int64_t cnt, double eps_g, double e_r,
                int32_t *passes, double *tau, double *dropped);

/* N3: the reverse Cuthill-McKee permutation (perm[new] = old) of pattern(A + A^T) for a
 * device CSR A holding all n rows, as option `reorder` computes it (rules in DESIGN.md and
 * oracle or_rcm).  perm: n int64, host or device.  Runs on the plan's stream; synchronises. */
int sexpm_rcm(sexpm_plan_t p, const sexpm_csr_in *A, int64_t *perm);

/* Y = A X for any device CSR A (rows row_begin..row_end of an n x n matrix, global column
 * indices) and dense device X (n x m, row-major, ldx >= m) into Y (rows of A x m, ldy >= m):
 * the kernel of sexpm_apply.  Runs on the plan's stream and synchronises it. */
int sexpm_spmm(sexpm_plan_t p, const sexpm_csr_in *A, int64_t m, const double *X, int64_t ldx,
               double *Y, int64_t ldy);

/* Host only (no device work; callable without a GPU).  The scalar part of Algorithm 4.2
 * steps 1-3 for a given plan norm ||H||: (M, N) by Eq. (4.20) (
 * N in [N0, N0 + n_window], M in [0, m_cap], ties to the smaller N: reading R5), the budget
 * a = 1/(N+1) if normal (Eq. 4.19) else min(1, 1/||H||) (reading R8), r0 =
 * r0(||H|| 2^-N, M) (Eq. 4.5) and eps_g^(0) = a r0 / (M e^{2 ||H 2^-N||}).
 * sexpm_plan uses exactly this after measuring the norm on the device.  a, r0, eps_g0 may
 * be NULL.  Errors: SEXPM_EINVAL (negative / non-finite norm, normal not 0/1),
 * SEXPM_ETOL (eps_tol < 1e-16, reading R13), SEXPM_EINFEASIBLE (no (M, N) in range). */
int sexpm_plan_scalars(double norm, int normal, double eps_tol, int m_cap, int n_window,
                       int32_t *M, int32_t *N, double *a, double *r0, double *eps_g0);

/* Host-side halo planner for the row-partitioned multi-GPU squaring (Lemma 3.1):
 * rank g owns rows [bounds[g], bounds[g+1]); with T^_{i-1} of bandwidths (l1, l2) the
 * product rows of rank g need B rows [max(0, b_g - l2), min(n, b_{g+1} + l1)).  Writes, for
 * every peer h, the row range [lo, hi) rank g must receive from h (lo == hi when none). */
int sexpm_halo_ranges(int world, int rank, const int64_t *bounds, int64_t n, int64_t l1,
                      int64_t l2, int64_t *recv_lo, int64_t *recv_hi);

/* Row partition balanced by a per-row work estimate (contiguous blocks). */
int sexpm_partition_rows(int64_t n, const double *work, int world, int64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif /* SEXPM_H */
