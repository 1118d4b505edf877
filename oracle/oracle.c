/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the filtered
 * precise-integration matrix exponential of arXiv 2110.04493
 * (Wu, Zhang, Zhu, Hu, "High-performance computation of large sparse matrix
 * exponential").  PAPER.md line numbers are cited as P:<line>.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2110_04493_b200/csrc); neither side includes the other.
 *
 * Arithmetic: IEEE double, compiled with -ffp-contract=off and without
 * -ffast-math.  Scalar series and filter sums use long double.  Every
 * function follows the paper's algorithm step by step in its order and
 * notation; nothing is blocked, fused or reordered.
 *
 * Readings of the paper where it is silent / garbled are listed in
 * DESIGN.md §"Readings" (R1..R14) and cited below.
 *
 * Pinned by tests/test_oracle_*.py against: Table 1 closed forms,
 * Table 2 and Table 3 bandwidth sequences, the (M, N) = (20, 8)
 * plan, closed forms of r0 (Eq. 4.5), the 1D/2D Dirichlet heat
 * closed forms, diagonal H, zero-row-sum and skew-symmetric invariants and a
 * 50-digit dense reference.  See DESIGN.md §"Oracle pins".
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* CSR owned by the oracle                                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  int64_t *rowptr; /* n+1 */
  int32_t *col;    /* nnz, strictly increasing per row */
  double *val;     /* nnz, no exact zeros */
} ocsr;

static ocsr csr_alloc(int64_t n, int64_t nnz) {
  ocsr A;
  A.n = n;
  A.rowptr = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
  A.col = (int32_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  A.val = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  return A;
}

static void csr_free(ocsr *A) {
  free(A->rowptr);
  free(A->col);
  free(A->val);
  A->rowptr = NULL;
  A->col = NULL;
  A->val = NULL;
}

static int64_t csr_nnz(const ocsr *A) { return A->rowptr[A->n]; }

static ocsr csr_copy_in(int64_t n, const int64_t *rp, const int32_t *ci, const double *v) {
  int64_t nnz = rp[n] - rp[0];
  ocsr A = csr_alloc(n, nnz);
  for (int64_t i = 0; i <= n; i++) A.rowptr[i] = rp[i] - rp[0];
  memcpy(A.col, ci, (size_t)nnz * sizeof(int32_t));
  memcpy(A.val, v, (size_t)nnz * sizeof(double));
  return A;
}

/* ------------------------------------------------------------------------- */
/* Norms ("any compatible norm"; P:432 Frobenius in all experiments)     */
/* ------------------------------------------------------------------------- */

/* ||A||_1 = max_j sum_i |a_ij|, column sums accumulated in row-major order. */
double or_norm_one(int64_t n, const int64_t *rp, const int32_t *ci, const double *v) {
  double *cs = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t i = 0; i < n; i++)
    for (int64_t p = rp[i]; p < rp[i + 1]; p++) cs[ci[p]] += fabs(v[p]);
  double m = 0.0;
  for (int64_t j = 0; j < n; j++)
    if (cs[j] > m) m = cs[j];
  free(cs);
  return m;
}

/* ||A||_F = sqrt(sum a_ij^2), summed in row-major order. */
double or_norm_fro(int64_t n, const int64_t *rp, const int32_t *ci, const double *v) {
  (void)ci;
  long double s = 0.0L;
  for (int64_t p = rp[0]; p < rp[n]; p++) s += (long double)v[p] * (long double)v[p];
  return (double)sqrtl(s);
}

/* ||I + T||_F: (1 + t_ii)^2 on the diagonal (t_ii = 0 if absent), t_ij^2 off it. */
static double norm_fro_I_plus(const ocsr *T) {
  long double s = 0.0L;
  for (int64_t i = 0; i < T->n; i++) {
    int have_diag = 0;
    for (int64_t p = T->rowptr[i]; p < T->rowptr[i + 1]; p++) {
      long double x = T->val[p];
      if (T->col[p] == i) {
        x += 1.0L;
        have_diag = 1;
      }
      s += x * x;
    }
    if (!have_diag) s += 1.0L;
  }
  return (double)sqrtl(s);
}

double or_norm_fro_I_plus(int64_t n, const int64_t *rp, const int32_t *ci, const double *v) {
  ocsr T = {n, (int64_t *)rp, (int32_t *)ci, (double *)v};
  return norm_fro_I_plus(&T);
}

/* Eq. (3.1): l1 = max (j - i), l2 = max (i - j) over nonzeros, 0 for the
 * zero matrix (reading R12). */
void or_bandwidth(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *l1, int64_t *l2) {
  int64_t a = 0, b = 0;
  for (int64_t i = 0; i < n; i++)
    for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
      int64_t d = (int64_t)ci[p] - i;
      if (d > a) a = d;
      if (-d > b) b = -d;
    }
  *l1 = a;
  *l2 = b;
}

/* ------------------------------------------------------------------------- */
/* Error model §4.1                                                          */
/* ------------------------------------------------------------------------- */

/* Eq. (4.5): r0(x, M) = (1/M!) sum_{i>=0} x^{M+1+i} / (i! (i+M+1)),
 * summed by the term recurrence
 *   term_0 = x^{M+1} / (M! (M+1)),
 *   term_{i+1} = term_i * x (i+M+1) / ((i+1)(i+M+2)),
 * until a term no longer changes the long-double partial sum. */
long double or_r0(long double x, int M) {
  if (x <= 0.0L) return 0.0L;
  long double t = 1.0L;
  for (int s = 1; s <= M; s++) t *= x / (long double)s; /* x^M / M! */
  t *= x / (long double)(M + 1);                       /* x^{M+1} / (M! (M+1)) */
  long double sum = 0.0L;
  for (int i = 0; i < 100000; i++) {
    long double ns = sum + t;
    if (ns == sum) break;
    sum = ns;
    t = t * x * (long double)(i + M + 1) / ((long double)(i + 1) * (long double)(i + M + 2));
  }
  return sum;
}

double or_r0_d(double x, int M) { return (double)or_r0((long double)x, M); }

/* Eq. (4.20): minimise M 2^N subject to ||H 2^-N|| <= 1 and
 * 2^N r0(||H|| 2^-N, M) <= eps_tol, N in [N0, N0 + n_window],
 * N0 = max(ceil(log2 ||H||), 0), M in [0, m_cap]; ties -> smaller N (R5).
 * Returns 0 on success, 1 if infeasible. ||H|| = 0 -> (0, 0). */
int or_plan(double norm, double eps_tol, int m_cap, int n_window, int *M_out, int *N_out) {
  if (norm == 0.0) {
    *M_out = 0;
    *N_out = 0;
    return 0;
  }
  int N0 = (int)ceil(log2(norm));
  if (N0 < 0) N0 = 0;
  while (ldexp(norm, -N0) > 1.0) N0++; /* guard log2 rounding */
  long double best = -1.0L;
  int bM = -1, bN = -1;
  for (int N = N0; N <= N0 + n_window; N++) {
    long double x = (long double)ldexp(norm, -N);
    for (int M = 0; M <= m_cap; M++) {
      long double r = ldexpl(or_r0(x, M), N);
      if (r <= (long double)eps_tol) {
        long double cost = (long double)M * ldexpl(1.0L, N);
        if (best < 0.0L || cost < best) {
          best = cost;
          bM = M;
          bN = N;
        }
        break; /* minimal M for this N */
      }
    }
  }
  if (bM < 0) return 1;
  *M_out = bM;
  *N_out = bN;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 4.1, literal.                                       */
/* ------------------------------------------------------------------------- */
/* Input: cnt values x (all stored entries of the matrix A, in row-major order).
 * Output: keep[p] = 1 for the entries of A~ = A - b_n.  Returns the number of
 * passes; *tau_final = last eps_f (entries kept are exactly |x| > tau_final);
 * *dropped = ||A - A~||_F.
 * Readings: R1 m_0 = 1 as printed and the first pass is unconditional:
 * Theorem 4.1's proof starts from "n = 0, m_0 = 1, eps_f^(1) = eps_g, b_1"
 * (P:384), and only then does ||A - A~|| <= eps_g (1 + e_r) hold for
 * every eps_g (the printed scalar b_0 = 1 would skip the loop and drop all of A
 * whenever eps_g (1 + e_r) >= 1).  Identical to the printed b_0 = 1 whenever
 * eps_g (1 + e_r) < 1.  R2 strict '>'.  R3 eps_g = 0 -> no filter. */
#define OR_MAX_PASSES 256
int or_alg41(int64_t cnt, const double *x, double eps_g, double e_r, uint8_t *keep,
             double *tau_final, double *dropped, double *tau_hist, int hist_cap) {
  if (eps_g == 0.0) { /* R3 */
    for (int64_t p = 0; p < cnt; p++) keep[p] = (x[p] != 0.0);
    *tau_final = 0.0;
    *dropped = 0.0;
    return 0;
  }
  /* step 1: m_0 = 1, n = 0, residual matrix b_0 = A (R1: first pass always runs) */
  uint8_t *in_res = (uint8_t *)malloc((size_t)(cnt > 0 ? cnt : 1));
  for (int64_t p = 0; p < cnt; p++) in_res[p] = 1;
  long double m = 1.0L, b = 1.0L;
  long double eg = eps_g;
  long double epsf = INFINITY;
  int n = 0;
  /* step 2 (R1: tested after each pass, the first pass unconditional) */
  do {
    epsf = eg / m;                             /* eps_f^{(n+1)} = eps_g / m_n */
    long double s = 0.0L;
    for (int64_t p = 0; p < cnt; p++) {
      if (!in_res[p]) continue;
      if (fabsl((long double)x[p]) > epsf) {   /* p = find(|b_n| > eps_f) */
        in_res[p] = 0;                         /* b_n(p) = 0 */
      } else {
        s += (long double)x[p] * (long double)x[p];
      }
    }
    b = sqrtl(s);                              /* b_{n+1} = ||b_{n+1}||_F */
    m = b / epsf;                              /* m_{n+1} = b_{n+1} / eps_f */
    if (n < hist_cap && tau_hist) tau_hist[n] = (double)epsf;
    n++;
    if (n >= OR_MAX_PASSES) break;             /* Theorem 4.1 guard; never hit in tests */
  } while (b > eg * (1.0L + (long double)e_r));
  /* step 3: A~ = A - b_n */
  long double d = 0.0L;
  for (int64_t p = 0; p < cnt; p++) {
    keep[p] = (uint8_t)(!in_res[p]);
    if (in_res[p]) d += (long double)x[p] * (long double)x[p];
  }
  *tau_final = (double)epsf;
  *dropped = (double)sqrtl(d);
  free(in_res);
  return n;
}

static ocsr csr_select(const ocsr *A, const uint8_t *keep) {
  int64_t nnz = 0;
  for (int64_t p = 0; p < csr_nnz(A); p++) nnz += keep[p];
  ocsr B = csr_alloc(A->n, nnz);
  int64_t q = 0;
  for (int64_t i = 0; i < A->n; i++) {
    for (int64_t p = A->rowptr[i]; p < A->rowptr[i + 1]; p++)
      if (keep[p]) {
        B.col[q] = A->col[p];
        B.val[q] = A->val[p];
        q++;
      }
    B.rowptr[i + 1] = q;
  }
  return B;
}

/* ------------------------------------------------------------------------- */
/* Row-wise products (Gustavson with a dense scatter workspace, SPEC design)  */
/* ------------------------------------------------------------------------- */
typedef struct {
  double *acc;
  uint8_t *mark;
  int32_t *list;
} workspace;

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* C = self_coef * A + A * B, then every value divided by `divisor`.
 * Row r: the accumulator starts with self_coef * a_rj (if self_coef != 0),
 * then adds a_rk * b_kj for k ascending in row r of A, j ascending in row k
 * of B (Eq. 2.7 / 4.15 with self_coef = 2, divisor = 1; Eq. 4.11 with
 * self_coef = 0, divisor = i — reading R7: divide after accumulation).
 * Exact zeros are purged (R11). */
static ocsr spgemm_rows(const ocsr *A, const ocsr *B, double self_coef, double divisor,
                        int nthreads) {
  int64_t n = A->n;
  int32_t **rc = (int32_t **)calloc((size_t)n, sizeof(int32_t *));
  double **rv = (double **)calloc((size_t)n, sizeof(double *));
  int64_t *rn = (int64_t *)calloc((size_t)n, sizeof(int64_t));
#ifdef _OPENMP
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
#endif
  {
    workspace w;
    w.acc = (double *)calloc((size_t)n, sizeof(double));
    w.mark = (uint8_t *)calloc((size_t)n, 1);
    w.list = (int32_t *)malloc((size_t)n * sizeof(int32_t));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
    for (int64_t r = 0; r < n; r++) {
      int64_t cnt = 0;
      if (self_coef != 0.0) {
        for (int64_t p = A->rowptr[r]; p < A->rowptr[r + 1]; p++) {
          int32_t j = A->col[p];
          w.acc[j] = self_coef * A->val[p];
          w.mark[j] = 1;
          w.list[cnt++] = j;
        }
      }
      for (int64_t p = A->rowptr[r]; p < A->rowptr[r + 1]; p++) {
        int32_t k = A->col[p];
        double a = A->val[p];
        for (int64_t q = B->rowptr[k]; q < B->rowptr[k + 1]; q++) {
          int32_t j = B->col[q];
          if (!w.mark[j]) {
            w.mark[j] = 1;
            w.acc[j] = 0.0;
            w.list[cnt++] = j;
          }
          double prod = a * B->val[q];
          w.acc[j] = w.acc[j] + prod;
        }
      }
      qsort(w.list, (size_t)cnt, sizeof(int32_t), cmp_i32);
      int64_t keep = 0;
      for (int64_t t = 0; t < cnt; t++) {
        double v = w.acc[w.list[t]] / divisor;
        if (v != 0.0) keep++;
      }
      rc[r] = (int32_t *)malloc((size_t)(keep > 0 ? keep : 1) * sizeof(int32_t));
      rv[r] = (double *)malloc((size_t)(keep > 0 ? keep : 1) * sizeof(double));
      int64_t q = 0;
      for (int64_t t = 0; t < cnt; t++) {
        int32_t j = w.list[t];
        double v = w.acc[j] / divisor;
        if (v != 0.0) {
          rc[r][q] = j;
          rv[r][q] = v;
          q++;
        }
        w.mark[j] = 0;
        w.acc[j] = 0.0;
      }
      rn[r] = keep;
    }
    free(w.acc);
    free(w.mark);
    free(w.list);
  }
  int64_t nnz = 0;
  for (int64_t r = 0; r < n; r++) nnz += rn[r];
  ocsr C = csr_alloc(n, nnz);
  int64_t q = 0;
  for (int64_t r = 0; r < n; r++) {
    memcpy(C.col + q, rc[r], (size_t)rn[r] * sizeof(int32_t));
    memcpy(C.val + q, rv[r], (size_t)rn[r] * sizeof(double));
    q += rn[r];
    C.rowptr[r + 1] = q;
    free(rc[r]);
    free(rv[r]);
  }
  free(rc);
  free(rv);
  free(rn);
  return C;
}

/* C = A + B (exact merge; sums that are exactly zero are purged, R11). */
static ocsr csr_add(const ocsr *A, const ocsr *B) {
  int64_t n = A->n;
  ocsr C = csr_alloc(n, csr_nnz(A) + csr_nnz(B));
  int64_t q = 0;
  for (int64_t r = 0; r < n; r++) {
    int64_t p = A->rowptr[r], pe = A->rowptr[r + 1];
    int64_t s = B->rowptr[r], se = B->rowptr[r + 1];
    while (p < pe || s < se) {
      int32_t j;
      double v;
      if (s >= se || (p < pe && A->col[p] < B->col[s])) {
        j = A->col[p];
        v = A->val[p++];
      } else if (p >= pe || B->col[s] < A->col[p]) {
        j = B->col[s];
        v = B->val[s++];
      } else {
        j = A->col[p];
        v = A->val[p++] + B->val[s++];
      }
      if (v != 0.0) {
        C.col[q] = j;
        C.val[q] = v;
        q++;
      }
    }
    C.rowptr[r + 1] = q;
  }
  return C;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 4.2                                                  */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t plan_norm;      /* 0 = 1-norm (BASELINE default), 1 = Frobenius */
  int32_t normal;         /* -1 auto (bit-exact symmetric or skew-symmetric), 0, 1 */
  int32_t threshold_mode; /* 0 = REL_PREV a r_i ||I+T^_{i-1}||_F (R4), 1 = ABS a r_i */
  int32_t filter;         /* 1 = filtered (paper), 0 = unfiltered PIM (eps_g = 0) */
  int32_t m_cap, n_window;
  int32_t force_M, force_N; /* -1 = use Eq. (4.20) */
  int32_t output_T;       /* 1 = return T^_N, 0 = E = I + T^_N */
  int32_t nthreads;
  int32_t ssat;           /* 1 = SSAT baseline (Table 1): E_0 = I + T^_0, E_i = E_{i-1}^2 */
  double e_r;             /* Algorithm 4.1 tolerance (R6: 0.1) */
} or_options;

#define OR_MAXSTEP 160
typedef struct {
  int32_t status; /* 0 ok, 1 infeasible plan, 2 bad input, 3 eps_tol < u */
  int32_t M, N, M_eff, normal;
  double norm, a, r0, eps_g0;
  /* Taylor terms i = 2..M stored at index i */
  int64_t taylor_nnz_unf[OR_MAXSTEP], taylor_nnz[OR_MAXSTEP];
  int32_t taylor_passes[OR_MAXSTEP];
  double taylor_tau[OR_MAXSTEP], taylor_dropped[OR_MAXSTEP];
  int64_t taylor_l1[OR_MAXSTEP], taylor_l2[OR_MAXSTEP];
  /* squarings i = 1..N stored at index i; index 0 = T^_0 */
  int64_t sq_nnz_unf[OR_MAXSTEP], sq_nnz[OR_MAXSTEP];
  int32_t sq_passes[OR_MAXSTEP];
  double sq_eps_g[OR_MAXSTEP], sq_tau[OR_MAXSTEP], sq_dropped[OR_MAXSTEP], sq_normIT[OR_MAXSTEP];
  int64_t sq_l1[OR_MAXSTEP], sq_l2[OR_MAXSTEP];
  double sq_fmas[OR_MAXSTEP];
} or_trace;

typedef struct {
  ocsr out;
  or_trace tr;
} or_result;

static int is_symmetric_sign(const ocsr *H, double sign) {
  /* H == sign * H^T bit-exactly (binary search in the sorted transpose row) */
  for (int64_t i = 0; i < H->n; i++)
    for (int64_t p = H->rowptr[i]; p < H->rowptr[i + 1]; p++) {
      int64_t j = H->col[p];
      int64_t lo = H->rowptr[j], hi = H->rowptr[j + 1];
      int found = 0;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (H->col[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      if (lo < H->rowptr[j + 1] && H->col[lo] == i && H->val[lo] == sign * H->val[p]) found = 1;
      if (!found) return 0;
    }
  return 1;
}

static double count_fmas(const ocsr *A, const ocsr *B) {
  double f = 0;
  for (int64_t p = 0; p < csr_nnz(A); p++) f += (double)(B->rowptr[A->col[p] + 1] - B->rowptr[A->col[p]]);
  return f;
}

static void filter_inplace(ocsr *S, double eps_g, double e_r, int32_t *passes, double *tau,
                           double *dropped) {
  int64_t nnz = csr_nnz(S);
  uint8_t *keep = (uint8_t *)malloc((size_t)(nnz > 0 ? nnz : 1));
  *passes = or_alg41(nnz, S->val, eps_g, e_r, keep, tau, dropped, NULL, 0);
  ocsr F = csr_select(S, keep);
  free(keep);
  csr_free(S);
  *S = F;
}

or_result *or_expm(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   double eps_tol, const or_options *o) {
  or_result *R = (or_result *)calloc(1, sizeof(or_result));
  or_trace *tr = &R->tr;
  ocsr H = csr_copy_in(n, rp, ci, v);
  for (int64_t p = 0; p < csr_nnz(&H); p++)
    if (!isfinite(H.val[p])) tr->status = 2;
  if (!(eps_tol >= 1e-16) || !isfinite(eps_tol)) tr->status = 3; /* R13: eps_tol >= u read as 1e-16 */
  if (o->ssat && o->output_T) tr->status = 2; /* SSAT has no incremental part to return */
  if (tr->status) {
    R->out = csr_alloc(n, 0);
    csr_free(&H);
    return R;
  }
  /* Step 1: M, N from Eq. (4.20) */
  double norm = (o->plan_norm == 0) ? or_norm_one(n, H.rowptr, H.col, H.val)
                                    : or_norm_fro(n, H.rowptr, H.col, H.val);
  int M, N;
  if (or_plan(norm, eps_tol, o->m_cap, o->n_window, &M, &N)) {
    tr->status = 1;
    R->out = csr_alloc(n, 0);
    csr_free(&H);
    return R;
  }
  if (o->force_M >= 0) M = o->force_M;
  if (o->force_N >= 0) N = o->force_N;
  tr->M = M;
  tr->N = N;
  tr->norm = norm;
  /* Step 2: a = 1/(1+N) if H normal, else ||H||^{-1} (R8: min(1, 1/||H||)) */
  int normal = o->normal;
  if (normal < 0) normal = is_symmetric_sign(&H, 1.0) || is_symmetric_sign(&H, -1.0);
  tr->normal = normal;
  double a;
  if (normal) a = 1.0 / (1.0 + (double)N);
  else a = (norm > 1.0) ? 1.0 / norm : 1.0;
  tr->a = a;
  /* Step 3: H0 = H 2^-N, S1 = H0, T0 = S1 */
  ocsr H0 = csr_copy_in(n, H.rowptr, H.col, H.val);
  for (int64_t p = 0; p < csr_nnz(&H0); p++) H0.val[p] = ldexp(H0.val[p], -N);
  double normH0 = ldexp(norm, -N);
  long double r0 = or_r0((long double)normH0, M);
  tr->r0 = (double)r0;
  double eps_g0 = 0.0;
  if (M >= 1) eps_g0 = (double)((long double)a * r0 / ((long double)M * expl(2.0L * (long double)normH0)));
  if (!o->filter) eps_g0 = 0.0;
  tr->eps_g0 = eps_g0;
  ocsr T;
  int M_eff = 0;
  if (M == 0) { /* R9: M = 0 -> T0 = 0 */
    T = csr_alloc(n, 0);
  } else {
    T = csr_copy_in(n, H0.rowptr, H0.col, H0.val);
    ocsr S = csr_copy_in(n, H0.rowptr, H0.col, H0.val);
    M_eff = 1;
    for (int i = 2; i <= M; i++) {
      /* S~_i = S^_{i-1} H0 / i */
      ocsr St = spgemm_rows(&S, &H0, 0.0, (double)i, o->nthreads);
      csr_free(&S);
      S = St;
      if (i < OR_MAXSTEP) tr->taylor_nnz_unf[i] = csr_nnz(&S);
      /* Algorithm 4.1 with eps_g^(0) */
      int32_t ps;
      double tau, dr;
      filter_inplace(&S, eps_g0, o->e_r, &ps, &tau, &dr);
      if (i < OR_MAXSTEP) {
        tr->taylor_nnz[i] = csr_nnz(&S);
        tr->taylor_passes[i] = ps;
        tr->taylor_tau[i] = tau;
        tr->taylor_dropped[i] = dr;
        or_bandwidth(n, S.rowptr, S.col, &tr->taylor_l1[i], &tr->taylor_l2[i]);
      }
      if (csr_nnz(&S) == 0) break; /* over-scaling: S^_i = 0 => all later terms 0 */
      M_eff = i;
      /* T^_0^(i) = T^_0^(i-1) + S^_i */
      ocsr Tn = csr_add(&T, &S);
      csr_free(&T);
      T = Tn;
    }
    csr_free(&S);
  }
  tr->M_eff = M_eff;
  tr->sq_nnz[0] = csr_nnz(&T);
  tr->sq_normIT[0] = norm_fro_I_plus(&T);
  or_bandwidth(n, T.rowptr, T.col, &tr->sq_l1[0], &tr->sq_l2[0]);
  if (o->ssat) {
    /* SSAT, the paper's scaling-and-squaring baseline (Table 1 column "SSAT", P:442-451;
     * SURVEY §8(f) N2): the same Taylor phase, then E_0 = I + T^_0 and N plain squarings
     * E_i = E_{i-1} E_{i-1} (rows in ascending k, Eq. 2.5's S(H)^2 without the incremental
     * split of Eq. 2.7), no filter; exact zeros purged (R11). */
    ocsr I = csr_alloc(n, n);
    for (int64_t r = 0; r < n; r++) {
      I.col[r] = (int32_t)r;
      I.val[r] = 1.0;
      I.rowptr[r + 1] = r + 1;
    }
    ocsr E = csr_add(&T, &I);
    csr_free(&I);
    csr_free(&T);
    for (int i = 1; i <= N; i++) {
      double fm = count_fmas(&E, &E);
      ocsr Et = spgemm_rows(&E, &E, 0.0, 1.0, o->nthreads);
      csr_free(&E);
      E = Et;
      int32_t ps;
      double tau, dr;
      filter_inplace(&E, 0.0, o->e_r, &ps, &tau, &dr);
      if (i < OR_MAXSTEP) {
        tr->sq_nnz_unf[i] = csr_nnz(&E);
        tr->sq_nnz[i] = csr_nnz(&E);
        tr->sq_fmas[i] = fm;
        or_bandwidth(n, E.rowptr, E.col, &tr->sq_l1[i], &tr->sq_l2[i]);
      }
    }
    R->out = E;
    csr_free(&H);
    csr_free(&H0);
    return R;
  }
  /* Step 4: squarings */
  long double ri = r0;
  for (int i = 1; i <= N; i++) {
    ri = 2.0L * ri; /* r_i = 2 r_{i-1} */
    double eps_g;
    if (o->threshold_mode == 1) eps_g = (double)((long double)a * ri);
    else eps_g = (double)((long double)a * ri * (long double)norm_fro_I_plus(&T));
    if (!o->filter) eps_g = 0.0;
    double fm = count_fmas(&T, &T);
    /* T~_i = 2 T^_{i-1} + T^_{i-1}^2 (Eq. 4.15; R10 index typo) */
    ocsr Tt = spgemm_rows(&T, &T, 2.0, 1.0, o->nthreads);
    csr_free(&T);
    T = Tt;
    int32_t ps;
    double tau, dr;
    int64_t nu = csr_nnz(&T);
    filter_inplace(&T, eps_g, o->e_r, &ps, &tau, &dr);
    if (i < OR_MAXSTEP) {
      tr->sq_nnz_unf[i] = nu;
      tr->sq_nnz[i] = csr_nnz(&T);
      tr->sq_passes[i] = ps;
      tr->sq_eps_g[i] = eps_g;
      tr->sq_tau[i] = tau;
      tr->sq_dropped[i] = dr;
      tr->sq_fmas[i] = fm;
      tr->sq_normIT[i] = norm_fro_I_plus(&T);
      or_bandwidth(n, T.rowptr, T.col, &tr->sq_l1[i], &tr->sq_l2[i]);
    }
  }
  /* Step 5: e^H = I + T^_N */
  if (o->output_T) {
    R->out = T;
  } else {
    ocsr I = csr_alloc(n, n);
    for (int64_t r = 0; r < n; r++) {
      I.col[r] = (int32_t)r;
      I.val[r] = 1.0;
      I.rowptr[r + 1] = r + 1;
    }
    R->out = csr_add(&T, &I);
    csr_free(&I);
    csr_free(&T);
  }
  csr_free(&H);
  csr_free(&H0);
  return R;
}

/* Accessors for ctypes */
int64_t or_result_nnz(const or_result *R) { return csr_nnz(&R->out); }
int64_t or_result_n(const or_result *R) { return R->out.n; }
void or_result_copy(const or_result *R, int64_t *rp, int32_t *ci, double *v) {
  memcpy(rp, R->out.rowptr, (size_t)(R->out.n + 1) * sizeof(int64_t));
  memcpy(ci, R->out.col, (size_t)csr_nnz(&R->out) * sizeof(int32_t));
  memcpy(v, R->out.val, (size_t)csr_nnz(&R->out) * sizeof(double));
}
const or_trace *or_result_trace(const or_result *R) { return &R->tr; }
void or_result_free(or_result *R) {
  if (!R) return;
  csr_free(&R->out);
  free(R);
}
int or_trace_size(void) { return (int)sizeof(or_trace); }
int or_options_size(void) { return (int)sizeof(or_options); }

/* Building blocks exported for the pin tests. */
static or_result *wrap(ocsr C) {
  or_result *R = (or_result *)calloc(1, sizeof(or_result));
  R->out = C;
  return R;
}
or_result *or_spgemm(int64_t n, const int64_t *arp, const int32_t *aci, const double *av,
                     const int64_t *brp, const int32_t *bci, const double *bv, double self_coef,
                     double divisor, int nthreads) {
  ocsr A = {n, (int64_t *)arp, (int32_t *)aci, (double *)av};
  ocsr B = {n, (int64_t *)brp, (int32_t *)bci, (double *)bv};
  return wrap(spgemm_rows(&A, &B, self_coef, divisor, nthreads));
}
or_result *or_add(int64_t n, const int64_t *arp, const int32_t *aci, const double *av,
                  const int64_t *brp, const int32_t *bci, const double *bv) {
  ocsr A = {n, (int64_t *)arp, (int32_t *)aci, (double *)av};
  ocsr B = {n, (int64_t *)brp, (int32_t *)bci, (double *)bv};
  return wrap(csr_add(&A, &B));
}

/* ------------------------------------------------------------------------- */
/* N1 apply: one step of the discretised system            */
/*   u_{k+1} = e^H u_k            (Eq. 2.2; validation of P:501-503)   */
/* for a block of m vectors: Y = A X, A CSR (n x n), X, Y dense row-major    */
/* (n x m).  Y(r, j) = sum over the entries of row r in ascending column     */
/* order of a_rk * X(k, j), starting from 0 (products rounded separately,    */
/* -ffp-contract=off).  steps > 1 applies A `steps` times: Y = A^steps X.    */
/* Parity pinned by tests/test_oracle_apply.py (dense matmul, E^k = e^{kH},  */
/* E 1 = 1 for zero-row-sum generators).                                     */
/* ------------------------------------------------------------------------- */
static void spmm_once(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                      int64_t m, const double *X, double *Y) {
  for (int64_t r = 0; r < n; r++) {
    for (int64_t j = 0; j < m; j++) {
      double y = 0.0;
      for (int64_t p = rp[r]; p < rp[r + 1]; p++) y = y + v[p] * X[(int64_t)ci[p] * m + j];
      Y[r * m + j] = y;
    }
  }
}

int or_spmm(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, int64_t m,
            const double *X, double *Y, int steps) {
  if (n < 0 || m < 0 || steps < 1) return 1;
  if (steps == 1) {
    spmm_once(n, rp, ci, v, m, X, Y);
    return 0;
  }
  double *a = (double *)malloc(sizeof(double) * (size_t)(n * m > 0 ? n * m : 1));
  double *b = (double *)malloc(sizeof(double) * (size_t)(n * m > 0 ? n * m : 1));
  if (!a || !b) {
    free(a);
    free(b);
    return 2;
  }
  const double *src = X;
  for (int s = 1; s <= steps; s++) {
    double *dst = s == steps ? Y : (s & 1 ? a : b);
    spmm_once(n, rp, ci, v, m, src, dst);
    src = dst;
  }
  free(a);
  free(b);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* N3 reordering: reverse Cuthill-McKee, the standard      */
/* heuristic for the real bandwidth lambda(A) = min_P l(P A P^T) of Def. 3.2a */
/* (P:134-136), whose computation is NP-hard.  Graph: the pattern of A + A^T */
/* without the diagonal.  Deterministic rules (the GPU follows the same):    */
/*  - components are started in ascending order of their smallest-degree,   */
/*    smallest-index unvisited node (isolated nodes are components too);     */
/*  - the start node is pseudo-peripheral (George-Liu): BFS from the        */
/*    candidate, take the last level's smallest-degree, smallest-index node,  */
/*    repeat while the number of levels grows;                               */
/*  - Cuthill-McKee: BFS levels in order; inside level L+1 the nodes are      */
/*    ordered by (smallest CM position of a neighbour in level L, degree,     */
/*    index);                                                                */
/*  - the whole CM sequence is reversed.  perm[new] = old.                   */
/* Pinned by tests/test_oracle_rcm.py (a permutation; bandwidth of banded   */
/* matrices under random relabelling restored; vs scipy's RCM bandwidth).   */
/* ------------------------------------------------------------------------- */
static int bfs_levels(int64_t n, const int64_t *rp, const int32_t *ci, int64_t s,
                      int32_t *level, int64_t *queue, int64_t *qlen) {
  /* level[] must be -1 on the component; returns the number of levels */
  int64_t head = 0, tail = 0;
  queue[tail++] = s;
  level[s] = 0;
  int maxl = 0;
  while (head < tail) {
    int64_t v = queue[head++];
    for (int64_t p = rp[v]; p < rp[v + 1]; p++) {
      int64_t u = ci[p];
      if (level[u] < 0) {
        level[u] = level[v] + 1;
        if (level[u] > maxl) maxl = level[u];
        queue[tail++] = u;
      }
    }
  }
  *qlen = tail;
  (void)n;
  return maxl + 1;
}

int or_rcm(int64_t n, const int64_t *rp0, const int32_t *ci0, int64_t *perm) {
  /* symmetric pattern G = pattern(A + A^T) minus the diagonal, rows sorted */
  int64_t nnz = rp0[n];
  int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t r = 0; r < n; r++)
    for (int64_t p = rp0[r]; p < rp0[r + 1]; p++)
      if (ci0[p] != r) {
        cnt[r + 1]++;
        cnt[ci0[p] + 1]++;
      }
  for (int64_t r = 0; r < n; r++) cnt[r + 1] += cnt[r];
  int32_t *adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cnt[n] > 0 ? cnt[n] : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t r = 0; r < n; r++) fill[r] = cnt[r];
  for (int64_t r = 0; r < n; r++)
    for (int64_t p = rp0[r]; p < rp0[r + 1]; p++)
      if (ci0[p] != r) {
        adj[fill[r]++] = ci0[p];
        adj[fill[ci0[p]]++] = (int32_t)r;
      }
  /* sort + dedupe each row */
  int64_t *rp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t w = 0;
  for (int64_t r = 0; r < n; r++) {
    int64_t b = cnt[r], e = fill[r];
    qsort(adj + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    rp[r] = w;
    for (int64_t p = b; p < e; p++)
      if (p == b || adj[p] != adj[p - 1]) adj[w++] = adj[p];
  }
  rp[n] = w;
  (void)nnz;
  int64_t *deg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t r = 0; r < n; r++) deg[r] = rp[r + 1] - rp[r];
  int32_t *level = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t *done = (int32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
  int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t *cm = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t ncm = 0;
  for (int64_t r = 0; r < n; r++) level[r] = -1;
  for (;;) {
    /* next component: smallest (degree, index) among unplaced nodes */
    int64_t s = -1;
    for (int64_t r = 0; r < n; r++)
      if (!done[r] && (s < 0 || deg[r] < deg[s])) s = r;
    if (s < 0) break;
    /* pseudo-peripheral start (George-Liu) */
    int64_t qlen;
    int nl = bfs_levels(n, rp, adj, s, level, queue, &qlen);
    for (;;) {
      int64_t c = -1;
      for (int64_t q = 0; q < qlen; q++) {
        int64_t v = queue[q];
        if (level[v] == nl - 1 && (c < 0 || deg[v] < deg[c] || (deg[v] == deg[c] && v < c))) c = v;
      }
      for (int64_t q = 0; q < qlen; q++) level[queue[q]] = -1;
      int64_t ql2;
      int nl2 = bfs_levels(n, rp, adj, c, level, queue, &ql2);
      if (nl2 > nl) {
        s = c;
        nl = nl2;
        qlen = ql2;
      } else {
        for (int64_t q = 0; q < ql2; q++) level[queue[q]] = -1;
        bfs_levels(n, rp, adj, s, level, queue, &qlen);
        break;
      }
    }
    /* Cuthill-McKee over the levels of s */
    int64_t lstart = ncm;
    cm[ncm] = s;
    pos[s] = ncm;
    ncm++;
    for (int L = 1; L < nl; L++) {
      int64_t b = ncm;
      for (int64_t q = 0; q < qlen; q++) {
        int64_t v = queue[q];
        if (level[v] == L) cm[ncm++] = v;
      }
      /* insertion sort by (key, degree, index), key = smallest CM position of a neighbour
       * in level L-1: plain and obviously correct */
      for (int64_t a = b + 1; a < ncm; a++) {
        int64_t v = cm[a];
        int64_t j = a - 1;
        while (j >= b) {
          int64_t u = cm[j];
          int64_t ku = INT64_MAX, kv = INT64_MAX;
          for (int64_t p = rp[u]; p < rp[u + 1]; p++)
            if (level[adj[p]] == L - 1 && pos[adj[p]] < ku) ku = pos[adj[p]];
          for (int64_t p = rp[v]; p < rp[v + 1]; p++)
            if (level[adj[p]] == L - 1 && pos[adj[p]] < kv) kv = pos[adj[p]];
          int gt = ku > kv || (ku == kv && (deg[u] > deg[v] || (deg[u] == deg[v] && u > v)));
          if (!gt) break;
          cm[j + 1] = u;
          j--;
        }
        cm[j + 1] = v;
      }
      for (int64_t a = b; a < ncm; a++) pos[cm[a]] = a;
    }
    for (int64_t a = lstart; a < ncm; a++) done[cm[a]] = 1;
    for (int64_t a = lstart; a < ncm; a++) level[cm[a]] = -1;
  }
  for (int64_t a = 0; a < n; a++) perm[a] = cm[n - 1 - a];
  free(cnt); free(adj); free(fill); free(rp); free(deg); free(level); free(done); free(queue);
  free(cm); free(pos);
  return 0;
}
