// kernels.cuh — internal launchers of the sm_100a kernels of libsexpm.
// Each launcher enqueues on `st` and never synchronises.  See kernels.cu for the
// paper passage every kernel implements.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace sx {

extern std::atomic<long long> g_kernel_launches;  // incremented by every launcher

constexpr int kThreads = 256;                 // row kernels: 8 warps per CTA
constexpr int kWarps = kThreads / 32;

// Device CSR view over a contiguous block of rows. Row r of the view is global row
// row0 + r; columns are global.
struct CsrView {
  int64_t nrows = 0;
  int64_t row0 = 0;
  int64_t nnz = 0;
  const int64_t *rp = nullptr;
  const int32_t *col = nullptr;
  const double *val = nullptr;
};

// --- K8: norms, validation, transpose-based checks (plan time) --------------------
void launch_validate(const CsrView &A, int64_t n, int *flags, cudaStream_t st);
void launch_col_count(const CsrView &A, int32_t *cnt, cudaStream_t st);
void launch_transpose_fill(const CsrView &A, int64_t *cursor, int32_t *trow, double *tval,
                           cudaStream_t st);
void launch_sort_columns(int64_t ncols, const int64_t *cp, int32_t *trow, double *tval,
                         cudaStream_t st);
void launch_col_abs_sum(int64_t ncols, const int64_t *cp, const double *tval, double *out,
                        cudaStream_t st);
void launch_compare_transpose(const CsrView &A, const int64_t *cp, const int32_t *trow,
                              const double *tval, int *flags, cudaStream_t st);
// deterministic reductions into out[0] (fixed grid, fixed order)
void launch_reduce_max(const double *x, int64_t cnt, double *partial, double *out,
                       cudaStream_t st);
void launch_reduce_sumsq(const double *x, int64_t cnt, double *partial, double *out,
                         cudaStream_t st);
void launch_reduce_sum(const double *x, int64_t cnt, double *partial, double *out,
                       cudaStream_t st);
void launch_reduce_max_i64(const int64_t *x, int64_t cnt, int64_t *out, cudaStream_t st);
void launch_reduce_sum_i64(const int64_t *x, int64_t cnt, int64_t *out, cudaStream_t st);
void launch_scale_pow2(double *v, int64_t cnt, int e, cudaStream_t st);
void launch_row_lengths(const int64_t *rp, int64_t nrows, int64_t *out, cudaStream_t st);
void launch_rowlen_sq(const int64_t *rp, int64_t nrows, int64_t *out, cudaStream_t st);  // out[r] = len(r)^2
void launch_copy_i64_offset(const int64_t *src, int64_t cnt, int64_t off, int64_t *dst,
                            cudaStream_t st);

// --- scan ------------------------------------------------------------------------
// exclusive scan of cnt int64 values into out[0..cnt]; out[cnt] = total.
// tmp needs scan_tmp_elems(cnt) int64s.
int64_t scan_tmp_elems(int64_t cnt);
void launch_exclusive_scan(const int64_t *in, int64_t cnt, int64_t *out, int64_t *tmp,
                           cudaStream_t st);

// --- K1 symbolic bound -----------------------------------------------------------
// For each row r of A: lo/hi = min/max column reachable (B rows of A's columns and, if
// self, A's own row), prod = sum of nnz(B row k) (+ nnz(A row)), bound = min(span, prod).
void launch_symbolic(const CsrView &A, const CsrView &B, int self, int32_t *lo, int32_t *hi,
                     int64_t *prod, int64_t *bound, cudaStream_t st);

// --- K2 binning ------------------------------------------------------------------
// order = row ids sorted by descending work (counting sort on floor(log2(work+1))).
void launch_bin_rows(int64_t nrows, const int64_t *work, int32_t *bin_cnt, int32_t *bin_off,
                     int32_t *order, cudaStream_t st);

// --- K3 numeric filtered SpGEMM with fused 2T add + classification ---------------
struct NumericArgs {
  CsrView A, B;
  double self_coef = 0.0;   // 2 for squaring (Eq. 4.15), 0 for Taylor (Eq. 4.11)
  double divisor = 1.0;     // i for Taylor terms, 1 otherwise
  double floor_tau = 0.0;   // entries with 0 < |x| <= floor_tau are dropped, x^2 summed
  const int32_t *lo = nullptr, *hi = nullptr;
  const int32_t *order = nullptr;
  int window = 8192;
  int64_t *cursor = nullptr;      // per-CTA scratch [grid][cursor_cap]
  int64_t cursor_cap = 0;
  int32_t *scr_col = nullptr;     // per-CTA staging [grid][scr_cap]
  double *scr_val = nullptr;
  int64_t scr_cap = 0;
  int32_t *pool_col = nullptr;    // global staging pool
  double *pool_val = nullptr;
  int64_t pool_cap = 0;
  unsigned long long *pool_used = nullptr;
  int64_t *row_off = nullptr;     // per row: offset in pool
  int64_t *row_cnt = nullptr;     // per row: staged count
  double *row_fsum = nullptr;     // per row: sum of x^2 below the floor
  int64_t *row_nnz = nullptr;     // per row: distinct nonzeros of C~
  int *row_counter = nullptr;     // dynamic scheduler
  int *flags = nullptr;           // flags[0] |= 1 on pool overflow, 2 on scratch overflow
  int grid = 0;
  int64_t nlist = 0;              // rows to process: order[0..nlist) (or 0..nlist)
  // first Algorithm 4.1 pass fused into the flush (kernels 5 and 7): per row, the sum of
  // x^2 over staged |x| <= eps_g (tau_1 = eps_g) and the count of staged |x| > eps_g
  double *row_p1 = nullptr;
  int64_t *row_c1 = nullptr;
  double eps_g = 0.0;
  const int32_t *gstart = nullptr;     // grouped kernels: group g = order[gstart[g], gstart[g+1])
  int64_t ngroups = 0;
  unsigned long long *prof = nullptr;  // optional phase clocks (grouped kernel): setup,
                                       // products, flush, groups, union k's, failed groups
};
int numeric_smem_bytes(int window);
void launch_numeric(const NumericArgs &a, cudaStream_t st);
// k-synchronous paged variant (no probing, sorted flush, bit-identical order)
int paged_smem_bytes();
void launch_numeric_paged(const NumericArgs &a, int32_t *fail_rows, int *fail_count,
                          cudaStream_t st);
// Taylor term by pull over H0^T (bit-identical order); BT = CSC of B (= B^T as CSR)
int taylor_pull_smem_bytes();
void launch_taylor_pull(const NumericArgs &a, const CsrView &BT, int32_t *fail_rows,
                        int *fail_count, cudaStream_t st);
// H0 as diagonals: val[di * n + k] = H0(k, k + off[di]) (0 where absent), off descending
struct DiaView {
  int ndiag = 0;
  const int32_t *off = nullptr;   // device, ndiag offsets, descending
  const double *val = nullptr;    // device, ndiag * n
  int64_t n = 0;
  int32_t dmin = 0, dmax = 0;
  unsigned long long *prod_count = nullptr;  // += products (a_rk h_kj pairs) computed
  int *need_max = nullptr;  // max over rows of the accumulator slots a row needed (span-fit rows)
};
constexpr int kDiaMax = 16;       // most offsets the diagonal kernel handles
constexpr int kDiaWarpsPerCta = 4;
// plan time: bitmap over offsets j - k + (n - 1) present in H; diagonals from offsets
void launch_mark_offsets(const CsrView &H, unsigned *bits, int64_t n, cudaStream_t st);
void launch_fill_dia(const CsrView &H, const int32_t *off_host, int nd, double *dia, int64_t n,
                     cudaStream_t st);
int taylor_dia_smem_bytes(int slots);
// Taylor term by diagonal push (bit-identical order); rows that do not fit -> fail_rows
void launch_taylor_dia(const NumericArgs &a, const DiaView &D, int slots, int32_t *fail_rows,
                       int *fail_count, cudaStream_t st);
// K5w: Taylor terms on the dense offset window (kernels.cu), position-major dense rows
struct WinArgs {
  int64_t nrows = 0, row0 = 0, n = 0;  // local rows, first global row, matrix order
  int nd = 0;
  const double *dia = nullptr;     // DiaView layout
  const int32_t *doff = nullptr;   // descending
  int dzero = -1;                  // index of the offset 0 in doff (-1: none)
  int prev_is_h0 = 0;              // S~_{i-1} = H0 (i = 2; FINAL with m = 1): read from dia
  const double *pS = nullptr;      // S~_{i-1}: [|W_{i-1}|][nrows]
  double tau_prev = 0.0;           // S^_{i-1} keeps |x| > tau_prev
  const double *T0old = nullptr;   // T^_0 over U: [|U| + 1][nrows] (the last plane zero),
  double *T0new = nullptr;         // updated in place (TERM: T0new == T0old)
  int c1cnt = 0;                   // |cum_{i-1}| (TERM) / |cum_m| (FINAL)
  const int16_t *mapC = nullptr;   // per cum position: its U-index if in the previous cum, or -1
  const int16_t *mapW = nullptr;   // per cum position: position in W_{i-1} (W_m), or -1
  const int16_t *cumU = nullptr;   // per cum position: its U-index (T^_0 is stored over U)
  const int32_t *coffs = nullptr;  // per cum position: its offset (FINAL)
  int sym = 0;                     // FINAL: lower entries read as their mirrors (K3s input)
  int half = 0;                    // half window (symmetric path): offsets o >= 0 only; each
                                   // off-diagonal value counted twice in the filter's sums
  int64_t plane = 0;               // S~ plane stride (rows + padr); 0: nrows
  int64_t padr = 0;                // zero rows in front of each S~ plane (mirrored reads)
  int ncnt = 0;                    // |W_i| (TERM)
  const int32_t *rec = nullptr;    // TERM: per position t of W_i a record of element offsets
                                   // (kernels.cu k_taylor_win; taylor_win_rec_words(nd) int32)
  const double *dpad = nullptr;    // H0's diagonals zero-padded: h_d(k) = dpad[di * npad + k]
                                   // (the pointer is at the padding's end: k may be negative)
  int32_t hoff[kDiaMax] = {0};     // di * npad - d_di
  int32_t hpad = 0;                // the padding (dpad - hpad is the array's start)
  double *nS = nullptr;            // S~_i: [|W_i|][nrows]
  double divisor = 1.0, floor_tau = 0.0, eps_g = 0.0;
  double *band_val = nullptr;      // [band_cap][nrows] staged floor < |x| <= eps_g
  int32_t *band_col = nullptr;
  int64_t band_cap = 0;
  unsigned long long *band_need = nullptr;  // atomicMax of a row's band count over band_cap
  int64_t *row_cnt = nullptr, *row_nnz = nullptr, *row_c1 = nullptr;
  double *row_fsum = nullptr, *row_p1 = nullptr;
  unsigned long long *prod_count = nullptr;
};
// the TERM kernel is compiled for 1..9 and 16 diagonals; records are built for that count
// (extra diagonals read the zero plane)
inline int taylor_win_kernel_nd(int nd) { return nd <= 9 ? nd : kDiaMax; }
int taylor_win_smem_bytes(int nd, int ncnt, int ccnt);
int taylor_win_rec_words(int nd);
void launch_taylor_win_t0(const WinArgs &a, cudaStream_t st);  // T^_0 update when 0 is not in D
// persistent grid of ctas_per_sm CTAs per SM over tiles of 128 rows
void launch_taylor_win(const WinArgs &a, int ctas_per_sm, int sms, cudaStream_t st);
// half: each staged value whose column is not its row's counted twice (its mirror)
void launch_win_band_pass(int64_t nl, const int64_t *cnt, const double *band_val, double tau, double *rowsum,
                          int64_t *rowcnt, cudaStream_t st, int half = 0, const int32_t *band_col = nullptr,
                          int64_t row0 = 0);
// FINAL: rp_out null -> per-row counts of T^_0 into cnt; else write T^_0's rows (CSR)
void launch_taylor_win_final(const WinArgs &a, int64_t *cnt, const int64_t *rp_out, int32_t *col_out,
                             double *val_out, cudaStream_t st);
void launch_count_above(const double *x, int64_t cnt, double tau, unsigned long long *out, cudaStream_t st);

// squaring order of a lattice-structured H (kernels.cu): 2D diamond tiles / 3D cubes of 8 rows
struct LatticeDesc {
  int dims = 0;              // 2 or 3
  int64_t n = 0;
  int64_t G = 0, Gy = 0;     // extents of the first two dimensions (row r = x + G y [+ G Gy z])
  int64_t GH = 0;            // G * Gy
  int64_t Dp = 0;            // 2D: even shift making x - y + Dp >= 0
  int64_t nv = 0, nv16 = 0;  // 2D: tiles / supertiles along v
  int64_t ntx = 0, nty = 0;  // 3D: tiles along x, y
  int64_t nx8 = 0, ny8 = 0;  // 3D: supertiles along x, y
  int64_t ntiles = 0, nsuper = 0;
};
// perm[new] = old, inv[old] = new, border = the block rows in supertile order (see kernels.cu
// for the scratch sizes)
void launch_lattice_order(const LatticeDesc &L, unsigned *mask, int64_t *cnt, int64_t *off, int64_t *scan_tmp,
                          int32_t *key, int32_t *scnt, int32_t *cur, int *flag, int64_t *perm, int64_t *inv,
                          int32_t *border, cudaStream_t st);
void launch_iota_i32(int64_t n, int32_t *x, cudaStream_t st);

// BSR-8 view (squarings on one GPU): conversion, block transpose, numeric kernel
struct BsrView {
  int64_t nbr = 0;
  const int64_t *brp = nullptr;
  const int32_t *bcol = nullptr;
  const double *bval = nullptr;
  const int64_t *tp = nullptr;
  const int32_t *tk = nullptr;
  const int64_t *tb = nullptr;
  const int32_t *border = nullptr;  // block rows in processing order (locality), or identity
  // the rows multiplied (A) may be a slice of the view's rows (B, e.g. a rank's rows inside
  // its halo): A has nbr_a block rows, its block row I is the view's block row I + ib0, and
  // the view's first block row is global block row kb0 (block columns are global)
  int64_t nbr_a = 0, ib0 = 0, kb0 = 0;
  // K3m only: A's own BSR view (Taylor terms S~ = S^ H0 / i: A = S^_{i-1}, B = H0); null when
  // A's blocks are B's rows (squarings)
  const int64_t *abrp = nullptr;
  const int32_t *abcol = nullptr;
  const double *abval = nullptr;
};
constexpr int kBsrScratchPerCta = 512 * 64;  // doubles of output-block scratch per CTA
constexpr int kBsrMaxRowBlocks = 136;        // blocks of a block row the numeric kernel holds
// optional relabelling fused into the BSR build: view row r = A's row rowmap[r], A's column c
// = the view's column colmap[c] (null: identity)
struct RowColMap {
  const int64_t *rowmap = nullptr, *colmap = nullptr;
};
void launch_bsr_count(const CsrView &A, int64_t nbr, int64_t *bcnt, int *flags, cudaStream_t st,
                      RowColMap map = RowColMap{});
// frag = true: values in K3m's tensor-core fragment order (see kernels.cu), else row-major
void launch_bsr_fill(const CsrView &A, int64_t nbr, const int64_t *brp, int32_t *bcol,
                     double *bval, int *flags, cudaStream_t st, bool frag = false,
                     RowColMap map = RowColMap{});
// tk_tmp / tb_tmp: nb-sized scratch; keys_out: nb int32 scratch; sort_tmp: bytes from
// bsr_transpose_temp_bytes(nb)
size_t bsr_transpose_temp_bytes(int64_t nb);
void launch_bsr_transpose(int64_t nbr, int64_t nbc, int64_t nb, const int64_t *brp,
                          const int32_t *bcol, int32_t *tcnt, int64_t *tp, int32_t *tk_tmp,
                          int64_t *tb_tmp, int32_t *tk, int64_t *tb, int64_t *scan_tmp,
                          int64_t *cnt64, void *sort_tmp, size_t sort_tmp_bytes, int32_t *keys_out,
                          cudaStream_t st);
int bsr_numeric_smem_bytes();
void launch_numeric_bsr(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                        int32_t *fail_rows, int *fail_count, cudaStream_t st);
// K3m: the block product on the fp64 tensor-core instruction (DMMA m8n8k4; BSR values in
// fragment order, launch_bsr_fill(frag = true)); no limit on the blocks of a row of A; scratch
// of kBsrMJCap * 66 doubles per CTA; rows it cannot hold -> fail_rows
constexpr int kBsrMJCap = 8192;              // output blocks per block row (K3m)
// K3m CTAs per SM: 4 (short match lists, 2 products in flight per operand set) or 2 (long
// lists: a block row of A with more than kBsrMLongRow blocks on average, 4 per set)
constexpr int kBsrMBlocksPerSm = 4, kBsrMBlocksPerSmLong = 2, kBsrMLongRow = 200;
int bsrm_numeric_smem_bytes();
void launch_numeric_bsrm(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                         int32_t *fail_rows, int *fail_count, cudaStream_t st, bool long_lists);

// K3s: the squaring of an exactly symmetric iterate T (T~ = 2T + T^2 is symmetric): K3m over
// the output blocks J >= I of every block row only.  Per block row I the candidate list
// cand(I) (all J, ascending) goes to cj[cj_off[I] ..), nlow[I] of them below I; the upper
// blocks C_IJ (raw, row-major 8 x 8) to bstore[(ob_off[I] + q - nlow[I]) * 64 ..].
// K3a then assembles every row r = 8I + i in column order -- column i of C_JI for J < I
// (found in J's list), the diagonal block mirrored from its upper triangle, row i of C_IJ
// for J > I -- classifies (Algorithm 4.1 floor, fused first pass) and stages exactly like the
// full kernels, so Algorithm 4.1 and the compaction run unchanged.
struct SymOut {
  double *bstore = nullptr;               // per upper block: its kept values, packed
  unsigned long long *bmask = nullptr;    // per upper block: kept elements (bit 8 row + col)
  double *fsI = nullptr;                  // per block row: dropped sum x^2 (mirrors counted)
  int64_t *nzI = nullptr;                 // per block row: distinct nonzeros (mirrors counted)
  int64_t *rowcnt = nullptr;              // per row: kept entries (K3s, atomics; zeroed before)
  const int64_t *rowoff = nullptr;        // its exclusive scan: the row's pool offset (K3a)
  int32_t *lidx = nullptr;                // per candidate (cj layout): a lower block's global index
  int32_t *cj = nullptr;
  const int64_t *ob_off = nullptr, *cj_off = nullptr;  // scans of K3c's counts
  const int64_t *nj = nullptr, *nup = nullptr;         // K3c: |cand(I)|, |cand(I) >= I|
  const int32_t *wlo = nullptr, *whi = nullptr;        // K3c: the union's block-column extent
  int *flag = nullptr;  // 1: a block row K3s or K3c could not hold, 2: K3s's list differs from
                        // K3c's count, 4: pattern not symmetric (a lower block missing from its
                        // mirror's list), 8: K3a's lower-list cap, 16: a row's count
};
// K3c: nj[I] = |cand(I)|, nup[I] = |cand(I) >= I| over the view's block rows (A = B)
// and the union's block-column extent [wlo, whi] (K3s's window: cand(I) is then the exact block
// union, symmetric for a symmetric block pattern)
void launch_sym_count(const BsrView &Bv, int64_t *nj, int64_t *nup, int32_t *wlo, int32_t *whi, int *flag,
                      cudaStream_t st, bool wide = false);
void launch_numeric_bsrm_sym(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                             const SymOut &so, cudaStream_t st, bool long_lists);
void launch_sym_lidx(const SymOut &so, int64_t nbr, cudaStream_t st);
// after K3s (+ lidx): Algorithm 4.1's pass over the store (psum per block row, x 2 mirrors)
void launch_sym_pass(const SymOut &so, int64_t nbr, double tau, double *psum, cudaStream_t st);
// the next squaring's BSR-8 view (fragment order) from the store, |x| > tau (kernels.cu)
struct SymFin {
  int64_t *bcnt = nullptr;                    // COUNT: non-empty blocks per block row (zeroed before)
  int64_t *rowcnt = nullptr;                  // COUNT: kept entries per row (zeroed before)
  uint8_t *flag = nullptr;                    // COUNT: per upper block, non-empty after tau
  double *rsI = nullptr;                      // COUNT: ||I + T^||_F^2 share of the block row
  int64_t *l1I = nullptr;                     // COUNT: bandwidth (symmetric: l1 = l2)
  const int64_t *brp = nullptr;               // WRITE: the scan of bcnt
  int32_t *bcol = nullptr;                    // WRITE
  double *bval = nullptr;                     // WRITE
};
void launch_sym_fin(const SymOut &so, int64_t nbr, int64_t nrows, double tau, const SymFin &f, bool write,
                    cudaStream_t st);
void launch_rowcnt_sq(const int64_t *rc, int64_t n, int64_t *sq, cudaStream_t st);  // sq[r] = rc[r]^2
// CSR rows of a fragment-order BSR view: counts (rp null) or the rows
void launch_bsr_to_csr(const BsrView &V, int64_t nrows, int64_t *cnt, const int64_t *rp, int32_t *col,
                       double *val, cudaStream_t st);
void launch_sym_assemble(const NumericArgs &a, const SymOut &so, int64_t nbr, int64_t nrows, int grid,
                         cudaStream_t st);
// T := the symmetric part read from the upper triangle: entry (r, c) kept iff (c, r) is
// present, value T(min(r,c), max(r,c)) (binary search in row c); count pass (cnt) or write
void launch_sym_intersect(const CsrView &A, int64_t *cnt, const int64_t *rp_out, int32_t *col_out,
                          double *val_out, cudaStream_t st);

// --- K6 Algorithm 4.1 pass -------------------------------------------------------
// out[0] = sum over x[0..cnt) of x^2 for |x| <= tau (deterministic order for fixed layout)
void launch_alg41_pass(const double *x, int64_t cnt, double tau, double *partial,
                       double *out, cudaStream_t st);

// the same pass summed per staged row (column order) then over rows in row order:
// independent of the order the product kernel staged rows in (run-to-run deterministic)
void launch_alg41_pass_rows(int64_t nrows, const int64_t *row_off, const int64_t *row_cnt,
                            const double *pool_val, double tau, double *rowsum, double *partial,
                            double *out, cudaStream_t st);

// --- K4 compaction -----------------------------------------------------------------
void launch_compact_count(int64_t nrows, const int64_t *row_off, const int64_t *row_cnt,
                          const double *pool_val, double tau, int64_t *cnt, cudaStream_t st);
// writes C rows; per-row stats: rs = ||row of (I + C)||^2 (identity on global row),
// l1r/l2r = max(col - row) / max(row - col) clamped at 0.
void launch_compact_write(int64_t nrows, int64_t row0, const int64_t *row_off,
                          const int64_t *row_cnt, const int32_t *pool_col,
                          const double *pool_val, double tau, const int64_t *rp_out,
                          int32_t *col_out, double *val_out, double *rs, int64_t *l1r,
                          int64_t *l2r, cudaStream_t st, const int8_t *ident = nullptr);
// E = I + T^_N fused into the last compaction: counts E's rows and records per-row
// diagonal status (0 insert 1.0, 1 write 1 + t, 2 purge) for launch_compact_write(ident).
void launch_compact_count_ident(int64_t nrows, int64_t row0, const int64_t *row_off,
                                const int64_t *row_cnt, const int32_t *pool_col,
                                const double *pool_val, double tau, int64_t *cnt, int8_t *ident,
                                cudaStream_t st);
// out2[0] = rows whose diagonal was inserted, out2[1] = rows whose diagonal was purged
void launch_count_ident(const int8_t *ident, int64_t nrows, int64_t *out2, cudaStream_t st);
// per-row ||row of (I + C)||^2 and bandwidth stats for an existing CSR
void launch_row_stats(const CsrView &C, double *rs, int64_t *l1r, int64_t *l2r,
                      cudaStream_t st);

// --- merge C = A + B (exact, zero sums purged): count then write ---------------------
void launch_merge_count(const CsrView &A, const CsrView &B, int64_t *cnt, cudaStream_t st);
void launch_merge_write(const CsrView &A, const CsrView &B, const int64_t *rp_out,
                        int32_t *col_out, double *val_out, cudaStream_t st);
// C = A + (staged S~ under tau), writing S^ (the kept staged entries) as well (Taylor terms).
// A's row r is A.col/val[A.rp[r] .. + alen[r]) (alen null: A.rp[r+1] - A.rp[r]); C's row r is
// written from rp_out[r] (a capacity offset) and its length stored in len_out[r]
void launch_merge_staged_count(const CsrView &A, const int64_t *alen, const int64_t *row_off,
                               const int64_t *row_cnt, const int32_t *pcol, const double *pval,
                               double tau, int64_t *cnt, cudaStream_t st);
void launch_merge_staged_write(const CsrView &A, const int64_t *alen, const int64_t *row_off,
                               const int64_t *row_cnt, const int32_t *pcol, const double *pval,
                               double tau, const int64_t *rp_out, int32_t *col_out, double *val_out,
                               int64_t *len_out, const int64_t *s_rp, int32_t *s_col, double *s_val,
                               cudaStream_t st);
// N1 apply: Y = A X, A CSR (rows A.nrows, global columns), X dense row-major (rows = A's
// column range, ldx >= m), Y row-major (A.nrows x m, ldy >= m)
// result copy-out by resident CTAs (false: pointers not 16-byte aligned, nothing launched)
bool launch_copy_out(void *dst, const void *src, size_t bytes, int ctas, cudaStream_t st);
void launch_spmm(const CsrView &A, int64_t m, const double *X, int64_t ldx, double *Y, int64_t ldy,
                 cudaStream_t st);
// N3 reverse Cuthill-McKee (driver.cu compute_rcm runs the level loop)
void launch_degree_nodiag(const CsrView &G, int32_t *deg, cudaStream_t st);
void launch_bfs_expand(const CsrView &G, int64_t *queue, int64_t a, int64_t b, int32_t *level,
                       int32_t L, unsigned long long *tail, cudaStream_t st);
void launch_min_deg(const int64_t *queue, int64_t a, int64_t b, const int32_t *deg,
                    const int8_t *done, unsigned long long *out, cudaStream_t st);
void launch_reset_level(const int64_t *queue, int64_t a, int64_t b, int32_t *level, cudaStream_t st);
void launch_cm_key(const CsrView &G, const int64_t *queue, int64_t a, int64_t b, const int32_t *level,
                   int32_t L, const int64_t *pos, const int32_t *deg, unsigned long long *key,
                   int32_t *ids, cudaStream_t st);
size_t cm_sort_temp_bytes(int64_t cnt);
void launch_cm_sort_place(unsigned long long *key, int32_t *ids, int64_t cnt, unsigned long long *key2,
                          int32_t *ids2, unsigned long long *keyv, void *tmp, size_t tmp_bytes,
                          int64_t base, int64_t *pos, int64_t *cm, cudaStream_t st);
void launch_mark_done(const int64_t *cm, int64_t a, int64_t b, int8_t *done, int32_t *level, cudaStream_t st);
void launch_reverse_perm(const int64_t *cm, int64_t n, int64_t *perm, int64_t *inv, cudaStream_t st);
void launch_perm_count(const int64_t *arp, const int64_t *rowmap, int64_t n, int64_t *cnt, cudaStream_t st);
void launch_perm_write(const CsrView &A, const int64_t *rowmap, const int64_t *colmap, int64_t n,
                       const int64_t *rp_out, int32_t *col_out, double *val_out, cudaStream_t st);
size_t seg_sort_temp_bytes(int64_t nnz, int64_t n, const int64_t *rp);
void launch_seg_sort(int32_t **k_cur, int32_t *k_alt, double **v_cur, double *v_alt, int64_t nnz,
                     int64_t n, const int64_t *rp, void *tmp, size_t tmp_bytes, cudaStream_t st);
// flag |= 1 unless A's rows equal (bit for bit) B's rows at offset A.row0 - B.row0
void launch_rows_equal(const CsrView &A, const CsrView &B, int *flag, cudaStream_t st);
// sort every row (<= 1024 entries) of relabelled CSR rows by column: warp-per-row bitonic
constexpr int kSortRowsCap = 1024;
void launch_sort_rows(const int64_t *rp, int64_t n, const int32_t *kin, const double *vin, int32_t *kout,
                      double *vout, cudaStream_t st);
// relabel + sort in one pass: output row r = input row rowmap[r] with keys colmap[k], sorted
// (rows <= kSortRowsCap entries)
void launch_perm_sort_rows(const CsrView &A, const int64_t *rowmap, const int64_t *colmap, int64_t n,
                           const int64_t *rp_out, int32_t *col_out, double *val_out, cudaStream_t st);
// K5s: Taylor product for short rows (thread per row, output span <= 64 columns)
void launch_taylor_dia_short(const NumericArgs &a, const DiaView &D, int32_t *fail_rows, int *fail_count,
                             cudaStream_t st);
void launch_i32_to_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st);
void launch_add_rowlen(const int64_t *rp, const int64_t *alen, const int64_t *b, int64_t n,
                       int64_t *out, cudaStream_t st);
// identity rows for rows [row0, row0+nrows)
void launch_identity(int64_t nrows, int64_t row0, int64_t *rp, int32_t *col, double *val,
                     cudaStream_t st);
// rowptr fix-up: dst[i] = src[i] - src[0] + base for i in [0, cnt]
void launch_rebase_rowptr(const int64_t *src, int64_t cnt, int64_t base, int64_t *dst,
                          cudaStream_t st);

// fp64 peak microbenchmark: which = 0 DFMA chains, 1 DMMA accumulators; out: sms*8*256 doubles
double fp64_peak_flops_per_launch(int which, int sms);
void launch_fp64_peak(int which, int sms, double *out, cudaStream_t st);

}  // namespace sx
