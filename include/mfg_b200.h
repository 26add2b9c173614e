/*
 * mfg_b200.h — C ABI of the B200-native Omega-sweep library (libmfg_b200.so).
 *
 * The reference (mfglobal 0.1.0, pure Python) has no FFI of its own: its hot
 * path bottoms out in numpy/scipy C extensions. Each entry point below
 * replaces one of those call sites; the reference interface it stands in for
 * is cited as mfg/<file>:<line> with mfg = /root/reference/pkg/src/mfglobal.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless the name ends in _host.
 *  - Nothing here allocates device memory: callers size workspaces with the
 *    *_workspace() queries and pass them in.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    and returns an mfg_status; mfg_last_error() gives a message.
 *  - dtype selects the storage type of Omega values and dense factors:
 *    MFG_F32 (float) or MFG_F64 (double). Reductions are always fp64.
 *  - Dense matrices are row-major with a leading dimension (elements).
 *  - Omega indices are int32 (|Omega| < 2^31; checked at build time).
 *  - Entry-stream arrays (layout idx / row_of and the value arrays passed to
 *    mfg_sweep) must be readable for 64 entries past nnz (zero padding):
 *    the grouped sweep kernel prefetches without bounds guards.
 */
#ifndef MFG_B200_H
#define MFG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MFG_OK = 0,
  MFG_ERR_ARG = 1,          /* shape / argument error      -> ValueError        */
  MFG_ERR_DATASET = 2,      /* range / duplicate in Omega  -> DatasetError      */
  MFG_ERR_CAPACITY = 3,     /* too large for int32 / ws    -> CapacityError     */
  MFG_ERR_CUDA = 4,         /* CUDA runtime error          -> RuntimeError      */
  MFG_ERR_NUMERICAL = 5     /* non-SPD normal matrix etc.  -> NumericalError    */
} mfg_status;

typedef enum { MFG_F32 = 0, MFG_F64 = 1 } mfg_dtype;

/* One orientation of Omega (CSR over rows, or CSC = CSR of the transpose).
 * Built by mfg_omega_build / mfg_layout_build; the scheduling metadata
 * (batch masks, nonempty-row ranks) drives the load-balanced flat-chunk
 * kernels, so Zipf-skewed rows need no special casing. */
typedef struct {
  int32_t nrows;            /* rows in this orientation                         */
  int32_t ncols;            /* columns in this orientation                      */
  int64_t nnz;
  const int32_t* ptr;       /* [nrows+1]  row pointers                          */
  const int32_t* idx;       /* [nnz]      column index of each entry            */
  const int32_t* row_of;    /* [nnz]      row of each entry (COO)               */
  const uint32_t* bmask;    /* [ceil(nnz/32)] bit l: entry 32b+l starts a row    */
  const int32_t* brank;     /* [ceil(nnz/32)] nonempty-row rank of entry 32b    */
  const int32_t* nzrows;    /* [n_nonempty] rank -> row                          */
  int32_t n_nonempty;
  const int32_t* empty_rows;/* [n_empty]  rows without entries                   */
  int32_t n_empty;
} mfg_layout;

const char* mfg_last_error(void);
int mfg_version(void);
/* number of kernel launches issued by this library since load (diagnostics) */
int64_t mfg_launch_count(void);

/* ---- Omega build ------------------------------------------------------
 * Replaces ObservationSet.from_coo (mfg/data.py:70-102): range checks,
 * (row, col) lexicographic sort, duplicate rejection, CSR row pointers; and
 * the CSC view a_csr_t = a_csr.T.tocsr() (mfg/data.py:113-119, 156-158).
 * Inputs are int64 COO (as the reference stores them) and fp64 values.
 * Outputs (all device): CSR (rows_out/cols_out/vals_out in (row,col) order,
 * ptr), CSC (csc_ptr, csc_rows, csc_perm = CSR position of each CSC entry).
 * On duplicates returns MFG_ERR_DATASET and writes the first duplicate's
 * sorted position to *dup_pos_host (-1 otherwise; host pointer).          */
size_t mfg_omega_build_workspace(int64_t nnz, int32_t m, int32_t n);
int mfg_omega_build(int32_t m, int32_t n, int64_t nnz,
                    const int64_t* rows_in, const int64_t* cols_in,
                    const double* vals_in,
                    int32_t* rows_out, int32_t* cols_out, double* vals_out,
                    int32_t* ptr, int32_t* csc_ptr, int32_t* csc_rows,
                    int32_t* csc_cols, int32_t* csc_perm,
                    int64_t* dup_pos_host, int32_t* range_err_host,
                    void* workspace, size_t ws_bytes, void* stream);

/* Scheduling metadata for one orientation, from its ptr/row_of arrays.
 * bmask/brank sized ceil(nnz/32); nzrows sized nrows; empty_rows sized nrows.
 * Writes counts to the host ints.                                          */
size_t mfg_layout_workspace(int64_t nnz, int32_t nrows);
int mfg_layout_build(int32_t nrows, int64_t nnz, const int32_t* ptr,
                     const int32_t* row_of, uint32_t* bmask, int32_t* brank,
                     int32_t* nzrows, int32_t* empty_rows,
                     int32_t* n_nonempty_host, int32_t* n_empty_host,
                     void* workspace, size_t ws_bytes, void* stream);

/* Gather: out[e] = src[perm[e]] (values into the CSC order).               */
int mfg_gather(int dtype, int64_t nnz, const int32_t* perm, const void* src,
               void* out, void* stream);
/* dtype conversion of a flat array (f64 <-> f32)                           */
int mfg_convert(int dtype_out, int dtype_in, int64_t count, const void* src,
                void* out, void* stream);

/* ---- The Omega sweep (the metric's unit of work) ----------------------
 * One launch pair computing, for fixed W (m x k) and H (n x k):
 *   R = P_Omega(W H^T) - A            (SDDMM; pair_values/residual_on_omega,
 *                                      mfg/data.py:253-280)
 *   RH  = R . H     (m x k)           (CSR SpMM, mfg/operators.py:108 /
 *                                      mfg/mfsolver.py:74)
 *   RtW = R^T . W   (n x k)           (CSC SpMM, mfg/operators.py:117)
 *   sums[0] = sum r^2 (loss_quad, mfg/data.py:291-293),
 *   sums[1] = ||W||_F^2, sums[2] = ||H||_F^2 (FactorPair.frob_sq,
 *                                      mfg/operators.py:53-55).
 * Both orientations are processed in the same launch (the CSC pass
 * recomputes r from its own value copy instead of gathering R).
 * Any of R/RH/RtW may be NULL to skip that output. out_scale multiplies
 * RH and RtW (e.g. 2 for gradients). vals_csc is A in CSC order.
 * compute_f64 != 0 forces fp64 arithmetic on f32 storage.
 * ldw/ldh >= k; padding columns must be zero. The single-launch grouped
 * kernel (row pieces finished in-kernel, last-block fp64 reductions) runs
 * when RH and RtW are both wanted and ldw == ldh == mfg_sweep_ld(dtype,
 * compute_f64, k): k itself when k*sizeof(elem) is a multiple of 16
 * (unpadded), else the grouped width kp (32/64 for f32, 16/32 for f64).
 * Other ld take the warp-per-chunk kernel plus a deterministic epilogue.
 * The workspace must be zero-filled before its first use and not shared
 * with concurrent calls; the sweep leaves its counters zeroed.           */
size_t mfg_sweep_workspace(const mfg_layout* csr, const mfg_layout* csc, int k);
/* Factor row stride (elements) the single-launch sweep kernels take for
 * width k (>= k; the columns beyond k must be zero).                     */
int mfg_sweep_ld(int dtype, int compute_f64, int k);

/* The sweep of one rank's shards: rows_csr is the CSR of
 * the rank's row block R_p (local row ids, global column ids), cols_csc the
 * CSC of its column block C_p (local column ids, global row ids). W_rows /
 * H_cols point at the rows R_p of W / C_p of H (the self rows), W_full /
 * H_full at the replicas the passes gather from. Outputs: R over the row
 * shard, the rows R_p of R.H and C_p of R^T.W -- final, with no exchange --
 * and sums = [sum r^2 over the row shard, ||W_rows||^2, ||H_cols||^2], whose
 * rank-ordered sums are the full sweep's. Same kernels and preconditions as
 * mfg_sweep; mfg_sweep_workspace(rows_csr, cols_csc, k) sizes the workspace. */
int mfg_sweep_sharded(int dtype, int compute_f64, const mfg_layout* rows_csr,
                      const mfg_layout* cols_csc, int k, const void* vals_rows,
                      const void* vals_cols, const void* W_rows, const void* W_full,
                      int ldw, const void* H_cols, const void* H_full, int ldh,
                      void* R, void* RH, void* RtW, double out_scale, double* sums,
                      void* workspace, size_t ws_bytes, void* stream);

/* mfg_sweep from HOST factors, as a host caller of the reference's sweep
 * (residual_on_omega + loss_quad + res.csr @ H + res.csr_t @ W,
 * mfg/data.py:272-293, mfg/operators.py:108,117) holds them: enqueues on
 * `stream` the H2D of W_host (m x k, row-major) and H_host (n x k) into the
 * device factors W (ld ldw) and H (ld ldh) -- one copy each, strided when
 * ld > k -- then the sweep, then one D2H of the packed results
 *   out = [sums (3 doubles, padded to 32 B) | RH (m x k) | RtW (n x k)]
 * into out_host (skipped when NULL). Host buffers should be pinned for the
 * copies to be asynchronous. Same preconditions as mfg_sweep.            */
int mfg_sweep_host(int dtype, int compute_f64, const mfg_layout* csr,
                   const mfg_layout* csc, int k, const void* vals_csr,
                   const void* vals_csc, const void* W_host, const void* H_host,
                   void* W, int ldw, void* H, int ldh, void* R, void* out,
                   void* out_host, double out_scale, void* workspace,
                   size_t ws_bytes, void* stream);
int mfg_sweep(int dtype, int compute_f64, const mfg_layout* csr,
              const mfg_layout* csc, int k, const void* vals_csr,
              const void* vals_csc, const void* W, int ldw, const void* H,
              int ldh, void* R, void* RH, void* RtW, double out_scale,
              double* sums, void* workspace, size_t ws_bytes, void* stream);

/* ---- panel passes: the hot part of the sweep from shared memory --------
 * The same arithmetic as mfg_sweep (mfg/data.py:253-263 pair_values,
 * mfg/operators.py:108,117 the two SpMMs), for the entries whose gathered
 * factor row is among the most frequently gathered ones: those rows are
 * staged in shared memory in panels of mfg_panel_rows(ld) rows, and every
 * run of a self row's entries inside one panel (a piece) is walked by an
 * 8-lane group. The remaining (cold) entries go through mfg_sweep_sharded
 * on their own layouts; mfg_panel_fold then adds each self row's piece
 * outputs to the cold part in a fixed order (bitwise reproducible).
 * fp32 storage and arithmetic; ld (= ldw = ldh) must be 32, 40 or 64.
 * The panel layout is built by paper_2204_14067_b200/panel.py (device-side
 * sort/scan); its arrays are documented in csrc/panel.cu.                  */
typedef struct {
  int32_t n_pieces;          /* pieces = output slots                        */
  int32_t n_frows;           /* self rows that own pieces                    */
  int32_t n_light;           /* the first n_light of them have few slots (folded
                                by one thread per 16-byte chunk); the rest get a
                                block each                                    */
  const int32_t* panel_ids;  /* [n_panels * mfg_panel_rows(ld)] gathered-row id, -1 = none */
  const int32_t* pieces;     /* [n_pieces][4] {self row, first record block, length, slot},
                                per panel by decreasing length               */
  const int32_t* recs;       /* record blocks of 16 entries, 96 B each: 16 x u16
                                panel-local rows, 16 x f32 A; a piece owns whole
                                blocks; 2 blocks of padding at the end        */
  const int32_t* frows;      /* [n_frows] self row                           */
  const int32_t* fbeg;       /* [n_frows] first slot of the row              */
  const int32_t* fcnt;       /* [n_frows] number of slots of the row         */
  void* r_hot;               /* out: residuals in record order, 16 per block (NULL: not wanted) */
  void* piece_out;           /* scratch [n_pieces][ld] fp32                  */
  void* piece_sq;            /* scratch [n_pieces] fp64 (NULL: no sum r^2)   */
} mfg_panel_pass;

/* rows of one panel for factor rows of ld floats (0: width not supported)   */
int mfg_panel_rows(int ld);
/* CTAs of the panel kernel (the length of cta_start)                        */
int mfg_panel_ctas(void);
/* Both passes' hot entries in one launch. plist: [n_list][4] {pass (0 CSR,
 * 1 CSC), panel, first piece, end piece}, one element per panel; cta_start:
 * [mfg_panel_ctas()] the list element each CTA starts its cyclic walk at;
 * counters: n_list + 1 zeroed int32 (left zeroed). W, H: the factors (row
 * stride ld).                                                              */
int mfg_panel_sweep(int ld, int n_list, const int32_t* plist, const int32_t* cta_start,
                    const mfg_panel_pass* csr, const mfg_panel_pass* csc, const void* W,
                    const void* H, int32_t* counters, void* stream);
/* out[row] += out_scale * (sum of the row's piece outputs, slot order), for
 * the rows that own slots; assign != 0: out[row] = ... instead (every entry of
 * those rows is in a piece: the cold pieces of mfg_cold_sweep share the slots).
 * sums[0] += sum of piece_sq (when both are non-NULL; sq_ws: 1 KB of zeroed
 * device scratch, left zeroed).                                            */
int mfg_panel_fold(int ld, int k, const mfg_panel_pass* pass, void* out, int ldout,
                   double out_scale, int assign, double* sums, void* sq_ws, void* stream);

/* The cold entries of both passes walked like panel pieces, their rows read
 * with global loads (ld = 32 or 40). The structs' pieces / recs / r_hot
 * describe the cold pieces (record blocks: 16 x u32 gathered-row ids, then
 * 16 x f32 A, 128 B; 2 blocks of padding); piece_out / piece_sq are the
 * arrays of the panel passes (slots are shared); panel_ids, frows, fbeg and
 * fcnt are not read. A piece whose length field has bit 30 set is its self
 * row's only slot: out_scale times its vector goes straight to that row of
 * RH / RtW (row stride ld; only used when k == ld) and the row is not in the
 * fold lists. counters: 3 zeroed int32 (left zeroed).                      */
int mfg_cold_sweep(int ld, const mfg_panel_pass* csr, const mfg_panel_pass* csc,
                   const void* W, const void* H, void* RH, void* RtW, double out_scale,
                   int32_t* counters, void* stream);

/* ---- SDDMM with fused reductions --------------------------------------
 * p_e = sum_d L[row_e, d] * (scale ? scale[d] : 1) * Rt[col_e, d]
 * r_e = p_e - A_e (A may be NULL -> 0)
 * out_e = out_mult * r_e (out may be NULL)
 * sums[0] += sum r_e^2;   if G: sums[1] += sum G_e (r_e - G_e/2);
 * sums[2] += sum G_e p_e   (all fp64; sums must hold 3 doubles)
 * Covers residual_on_omega(_svd) (mfg/data.py:272-288), triplet_values
 * (266-269), the Eq.5 terms f_next / g_inner (mfg/proxlift.py:374-377) and
 * ShiftedOperator.frob_sq's x_Omega.g (mfg/operators.py:142-152).         */
size_t mfg_sddmm_workspace(const mfg_layout* lay, int k);
int mfg_sddmm(int dtype, int compute_f64, const mfg_layout* lay, int k,
              const void* L, int ldl, const double* scale, const void* Rt,
              int ldr, const void* A, const void* G, double out_mult,
              void* out, double* sums, void* workspace, size_t ws_bytes,
              void* stream);

/* ---- SpMM over Omega --------------------------------------------------
 * Y = alpha * S X + beta * Y, S the sparse matrix with values `vals` in the
 * layout's order (CSR: grad.csr @ block, mfg/operators.py:108; pass the CSC
 * layout and CSC-ordered values for grad.csr_t @ block, 117/135).
 * X is (ncols x p), Y is (nrows x p).                                     */
size_t mfg_spmm_workspace(const mfg_layout* lay, int p);
int mfg_spmm(int dtype, const mfg_layout* lay, int p, const void* vals,
             const void* X, int ldx, double alpha, double beta, void* Y,
             int ldy, void* workspace, size_t ws_bytes, void* stream);

/* ---- BCD half-sweep ---------------------------------------------------
 * Exact row minimisers (mfg/mfsolver.py:53-75):
 *   (lam I + 2 sum_{j in Omega_i} o_j o_j^T) w_i = 2 sum_j A_ij o_j
 * Gram assembly and a per-row Cholesky solve, fp64 arithmetic for either
 * storage type. OUT is (nrows x k).                                       */
size_t mfg_bcd_workspace(const mfg_layout* lay, int k);
int mfg_bcd_half_sweep(int dtype, const mfg_layout* lay, int k,
                       const void* vals, const void* other, int ldo,
                       double lam, void* out, int ldout, void* workspace,
                       size_t ws_bytes, void* stream);
/* Enqueue (on `stream`) a copy of the last half-sweep's status word from its
 * workspace into *flag_host (pinned host memory for an asynchronous copy):
 * nonzero when a Cholesky pivot was <= 0 or NaN (a non-SPD normal matrix,
 * i.e. non-finite factors or values), which the reference's batched
 * np.linalg.solve (mfg/mfsolver.py:75) would turn into NaN rows. The Python
 * layer raises NumericalError (mfg/driver.py:52) for it.                   */
int mfg_bcd_status(const void* workspace, int* flag_host, void* stream);

/* ---- dense fp64 contractions of the lifting step (fp64 tensor cores) ---
 * Row-major operands. mfg_gemm_tn: C (p x q) = alpha A^T B for tall A
 * (m x p) and B (m x q) -- the k x k Grams of inner_product / frob_dist_sq
 * (mfg/operators.py:67-81), H^T V and W^T U of ShiftedOperator.apply /
 * apply_t (mfg/operators.py:102-118), the CholeskyQR Gram B^T B
 * (orthonormalize, mfg/kernels.py:76-105), q^T S q of _ritz
 * (mfg/eigensolver.py:81-92) and M M^T of exact_svd_short_fat
 * (mfg/kernels.py:108-135). The contraction is split over row slices whose
 * partials are added in slice order (bitwise reproducible); workspace from
 * mfg_gemm_tn_workspace (0 bytes: none needed).
 * mfg_gemm_nn: C (m x q) = alpha A (m x p) B (p x q) + beta C -- W (H^T V),
 * the Ritz rotations q P and S q P, and V = M^T U / sigma.               */
size_t mfg_gemm_tn_workspace(int m, int p, int q);
int mfg_gemm_tn(int m, int p, int q, const double* A, int lda, const double* B,
                int ldb, double alpha, double* C, int ldc, void* workspace,
                size_t ws_bytes, void* stream);
int mfg_gemm_nn(int m, int p, int q, const double* A, int lda, const double* B,
                int ldb, double alpha, double beta, double* C, int ldc,
                void* stream);

/* ---- tall-skinny QR of the lifting step --------------------------------
 * Q (m x p, orthonormal columns) and diag[j] = |R_jj| of B = Q R for a
 * row-major B (m x p, m >= p >= 1): the Householder QR of orthonormalize
 * (mfg/kernels.py:76-105, np.linalg.qr + the |R_jj| <= tol ||B||_F column
 * screening, which the caller applies to diag on the host) and of
 * svd_from_factors (mfg/mfsolver.py:35-45). 32-column panels: block
 * Gram-Schmidt with re-orthogonalisation against the finished columns (on
 * the DMMA products above) around a Householder TSQR of the panel in shared
 * memory. Q equals LAPACK's up to column signs. The workspace's first bytes
 * are a mfg_gemm_tn workspace (zero before the first use, left zero).     */
size_t mfg_qr_workspace(int m, int p);
int mfg_qr(int m, int p, const double* B, int ldb, double* Q, int ldq,
           double* diag, void* workspace, size_t ws_bytes, void* stream);

/* ---- dense reductions ---------------------------------------------------
 * sums_host-free fp64 dot: out[0] = sum_i x_i y_i over `count` entries.    */
int mfg_dot(int dtype, int64_t count, const void* x, const void* y,
            double* out, void* workspace, size_t ws_bytes, void* stream);

/* ---- diagnostics ------------------------------------------------------
 * CUDA-event timing of the main sweep kernel on its launching stream, for
 * the roofline figure of bench.py: enable with room for max_records
 * launches (0 disables), then collect the summed milliseconds.            */
int mfg_profile_enable(int max_records);
int mfg_profile_collect(double* total_ms, int* count);
/* ---- text ingest (host) -------------------------------------------------
 * Multi-threaded parser of the whitespace "user item rating [timestamp]"
 * format (replaces mfg/data.py:164-200 _parse_stream on files/bytes).
 * mfg_count_lines gives an upper bound on the records. mfg_parse_ratings
 * fills users/items/ratings (cap entries) in file order and sets *count;
 * it returns MFG_ERR_ARG with *first_odd_line (1-based) at the first line
 * whose parse is not a plain ASCII "id id decimal [field]" with positive
 * ids -- the caller then re-parses with the reference's rules, which accept
 * the line or raise the reference's exact ParseError. nthreads <= 0 uses
 * all hardware threads.                                                     */
int64_t mfg_count_lines(const char* buf, size_t len);
int mfg_parse_ratings(const char* buf, size_t len, int nthreads, int64_t* users,
                      int64_t* items, double* ratings, size_t cap, size_t* count,
                      int64_t* first_odd_line);

/* per-worker clock64 stamps of the grouped sweep (start, init, loop, end),
 * [workers][4] int64 on the device; NULL disables.                        */
int mfg_set_probe(void* dev_buffer);

#ifdef __cplusplus
}
#endif
#endif /* MFG_B200_H */
