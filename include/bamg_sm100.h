/*
 * bamg_sm100.h -- C ABI of libbamg_sm100.so, the B200 (sm_100a) engine behind
 * the BAMG setup + AMG-preconditioned GMRES path of arxiv/paper_1402_4005.
 *
 * The reference (`markovmg`, pure Python) has no FFI of its own: its
 * "operator API" is a set of module-level Python functions.  Every entry point
 * below replaces the arithmetic of one of those functions (cited per
 * declaration as reference file:line, relative to
 * /root/reference/pkg/src/markovmg/).  The Python package
 * `paper_1402_4005_b200` binds these through ctypes (INTEGRATION.md shows the
 * stub) and re-exports the reference's names and signatures.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the name ends in `_host`.
 *     Buffers passed in are caller-owned; library workspaces and hierarchy /
 *     basis storage are owned by the handle and released by *_destroy.
 *   - Values are fp64, CSR indices int32 (every nnz in scope is < 2^31),
 *     vector blocks of k test vectors are n x k row-major ("interleaved":
 *     the k values of one state are contiguous).
 *   - Calls are stream-ordered on the stream given to bamg_ctx_create and are
 *     not re-entrant per context.  One context per (device, stream).
 *   - Return codes: 0 ok; < 0 CUDA / argument error (text via
 *     bamg_last_error); > 0 numerical status (1 = not converged,
 *     2 = singular pivot / not positive definite).
 *   - Kernels tagged BIT-EXACT reproduce the reference's scipy arithmetic bit
 *     for bit (sequential ascending-column sums, no FMA contraction).
 */
#ifndef BAMG_SM100_H
#define BAMG_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bamg_ctx bamg_ctx;
typedef struct bamg_hier bamg_hier;

/* A CSR matrix in device memory (canonical form: sorted, no duplicates). */
typedef struct bamg_csr {
  int32_t nrows;
  int32_t ncols;
  int64_t nnz;
  const int32_t* rowptr; /* nrows + 1 */
  const int32_t* col;    /* nnz */
  const double* val;     /* nnz */
  /* optional packed copy made by bamg_csr_pack_plan / _fill (NULL: none): one 32-bit word
   * per entry, (col - row) << 8 | value code, stored slice-major over 32-row slices (word u of
   * row 32 s + l at pslice[s] + 32 u + l; rows shorter than the slice's longest are padded with
   * code 255), the slice offsets pslice[nrows / 32 + 1] (in words), and the 512-double
   * dictionary (values, then their correctly rounded reciprocals).  The k = 1 kernels read it
   * instead of rowptr / col / val; results are bit-identical. */
  const uint32_t* packed; /* pwords */
  const double* dict;     /* 512 */
  const int32_t* pslice;  /* ceil(nrows / 32) + 1 */
  int64_t pwords;
  /* optional stencil (bamg_csr_stencil; ptiles NULL: none): the lattice
   * generators' interior rows all carry the same (col - row, value) list, so a 256-row tile whose
   * rows all equal that list is flagged in ptiles[ceil(nrows / 256)] and swept without reading its
   * packed words at all -- offsets and values come from the kernel's parameter space.  Same
   * products, same order: bit-identical. */
  const uint8_t* ptiles;
  int32_t st_w;        /* entries of the stencil row (1..8) */
  int32_t st_diag;     /* index of its diagonal entry */
  int32_t st_delta[8]; /* col - row, ascending */
  double st_val[8];
  double st_d, st_rd;  /* the diagonal value and RN(1 / d) */
  int64_t st_tiles;    /* flagged tiles (the bytes the sweeps no longer read) */
} bamg_csr;

/* ---------------------------------------------------------------- context */
int bamg_ctx_create(int device, void* cuda_stream, bamg_ctx** out);
int bamg_ctx_destroy(bamg_ctx* ctx);
const char* bamg_last_error(bamg_ctx* ctx);
int bamg_version(void);
/* Number of kernels this context has launched (evidence for bench.py). */
int64_t bamg_launch_count(bamg_ctx* ctx);
/* Number of times the engine made the host wait on its stream. */
int64_t bamg_sync_count(bamg_ctx* ctx);
int bamg_sync(bamg_ctx* ctx);
/* Live per-kernel-family timing with CUDA events on the context's stream.
 * Families: 0 CSR-stream SpMV/SpMM/Jacobi, 1 LS fit, 2 SpGEMM, 3 GMRES
 * orthogonalisation, 4 dense coarsest, 5 other.  enable() resets counters. */
int bamg_prof_enable(bamg_ctx* ctx, unsigned family_mask);
int bamg_prof_read(bamg_ctx* ctx, int family, double* ms_host, int64_t* launches_host,
                   double* bytes_host);
/* Measured fp64 FMA throughput of this device in TFLOP/s (best of `reps`
 * ~1 ms launches).  No reference counterpart: SURVEY.md §8(d) asks for the LS
 * fit to be reported against a measured fp64 CUDA-core peak. */
int bamg_fp64_peak(bamg_ctx* ctx, int reps, double* tflops_host);
/* C = alpha op(A) op(B) + beta C, column-major fp64, BLAS argument order
 * (device pointers, stream-ordered).  The dense kernels behind the coarsest
 * level (gemm.cu: DMMA m8n8k4 tiles, GEMV); replaces the LAPACK/BLAS the
 * reference reaches through numpy (dense.py:53-131). */
int bamg_dgemm(bamg_ctx* ctx, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
               const double* B, int ldb, double beta, double* C, int ldc);
/* Development trace: event pair around every launch, aggregated by kernel
 * name into "name total_ms count" lines. */
int bamg_trace_enable(bamg_ctx* ctx, int on);
int bamg_trace_dump(bamg_ctx* ctx, char* buf, int64_t cap);
/* Same trace as a per-launch timeline: "name start_us end_us" lines. */
int bamg_trace_timeline(bamg_ctx* ctx, char* buf, int64_t cap);
/* Number of trace events recorded so far (timeline phase markers). */
int64_t bamg_trace_position(bamg_ctx* ctx);

/* ------------------------------------------------------- sparse (sparse.py) */
/* y = A x.  BIT-EXACT vs scipy csr_matvec.  Replaces spmv, sparse.py:81-86;
 * with A = explicit transpose it replaces spmv_transpose, sparse.py:89-94. */
int bamg_spmv(bamg_ctx* ctx, const bamg_csr* A, const double* x, double* y);
/* Packed (value-indexed, 32-bit, slice-major) copy of a square operator for the HBM-bound
 * k = 1 kernels (SpMV, V-cycle Jacobi sweeps and residuals).  _plan fills dict[512] and
 * pslice[ceil(nrows / 32) + 1] and sets *ok_host = the number of dictionary entries and
 * *words_host = the packed length when A
 * has at most 254 distinct values and |col - row| < 2^23 (the generators' B = I - A,
 * chains.py:95-302), else *ok_host = 0 and the caller keeps the plain CSR; _fill writes the
 * words (ndict = the plan's *ok_host).  Storage
 * only -- no reference counterpart; replaces nothing in sparse.py:21-46 (the CSR stays). */
int bamg_csr_pack_plan(bamg_ctx* ctx, const bamg_csr* A, int32_t* pslice, double* dict, int* ok_host,
                       int64_t* words_host);
int bamg_csr_pack_fill(bamg_ctx* ctx, const bamg_csr* A, const int32_t* pslice, const double* dict, int ndict,
                       uint32_t* packed);
/* Stencil of a lattice operator: the (col - row, value) list of row nrows / 2 + sqrt(nrows) / 4
 * (an interior point of a square lattice) is the candidate; tiles[ceil(nrows / 256)] gets 1 for every
 * 256-row tile whose rows all carry exactly that list.  *out receives a copy of A with ptiles = tiles
 * and the st_* fields filled when the candidate has 1..8 entries, a diagonal, and at least half of the
 * tiles match (one host read); otherwise *out = *A with ptiles = NULL.  The k = 1 packed kernels and
 * the k-wide sweeps of such an operator take offsets and values of flagged tiles from their
 * parameter space.  Storage only, like bamg_csr_pack_plan. */
int bamg_csr_stencil(bamg_ctx* ctx, const bamg_csr* A, uint8_t* tiles, bamg_csr* out);
/* Y = A X for k interleaved vectors (n x k).  BIT-EXACT per column vs
 * csr_matvecs (interp.py:95, bootstrap.py:384-385). */
int bamg_spmm(bamg_ctx* ctx, const bamg_csr* A, const double* X, double* Y, int k);
/* Explicit transpose with sorted columns: out arrays sized ncols+1 / nnz.
 * Replaces transpose, sparse.py:97-99. */
int bamg_csr_transpose(bamg_ctx* ctx, const bamg_csr* A, int32_t* rowptr_t,
                       int32_t* col_t, double* val_t);
/* Pattern of A + A^T without the diagonal (unit weights implicit).
 * Two calls: rowptr (n+1) first, then columns.  A_t is the explicit
 * transpose of A.  Replaces adjacency_structure, sparse.py:120-128. */
int bamg_sym_pattern_count(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                           int32_t* rowptr_s, int64_t* nnz_host);
int bamg_sym_pattern_fill(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                          const int32_t* rowptr_s, int32_t* col_s);
/* d_i = A_ii (0 when not stored).  B.diagonal(). */
int bamg_diag(bamg_ctx* ctx, const bamg_csr* A, double* d);
/* Count of d_i <= 0 (bootstrap.py:332-334, _operator_degenerate). */
int bamg_count_nonpositive(bamg_ctx* ctx, const double* d, int64_t n, int64_t* count_host);

/* Two-pass SpGEMM C = A B with scipy csr_matmat semantics: sums accumulated in
 * A-row order then B-row order, exact-zero results dropped.  `order`:
 *   0 = canonical (sorted columns, |v| < 1e-300 also dropped: make_csr),
 *   1 = scipy storage order (reverse first touch), exact zeros dropped only.
 * Flags or'ed into `order`: 2 = walk each row of A in reverse storage order,
 * 4 = walk each row of B in reverse.  They give (A I) B and A (I B) with an
 * identity mass I bit-identically without forming the identity product
 * (scipy stores A I / I B with every row reversed: bootstrap.py:372-373 at the
 * finest level, where M = N = I).
 * Count pass fills rowptr_c (nrows+1) and returns nnz; fill pass writes.
 * Replaces triple_product, sparse.py:102-117 and bootstrap.py:372-373. */
int bamg_spgemm_count(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                      int32_t* rowptr_c, int64_t* nnz_host);
int bamg_spgemm_fill(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                     const int32_t* rowptr_c, int32_t* col_c, double* val_c);
/* Independent products counted together: bamg_spgemm_count_slot launches the
 * count into one of 4 slots without any host read; bamg_spgemm_count_wait
 * reads nnz of the listed slots with ONE synchronisation; each product is
 * then finished with bamg_spgemm_fill_slot on its slot.  (The Galerkin
 * products of one level -- QB, Q M, N P -- share one wait.) */
int bamg_spgemm_count_slot(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                           int32_t* rowptr_c, int slot);
int bamg_spgemm_count_wait(bamg_ctx* ctx, int nslots, const int32_t* slots, int64_t* nnz_host);
int bamg_spgemm_fill_slot(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                          const int32_t* rowptr_c, int32_t* col_c, double* val_c, int slot);

/* ------------------------------------------------ chains (chains.py, inputs) */
/* On-device assembly of the lattice chains' B = I - A (SURVEY.md section 8(f)
 * row 1): family 0 = tandem queue (chains.py:134-179, rates lam, mu1, mu2),
 * 1 = uniform 2-D walk (chains.py:95-131).  Count writes rowptr (side^2 + 1),
 * the per-axis geometry (2 x side^2, may be null) and returns nnz; fill writes
 * col/val.  Bit-identical to the host generators (canonical CSR). */
int bamg_chain_lattice_count(bamg_ctx* ctx, int family, int side, double lam, double mu1, double mu2,
                             int32_t* rowptr, double* geometry, int64_t* nnz_host);
int bamg_chain_lattice_fill(bamg_ctx* ctx, int family, int side, double lam, double mu1, double mu2,
                            const int32_t* rowptr, int32_t* col, double* val);
/* B = I - A of the random planar walk (chains.py:270-302) from its Delaunay
 * triangles (ntri x 3 int32 vertex ids; Qhull on the host): count writes
 * rowptr (n + 1) and nnz, fill writes col / val.  Bit-identical to the
 * reference's make_csr(I - A) on the same edge set. */
int bamg_chain_planar_count(bamg_ctx* ctx, const int32_t* tri, int64_t ntri, int n, int32_t* rowptr,
                            int64_t* nnz_host);
int bamg_chain_planar_fill(bamg_ctx* ctx, const int32_t* tri, int64_t ntri, int n, const int32_t* rowptr,
                           int32_t* col, double* val);
/* BASELINE's test vectors without the host: numpy default_rng(seed).random((k, n))
 * twice (right, then left) from the PCG64 state (st, inc) numpy derives from the
 * seed, bit-identical, written n x k interleaved (the layout run_setup takes). */
int bamg_uniform_draws(bamg_ctx* ctx, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int k,
                       int64_t n, double* right, double* left);

/* ------------------------------------------------------ relax (relax.py) */
/* skip_i = d_i <= 0 || (sum_j |A_ij| - |d_i|) > 4 d_i.  Pass the explicit
 * transpose for the column variant.  Replaces degenerate_rows, relax.py:47-63. */
int bamg_degenerate_rows(bamg_ctx* ctx, const bamg_csr* A, const double* d, uint8_t* skip);
/* Self-test of the Jacobi epilogue's division: the engine divides by d through
 * the correctly rounded reciprocal plus one FMA correction (Markstein), which
 * must equal IEEE x / d bit for bit.  Compares both on n reproducible random
 * operand pairs (mode 0: |exponent| <= 40, 1: the fast-path range, 2: all
 * finite doubles incl. subnormals and zeros, 3: near-power-of-two and all-ones
 * mantissas) and returns the number of differing results.  No reference
 * counterpart: it certifies the bit-exactness claim of bamg_jacobi. */
int bamg_selftest_div(bamg_ctx* ctx, int64_t n, uint64_t seed, int mode, int64_t* mismatches_host);
/* One weighted-Jacobi sweep on k interleaved vectors, BIT-EXACT vs
 * _apply_sweep (relax.py:66-83):  x' = x + (omega (b - A x)) / d on unskipped
 * rows.  b may be NULL (homogeneous).  When b_scale is non-NULL the
 * right-hand side is b_scale[c] * b (the sigma * M u of bootstrap.py:296).
 * peak (k doubles, may be NULL) receives max |x'| per vector. */
int bamg_jacobi(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip,
                const double* b, const double* b_scale, const double* x, double* x_out,
                int k, double omega, double* peak);

/* --------------------------------------------------- dense block reductions */
/* out[c] = ||X[:, c]||_2 for n x k interleaved X (deterministic tree). */
int bamg_col_norms(bamg_ctx* ctx, const double* X, int64_t n, int k, double* out);
/* out[c] = sum_i X[i,c] * Y[i,c]. */
int bamg_col_dots(bamg_ctx* ctx, const double* X, const double* Y, int64_t n, int k,
                  double* out);
/* X[:, c] /= s[c] where s[c] != 0 (zero norms left as 1: bootstrap.py:160-163). */
int bamg_col_scale_div(bamg_ctx* ctx, double* X, int64_t n, int k, const double* s);
/* X[i, c] = value for all i (pinning the constant left vector). */
int bamg_col_fill(bamg_ctx* ctx, double* X, int64_t n, int k, int c, double value);
/* Y[i, :] = X[idx[i], :] (triplet injection, bootstrap.py:375-377). */
int bamg_gather_rows(bamg_ctx* ctx, const double* X, const int32_t* idx, int64_t m, int k,
                     double* Y);

/* -------------------------------------------------- bootstrap (bootstrap.py) */
/* One _smooth_block (bootstrap.py:284-314) on device: nsweeps coupled sweeps
 * of the k right vectors V (with A) and the k left vectors U (with A^T),
 * optional inhomogeneous rhs sigma*M u / sigma*N v with per-sweep Rayleigh
 * updates, runaway rescaling, row normalisation, the pinned constant left
 * slot and the sigma refresh (bootstrap.py:166-177).  M / N NULL = identity.
 * U, V are updated in place; sigma (k doubles, device) in place. */
int bamg_smooth_block(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                      const bamg_csr* M, const bamg_csr* N, const double* d,
                      const uint8_t* skip, const uint8_t* skip_t, double* U, double* V,
                      double* sigma, int k, int nsweeps, double omega, int inhomogeneous,
                      int smooth, int refresh);
/* Rayleigh refresh only (bootstrap.py:166-177). */
int bamg_refresh_sigmas(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* M,
                        const bamg_csr* N, const double* U, const double* V, double* U_flip,
                        double* sigma, int k);

/* ------------------------------------------------------ interp (interp.py) */
/* Normalised test vectors and weights 1/||A v||^2 with the caps of
 * singular_test_weights (interp.py:82-102).  Pass A^T for the left side.
 * inf_slot < 0 for none.  Xn (n x k) receives the unit vectors. */
int bamg_test_weights(bamg_ctx* ctx, const bamg_csr* A, const double* X, int64_t n, int k,
                      int inf_slot, double* Xn, double* w);
/* Greedy caliber-bounded weighted ridge LS per fine point (interp.py:129-289).
 * Production path: one thread per point (register Cholesky of the ridge normal
 * equations + two refinement steps on the original rows); points it cannot
 * take are finished by the one-warp-per-point Householder-QR kernel.
 * adj: pattern(A+A^T) without diagonal; coarse_rank[i] >= 0 marks a C point.
 * ridge_override < 0: lambda = 0.1 * level scale (interp.py:266-268), else
 * the given lambda.  Writes, per state i, up to `caliber` (column, value) pairs
 * into out_col/out_val (n x caliber) and out_cnt[i] (C points: identity entry;
 * no-candidate F points: 0).  status_host (2 int64): [0] fits that took the
 * rank-deficient pseudo-inverse branch, [1] points deferred to the warp path. */
/* Multi-GPU setup: restrict every following LS fit of this context to the
 * fine points in rows [row_lo, row_hi) -- the per-point loop of _build_rows
 * (interp.py:258-289) is independent per point, so each rank fits its own row block and
 * the fixed-stride outputs (out_cnt / out_col / out_val) are all-gathered by rows.  Rows
 * outside the range get out_cnt = 0.  row_lo < 0 restores the full range.  (The warp-only
 * fallback path, k > 16 or caliber > 4, ignores the range and fits every row.) */
int bamg_fit_set_row_range(bamg_ctx* ctx, int64_t row_lo, int64_t row_hi);
int bamg_fit_rows(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank,
                  const double* X, const double* w, int64_t n, int k, int caliber,
                  int radius, double improvement_tol, int constrain, int nonnegative,
                  double ridge_override, int32_t* out_cnt, int32_t* out_col, double* out_val,
                  int64_t* status_host);
/* bamg_fit_rows + bamg_rows_count in one call with ONE host read (status as
 * bamg_fit_rows, nnz of the compacted CSR); rowptr (n + 1) is written, the
 * caller allocates nnz entries and finishes with bamg_rows_fill.  Replaces
 * _build_rows, interp.py:252-289. */
int bamg_fit_rows_csr(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank,
                      const double* X, const double* w, int64_t n, int k, int caliber,
                      int radius, double improvement_tol, int constrain, int nonnegative,
                      double ridge_override, int32_t* out_cnt, int32_t* out_col, double* out_val,
                      int32_t* rowptr, int64_t* status_host, int64_t* nnz_host);
/* Asynchronous bamg_fit_rows_csr into one of 4 slots (no host read), and the
 * ONE synchronisation that returns status (2 per slot) and nnz of the listed
 * slots: the P and W fits of a level share it.  Each slot call forks from the
 * context stream at the call (everything enqueued before it, its inputs
 * included, is ordered before the fit) onto the slot's own side stream with
 * its own scratch; bamg_fit_rows_wait joins every pending slot back into the
 * context stream.  Until then the caller must not enqueue work that reads a
 * pending slot's outputs (out_cnt / out_col / out_val / rowptr) nor free
 * them; other work, including other entry points, may run in between. */
int bamg_fit_rows_csr_slot(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank,
                           const double* X, const double* w, int64_t n, int k, int caliber,
                           int radius, double improvement_tol, int constrain, int nonnegative,
                           double ridge_override, int32_t* out_cnt, int32_t* out_col, double* out_val,
                           int32_t* rowptr, int slot);
int bamg_fit_rows_wait(bamg_ctx* ctx, int nslots, const int32_t* slots, int64_t* status_host,
                       int64_t* nnz_host);
/* Compact the fixed-stride rows into canonical CSR (sorted columns, |v| <
 * 1e-300 dropped: csr_from_coo, sparse.py:42-46).  Two calls. */
int bamg_rows_count(bamg_ctx* ctx, const int32_t* cnt, const double* val, int64_t n,
                    int stride, int32_t* rowptr, int64_t* nnz_host);
int bamg_rows_fill(bamg_ctx* ctx, const int32_t* cnt, const int32_t* col, const double* val,
                   int64_t n, int stride, const int32_t* rowptr, int32_t* col_out,
                   double* val_out);

/* ---------------------------------------------------- coarsen (coarsen.py) */
/* Rank of every coordinate among the distinct values of its axis
 * (np.unique(..., return_inverse=True), coarsen.py:84-87). */
int bamg_axis_ranks(bamg_ctx* ctx, const double* coord, int64_t n, int32_t* rank,
                    int64_t* nvalues_host);
/* Ranks on the coarse level from the parent ranks of the kept points. */
int bamg_rerank(bamg_ctx* ctx, const int32_t* parent_rank, const int32_t* coarse_idx,
                int64_t nc, int64_t nvalues_parent, int32_t* rank_out, int64_t* nvalues_host);
/* mask from per-axis ranks: every rank even (geometric_coarsen, coarsen.py:90-109). */
int bamg_even_mask(bamg_ctx* ctx, const int32_t* const* ranks_host, int ndim, int64_t n,
                   uint8_t* mask);
/* coarse list / fine list / coarse_rank from a mask (CfSplitting, coarsen.py:23-52). */
int bamg_split_from_mask(bamg_ctx* ctx, const uint8_t* mask, int64_t n, int32_t* coarse,
                         int32_t* fine, int32_t* coarse_rank, int64_t* nc_host);
/* One compatible-relaxation pass (coarsen.py:129-166): x_F from the host draw,
 * unit-RMS scaling, `sweeps` F-relaxation sweeps, mu, and the greedy MIS in
 * (-mu, index) order computed as a parallel lexicographically-first MIS.
 * `normals` holds the n_fine draws in ascending fine-index order.  Sets new
 * coarse points in cmask; returns the number of candidates in *ncand_host.
 * When there are none and coarse_empty is set, argmax(mu) over the fine
 * points is promoted instead (coarsen.py:148-152). */
int bamg_cr_pass(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* adj, const double* d,
                 uint8_t* cmask, const double* normals, int64_t n_fine, int sweeps,
                 double omega, double threshold, int coarse_empty, int64_t* ncand_host,
                 int64_t* ncoarse_host);
/* Rows without stored entries (cr_coarsen rejects them, coarsen.py:119-121). */
int bamg_count_empty_rows(bamg_ctx* ctx, const bamg_csr* A, int64_t* count_host);
/* Column permutation of an n x k block: Y[:, j] = X[:, perm_host[j]]. */
int bamg_permute_cols(bamg_ctx* ctx, const double* X, int64_t n, int k, const int32_t* perm_host,
                      double* Y);

/* ------------------------------------------------------------ dense (dense.py) */
/* Scatter a CSR into a dense column-major n x n matrix. */
int bamg_csr_to_dense(bamg_ctx* ctx, const bamg_csr* A, double* D, int ld, int transpose);
/* Explicit pseudo-inverse Z = A^+ (column-major n x n) by one-sided Jacobi SVD
 * with rank_tol * sigma_max (PinvOperator, dense.py:118-131). */
int bamg_dense_pinv(bamg_ctx* ctx, const double* A, int n, double rank_tol, double* Z);
/* Coarsest generalized singular triplets (coarsest_triplets, bootstrap.py:205-281):
 * M = L_M L_M^T, N = L_N L_N^T, SVD of L_M^-1 B L_N^-T, r smallest triplets,
 * halves normalised, sign so u^T B v >= 0, null-slot cleanup.  Inputs dense
 * column-major; outputs U, V as n x r interleaved and sigma (r). */
int bamg_coarsest_triplets(bamg_ctx* ctx, const double* Bd, const double* Md,
                           const double* Nd, int n, int r, double* U, double* V,
                           double* sigma);
/* Same, and for the large (blocked) path also the V-cycle's pseudo-inverse of
 * B (row-major n x n into Z, as bamg_dense_pinv) derived from the same
 * factors: B^+ = (I - z z^T) L_N^-T K^+ L_M^-1 (I - y y^T).  *z_valid = 1 when
 * it was computed and certified (else the caller builds it with
 * bamg_dense_pinv).  Replaces the second factorisation behind PinvOperator
 * (dense.py:118-131, built solver.py:93-94) for the coarsest level. */
int bamg_coarsest_triplets_pinv(bamg_ctx* ctx, const double* Bd, const double* Md, const double* Nd, int n, int r,
                                double* U, double* V, double* sigma, double* Z, int* z_valid);
/* As bamg_coarsest_triplets_pinv (Z may be null); when the large coarsest
 * level took the implicit path (the bordered LU of B, no explicit K^+),
 * *lu_out receives that LU for the V-cycle (bamg_hier_set_coarsest_lu) and Z
 * is not formed.  Free with bamg_coarse_lu_destroy. */
typedef struct bamg_coarse_lu bamg_coarse_lu;
int bamg_coarsest_triplets_ex(bamg_ctx* ctx, const double* Bd, const double* Md, const double* Nd, int n, int r,
                              double* U, double* V, double* sigma, double* Z, int* z_valid,
                              bamg_coarse_lu** lu_out);
/* x = B^+ b through the kept LU: (I - z z^T) B^g (I - y y^T) b. */
int bamg_coarse_lu_apply(bamg_ctx* ctx, const bamg_coarse_lu* lu, const double* b, double* x);
int bamg_coarse_lu_destroy(bamg_ctx* ctx, bamg_coarse_lu* lu);
/* Banded coarsest level: the same triplets as bamg_coarsest_triplets
 * (coarsest_triplets, bootstrap.py:205-281) and the V-cycle's B^+
 * (PinvOperator, dense.py:118-131) from block-tridiagonal factorisations of
 * the CSR operators (B, its explicit transpose Bt, M, N; no dense n x n
 * matrix is formed).  Returns 1 -- nothing written -- when the half-bandwidth
 * exceeds 160 or n / 4, or the factorisation is not certified; the caller
 * then takes the dense path.  Vin (n x r interleaved, may be NULL): the
 * level's incoming right test vectors, a warm start for the subspace
 * iteration.  *lu_out: free with bamg_coarse_lu_destroy. */
int bamg_coarsest_band(bamg_ctx* ctx, const bamg_csr* B, const bamg_csr* Bt, const bamg_csr* M, const bamg_csr* N,
                       int r, const double* Vin, double* U, double* V, double* sigma, bamg_coarse_lu** lu_out);

/* ----------------------------------------------------------- solver (solver.py) */
/* Hierarchy for the V-cycle (VCycleOperator, solver.py:79-124).  Level
 * matrices are borrowed (caller keeps them alive); the library owns the
 * per-level work vectors.  The coarsest level is applied as Z b with the
 * explicit pseudo-inverse Z (n_L x n_L, column-major, borrowed). */
int bamg_hier_create(bamg_ctx* ctx, int nlevels, bamg_hier** out);
int bamg_hier_destroy(bamg_hier* h);
int bamg_hier_set_level(bamg_hier* h, int level, const bamg_csr* B, const double* d,
                        const uint8_t* skip, const bamg_csr* P, const bamg_csr* Q);
int bamg_hier_set_coarsest(bamg_hier* h, const double* Z, int n);
/* The coarsest solve through a kept coarse LU instead of an explicit Z. */
int bamg_hier_set_coarsest_lu(bamg_hier* h, const bamg_coarse_lu* lu, int n);
int bamg_hier_set_smoother(bamg_hier* h, double omega, int nu_pre, int nu_post);
/* x = C b, one V-cycle from a zero guess. */
int bamg_vcycle(bamg_ctx* ctx, bamg_hier* h, const double* b, double* x);
/* Left-preconditioned GMRES (solver.py:136-226): Arnoldi with two-pass
 * classical Gram-Schmidt (CGS2) as fused multi-vector reductions, Givens
 * rotations on device, per-iteration true residual ||Bx||/||x||.
 * h may be NULL (unpreconditioned).  restart <= 0 = unrestarted.  stopping:
 * 0 = ||Bx||/||x|| ("scaled_bx"), 1 = ||b-Bx||/||b-Bx0|| ("relative").
 * history_host receives max_iters + 1 doubles; returns 0 converged, 1 not. */
int bamg_gmres(bamg_ctx* ctx, const bamg_csr* B, bamg_hier* h, const double* b,
               const double* x0, double* x, int restart, int max_iters, double rtol,
               int stopping, int* iters_host, double* history_host, int* nhistory_host);
/* y = Z b for a row-major dense n x n Z (the coarsest pseudo-inverse apply,
 * dense.py:130-131). */
int bamg_dense_gemv(bamg_ctx* ctx, const double* Z, int n, const double* b, double* y);
/* Rank-local building blocks of the row-partitioned solve (distributed.py):
 * operators use halo-extended column numbering; mdot / mupdate return local
 * partial sums that the caller all-reduces over NCCL.  Vp is a DEVICE array
 * of m basis-vector pointers. */
int bamg_residual(bamg_ctx* ctx, const bamg_csr* A, const double* b, const double* x, double* r);
int bamg_addmv(bamg_ctx* ctx, const bamg_csr* A, const double* xc, const double* xold, double* y);
int bamg_jacobi_zero(bamg_ctx* ctx, int64_t n, const double* b, const double* d, const uint8_t* skip,
                     double omega, double* x);
int bamg_dense_gemv_rows(bamg_ctx* ctx, const double* Z, int n, const double* b, double* y);
int bamg_mdot(bamg_ctx* ctx, const double* const* Vp, int m, const double* w, int64_t n, double* out);
int bamg_mupdate(bamg_ctx* ctx, const double* const* Vp, int m, const double* c, double* w, int64_t n,
                 double* nrm2);
/* The two fused basis passes of bamg_gmres' Arnoldi step (two-pass CGS2 through the
 * Gram matrix G = V^T V, solver.py:183-196 replaced) on the caller's row block, m <= 64:
 *   bamg_cgs_dots:   out[0..m) = V^T w, out[m] = |w|^2
 *   bamg_cgs_update: ww = w - V c (c = 2 h1 - G h1), vnew = ww * inv_norm unless happy,
 *                    x = x0 + e + V y, out = [V^T ww (m), |ww|^2, |x|^2]
 * The caller all-reduces `out` over its ranks between the passes (one all-reduce each). */
int bamg_cgs_dots(bamg_ctx* ctx, const double* const* Vp, int m, const double* w, int64_t n, double* out);
int bamg_cgs_update(bamg_ctx* ctx, const double* const* Vp, int m, const double* c, const double* y,
                    const double* w, const double* x0, const double* e, double inv_norm, int happy,
                    int64_t n, double* vnew, double* x, double* out);
int bamg_combine(bamg_ctx* ctx, const double* const* Vp, int m, const double* y, const double* base,
                 const double* add, int64_t n, double* out);

/* x0 finalisation (bootstrap.py:420-428 and solver.py:229-235): non-finite or
 * all-zero -> uniform 1/n, sign so the max-|.| entry is positive, l1 = 1. */
int bamg_sign_fix_l1(bamg_ctx* ctx, const double* x, int64_t n, int stride, double* out,
                     int uniform_fallback);

/* ---- field-of-values diagnostics (fov.cu; reference markovmg/fov.py) ----
 * Dense column-major fp64 n x n on device, n <= 1200 in the Python mirror
 * (fov.py:22 DENSE_CAP).
 * bamg_fov_points replaces the angle sweep of fov_boundary (fov.py:85-115):
 *   points[2t], points[2t+1] = re, im of the supporting point v^H A v of angle
 *   theta_t = 2 pi t / n_angles (v the unit top eigenvector of the Hermitian
 *   part of e^{i theta} A).  tol: Lanczos residual bound relative to |A|_F
 *   (0 -> 1e-13).  *iterations: Lanczos steps taken (host, may be NULL).
 * bamg_eigvals replaces eigenvalue_dots' np.linalg.eigvals (fov.py:60-67):
 *   unsorted wr, wi (device, n each); returns 2 if the QR iteration stalls.
 * bamg_range_basis replaces project_range / projected_preconditioned's
 *   SVD range basis (fov.py:194-223): *rank (host) = #{sigma > rank_tol
 *   sigma_max}; basis (n x rank, descending sigma, column-major) and
 *   projected = basis^T A basis (rank x rank); basis == NULL queries the rank
 *   only.  A zero matrix is an argument error (-2), like the reference's
 *   ValueError. */
int bamg_fov_points(bamg_ctx* ctx, const double* A, int n, int n_angles, double tol, double* points,
                    int* iterations);
int bamg_eigvals(bamg_ctx* ctx, const double* A, int n, double* wr, double* wi);
int bamg_range_basis(bamg_ctx* ctx, const double* A, int n, double rank_tol, double* basis,
                     double* projected, int* rank);

#ifdef __cplusplus
}
#endif
#endif /* BAMG_SM100_H */
