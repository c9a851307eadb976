// internal.cuh -- cross-translation-unit entry points (no arena reset inside;
// the exported extern "C" wrapper owns the reset).
#pragma once
#include "common.cuh"

int spmm_dev(bamg_ctx* ctx, const bamg_csr* A, const double* X, double* Y, int k);
int resid_dev(bamg_ctx* ctx, const bamg_csr* A, const double* b, const double* X, double* R);
int addmv_dev(bamg_ctx* ctx, const bamg_csr* A, const double* Xc, const double* Xold, double* Y, int k);
int jacobi_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip,
               const double* b, const double* b_scale, const double* x, double* x_out, int k,
               double omega, double* peak, const double* rd = nullptr);
int recip_dev(bamg_ctx* ctx, const double* d, int64_t n, double* rd);
int jacobi_mass_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip, const bamg_csr* M,
                    const double* mx, const double* sigma, const double* x, double* x_out, int k, double omega,
                    double* peak, const double* rd);
int rayleigh_fused_dev(bamg_ctx* ctx, const bamg_csr* A, const double* U, const double* V, int k, double* sigma,
                       double* flip, int mode, double* dots, const bamg_csr* M = nullptr,
                       const bamg_csr* N = nullptr);
int diag_dev(bamg_ctx* ctx, const bamg_csr* A, double* d);
int degenerate_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, uint8_t* skip);
int transpose_dev(bamg_ctx* ctx, const bamg_csr* A, int32_t* rowptr_t, int32_t* col_t, double* val_t);

// per-vector helpers on n x k interleaved blocks (reduce.cu)
int rayleigh_dev(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* M, const bamg_csr* N,
                 const double* U, const double* V, int64_t n, int k, double* sigma,
                 double* U_flip_or_null, int mode, double* work3);
int normalize_cols_dev(bamg_ctx* ctx, double* X, int64_t n, int k);
// src non-null: X = src / s (out of place)
int col_scale_div_dev(bamg_ctx* ctx, double* X, int64_t n, int k, const double* s, int fill_c = -1,
                      double fill_v = 0.0, const double* src = nullptr);
int col_fill_dev(bamg_ctx* ctx, double* X, int64_t n, int k, int c, double value);

// C = alpha op(A) op(B) + beta C, column-major fp64 (gemm.cu)
int dgemm_dev(bamg_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
              const double* B, int ldb, double beta, double* C, int ldc);
// strided batch: C_i = alpha op(A_i) op(B_i) + beta C_i, X_i = X + i * sX
int dgemm_batched_dev(bamg_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
                      int64_t sA, const double* B, int ldb, int64_t sB, double beta, double* C, int ldc, int64_t sC,
                      int batch);

// CholQR2 orthonormalisation of an n x p column-major block (dense_large.cu)
int dl_orthonormalize(bamg_ctx* ctx, double* Y, int n, int p, double* G, double* Rinv, double* tmp);
// Y <- Y R^-1 for a caller-computed Gram G = R^T R (dense_large.cu)
int dl_cholqr_apply(bamg_ctx* ctx, const double* G, double* Y, int n, int p, double* Rinv, double* tmp);
// one-sided Jacobi SVD of an nrows x ncols block (dense.cu)
int jacobi_svd_public(bamg_ctx* ctx, double* G, int nrows, int ncols, double* V, double* sig);

// banded coarsest level (band.cu)
struct BandPinv;
int band_coarsest_triplets(bamg_ctx* ctx, const bamg_csr* B, const bamg_csr* Bt, const bamg_csr* M,
                           const bamg_csr* N, int r, const double* Vin, double* U, double* V, double* sigma,
                           BandPinv** keep);
int band_pinv_apply(bamg_ctx* ctx, const BandPinv* h, const double* b, double* x);
void band_pinv_free(bamg_ctx* ctx, BandPinv* h);

struct bamg_coarse_lu;
// x = B^+ b through the kept coarsest LU (dense_large.cu)
int coarse_lu_apply(bamg_ctx* ctx, const bamg_coarse_lu* h, const double* b, double* x);
