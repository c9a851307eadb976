// spgemm.cu -- two-pass sparse matrix product C = A B with scipy csr_matmat
// semantics (the Galerkin products of sparse.py:102-117 and
// bootstrap.py:372-373).
//
// One thread owns one output row.  It walks row i of A in storage order and,
// for each a_ij, row j of B in storage order, accumulating a_ij * b_jk into a
// per-row list kept in FIRST-TOUCH order -- exactly the sequence of
// `sums[k] += v * Bx[kk]` updates scipy performs, so every value is the same
// sequential non-FMA sum.  Pass 1 counts the kept entries (exact zeros
// dropped; canonical mode additionally drops |v| < 1e-300 as make_csr does),
// an exclusive scan gives the row pointer, pass 2 recomputes and writes:
//   order 1 = scipy storage order (reverse first touch), used for the
//             intermediate Q*B that feeds the second product (its storage
//             order fixes the accumulation order of (QB)P);
//   order 0 = canonical (sorted columns), the make_csr'd result.
// The per-row lists live in a global scratch slice sized by the structural
// upper bound sum_j nnz(B_j) (row-chunked so the slice stays bounded).
#include "internal.cuh"

__global__ void spgemm_ub_kernel(int r0, int nr, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                 const int32_t* __restrict__ brp, int32_t* __restrict__ ub) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nr) return;
  int i = r0 + t;
  int s = 0;
  for (int jj = arp[i]; jj < arp[i + 1]; ++jj) {
    int j = acol[jj];
    s += brp[j + 1] - brp[j];
  }
  ub[t] = s;
}

template <int PASS>
__global__ void spgemm_row_kernel(int r0, int nr, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                  const double* __restrict__ aval, const int32_t* __restrict__ brp,
                                  const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                  const int32_t* __restrict__ soff, int32_t* __restrict__ skey,
                                  double* __restrict__ sval, int order, int32_t* __restrict__ cnt,
                                  const int32_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                  double* __restrict__ cval) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nr) return;
  int i = r0 + t;
  int32_t* key = skey + soff[t];
  double* val = sval + soff[t];
  int len = 0;
  for (int jj = arp[i]; jj < arp[i + 1]; ++jj) {
    int j = acol[jj];
    double v = aval[jj];
    for (int kk = brp[j]; kk < brp[j + 1]; ++kk) {
      int c = bcol[kk];
      double p = __dmul_rn(v, bval[kk]);
      int q = 0;
      while (q < len && key[q] != c) ++q;
      if (q == len) {
        key[len] = c;
        val[len] = __dadd_rn(0.0, p);
        ++len;
      } else {
        val[q] = __dadd_rn(val[q], p);
      }
    }
  }
  auto keep = [&](double x) { return order == 0 ? !(fabs(x) < 1e-300) : (x != 0.0); };
  if (PASS == 0) {
    int c = 0;
    for (int q = 0; q < len; ++q) c += keep(val[q]) ? 1 : 0;
    cnt[t] = c;
    return;
  }
  int w = crp[i];
  if (order == 1) {  // reverse first touch
    for (int q = len - 1; q >= 0; --q)
      if (keep(val[q])) {
        ccol[w] = key[q];
        cval[w] = val[q];
        ++w;
      }
  } else {  // sorted by column
    int start = w;
    for (int q = 0; q < len; ++q) {
      if (!keep(val[q])) continue;
      int c = key[q];
      double x = val[q];
      int p = w++;
      while (p > start && ccol[p - 1] > c) {
        ccol[p] = ccol[p - 1];
        cval[p] = cval[p - 1];
        --p;
      }
      ccol[p] = c;
      cval[p] = x;
    }
  }
}

__global__ void copy_counts_kernel(const int32_t* __restrict__ src, int nr, int32_t* __restrict__ dst) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nr) dst[t] = src[t];
}

constexpr int64_t SPGEMM_SCRATCH = int64_t(1) << 28;  // entries per chunk

static int spgemm_pass(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order, int pass,
                       int32_t* counts_all, const int32_t* crp, int32_t* ccol, double* cval) {
  const int n = A->nrows;
  int32_t* ub;
  int32_t* off;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &ub));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &off));
  // chunk rows so the scratch slice stays below SPGEMM_SCRATCH entries;
  // rows per chunk shrink geometrically when a chunk overflows
  int r0 = 0;
  int chunk = n > 0 ? n : 1;
  int32_t* skey = nullptr;
  double* sval = nullptr;
  int64_t scap = 0;
  while (r0 < n) {
    int nr = chunk < n - r0 ? chunk : n - r0;
    BAMG_LAUNCH(ctx, spgemm_ub_kernel, grid_for(nr, 256), 256, 0, r0, nr, A->rowptr, A->col, B->rowptr, ub);
    int64_t total = 0;
    BAMG_TRY(scan_i32(ctx, ub, off, nr, &total));
    if (total > SPGEMM_SCRATCH && nr > 1) {
      chunk = nr / 2;
      continue;
    }
    if (total > scap) {
      int64_t want = total > 1024 ? total : 1024;
      BAMG_TRY(arena_get(ctx, (size_t)want, &skey));
      BAMG_TRY(arena_get(ctx, (size_t)want, &sval));
      scap = want;
    }
    if (pass == 0) {
      BAMG_LAUNCH(ctx, spgemm_row_kernel<0>, grid_for(nr, 128), 128, 0, r0, nr, A->rowptr, A->col, A->val,
                  B->rowptr, B->col, B->val, off, skey, sval, order, counts_all + r0, crp, ccol, cval);
    } else {
      BAMG_LAUNCH(ctx, spgemm_row_kernel<1>, grid_for(nr, 128), 128, 0, r0, nr, A->rowptr, A->col, A->val,
                  B->rowptr, B->col, B->val, off, skey, sval, order, nullptr, crp, ccol, cval);
    }
    r0 += nr;
  }
  return 0;
}

extern "C" int bamg_spgemm_count(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order, int32_t* rowptr_c,
                                 int64_t* nnz_host) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, A && B && A->ncols == B->nrows, "dimension mismatch in sparse product");
  BAMG_REQUIRE(ctx, order == 0 || order == 1, "order must be 0 (canonical) or 1 (scipy storage order)");
  int32_t* counts;
  BAMG_TRY(arena_get(ctx, (size_t)A->nrows + 1, &counts));
  BAMG_TRY(spgemm_pass(ctx, A, B, order, 0, counts, nullptr, nullptr, nullptr));
  return scan_i32(ctx, counts, rowptr_c, A->nrows, nnz_host);
}

extern "C" int bamg_spgemm_fill(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                                const int32_t* rowptr_c, int32_t* col_c, double* val_c) {
  ctx->arena.reset();
  return spgemm_pass(ctx, A, B, order, 1, nullptr, rowptr_c, col_c, val_c);
}
