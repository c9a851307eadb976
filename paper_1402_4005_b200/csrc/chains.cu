// chains.cu -- on-device assembly of the lattice benchmark chains (SURVEY.md
// section 8(f), row 1): B = I - A of the tandem queue (chains.py:134-179) and
// of the uniform 2-D random walk (chains.py:95-131) written straight into
// device CSR, with the per-axis geometry columns -- no host scipy matrix, no
// 0.8 GB upload for the 16.8M-state chain.  Canonical form and every value
// bit-identical to paper_1402_4005_b200/chains.py (itself bit-identical to the
// reference): the same stencil slots in ascending column order, the same
// self-loop mass accumulation order, the same 1/deg divisions.
//
// Two passes over the rows: count (entries per row) -> exclusive scan ->
// fill.  Node numbering node = q2 * side + q1 (tandem), iy * side + ix
// (uniform), as the reference.
#include "internal.cuh"

struct TandemRow {
  int64_t col[4];
  double val[4];
  int len;
};

__device__ __forceinline__ TandemRow tandem_row(int64_t i, int side, double lam, double mu1, double mu2) {
  const int64_t q1 = i % side, q2 = i / side;
  // self-loop mass of node i, accumulated in the reference's order
  double stay = 0.0;
  if (q1 + 1 > side - 1) stay = stay + lam;
  if (!((q1 >= 1) && (q2 + 1 <= side - 1))) stay = stay + mu1;
  if (q2 < 1) stay = stay + mu2;
  const double d = stay > 0.0 ? 1.0 - stay : 1.0;
  TandemRow r;
  r.len = 0;
  // sources j -> i: (q1+1, q2-1) via mu1 [i-side+1], (q1-1, q2) via lam [i-1],
  // diagonal [i], (q1, q2+1) via mu2 [i+side]
  if ((q1 + 1 <= side - 1) && (q2 >= 1)) {
    r.col[r.len] = i - side + 1;
    r.val[r.len++] = -mu1;
  }
  if (q1 >= 1) {
    r.col[r.len] = i - 1;
    r.val[r.len++] = -lam;
  }
  if (d != 0.0) {
    r.col[r.len] = i;
    r.val[r.len++] = d;
  }
  if (q2 + 1 <= side - 1) {
    r.col[r.len] = i + side;
    r.val[r.len++] = -mu2;
  }
  return r;
}

struct UniformRow {
  int64_t col[5];
  double val[5];
  int len;
};

__device__ __forceinline__ double uniform_p(int64_t j, int side) {
  const int64_t ix = j % side, iy = j / side;
  const int deg = (ix > 0) + (ix < side - 1) + (iy > 0) + (iy < side - 1);
  return 1.0 / (double)deg;
}

__device__ __forceinline__ UniformRow uniform_row(int64_t i, int side) {
  const int64_t ix = i % side, iy = i / side;
  UniformRow r;
  r.len = 0;
  if (iy > 0) {
    r.col[r.len] = i - side;
    r.val[r.len++] = -uniform_p(i - side, side);
  }
  if (ix > 0) {
    r.col[r.len] = i - 1;
    r.val[r.len++] = -uniform_p(i - 1, side);
  }
  r.col[r.len] = i;
  r.val[r.len++] = 1.0;
  if (ix < side - 1) {
    r.col[r.len] = i + 1;
    r.val[r.len++] = -uniform_p(i + 1, side);
  }
  if (iy < side - 1) {
    r.col[r.len] = i + side;
    r.val[r.len++] = -uniform_p(i + side, side);
  }
  return r;
}

// family 0: tandem, 1: uniform.  PASS 0 writes the row lengths (and the
// geometry), PASS 1 the entries at rowptr.
template <int PASS>
__global__ void lattice_chain_kernel(int family, int side, double lam, double mu1, double mu2, int32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ rowptr, int32_t* __restrict__ col,
                                     double* __restrict__ val, double* __restrict__ geo) {
  BAMG_PDL_PROLOGUE();
  const int64_t n = (int64_t)side * side;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int len;
  int64_t cc[5];
  double vv[5];
  if (family == 0) {
    const TandemRow r = tandem_row(i, side, lam, mu1, mu2);
    len = r.len;
    for (int q = 0; q < 4; ++q) {
      cc[q] = r.col[q];
      vv[q] = r.val[q];
    }
  } else {
    const UniformRow r = uniform_row(i, side);
    len = r.len;
    for (int q = 0; q < 5; ++q) {
      cc[q] = r.col[q];
      vv[q] = r.val[q];
    }
  }
  if (PASS == 0) {
    cnt[i] = len;
    if (geo) {  // per-axis columns: [0, n) first coordinate, [n, 2n) second
      geo[i] = (double)(i % side);
      geo[n + i] = (double)(i / side);
    }
    return;
  }
  const int64_t b = rowptr[i];
  for (int q = 0; q < len; ++q) {
    col[b + q] = (int32_t)cc[q];
    val[b + q] = vv[q];
  }
}

extern "C" int bamg_chain_lattice_count(bamg_ctx* ctx, int family, int side, double lam, double mu1, double mu2,
                                        int32_t* rowptr, double* geometry, int64_t* nnz_host) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, family == 0 || family == 1, "family must be 0 (tandem) or 1 (uniform2d)");
  BAMG_REQUIRE(ctx, side >= 2 && (int64_t)side * side < (int64_t)1 << 31, "side must lie in [2, 46340]");
  const int64_t n = (int64_t)side * side;
  int32_t* cnt;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &cnt));
  BAMG_LAUNCH(ctx, lattice_chain_kernel<0>, grid_for(n, 256), 256, 0, family, side, lam, mu1, mu2, cnt,
              (const int32_t*)nullptr, (int32_t*)nullptr, (double*)nullptr, geometry);
  return scan_i32(ctx, cnt, rowptr, n, nnz_host);
}

extern "C" int bamg_chain_lattice_fill(bamg_ctx* ctx, int family, int side, double lam, double mu1, double mu2,
                                       const int32_t* rowptr, int32_t* col, double* val) {
  BAMG_REQUIRE(ctx, family == 0 || family == 1, "family must be 0 (tandem) or 1 (uniform2d)");
  const int64_t n = (int64_t)side * side;
  BAMG_LAUNCH(ctx, lattice_chain_kernel<1>, grid_for(n, 256), 256, 0, family, side, lam, mu1, mu2, (int32_t*)nullptr,
              rowptr, col, val, (double*)nullptr);
  return 0;
}
