// gemm.cu -- fp64 GEMM / GEMV for the large coarsest level (dense_large.cu).
//
// C = alpha op(A) op(B) + beta C, column-major, BLAS argument convention.
// The reference's coarsest work is LAPACK (dense.py:53-131 -> dgesdd, dsyevd,
// dpotrf, dtrtrs); dense_large.cu restates it as blocked algorithms whose
// trailing updates and recursion nodes are GEMMs of three shape classes:
//   * square-ish products (n = 512 ... 24k): DMMA tensor-core tiles,
//     `mma.sync.aligned.m8n8k4 ... f64` (the fp64 MMA of sm_100a), 128 x 128
//     CTA tiles, k-tiles of 16 staged through a 3-deep cp.async ring,
//     8 warps of 32 x 64;
//   * tall-skinny products (one side <= 64: the subspace iteration's n x p
//     blocks) on 64 x 32 tiles; products with both m and n small but a long k
//     (Gram matrices Y^T Y) split k over CTAs with a fixed-order reduction
//     (deterministic run to run);
//   * matrix-vector products (n == 1 or m == 1): HBM-bound GEMV kernels
//     (column-major A: threads over rows with k split in fixed chunks;
//     transposed: one warp per column).
// Shared-memory tiles are k-major ([k][m] / [k][n], row pitch BM+4 / BN+4) so
// the DMMA fragment loads (lane -> (k = lane % 4, row = lane / 4)) hit 16
// distinct 8-byte bank pairs per half-warp.
#include "internal.cuh"

namespace {

constexpr int BK = 16;
constexpr int STAGES = 3;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// op(A)(i, p) and op(B)(p, j) tiles -> shared [p][i] / [p][j]
template <int BM, int BN, int NT, bool TA, bool TB>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* A, int lda, const double* B,
                                           int ldb, int m, int n, int k, int m0, int n0, int k0) {
  constexpr int LA = BM + 4, LB = BN + 4;
#pragma unroll
  for (int r = 0; r < BM * BK / NT; ++r) {
    const int e = threadIdx.x + r * NT;
    int i, p;
    if (!TA) {  // A col-major m x k: i contiguous
      i = e % BM;
      p = e / BM;
    } else {  // A stored k x m: p contiguous
      p = e % BK;
      i = e / BK;
    }
    const int gi = m0 + i, gp = k0 + p;
    const bool ok = gi < m && gp < k;
    const double* src = ok ? (!TA ? A + (int64_t)gp * lda + gi : A + (int64_t)gi * lda + gp) : A;
    cp_async8(sA + p * LA + i, src, ok);
  }
#pragma unroll
  for (int r = 0; r < BN * BK / NT; ++r) {
    const int e = threadIdx.x + r * NT;
    int j, p;
    if (!TB) {  // B col-major k x n: p contiguous
      p = e % BK;
      j = e / BK;
    } else {  // B stored n x k: j contiguous
      j = e % BN;
      p = e / BN;
    }
    const int gj = n0 + j, gp = k0 + p;
    const bool ok = gj < n && gp < k;
    const double* src = ok ? (!TB ? B + (int64_t)gj * ldb + gp : B + (int64_t)gp * ldb + gj) : B;
    cp_async8(sB + p * LB + j, src, ok);
  }
}

// One CTA computes a BM x BN tile of C over the k range of its split
// (blockIdx.z).  split == 1: C = alpha acc + beta C in place; split > 1: the
// raw partial tile goes to part[z][j][i] (m x n column-major slabs) and
// gemm_splitk_reduce finishes in fixed z order.
template <int BM, int BN, int WM, int WN, bool TA, bool TB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    dgemm_tile_kernel(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
                      const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc,
                      int kchunk, double* __restrict__ part, int64_t strA, int64_t strB, int64_t strC, int batched) {
  BAMG_PDL_PROLOGUE();
  if (batched) {  // blockIdx.z selects the problem of a strided batch (split-k off)
    A += strA * blockIdx.z;
    B += strB * blockIdx.z;
    C += strC * blockIdx.z;
  }
  constexpr int NW_M = BM / WM, NW_N = BN / WN, NT = NW_M * NW_N * 32;
  constexpr int MT = WM / 8, NTL = WN / 8;
  constexpr int LA = BM + 4, LB = BN + 4;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;                          // STAGES x BK x LA
  double* sB = smem + STAGES * BK * LA;       // STAGES x BK x LB
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb = batched ? 0 : blockIdx.z * kchunk;
  const int ke = min(k, kb + kchunk);
  const int KT = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % NW_M) * WM, wn0 = (warp / NW_M) * WN;
  const int fr = lane >> 2, fk = lane & 3;

  double acc[MT][NTL][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NTL; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT)
      load_stage<BM, BN, NT, TA, TB>(sA + s * BK * LA, sB + s * BK * LB, A, lda, B, ldb, m, n, ke, m0, n0,
                                     kb + s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      const int st = nk % STAGES;
      load_stage<BM, BN, NT, TA, TB>(sA + st * BK * LA, sB + st * BK * LB, A, lda, B, ldb, m, n, ke, m0, n0,
                                     kb + nk * BK);
    }
    cp_async_commit();
    const double* a_s = sA + (kt % STAGES) * BK * LA;
    const double* b_s = sB + (kt % STAGES) * BK * LB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MT], bf[NTL];
#pragma unroll
      for (int a = 0; a < MT; ++a) af[a] = a_s[(kk + fk) * LA + wm0 + a * 8 + fr];
#pragma unroll
      for (int b = 0; b < NTL; ++b) bf[b] = b_s[(kk + fk) * LB + wn0 + b * 8 + fr];
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NTL; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

  // accumulator (a, b, h): row wm0 + 8a + fr, column wn0 + 8b + 2 fk + h
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    const int i = m0 + wm0 + a * 8 + fr;
    if (i >= m) continue;
#pragma unroll
    for (int b = 0; b < NTL; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = n0 + wn0 + b * 8 + 2 * fk + h;
        if (j >= n) continue;
        if (part) {
          part[((int64_t)blockIdx.z * n + j) * m + i] = acc[a][b][h];
        } else {
          double* c = C + (int64_t)j * ldc + i;
          *c = beta == 0.0 ? alpha * acc[a][b][h] : alpha * acc[a][b][h] + beta * *c;
        }
      }
  }
}

__global__ void gemm_splitk_reduce(int m, int n, int splits, double alpha, const double* __restrict__ part,
                                   double beta, double* __restrict__ C, int ldc) {
  BAMG_PDL_PROLOGUE();
  const int64_t mn = (int64_t)m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * mn + e];
    const int64_t j = e / m, i = e - j * m;
    double* c = C + j * ldc + i;
    *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
  }
}

// y = op(A) x for column-major A (m x k) without transpose: CTA (bx, by)
// sums rows [256 bx, +256) over the k chunk by; partials reduced in order.
constexpr int GEMV_CHUNK = 256;
__global__ void __launch_bounds__(256) gemv_n_partial(int m, int k, const double* __restrict__ A, int lda,
                                                      const double* __restrict__ x, int incx,
                                                      double* __restrict__ part) {
  BAMG_PDL_PROLOGUE();
  const int rblocks = (m + 255) / 256;
  const int rb = blockIdx.x % rblocks, chunk = blockIdx.x / rblocks;
  const int i = rb * 256 + threadIdx.x;
  const int p0 = chunk * GEMV_CHUNK, p1 = min(k, p0 + GEMV_CHUNK);
  __shared__ double xs[GEMV_CHUNK];
  for (int p = p0 + threadIdx.x; p < p1; p += 256) xs[p - p0] = x[(int64_t)p * incx];
  __syncthreads();
  if (i >= m) return;
  const double* a = A + (int64_t)p0 * lda + i;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int p = p0;
  for (; p + 4 <= p1; p += 4, a += 4 * (int64_t)lda) {
    const double a0 = __ldg(a), a1 = __ldg(a + lda), a2 = __ldg(a + 2 * (int64_t)lda), a3 = __ldg(a + 3 * (int64_t)lda);
    s0 = fma(a0, xs[p - p0], s0);
    s1 = fma(a1, xs[p - p0 + 1], s1);
    s2 = fma(a2, xs[p - p0 + 2], s2);
    s3 = fma(a3, xs[p - p0 + 3], s3);
  }
  for (; p < p1; ++p, a += lda) s0 = fma(__ldg(a), xs[p - p0], s0);
  part[(int64_t)chunk * m + i] = (s0 + s1) + (s2 + s3);
}

__global__ void gemv_n_finish(int m, int chunks, double alpha, const double* __restrict__ part, double beta,
                              double* __restrict__ y, int incy) {
  BAMG_PDL_PROLOGUE();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(int64_t)c * m + i];
  double* o = y + (int64_t)i * incy;
  *o = beta == 0.0 ? alpha * s : alpha * s + beta * *o;
}

// y_j = alpha A(:, j) . x + beta y_j (A column j contiguous): warp per column
__global__ void __launch_bounds__(256) gemv_t_kernel(int n, int k, double alpha, const double* __restrict__ A,
                                                     int lda, const double* __restrict__ x, int incx, double beta,
                                                     double* __restrict__ y, int incy) {
  BAMG_PDL_PROLOGUE();
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= n) return;
  const double* a = A + (int64_t)j * lda;
  double s0 = 0.0, s1 = 0.0;
  int p = lane;
  for (; p + 32 < k; p += 64) {
    s0 = fma(__ldg(a + p), __ldg(x + (int64_t)p * incx), s0);
    s1 = fma(__ldg(a + p + 32), __ldg(x + (int64_t)(p + 32) * incx), s1);
  }
  if (p < k) s0 = fma(__ldg(a + p), __ldg(x + (int64_t)p * incx), s0);
  const double s = warp_sum(s0 + s1);
  if (lane == 0) {
    double* o = y + (int64_t)j * incy;
    *o = beta == 0.0 ? alpha * s : alpha * s + beta * *o;
  }
}

__global__ void scale_kernel(int m, int n, double beta, double* __restrict__ C, int ldc) {
  BAMG_PDL_PROLOGUE();
  const int64_t mn = (int64_t)m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    double* c = C + j * ldc + i;
    *c = beta == 0.0 ? 0.0 : beta * *c;
  }
}

template <int BM, int BN>
constexpr size_t tile_smem() {
  return (size_t)STAGES * BK * ((BM + 4) + (BN + 4)) * sizeof(double);
}

template <int BM, int BN, int WM, int WN, bool TA, bool TB>
int launch_tiles(bamg_ctx* ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B,
                 int ldb, double beta, double* C, int ldc, int batch = 1, int64_t sA = 0, int64_t sB = 0,
                 int64_t sC = 0) {
  auto kern = dgemm_tile_kernel<BM, BN, WM, WN, TA, TB>;
  constexpr size_t smem = tile_smem<BM, BN>();
  BAMG_TRY(smem_optin(ctx, (const void*)kern, smem));
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const int gm = (m + BM - 1) / BM, gn = (n + BN - 1) / BN;
  const int64_t tiles = (int64_t)gm * gn;
  // split k when the tile grid cannot fill the GPU and k is long: each split
  // keeps >= 512 of k; the partials are reduced in fixed order
  int splits = 1;
  const int want = 2 * ctx->num_sms;
  if (batch == 1 && tiles < want && k >= 1024) {
    splits = (int)std::min<int64_t>((want + tiles - 1) / tiles, k / 512);
    splits = std::max(1, std::min(splits, 64));
  }
  int kchunk = (k + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = k > 0 ? (k + kchunk - 1) / kchunk : 1;
  if (batch > 1) {
    splits = 1;
    kchunk = k;
  }
  double* part = nullptr;
  if (splits > 1) BAMG_TRY(arena_get(ctx, (size_t)splits * m * n, &part));
  ctx->prof.flops[FAM_DENSE] += 2.0 * m * n * (double)k * batch;
  const int gz = batch > 1 ? batch : splits;
  const int bflag = batch > 1 ? 1 : 0;
  if (bamg_pdl_enabled()) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(gm, gn, gz);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ctx->trace.on) trace_mark(ctx, "dgemm_tile_kernel");
    BAMG_CHECK_CUDA(ctx, cudaLaunchKernelEx(&cfg, kern, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part,
                                            sA, sB, sC, bflag));
  } else {
    if (ctx->trace.on) trace_mark(ctx, "dgemm_tile_kernel");
    kern<<<dim3(gm, gn, gz), NT, smem, ctx->stream>>>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part,
                                                      sA, sB, sC, bflag);
  }
  ctx->launches++;
  BAMG_CHECK_CUDA(ctx, cudaGetLastError());
  if (ctx->trace.on) trace_mark(ctx, nullptr);
  if (splits > 1) {
    const int64_t mn = (int64_t)m * n;
    BAMG_LAUNCH(ctx, gemm_splitk_reduce, (int)std::min<int64_t>(grid_for(mn, 256), 4 * ctx->num_sms), 256, 0, m,
                n, splits, alpha, (const double*)part, beta, C, ldc);
  }
  return 0;
}

template <int BM, int BN, int WM, int WN>
int dispatch_tiles(bamg_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
                   const double* B, int ldb, double beta, double* C, int ldc, int batch = 1, int64_t sA = 0,
                   int64_t sB = 0, int64_t sC = 0) {
  if (!ta && !tb)
    return launch_tiles<BM, BN, WM, WN, false, false>(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, batch, sA, sB,
                                                      sC);
  if (ta && !tb)
    return launch_tiles<BM, BN, WM, WN, true, false>(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, batch, sA, sB,
                                                     sC);
  if (!ta && tb)
    return launch_tiles<BM, BN, WM, WN, false, true>(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, batch, sA, sB,
                                                     sC);
  return launch_tiles<BM, BN, WM, WN, true, true>(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, batch, sA, sB,
                                                  sC);
}

// y (len rows, stride incy) = alpha op(M) x + beta y, op(M) rows x cols
int gemv(bamg_ctx* ctx, bool trans, int rows, int cols, double alpha, const double* M, int ldm, const double* x,
         int incx, double beta, double* y, int incy) {
  if (rows <= 0) return 0;
  ctx->prof.flops[FAM_DENSE] += 2.0 * rows * (double)cols;
  if (cols <= 0) {
    BAMG_LAUNCH(ctx, scale_kernel, grid_for(rows, 256), 256, 0, 1, rows, beta, y, incy);
    return 0;
  }
  if (trans) {  // y_j = M(:, j) . x, M stored cols x rows
    BAMG_LAUNCH(ctx, gemv_t_kernel, grid_for(rows, 8), 256, 0, rows, cols, alpha, M, ldm, x, incx, beta, y, incy);
    return 0;
  }
  const int chunks = (cols + GEMV_CHUNK - 1) / GEMV_CHUNK;
  double* part = nullptr;
  BAMG_TRY(arena_get(ctx, (size_t)chunks * rows, &part));
  BAMG_LAUNCH(ctx, gemv_n_partial, grid_for(rows, 256) * chunks, 256, 0, rows, cols, M, ldm, x, incx, part);
  BAMG_LAUNCH(ctx, gemv_n_finish, grid_for(rows, 256), 256, 0, rows, chunks, alpha, (const double*)part, beta, y,
              incy);
  return 0;
}

}  // namespace

int dgemm_dev(bamg_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
              const double* B, int ldb, double beta, double* C, int ldc) {
  if (m <= 0 || n <= 0) return 0;
  static const bool log = getenv("BAMG_GEMM_LOG") != nullptr;
  if (log) fprintf(stderr, "gemm %d %d %d %d %d\n", (int)ta, (int)tb, m, n, k);
  if (k <= 0 || alpha == 0.0) {
    if (beta == 1.0) return 0;
    BAMG_LAUNCH(ctx, scale_kernel, std::min(grid_for((int64_t)m * n, 256), 4 * ctx->num_sms), 256, 0, m, n, beta,
                C, ldc);
    return 0;
  }
  if (n == 1)  // C(:, 0) = op(A) op(B)(:, 0); op(B)(p, 0) = tb ? B[p ldb] : B[p]
    return gemv(ctx, ta, m, k, alpha, A, lda, B, tb ? ldb : 1, beta, C, 1);
  if (m == 1)  // C(0, j) = sum_p op(A)(0, p) op(B)(p, j): op(B)^T a
    return gemv(ctx, !tb, n, k, alpha, B, ldb, A, ta ? 1 : lda, beta, C, ldc);
  // 128 x 128 tiles only when they fill the GPU; small products on 64 x 32
  // tiles (more CTAs, shorter serial k loops per SM)
  const int64_t big_tiles = (int64_t)((m + 127) / 128) * ((n + 127) / 128);
  if (m <= 64 || n <= 64 || big_tiles < ctx->num_sms)
    return dispatch_tiles<64, 32, 32, 16>(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  return dispatch_tiles<128, 128, 32, 64>(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

// Strided batch of `batch` independent products C_i = alpha op(A_i) op(B_i) +
// beta C_i (X_i = X + i * sX): one launch, blockIdx.z = i.
int dgemm_batched_dev(bamg_ctx* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
                      int64_t sA, const double* B, int ldb, int64_t sB, double beta, double* C, int ldc, int64_t sC,
                      int batch) {
  if (m <= 0 || n <= 0 || batch <= 0) return 0;
  if (batch == 1) return dgemm_dev(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  BAMG_REQUIRE(ctx, k > 0, "batched GEMM needs k > 0");
  return dispatch_tiles<64, 32, 32, 16>(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, batch, sA, sB, sC);
}

// C ABI (tests / tools): device pointers, stream-ordered on the context.
extern "C" int bamg_dgemm(bamg_ctx* ctx, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
                          const double* B, int ldb, double beta, double* C, int ldc) {
  if (!ctx) return -2;
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, m >= 0 && n >= 0 && k >= 0, "negative dimension");
  BAMG_REQUIRE(ctx, lda >= std::max(1, ta ? k : m) && ldb >= std::max(1, tb ? n : k) && ldc >= std::max(1, m),
               "leading dimension too small");
  return dgemm_dev(ctx, ta != 0, tb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}
