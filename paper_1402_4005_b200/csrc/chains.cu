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
#include <algorithm>

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

// ------------------------------------------------------------ planar chain
// B = I - A of the random planar walk (chains.py:270-302) from the Delaunay
// triangles (the triangulation itself is Qhull on the host; the reference's
// Bowyer-Watson is O(n^2)): every triangle lists its two other corners at
// each corner, each row's list is sorted and de-duplicated (an interior edge
// comes from two triangles), deg = unique neighbour count, and row i of B
// holds 1.0 on the diagonal and -(1.0 / deg[j]) at every neighbour j -- the
// reference's A has 1/deg[j] in column j (chains.py:296-299), so the values
// and the canonical column order are bit-identical to make_csr(I - A).
__global__ void planar_tri_count_kernel(const int32_t* __restrict__ tri, int64_t ntri, int32_t* __restrict__ cnt) {
  BAMG_PDL_PROLOGUE();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntri; t += (int64_t)gridDim.x * blockDim.x)
    for (int q = 0; q < 3; ++q) atomicAdd(&cnt[tri[3 * t + q]], 2);
}

__global__ void planar_tri_fill_kernel(const int32_t* __restrict__ tri, int64_t ntri, int32_t* __restrict__ cur,
                                       int32_t* __restrict__ nbr) {
  BAMG_PDL_PROLOGUE();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntri; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v[3] = {tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
    for (int q = 0; q < 3; ++q) {
      const int32_t p = atomicAdd(&cur[v[q]], 2);
      nbr[p] = v[(q + 1) % 3];
      nbr[p + 1] = v[(q + 2) % 3];
    }
  }
}

// sort + de-duplicate each row's list in place; deg[i] = unique count,
// cnt1[i] = deg[i] + 1 (row length of B: neighbours and the diagonal)
__global__ void planar_row_unique_kernel(const int32_t* __restrict__ off, int32_t* __restrict__ nbr, int n,
                                         int32_t* __restrict__ deg, int32_t* __restrict__ cnt1,
                                         int* __restrict__ isolated) {
  BAMG_PDL_PROLOGUE();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t* a = nbr + off[i];
  const int len = off[i + 1] - off[i];
  for (int x = 1; x < len; ++x) {  // insertion sort (mean degree ~6)
    const int32_t v = a[x];
    int y = x - 1;
    while (y >= 0 && a[y] > v) {
      a[y + 1] = a[y];
      --y;
    }
    a[y + 1] = v;
  }
  int u = 0;
  for (int x = 0; x < len; ++x)
    if (u == 0 || a[x] != a[u - 1]) a[u++] = a[x];
  deg[i] = u;
  cnt1[i] = u + 1;
  if (u == 0) atomicExch(isolated, 1);
}

__global__ void planar_fill_b_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                     const int32_t* __restrict__ deg, int n, const int32_t* __restrict__ rowptr,
                                     int32_t* __restrict__ col, double* __restrict__ val) {
  BAMG_PDL_PROLOGUE();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t* a = nbr + off[i];
  const int u = deg[i];
  int w = rowptr[i];
  bool diag = false;
  for (int x = 0; x < u; ++x) {
    const int32_t j = a[x];
    if (!diag && j > i) {
      col[w] = i;
      val[w++] = 1.0;
      diag = true;
    }
    col[w] = j;
    val[w++] = -(1.0 / (double)deg[j]);
  }
  if (!diag) {
    col[w] = i;
    val[w] = 1.0;
  }
}

// both calls rebuild the (cheap) sorted neighbour lists in the arena
static int planar_lists(bamg_ctx* ctx, const int32_t* tri, int64_t ntri, int n, int32_t** off, int32_t** nbr,
                        int32_t** deg, int32_t** cnt1, int* isolated_host) {
  int32_t *cnt, *cur;
  int* iso;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &cnt));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, off));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &cur));
  BAMG_TRY(arena_get(ctx, (size_t)6 * ntri + 1, nbr));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, deg));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, cnt1));
  BAMG_TRY(arena_get(ctx, 1, &iso));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n, ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(iso, 0, sizeof(int), ctx->stream));
  const int g = std::min(grid_for(ntri, 256), 8 * ctx->num_sms);
  BAMG_LAUNCH(ctx, planar_tri_count_kernel, g, 256, 0, tri, ntri, cnt);
  int64_t total = 0;
  BAMG_TRY(scan_i32(ctx, cnt, *off, n, &total));
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(cur, *off, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  BAMG_LAUNCH(ctx, planar_tri_fill_kernel, g, 256, 0, tri, ntri, cur, *nbr);
  BAMG_LAUNCH(ctx, planar_row_unique_kernel, grid_for(n, 256), 256, 0, (const int32_t*)*off, *nbr, n, *deg, *cnt1,
              iso);
  BAMG_TRY(ctx_read_i32(ctx, iso, 1, isolated_host));
  return 0;
}

extern "C" int bamg_chain_planar_count(bamg_ctx* ctx, const int32_t* tri, int64_t ntri, int n, int32_t* rowptr,
                                       int64_t* nnz_host) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, n >= 4 && ntri >= 1 && 6 * ntri < ((int64_t)1 << 31), "planar chain: bad sizes");
  int32_t *off, *nbr, *deg, *cnt1;
  int iso = 0;
  BAMG_TRY(planar_lists(ctx, tri, ntri, n, &off, &nbr, &deg, &cnt1, &iso));
  BAMG_REQUIRE(ctx, iso == 0, "triangulation left an isolated point");
  return scan_i32(ctx, cnt1, rowptr, n, nnz_host);
}

extern "C" int bamg_chain_planar_fill(bamg_ctx* ctx, const int32_t* tri, int64_t ntri, int n, const int32_t* rowptr,
                                      int32_t* col, double* val) {
  ctx->arena.reset();
  int32_t *off, *nbr, *deg, *cnt1;
  int iso = 0;
  BAMG_TRY(planar_lists(ctx, tri, ntri, n, &off, &nbr, &deg, &cnt1, &iso));
  BAMG_LAUNCH(ctx, planar_fill_b_kernel, grid_for(n, 256), 256, 0, (const int32_t*)off, (const int32_t*)nbr,
              (const int32_t*)deg, n, rowptr, col, val);
  return 0;
}

// ------------------------------------------- seeded test vectors on device
// BASELINE.json's test vectors are numpy's default_rng(seed).random((k, n))
// twice (right, then left).  numpy's PCG64 is a 128-bit LCG (multiplier
// 0x2360ed051fc65da44385df649fccf645) with the XSL-RR 128/64 output, and
// random() maps a draw u to (u >> 11) * 2^-53.  Each thread jumps its LCG
// ahead to the start of its chunk (binary powers of the affine step) and
// produces the chunk: the same doubles as numpy, bit for bit, written in the
// engine's n x k interleaved layout -- no 2 k n x 8-byte host upload.
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;
}

__device__ __forceinline__ uint64_t pcg_xsl_rr(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__global__ void pcg64_uniform_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                     int64_t total, int64_t chunk, int k, int64_t n, double* __restrict__ right,
                                     double* __restrict__ left) {
  BAMG_PDL_PROLOGUE();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = t * chunk;
  if (i0 >= total) return;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  u128 s = ((u128)st_hi << 64) | st_lo;
  // s <- state after i0 steps: (A, C) = step^i0 by binary powers
  u128 A = 1, C = 0, a = pcg_mult(), c = inc;
  for (int64_t e = i0; e; e >>= 1) {
    if (e & 1) {
      A = a * A;
      C = a * C + c;
    }
    c = a * c + c;
    a = a * a;
  }
  s = A * s + C;
  const int64_t kn = (int64_t)k * n;
  const int64_t i1 = min(total, i0 + chunk);
  const u128 m = pcg_mult();
  for (int64_t i = i0; i < i1; ++i) {
    s = s * m + inc;
    const double v = (double)(pcg_xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
    const int64_t j = i < kn ? i : i - kn;  // position in the (k, n) C-order draw
    const int64_t c = j / n, row = j - c * n;
    (i < kn ? right : left)[row * k + c] = v;
  }
}

extern "C" int bamg_uniform_draws(bamg_ctx* ctx, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                                  int k, int64_t n, double* right, double* left) {
  BAMG_REQUIRE(ctx, k >= 1 && n >= 1 && right && left, "bad draw shape");
  const int64_t total = 2 * (int64_t)k * n;
  const int64_t chunk = 256;
  const int64_t threads = (total + chunk - 1) / chunk;
  BAMG_LAUNCH(ctx, pcg64_uniform_kernel, grid_for(threads, 128), 128, 0, st_hi, st_lo, inc_hi, inc_lo, total, chunk, k,
              n, right, left);
  return 0;
}
