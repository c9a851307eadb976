// setup.cu -- bootstrap relaxation of the k left / k right test vectors and
// the singular-test weights, all on device.
//
// _smooth_block (bootstrap.py:284-314): per sweep one fused k-wide Jacobi
// launch per side (right vectors with B, left vectors with the explicit B^T,
// both through the bit-exact CSR-stream kernel of sparse.cu), the optional
// inhomogeneous right-hand sides sigma*M u / sigma*N v folded into the
// Jacobi epilogue, runaway rescaling driven by the per-vector peak the
// Jacobi epilogue already reduces, and the per-sweep Rayleigh quotient
// (bootstrap.py:144-153) from three k-wide SpMMs and one fused column-dot
// pass.  Row normalisation, the pinned constant left slot and the sigma
// refresh (bootstrap.py:160-177) close the block.  No host synchronisation.
//
// singular_test_weights (interp.py:82-102): unit-normalise, ||A v||, then the
// caps 1e16 / 1e4 x median and the infinite constraint slot, in one tiny
// single-CTA kernel over the k residual norms.
#include <cmath>

#include "internal.cuh"

// X[:, c] /= peak[c] when peak[c] > 1e100 (bootstrap.py:302-306), both sides
// in one launch: elements [0, total) of X0 with peak[0..k), then X1 with
// peak[k..2k)
// Fixed grid, grid-stride; every CTA first checks the 2k peaks and leaves at
// once when none exceeds the threshold (the common case), so a sweep's
// rescale costs one short launch instead of a thread per vector entry.
__global__ void rescale_kernel(double* __restrict__ X0, double* __restrict__ X1, int64_t total, int k,
                               const double* __restrict__ peak) {
  BAMG_PDL_PROLOGUE();
  const int t = threadIdx.x;
  const bool big = t < 2 * k && peak[t] > 1e100;
  if (!__syncthreads_or(big)) return;
  const int64_t n = total / k;  // rows per block; thread per row
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + t; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool second = i >= n;
    double* x = (second ? X1 : X0) + (second ? i - n : i) * k;
    const double* pk = peak + (second ? k : 0);
    for (int c = 0; c < k; ++c) {
      const double p = pk[c];
      if (p > 1e100) x[c] = x[c] / p;
    }
  }
}

// u_c <- -u_c for flagged columns
// k in {8, 16}: flat double2 form (consecutive threads on consecutive 16-byte
// words), a word written only when one of its columns flips
template <int KK>
__global__ void flip_flat_kernel(double* __restrict__ X, int64_t total2, const double* __restrict__ flip) {
  BAMG_PDL_PROLOGUE();
  bool any = false;
#pragma unroll
  for (int c = 0; c < KK; ++c) any |= flip[c] != 0.0;
  if (!any) return;
  double2* x2 = reinterpret_cast<double2*>(X);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total2; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)((2 * i) & (KK - 1));
    const bool f0 = flip[c] != 0.0, f1 = flip[c + 1] != 0.0;
    if (f0 || f1) {
      double2 v = x2[i];
      if (f0) v.x = -v.x;
      if (f1) v.y = -v.y;
      x2[i] = v;
    }
  }
}

__global__ void flip_kernel(double* __restrict__ X, int64_t total, int k, const double* __restrict__ flip);

static int flip_dev(bamg_ctx* ctx, double* X, int64_t total, int k, const double* flip) {
  const bool al16 = (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  const int cap = ctx->num_sms * 8;
  if (al16 && (k == 8 || k == 16)) {
    const int g = std::min(grid_for(total / 2, 256), cap);
    if (k == 8) BAMG_LAUNCH(ctx, flip_flat_kernel<8>, g, 256, 0, X, total / 2, flip);
    else BAMG_LAUNCH(ctx, flip_flat_kernel<16>, g, 256, 0, X, total / 2, flip);
    return 0;
  }
  BAMG_LAUNCH(ctx, flip_kernel, std::min(grid_for(total / k, 256), cap), 256, 0, X, total, k, flip);
  return 0;
}

// grid-stride, thread per row; a CTA leaves at once when no column flips
// (the common case: the launch is then a few microseconds, not a 1M-thread pass)
__global__ void flip_kernel(double* __restrict__ X, int64_t total, int k, const double* __restrict__ flip) {
  BAMG_PDL_PROLOGUE();
  bool any = false;
  for (int c = 0; c < k; ++c) any |= flip[c] != 0.0;
  if (!any) return;
  const int64_t rows = total / k;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double* x = X + r * k;
    for (int c = 0; c < k; ++c)
      if (flip[c] != 0.0) x[c] = -x[c];
  }
}

// three column-dot sums in one pass (a.b, c.d, e.f per column), then -- in
// the last CTA to arrive -- the fixed-order sum of the per-CTA partials and
// the Rayleigh quotient finish (one launch instead of three)
__global__ void __launch_bounds__(RED_THREADS)
rayleigh_reduce_kernel(const double* __restrict__ A, const double* __restrict__ Bm, const double* __restrict__ Cm,
                       const double* __restrict__ Dm, const double* __restrict__ Em, const double* __restrict__ Fm,
                       int64_t n, int k, double* __restrict__ partial, unsigned int* __restrict__ counter,
                       double* __restrict__ dots, double* __restrict__ sigma, double* __restrict__ flip, int mode) {
  BAMG_PDL_PROLOGUE();
  constexpr int KM = 32;
  __shared__ double sh[RED_THREADS / 32][3 * KM];
  __shared__ bool last;
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = min(r0 + per, n);
  double a0[KM], a1[KM], a2[KM];
#pragma unroll
  for (int c = 0; c < KM; ++c) a0[c] = a1[c] = a2[c] = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    int64_t o = r * k;
#pragma unroll
    for (int c = 0; c < KM; ++c) {
      if (c < k) {
        a0[c] += A[o + c] * Bm[o + c];
        a1[c] += Cm[o + c] * Dm[o + c];
        a2[c] += Em[o + c] * Fm[o + c];
      }
    }
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < KM; ++c) {
    if (c < k) {
      double v0 = warp_sum(a0[c]), v1 = warp_sum(a1[c]), v2 = warp_sum(a2[c]);
      if (lane == 0) {
        sh[wid][c] = v0;
        sh[wid][k + c] = v1;
        sh[wid][2 * k + c] = v2;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 3 * k) {
    double v = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) v += sh[w][threadIdx.x];
    partial[(int64_t)blockIdx.x * 3 * k + threadIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int m = 3 * k, nb = gridDim.x;
  for (int i = wid; i < m; i += RED_THREADS / 32) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(partial + (int64_t)b * m + i);
    v = warp_sum(v);
    if (lane == 0) dots[i] = v;
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < k) {
    double du = sqrt(fmax(dots[c], 0.0));
    double dv = sqrt(fmax(dots[k + c], 0.0));
    double prev = sigma[c];
    double s = (du < 1e-15 || dv < 1e-15) ? prev : dots[2 * k + c] / (du * dv);
    if (mode == 0) {
      sigma[c] = s;
    } else {
      double f = 0.0;
      if (s < -1e-13) {
        f = 1.0;
        s = -s;
      }
      flip[c] = f;
      sigma[c] = fabs(s);
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// sigma update from (U, V): mode 0 smoothing, mode 1 refresh (+ flips of U).
int rayleigh_dev(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* M, const bamg_csr* N,
                 const double* U, const double* V, int64_t n, int k, double* sigma,
                 double* U_flip_or_null, int mode, double* work3) {
  double *MU, *NV, *AV, *dots, *partial, *flip;
  const double* mu = U;
  const double* nv = V;
  {  // one fused pass over A (and M, N): sparse.cu rayleigh_fused_kernel
    BAMG_TRY(arena_get(ctx, (size_t)3 * k, &dots));
    BAMG_TRY(arena_get(ctx, (size_t)k, &flip));
    int rc = rayleigh_fused_dev(ctx, A, U, V, k, sigma, flip, mode, dots, M, N);
    if (rc < 0) return rc;
    if (rc == 0) {
      if (mode == 1 && U_flip_or_null) {
        int64_t total = n * k;
        BAMG_TRY(flip_dev(ctx, U_flip_or_null, total, k, flip));
      }
      return 0;
    }
  }
  if (!work3) BAMG_TRY(arena_get(ctx, (size_t)3 * n * k, &work3));
  MU = work3;
  NV = work3 + (size_t)n * k;
  AV = work3 + (size_t)2 * n * k;
  if (M) {
    BAMG_TRY(spmm_dev(ctx, M, U, MU, k));
    mu = MU;
  }
  if (N) {
    BAMG_TRY(spmm_dev(ctx, N, V, NV, k));
    nv = NV;
  }
  BAMG_TRY(spmm_dev(ctx, A, V, AV, k));
  BAMG_TRY(arena_get(ctx, (size_t)3 * k, &dots));
  BAMG_TRY(arena_get(ctx, (size_t)RED_BLOCKS * 3 * k, &partial));
  BAMG_TRY(arena_get(ctx, (size_t)k, &flip));
  // rayleigh quotient: dots = [uMu(k) | vNv(k) | uBv(k)]; mode 0: sigma = s (or
  // prev when a normaliser collapses); mode 1 (refresh): s < -1e-13 -> flip
  BAMG_LAUNCH(ctx, rayleigh_reduce_kernel, red_blocks_for(n), RED_THREADS, 0, U, mu, V, nv, U, AV, n, k, partial,
              ctx->counters + 1, dots, sigma, flip, mode);
  if (mode == 1 && U_flip_or_null) {
    int64_t total = n * k;
    BAMG_TRY(flip_dev(ctx, U_flip_or_null, total, k, flip));
  }
  return 0;
}

int normalize_cols_dev(bamg_ctx* ctx, double* X, int64_t n, int k) {
  double* nrm;
  BAMG_TRY(arena_get(ctx, (size_t)k, &nrm));
  BAMG_TRY(colreduce(ctx, X, nullptr, n, k, 0, nrm, 1));
  int64_t total = n * k;
  (void)total;
  return col_scale_div_dev(ctx, X, n, k, nrm);
}

extern "C" int bamg_smooth_block(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                                 const bamg_csr* M, const bamg_csr* N, const double* d,
                                 const uint8_t* skip, const uint8_t* skip_t, double* U, double* V,
                                 double* sigma, int k, int nsweeps, double omega, int inhomogeneous,
                                 int smooth, int refresh) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, A && A_t && A->nrows == A->ncols, "square operator and its transpose expected");
  BAMG_REQUIRE(ctx, k >= 1 && k <= 32, "k must lie in [1, 32]");
  const int64_t n = A->nrows;
  const int64_t total = n * k;
  if (smooth && nsweeps > 0) {
    double *U2, *V2, *MU = nullptr, *NV = nullptr, *peak, *work3 = nullptr, *rd;
    if (inhomogeneous) BAMG_TRY(arena_get(ctx, (size_t)3 * total, &work3));
    // reciprocal diagonal once per block: every sweep divides through it
    // (div_rn_recip, bit-identical to the IEEE division)
    BAMG_TRY(arena_get(ctx, (size_t)n, &rd));
    BAMG_TRY(recip_dev(ctx, d, n, rd));
    BAMG_TRY(arena_get(ctx, (size_t)total, &U2));
    BAMG_TRY(arena_get(ctx, (size_t)total, &V2));
    BAMG_TRY(arena_get(ctx, (size_t)2 * k, &peak));
    if (inhomogeneous) {
      if (M) BAMG_TRY(arena_get(ctx, (size_t)total, &MU));
      if (N) BAMG_TRY(arena_get(ctx, (size_t)total, &NV));
    }
    // an odd number (>= 3) of sweeps would leave the result in the scratch pair and cost a
    // device copy of both blocks: a third buffer per side routes the last sweep into U / V
    // (U -> U2 -> U3 -> U)
    double *U3 = nullptr, *V3 = nullptr;
    if ((nsweeps & 1) && nsweeps >= 3) {
      BAMG_TRY(arena_get(ctx, (size_t)total, &U3));
      BAMG_TRY(arena_get(ctx, (size_t)total, &V3));
    }
    double *u = U, *v = V, *uo = U2, *vo = V2;
    for (int s = 0; s < nsweeps; ++s) {
      if (U3 && s >= 1) {  // sweeps 1 .. n-1 alternate U2 <-> U3 and the last one lands in U / V
        uo = s == nsweeps - 1 ? U : (u == U2 ? U3 : U2);
        vo = s == nsweeps - 1 ? V : (v == V2 ? V3 : V2);
      }
      BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(peak, 0, sizeof(double) * 2 * k, ctx->stream));
      // right vectors: rhs sigma * M u (the mass product fused into the sweep
      // when the rows kernel covers k), left vectors: sigma * N v
      int rcv = 1, rcu = 1;
      if (inhomogeneous && M) rcv = jacobi_mass_dev(ctx, A, d, skip, M, u, sigma, v, vo, k, omega, peak, rd);
      if (rcv < 0) return rcv;
      if (rcv == 1) {
        const double* bv = nullptr;
        if (inhomogeneous) {
          if (M) {
            BAMG_TRY(spmm_dev(ctx, M, u, MU, k));
            bv = MU;
          } else {
            bv = u;
          }
        }
        BAMG_TRY(jacobi_dev(ctx, A, d, skip, bv, inhomogeneous ? sigma : nullptr, v, vo, k, omega, peak, rd));
      }
      if (inhomogeneous && N) rcu = jacobi_mass_dev(ctx, A_t, d, skip_t, N, v, sigma, u, uo, k, omega, peak + k, rd);
      if (rcu < 0) return rcu;
      if (rcu == 1) {
        const double* bu = nullptr;
        if (inhomogeneous) {
          if (N) {
            BAMG_TRY(spmm_dev(ctx, N, v, NV, k));
            bu = NV;
          } else {
            bu = v;
          }
        }
        BAMG_TRY(jacobi_dev(ctx, A_t, d, skip_t, bu, inhomogeneous ? sigma : nullptr, u, uo, k, omega, peak + k, rd));
      }
      if (smooth == 1) {  // init_test_vectors (smooth == 2) has no runaway rescaling
        const int rg = grid_for(2 * n, 256);
        BAMG_LAUNCH(ctx, rescale_kernel, rg < ctx->num_sms * 8 ? rg : ctx->num_sms * 8, 256, 0, vo, uo, total, k,
                    peak);
      }
      std::swap(u, uo);
      std::swap(v, vo);
      if (inhomogeneous) BAMG_TRY(rayleigh_dev(ctx, A, M, N, u, v, n, k, sigma, nullptr, 0, work3));
    }
    if (u != U) BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(U, u, sizeof(double) * total, cudaMemcpyDeviceToDevice, ctx->stream));
    if (v != V) BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(V, v, sizeof(double) * total, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (refresh) {
    // normalise U and V, then U[:, 0] = 1/sqrt(n): the fill rides on U's division pass
    double *nu, *nv;
    BAMG_TRY(arena_get(ctx, (size_t)k, &nu));
    BAMG_TRY(arena_get(ctx, (size_t)k, &nv));
    BAMG_TRY(colreduce(ctx, U, nullptr, n, k, 0, nu, 1));
    BAMG_TRY(colreduce(ctx, V, nullptr, n, k, 0, nv, 1));
    BAMG_TRY(col_scale_div_dev(ctx, U, n, k, nu, 0, 1.0 / std::sqrt((double)n)));
    BAMG_TRY(col_scale_div_dev(ctx, V, n, k, nv));
    BAMG_TRY(rayleigh_dev(ctx, A, M, N, U, V, n, k, sigma, U, 1, nullptr));
  }
  return 0;
}

extern "C" int bamg_refresh_sigmas(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* M, const bamg_csr* N,
                                   const double* U, const double* V, double* U_flip, double* sigma, int k) {
  ctx->arena.reset();
  return rayleigh_dev(ctx, A, M, N, U, V, A->nrows, k, sigma, U_flip, 1, nullptr);
}

// --------------------------------------------------- singular test weights
// w = 1/res^2; nan/inf -> 1e16; min(w, 1e16); min(w, 1e4 * max(median, 1e-16));
// w[inf_slot] = inf   (interp.py:96-101)
__global__ void weights_finish_kernel(const double* __restrict__ res, int k, int inf_slot, double* __restrict__ w) {
  BAMG_PDL_PROLOGUE();
  if (threadIdx.x != 0) return;
  const double CAP = 1e16, SPREAD = 1e4;
  double t[32], s[32];
  for (int c = 0; c < k; ++c) {
    double r2 = res[c] * res[c];
    double v = 1.0 / r2;
    if (isnan(v)) v = CAP;
    if (isinf(v) && v > 0) v = CAP;
    v = fmin(v, CAP);
    t[c] = v;
    s[c] = v;
  }
  for (int i = 1; i < k; ++i) {  // insertion sort for the median
    double x = s[i];
    int j = i - 1;
    while (j >= 0 && s[j] > x) {
      s[j + 1] = s[j];
      --j;
    }
    s[j + 1] = x;
  }
  double med = (k & 1) ? s[k / 2] : (s[k / 2 - 1] + s[k / 2]) / 2.0;
  double lim = SPREAD * fmax(med, 1.0 / CAP);
  for (int c = 0; c < k; ++c) w[c] = fmin(t[c], lim);
  if (inf_slot >= 0 && inf_slot < k) w[inf_slot] = INFINITY;
}

extern "C" int bamg_test_weights(bamg_ctx* ctx, const bamg_csr* A, const double* X, int64_t n, int k,
                                 int inf_slot, double* Xn, double* w) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, k >= 1 && k <= 32, "k must lie in [1, 32]");
  const int64_t total = n * k;
  // Xn = X / |X| column-wise: the norms from X, the division straight into Xn (no copy of the block)
  double* nrm;
  BAMG_TRY(arena_get(ctx, (size_t)k, &nrm));
  BAMG_TRY(colreduce(ctx, X, nullptr, n, k, 0, nrm, 1));
  BAMG_TRY(col_scale_div_dev(ctx, Xn, n, k, nrm, -1, 0.0, X));
  double *R, *res;
  BAMG_TRY(arena_get(ctx, (size_t)total, &R));
  BAMG_TRY(arena_get(ctx, (size_t)k, &res));
  BAMG_TRY(spmm_dev(ctx, A, Xn, R, k));
  BAMG_TRY(colreduce(ctx, R, nullptr, n, k, 0, res, 1));
  BAMG_LAUNCH(ctx, weights_finish_kernel, 1, 32, 0, res, k, inf_slot, w);
  return 0;
}
