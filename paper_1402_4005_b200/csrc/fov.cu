// fov.cu -- field-of-values diagnostics on device (the
// reference's markovmg/fov.py).  Dense, n <= 1200 (fov.py:22 DENSE_CAP).
//
//  * bamg_fov_points: the angle sweep of fov_boundary (fov.py:85-115).  For
//    every angle theta_t = 2 pi t / T the top eigenvector of the Hermitian
//    part of e^{i theta} A,  H_t = cos(theta) H + i sin(theta) K  with
//    H = (A + A^T)/2 and K = (A - A^T)/2 (A real), supplies the supporting
//    point <A v, v>.  All T angles run together: Lanczos with full (CGS2)
//    reorthogonalisation on the real 2n x 2n form [[cH, -sK], [sK, cH]],
//    where one DMMA GEMM of [H; K] (2n x n) with the n x 2T block of every
//    angle's current Lanczos vector applies all T operators at once.  The
//    tridiagonal top eigenpair per angle: Sturm bisection + inverse
//    iteration, one thread per angle.  Convergence test |beta_m s_m| <=
//    tol |A|_F per angle; converged angles stop stepping.  The reference
//    warm-starts each angle from the previous angle's vector (eigsh, tol
//    1e-10) -- a start vector changes only the iteration count, not the
//    (unique) supporting point, so the angles are independent here.
//  * bamg_eigvals: eigenvalue_dots (fov.py:60-67, np.linalg.eigvals = LAPACK
//    dgeev): diagonal balancing by powers of 2 (dgebal's scaling), Householder reduction to upper
//    Hessenberg form (three launches per column), then the Francis
//    double-shift QR iteration with deflation in one CTA (the scalar control
//    on thread 0, each bulge step's row and column modifications spread over
//    the CTA; the matrix sits in shared memory when n <= 165, else in L2).
//  * bamg_range_basis: project_range / projected_preconditioned
//    (fov.py:194-223): one-sided Jacobi SVD (dense.cu), columns with
//    sigma > rank_tol sigma_max in descending order, basis^T A basis by two
//    DMMA GEMMs.
#include "common.cuh"
#include "internal.cuh"

#include <cmath>
#include <vector>

namespace {

constexpr int FOV_THREADS = 256;

__device__ __forceinline__ double fov_block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < nw; ++q) t += sh[q];
  __syncthreads();
  return t;
}

}  // namespace

// ------------------------------------------------------------ angle sweep
// HK (2n x n, column-major, ld 2n): rows 0..n-1 = H, rows n..2n-1 = K.
__global__ void fov_split_kernel(const double* __restrict__ A, int n, double* __restrict__ HK) {
  BAMG_PDL_PROLOGUE();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * n) return;
  const int i = (int)(t % n), j = (int)(t / n);
  const double a = A[t], b = A[(int64_t)i * n + j];  // A(i,j), A(j,i)
  HK[(int64_t)j * 2 * n + i] = 0.5 * (a + b);
  HK[(int64_t)j * 2 * n + n + i] = 0.5 * (a - b);
}

__global__ void fov_fro_kernel(const double* __restrict__ A, int64_t total, double* out) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) a += A[t] * A[t];
  a = fov_block_sum(a, sh);
  if (threadIdx.x == 0) out[0] = sqrt(a);
}

// q_0 of every angle: x = the reference's v0 (fov.py:100-102), y = 0.
__global__ void fov_start_kernel(double* __restrict__ Q0, int n, int T) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[32];
  __shared__ double inv;
  double a = 0.0;
  const double r = 1.0 / sqrt((double)n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = r + 1e-3 * cos((double)i) * r;
    a += v * v;
  }
  a = fov_block_sum(a, sh);
  if (threadIdx.x == 0) inv = 1.0 / sqrt(a);
  __syncthreads();
  const int t = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    Q0[(int64_t)t * n + i] = (r + 1e-3 * cos((double)i) * r) * inv;
    Q0[(int64_t)(T + t) * n + i] = 0.0;
  }
}

// One Lanczos step for every active angle (one CTA per angle):
//   w = R_t q_j  (from W = [H; K] [X Y]),  two classical Gram-Schmidt passes
//   against q_0..q_j, alpha_j = q_j^T w (both passes), beta_j = |w|,
//   q_{j+1} = w / beta_j.  status: 0 active, 1 converged, 2 invariant subspace.
// Basis slot i is an n x 2T column-major block (column t = x part of angle t,
// column T + t = its y part).
__global__ void __launch_bounds__(FOV_THREADS)
fov_lanczos_step_kernel(const double* __restrict__ W, int n, int T, const double* __restrict__ cs,
                        const double* __restrict__ sn, double* __restrict__ Q, int j, int mmax,
                        double* __restrict__ alpha, double* __restrict__ beta, int* __restrict__ status,
                        int* __restrict__ kdim, double brk) {
  BAMG_PDL_PROLOGUE();
  const int t = blockIdx.x;
  if (status[t] != 0) return;
  extern __shared__ double sm[];
  double* w = sm;            // 2n
  double* d = sm + 2 * n;    // j + 1 coefficients
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t ld2 = 2 * (int64_t)n, slot = 2 * (int64_t)n * T;
  const double c = cs[t], s = sn[t];
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const double hx = W[(int64_t)t * ld2 + r], kx = W[(int64_t)t * ld2 + n + r];
    const double hy = W[(int64_t)(T + t) * ld2 + r], ky = W[(int64_t)(T + t) * ld2 + n + r];
    w[r] = c * hx - s * ky;
    w[n + r] = c * hy + s * kx;
  }
  __syncthreads();
  double a_j = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = wid; i <= j; i += nw) {
      const double* xq = Q + i * slot + (int64_t)t * n;
      const double* yq = Q + i * slot + (int64_t)(T + t) * n;
      double acc = 0.0;
      for (int r = lane; r < n; r += 32) acc += xq[r] * w[r] + yq[r] * w[n + r];
      acc = warp_sum(acc);
      if (lane == 0) d[i] = acc;
    }
    __syncthreads();
    a_j += d[j];
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double sx = 0.0, sy = 0.0;
      for (int i = 0; i <= j; ++i) {
        sx += d[i] * Q[i * slot + (int64_t)t * n + r];
        sy += d[i] * Q[i * slot + (int64_t)(T + t) * n + r];
      }
      w[r] -= sx;
      w[n + r] -= sy;
    }
    __syncthreads();
  }
  double nrm = 0.0;
  for (int r = threadIdx.x; r < 2 * n; r += blockDim.x) nrm += w[r] * w[r];
  nrm = sqrt(fov_block_sum(nrm, sh));
  if (threadIdx.x == 0) {
    alpha[(int64_t)t * mmax + j] = a_j;
    beta[(int64_t)t * mmax + j] = nrm;
    kdim[t] = j + 1;
  }
  if (j + 1 >= mmax) return;
  const bool stop = !(nrm > brk);
  const double inv = stop ? 0.0 : 1.0 / nrm;
  double* xo = Q + (j + 1) * slot + (int64_t)t * n;
  double* yo = Q + (j + 1) * slot + (int64_t)(T + t) * n;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    xo[r] = w[r] * inv;
    yo[r] = w[n + r] * inv;
  }
  if (stop && threadIdx.x == 0) status[t] = 2;
}

// Top eigenpair of the m x m symmetric tridiagonal (alpha, beta) of every
// angle still in play: Sturm-count bisection for the largest eigenvalue, then
// three steps of inverse iteration (tridiagonal LU with partial pivoting).
// Marks angles converged when |beta_{m-1} s_{m-1}| <= tol (or the Krylov
// space is invariant).  `final` forces the eigenvector for every angle.
__global__ void fov_tridiag_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                                   const int* __restrict__ kdim, int T, int mmax, double tol, int* __restrict__ status,
                                   double* __restrict__ S, double* __restrict__ scratch, int* __restrict__ done_now,
                                   int final_pass) {
  BAMG_PDL_PROLOGUE();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  done_now[t] = 0;
  const int st = status[t];
  if (st == 1) return;  // converged earlier: its Ritz vector is already formed
  const int m = kdim[t];
  if (m <= 0) return;
  const double* a = alpha + (int64_t)t * mmax;
  const double* b = beta + (int64_t)t * mmax;
  double* s = S + (int64_t)t * mmax;
  double* dl = scratch + (int64_t)t * 5 * mmax;
  double* dd = dl + mmax;
  double* du = dd + mmax;
  double* du2 = du + mmax;
  double* y = du2 + mmax;
  // Gershgorin interval and scale
  double lo = 1e300, hi = -1e300, tn = 0.0;
  for (int i = 0; i < m; ++i) {
    const double off = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < m ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - off);
    hi = fmax(hi, a[i] + off);
    tn = fmax(tn, fabs(a[i]) + off);
  }
  const double eps = 2.220446049250313e-16;
  const double pivmin = fmax(1e-300, eps * eps * fmax(tn, 1e-300));
  // bisection: count(x) = # eigenvalues < x
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (!(mid > lo && mid < hi)) break;
    if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + pivmin) break;
    int cnt = 0;
    double q = a[0] - mid;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < m; ++i) {
      q = a[i] - mid - b[i - 1] * b[i - 1] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += q < 0.0;
    }
    if (cnt == m) hi = mid;
    else lo = mid;
  }
  const double lam = hi;
  // inverse iteration on (T - lam I)
  const double floorp = eps * fmax(tn, 1e-300);
  for (int i = 0; i < m; ++i) y[i] = 1.0 + 1e-2 * (double)((i * 7919) % 17) / 17.0;
  for (int it = 0; it < 3; ++it) {
    for (int i = 0; i < m; ++i) {
      dd[i] = a[i] - lam;
      du[i] = (i + 1 < m) ? b[i] : 0.0;
      dl[i] = (i + 1 < m) ? b[i] : 0.0;  // sub-diagonal entry (i+1, i)
      du2[i] = 0.0;
    }
    // factor with partial pivoting, solve in place on y
    for (int i = 0; i + 1 < m; ++i) {
      if (fabs(dd[i]) >= fabs(dl[i])) {
        if (dd[i] == 0.0) dd[i] = floorp;
        const double f = dl[i] / dd[i];
        dd[i + 1] -= f * du[i];
        y[i + 1] -= f * y[i];
        dl[i] = 0.0;  // marks "no swap" for nothing further
      } else {
        const double f = dd[i] / dl[i];
        dd[i] = dl[i];
        const double tmp = dd[i + 1];
        dd[i + 1] = du[i] - f * tmp;
        du[i] = tmp;
        if (i + 2 < m) {
          du2[i] = du[i + 1];
          du[i + 1] = -f * du[i + 1];
        }
        const double yt = y[i];
        y[i] = y[i + 1];
        y[i + 1] = yt - f * y[i + 1];
      }
    }
    if (fabs(dd[m - 1]) < floorp) dd[m - 1] = dd[m - 1] < 0.0 ? -floorp : floorp;
    for (int i = m - 1; i >= 0; --i) {
      if (fabs(dd[i]) < floorp) dd[i] = dd[i] < 0.0 ? -floorp : floorp;
      double v = y[i];
      if (i + 1 < m) v -= du[i] * y[i + 1];
      if (i + 2 < m) v -= du2[i] * y[i + 2];
      y[i] = v / dd[i];
    }
    double nr = 0.0;
    for (int i = 0; i < m; ++i) nr += y[i] * y[i];
    nr = sqrt(nr);
    if (!(nr > 0.0) || !isfinite(nr)) {
      for (int i = 0; i < m; ++i) y[i] = (i == m - 1) ? 1.0 : 0.0;
      nr = 1.0;
    }
    for (int i = 0; i < m; ++i) y[i] /= nr;
  }
  for (int i = 0; i < m; ++i) s[i] = y[i];
  const double res = fabs(b[m - 1] * y[m - 1]);
  if (st == 2 || res <= tol || final_pass) {
    status[t] = 1;
    done_now[t] = 1;
  }
}

// Ritz vectors v_t = sum_i s_t[i] q_i for the angles that converged in this
// check (done_now), normalised; written to V (n x 2T layout).
__global__ void __launch_bounds__(FOV_THREADS)
fov_ritz_kernel(const double* __restrict__ Q, const double* __restrict__ S, const int* __restrict__ kdim,
                const int* __restrict__ done_now, int n, int T, int mmax, double* __restrict__ V) {
  BAMG_PDL_PROLOGUE();
  const int t = blockIdx.x;
  if (!done_now[t]) return;
  __shared__ double sh[32];
  const int m = kdim[t];
  const int64_t slot = 2 * (int64_t)n * T;
  const double* s = S + (int64_t)t * mmax;
  double nrm = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < m; ++i) {
      x += s[i] * Q[i * slot + (int64_t)t * n + r];
      y += s[i] * Q[i * slot + (int64_t)(T + t) * n + r];
    }
    V[(int64_t)t * n + r] = x;
    V[(int64_t)(T + t) * n + r] = y;
    nrm += x * x + y * y;
  }
  nrm = sqrt(fov_block_sum(nrm, sh));
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    V[(int64_t)t * n + r] *= inv;
    V[(int64_t)(T + t) * n + r] *= inv;
  }
}

__global__ void fov_mark_active_kernel(const int* __restrict__ status, int T, int* __restrict__ flag) {
  BAMG_PDL_PROLOGUE();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) flag[t] = status[t] == 1 ? 0 : 1;
}

// restart: unconverged angles continue from their current Ritz vector
__global__ void fov_restart_kernel(const double* __restrict__ V, const int* __restrict__ status, int n, int T,
                                   double* __restrict__ Q0) {
  BAMG_PDL_PROLOGUE();
  const int t = blockIdx.x;
  if (status[t] == 1) return;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    Q0[(int64_t)t * n + r] = V[(int64_t)t * n + r];
    Q0[(int64_t)(T + t) * n + r] = V[(int64_t)(T + t) * n + r];
  }
}

// supporting point of angle t: v^H A v with v = x + i y,
//   = x^T H x + y^T H y + i (2 x^T K y)       (W = [H; K] [X Y])
__global__ void fov_points_kernel(const double* __restrict__ W, const double* __restrict__ V, int n, int T,
                                  double* __restrict__ pts) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[32];
  const int t = blockIdx.x;
  const int64_t ld2 = 2 * (int64_t)n;
  double re = 0.0, im = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const double x = V[(int64_t)t * n + r], y = V[(int64_t)(T + t) * n + r];
    re += x * W[(int64_t)t * ld2 + r] + y * W[(int64_t)(T + t) * ld2 + r];
    im += x * W[(int64_t)(T + t) * ld2 + n + r];
  }
  re = fov_block_sum(re, sh);
  im = fov_block_sum(im, sh);
  if (threadIdx.x == 0) {
    pts[2 * t] = re;
    pts[2 * t + 1] = 2.0 * im;
  }
}

// ------------------------------------------------------------ eigenvalues
// Diagonal balancing by powers of two, LAPACK dgebal's scaling loop (the
// permutation stage isolates nothing for an irreducible chain and is not
// done): 2-norms of column i and row i (diagonal included), scale by 2^k while
// the pair gets more than 5 % closer; exact in floating point.  One CTA.
__global__ void __launch_bounds__(1024) eig_balance_kernel(double* A, int n) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[32];
  __shared__ int again;
  for (int sweep = 0; sweep < 200; ++sweep) {
    if (threadIdx.x == 0) again = 0;
    __syncthreads();
    for (int i = 0; i < n; ++i) {
      double c = 0.0, r = 0.0;
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double x = A[(int64_t)i * n + j];  // column i
        const double y = A[(int64_t)j * n + i];  // row i
        c += x * x;
        r += y * y;
      }
      c = sqrt(fov_block_sum(c, sh));
      r = sqrt(fov_block_sum(r, sh));
      if (c == 0.0 || r == 0.0) continue;
      double g = r / 2.0, f = 1.0;
      const double s = c + r;
      while (c < g && f < 1e300 && c < 1e300) {
        f *= 2.0;
        c *= 2.0;
        r /= 2.0;
        g /= 2.0;
      }
      g = c / 2.0;
      while (g >= r && f > 1e-300 && r < 1e300) {
        f /= 2.0;
        c /= 2.0;
        g /= 2.0;
        r *= 2.0;
      }
      if (c + r < 0.95 * s) {
        const double gi = 1.0 / f;
        for (int j = threadIdx.x; j < n; j += blockDim.x) A[(int64_t)j * n + i] *= gi;  // row i
        __syncthreads();
        for (int j = threadIdx.x; j < n; j += blockDim.x) A[(int64_t)i * n + j] *= f;   // column i
        if (threadIdx.x == 0) again = 1;
      }
      __syncthreads();
    }
    __syncthreads();
    if (!again) break;
    __syncthreads();
  }
}

// Householder vector of column k below the subdiagonal: v (rows k+1..n-1),
// beta = 2 / v^T v; column k becomes (.., s, 0, .., 0).
__global__ void eig_hh_vec_kernel(double* A, int n, int k, double* __restrict__ v, double* __restrict__ beta) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[32];
  double* col = A + (int64_t)k * n;
  double a = 0.0;
  for (int i = k + 2 + threadIdx.x; i < n; i += blockDim.x) a += col[i] * col[i];
  const double tail = fov_block_sum(a, sh);
  const double x0 = col[k + 1];
  if (tail == 0.0) {  // already Hessenberg in this column
    if (threadIdx.x == 0) beta[0] = 0.0;
    return;
  }
  const double nx = sqrt(x0 * x0 + tail);
  const double sg = x0 >= 0.0 ? 1.0 : -1.0;
  const double v0 = x0 + sg * nx;
  for (int i = k + 2 + threadIdx.x; i < n; i += blockDim.x) {
    v[i] = col[i];
    col[i] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    v[k + 1] = v0;
    col[k + 1] = -sg * nx;
    beta[0] = 2.0 / (v0 * v0 + tail);
  }
}

// A(k+1:, j) -= beta v (v^T A(k+1:, j)) for j > k: one warp per column
__global__ void eig_hh_left_kernel(double* A, int n, int k, const double* __restrict__ v,
                                   const double* __restrict__ beta) {
  BAMG_PDL_PROLOGUE();
  const double b = beta[0];
  if (b == 0.0) return;
  const int lane = threadIdx.x & 31;
  const int j = k + 1 + (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (j >= n) return;
  double* col = A + (int64_t)j * n;
  double w = 0.0;
  for (int i = k + 1 + lane; i < n; i += 32) w += v[i] * col[i];
  w = warp_sum(w) * b;
  for (int i = k + 1 + lane; i < n; i += 32) col[i] -= w * v[i];
}

// A(:, k+1:) -= beta (A(:, k+1:) v) v^T: 32 rows x 8 column slices per CTA
__global__ void __launch_bounds__(256) eig_hh_right_kernel(double* A, int n, int k, const double* __restrict__ v,
                                                           const double* __restrict__ beta) {
  BAMG_PDL_PROLOGUE();
  const double b = beta[0];
  if (b == 0.0) return;
  __shared__ double part[8][33];
  const int rl = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + rl;
  double u = 0.0;
  if (i < n)
    for (int j = k + 1 + sl; j < n; j += 8) u += A[(int64_t)j * n + i] * v[j];
  part[sl][rl] = u;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) tot += part[q][rl];
  tot *= b;
  if (i < n)
    for (int j = k + 1 + sl; j < n; j += 8) A[(int64_t)j * n + i] -= tot * v[j];
}

// Francis double-shift QR on the upper Hessenberg matrix (eigenvalues only),
// one CTA.  Scalar control on thread 0; each bulge step's row modification
// (columns k..nn) and column modification (rows l..min(nn, k+3)) run across
// the CTA.  `M` is the matrix (global, or a shared-memory copy), ld = n.
constexpr int HQR_THREADS = 512;
constexpr int HQR_SMEM_N = 165;
__global__ void __launch_bounds__(HQR_THREADS)
eig_hqr_kernel(double* Ag, int n, double* __restrict__ wr, double* __restrict__ wi, int* __restrict__ info) {
  BAMG_PDL_PROLOGUE();
  extern __shared__ double smA[];
  __shared__ double sh[32];
  __shared__ double par[8];
  __shared__ int ctl[6];
  const bool in_smem = n <= HQR_SMEM_N;
  double* A = in_smem ? smA : Ag;
  if (in_smem) {
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) smA[t] = Ag[t];
    __syncthreads();
  }
#define HA(i, j) A[(int64_t)(j) * n + (i)]
  double loc = 0.0;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int i = t % n, j = t / n;
    if (i <= j + 1) loc += fabs(A[t]);
  }
  const double anorm = fov_block_sum(loc, sh);
  // thread-0 state
  int nn = n - 1, its = 0, l = 0;
  double tshift = 0.0, x = 0.0, y = 0.0, w = 0.0;
  if (threadIdx.x == 0) info[0] = 0;
  constexpr int ITMAX = 60;
  for (;;) {
    // ---- thread 0 decides the next action: 0 = done, 1 = deflated, 2 = QR sweep, 3 = failure
    if (threadIdx.x == 0) {
      int action = 1;
      if (nn < 0) {
        action = 0;
      } else {
        for (l = nn; l >= 1; --l) {
          double s = fabs(HA(l - 1, l - 1)) + fabs(HA(l, l));
          if (s == 0.0) s = anorm;
          if (fabs(HA(l, l - 1)) + s == s) {
            HA(l, l - 1) = 0.0;
            break;
          }
        }
        x = HA(nn, nn);
        if (l == nn) {
          wr[nn] = x + tshift;
          wi[nn] = 0.0;
          --nn;
          its = 0;
        } else {
          y = HA(nn - 1, nn - 1);
          w = HA(nn, nn - 1) * HA(nn - 1, nn);
          if (l == nn - 1) {
            const double p = 0.5 * (y - x);
            const double q = p * p + w;
            double z = sqrt(fabs(q));
            x += tshift;
            if (q >= 0.0) {
              z = p + (p >= 0.0 ? fabs(z) : -fabs(z));
              wr[nn - 1] = wr[nn] = x + z;
              if (z != 0.0) wr[nn] = x - w / z;
              wi[nn - 1] = wi[nn] = 0.0;
            } else {
              wr[nn - 1] = wr[nn] = x + p;
              wi[nn - 1] = -z;
              wi[nn] = z;
            }
            nn -= 2;
            its = 0;
          } else if (its >= ITMAX) {
            info[0] = nn + 1;
            action = 3;
          } else {
            if (its == 10 || its == 20) {  // exceptional shift
              tshift += x;
              for (int i = 0; i <= nn; ++i) HA(i, i) -= x;
              const double s = fabs(HA(nn, nn - 1)) + fabs(HA(nn - 1, nn - 2));
              y = x = 0.75 * s;
              w = -0.4375 * s * s;
            }
            ++its;
            int m;
            double p = 0.0, q = 0.0, r = 0.0;
            for (m = nn - 2; m >= l; --m) {
              const double z = HA(m, m);
              double rr = x - z, ss = y - z;
              p = (rr * ss - w) / HA(m + 1, m) + HA(m, m + 1);
              q = HA(m + 1, m + 1) - z - rr - ss;
              r = HA(m + 2, m + 1);
              ss = fabs(p) + fabs(q) + fabs(r);
              p /= ss;
              q /= ss;
              r /= ss;
              if (m == l) break;
              const double u = fabs(HA(m, m - 1)) * (fabs(q) + fabs(r));
              const double vv = fabs(p) * (fabs(HA(m - 1, m - 1)) + fabs(z) + fabs(HA(m + 1, m + 1)));
              if (u + vv == vv) break;
            }
            for (int i = m + 2; i <= nn; ++i) {
              HA(i, i - 2) = 0.0;
              if (i != m + 2) HA(i, i - 3) = 0.0;
            }
            par[0] = p;
            par[1] = q;
            par[2] = r;
            ctl[1] = m;
            action = 2;
          }
        }
      }
      ctl[0] = action;
      ctl[2] = nn;
      ctl[3] = l;
    }
    __syncthreads();
    const int action = ctl[0];
    if (action == 0 || action == 3) break;
    if (action == 1) continue;
    const int m = ctl[1], nnq = ctl[2], lq = ctl[3];
    double p = par[0], q = par[1], r = par[2];
    __syncthreads();
    for (int k = m; k <= nnq - 1; ++k) {
      if (threadIdx.x == 0) {
        double xx = 0.0;
        if (k != m) {
          p = HA(k, k - 1);
          q = HA(k + 1, k - 1);
          r = 0.0;
          if (k != nnq - 1) r = HA(k + 2, k - 1);
          xx = fabs(p) + fabs(q) + fabs(r);
          if (xx != 0.0) {
            p /= xx;
            q /= xx;
            r /= xx;
          }
        }
        const double nrm = sqrt(p * p + q * q + r * r);
        const double s = p >= 0.0 ? nrm : -nrm;
        int go = 0;
        if (s != 0.0) {
          if (k == m) {
            if (lq != m) HA(k, k - 1) = -HA(k, k - 1);
          } else {
            HA(k, k - 1) = -s * xx;
          }
          p += s;
          par[3] = p / s;  // x
          par[4] = q / s;  // y
          par[5] = r / s;  // z
          par[6] = q / p;  // q
          par[7] = r / p;  // r
          go = 1;
        }
        ctl[4] = go;
      }
      __syncthreads();
      if (ctl[4]) {
        const double hx = par[3], hy = par[4], hz = par[5], hq = par[6], hr = par[7];
        const bool three = k != nnq - 1;
        for (int j = k + threadIdx.x; j <= nnq; j += blockDim.x) {  // row modification
          double pp = HA(k, j) + hq * HA(k + 1, j);
          if (three) {
            pp += hr * HA(k + 2, j);
            HA(k + 2, j) -= pp * hz;
          }
          HA(k + 1, j) -= pp * hy;
          HA(k, j) -= pp * hx;
        }
        __syncthreads();
        const int mmin = nnq < k + 3 ? nnq : k + 3;
        for (int i = lq + threadIdx.x; i <= mmin; i += blockDim.x) {  // column modification
          double pp = hx * HA(i, k) + hy * HA(i, k + 1);
          if (three) {
            pp += hz * HA(i, k + 2);
            HA(i, k + 2) -= pp * hr;
          }
          HA(i, k + 1) -= pp * hq;
          HA(i, k) -= pp;
        }
      }
      __syncthreads();
    }
  }
#undef HA
}

// ------------------------------------------------------------ range basis
// basis[:, c] = G[:, perm[n-1-c]] / sig[perm[n-1-c]]   (descending sigma)
__global__ void range_gather_kernel(const double* __restrict__ G, const double* __restrict__ sig,
                                    const int* __restrict__ perm, int n, int r, double* __restrict__ basis) {
  BAMG_PDL_PROLOGUE();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * r) return;
  const int c = (int)(t / n), i = (int)(t % n);
  const int idx = perm[n - 1 - c];
  basis[t] = G[(int64_t)idx * n + i] / sig[idx];
}

__global__ void range_sort_kernel(const double* __restrict__ sig, int n, int* __restrict__ perm) {
  BAMG_PDL_PROLOGUE();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double si = sig[i];
  int rk = 0;
  for (int j = 0; j < n; ++j) {
    const double sj = sig[j];
    if (sj < si || (sj == si && j > i)) ++rk;  // ties: lower index ranks higher (first in descending order)
  }
  perm[rk] = i;
}

// ================================================================= C ABI
extern "C" int bamg_fov_points(bamg_ctx* ctx, const double* A, int n, int n_angles, double tol, double* points,
                               int* iterations) {
  if (!ctx) return -2;
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, n >= 1, "empty matrix");
  BAMG_REQUIRE(ctx, n_angles >= 1, "need at least one angle");
  const int T = n_angles;
  const int mmax = std::min(2 * n, 400);
  const int64_t slot = 2 * (int64_t)n * T;
  double *HK, *Q, *W, *V, *alpha, *beta, *S, *scr, *cs, *sn, *fro;
  int *status, *kdim, *done_now;
  BAMG_TRY(arena_get(ctx, (size_t)2 * n * n, &HK));
  BAMG_TRY(arena_get(ctx, (size_t)mmax * slot, &Q));
  BAMG_TRY(arena_get(ctx, (size_t)2 * slot, &W));
  BAMG_TRY(arena_get(ctx, (size_t)slot, &V));
  BAMG_TRY(arena_get(ctx, (size_t)T * mmax, &alpha));
  BAMG_TRY(arena_get(ctx, (size_t)T * mmax, &beta));
  BAMG_TRY(arena_get(ctx, (size_t)T * mmax, &S));
  BAMG_TRY(arena_get(ctx, (size_t)T * mmax * 5, &scr));
  BAMG_TRY(arena_get(ctx, (size_t)T, &cs));
  BAMG_TRY(arena_get(ctx, (size_t)T, &sn));
  BAMG_TRY(arena_get(ctx, 1, &fro));
  BAMG_TRY(arena_get(ctx, (size_t)T, &status));
  BAMG_TRY(arena_get(ctx, (size_t)T, &kdim));
  BAMG_TRY(arena_get(ctx, (size_t)T, &done_now));
  {
    std::vector<double> c(T), s(T);
    for (int t = 0; t < T; ++t) {
      const double th = 2.0 * M_PI * t / T;  // fov.py:103-104
      c[t] = std::cos(th);
      s[t] = std::sin(th);
    }
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(cs, c.data(), sizeof(double) * T, cudaMemcpyHostToDevice, ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(sn, s.data(), sizeof(double) * T, cudaMemcpyHostToDevice, ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
  }
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(status, 0, sizeof(int) * T, ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(kdim, 0, sizeof(int) * T, ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(V, 0, sizeof(double) * slot, ctx->stream));
  BAMG_LAUNCH(ctx, fov_split_kernel, grid_for((int64_t)n * n, 256), 256, 0, A, n, HK);
  BAMG_LAUNCH(ctx, fov_fro_kernel, 1, 1024, 0, A, (int64_t)n * n, fro);
  double afro;
  BAMG_TRY(ctx_read_doubles(ctx, fro, 1, &afro));
  const double scale = afro > 0.0 ? afro : 1.0;
  const double rtol = (tol > 0.0 ? tol : 1e-13) * scale;
  const double brk = 1e-14 * scale;
  BAMG_LAUNCH(ctx, fov_start_kernel, T, 256, 0, Q, n, T);
  const size_t smem = sizeof(double) * (2 * (size_t)n + mmax);
  BAMG_TRY(smem_optin(ctx, (const void*)fov_lanczos_step_kernel, smem));
  int total_steps = 0;
  // after MAX_RESTARTS cycles the last check accepts every angle's current
  // Ritz vector (the reference's eigsh falls back to a dense eigh instead)
  constexpr int MAX_RESTARTS = 40, CHECK_EVERY = 16;
  int restarts = 0;
  std::vector<int> hstat(T);
  for (;;) {
    bool all_done = false;
    for (int j = 0; j < mmax; ++j) {
      BAMG_TRY(dgemm_dev(ctx, false, false, 2 * n, 2 * T, n, 1.0, HK, 2 * n, Q + j * slot, n, 0.0, W, 2 * n));
      BAMG_LAUNCH(ctx, fov_lanczos_step_kernel, T, FOV_THREADS, smem, W, n, T, cs, sn, Q, j, mmax, alpha, beta,
                  status, kdim, brk);
      ++total_steps;
      const bool last = (j + 1 == mmax);
      if (((j + 1) % CHECK_EVERY == 0) || last) {
        const int final_pass = (last && restarts + 1 >= MAX_RESTARTS) ? 1 : 0;
        BAMG_LAUNCH(ctx, fov_tridiag_kernel, grid_for(T, 64), 64, 0, alpha, beta, kdim, T, mmax, rtol, status, S,
                    scr, done_now, final_pass);
        BAMG_LAUNCH(ctx, fov_ritz_kernel, T, FOV_THREADS, 0, Q, S, kdim, done_now, n, T, mmax, V);
        BAMG_TRY(ctx_read_i32(ctx, status, T, hstat.data()));
        all_done = true;
        for (int t = 0; t < T; ++t) all_done &= hstat[t] == 1;
        if (all_done) break;
      }
    }
    if (all_done) break;
    ++restarts;
    // still-active angles: Ritz vector of the full basis (S holds their
    // tridiagonal eigenvectors from the last check), restart from it
    BAMG_LAUNCH(ctx, fov_mark_active_kernel, grid_for(T, 256), 256, 0, (const int*)status, T, done_now);
    BAMG_LAUNCH(ctx, fov_ritz_kernel, T, FOV_THREADS, 0, Q, S, kdim, done_now, n, T, mmax, V);
    BAMG_LAUNCH(ctx, fov_restart_kernel, T, 256, 0, V, status, n, T, Q);
  }
  BAMG_TRY(dgemm_dev(ctx, false, false, 2 * n, 2 * T, n, 1.0, HK, 2 * n, V, n, 0.0, W, 2 * n));
  BAMG_LAUNCH(ctx, fov_points_kernel, T, 256, 0, W, V, n, T, points);
  if (iterations) *iterations = total_steps;
  return 0;
}

extern "C" int bamg_eigvals(bamg_ctx* ctx, const double* A, int n, double* wr, double* wi) {
  if (!ctx) return -2;
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, n >= 1, "empty matrix");
  double *H, *v, *beta;
  int* info;
  BAMG_TRY(arena_get(ctx, (size_t)n * n, &H));
  BAMG_TRY(arena_get(ctx, (size_t)n + 2, &v));
  BAMG_TRY(arena_get(ctx, 1, &beta));
  BAMG_TRY(arena_get(ctx, 1, &info));
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(H, A, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, ctx->stream));
  BAMG_LAUNCH(ctx, eig_balance_kernel, 1, 1024, 0, H, n);
  for (int k = 0; k + 2 < n; ++k) {
    BAMG_LAUNCH(ctx, eig_hh_vec_kernel, 1, 256, 0, H, n, k, v, beta);
    BAMG_LAUNCH(ctx, eig_hh_left_kernel, grid_for((int64_t)(n - k - 1) * 32, 256), 256, 0, H, n, k, (const double*)v,
                (const double*)beta);
    BAMG_LAUNCH(ctx, eig_hh_right_kernel, (n + 31) / 32, 256, 0, H, n, k, (const double*)v, (const double*)beta);
  }
  const size_t smem = n <= HQR_SMEM_N ? sizeof(double) * (size_t)n * n : 0;
  if (smem) BAMG_TRY(smem_optin(ctx, (const void*)eig_hqr_kernel, smem));
  BAMG_LAUNCH(ctx, eig_hqr_kernel, 1, HQR_THREADS, smem, H, n, wr, wi, info);
  int h;
  BAMG_TRY(ctx_read_i32(ctx, info, 1, &h));
  if (h != 0) {
    ctx->err = "eigenvalue QR iteration did not converge";
    return 2;
  }
  return 0;
}

extern "C" int bamg_range_basis(bamg_ctx* ctx, const double* A, int n, double rank_tol, double* basis,
                                double* projected, int* rank) {
  if (!ctx) return -2;
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, n >= 1, "empty matrix");
  double *G, *Vr, *sig, *T1;
  int* perm;
  BAMG_TRY(arena_get(ctx, (size_t)n * n, &G));
  BAMG_TRY(arena_get(ctx, (size_t)n * n, &Vr));
  BAMG_TRY(arena_get(ctx, (size_t)n, &sig));
  BAMG_TRY(arena_get(ctx, (size_t)n * n, &T1));
  BAMG_TRY(arena_get(ctx, (size_t)n, &perm));
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(G, A, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (n >= 2) {
    BAMG_TRY(jacobi_svd_public(ctx, G, n, n, Vr, sig));
  } else {
    BAMG_LAUNCH(ctx, fov_fro_kernel, 1, 32, 0, (const double*)G, (int64_t)1, sig);
  }
  std::vector<double> hs(n);
  BAMG_TRY(ctx_read_doubles(ctx, sig, n, hs.data()));
  double smax = 0.0;
  for (double s : hs) smax = std::max(smax, s);
  if (!(smax > 0.0)) {
    ctx->err = "argument error: zero matrix has no range to project onto";
    return -2;
  }
  int r = 0;
  for (double s : hs) r += s > rank_tol * smax;
  *rank = r;
  if (!basis) return 0;  // rank query only
  BAMG_LAUNCH(ctx, range_sort_kernel, grid_for(n, 256), 256, 0, sig, n, perm);
  BAMG_LAUNCH(ctx, range_gather_kernel, grid_for((int64_t)n * r, 256), 256, 0, G, sig, perm, n, r, basis);
  // projected = basis^T (A basis)
  BAMG_TRY(dgemm_dev(ctx, false, false, n, r, n, 1.0, A, n, basis, n, 0.0, T1, n));
  BAMG_TRY(dgemm_dev(ctx, true, false, r, r, n, 1.0, basis, n, T1, n, 0.0, projected, r));
  return 0;
}
