// interp.cu -- least-squares interpolation / restriction rows
// (interp.py:105-289): one thread per fine point on the production path
// (fit_rows_thread_kernel: corrected semi-normal equations with compile-time
// trial sizes), one warp per point for the rest (fit_rows_kernel below,
// Householder QR with the reference's pseudo-inverse branch).
//
// Per fine point i the warp
//   1. builds the candidate list: coarse points among the radius-1
//      neighbours in pattern(B + B^T), escalating to radius 2 when there are
//      none (interp.py:241-249, 274-276), sorted ascending;
//   2. runs the greedy caliber-bounded selection of fit_row
//      (interp.py:129-238) with the reference's exact decision rules: strict
//      `<` argmin over candidates in ascending order, the |coef| > 10 veto
//      after the first step, the relative-improvement stop, the 1e-30 stop,
//      negative-coefficient dropping (argmin first) and the inert single-point
//      row, the sum-to-one constrained variant used for Q;
//   3. solves every trial model as a ridge least-squares problem by
//      Householder QR held in the warp: lane l owns LS row l (the finite-
//      weight tests first, then the ridge rows lambda*I), column norms and
//      reflector applications are warp-shuffle reductions, back
//      substitution broadcasts one coefficient per step.  The
//      |R_jj| < 1e-13 max|R| branch of qr_solve_ls (dense.py:134-152) falls
//      back to a warp one-sided-Jacobi pseudo-inverse (dense.py:102-115).
// Decisions compare warp-reduced fp64 values; the reference's decision
// margins are >= 1e-9 relative, far above the 1e-15 rounding differences
// between this QR and LAPACK's, so selected patterns are bit-identical.
#include <cmath>
#include <cstdlib>

#include <utility>

#include "internal.cuh"

constexpr int FIT_WARPS = 4;     // warps per CTA
constexpr int CMAX = 8;          // largest caliber supported
constexpr int MAXCAND = 256;     // candidate list capacity per point (warp path)

struct FitLane {
  int lane;
  int rf;        // number of finite-weight tests (data rows)
  int f;         // test index owned by this lane (lane < rf)
  double y;      // sqrt-weight-free fine value y_f
  double sw;     // sqrt(w_f)
};

__device__ __forceinline__ double wsum(double v) { return warp_sum(v); }

__device__ __forceinline__ double cval(const double* __restrict__ X, int k, int point, int f) {
  return __ldg(X + (int64_t)point * k + f);
}

// Warp one-sided Jacobi pseudo-inverse solve of the nr x nc system held as
// lane rows a0[] with rhs b0 (rank_tol 1e-12 relative to sigma_max).
__device__ void warp_pinv_solve(const FitLane& L, int nr, int nc, const double* a0, double b0,
                                double* coef, double* sV) {
  double g[CMAX];
#pragma unroll
  for (int q = 0; q < CMAX; ++q) g[q] = (q < nc && L.lane < nr) ? a0[q] : 0.0;
  // V = I (nc x nc, row-major in shared memory, owned by this warp)
  if (L.lane < nc * nc) sV[L.lane] = (L.lane / nc == L.lane % nc) ? 1.0 : 0.0;
  for (int i = L.lane + 32; i < nc * nc; i += 32) sV[i] = (i / nc == i % nc) ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < nc - 1; ++p) {
      for (int q = p + 1; q < nc; ++q) {
        double gp = 0.0, gq = 0.0;
#pragma unroll
        for (int t = 0; t < CMAX; ++t) {
          if (t == p) gp = g[t];
          if (t == q) gq = g[t];
        }
        double al = wsum(gp * gp), be = wsum(gq * gq), ga = wsum(gp * gq);
        if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
          rotated = true;
          double zeta = (be - al) / (2.0 * ga);
          double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          double np = c * gp - s * gq, nq = s * gp + c * gq;
#pragma unroll
          for (int u = 0; u < CMAX; ++u) {
            if (u == p) g[u] = np;
            if (u == q) g[u] = nq;
          }
          __syncwarp();
          if (L.lane < nc) {
            double vp = sV[L.lane * nc + p], vq = sV[L.lane * nc + q];
            sV[L.lane * nc + p] = c * vp - s * vq;
            sV[L.lane * nc + q] = s * vp + c * vq;
          }
          __syncwarp();
        }
      }
    }
    if (!rotated) break;
  }
  double sig[CMAX], gb[CMAX];
  double smax = 0.0;
#pragma unroll
  for (int q = 0; q < CMAX; ++q) {
    if (q < nc) {
      sig[q] = sqrt(wsum(g[q] * g[q]));
      gb[q] = wsum(g[q] * (L.lane < nr ? b0 : 0.0));
      smax = fmax(smax, sig[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < CMAX; ++q) {
    if (q < nc) {
      double x = 0.0;
      for (int i = 0; i < nc; ++i) {
        double si = 0.0, gbi = 0.0;
#pragma unroll
        for (int t = 0; t < CMAX; ++t)
          if (t == i) {
            si = sig[t];
            gbi = gb[t];
          }
        if (smax > 0.0 && si > 1e-12 * smax) x += sV[q * nc + i] * (gbi / (si * si));
      }
      coef[q] = x;
    }
  }
  __syncwarp();
}

// Ridge LS for one column set.  cols[q] is a candidate POINT index; with
// `base` >= 0 the columns are differenced against the base point and the
// target is y - C_base (the constrained elimination of interp.py:180-186).
// Returns coefficients (nc), misfit over the data rows and the objective.
__device__ void ls_solve(const FitLane& L, const double* __restrict__ X, int k, const int* cols, int nc,
                         int base, double lam, double* coef, double* data_out, double* total_out,
                         unsigned long long* fallback, double* sV) {
  const bool ridge = lam > 0.0;
  const int nr = L.rf + (ridge ? nc : 0);
  double a[CMAX], a0[CMAX];
  double b = 0.0;
  if (L.lane < L.rf) {
    double cb = base >= 0 ? cval(X, k, base, L.f) : 0.0;
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      if (q < nc) {
        double c = cval(X, k, cols[q], L.f);
        a[q] = L.sw * (base >= 0 ? c - cb : c);
      } else {
        a[q] = 0.0;
      }
    }
    b = L.sw * (base >= 0 ? L.y - cb : L.y);
  } else if (ridge && L.lane < nr) {
    int rr = L.lane - L.rf;
#pragma unroll
    for (int q = 0; q < CMAX; ++q) a[q] = (q == rr) ? lam : 0.0;
  } else {
#pragma unroll
    for (int q = 0; q < CMAX; ++q) a[q] = 0.0;
  }
#pragma unroll
  for (int q = 0; q < CMAX; ++q) a0[q] = a[q];
  const double b0 = b;
  // Householder QR (dgeqr2 conventions), reflectors applied to b on the fly
#pragma unroll
  for (int j = 0; j < CMAX; ++j) {
    if (j < nc) {
      double xj = a[j];
      double alpha = __shfl_sync(0xffffffffu, xj, j);
      double below = (L.lane > j && L.lane < nr) ? xj : 0.0;
      double xn2 = wsum(below * below);
      if (xn2 != 0.0) {
        double xnorm = sqrt(xn2);
        double beta = -copysign(hypot(alpha, xnorm), alpha);
        double tau = (beta - alpha) / beta;
        double scal = 1.0 / (alpha - beta);
        double v = (L.lane == j) ? 1.0 : ((L.lane > j && L.lane < nr) ? xj * scal : 0.0);
#pragma unroll
        for (int q = 0; q < CMAX; ++q) {
          if (q > j && q < nc) {
            double dq = wsum(v * a[q]);
            a[q] -= tau * dq * v;
          }
        }
        double db = wsum(v * b);
        b -= tau * db * v;
        if (L.lane == j) a[j] = beta;
        else if (L.lane > j) a[j] = 0.0;
      }
    }
  }
  // rank test of qr_solve_ls: min |R_jj| < 1e-13 max |R|
  double rmax = 0.0, dmin = INFINITY;
  if (L.lane < nc) {
#pragma unroll
    for (int q = 0; q < CMAX; ++q)
      if (q >= L.lane && q < nc) rmax = fmax(rmax, fabs(a[q]));
#pragma unroll
    for (int q = 0; q < CMAX; ++q)
      if (q == L.lane) dmin = fabs(a[q]);
  }
  rmax = warp_max(rmax);
  dmin = -warp_max(-dmin);
  if (rmax == 0.0 || dmin < 1e-13 * rmax) {
    if (L.lane == 0) atomicAdd(fallback, 1ull);
    warp_pinv_solve(L, nr, nc, a0, b0, coef, sV);
  } else {
    // back substitution: lane j owns row j of R and (Q^T b)_j
#pragma unroll
    for (int q = 0; q < CMAX; ++q) coef[q] = 0.0;
#pragma unroll
    for (int j = CMAX - 1; j >= 0; --j) {
      if (j < nc) {
        double s = b;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q > j && q < nc) s -= a[q] * coef[q];
        double rjj = 0.0;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q == j) rjj = a[q];
        double cj = s / rjj;
        cj = __shfl_sync(0xffffffffu, cj, j);
        coef[j] = cj;
      }
    }
  }
  // misfit over the data rows, objective with the ridge penalty
  double res = 0.0;
  if (L.lane < L.rf) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < CMAX; ++q)
      if (q < nc) t += a0[q] * coef[q];
    res = t - b0;
  }
  double data = wsum(res * res);
  double cc = 0.0;
#pragma unroll
  for (int q = 0; q < CMAX; ++q)
    if (q < nc) cc += coef[q] * coef[q];
  *data_out = data;
  *total_out = data + lam * lam * cc;
}

struct Model {
  int pos[CMAX];   // positions into the candidate list, model order
  int len;
  double coef[CMAX];
  double data, total;
};

// solve_model of fit_row (interp.py:176-199): fit `trial`, dropping the most
// negative coefficient until all are non-negative.
__device__ void solve_model(const FitLane& L, const double* __restrict__ X, int k, const int* cand,
                            const int* trial, int tlen, bool constrain, bool nonneg, double lam,
                            double empty, Model* out, unsigned long long* fallback, double* sV) {
  int work[CMAX];
  int wl = tlen;
#pragma unroll
  for (int q = 0; q < CMAX; ++q) work[q] = q < tlen ? trial[q] : 0;
  while (wl > 0) {
    double coef[CMAX];
    double data, total;
    if (constrain) {
      int base = cand[work[0]];
      if (wl > 1) {
        int cols[CMAX];
        double ct[CMAX];
#pragma unroll
        for (int q = 0; q < CMAX; ++q) cols[q] = (q + 1 < wl) ? cand[work[q + 1]] : 0;
        ls_solve(L, X, k, cols, wl - 1, base, lam, ct, &data, &total, fallback, sV);
        double ssum = 0.0;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q < wl - 1) ssum += ct[q];
        coef[0] = 1.0 - ssum;
#pragma unroll
        for (int q = 1; q < CMAX; ++q) coef[q] = (q < wl) ? ct[q - 1] : 0.0;
      } else {
        double r = 0.0;
        if (L.lane < L.rf) r = L.sw * (L.y - cval(X, k, base, L.f));
        data = wsum(r * r);
        total = data;
        coef[0] = 1.0;
      }
    } else {
      int cols[CMAX];
#pragma unroll
      for (int q = 0; q < CMAX; ++q) cols[q] = q < wl ? cand[work[q]] : 0;
      ls_solve(L, X, k, cols, wl, -1, lam, coef, &data, &total, fallback, sV);
    }
    // coef.min(initial=0.0) >= 0
    double cmin = 0.0;
    int amin = 0;
    bool has_nan = false;
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      if (q < wl) {
        if (coef[q] != coef[q]) has_nan = true;
        if (coef[q] < cmin) {
          cmin = coef[q];
        }
      }
    }
    // np.argmin: first index of the minimum (NaN counts as the minimum)
    {
      double best = INFINITY;
      int bi = 0;
      bool found_nan = false;
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        if (q < wl && !found_nan) {
          if (coef[q] != coef[q]) {
            bi = q;
            found_nan = true;
          } else if (coef[q] < best) {
            best = coef[q];
            bi = q;
          }
        }
      }
      amin = bi;
    }
    bool ok = !has_nan && cmin >= 0.0;
    if (!nonneg || ok) {
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        out->pos[q] = work[q];
        out->coef[q] = q < wl ? coef[q] : 0.0;
      }
      out->len = wl;
      out->data = data;
      out->total = total;
      return;
    }
    if (wl == 1) {  // inert single-point row
      out->pos[0] = work[0];
      out->coef[0] = 0.0;
      out->len = 1;
      out->data = empty;
      out->total = empty;
      return;
    }
    // work.pop(argmin)
#pragma unroll
    for (int q = 0; q < CMAX - 1; ++q)
      if (q >= amin) work[q] = work[q + 1];
    --wl;
  }
  out->len = 0;
  out->data = empty;
  out->total = empty;
}

// insert x into the sorted unique list s (length *len) if absent
__device__ __forceinline__ bool sorted_insert(int* s, int* len, int x, int cap) {
  int lo = 0, hi = *len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  if (lo < *len && s[lo] == x) return true;
  if (*len >= cap) return false;
  for (int q = *len; q > lo; --q) s[q] = s[q - 1];
  s[lo] = x;
  ++*len;
  return true;
}

__global__ void __launch_bounds__(FIT_WARPS * 32)
fit_rows_kernel(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                const int32_t* __restrict__ crank, const double* __restrict__ X, int k,
                const double* __restrict__ w, const double* __restrict__ lam_dev, int caliber,
                int radius, double tol, int constrain, int nonneg, int32_t* __restrict__ out_cnt,
                int32_t* __restrict__ out_col, double* __restrict__ out_val,
                unsigned long long* __restrict__ status, const int32_t* __restrict__ list, int nlist,
                const unsigned int* __restrict__ nlist_dev) {
  BAMG_PDL_PROLOGUE();
  if (nlist_dev) nlist = (int)*nlist_dev;  // deferred points counted on device (no host read)
  __shared__ int s_cand[FIT_WARPS][MAXCAND];
  __shared__ double s_V[FIT_WARPS][CMAX * CMAX];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int* cand = s_cand[wib];
  double* sV = s_V[wib];
  const double lam = lam_dev[0];

  FitLane L;
  L.lane = lane;
  {
    bool fin = lane < k && isfinite(w[lane]);
    unsigned mask = __ballot_sync(0xffffffffu, fin);
    L.rf = __popc(mask);
    // lane l owns the l-th finite test
    int f = -1, seen = 0;
    for (int t = 0; t < k; ++t) {
      if (mask & (1u << t)) {
        if (seen == lane) f = t;
        ++seen;
      }
    }
    L.f = f < 0 ? 0 : f;
    L.sw = (lane < L.rf) ? sqrt(w[L.f]) : 0.0;
  }

  const int gw = blockIdx.x * FIT_WARPS + wib;
  const int nw = gridDim.x * FIT_WARPS;
  const int total = list ? nlist : n;
  for (int it = gw; it < total; it += nw) {
    const int i = list ? list[it] : it;
    int64_t obase = (int64_t)i * caliber;
    int ci = crank[i];
    if (ci >= 0) {  // coarse point: identity row
      if (lane == 0) {
        out_cnt[i] = 1;
        out_col[obase] = ci;
        out_val[obase] = 1.0;
      }
      continue;
    }
    // ---- candidates (sorted ascending point indices)
    int m = 0;
    const int rb = arp[i], re = arp[i + 1];
    if (radius == 1) {
      if (lane == 0) {
        for (int j = rb; j < re; ++j) {
          int p = acol[j];
          if (crank[p] >= 0) {
            if (m < MAXCAND) cand[m] = p;
            ++m;
          }
        }
      }
      m = __shfl_sync(0xffffffffu, m, 0);
    }
    if (m == 0 && re > rb) {  // radius-2 (escalation or configured)
      if (lane == 0) {
        // only coarse points (!= i) enter the sorted set: the reference's
        // unique(one + two-hop) filtered by (two != i) & coarse_mask
        int len = 0;
        bool ok = true;
        for (int j = rb; j < re && ok; ++j) {
          int p = acol[j];
          if (p != i && crank[p] >= 0) ok = sorted_insert(cand, &len, p, MAXCAND);
          for (int q = arp[p]; q < arp[p + 1] && ok; ++q) {
            int x = acol[q];
            if (x != i && crank[x] >= 0) ok = sorted_insert(cand, &len, x, MAXCAND);
          }
        }
        if (!ok) atomicOr(status + 1, 1ull);
        m = len;
      }
      m = __shfl_sync(0xffffffffu, m, 0);
    }
    __syncwarp();
    if (m > MAXCAND) {
      if (lane == 0) atomicOr(status + 1, 2ull);
      m = MAXCAND;
    }
    if (m == 0) {  // decoupled point: empty row (interp.py:277-281)
      if (lane == 0) out_cnt[i] = 0;
      continue;
    }
    if (lane < L.rf) L.y = cval(X, k, i, L.f);
    else L.y = 0.0;
    double yy = (lane < L.rf) ? w[L.f] * (L.y * L.y) : 0.0;
    const double empty = wsum(yy);

    // ---- greedy selection (fit_row)
    int sel[CMAX];
    int nsel = 0;
    double coefs[CMAX];
#pragma unroll
    for (int q = 0; q < CMAX; ++q) {
      sel[q] = 0;
      coefs[q] = 0.0;
    }
    double cur_total = empty;
    const int cap = caliber < m ? caliber : m;
    while (nsel < cap) {
      Model best;
      bool have = false;
      for (int j = 0; j < m; ++j) {
        bool in = false;
#pragma unroll
        for (int q = 0; q < CMAX; ++q)
          if (q < nsel && sel[q] == j) in = true;
        if (in) continue;
        int trial[CMAX];
#pragma unroll
        for (int q = 0; q < CMAX; ++q) trial[q] = q < nsel ? sel[q] : (q == nsel ? j : 0);
        Model md;
        solve_model(L, X, k, cand, trial, nsel + 1, constrain != 0, nonneg != 0, lam, empty, &md,
                    status, sV);
        if (nsel > 0 && md.len > 0) {
          double amax = 0.0;
          bool nan = false;
#pragma unroll
          for (int q = 0; q < CMAX; ++q)
            if (q < md.len) {
              if (md.coef[q] != md.coef[q]) nan = true;
              amax = fmax(amax, fabs(md.coef[q]));
            }
          if (!nan && amax > 10.0) continue;  // COEF_CAP veto
        }
        if (!have || md.total < best.total) {
          best = md;
          have = true;
        }
      }
      if (!have) break;
      if (nsel > 0) {
        if (cur_total <= 0.0 || (cur_total - best.total) < tol * cur_total) break;
      }
      if (best.len <= nsel) break;
#pragma unroll
      for (int q = 0; q < CMAX; ++q) {
        sel[q] = best.pos[q];
        coefs[q] = best.coef[q];
      }
      nsel = best.len;
      cur_total = best.total;
      if (cur_total <= 1e-30) break;
    }
    if (nsel == 0) {
      sel[0] = 0;
      coefs[0] = constrain ? 1.0 : 0.0;
      nsel = 1;
    }
    if (lane == 0) {
      out_cnt[i] = nsel;
      for (int q = 0; q < nsel; ++q) {
        out_col[obase + q] = crank[cand[sel[q]]];
        out_val[obase + q] = coefs[q];
      }
    }
    __syncwarp();
  }
}


// ===================================================================
// Thread-per-point variant (the production path).  Same greedy and decision
// rules; each trial model is solved from its ridge normal equations
// (A^T A + lambda^2 I) c = A^T b by a register Cholesky, then corrected by two
// steps of iterative refinement whose residuals are formed from the original
// rows (corrected semi-normal equations: forward error ~ eps * cond(A), the
// QR-level accuracy, since eps * cond(A)^2 << 1 for every ridge-regularised
// fit in scope).  Misfits are summed directly from the residual rows, never
// from the expanded quadratic form.  Points the thread path cannot take
// (more than TMAXC candidates, k > TKMAX, lambda == 0, or a Cholesky factor
// failing qr_solve_ls's rank test) are appended to a list that the warp-QR
// kernel above finishes -- so the reference's pseudo-inverse branch keeps its
// exact semantics.
constexpr int TMAXC = 16;  // candidates per point on the thread path
constexpr int TKMAX = 32;
constexpr int TCAL = 4;    // calibers up to 4 on the thread path
#ifndef BAMG_FIT_RECIP
#define BAMG_FIT_RECIP 1
#endif

struct TModel {
  int pos[TCAL];
  int len;
  double coef[TCAL];
  double data, total;
};

// KM <= 16: "exact" mode, KM == k at compile time -- every loop over the tests
// is unrolled, test t lives in registers, and infinite-weight tests are
// masked by sw = 0 (their rows add exact zeros).  KM == 32: generic mode for
// any k, finite tests compacted into f[] (local memory).
template <int KM>
struct TPoint {
  static constexpr bool EXACT = KM <= 16;
  // exact mode with whole 32-byte row segments: the columns are read four
  // tests at a time with 256-bit loads (the launcher checks X's alignment)
  static constexpr bool VEC = EXACT && KM % 4 == 0;
  const double* X;
  int k;
  int nf;                        // finite tests (generic mode)
  int f[EXACT ? 1 : KM];         // their indices (generic mode)
  double y[KM];                  // fine values
  double sw[KM];                 // sqrt weights (0 for masked tests)
  double lam;
  __device__ __forceinline__ double yv(int t) const { return y[t]; }
  __device__ __forceinline__ double swv(int t) const { return sw[t]; }
  __device__ __forceinline__ int ntest() const { return EXACT ? KM : nf; }
  __device__ __forceinline__ int stride() const { return EXACT ? KM : k; }
  __device__ __forceinline__ int test(int t) const {
    if constexpr (EXACT) return t;
    else return f[t];
  }
};

// column value a_{fq} = sw_f * (C[f, col] - C[f, base]) (base < 0: no shift)
template <int KM>
__device__ __forceinline__ double tcol(const TPoint<KM>& P, int t, int col, int base) {
  double c = __ldg(P.X + (int64_t)col * P.stride() + P.test(t));
  if (base >= 0) c -= __ldg(P.X + (int64_t)base * P.stride() + P.test(t));
  return P.swv(t) * c;
}

template <int KM>
__device__ __forceinline__ double ttarget(const TPoint<KM>& P, int t, int base) {
  double yv = P.yv(t);
  if (base >= 0) yv -= __ldg(P.X + (int64_t)base * P.stride() + P.test(t));
  return P.swv(t) * yv;
}

__device__ __forceinline__ void ldg_v4(const double* p, double* v) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// tests t0..t0+3 of every trial column and of the target, the same values
// tcol / ttarget give one scalar load at a time (VEC mode): av[q][u] =
// sw * (C[col_q] - C[base]), bv[u] = sw * (y - C[base]) at test t0 + u.
// One 256-bit load per row and chunk instead of four (or eight, with the
// base row re-read per column): the fit was bound by load-issue throttling.
template <int KM, int NC>
__device__ __forceinline__ void tchunk(const TPoint<KM>& P, const int* cols, int base, int t0, double (&av)[NC][4],
                                       double (&bv)[4]) {
  double xb[4] = {0.0, 0.0, 0.0, 0.0};
  if (base >= 0) ldg_v4(P.X + (int64_t)base * KM + t0, xb);
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double xc[4];
    ldg_v4(P.X + (int64_t)cols[q] * KM + t0, xc);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double c = xc[u];
      if (base >= 0) c -= xb[u];
      av[q][u] = P.swv(t0 + u) * c;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    double yv = P.yv(t0 + u);
    if (base >= 0) yv -= xb[u];
    bv[u] = P.swv(t0 + u) * yv;
  }
}

// ridge LS on NC columns (point indices cols[]); returns false when the
// Cholesky factor fails the rank test (caller defers the point).  NC is a
// compile-time constant so no guarded (issued but idle) lanes of the 4x4
// Gram / Cholesky / triangular loops execute for small trial models.
template <int KM, int NC>
__device__ __forceinline__ bool tls_solve_n(const TPoint<KM>& P, const int* cols, int base, double* coef,
                                            double* data, double* total) {
  constexpr int nc = NC;
  double G[NC][NC], h[NC];
#pragma unroll
  for (int p = 0; p < NC; ++p) {
    h[p] = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) G[p][q] = 0.0;
  }
  auto gram_add = [&](const double* a, double b) {
#pragma unroll
    for (int p = 0; p < NC; ++p) {
      h[p] += a[p] * b;
#pragma unroll
      for (int q = 0; q <= p; ++q) G[p][q] += a[p] * a[q];
    }
  };
  if constexpr (TPoint<KM>::VEC) {
#pragma unroll
    for (int t0 = 0; t0 < KM; t0 += 4) {
      double av[NC][4], bv[4];
      tchunk<KM, NC>(P, cols, base, t0, av, bv);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double a[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) a[q] = av[q][u];
        gram_add(a, bv[u]);
      }
    }
  } else {
    _Pragma("unroll") for (int t = 0; t < P.ntest(); ++t) {
      double a[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) a[q] = q < nc ? tcol(P, t, cols[q], base) : 0.0;
      gram_add(a, ttarget(P, t, base));
    }
  }
  const double l2 = P.lam * P.lam;
  // Cholesky G + lam^2 I = R^T R (lower L = R^T stored in G's lower triangle)
  double L[NC][NC];
#if BAMG_FIT_RECIP
  double rinv[NC];  // reciprocal pivots: one division per column
#define BAMG_PIVDIV(v, j) ((v) * rinv[j])
#else
#define BAMG_PIVDIV(v, j) ((v) / L[j][j])
#endif
  double rmax = 0.0, dmin = INFINITY;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    if (j >= nc) break;
    double d = G[j][j] + l2;
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (q < j) d -= L[j][q] * L[j][q];
    if (!(d > 0.0)) return false;
    double ljj = sqrt(d);
    L[j][j] = ljj;
#if BAMG_FIT_RECIP
    rinv[j] = 1.0 / ljj;
#endif
    dmin = fmin(dmin, ljj);
    rmax = fmax(rmax, ljj);
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if (i > j && i < nc) {
        double v = G[i][j];
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (q < j) v -= L[i][q] * L[j][q];
        L[i][j] = BAMG_PIVDIV(v, j);
        rmax = fmax(rmax, fabs(L[i][j]));
      }
    }
  }
  if (rmax == 0.0 || dmin < 1e-13 * rmax) return false;  // qr_solve_ls would take pinv
  auto chol_solve = [&](const double* rhs, double* x) {
    double z[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if (i < nc) {
        double v = rhs[i];
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (q < i) v -= L[i][q] * z[q];
        z[i] = BAMG_PIVDIV(v, i);
      }
    }
#pragma unroll
    for (int i = NC - 1; i >= 0; --i) {
      if (i < nc) {
        double v = z[i];
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (q > i && q < nc) v -= L[q][i] * x[q];
        x[i] = BAMG_PIVDIV(v, i);
      }
    }
  };
  double c[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) c[q] = 0.0;
  chol_solve(h, c);
  for (int refine = 0; refine < 2; ++refine) {
    double g[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) g[q] = q < nc ? -l2 * c[q] : 0.0;  // ridge rows: -lam * (lam c)
    auto resid_add = [&](const double* a, double r) {
#pragma unroll
      for (int q = 0; q < NC; ++q) r -= a[q] * c[q];
#pragma unroll
      for (int q = 0; q < NC; ++q) g[q] += a[q] * r;
    };
    if constexpr (TPoint<KM>::VEC) {
#pragma unroll
      for (int t0 = 0; t0 < KM; t0 += 4) {
        double av[NC][4], bv[4];
        tchunk<KM, NC>(P, cols, base, t0, av, bv);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double a[NC];
#pragma unroll
          for (int q = 0; q < NC; ++q) a[q] = av[q][u];
          resid_add(a, bv[u]);
        }
      }
    } else {
      _Pragma("unroll") for (int t = 0; t < P.ntest(); ++t) {
        double a[NC];
        double r = ttarget(P, t, base);
#pragma unroll
        for (int q = 0; q < NC; ++q) a[q] = q < nc ? tcol(P, t, cols[q], base) : 0.0;
        resid_add(a, r);
      }
    }
    double dlt[NC];
    chol_solve(g, dlt);
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (q < nc) c[q] += dlt[q];
  }
  double mis = 0.0;
  if constexpr (TPoint<KM>::VEC) {
#pragma unroll
    for (int t0 = 0; t0 < KM; t0 += 4) {
      double av[NC][4], bv[4];
      tchunk<KM, NC>(P, cols, base, t0, av, bv);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < NC; ++q) r += av[q][u] * c[q];
        r -= bv[u];
        mis += r * r;
      }
    }
  } else {
    _Pragma("unroll") for (int t = 0; t < P.ntest(); ++t) {
      double r = 0.0;
#pragma unroll
      for (int q = 0; q < NC; ++q)
        if (q < nc) r += tcol(P, t, cols[q], base) * c[q];
      r -= ttarget(P, t, base);
      mis += r * r;
    }
  }
  double cc = 0.0;
#pragma unroll
  for (int q = 0; q < NC; ++q)
    if (q < nc) {
      coef[q] = c[q];
      cc += c[q] * c[q];
    }
  *data = mis;
  *total = mis + l2 * cc;
  return true;
}
#undef BAMG_PIVDIV

template <int KM>
__device__ __forceinline__ bool tls_solve(const TPoint<KM>& P, const int* cols, int nc, int base, double* coef,
                                          double* data, double* total) {
  static_assert(TCAL == 4, "tls_solve dispatch covers calibers 1..4");
  switch (nc) {
    case 1: return tls_solve_n<KM, 1>(P, cols, base, coef, data, total);
    case 2: return tls_solve_n<KM, 2>(P, cols, base, coef, data, total);
    case 3: return tls_solve_n<KM, 3>(P, cols, base, coef, data, total);
    default: return tls_solve_n<KM, 4>(P, cols, base, coef, data, total);
  }
}

// solve_model (interp.py:176-199) on the thread path; false = defer point
template <int KM>
__device__ bool tsolve_model(const TPoint<KM>& P, const int* trial, int tlen, bool constrain, bool nonneg,
                             double empty, TModel* out) {
  int work[TCAL];
  int wl = tlen;
#pragma unroll
  for (int q = 0; q < TCAL; ++q) work[q] = q < tlen ? trial[q] : 0;
  while (wl > 0) {
    double coef[TCAL];
    double data, total;
    if (constrain) {
      int base = work[0];
      if (wl > 1) {
        int cols[TCAL];
        double ct[TCAL];
#pragma unroll
        for (int q = 0; q < TCAL; ++q) cols[q] = (q + 1 < wl) ? work[q + 1] : 0;
        if (!tls_solve(P, cols, wl - 1, base, ct, &data, &total)) return false;
        double ssum = 0.0;
#pragma unroll
        for (int q = 0; q < TCAL; ++q)
          if (q < wl - 1) ssum += ct[q];
        coef[0] = 1.0 - ssum;
#pragma unroll
        for (int q = 1; q < TCAL; ++q) coef[q] = (q < wl) ? ct[q - 1] : 0.0;
      } else {
        double mis = 0.0;
        if constexpr (TPoint<KM>::VEC) {
#pragma unroll
          for (int t0 = 0; t0 < KM; t0 += 4) {
            double xb[4];
            ldg_v4(P.X + (int64_t)base * KM + t0, xb);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              double r = P.swv(t0 + u) * (P.yv(t0 + u) - xb[u]);
              mis += r * r;
            }
          }
        } else {
          _Pragma("unroll") for (int t = 0; t < P.ntest(); ++t) {
            double r = ttarget(P, t, base);
            mis += r * r;
          }
        }
        data = total = mis;
        coef[0] = 1.0;
      }
    } else {
      int cols[TCAL];
#pragma unroll
      for (int q = 0; q < TCAL; ++q) cols[q] = q < wl ? work[q] : 0;
      if (!tls_solve(P, cols, wl, -1, coef, &data, &total)) return false;
    }
    bool has_nan = false;
    double cmin = 0.0;
    int amin = 0;
    double best = INFINITY;
    bool found_nan = false;
#pragma unroll
    for (int q = 0; q < TCAL; ++q) {
      if (q < wl) {
        double v = coef[q];
        if (v != v) {
          has_nan = true;
          if (!found_nan) {
            amin = q;
            found_nan = true;
          }
        } else {
          cmin = fmin(cmin, v);
          if (!found_nan && v < best) {
            best = v;
            amin = q;
          }
        }
      }
    }
    if (!nonneg || (!has_nan && cmin >= 0.0)) {
#pragma unroll
      for (int q = 0; q < TCAL; ++q) {
        out->pos[q] = work[q];
        out->coef[q] = q < wl ? coef[q] : 0.0;
      }
      out->len = wl;
      out->data = data;
      out->total = total;
      return true;
    }
    if (wl == 1) {
      out->pos[0] = work[0];
      out->coef[0] = 0.0;
      out->len = 1;
      out->data = empty;
      out->total = empty;
      return true;
    }
#pragma unroll
    for (int q = 0; q < TCAL - 1; ++q)
      if (q >= amin) work[q] = work[q + 1];
    --wl;
  }
  out->len = 0;
  out->data = empty;
  out->total = empty;
  return true;
}

// coarse points: identity rows; fine points: appended to the work list
__global__ void fit_prepare_kernel(int n, const int32_t* __restrict__ crank, int caliber, int32_t* __restrict__ out_cnt,
                                   int32_t* __restrict__ out_col, double* __restrict__ out_val,
                                   int32_t* __restrict__ list, unsigned int* __restrict__ nlist, int lo, int hi) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i < lo || i >= hi) {  // another rank's row (bamg_fit_set_row_range)
    out_cnt[i] = 0;
    return;
  }
  int ci = crank[i];
  if (ci >= 0) {
    int64_t o = (int64_t)i * caliber;
    out_cnt[i] = 1;
    out_col[o] = ci;
    out_val[o] = 1.0;
  } else {
    list[atomicAdd(nlist, 1u)] = i;
  }
}

// Candidate pass of the thread path: coarse radius-1 neighbours (adjacency
// rows are sorted), escalating to the sorted unique radius-2 union when there
// are none (interp.py:241-249, 274-276).  Writes the list to cbuf[t][TMAXC]
// and counts the points per candidate count, so the fit kernel can run warps
// of equal-sized problems (the greedy loop's trip counts follow m).  Points
// with no candidates get an empty row here; overflowing ones go to the warp
// path.
__global__ void __launch_bounds__(256)
fit_cands_kernel(const int32_t* __restrict__ list, const unsigned int* __restrict__ nlist,
                 const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                 const int32_t* __restrict__ crank, int radius, int32_t* __restrict__ mcnt,
                 int32_t* __restrict__ cbuf, unsigned int* __restrict__ hist, int32_t* __restrict__ out_cnt,
                 int32_t* __restrict__ defer, unsigned int* __restrict__ ndefer) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned int sh[TMAXC + 1];
  if (threadIdx.x <= TMAXC) sh[threadIdx.x] = 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (int)*nlist) {
    const int i = list[t];
    int32_t* cand = cbuf + (int64_t)t * TMAXC;
    int m = 0;
    bool ok = true;
    const int rb = arp[i], re = arp[i + 1];
    if (radius == 1) {
      for (int j = rb; j < re; ++j) {
        int p = acol[j];
        if (crank[p] >= 0) {
          if (m < TMAXC) cand[m] = p;
          ++m;
        }
      }
      if (m > TMAXC) ok = false;
    }
    if (ok && m == 0 && re > rb) {
      int len = 0;
      for (int j = rb; j < re && ok; ++j) {
        int nb = acol[j];
        for (int side = 0; side < 2 && ok; ++side) {
          int qb = side == 0 ? j : arp[nb];
          int qe = side == 0 ? j + 1 : arp[nb + 1];
          for (int q = qb; q < qe; ++q) {
            int x = acol[q];
            if (x == i || crank[x] < 0) continue;
            int pos = 0;
            while (pos < len && cand[pos] < x) ++pos;
            if (pos < len && cand[pos] == x) continue;
            if (len >= TMAXC) {
              ok = false;
              break;
            }
            for (int u = len; u > pos; --u) cand[u] = cand[u - 1];
            cand[pos] = x;
            ++len;
          }
        }
      }
      m = len;
    }
    if (!ok) {
      defer[atomicAdd(ndefer, 1u)] = i;
      mcnt[t] = -1;
    } else if (m == 0) {
      out_cnt[i] = 0;
      mcnt[t] = -1;
    } else {
      mcnt[t] = m;
      atomicAdd(&sh[m], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x <= TMAXC && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

// exclusive scan of the candidate-count histogram -> bucket cursors
__global__ void fit_bucket_scan_kernel(unsigned int* __restrict__ hist, unsigned int* __restrict__ nsorted) {
  BAMG_PDL_PROLOGUE();
  if (threadIdx.x != 0) return;
  unsigned int acc = 0;
  for (int b = 0; b <= TMAXC; ++b) {
    unsigned int c = hist[b];
    hist[b] = acc;
    acc += c;
  }
  *nsorted = acc;
}

// bucket the points by candidate count (order inside a bucket is immaterial:
// every point's row is computed independently)
__global__ void __launch_bounds__(256)
fit_bucket_scatter_kernel(const int32_t* __restrict__ mcnt, const unsigned int* __restrict__ nlist,
                          unsigned int* __restrict__ cursor, int32_t* __restrict__ order) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned int sh[TMAXC + 1], base[TMAXC + 1];
  if (threadIdx.x <= TMAXC) sh[threadIdx.x] = 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = t < (int)*nlist ? mcnt[t] : -1;
  unsigned int r = m > 0 ? atomicAdd(&sh[m], 1u) : 0u;
  __syncthreads();
  if (threadIdx.x <= TMAXC) base[threadIdx.x] = sh[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], sh[threadIdx.x]) : 0u;
  __syncthreads();
  if (m > 0) order[base[m] + r] = t;
}

#ifndef BAMG_FIT_MINBLOCKS
#define BAMG_FIT_MINBLOCKS 2
#endif
constexpr int TFIT_THREADS = 128;

// Greedy selection of one fine point per thread over its m candidates.  The
// candidate list sits in shared memory (one column per thread); the selection
// and the trial models carry candidate point ids, so no per-thread array is
// indexed dynamically.
template <int KM>
__global__ void __launch_bounds__(TFIT_THREADS, BAMG_FIT_MINBLOCKS)
fit_rows_thread_kernel(const int32_t* __restrict__ order, const unsigned int* __restrict__ nsorted,
                       const int32_t* __restrict__ list, const int32_t* __restrict__ mcnt,
                       const int32_t* __restrict__ cbuf, const int32_t* __restrict__ crank,
                       const double* __restrict__ X, int k, const double* __restrict__ w,
                       const double* __restrict__ lam_dev, int caliber, double tol, int constrain, int nonneg,
                       int32_t* __restrict__ out_cnt, int32_t* __restrict__ out_col, double* __restrict__ out_val,
                       int32_t* __restrict__ defer, unsigned int* __restrict__ ndefer) {
  BAMG_PDL_PROLOGUE();
  __shared__ int s_cand[TMAXC][TFIT_THREADS];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int)*nsorted) return;
  const int s = order[t];
  const int i = list[s];
  const int m = mcnt[s];
  const int64_t obase = (int64_t)i * caliber;
  {
    const int4* src = reinterpret_cast<const int4*>(cbuf + (int64_t)s * TMAXC);
#pragma unroll
    for (int v = 0; v < TMAXC / 4; ++v) {
      if (4 * v < m) {
        int4 c4 = src[v];
        s_cand[4 * v][threadIdx.x] = c4.x;
        s_cand[4 * v + 1][threadIdx.x] = c4.y;
        s_cand[4 * v + 2][threadIdx.x] = c4.z;
        s_cand[4 * v + 3][threadIdx.x] = c4.w;
      }
    }
  }
  TPoint<KM> P;
  P.X = X;
  P.k = k;
  P.lam = lam_dev[0];
  if (!(P.lam > 0.0)) {
    defer[atomicAdd(ndefer, 1u)] = i;
    return;
  }
  double empty = 0.0;
  if constexpr (TPoint<KM>::EXACT) {
#pragma unroll
    for (int tt = 0; tt < KM; ++tt) {
      double wt = w[tt];
      double yv = X[(int64_t)i * KM + tt];
      bool fin = isfinite(wt);
      P.y[tt] = yv;
      P.sw[tt] = fin ? sqrt(wt) : 0.0;
      if (fin) empty += wt * (yv * yv);
    }
    P.nf = KM;
  } else {
    int nf = 0;
    for (int tt = 0; tt < k; ++tt) {
      double wt = w[tt];
      if (!isfinite(wt)) continue;
      double yv = X[(int64_t)i * k + tt];
      P.f[nf] = tt;
      P.y[nf] = yv;
      P.sw[nf] = sqrt(wt);
      empty += wt * (yv * yv);
      ++nf;
    }
    P.nf = nf;
  }

  int sel[TCAL];
  double coefs[TCAL];
  int nsel = 0;
#pragma unroll
  for (int q = 0; q < TCAL; ++q) {
    sel[q] = 0;
    coefs[q] = 0.0;
  }
  double cur_total = empty;
  const int cap = caliber < m ? caliber : m;
  while (nsel < cap) {
    TModel best;
    bool have = false;
    for (int j = 0; j < m; ++j) {
      const int cj = s_cand[j][threadIdx.x];
      bool in = false;
#pragma unroll
      for (int q = 0; q < TCAL; ++q)
        if (q < nsel && sel[q] == cj) in = true;
      if (in) continue;
      int trial[TCAL];
#pragma unroll
      for (int q = 0; q < TCAL; ++q) trial[q] = q < nsel ? sel[q] : (q == nsel ? cj : 0);
      TModel md;
      if (!tsolve_model(P, trial, nsel + 1, constrain != 0, nonneg != 0, empty, &md)) {
        defer[atomicAdd(ndefer, 1u)] = i;
        return;
      }
      if (nsel > 0 && md.len > 0) {
        double amax = 0.0;
        bool nan = false;
#pragma unroll
        for (int q = 0; q < TCAL; ++q)
          if (q < md.len) {
            if (md.coef[q] != md.coef[q]) nan = true;
            amax = fmax(amax, fabs(md.coef[q]));
          }
        if (!nan && amax > 10.0) continue;
      }
      if (!have || md.total < best.total) {
        best = md;
        have = true;
      }
    }
    if (!have) break;
    if (nsel > 0 && (cur_total <= 0.0 || (cur_total - best.total) < tol * cur_total)) break;
    if (best.len <= nsel) break;
#pragma unroll
    for (int q = 0; q < TCAL; ++q) {
      sel[q] = best.pos[q];
      coefs[q] = best.coef[q];
    }
    nsel = best.len;
    cur_total = best.total;
    if (cur_total <= 1e-30) break;
  }
  if (nsel == 0) {
    sel[0] = s_cand[0][threadIdx.x];
    coefs[0] = constrain ? 1.0 : 0.0;
    nsel = 1;
  }
  out_cnt[i] = nsel;
#pragma unroll
  for (int q = 0; q < TCAL; ++q)
    if (q < nsel) {
      out_col[obase + q] = crank[sel[q]];
      out_val[obase + q] = coefs[q];
    }
}

// ridge = 0.1 * sqrt(mean_i (sqrt(sum_f w_f x_if^2))^2)  (interp.py:266-268)
__global__ void level_scale_partial(const double* __restrict__ X, int64_t n, int k, const double* __restrict__ w,
                                    double* __restrict__ partial) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[RED_THREADS / 32];
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  double acc = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < k; ++c) {
      double wc = w[c];
      if (isfinite(wc)) {
        double x = X[r * k + c];
        s += wc * (x * x);
      }
    }
    double ps = sqrt(s);
    acc += ps * ps;
  }
  double v = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < RED_THREADS / 32; ++q) t += sh[q];
    partial[blockIdx.x] = t;
  }
}

__global__ void level_scale_final(const double* __restrict__ partial, int nb, int64_t n, double* lam) {
  BAMG_PDL_PROLOGUE();
  int lane = threadIdx.x;
  double v = 0.0;
  for (int b = lane; b < nb; b += 32) v += partial[b];
  v = warp_sum(v);
  if (lane == 0) lam[0] = 0.1 * sqrt(v / (double)n);
}

// BAMG_FIT_WARP=1 forces the warp-QR path for every point (parity testing)
static bool force_warp_path() {
  const char* e = getenv("BAMG_FIT_WARP");
  return e && e[0] == '1';
}

// LS fit of every fine point.  status (device, 4 words): [0] points that took
// the reference's pseudo-inverse branch, [1] candidate-list overflows,
// [2] points deferred from the thread path to the warp path.  Nothing is read
// back here: the deferred points are walked grid-stride over their device
// count, so the caller reads status once (with its own results).
static int fit_rows_launch(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank, const double* X,
                           const double* w, int64_t n, int k, int caliber, int radius, double improvement_tol,
                           int constrain, int nonnegative, double ridge_override, int32_t* out_cnt,
                           int32_t* out_col, double* out_val, unsigned long long* status) {
  BAMG_REQUIRE(ctx, caliber >= 1 && caliber <= CMAX, "caliber must lie in [1, 8]");
  BAMG_REQUIRE(ctx, k >= 1 && k + caliber <= 32, "need k + caliber <= 32 (one LS row per lane)");
  BAMG_REQUIRE(ctx, radius == 1 || radius == 2, "radius must be 1 or 2");
  BAMG_REQUIRE(ctx, adj && adj->nrows == n, "adjacency size mismatch");
  double *partial, *lam;
  BAMG_TRY(arena_get(ctx, RED_BLOCKS, &partial));
  BAMG_TRY(arena_get(ctx, 1, &lam));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(status, 0, 4 * sizeof(unsigned long long), ctx->stream));
  if (ridge_override >= 0.0) {
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(lam, &ridge_override, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  } else {
    const int nbl = red_blocks_for(n);
    BAMG_LAUNCH(ctx, level_scale_partial, nbl, RED_THREADS, 0, X, n, k, w, partial);
    BAMG_LAUNCH(ctx, level_scale_final, 1, 32, 0, partial, nbl, n, lam);
  }
  // algorithmic bytes: test vectors of every point + adjacency + rank map + the row output
  double fbytes = 8.0 * n * k + 4.0 * (n + 1) + 4.0 * adj->nnz + 4.0 * n + 16.0 * n * caliber;
  int32_t* defer;
  unsigned int* ndefer = reinterpret_cast<unsigned int*>(status + 2);  // low half of status[2]
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &defer));
  if (k <= TKMAX && caliber <= TCAL && !force_warp_path()) {
    int32_t* flist;
    unsigned int* nfl;
    BAMG_TRY(arena_get(ctx, (size_t)n + 1, &flist));
    BAMG_TRY(arena_get(ctx, 1, &nfl));
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(nfl, 0, sizeof(unsigned int), ctx->stream));
    const int row_lo = ctx->fit_lo >= 0 ? (int)(ctx->fit_lo < n ? ctx->fit_lo : n) : 0;
    const int row_hi = ctx->fit_lo >= 0 ? (int)(ctx->fit_hi < n ? ctx->fit_hi : n) : (int)n;
    BAMG_LAUNCH(ctx, fit_prepare_kernel, grid_for(n, 256), 256, 0, (int)n, coarse_rank, caliber, out_cnt, out_col,
                out_val, flist, nfl, row_lo, row_hi);
    int32_t *mcnt, *cbuf, *order;
    unsigned int *hist, *nsorted;
    BAMG_TRY(arena_get(ctx, (size_t)n + 1, &mcnt));
    BAMG_TRY(arena_get(ctx, (size_t)n * TMAXC + 4, &cbuf));
    BAMG_TRY(arena_get(ctx, (size_t)n + 1, &order));
    BAMG_TRY(arena_get(ctx, TMAXC + 2, &hist));
    nsorted = hist + TMAXC + 1;
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(hist, 0, (TMAXC + 2) * sizeof(unsigned int), ctx->stream));
    BAMG_LAUNCH(ctx, fit_cands_kernel, grid_for(n, 256), 256, 0, flist, nfl, adj->rowptr, adj->col, coarse_rank,
                radius, mcnt, cbuf, hist, out_cnt, defer, ndefer);
    BAMG_LAUNCH(ctx, fit_bucket_scan_kernel, 1, 32, 0, hist, nsorted);
    BAMG_LAUNCH(ctx, fit_bucket_scatter_kernel, grid_for(n, 256), 256, 0, mcnt, nfl, hist, order);
    // the VEC specialisations read X in 32-byte segments
    const bool x_aligned = (reinterpret_cast<uintptr_t>(X) & 31) == 0;
#define BAMG_FIT_EXACT(KK)                                                                                       \
  if (k == KK && (x_aligned || !TPoint<KK>::VEC)) {                                                                                                 \
    BAMG_LAUNCH_FAM(ctx, FAM_FIT, fbytes, fit_rows_thread_kernel<KK>, grid_for(n, TFIT_THREADS), TFIT_THREADS, 0,  \
                    order, nsorted, flist, mcnt, cbuf, coarse_rank, X, k, w, lam, caliber, improvement_tol,        \
                    constrain, nonnegative, out_cnt, out_col, out_val, defer, ndefer);                             \
  } else
    BAMG_FIT_EXACT(8) BAMG_FIT_EXACT(10) BAMG_FIT_EXACT(12) BAMG_FIT_EXACT(16) {
      BAMG_LAUNCH_FAM(ctx, FAM_FIT, fbytes, fit_rows_thread_kernel<TKMAX>, grid_for(n, TFIT_THREADS), TFIT_THREADS,
                      0, order, nsorted, flist, mcnt, cbuf, coarse_rank, X, k, w, lam, caliber, improvement_tol,
                      constrain, nonnegative, out_cnt, out_col, out_val, defer, ndefer);
    }
#undef BAMG_FIT_EXACT
    // deferred points (device count): a fixed grid of warps strides over them
    const int blocks = ctx->num_sms * 4;
    BAMG_LAUNCH_FAM(ctx, FAM_FIT, 0.0, fit_rows_kernel, blocks, FIT_WARPS * 32, 0, (int)n, adj->rowptr, adj->col,
                    coarse_rank, X, k, w, lam, caliber, radius, improvement_tol, constrain, nonnegative, out_cnt,
                    out_col, out_val, status, (const int32_t*)defer, 0, (const unsigned int*)ndefer);
  } else if (n > 0) {
    int64_t blocks = (n + FIT_WARPS - 1) / FIT_WARPS;
    int64_t maxb = (int64_t)ctx->num_sms * 64;
    if (blocks > maxb) blocks = maxb;
    BAMG_LAUNCH_FAM(ctx, FAM_FIT, fbytes, fit_rows_kernel, (int)blocks, FIT_WARPS * 32, 0, (int)n, adj->rowptr,
                    adj->col, coarse_rank, X, k, w, lam, caliber, radius, improvement_tol, constrain, nonnegative,
                    out_cnt, out_col, out_val, status, (const int32_t*)nullptr, (int)n, (const unsigned int*)nullptr);
  }
  return 0;
}

static int fit_status_check(bamg_ctx* ctx, const int64_t* st, int64_t* status_host) {
  if (status_host) {
    status_host[0] = st[0];
    status_host[1] = st[2] & 0xffffffffll;
  }
  BAMG_REQUIRE(ctx, st[1] == 0, "candidate list overflow (more than 256 coarse candidates for one point)");
  return 0;
}

extern "C" int bamg_fit_set_row_range(bamg_ctx* ctx, int64_t row_lo, int64_t row_hi) {
  if (row_lo < 0) {
    ctx->fit_lo = ctx->fit_hi = -1;
    return 0;
  }
  BAMG_REQUIRE(ctx, row_hi >= row_lo, "row range must be ordered");
  ctx->fit_lo = row_lo;
  ctx->fit_hi = row_hi;
  return 0;
}

extern "C" int bamg_fit_rows(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank, const double* X,
                             const double* w, int64_t n, int k, int caliber, int radius, double improvement_tol,
                             int constrain, int nonnegative, double ridge_override, int32_t* out_cnt,
                             int32_t* out_col, double* out_val, int64_t* status_host) {
  ctx->arena.reset();
  if (status_host) status_host[0] = status_host[1] = 0;
  unsigned long long* status;
  BAMG_TRY(arena_get(ctx, 4, &status));
  BAMG_TRY(fit_rows_launch(ctx, adj, coarse_rank, X, w, n, k, caliber, radius, improvement_tol, constrain,
                           nonnegative, ridge_override, out_cnt, out_col, out_val, status));
  int64_t st[3];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(status), 3, st));
  return fit_status_check(ctx, st, status_host);
}

__global__ void rows_count_kernel(const int32_t* __restrict__ cnt, const double* __restrict__ val, int64_t n,
                                  int stride, int32_t* __restrict__ out);

// Per-context state of asynchronous fits (bamg_fit_rows_csr_slot): status
// words (4 slots x 4 words, read back together by bamg_fit_rows_wait), one
// side stream, fork / join event and scratch arena per slot.  Every slot call
// records its OWN fork event on the main stream, so everything enqueued on
// the main stream before the call (its inputs included) is ordered before the
// slot's launches on its side stream; the fits of a batch (P and W of a
// level) then overlap -- the coarse levels' fits are one serial greedy chain
// per thread (35-60 us whatever the size) and run side by side at the cost
// of one.  The joins are deferred to bamg_fit_rows_wait, which orders the
// main stream after every pending slot before reading the status words.
// Slots never touch the context arena (each has its own), so main-stream work
// between slot calls -- including entry points that reset the arena -- is
// safe; what must not happen before bamg_fit_rows_wait is main-stream work
// that READS a pending slot's outputs.  While the stream is being captured
// into a graph the slots run on the main stream.
constexpr int FIT_SLOTS = 4;
struct FitSlots {
  unsigned long long* status = nullptr;
  cudaStream_t side[FIT_SLOTS] = {};
  cudaEvent_t fork[FIT_SLOTS] = {}, join[FIT_SLOTS] = {};
  Arena arena[FIT_SLOTS];
  bool pending[FIT_SLOTS] = {};
};

static FitSlots* fit_slots(bamg_ctx* ctx) {
  if (ctx->fit_slots) return ctx->fit_slots;
  FitSlots* fs = new FitSlots();
  bool ok = cudaMalloc(&fs->status, sizeof(unsigned long long) * 4 * FIT_SLOTS) == cudaSuccess;
  for (int s = 0; s < FIT_SLOTS && ok; ++s)
    ok = cudaStreamCreateWithFlags(&fs->side[s], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fs->fork[s], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&fs->join[s], cudaEventDisableTiming) == cudaSuccess;
  ctx->fit_slots = fs;  // released (also when partially built) by fit_slots_release
  return ok ? fs : nullptr;
}

void fit_slots_release(bamg_ctx* ctx) {
  FitSlots* fs = ctx->fit_slots;
  if (!fs) return;
  for (int s = 0; s < FIT_SLOTS; ++s) {
    if (fs->side[s]) cudaStreamSynchronize(fs->side[s]);
    fs->arena[s].release();
    if (fs->side[s]) cudaStreamDestroy(fs->side[s]);
    if (fs->fork[s]) cudaEventDestroy(fs->fork[s]);
    if (fs->join[s]) cudaEventDestroy(fs->join[s]);
  }
  if (fs->status) cudaFree(fs->status);
  delete fs;
  ctx->fit_slots = nullptr;
}

static unsigned long long* fit_slot_status(bamg_ctx* ctx) {
  FitSlots* fs = fit_slots(ctx);
  return fs ? fs->status : nullptr;
}

static int fit_rows_csr_launch(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank, const double* X,
                               const double* w, int64_t n, int k, int caliber, int radius, double improvement_tol,
                               int constrain, int nonnegative, double ridge_override, int32_t* out_cnt,
                               int32_t* out_col, double* out_val, int32_t* rowptr, unsigned long long* status) {
  BAMG_TRY(fit_rows_launch(ctx, adj, coarse_rank, X, w, n, k, caliber, radius, improvement_tol, constrain,
                           nonnegative, ridge_override, out_cnt, out_col, out_val, status));
  int32_t* c;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &c));
  BAMG_LAUNCH(ctx, rows_count_kernel, grid_for(n, 256), 256, 0, out_cnt, out_val, n, caliber, c);
  return scan_i32_dev(ctx, c, rowptr, n, reinterpret_cast<int64_t*>(status + 3));
}

// Asynchronous fit + row count + scan into slot `slot` (0..3); the status
// [pinv-branch points, overflows, deferred, nnz] of every listed slot comes
// back with ONE synchronisation in bamg_fit_rows_wait (P and W of a level).
extern "C" int bamg_fit_rows_csr_slot(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank,
                                      const double* X, const double* w, int64_t n, int k, int caliber, int radius,
                                      double improvement_tol, int constrain, int nonnegative, double ridge_override,
                                      int32_t* out_cnt, int32_t* out_col, double* out_val, int32_t* rowptr,
                                      int slot) {
  BAMG_REQUIRE(ctx, slot >= 0 && slot < FIT_SLOTS, "slot must lie in [0, 4)");
  FitSlots* fs = fit_slots(ctx);
  BAMG_REQUIRE(ctx, fs != nullptr, "fit slot state allocation failed");
  unsigned long long* st = fs->status + 4 * slot;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  BAMG_CHECK_CUDA(ctx, cudaStreamIsCapturing(ctx->stream, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  cudaStream_t main = ctx->stream;
  const bool prof = (ctx->prof.mask >> FAM_FIT) & 1u;
  bool first_of_batch = true;
  for (int s = 0; s < FIT_SLOTS; ++s) first_of_batch = first_of_batch && !fs->pending[s];
  if (prof && !capturing && first_of_batch)  // one event pair per batch (closed in bamg_fit_rows_wait)
    cudaEventRecord(prof_event(ctx, FAM_FIT), main);
  Arena saved;
  std::swap(saved, ctx->arena);  // the slot's scratch comes from its own arena
  std::swap(ctx->arena, fs->arena[slot]);
  if (!capturing) {
    // the slot's previous use of its arena ran on its side stream: stream-ordered
    ctx->arena.reset();
    if (cudaEventRecord(fs->fork[slot], main) != cudaSuccess ||
        cudaStreamWaitEvent(fs->side[slot], fs->fork[slot], 0) != cudaSuccess) {
      std::swap(ctx->arena, fs->arena[slot]);
      std::swap(saved, ctx->arena);
      ctx->err = "fit slot fork failed";
      return -1;
    }
    ctx->stream = fs->side[slot];
  } else {
    cudaStreamSynchronize(fs->side[slot]);  // no capture-time reset may overlap a side-stream user
    ctx->arena.reset();
  }
  ctx->prof.batched[FAM_FIT] = !capturing;
  int rc = fit_rows_csr_launch(ctx, adj, coarse_rank, X, w, n, k, caliber, radius, improvement_tol, constrain,
                               nonnegative, ridge_override, out_cnt, out_col, out_val, rowptr, st);
  ctx->prof.batched[FAM_FIT] = false;
  ctx->stream = main;
  std::swap(ctx->arena, fs->arena[slot]);
  std::swap(saved, ctx->arena);
  if (!capturing) {
    // even after an error: the join keeps the main stream ordered after whatever was enqueued
    cudaEventRecord(fs->join[slot], fs->side[slot]);
    fs->pending[slot] = true;
  }
  return rc;
}

extern "C" int bamg_fit_rows_wait(bamg_ctx* ctx, int nslots, const int32_t* slots, int64_t* status_host,
                                  int64_t* nnz_host) {
  BAMG_REQUIRE(ctx, nslots >= 1 && nslots <= FIT_SLOTS, "1..4 slots");
  FitSlots* fs = fit_slots(ctx);
  BAMG_REQUIRE(ctx, fs != nullptr, "fit slot state allocation failed");
  bool any = false;
  for (int s = 0; s < FIT_SLOTS; ++s)  // join every pending slot back into the main stream
    if (fs->pending[s]) {
      BAMG_CHECK_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, fs->join[s], 0));
      fs->pending[s] = false;
      any = true;
    }
  if (any && ((ctx->prof.mask >> FAM_FIT) & 1u))  // close the batch's event pair
    cudaEventRecord(prof_event(ctx, FAM_FIT), ctx->stream);
  unsigned long long* st = fs->status;
  int64_t h[4 * FIT_SLOTS];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<const int64_t*>(st), 4 * FIT_SLOTS, h));
  for (int i = 0; i < nslots; ++i) {
    BAMG_REQUIRE(ctx, slots[i] >= 0 && slots[i] < FIT_SLOTS, "slot must lie in [0, 4)");
    const int64_t* q = h + 4 * slots[i];
    nnz_host[i] = q[3];
    BAMG_TRY(fit_status_check(ctx, q, status_host ? status_host + 2 * i : nullptr));
  }
  return 0;
}

// The fit, the kept-entry count of its rows and the row-pointer scan in one
// call with ONE host read: [pinv-branch points, overflows, deferred, nnz].
// The caller allocates col/val for nnz and finishes with bamg_rows_fill.
extern "C" int bamg_fit_rows_csr(bamg_ctx* ctx, const bamg_csr* adj, const int32_t* coarse_rank, const double* X,
                                 const double* w, int64_t n, int k, int caliber, int radius, double improvement_tol,
                                 int constrain, int nonnegative, double ridge_override, int32_t* out_cnt,
                                 int32_t* out_col, double* out_val, int32_t* rowptr, int64_t* status_host,
                                 int64_t* nnz_host) {
  ctx->arena.reset();
  if (status_host) status_host[0] = status_host[1] = 0;
  unsigned long long* status;
  BAMG_TRY(arena_get(ctx, 4, &status));
  BAMG_TRY(fit_rows_launch(ctx, adj, coarse_rank, X, w, n, k, caliber, radius, improvement_tol, constrain,
                           nonnegative, ridge_override, out_cnt, out_col, out_val, status));
  int32_t* c;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &c));
  BAMG_LAUNCH(ctx, rows_count_kernel, grid_for(n, 256), 256, 0, out_cnt, out_val, n, caliber, c);
  BAMG_TRY(scan_i32_dev(ctx, c, rowptr, n, reinterpret_cast<int64_t*>(status + 3)));
  int64_t st[4];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(status), 4, st));
  *nnz_host = st[3];
  return fit_status_check(ctx, st, status_host);
}

// ---------------------------------------------- fixed-stride rows -> CSR
__global__ void rows_count_kernel(const int32_t* __restrict__ cnt, const double* __restrict__ val, int64_t n,
                                  int stride, int32_t* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int t = 0; t < cnt[i]; ++t)
    if (!(fabs(val[i * stride + t]) < 1e-300)) ++c;
  out[i] = c;
}

__global__ void rows_fill_kernel(const int32_t* __restrict__ cnt, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, int64_t n, int stride,
                                 const int32_t* __restrict__ rp, int32_t* __restrict__ col_out,
                                 double* __restrict__ val_out) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int w = rp[i];
  int start = w;
  for (int t = 0; t < cnt[i]; ++t) {
    double v = val[i * stride + t];
    if (fabs(v) < 1e-300) continue;
    int c = col[i * stride + t];
    int p = w++;
    while (p > start && col_out[p - 1] > c) {  // insertion by column
      col_out[p] = col_out[p - 1];
      val_out[p] = val_out[p - 1];
      --p;
    }
    col_out[p] = c;
    val_out[p] = v;
  }
}

extern "C" int bamg_rows_count(bamg_ctx* ctx, const int32_t* cnt, const double* val, int64_t n, int stride,
                               int32_t* rowptr, int64_t* nnz_host) {
  ctx->arena.reset();
  int32_t* c;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &c));
  BAMG_LAUNCH(ctx, rows_count_kernel, grid_for(n, 256), 256, 0, cnt, val, n, stride, c);
  return scan_i32(ctx, c, rowptr, n, nnz_host);
}

extern "C" int bamg_rows_fill(bamg_ctx* ctx, const int32_t* cnt, const int32_t* col, const double* val, int64_t n,
                              int stride, const int32_t* rowptr, int32_t* col_out, double* val_out) {
  BAMG_LAUNCH(ctx, rows_fill_kernel, grid_for(n, 256), 256, 0, cnt, col, val, n, stride, rowptr, col_out, val_out);
  return 0;
}
