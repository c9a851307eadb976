// solver.cu -- V-cycle preconditioner and left-preconditioned GMRES.
//
// VCycleOperator (solver.py:79-124): per level nu1 weighted-Jacobi sweeps
// from a zero guess, residual, restriction by Q, recursion, prolongation +
// correction by P, nu2 sweeps; the coarsest level applies the explicit
// pseudo-inverse Z = B_L^+ (built once in setup by dense.cu) as one GEMV.
// All level kernels are the bit-exact CSR-stream kernels of sparse.cu, so a
// V-cycle on identical operators reproduces the reference bit for bit apart
// from the coarsest GEMV.
//
// GMRES (solver.py:136-226): left preconditioning op(v) = C(Bv), Arnoldi
// orthogonalisation by two-pass classical Gram-Schmidt (CGS2: three fused
// passes over the basis -- dot, update+dot, update+norm -- instead of the
// reference's 2(j+1) serial MGS dot/axpy pairs), Givens rotations and the
// triangular solve in a one-CTA kernel, x = x0 + e + V y fused, and the true
// residual ||Bx||/||x|| every iteration (one 3-double device->host read per
// iteration, the only host synchronisation of the solve).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

struct HLevel {
  bamg_csr B{}, P{}, Q{};
  const double* d = nullptr;
  const uint8_t* skip = nullptr;
  int n = 0;
  double* x = nullptr;   // iterate
  double* x2 = nullptr;  // ping-pong partner
  double* b = nullptr;   // rhs (levels >= 1)
  double* r = nullptr;   // residual
  double* rd = nullptr;  // RN(1/d) for the sweeps' division
};

// A captured V-cycle for one (b, x) pointer pair: the ~10 launches per level
// of the V-cycle replay as one cudaGraphLaunch (no per-kernel CPU launch cost,
// device-side back-to-back scheduling of the dependent level kernels).
struct VGraph {
  const double* b;
  double* x;
  cudaGraphExec_t exec;
  int nkernels;
};

struct bamg_hier {
  bamg_ctx* ctx = nullptr;
  std::vector<HLevel> lv;
  const double* Z = nullptr;
  int nz = 0;
  const bamg_coarse_lu* clu = nullptr;  // coarsest solve through the kept LU (large n)
  double omega = 0.7;
  int nu1 = 3, nu2 = 3;
  std::vector<std::pair<char*, size_t>> owned;  // level buffers (from / back to ctx->buf_pool)
  bool ready = false;
  std::vector<VGraph> graphs;
};

constexpr size_t EXEC_POOL_MAX = 16;

// graphs go back to the context pool (a later hierarchy re-points them)
static void hier_drop_graphs(bamg_hier* h) {
  bamg_ctx* ctx = h->ctx;
  for (auto& g : h->graphs) {
    if (ctx->exec_pool.size() < EXEC_POOL_MAX) ctx->exec_pool.push_back(g.exec);
    else cudaGraphExecDestroy(g.exec);
  }
  h->graphs.clear();
}

extern "C" int bamg_hier_create(bamg_ctx* ctx, int nlevels, bamg_hier** out) {
  BAMG_REQUIRE(ctx, nlevels >= 1 && out, "hierarchy needs at least one level");
  bamg_hier* h = new bamg_hier();
  h->ctx = ctx;
  h->lv.resize(nlevels);
  *out = h;
  return 0;
}

extern "C" int bamg_hier_destroy(bamg_hier* h) {
  if (!h) return 0;
  // in-flight replays of this hierarchy's graphs must finish before their
  // executables and buffers are handed to the next hierarchy
  cudaStreamSynchronize(h->ctx->stream);
  hier_drop_graphs(h);
  for (auto& b : h->owned) pool_give(h->ctx, b.first, b.second);
  delete h;
  return 0;
}

extern "C" int bamg_hier_set_level(bamg_hier* h, int level, const bamg_csr* B, const double* d,
                                   const uint8_t* skip, const bamg_csr* P, const bamg_csr* Q) {
  bamg_ctx* ctx = h->ctx;
  BAMG_REQUIRE(ctx, level >= 0 && level < (int)h->lv.size(), "level out of range");
  HLevel& L = h->lv[level];
  L.B = *B;
  L.d = d;
  L.skip = skip;
  L.n = B->nrows;
  if (P) L.P = *P;
  if (Q) L.Q = *Q;
  h->ready = false;
  hier_drop_graphs(h);
  return 0;
}

extern "C" int bamg_hier_set_coarsest(bamg_hier* h, const double* Z, int n) {
  h->Z = Z;
  h->nz = n;
  h->clu = nullptr;
  hier_drop_graphs(h);
  return 0;
}

extern "C" int bamg_hier_set_coarsest_lu(bamg_hier* h, const bamg_coarse_lu* lu, int n) {
  h->clu = lu;
  h->Z = nullptr;
  h->nz = n;
  hier_drop_graphs(h);
  return 0;
}

extern "C" int bamg_hier_set_smoother(bamg_hier* h, double omega, int nu_pre, int nu_post) {
  h->omega = omega;
  h->nu1 = nu_pre;
  h->nu2 = nu_post;
  hier_drop_graphs(h);
  return 0;
}

static int hier_prepare(bamg_hier* h) {
  if (h->ready) return 0;
  bamg_ctx* ctx = h->ctx;
  int L = (int)h->lv.size();
  BAMG_REQUIRE(ctx, (h->Z || h->clu) && h->nz == h->lv[L - 1].n, "coarsest pseudo-inverse missing or wrong size");
  size_t total = 0;
  for (int l = 0; l < L; ++l) {
    HLevel& v = h->lv[l];
    BAMG_REQUIRE(ctx, v.B.rowptr != nullptr, "level operator missing");
    if (l + 1 < L) BAMG_REQUIRE(ctx, v.P.rowptr && v.Q.rowptr, "transfer operators missing");
    total += (size_t)5 * (v.n > 0 ? v.n : 1) + 32;  // 256-byte aligned level slices
  }
  if (h->owned.empty() || h->owned[0].second < total * sizeof(double)) {
    for (auto& b : h->owned) pool_give(ctx, b.first, b.second);
    h->owned.clear();
    char* p = nullptr;
    BAMG_TRY(pool_take(ctx, total * sizeof(double), &p));
    h->owned.push_back({p, total * sizeof(double)});
  }
  double* buf = reinterpret_cast<double*>(h->owned[0].first);
  for (int l = 0; l < L; ++l) {
    HLevel& v = h->lv[l];
    size_t n = (size_t)(v.n > 0 ? v.n : 1);
    v.x = buf;
    v.x2 = buf + n;
    v.b = buf + 2 * n;
    v.r = buf + 3 * n;
    v.rd = buf + 4 * n;
    buf += ((5 * n + 31) / 32) * 32;
    if (v.n > 0 && v.d) BAMG_TRY(recip_dev(ctx, v.d, v.n, v.rd));
  }
  h->ready = true;
  return 0;
}

// x = 0 + (omega * (b - 0)) / d  on unskipped rows (the first sweep from the
// zero guess, bit-identical to relax.py:78-83 with x = 0).
template <bool VEC>
__global__ void jacobi_from_zero_kernel(int n, const double* __restrict__ b, const double* __restrict__ d,
                                        const uint8_t* __restrict__ skip, double omega,
                                        double* __restrict__ x, const double* __restrict__ rd) {
  BAMG_PDL_PROLOGUE();
  // two rows per thread (16-byte loads); the plain IEEE division needs no 1/d stream here --
  // a pure streaming kernel has the issue slots for it (25 instead of 33 bytes per row)
  (void)rd;
  const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (!VEC) {  // misaligned caller buffers: scalar loads, same arithmetic
    for (int r = i; r < min(i + 2, n); ++r) x[r] = __dadd_rn(0.0, skip[r] ? 0.0 : __ddiv_rn(__dmul_rn(omega, b[r]), d[r]));
    return;
  }
  if (i + 1 < n) {
    const double2 bv = *reinterpret_cast<const double2*>(b + i);
    const double2 dv = *reinterpret_cast<const double2*>(d + i);
    const uchar2 sk = *reinterpret_cast<const uchar2*>(skip + i);
    double2 out;
    out.x = __dadd_rn(0.0, sk.x ? 0.0 : __ddiv_rn(__dmul_rn(omega, bv.x), dv.x));
    out.y = __dadd_rn(0.0, sk.y ? 0.0 : __ddiv_rn(__dmul_rn(omega, bv.y), dv.y));
    *reinterpret_cast<double2*>(x + i) = out;
  } else if (i < n) {
    x[i] = __dadd_rn(0.0, skip[i] ? 0.0 : __ddiv_rn(__dmul_rn(omega, b[i]), d[i]));
  }
}

static int jacobi_from_zero(bamg_ctx* ctx, int64_t n, const double* b, const double* d, const uint8_t* skip,
                            double omega, double* x) {
  const bool vec = ((reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(x)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(skip) & 1) == 0;
  const int g = grid_for((n + 1) / 2, 256);
  if (vec) BAMG_LAUNCH(ctx, jacobi_from_zero_kernel<true>, g, 256, 0, (int)n, b, d, skip, omega, x, (const double*)nullptr);
  else BAMG_LAUNCH(ctx, jacobi_from_zero_kernel<false>, g, 256, 0, (int)n, b, d, skip, omega, x, (const double*)nullptr);
  return 0;
}

// y = Z b, Z row-major n x n (warp per row, coalesced).
__global__ void gemv_rowmajor_kernel(int n, const double* __restrict__ Z, const double* __restrict__ b,
                                     double* __restrict__ y) {
  BAMG_PDL_PROLOGUE();
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const double* zr = Z + (int64_t)warp * n;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s += zr[j] * b[j];
  s = warp_sum(s);
  if (lane == 0) y[warp] = s;
}

static int vcycle_impl(bamg_ctx* ctx, bamg_hier* h, const double* b_in, double* x_out) {
  BAMG_TRY(hier_prepare(h));
  int L = (int)h->lv.size();
  const double om = h->omega;
  // downward
  const double* bl = b_in;
  std::vector<double*> xs(L);
  for (int l = 0; l < L - 1; ++l) {
    HLevel& v = h->lv[l];
    double* cur = v.x;
    double* oth = v.x2;
    if (h->nu1 > 0) {
      BAMG_TRY(jacobi_from_zero(ctx, v.n, bl, v.d, v.skip, om, cur));
      for (int s = 1; s < h->nu1; ++s) {
        BAMG_TRY(jacobi_dev(ctx, &v.B, v.d, v.skip, bl, nullptr, cur, oth, 1, om, nullptr, v.rd));
        std::swap(cur, oth);
      }
    } else {
      BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(cur, 0, sizeof(double) * v.n, ctx->stream));
    }
    xs[l] = cur;
    v.x2 = oth;
    v.x = cur;
    BAMG_TRY(resid_dev(ctx, &v.B, bl, cur, v.r));
    HLevel& c = h->lv[l + 1];
    BAMG_TRY(spmm_dev(ctx, &v.Q, v.r, c.b, 1));
    bl = c.b;
  }
  // coarsest: x_L = Z b_L
  HLevel& cl = h->lv[L - 1];
  double* xc = (L == 1) ? x_out : cl.x;
  if (h->clu) {
    BAMG_TRY(coarse_lu_apply(ctx, h->clu, bl, xc));
  } else {
    BAMG_LAUNCH(ctx, gemv_rowmajor_kernel, grid_for((int64_t)h->nz * 32, 256), 256, 0, h->nz, h->Z, bl, xc);
  }
  // upward
  for (int l = L - 2; l >= 0; --l) {
    HLevel& v = h->lv[l];
    const double* blv = (l == 0) ? b_in : v.b;
    double* cur = v.x;
    double* oth = v.x2;
    // x <- x + P xc  (written to the partner buffer, then ping-pong)
    BAMG_TRY(addmv_dev(ctx, &v.P, xc, cur, oth, 1));
    std::swap(cur, oth);
    for (int s = 0; s < h->nu2; ++s) {
      double* dst = (l == 0 && s == h->nu2 - 1) ? x_out : oth;
      BAMG_TRY(jacobi_dev(ctx, &v.B, v.d, v.skip, blv, nullptr, cur, dst, 1, om, nullptr, v.rd));
      if (dst == x_out) {
        cur = x_out;
      } else {
        std::swap(cur, oth);
      }
    }
    if (l == 0 && h->nu2 == 0)
      BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(x_out, cur, sizeof(double) * v.n, cudaMemcpyDeviceToDevice, ctx->stream));
    v.x = cur == x_out ? v.x : cur;
    xc = cur;
  }
  return 0;
}

static bool graphs_enabled(bamg_ctx* ctx) {
  // the development trace wants every launch, unless BAMG_TRACE_GRAPHS=1 (one
  // timeline entry per V-cycle graph replay)
  const char* tg = getenv("BAMG_TRACE_GRAPHS");
  if (ctx->trace.on && !(tg && tg[0] == '1')) return false;
  const char* e = getenv("BAMG_NO_GRAPHS");
  return !(e && e[0] == '1');
}

// V-cycle through a cached CUDA graph keyed by (b, x); captured on a private
// non-blocking stream (the context stream may be the legacy default stream,
// which cannot capture) and replayed on the context stream.
static int vcycle_run(bamg_ctx* ctx, bamg_hier* h, const double* b, double* x) {
  if (!graphs_enabled(ctx)) return vcycle_impl(ctx, h, b, x);
  BAMG_TRY(hier_prepare(h));
  VGraph* g = nullptr;
  for (auto& e : h->graphs)
    if (e.b == b && e.x == x) g = &e;
  if (!g) {
    if (h->graphs.size() >= 8) hier_drop_graphs(h);
    if (!ctx->cap_stream) BAMG_CHECK_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaStream_t cap = ctx->cap_stream;
    cudaStream_t saved = ctx->stream;
    int64_t l0 = ctx->launches;
    unsigned saved_mask = ctx->prof.mask;  // no profiler events inside the graph
    ctx->prof.mask = 0;
    const bool saved_trace = ctx->trace.on;  // nor trace events
    ctx->trace.on = false;
    ctx->stream = cap;
    cudaGraph_t graph;
    cudaError_t e1 = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    int rc = e1 == cudaSuccess ? vcycle_impl(ctx, h, b, x) : -1;
    cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    ctx->stream = saved;
    ctx->prof.mask = saved_mask;
    ctx->trace.on = saved_trace;
    int nk = (int)(ctx->launches - l0);
    ctx->launches = l0;
    if (e1 != cudaSuccess || e2 != cudaSuccess || rc != 0) {
      ctx->err = std::string("V-cycle graph capture failed: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
      return rc != 0 ? rc : -1;
    }
    // re-point a pooled executable of the same topology (a V-cycle of another
    // hierarchy with the same level count); instantiate only when none fits
    cudaGraphExec_t exec = nullptr;
    while (!exec && !ctx->exec_pool.empty()) {
      cudaGraphExec_t cand = ctx->exec_pool.back();
      ctx->exec_pool.pop_back();
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(cand, graph, &info) == cudaSuccess) {
        exec = cand;
      } else {
        (void)cudaGetLastError();  // clear the non-sticky update failure
        cudaGraphExecDestroy(cand);
      }
    }
    if (!exec) BAMG_CHECK_CUDA(ctx, cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    h->graphs.push_back({b, x, exec, nk});
    g = &h->graphs.back();
  }
  if (ctx->trace.on) trace_mark(ctx, "vcycle_graph");
  BAMG_CHECK_CUDA(ctx, cudaGraphLaunch(g->exec, ctx->stream));
  if (ctx->trace.on) trace_mark(ctx, nullptr);
  ctx->launches += g->nkernels;
  return 0;
}

extern "C" int bamg_vcycle(bamg_ctx* ctx, bamg_hier* h, const double* b, double* x) {
  ctx->arena.reset();
  return vcycle_run(ctx, h, b, x);
}

// ===================================================================== GMRES
constexpr int GM_BLOCKS = RED_BLOCKS;
constexpr int GM_THREADS = 256;
constexpr int GM_GROUP = 16;  // basis vectors per register group

// state code of an Arnoldi step (code[0]): 1 = one projection suffices (DGKS),
// 0 = second projection, safe Pythagorean norm, 2 = second projection with the
// explicit norm.  A kernel gated on `mask` runs iff bit code[0] is set.
__device__ __forceinline__ bool cgs_gate(const double* code, unsigned mask) {
  return !code || ((mask >> (int)code[0]) & 1u);
}


// partial[b * m + i] = sum over block b's chunk of V_i . w   (i < m)
__global__ void __launch_bounds__(GM_THREADS)
mdot_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ w, int64_t n,
            double* __restrict__ partial) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[GM_THREADS / 32][GM_GROUP];
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = min(r0 + per, n);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g0 = 0; g0 < m; g0 += GM_GROUP) {
    double acc[GM_GROUP];
#pragma unroll
    for (int g = 0; g < GM_GROUP; ++g) acc[g] = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += GM_THREADS) {
      double wi = w[i];
#pragma unroll
      for (int g = 0; g < GM_GROUP; ++g)
        if (g0 + g < m) acc[g] += Vp[g0 + g][i] * wi;
    }
#pragma unroll
    for (int g = 0; g < GM_GROUP; ++g) {
      double v = warp_sum(acc[g]);
      if (lane == 0) sh[wid][g] = v;
    }
    __syncthreads();
    if (threadIdx.x < GM_GROUP && g0 + threadIdx.x < m) {
      double v = 0.0;
      for (int q = 0; q < GM_THREADS / 32; ++q) v += sh[q][threadIdx.x];
      partial[(int64_t)blockIdx.x * m + g0 + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

// w -= sum_i c_i V_i ; then optionally partial dots V_i . w_new (mode 1) or
// the partial |w_new|^2 (mode 2).  c read from device.
template <int MODE>
__global__ void __launch_bounds__(GM_THREADS)
mupdate_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ c,
               double* __restrict__ w, int64_t n, double* __restrict__ partial) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[GM_THREADS / 32][GM_GROUP];
  __shared__ double sc[1024];
  for (int i = threadIdx.x; i < m && i < 1024; i += GM_THREADS) sc[i] = c[i];
  __syncthreads();
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = min(r0 + per, n);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += GM_THREADS) {
    double t = 0.0;
    for (int g = 0; g < m; ++g) t += (g < 1024 ? sc[g] : c[g]) * Vp[g][i];
    double wn = w[i] - t;
    w[i] = wn;
    if (MODE == 2) nrm += wn * wn;
  }
  if (MODE == 2) {
    double v = warp_sum(nrm);
    if (lane == 0) sh[wid][0] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < GM_THREADS / 32; ++q) s += sh[q][0];
      partial[blockIdx.x] = s;
    }
  }
}

// out[i] = sum_b partial[b * m + i]  (fixed order -> deterministic)
__global__ void mreduce_kernel(const double* __restrict__ partial, int nb, int m, double* __restrict__ out,
                               int accumulate) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (i >= m) return;
  double v = 0.0;
  for (int b = lane; b < nb; b += 32) v += partial[(int64_t)b * m + i];
  v = warp_sum(v);
  if (lane == 0) out[i] = accumulate ? out[i] + v : v;
}

// Arnoldi bookkeeping for column j (solver.py:189-209), one thread:
//   h[j+1] = sqrt(nrm2); happy test; previous rotations; new rotation;
//   R[:, j]; g; y = R^-1 g (back substitution).  state[0] = happy flag,
//   state[1] = h[j+1].
// flag / mask: with a CGS step code (see cgs_gate) the kernel runs only when
// bit flag[0] of mask is set, so each branch's norm reaches the rotation
// exactly once.
__global__ void givens_kernel(int j, int ldr, double* __restrict__ h, const double* __restrict__ nrm2,
                              double beta, double* __restrict__ R, double* __restrict__ g,
                              double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ y,
                              double* __restrict__ state, const double* __restrict__ flag, unsigned mask) {
  BAMG_PDL_PROLOGUE();
  if (!cgs_gate(flag, mask)) return;
  extern __shared__ double sg[];  // j+1 working entries of g during the back substitution
  if (threadIdx.x == 0) {
    double hj1 = sqrt(nrm2[0]);
    h[j + 1] = hj1;
    double happy = (hj1 <= 1e-14 * beta) ? 1.0 : 0.0;
    for (int i = 0; i < j; ++i) {
      double t = cs[i] * h[i] + sn[i] * h[i + 1];
      h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
      h[i] = t;
    }
    double rad = hypot(h[j], h[j + 1]);
    if (rad == 0.0) {
      cs[j] = 1.0;
      sn[j] = 0.0;
    } else {
      cs[j] = h[j] / rad;
      sn[j] = h[j + 1] / rad;
    }
    for (int i = 0; i < j; ++i) R[(int64_t)j * ldr + i] = h[i];  // column j (column-major)
    R[(int64_t)j * ldr + j] = rad;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    state[0] = happy;
    state[1] = hj1;
  }
  __syncthreads();
  // back substitution R[:j+1, :j+1] y = g[:j+1], column-oriented: y_i, then
  // the CTA removes column i of R from the remaining right-hand side
  for (int q = threadIdx.x; q <= j; q += blockDim.x) sg[q] = g[q];
  __syncthreads();
  for (int i = j; i >= 0; --i) {
    const double yi = sg[i] / R[(int64_t)i * ldr + i];
    if (threadIdx.x == 0) y[i] = yi;
    for (int q = threadIdx.x; q < i; q += blockDim.x) sg[q] -= R[(int64_t)i * ldr + q] * yi;
    __syncthreads();
  }
}

// dst = w / h  unless the happy-breakdown flag is set
__global__ void scale_new_basis_kernel(const double* __restrict__ w, const double* __restrict__ state,
                                       int64_t n, double* __restrict__ dst) {
  BAMG_PDL_PROLOGUE();
  if (state[0] != 0.0) return;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double h = state[1];
  if (i < n) dst[i] = w[i] / h;
}

// out = base + add + sum_g y_g V_g   (add may be null)
__global__ void combine_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ y,
                               const double* __restrict__ base, const double* __restrict__ e_add,
                               const double* __restrict__ e_add2, int64_t n, double* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sy[1024];
  for (int i = threadIdx.x; i < m && i < 1024; i += blockDim.x) sy[i] = y[i];
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = 0.0;
  for (int g = 0; g < m; ++g) t += (g < 1024 ? sy[g] : y[g]) * Vp[g][i];
  double e = e_add ? e_add[i] + t : t;   // e_try = e + V y
  out[i] = base ? base[i] + e : e;        // x = x0 + e_try
  (void)e_add2;
}

__global__ void axpby_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                             double* __restrict__ out) {
  BAMG_PDL_PROLOGUE();  // out = a - b
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}

__global__ void scale_div_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ s,
                                 double* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] / s[0];
}

// ---- register-resident CGS2 passes (basis of <= CGS_MAXM vectors)
// Reorthogonalisation is applied only where it is needed (the DGKS criterion,
// eta = 1/sqrt(2)): pass A also forms |w|^2, and when the first projection
// keeps |w - V h|^2 = |w|^2 - |h|^2 >= |w|^2 / 2 the step is ONE more pass
// (pass C with h, straight from w) -- two passes over V instead of three.
// Otherwise the classical second pass runs (below).  Which branch a step
// takes is decided on the device (a state code, every kernel gated on it),
// so the host never waits for it.
// One Arnoldi step in three passes over the basis instead of five:
//   A: h  = V^T w                                   (dots)
//   B: w' = w - V h ; h2 = V^T w' ; |w'|^2          (update + dots, one read of V)
//   C: v_{j+1} = (w' - V h2) / h_{j+1} ; x = x0 + e + V y ; |x|^2
// with h_{j+1}^2 = |w'|^2 - |h2|^2 (Pythagoras: w'' = w' - V h2 is w' minus
// its projection on the orthonormal basis), so the Givens update and the
// least-squares y of column j are known before pass C and the iterate x the
// stopping test needs is formed in the same read of V.  Where the difference
// loses more than two digits (|w''|^2 < 1e-2 |w'|^2: w' nearly inside span V)
// the step falls back on device to the explicit norm (cgs_fix_*).  Each CTA
// owns a fixed contiguous row chunk and reduces its partial sums in a fixed
// order (deterministic).  Values V_g[i] of a row stay in registers between
// the update and the dots of pass B.
constexpr int CGS_MAXM = 64;
__constant__ bool cgs_force_two_pass = false;  // BAMG_CGS_ALWAYS_REORTH=1 (development)
constexpr int CGS_THREADS = 128;
constexpr int CGS_WARPS = CGS_THREADS / 32;
constexpr int CGS_MAX_BLOCKS = 32 * 148;  // partial-sum slots per CTA: CGS_MAXM + 1

// rows per CTA chunk, a multiple of 32: with the 256-byte aligned basis vectors every warp load
// (32 consecutive doubles) then covers exactly two whole 128-byte lines.  Unaligned chunks made
// each load straddle a line shared with the neighbouring warp's, and under the evict-first
// streaming loads that line was fetched from DRAM twice: ncu showed the passes at the DRAM peak
// (6.0-6.6 TB/s) while reading 1.15-1.22x their algorithmic bytes at m = 32 ... 60.
__device__ __forceinline__ int64_t cgs_chunk_rows(int64_t n, int nblk) {
  const int64_t per = (n + nblk - 1) / nblk;
  return (per + 31) & ~(int64_t)31;
}

template <int MAXM>
__device__ __forceinline__ void cgs_load_ptrs(const double* const* __restrict__ Vp, int m, const double** sp) {
  // slots past m alias V_0 (their coefficients are zero): the loads stay
  // unconditional, so all of a row's loads issue back to back
  for (int g = threadIdx.x; g < MAXM; g += blockDim.x) sp[g] = Vp[g < m ? g : 0];
  __syncthreads();
}

// per-warp partial sums acc[warp][slot] -> part[block * stride + slot], fixed order
__device__ __forceinline__ void cgs_flush(double (*acc)[CGS_MAXM + 2], int nslots, double* __restrict__ part,
                                          int stride) {
  __syncthreads();
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < CGS_WARPS; ++w) v += acc[w][q];
    part[(int64_t)blockIdx.x * stride + q] = v;
  }
}

// Transpose reduction of 32 per-lane values: afterwards lane l holds
// sum over the warp's lanes of a[l] (in a[0]); 31 shuffles instead of the
// 160 of 32 separate butterfly sums.
__device__ __forceinline__ double warp_transpose_sum32(double (&a)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? a[i] : a[i + half];
      const double keep = hi ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return a[0];
}

// The same fold for NV = 8 or 16 values per lane: log2(NV) halving steps leave lane l with value
// l mod NV summed over its group of NV lanes, and the 32 / NV groups are added by plain butterfly
// steps (9 / 16 shuffles instead of 31); every lane ends with the total of value l mod NV.
template <int NV>
__device__ __forceinline__ double warp_transpose_sum_n(double (&a)[NV], int lane) {
#pragma unroll
  for (int half = NV / 2; half >= 1; half >>= 1) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? a[i] : a[i + half];
      const double keep = hi ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  double r = a[0];
#pragma unroll
  for (int o = NV; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// products of the row's NS values with s, folded over the warp (NS <= 32 slots of one group)
template <int NS>
__device__ __forceinline__ double cgs_fold(const double* v, double s, int lane) {
  constexpr int NV = NS <= 8 ? 8 : 32;  // (the 16-value fold compiles to more registers than the 32-value one)
  double pr[NV];
#pragma unroll
  for (int g = 0; g < NV; ++g) pr[g] = g < NS ? v[g < NS ? g : 0] * s : 0.0;
  return warp_transpose_sum_n<NV>(pr, lane);
}

// MODE 0 (pass A): part[b][g] = chunk sum of V_g . w, part[b][m] = |w|^2
// MODE 1 (pass B): w <- w - sum_g c_g V_g (in place); part[b][g] = V_g . w_new,
//                  part[b][m] = |w_new|^2  (runs only for code 0)
// A warp takes 32 consecutive rows (one per lane) at a time; the row's MAXM
// basis values stay in registers, the 32 x MAXM products are folded across
// the warp by transpose reductions, and lane l accumulates the dots of
// vectors l, l + 32 over all of the warp's rows.
// NS = the slots a thread really loads (a multiple of 8, >= the group's m): slots past m alias V_0
// with zero coefficients, and every aliased load is an L1 hit that still costs an LSU slot -- a
// group of 5 vectors read through 32 slots spent most of its load issue on them.
// RU = row sets in flight per thread: a short basis (NS = 8, 16) has too few loads per row to cover the
// memory latency at the kernel's occupancy (m = 1: 8 KB in flight per SM, 1.1 TB/s), so 32 / NS row
// sets are loaded before any is folded; the folds follow in row order (the sums are unchanged).
template <int NS, int MODE>
__device__ __forceinline__ void cgs_dots_body(const double* const* sp, const double* sc, double (*acc)[CGS_MAXM + 2],
                                              int m, double* __restrict__ w, int64_t r0, int64_t r1, int lane,
                                              int wid) {
  constexpr int NB = (NS + 31) / 32;
  constexpr int RU = NS <= 8 ? 4 : (NS <= 16 ? 2 : 1);
  double dot[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) dot[q] = 0.0;
  double wn2 = 0.0;
  for (int64_t base = r0 + wid * 32; base < r1; base += (int64_t)RU * CGS_THREADS) {
    double v[RU][NS], wi[RU];
    bool ok[RU];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int64_t i = base + (int64_t)r * CGS_THREADS + lane;
      ok[r] = i < r1;
      const int64_t ic = ok[r] ? i : r0;  // rows past the chunk read row r0 and contribute 0
#pragma unroll
      for (int g = 0; g < NS; ++g) v[r][g] = __ldcs(sp[g] + ic);
      wi[r] = w[ic];
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      if (r > 0 && base + (int64_t)r * CGS_THREADS >= r1) break;  // warp-uniform: no rows left
      if (MODE == 1) {
        double t = 0.0;
#pragma unroll
        for (int g = 0; g < NS; ++g) t = fma(sc[g], v[r][g], t);
        wi[r] -= t;
        if (ok[r]) w[base + (int64_t)r * CGS_THREADS + lane] = wi[r];
      }
      if (!ok[r]) wi[r] = 0.0;
      wn2 = fma(wi[r], wi[r], wn2);
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q * 32 >= m) break;
        if constexpr (NS <= 32) {
          dot[q] += cgs_fold<NS>(v[r], wi[r], lane);
        } else {
          double pr[32];
#pragma unroll
          for (int g = 0; g < 32; ++g) pr[g] = q * 32 + g < NS ? v[r][q * 32 + g < NS ? q * 32 + g : 0] * wi[r] : 0.0;
          dot[q] += warp_transpose_sum32(pr, lane);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) acc[wid][q * 32 + lane] = dot[q];
  wn2 = warp_sum(wn2);
  if (lane == 0) acc[wid][CGS_MAXM] = wn2;
}

template <int MAXM, int MODE>
__global__ void __launch_bounds__(CGS_THREADS)
cgs_dots_kernel(const double* const* __restrict__ Vp, int m_all, const double* __restrict__ c, double* __restrict__ w,
                int64_t n, double* __restrict__ part, const double* __restrict__ code, int nblk) {
  BAMG_PDL_PROLOGUE();
  if (MODE == 1 && !cgs_gate(code, 1u << 0)) return;
  // more than nblk CTAs (pass A only): CTAs [y nblk, (y + 1) nblk) take the basis vectors
  // [y MAXM, (y + 1) MAXM) -- two <32> groups keep 116 registers (4 CTAs per SM) where one <64>
  // pass needs 168 (2-3 per SM)
  const int by = blockIdx.x / nblk, bx = blockIdx.x - by * nblk;
  const int stride = m_all + 1, slot0 = by * MAXM;
  Vp += slot0;
  const int m = min(MAXM, m_all - slot0);
  static_assert(MAXM % 32 == 0, "basis slots come in warps of 32");
  __shared__ const double* sp[MAXM];
  __shared__ double sc[MAXM];
  __shared__ double acc[CGS_WARPS][CGS_MAXM + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (MODE == 1)
    for (int g = threadIdx.x; g < MAXM; g += blockDim.x) sc[g] = g < m ? c[g] : 0.0;
  cgs_load_ptrs<MAXM>(Vp, m, sp);
  const int64_t per = cgs_chunk_rows(n, nblk);
  const int64_t r0 = (int64_t)bx * per, r1 = min(r0 + per, n);
  if (MAXM == 32 && m <= 8) cgs_dots_body<8, MODE>(sp, sc, acc, m, w, r0, r1, lane, wid);
  else if (MAXM == 32 && m <= 16) cgs_dots_body<16, MODE>(sp, sc, acc, m, w, r0, r1, lane, wid);
  else if (MAXM == 32 && m <= 24) cgs_dots_body<24, MODE>(sp, sc, acc, m, w, r0, r1, lane, wid);
  else cgs_dots_body<MAXM, MODE>(sp, sc, acc, m, w, r0, r1, lane, wid);
  __syncthreads();
  const int nslots = m + (by == 0 ? 1 : 0);  // |w|^2 (slot m_all) from the first group only
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) {
    const int slot = q == m ? CGS_MAXM : q;
    double t = 0.0;
    for (int ww = 0; ww < CGS_WARPS; ++ww) t += acc[ww][slot];
    part[(int64_t)bx * stride + (q == m ? m_all : slot0 + q)] = t;
  }
}

// out[i] = sum_b part[b * stride + i], i < cnt (fixed order)
__global__ void cgs_reduce_kernel(const double* __restrict__ part, int nb, int stride, int cnt,
                                  double* __restrict__ out, const double* __restrict__ code, unsigned mask) {
  BAMG_PDL_PROLOGUE();
  if (!cgs_gate(code, mask)) return;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= cnt) return;
  double v = 0.0;
  for (int b = lane; b < nb; b += 32) v += part[(int64_t)b * stride + i];
  v = warp_sum(v);
  if (lane == 0) out[i] = v;
}

// DGKS decision after pass A: h = hv[0..m), |w|^2 = hv[m].  One projection
// suffices when |w|^2 - |h|^2 >= |w|^2 / 2 (code 1, nrm2 = that difference);
// else code 0 (the second pass runs).
// (code 1 also copies h to h2: pass C projects with h2, and the Givens update
// rotates hv in place)
__global__ void cgs_dgks_kernel(int m, const double* __restrict__ hv, double* __restrict__ nrm2,
                                double* __restrict__ code, double* __restrict__ h2) {
  BAMG_PDL_PROLOGUE();
  __shared__ double red[32];
  double q = 0.0;
  for (int g = threadIdx.x; g < m; g += blockDim.x) q = fma(hv[g], hv[g], q);
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    const double wn = hv[m], d = wn - t;
    const bool one = d >= 0.5 * wn && wn > 0.0 && !cgs_force_two_pass;
    code[0] = one ? 1.0 : 0.0;
    if (one) nrm2[0] = d;
    red[0] = one ? 1.0 : 0.0;
  }
  __syncthreads();
  if (red[0] == 1.0)
    for (int g = threadIdx.x; g < m; g += blockDim.x) h2[g] = hv[g];
}

// (code 0 only) hv[0..m) += h2[0..m);  nrm2 = |w'|^2 - |h2|^2 (h2 = sums[0..m),
// |w'|^2 = sums[m]); code 2 when the difference lost more than two digits
__global__ void cgs_pythag_kernel(int m, const double* __restrict__ sums, double* __restrict__ hv,
                                  double* __restrict__ nrm2, double* __restrict__ flag) {
  BAMG_PDL_PROLOGUE();
  if (!cgs_gate(flag, 1u << 0)) return;
  __shared__ double red[32];
  double q = 0.0;
  for (int g = threadIdx.x; g < m; g += blockDim.x) {
    const double h2 = sums[g];
    hv[g] += h2;
    q += h2 * h2;
  }
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    const double wn = sums[m];
    const double d = wn - t;
    const bool unsafe = !(d >= 1e-2 * wn);
    nrm2[0] = unsafe ? 0.0 : d;
    flag[0] = unsafe ? 2.0 : 0.0;
  }
}

// pass C: v_new = (w' - V h2) / state[1] (skipped on happy breakdown) and
// x = x0 + e + V y with part[b] = chunk |x|^2; when flag[0] is set (unsafe
// Pythagoras) the unscaled w'' goes to v_new and part[b] = chunk |w''|^2
// instead, and x is left to cgs_fix_x_kernel.
template <int MAXM>
__global__ void __launch_bounds__(CGS_THREADS, 4)
cgs_final_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ h2,
                 const double* __restrict__ h1, const double* __restrict__ y, const double* __restrict__ wp,
                 const double* __restrict__ x0,
                 const double* __restrict__ e, const double* __restrict__ state, const double* __restrict__ flag,
                 int64_t n, double* __restrict__ vnew, double* __restrict__ x, double* __restrict__ part) {
  BAMG_PDL_PROLOGUE();
  __shared__ const double* sp[MAXM];
  __shared__ double sh[MAXM], sy[MAXM];
  __shared__ double acc[CGS_WARPS][CGS_MAXM + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  (void)h1;  // h2 holds the projection coefficients of either branch
  for (int g = threadIdx.x; g < MAXM; g += blockDim.x) {
    sh[g] = g < m ? h2[g] : 0.0;
    sy[g] = g < m ? y[g] : 0.0;
  }
  if (threadIdx.x < CGS_WARPS) acc[threadIdx.x][0] = 0.0;
  cgs_load_ptrs<MAXM>(Vp, m, sp);
  const bool unsafe = flag[0] == 2.0;
  const bool happy = state[0] != 0.0;
  const double inv = 1.0 / state[1];
  const int64_t per = cgs_chunk_rows(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += CGS_THREADS) {
    double v[MAXM];  // every load of the row issued before the first FMA
#pragma unroll
    for (int g = 0; g < MAXM; ++g) v[g] = __ldcs(sp[g] + i);
    const double wpi = wp[i], x0i = x0[i], ei = e[i];
    double t = 0.0, u = 0.0;
#pragma unroll
    for (int g = 0; g < MAXM; ++g) {
      t = fma(sh[g], v[g], t);
      u = fma(sy[g], v[g], u);
    }
    const double ww = wpi - t;
    if (unsafe) {
      vnew[i] = ww;
      nrm = fma(ww, ww, nrm);
    } else {
      if (!happy) vnew[i] = ww * inv;
      const double xi = x0i + (ei + u);
      x[i] = xi;
      nrm = fma(xi, xi, nrm);
    }
  }
  nrm = warp_sum(nrm);
  if (lane == 0) acc[wid][0] = nrm;
  cgs_flush(acc, 1, part, 1);
}

// ---- two-pass CGS2 through the Gram matrix (the default)
// CGS2's second projection h2 = V^T (w - V h1) equals h1 - G h1 with
// G = V^T V, so when G is carried along the step needs no second sweep over V
// for it: pass A (dots, above) gives h1 and |w|^2, a one-CTA kernel forms the
// total coefficients c = h1 + h2 = 2 h1 - G h1 and the new vector's norm
// |w - V c|^2 = |w|^2 - 2 c.h1 + c^T G c, and ONE more pass writes
// v_new = (w - V c) / h_{j+1}, the iterate x = x0 + e + V y with |x|^2, and --
// from the same registers -- V^T v_new and |v_new|^2, the new row of G.  G holds
// the stored basis' true inner products (round-off defects and the new
// vector's actual norm included), so later projections compensate them to first
// order; the defects themselves are what CGS2 leaves, O(eps |w| / h_{j+1}).
// Two reads of the basis per Arnoldi step instead of three.  When the norm
// formula cancels more than six digits (w all but inside span V) the step
// writes w - V c unscaled and takes the explicit norm (cgs_fix_*).
constexpr int CGS_LDG = CGS_MAXM + 1;

__global__ void cgs_gram_init_kernel(double* __restrict__ G) {
  BAMG_PDL_PROLOGUE();
  for (int i = threadIdx.x; i < CGS_LDG * CGS_LDG; i += blockDim.x) G[i] = i == 0 ? 1.0 : 0.0;
}

// hv[0..m) = h1, hv[m] = |w|^2  ->  hv[0..m) = c2[0..m) = 2 h1 - G h1,
// nrm2 = |w - V c|^2; flag 0 (safe) or 2 (explicit norm)
__global__ void cgs_gram_coef_kernel(int m, const double* __restrict__ G, double* __restrict__ hv,
                                     double* __restrict__ c2, double* __restrict__ nrm2,
                                     double* __restrict__ flag) {
  BAMG_PDL_PROLOGUE();
  __shared__ double h1[CGS_MAXM], c[CGS_MAXM], gc[CGS_MAXM];
  const int g = threadIdx.x;
  if (g < m) h1[g] = hv[g];
  __syncthreads();
  if (g < m) {
    double t = 0.0;
    for (int a = 0; a < m; ++a) t = fma(G[g * CGS_LDG + a], h1[a], t);
    c[g] = h1[g] + (h1[g] - t);
  }
  __syncthreads();
  if (g < m) {
    double t = 0.0;
    for (int a = 0; a < m; ++a) t = fma(G[g * CGS_LDG + a], c[a], t);
    gc[g] = t;
    hv[g] = c[g];
    c2[g] = c[g];
  }
  __syncthreads();
  if (g == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int a = 0; a < m; ++a) {
      s1 = fma(c[a], h1[a], s1);
      s2 = fma(c[a], gc[a], s2);
    }
    const double wn = hv[m];
    const double d = (wn - s1) - (s1 - s2);
    const bool unsafe = !(d >= 1e-6 * wn) || !(wn > 0.0);
    nrm2[0] = unsafe ? 0.0 : d;
    flag[0] = unsafe ? 2.0 : 0.0;
  }
}

// the update pass: ww = w - V c; v_new = ww / state[1] (unscaled when flag = 2,
// skipped on happy breakdown); x = x0 + e + V y (flag 0 only);
// part[b][0..m) = V^T ww, part[b][m] = |ww|^2, part[b][m + 1] = |x|^2
template <int NS>
__device__ __forceinline__ void cgs_update_body(const double* const* sp, const double* sc, const double* sy,
                                                double (*acc)[CGS_MAXM + 2], int m, const double* __restrict__ w,
                                                const double* __restrict__ x0, const double* __restrict__ e,
                                                bool unsafe, bool happy, double inv, int64_t r0, int64_t r1,
                                                double* __restrict__ vnew, double* __restrict__ x, int lane, int wid) {
  constexpr int NB = (NS + 31) / 32;
  constexpr int RU = NS <= 8 ? 4 : (NS <= 16 ? 2 : 1);  // row sets in flight (see cgs_dots_body)
  double dot[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) dot[q] = 0.0;
  double wn2 = 0.0, xn2 = 0.0;
#pragma unroll 1
  for (int64_t base = r0 + wid * 32; base < r1; base += (int64_t)RU * CGS_THREADS) {
    double v[RU][NS], wi[RU], x0i[RU], ei[RU];
    bool ok[RU];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int64_t i = base + (int64_t)r * CGS_THREADS + lane;
      ok[r] = i < r1;
      const int64_t ic = ok[r] ? i : r0;  // rows past the chunk read row r0 and contribute 0
#pragma unroll
      for (int g = 0; g < NS; ++g) v[r][g] = __ldcs(sp[g] + ic);
      wi[r] = w[ic], x0i[r] = x0[ic], ei[r] = e[ic];
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      if (r > 0 && base + (int64_t)r * CGS_THREADS >= r1) break;  // warp-uniform: no rows left
      const int64_t i = base + (int64_t)r * CGS_THREADS + lane;
      double t = 0.0, u = 0.0;
#pragma unroll
      for (int g = 0; g < NS; ++g) {
        t = fma(sc[g], v[r][g], t);
        u = fma(sy[g], v[r][g], u);
      }
      double ww = wi[r] - t;
      if (ok[r]) {
        if (unsafe) {
          vnew[i] = ww;
        } else {
          if (!happy) vnew[i] = ww * inv;
          const double xi = x0i[r] + (ei[r] + u);
          x[i] = xi;
          xn2 = fma(xi, xi, xn2);
        }
      } else {
        ww = 0.0;
      }
      wn2 = fma(ww, ww, wn2);
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q * 32 >= m) break;
        if constexpr (NS <= 32) {
          dot[q] += cgs_fold<NS>(v[r], ww, lane);
        } else {
          double pr[32];
#pragma unroll
          for (int g = 0; g < 32; ++g) pr[g] = q * 32 + g < NS ? v[r][q * 32 + g < NS ? q * 32 + g : 0] * ww : 0.0;
          dot[q] += warp_transpose_sum32(pr, lane);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) acc[wid][q * 32 + lane] = dot[q];
  wn2 = warp_sum(wn2);
  xn2 = warp_sum(xn2);
  if (lane == 0) acc[wid][CGS_MAXM] = wn2, acc[wid][CGS_MAXM + 1] = xn2;
}

template <int MAXM, int NS = MAXM>
__global__ void __launch_bounds__(CGS_THREADS, (NS <= 32 ? 4 : NS <= 48 ? 3 : 2))
cgs_update_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ c,
                  const double* __restrict__ y, const double* __restrict__ w, const double* __restrict__ x0,
                  const double* __restrict__ e, const double* __restrict__ state, const double* __restrict__ flag,
                  int64_t n, double* __restrict__ vnew, double* __restrict__ x, double* __restrict__ part) {
  BAMG_PDL_PROLOGUE();
  static_assert(MAXM % 32 == 0, "basis slots come in warps of 32");
  __shared__ const double* sp[MAXM];
  __shared__ double sc[MAXM], sy[MAXM];
  __shared__ double acc[CGS_WARPS][CGS_MAXM + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g = threadIdx.x; g < MAXM; g += blockDim.x) {
    sc[g] = g < m ? c[g] : 0.0;
    sy[g] = g < m ? y[g] : 0.0;
  }
  cgs_load_ptrs<MAXM>(Vp, m, sp);
  const bool unsafe = flag[0] == 2.0;
  const bool happy = state[0] != 0.0;
  const double inv = 1.0 / state[1];
  const int64_t per = cgs_chunk_rows(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  // NS = the slots a thread loads: the next multiple of 8 above m (see cgs_dots_body); one kernel
  // per NS, so the short passes keep their own (small) register count and occupancy
  cgs_update_body<NS>(sp, sc, sy, acc, m, w, x0, e, unsafe, happy, inv, r0, r1, vnew, x, lane, wid);
  __syncthreads();
  const int nslots = m + 2;
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) {
    const int slot = q >= m ? CGS_MAXM + (q - m) : q;
    double t = 0.0;
    for (int ww2 = 0; ww2 < CGS_WARPS; ++ww2) t += acc[ww2][slot];
    part[(int64_t)blockIdx.x * (m + 2) + q] = t;
  }
}

// The update pass for 32 < m <= 64 with the row's vectors split over a warp
// pair: warp half h of a pair keeps vectors [32 h, 32 h + 32) of 32 rows in
// registers (118 registers, 4 CTAs per SM, against 190 and 2 for whole rows in
// one thread); the halves exchange their partial projections through shared
// memory (two 64-thread named barriers per 32 rows), half 0 forms ww, v_new and
// x, and both take their vectors' dots with ww from the registers they hold.
template <int NS>
__device__ __forceinline__ void cgs_pair_body(const double* const* sp, const double* sc, const double* sy,
                                              double (*acc)[CGS_MAXM + 2], double (*xt)[32], double (*xu)[32],
                                              double (*xw)[32], int m, const double* __restrict__ w,
                                              const double* __restrict__ x0, const double* __restrict__ e,
                                              bool unsafe, bool happy, double inv, int64_t r0, int64_t r1,
                                              double* __restrict__ vnew, double* __restrict__ x, int lane, int pair,
                                              int half, int npairs) {
  const int g0 = half * 32;
  double dot = 0.0, wn2 = 0.0, xn2 = 0.0;
  for (int64_t base = r0 + pair * 32; base < r1; base += 32 * npairs) {
    const int64_t i = base + lane;
    const bool ok = i < r1;
    const int64_t ic = ok ? i : r0;  // rows past the chunk read row r0 and contribute 0
    double v[NS];
#pragma unroll
    for (int g = 0; g < NS; ++g) v[g] = __ldcs(sp[g0 + g] + ic);
    double wi = 0.0, x0i = 0.0, ei = 0.0;
    if (half == 0) wi = w[ic], x0i = x0[ic], ei = e[ic];
    double t = 0.0, u = 0.0;
#pragma unroll
    for (int g = 0; g < NS; ++g) {
      t = fma(sc[g0 + g], v[g], t);
      u = fma(sy[g0 + g], v[g], u);
    }
    if (half == 1) xt[pair][lane] = t, xu[pair][lane] = u;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
    double ww = 0.0;
    if (half == 0) {
      t += xt[pair][lane];
      u += xu[pair][lane];
      ww = wi - t;
      if (ok) {
        if (unsafe) {
          vnew[i] = ww;
        } else {
          if (!happy) vnew[i] = ww * inv;
          const double xi = x0i + (ei + u);
          x[i] = xi;
          xn2 = fma(xi, xi, xn2);
        }
      } else {
        ww = 0.0;
      }
      wn2 = fma(ww, ww, wn2);
      xw[pair][lane] = ww;
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
    if (half == 1) ww = xw[pair][lane];
    if (g0 < m) dot += cgs_fold<NS>(v, ww, lane);
  }
  acc[pair][g0 + lane] = dot;
  if (half == 0) {
    wn2 = warp_sum(wn2);
    xn2 = warp_sum(xn2);
    if (lane == 0) acc[pair][CGS_MAXM] = wn2, acc[pair][CGS_MAXM + 1] = xn2;
  }
}

__global__ void __launch_bounds__(CGS_THREADS)
cgs_update_pair_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ c,
                       const double* __restrict__ y, const double* __restrict__ w, const double* __restrict__ x0,
                       const double* __restrict__ e, const double* __restrict__ state,
                       const double* __restrict__ flag, int64_t n, double* __restrict__ vnew,
                       double* __restrict__ x, double* __restrict__ part) {
  BAMG_PDL_PROLOGUE();
  constexpr int MAXM = 64, PAIRS = CGS_WARPS / 2;
  __shared__ const double* sp[MAXM];
  __shared__ double sc[MAXM], sy[MAXM];
  __shared__ double acc[PAIRS][CGS_MAXM + 2];
  __shared__ double xt[PAIRS][32], xu[PAIRS][32], xw[PAIRS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pair = wid >> 1, half = wid & 1;
  for (int g = threadIdx.x; g < MAXM; g += blockDim.x) {
    sc[g] = g < m ? c[g] : 0.0;
    sy[g] = g < m ? y[g] : 0.0;
  }
  cgs_load_ptrs<MAXM>(Vp, m, sp);
  const bool unsafe = flag[0] == 2.0;
  const bool happy = state[0] != 0.0;
  const double inv = 1.0 / state[1];
  const int64_t per = cgs_chunk_rows(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  // the upper half holds vectors [32, m): the slots it loads are the next multiple of 8 (the
  // branch is uniform per warp; both halves run the same trips and barriers)
  const int mh = half == 0 ? 32 : m - 32;
  if (mh <= 8)
    cgs_pair_body<8>(sp, sc, sy, acc, xt, xu, xw, m, w, x0, e, unsafe, happy, inv, r0, r1, vnew, x, lane, pair, half, PAIRS);
  else if (mh <= 16)
    cgs_pair_body<16>(sp, sc, sy, acc, xt, xu, xw, m, w, x0, e, unsafe, happy, inv, r0, r1, vnew, x, lane, pair, half, PAIRS);
  else if (mh <= 24)
    cgs_pair_body<24>(sp, sc, sy, acc, xt, xu, xw, m, w, x0, e, unsafe, happy, inv, r0, r1, vnew, x, lane, pair, half, PAIRS);
  else
    cgs_pair_body<32>(sp, sc, sy, acc, xt, xu, xw, m, w, x0, e, unsafe, happy, inv, r0, r1, vnew, x, lane, pair, half, PAIRS);
  __syncthreads();
  const int nslots = m + 2;
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) {
    const int slot = q >= m ? CGS_MAXM + (q - m) : q;
    double t = 0.0;
    for (int p = 0; p < PAIRS; ++p) t += acc[p][slot];
    part[(int64_t)blockIdx.x * (m + 2) + q] = t;
  }
}

typedef void (*cgs_update_fn)(const double* const*, int, const double*, const double*, const double*, const double*,
                              const double*, const double*, const double*, int64_t, double*, double*, double*);
static bool cgs_pair_enabled();
static cgs_update_fn cgs_update_select(int m) {
  if (m <= 8) return cgs_update_kernel<32, 8>;
  if (m <= 16) return cgs_update_kernel<32, 16>;
  if (m <= 24) return cgs_update_kernel<32, 24>;
  if (m <= 32) return cgs_update_kernel<32, 32>;
  // m = 33..48: whole rows per thread through 40 / 48 slots (139 / 154 registers, 3 CTAs per SM, no
  // pair barriers) beat the warp-pair split, whose upper half idles there; BAMG_CGS_MID=0 disables
  static const bool mid = !(getenv("BAMG_CGS_MID") && getenv("BAMG_CGS_MID")[0] == '0');
  if (mid && m <= 40) return cgs_update_kernel<64, 40>;
  if (mid && m <= 48) return cgs_update_kernel<64, 48>;
  return cgs_pair_enabled() ? cgs_update_pair_kernel : cgs_update_kernel<64, 64>;
}

// (flag 2 only) the explicit norm |w - V c|^2 = gs[m] for the Givens step
__global__ void cgs_gram_fix_norm_kernel(const double* __restrict__ flag, const double* __restrict__ gs, int m,
                                         double* __restrict__ nrm2) {
  BAMG_PDL_PROLOGUE();
  if (threadIdx.x == 0 && flag[0] == 2.0) nrm2[0] = gs[m];
}

// row / column m of G from gs = V^T ww, |ww|^2 (ww scaled by 1 / state[1] to
// v_new), and |x|: sqrt(gs[m + 1]), or from cgs_fix_x_kernel's partials after
// an explicit-norm step
__global__ void cgs_gram_update_kernel(int m, const double* __restrict__ gs, const double* __restrict__ state,
                                       const double* __restrict__ flag, const double* __restrict__ part_x, int nbx,
                                       double* __restrict__ G, double* __restrict__ xnorm) {
  BAMG_PDL_PROLOGUE();
  __shared__ double red[32];
  const bool unsafe = flag[0] == 2.0;
  const bool happy = state[0] != 0.0;
  const double inv = 1.0 / state[1];
  if (!happy && m < CGS_MAXM) {
    for (int g = threadIdx.x; g < m; g += blockDim.x) {
      const double v = gs[g] * inv;
      G[g * CGS_LDG + m] = v;
      G[m * CGS_LDG + g] = v;
    }
    if (threadIdx.x == 0) G[m * CGS_LDG + m] = gs[m] * inv * inv;
  }
  if (!unsafe) {
    if (threadIdx.x == 0) xnorm[0] = sqrt(gs[m + 1]);
    return;
  }
  double v = 0.0;
  for (int b = threadIdx.x; b < nbx; b += blockDim.x) v += part_x[b];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    xnorm[0] = sqrt(t);
  }
}

// unsafe step, part 1 (one CTA): |w''|^2 from pass C's partials -> the
// normal Givens path (givens_kernel is launched after this by the host loop
// with nrm2 = this value).  No-op when the Pythagorean norm was safe.
__global__ void cgs_fix_norm_kernel(const double* __restrict__ flag, const double* __restrict__ part, int nb,
                                    double* __restrict__ nrm2) {
  BAMG_PDL_PROLOGUE();
  if (flag[0] != 2.0) return;
  __shared__ double red[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[b];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    nrm2[0] = t;
  }
}

// out[0] = sqrt(sum_b part[b]) (fixed order, one CTA)
__global__ void sum_sqrt_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  __shared__ double red[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[b];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[0] = sqrt(t);
  }
}

// unsafe step, part 2: scale v_new by the explicit norm and form x (+ |x|^2
// partials).  No-op when safe.
__global__ void __launch_bounds__(256)
cgs_fix_x_kernel(const double* const* __restrict__ Vp, int m, const double* __restrict__ y,
                 const double* __restrict__ x0, const double* __restrict__ e, const double* __restrict__ state,
                 const double* __restrict__ flag, int64_t n, double* __restrict__ vnew, double* __restrict__ x,
                 double* __restrict__ part) {
  BAMG_PDL_PROLOGUE();
  if (flag[0] != 2.0) return;
  __shared__ double red[8];
  const bool happy = state[0] != 0.0;
  const double inv = 1.0 / state[1];
  const int64_t per = cgs_chunk_rows(n, gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  double nrm = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double u = 0.0;
    for (int g = 0; g < m; ++g) u = fma(y[g], Vp[g][i], u);
    const double xi = x0[i] + (e[i] + u);
    x[i] = xi;
    nrm = fma(xi, xi, nrm);
    if (!happy) vnew[i] *= inv;
  }
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

struct GmresWork {
  std::vector<double*> basis;     // device vectors (owned)
  double** dVp = nullptr;         // device pointer table
  size_t cap = 0;
  size_t uploaded = 0;
  int64_t n = 0;
};

static int basis_reserve(bamg_ctx* ctx, GmresWork& W, int64_t n, int count) {
  if (W.n != n) {
    for (double* p : W.basis) cudaFree(p);
    W.basis.clear();
    W.n = n;
    W.uploaded = 0;
  }
  if ((int)W.basis.size() >= count && W.uploaded >= W.basis.size()) return 0;
  // grow in chunks of 8 vectors so allocation stays off the per-iteration path
  int target = ((count + 7) / 8) * 8;
  while ((int)W.basis.size() < target) {
    double* p = nullptr;
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&p, sizeof(double) * (n > 0 ? n : 1)));
    W.basis.push_back(p);
  }
  if (W.cap < W.basis.size()) {
    if (W.dVp) {
      BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFree(W.dVp);
    }
    W.cap = W.basis.size() + 32;
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&W.dVp, sizeof(double*) * W.cap));
  }
  // the host table must stay alive until the copy lands: synchronous copy
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaMemcpy(W.dVp, W.basis.data(), sizeof(double*) * W.basis.size(),
                                  cudaMemcpyHostToDevice));
  W.uploaded = W.basis.size();
  return 0;
}

static int cgs_grid(bamg_ctx* ctx, const void* fn, int64_t n) {
  static std::vector<std::pair<const void*, int>> occ;  // per kernel (one device per process in practice)
  int per_sm = 0;
  for (auto& e : occ)
    if (e.first == fn) per_sm = e.second;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, CGS_THREADS, 0) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    occ.push_back({fn, per_sm});
  }
  const int64_t by_rows = (n + 4 * CGS_THREADS - 1) / (4 * CGS_THREADS);
  const int64_t g = std::min<int64_t>((int64_t)per_sm * ctx->num_sms, std::max<int64_t>(by_rows, 1));
  return (int)std::min<int64_t>(g, CGS_MAX_BLOCKS);
}

static void cgs_apply_env() {
  static bool done = false;
  if (done) return;
  done = true;
  const char* e = getenv("BAMG_CGS_ALWAYS_REORTH");
  const bool v = e && e[0] == '1';
  cudaMemcpyToSymbol(cgs_force_two_pass, &v, sizeof(bool));
}

// BAMG_CGS_GRAM=0: the three-pass CGS2 (explicit second projection) instead of the Gram form
static bool cgs_gram_enabled() {
  const char* e = getenv("BAMG_CGS_GRAM");
  return !(e && e[0] == '0');
}

static bool cgs_pair_enabled() {  // BAMG_CGS_PAIR=0: whole rows per thread for m > 32 (development)
  static const bool on = !(getenv("BAMG_CGS_PAIR") && getenv("BAMG_CGS_PAIR")[0] == '0');
  return on;
}

static bool cgs_fast_enabled() {
  static const bool on = !(getenv("BAMG_CGS_SLOW") && getenv("BAMG_CGS_SLOW")[0] == '1');
  return on;
}

static GmresWork& gmres_work(bamg_ctx* ctx) {
  if (!ctx->gmres_work) ctx->gmres_work = new GmresWork();
  return *ctx->gmres_work;
}

void gmres_work_release(bamg_ctx* ctx) {
  GmresWork* W = ctx->gmres_work;
  if (!W) return;
  for (double* p : W->basis) cudaFree(p);
  if (W->dVp) cudaFree(W->dVp);
  delete W;
  ctx->gmres_work = nullptr;
}

static int apply_op(bamg_ctx* ctx, const bamg_csr* B, bamg_hier* h, const double* v, double* tmp,
                    double* out) {
  if (h) {
    BAMG_TRY(spmm_dev(ctx, B, v, tmp, 1));
    return vcycle_run(ctx, h, tmp, out);
  }
  return spmm_dev(ctx, B, v, out, 1);
}

extern "C" int bamg_dense_gemv(bamg_ctx* ctx, const double* Z, int n, const double* b, double* y) {
  BAMG_LAUNCH(ctx, gemv_rowmajor_kernel, grid_for((int64_t)n * 32, 256), 256, 0, n, Z, b, y);
  return 0;
}

extern "C" int bamg_gmres(bamg_ctx* ctx, const bamg_csr* B, bamg_hier* h, const double* b,
                          const double* x0, double* x, int restart, int max_iters, double rtol,
                          int stopping, int* iters_host, double* history_host, int* nhistory_host) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, B && B->nrows == B->ncols, "square operator expected");
  BAMG_REQUIRE(ctx, max_iters >= 0, "max_iters must be nonnegative");
  cgs_apply_env();
  const int64_t n = B->nrows;
  const int nb = GM_BLOCKS;
  // workspace
  double *tmp, *w, *e, *rhs, *r, *R, *g, *cs, *sn, *y, *hv, *h2, *part, *scal, *state;
  int m_cap = (restart > 0 ? restart : max_iters);
  if (m_cap > max_iters) m_cap = max_iters;
  if (m_cap < 1) m_cap = 1;
  BAMG_TRY(arena_get(ctx, n, &tmp));
  BAMG_TRY(arena_get(ctx, n, &w));
  BAMG_TRY(arena_get(ctx, n, &e));
  BAMG_TRY(arena_get(ctx, n, &rhs));
  BAMG_TRY(arena_get(ctx, n, &r));
  BAMG_TRY(arena_get(ctx, (size_t)m_cap * m_cap, &R));
  BAMG_TRY(arena_get(ctx, m_cap + 1, &g));
  BAMG_TRY(arena_get(ctx, m_cap, &cs));
  BAMG_TRY(arena_get(ctx, m_cap, &sn));
  BAMG_TRY(arena_get(ctx, m_cap, &y));
  BAMG_TRY(arena_get(ctx, m_cap + 2, &hv));
  BAMG_TRY(arena_get(ctx, m_cap + 2, &h2));
  BAMG_TRY(arena_get(ctx, std::max((size_t)nb * (m_cap + 2), (size_t)CGS_MAX_BLOCKS * (CGS_MAXM + 2)), &part));
  BAMG_TRY(arena_get(ctx, 8, &scal));
  BAMG_TRY(arena_get(ctx, 4, &state));
  double *flag, *gram, *gsum;
  BAMG_TRY(arena_get(ctx, 2, &flag));
  BAMG_TRY(arena_get(ctx, (size_t)CGS_LDG * CGS_LDG, &gram));
  BAMG_TRY(arena_get(ctx, CGS_MAXM + 2, &gsum));
  GmresWork& W = gmres_work(ctx);
  const int blk = 256;
  const int grd = grid_for(n, blk);

  auto norm_into = [&](const double* v, double* out) -> int {
    return colreduce(ctx, v, nullptr, n, 1, 0, out, 1);
  };
  double denom0 = 1.0;
  // stopping 0: ||Bx|| / ||x||  ("scaled_bx");  1: ||b - Bx|| / max(||b - Bx0||, 1e-300)
  auto metric = [&](const double* xv, double* out_host) -> int {
    if (stopping == 1) {
      BAMG_TRY(resid_dev(ctx, B, b, xv, tmp));
      BAMG_TRY(norm_into(tmp, scal));
      double r0;
      BAMG_TRY(ctx_read_doubles(ctx, scal, 1, &r0));
      *out_host = r0 / denom0;
      return 0;
    }
    BAMG_TRY(spmm_dev(ctx, B, xv, tmp, 1));
    BAMG_TRY(norm_into(tmp, scal));
    BAMG_TRY(norm_into(xv, scal + 1));
    double hv2[2];
    BAMG_TRY(ctx_read_doubles(ctx, scal, 2, hv2));
    *out_host = hv2[1] == 0.0 ? INFINITY : hv2[0] / hv2[1];
    return 0;
  };
  // the iteration's metric and Givens state (happy flag) in ONE read
  double last_code = -1.0;  // the step's CGS code, read with the metric
  // x_norm_ready: |x| already in scal[1] (the CGS fast path forms it with x)
  auto metric_state = [&](const double* xv, double* out_host, bool* happy, bool x_norm_ready) -> int {
    if (stopping == 1) {
      BAMG_TRY(resid_dev(ctx, B, b, xv, tmp));
      BAMG_TRY(norm_into(tmp, scal));
    } else {
      BAMG_TRY(spmm_dev(ctx, B, xv, tmp, 1));
      BAMG_TRY(norm_into(tmp, scal));
      if (!x_norm_ready) BAMG_TRY(norm_into(xv, scal + 1));
    }
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(scal + 4, state, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(scal + 5, flag, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    double hv3[6];
    BAMG_TRY(ctx_read_doubles(ctx, scal, 6, hv3));
    last_code = hv3[5];
    if (stopping == 1) *out_host = hv3[0] / denom0;
    else *out_host = hv3[1] == 0.0 ? INFINITY : hv3[0] / hv3[1];
    *happy = hv3[4] != 0.0;
    return 0;
  };
  if (stopping == 1) {
    BAMG_TRY(resid_dev(ctx, B, b, x0, tmp));
    BAMG_TRY(norm_into(tmp, scal));
    double r0;
    BAMG_TRY(ctx_read_doubles(ctx, scal, 1, &r0));
    denom0 = r0 > 1e-300 ? r0 : 1e-300;
  }

  int nhist = 0;
  double m0;
  BAMG_TRY(metric(x0, &m0));
  history_host[nhist++] = m0;
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  *iters_host = 0;
  if (m0 <= rtol) {
    *nhistory_host = nhist;
    return 0;
  }
  // rhs = C(b - B x0)
  BAMG_TRY(spmm_dev(ctx, B, x0, tmp, 1));
  BAMG_LAUNCH(ctx, axpby_kernel, grd, blk, 0, n, b, tmp, w);
  if (h) {
    BAMG_TRY(vcycle_run(ctx, h, w, rhs));
  } else {
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(rhs, w, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(e, 0, sizeof(double) * n, ctx->stream));

  int iters = 0;
  int one_pass_steps = 0;  // Arnoldi steps that took the single projection (DGKS)
  int explicit_norm_steps = 0;  // Gram-path steps that fell back to the explicit norm
  bool converged = false;
  bool first_cycle = true;
  while (iters < max_iters && !converged) {
    // r = rhs - op(e)
    if (first_cycle) {
      BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(r, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      BAMG_TRY(apply_op(ctx, B, h, e, w, tmp));
      BAMG_LAUNCH(ctx, axpby_kernel, grd, blk, 0, n, rhs, tmp, r);
    }
    first_cycle = false;
    double beta;
    BAMG_TRY(norm_into(r, scal + 2));
    BAMG_TRY(ctx_read_doubles(ctx, scal + 2, 1, &beta));
    if (beta == 0.0) break;
    int m = (restart > 0 ? restart : max_iters);
    if (m > max_iters - iters) m = max_iters - iters;
    BAMG_TRY(basis_reserve(ctx, W, n, 1));
    BAMG_LAUNCH(ctx, scale_div_kernel, grd, blk, 0, n, r, scal + 2, W.basis[0]);
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(R, 0, sizeof(double) * (size_t)m_cap * m_cap, ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(g, 0, sizeof(double) * (m_cap + 1), ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(g, scal + 2, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    int used = 0;
    bool broke = false;
    for (int j = 0; j < m; ++j) {
      BAMG_TRY(basis_reserve(ctx, W, n, j + 2));
      // w = op(V_j)
      BAMG_TRY(apply_op(ctx, B, h, W.basis[j], tmp, w));
      if (j + 1 <= CGS_MAXM && cgs_fast_enabled() && cgs_gram_enabled()) {
        // two passes over V (see cgs_gram_coef_kernel): dots, then the update with x, |x| and G's new row
        const int mj = j + 1;
        if (j == 0) BAMG_LAUNCH(ctx, cgs_gram_init_kernel, 1, 256, 0, gram);
        auto dots = cgs_dots_kernel<32, 0>;
        auto upd = cgs_update_select(mj);
        // pass A in vector groups of 32 (one wave in total); the update pass keeps whole rows
        const int groups = (mj + 31) / 32;
        const int cbd = std::max(1, cgs_grid(ctx, (const void*)dots, n) / groups);
        const int cb = cgs_grid(ctx, (const void*)upd, n);
        BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (mj + groups) * n, dots, cbd * groups, CGS_THREADS, 0,
                        (const double* const*)W.dVp, mj, (const double*)nullptr, w, n, part, (const double*)nullptr, cbd);
        BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(mj + 1) * 32, 256), 256, 0, (const double*)part, cbd,
                    mj + 1, mj + 1, hv, (const double*)nullptr, 0u);  // h1 and |w|^2
        BAMG_LAUNCH(ctx, cgs_gram_coef_kernel, 1, CGS_MAXM, 0, mj, (const double*)gram, hv, h2, scal + 3, flag);
        BAMG_LAUNCH(ctx, givens_kernel, 1, 256, sizeof(double) * (j + 2), j, m_cap, hv, scal + 3, beta, R, g, cs, sn,
                    y, state, (const double*)flag, 0b011u);
        BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (mj + 5) * n, upd, cb, CGS_THREADS, 0, (const double* const*)W.dVp, mj,
                        (const double*)h2, (const double*)y, (const double*)w, x0, (const double*)e,
                        (const double*)state, (const double*)flag, n, W.basis[j + 1], x, part);
        BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(mj + 2) * 32, 256), 256, 0, (const double*)part, cb,
                    mj + 2, mj + 2, gsum, (const double*)nullptr, 0u);  // V^T ww, |ww|^2, |x|^2
        BAMG_LAUNCH(ctx, cgs_gram_fix_norm_kernel, 1, 32, 0, (const double*)flag, (const double*)gsum, mj, scal + 3);
        BAMG_LAUNCH(ctx, givens_kernel, 1, 256, sizeof(double) * (j + 2), j, m_cap, hv, scal + 3, beta, R, g, cs, sn,
                    y, state, (const double*)flag, 0b100u);
        BAMG_LAUNCH(ctx, cgs_fix_x_kernel, cb, 256, 0, (const double* const*)W.dVp, mj, (const double*)y, x0,
                    (const double*)e, (const double*)state, (const double*)flag, n, W.basis[j + 1], x, part);
        BAMG_LAUNCH(ctx, cgs_gram_update_kernel, 1, 256, 0, mj, (const double*)gsum, (const double*)state,
                    (const double*)flag, (const double*)part, cb, gram, scal + 1);
        ++iters;
        used = j + 1;
        double mval;
        bool happy = false;
        BAMG_TRY(metric_state(x, &mval, &happy, true));
        if (last_code == 2.0) ++explicit_norm_steps;
        history_host[nhist++] = mval;
        if (mval <= rtol) converged = true;
        if (converged || happy || iters >= max_iters) {
          if (happy) converged = true;
          BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, used, y, nullptr, e, nullptr, n, tmp);
          BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(e, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
          broke = true;
          break;
        }
        continue;
      }
      if (j + 1 <= CGS_MAXM && cgs_fast_enabled()) {
        // three passes over V (see cgs_dots_kernel); x and |x| formed in pass C
        const int mj = j + 1;
        auto dots = mj <= 32 ? cgs_dots_kernel<32, 0> : cgs_dots_kernel<64, 0>;
        auto upd = mj <= 32 ? cgs_dots_kernel<32, 1> : cgs_dots_kernel<64, 1>;
        auto fin = mj <= 16 ? cgs_final_kernel<16> : mj <= 32 ? cgs_final_kernel<32> : cgs_final_kernel<64>;  // NOLINT
        // one full wave: resident CTAs per SM x SMs (register-bound kernels),
        // capped so every CTA keeps >= 4 row batches; a fixed function of
        // (n, kernel, device), so the partial-sum tree is reproducible
        const int cb = std::min(cgs_grid(ctx, (const void*)upd, n), cgs_grid(ctx, (const void*)fin, n));
        BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (mj + 1) * n, dots, cb, CGS_THREADS, 0, (const double* const*)W.dVp, mj,
                        (const double*)nullptr, w, n, part, (const double*)nullptr, cb);
        BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(mj + 1) * 32, 256), 256, 0, (const double*)part, cb,
                    mj + 1, mj + 1, hv, (const double*)nullptr, 0u);  // h and |w|^2
        BAMG_LAUNCH(ctx, cgs_dgks_kernel, 1, 256, 0, mj, (const double*)hv, scal + 3, flag, h2);
        // second projection (code 0 only; its bytes are booked after the step's read-back)
        BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 0.0, upd, cb, CGS_THREADS, 0, (const double* const*)W.dVp, mj,
                        (const double*)hv, w, n, part, (const double*)flag, cb);
        BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(mj + 1) * 32, 256), 256, 0, (const double*)part, cb,
                    mj + 1, mj + 1, h2, (const double*)flag, 1u);
        BAMG_LAUNCH(ctx, cgs_pythag_kernel, 1, 256, 0, mj, (const double*)h2, hv, scal + 3, flag);
        BAMG_LAUNCH(ctx, givens_kernel, 1, 256, sizeof(double) * (j + 2), j, m_cap, hv, scal + 3, beta, R, g, cs, sn,
                    y, state, (const double*)flag, 0b011u);
        BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (mj + 5) * n, fin, cb, CGS_THREADS, 0, (const double* const*)W.dVp, mj,
                        (const double*)h2, (const double*)hv, (const double*)y, (const double*)w, x0, (const double*)e,
                        (const double*)state, (const double*)flag, n, W.basis[j + 1], x, part);
        BAMG_LAUNCH(ctx, cgs_fix_norm_kernel, 1, 256, 0, (const double*)flag, (const double*)part, cb, scal + 3);
        BAMG_LAUNCH(ctx, givens_kernel, 1, 256, sizeof(double) * (j + 2), j, m_cap, hv, scal + 3, beta, R, g, cs, sn,
                    y, state, (const double*)flag, 0b100u);
        BAMG_LAUNCH(ctx, cgs_fix_x_kernel, cb, 256, 0, (const double* const*)W.dVp, mj, (const double*)y, x0,
                    (const double*)e, (const double*)state, (const double*)flag, n, W.basis[j + 1], x, part);
        BAMG_LAUNCH(ctx, sum_sqrt_kernel, 1, 256, 0, (const double*)part, cb, scal + 1);
        ++iters;
        used = j + 1;
        double mval;
        bool happy = false;
        BAMG_TRY(metric_state(x, &mval, &happy, true));
        if (last_code != 1.0 && ((ctx->prof.mask >> FAM_ORTHO) & 1u))  // the second projection ran
          ctx->prof.bytes[FAM_ORTHO] += 8.0 * (mj + 2) * n;
        if (last_code == 1.0) ++one_pass_steps;
        history_host[nhist++] = mval;
        if (mval <= rtol) converged = true;
        if (converged || happy || iters >= max_iters) {
          if (happy) converged = true;
          BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, used, y, nullptr, e, nullptr, n, tmp);
          BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(e, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
          broke = true;
          break;
        }
        continue;
      }
      // CGS2: h = V^T w ; w -= V h ; h2 = V^T w ; w -= V h2 ; |w|^2
      BAMG_LAUNCH(ctx, mdot_kernel, nb, GM_THREADS, 0, W.dVp, j + 1, w, n, part);
      BAMG_LAUNCH(ctx, mreduce_kernel, grid_for((int64_t)(j + 1) * 32, 256), 256, 0, part, nb, j + 1, hv, 0);
      BAMG_LAUNCH(ctx, mupdate_kernel<0>, nb, GM_THREADS, 0, W.dVp, j + 1, hv, w, n, part);
      BAMG_LAUNCH(ctx, mdot_kernel, nb, GM_THREADS, 0, W.dVp, j + 1, w, n, part);
      BAMG_LAUNCH(ctx, mreduce_kernel, grid_for((int64_t)(j + 1) * 32, 256), 256, 0, part, nb, j + 1, h2, 0);
      BAMG_LAUNCH(ctx, mupdate_kernel<2>, nb, GM_THREADS, 0, W.dVp, j + 1, h2, w, n, part);
      BAMG_LAUNCH(ctx, mreduce_kernel, 1, 32, 0, part, nb, 1, scal + 3, 0);
      // h += h2 (length j+1) via the reduce kernel's accumulate path
      BAMG_LAUNCH(ctx, mreduce_kernel, grid_for((int64_t)(j + 1) * 32, 256), 256, 0, h2, 1, j + 1, hv, 1);
      BAMG_LAUNCH(ctx, givens_kernel, 1, 256, sizeof(double) * (j + 2), j, m_cap, hv, scal + 3, beta, R, g, cs, sn, y,
                  state, (const double*)nullptr, 0u);
      BAMG_LAUNCH(ctx, scale_new_basis_kernel, grd, blk, 0, w, state, n, W.basis[j + 1]);
      ++iters;
      used = j + 1;
      // x = x0 + (e + V y)
      BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, used, y, x0, e, nullptr, n, x);
      double mval;
      bool happy = false;
      BAMG_TRY(metric_state(x, &mval, &happy, false));
      history_host[nhist++] = mval;
      if (mval <= rtol) converged = true;
      if (converged || happy || iters >= max_iters) {
        if (happy) converged = true;
        BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, used, y, nullptr, e, nullptr, n, tmp);
        BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(e, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        broke = true;
        break;
      }
    }
    if (!broke) {
      // restart: e += V y (y of the last column is still current)
      BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, used, y, nullptr, e, nullptr, n, tmp);
      BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(e, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
      BAMG_LAUNCH(ctx, combine_kernel, grd, blk, 0, W.dVp, 0, y, x0, e, nullptr, n, x);
    }
  }
  *iters_host = iters;
  *nhistory_host = nhist;
  if (getenv("BAMG_DEBUG"))
    fprintf(stderr, "[bamg] gmres: %d iterations, %d with one projection (DGKS), %d with the explicit norm\n", iters,
            one_pass_steps, explicit_norm_steps);
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return converged ? 0 : 1;
}

// ===================================================== sign fix + l1 norm
// stats: [0] max|x| (bits), [1] first index of the max, [2] sum|x|,
// [3] non-finite flag
__global__ void signfix_extract_kernel(const double* __restrict__ x, int64_t n, int stride,
                                       double* __restrict__ out, unsigned long long* __restrict__ flags) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i * stride];
  out[i] = v;
  if (!isfinite(v)) atomicOr(flags, 1ull);
}

__global__ void absstats_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ psum,
                                        double* __restrict__ pmax, long long* __restrict__ pidx) {
  BAMG_PDL_PROLOGUE();
  __shared__ double ss[256], sm[256];
  __shared__ long long si[256];
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  double s = 0.0, mx = -1.0;
  long long mi = -1;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double a = fabs(x[i]);
    s += a;
    if (a > mx) {
      mx = a;
      mi = i;
    }
  }
  ss[threadIdx.x] = s;
  sm[threadIdx.x] = mx;
  si[threadIdx.x] = mi;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      ss[threadIdx.x] += ss[threadIdx.x + off];
      double m2 = sm[threadIdx.x + off];
      long long i2 = si[threadIdx.x + off];
      if (m2 > sm[threadIdx.x] || (m2 == sm[threadIdx.x] && i2 >= 0 && (si[threadIdx.x] < 0 || i2 < si[threadIdx.x]))) {
        sm[threadIdx.x] = m2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    psum[blockIdx.x] = ss[0];
    pmax[blockIdx.x] = sm[0];
    pidx[blockIdx.x] = si[0];
  }
}

__global__ void absstats_final_kernel(int nb, const double* psum, const double* pmax, const long long* pidx,
                                      double* stats) {
  BAMG_PDL_PROLOGUE();
  if (threadIdx.x != 0) return;
  double s = 0.0, mx = -1.0;
  long long mi = -1;
  for (int b = 0; b < nb; ++b) {
    s += psum[b];
    if (pmax[b] > mx) {
      mx = pmax[b];
      mi = pidx[b];
    }
  }
  stats[0] = mx;
  stats[1] = (double)mi;
  stats[2] = s;
}

__global__ void uniform_fill_kernel(double* out, int64_t n, const unsigned long long* flags,
                                    const double* stats) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (flags[0] != 0ull || stats[2] == 0.0) out[i] = 1.0 / (double)n;
}

__global__ void signfix_apply_kernel(double* out, int64_t n, const double* stats) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long pk = (long long)stats[1];
  double v = out[i];
  // stats computed on the current contents; peak value sign decides
  double sgn_src = stats[3];
  if (sgn_src < 0.0) v = -v;
  double tot = stats[2];
  out[i] = tot > 0.0 ? v / tot : v;
  (void)pk;
}

__global__ void peak_sign_kernel(const double* out, double* stats) {
  BAMG_PDL_PROLOGUE();
  long long pk = (long long)stats[1];
  stats[3] = pk >= 0 ? out[pk] : 1.0;
}

static int absstats(bamg_ctx* ctx, const double* x, int64_t n, double* stats) {
  double *psum, *pmax;
  long long* pidx;
  BAMG_TRY(arena_get(ctx, RED_BLOCKS, &psum));
  BAMG_TRY(arena_get(ctx, RED_BLOCKS, &pmax));
  BAMG_TRY(arena_get(ctx, RED_BLOCKS, &pidx));
  BAMG_LAUNCH(ctx, absstats_partial_kernel, RED_BLOCKS, 256, 0, x, n, psum, pmax, pidx);
  BAMG_LAUNCH(ctx, absstats_final_kernel, 1, 32, 0, RED_BLOCKS, psum, pmax, pidx, stats);
  return 0;
}

extern "C" int bamg_sign_fix_l1(bamg_ctx* ctx, const double* x, int64_t n, int stride, double* out,
                                int uniform_fallback) {
  ctx->arena.reset();
  unsigned long long* flags;
  double* stats;
  BAMG_TRY(arena_get(ctx, 1, &flags));
  BAMG_TRY(arena_get(ctx, 4, &stats));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(flags, 0, sizeof(*flags), ctx->stream));
  BAMG_LAUNCH(ctx, signfix_extract_kernel, grid_for(n, 256), 256, 0, x, n, stride, out, flags);
  BAMG_TRY(absstats(ctx, out, n, stats));
  if (uniform_fallback) {
    BAMG_LAUNCH(ctx, uniform_fill_kernel, grid_for(n, 256), 256, 0, out, n, flags, stats);
    BAMG_TRY(absstats(ctx, out, n, stats));
  }
  BAMG_LAUNCH(ctx, peak_sign_kernel, 1, 1, 0, out, stats);
  BAMG_LAUNCH(ctx, signfix_apply_kernel, grid_for(n, 256), 256, 0, out, n, stats);
  return 0;
}

// ===================================================== distributed building blocks
// Rank-local pieces of the V-cycle and of CGS2 for the row-partitioned solve
// (paper_1402_4005_b200/distributed.py): the operators carry halo-extended
// column numbering, dot products are local partial sums the caller all-reduces.
extern "C" int bamg_residual(bamg_ctx* ctx, const bamg_csr* A, const double* b, const double* x, double* r) {
  return resid_dev(ctx, A, b, x, r);
}

extern "C" int bamg_addmv(bamg_ctx* ctx, const bamg_csr* A, const double* xc, const double* xold, double* y) {
  return addmv_dev(ctx, A, xc, xold, y, 1);
}

extern "C" int bamg_jacobi_zero(bamg_ctx* ctx, int64_t n, const double* b, const double* d, const uint8_t* skip,
                                double omega, double* x) {
  return jacobi_from_zero(ctx, n, b, d, skip, omega, x);
}

extern "C" int bamg_dense_gemv_rows(bamg_ctx* ctx, const double* Z, int n, const double* b, double* y) {
  BAMG_LAUNCH(ctx, gemv_rowmajor_kernel, grid_for((int64_t)n * 32, 256), 256, 0, n, Z, b, y);
  return 0;
}

// out[i] = V_i . w  (local partial sums), i < m
extern "C" int bamg_mdot(bamg_ctx* ctx, const double* const* Vp, int m, const double* w, int64_t n, double* out) {
  ctx->arena.reset();
  double* part;
  BAMG_TRY(arena_get(ctx, (size_t)GM_BLOCKS * (m > 0 ? m : 1), &part));
  BAMG_LAUNCH(ctx, mdot_kernel, GM_BLOCKS, GM_THREADS, 0, Vp, m, w, n, part);
  BAMG_LAUNCH(ctx, mreduce_kernel, grid_for((int64_t)m * 32, 256), 256, 0, part, GM_BLOCKS, m, out, 0);
  return 0;
}

// w -= sum_i c_i V_i ; nrm2 (optional) = |w_new|^2 local partial
extern "C" int bamg_mupdate(bamg_ctx* ctx, const double* const* Vp, int m, const double* c, double* w, int64_t n,
                            double* nrm2) {
  ctx->arena.reset();
  double* part;
  BAMG_TRY(arena_get(ctx, (size_t)GM_BLOCKS + 1, &part));
  if (nrm2) {
    BAMG_LAUNCH(ctx, mupdate_kernel<2>, GM_BLOCKS, GM_THREADS, 0, Vp, m, c, w, n, part);
    BAMG_LAUNCH(ctx, mreduce_kernel, 1, 32, 0, part, GM_BLOCKS, 1, nrm2, 0);
  } else {
    BAMG_LAUNCH(ctx, mupdate_kernel<0>, GM_BLOCKS, GM_THREADS, 0, Vp, m, c, w, n, part);
  }
  return 0;
}

// ---- rank-local passes of the two-pass (Gram) CGS2 step for the row-partitioned solve
// (distributed.py): the same fused kernels bamg_gmres runs, on the caller's row block, with
// the partial sums left for the caller's all-reduce between them.
__global__ void cgs_set_state_kernel(double* __restrict__ state, double* __restrict__ flag, double happy,
                                     double norm, double code) {
  BAMG_PDL_PROLOGUE();
  state[0] = happy;
  state[1] = norm;
  flag[0] = code;
}

// out[0..m) = V^T w, out[m] = |w|^2 over the n local rows (m <= 64)
extern "C" int bamg_cgs_dots(bamg_ctx* ctx, const double* const* Vp, int m, const double* w, int64_t n,
                             double* out) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, m >= 1 && m <= CGS_MAXM, "1..64 basis vectors per fused pass");
  double* part;
  BAMG_TRY(arena_get(ctx, (size_t)CGS_MAX_BLOCKS * (CGS_MAXM + 2), &part));
  auto dots = cgs_dots_kernel<32, 0>;
  const int groups = (m + 31) / 32;
  const int cbd = std::max(1, cgs_grid(ctx, (const void*)dots, n) / groups);
  BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (m + groups) * n, dots, cbd * groups, CGS_THREADS, 0, Vp, m,
                  (const double*)nullptr, const_cast<double*>(w), n, part, (const double*)nullptr, cbd);
  BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(m + 1) * 32, 256), 256, 0, (const double*)part, cbd, m + 1,
              m + 1, out, (const double*)nullptr, 0u);
  return 0;
}

// ww = w - V c; vnew = ww * inv_norm (skipped when happy != 0); x = x0 + e + V y;
// out[0..m) = V^T ww, out[m] = |ww|^2, out[m + 1] = |x|^2 over the n local rows
extern "C" int bamg_cgs_update(bamg_ctx* ctx, const double* const* Vp, int m, const double* c, const double* y,
                               const double* w, const double* x0, const double* e, double inv_norm, int happy,
                               int64_t n, double* vnew, double* x, double* out) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, m >= 1 && m <= CGS_MAXM, "1..64 basis vectors per fused pass");
  double *part, *st;
  BAMG_TRY(arena_get(ctx, (size_t)CGS_MAX_BLOCKS * (CGS_MAXM + 2), &part));
  BAMG_TRY(arena_get(ctx, 4, &st));
  BAMG_LAUNCH(ctx, cgs_set_state_kernel, 1, 1, 0, st, st + 2, happy ? 1.0 : 0.0, 1.0 / inv_norm, 0.0);
  auto upd = cgs_update_select(m);
  const int cb = cgs_grid(ctx, (const void*)upd, n);
  BAMG_LAUNCH_FAM(ctx, FAM_ORTHO, 8.0 * (m + 5) * n, upd, cb, CGS_THREADS, 0, Vp, m, c, y, w, x0, e,
                  (const double*)st, (const double*)(st + 2), n, vnew, x, part);
  BAMG_LAUNCH(ctx, cgs_reduce_kernel, grid_for((int64_t)(m + 2) * 32, 256), 256, 0, (const double*)part, cb, m + 2,
              m + 2, out, (const double*)nullptr, 0u);
  return 0;
}

// out = base + add + sum_i y_i V_i   (base / add may be NULL)
extern "C" int bamg_combine(bamg_ctx* ctx, const double* const* Vp, int m, const double* y, const double* base,
                            const double* add, int64_t n, double* out) {
  BAMG_LAUNCH(ctx, combine_kernel, grid_for(n, 256), 256, 0, Vp, m, y, base, add, nullptr, n, out);
  return 0;
}
