// coarsen.cu -- C/F splitting on device (coarsen.py:23-176).
//
// Geometric mode: axis ranks among distinct coordinate values (np.unique
// return_inverse) by an LSD radix sort that only visits the key bits that
// actually vary, then "every rank even".  Coarse levels re-rank exactly by a
// presence scan over the parent ranks of the kept points (the distinct values
// on the coarse level are a subset of the parent's, order preserved).
//
// Compatible relaxation (cr_coarsen): per pass the host supplies the seeded
// standard-normal draw for the fine points (numpy PCG64 stream; the only
// host-generated input), the device does unit-RMS scaling, the F-relaxation
// sweeps (bit-exact CSR-stream SpMV), mu = min(|x|, 1e6)^(1/sweeps), the
// candidate test and the greedy maximal independent set in (-mu, index)
// order.  The sequential greedy is reproduced exactly by the parallel
// lexicographically-first MIS: a candidate joins when every higher-priority
// candidate neighbour is out, and leaves when any of them is in.
#include <cmath>

#include "internal.cuh"

// ------------------------------------------------------------ radix ranks
__device__ __forceinline__ unsigned long long order_key(double v) {
  if (v == 0.0) v = 0.0;  // -0.0 == 0.0 for np.unique
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void keys_init_kernel(const double* __restrict__ coord, int64_t n, unsigned long long* __restrict__ key,
                                 int32_t* __restrict__ idx, unsigned long long* orand) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned long long so[256], sa[256];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long k = 0ull, a = ~0ull;
  if (i < n) {
    k = order_key(coord[i]);
    key[i] = k;
    idx[i] = (int32_t)i;
    a = k;
  }
  so[threadIdx.x] = k;
  sa[threadIdx.x] = a;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      so[threadIdx.x] |= so[threadIdx.x + off];
      sa[threadIdx.x] &= sa[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicOr(&orand[0], so[0]);
    atomicAnd(&orand[1], sa[0]);
  }
}

__global__ void bit_flags_kernel(const unsigned long long* __restrict__ key, int64_t n, int bit,
                                 uint8_t* __restrict__ zero) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) zero[i] = ((key[i] >> bit) & 1ull) ? 0 : 1;
}

__global__ void bit_scatter_kernel(const unsigned long long* __restrict__ key, const int32_t* __restrict__ idx,
                                   int64_t n, int bit, const int32_t* __restrict__ zpos,
                                   unsigned long long* __restrict__ key2, int32_t* __restrict__ idx2) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t nz = zpos[n];
  unsigned long long k = key[i];
  int64_t dst = ((k >> bit) & 1ull) ? nz + (i - zpos[i]) : zpos[i];
  key2[dst] = k;
  idx2[dst] = idx[i];
}

__global__ void distinct_flags_kernel(const unsigned long long* __restrict__ key, int64_t n, uint8_t* __restrict__ f) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = (i > 0 && key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void rank_scatter_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ pos, const uint8_t* __restrict__ f,
                                    int64_t n, int32_t* __restrict__ rank) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rank[idx[i]] = pos[i] + f[i];  // inclusive count of "new value" flags
}

// Integer-coordinate fast path (lattice chains store grid positions): when
// every value is an integer in [0, 2^24), np.unique's inverse is the prefix
// count of the present values -- presence flags, one scan, one gather -- in
// place of the 64-bit LSD radix sort (~3 launches per varying key bit).
constexpr int64_t INT_RANK_MAX = 1 << 24;

__global__ void int_probe_kernel(const double* __restrict__ coord, int64_t n, unsigned int* __restrict__ probe) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool ok = true;
  int v = 0;
  if (i < n) {
    const double x = coord[i];
    ok = x >= 0.0 && x < (double)INT_RANK_MAX && x == floor(x);
    v = ok ? (int)x : 0;
  }
  if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(probe, 1u);
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(probe + 1, (unsigned)v);
}

__global__ void int_presence_kernel(const double* __restrict__ coord, int64_t n, uint8_t* __restrict__ present) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) present[(int)coord[i]] = 1;
}

__global__ void int_rank_kernel(const double* __restrict__ coord, int64_t n, const int32_t* __restrict__ pos,
                                int32_t* __restrict__ rank) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rank[i] = pos[(int)coord[i]];
}

extern "C" int bamg_axis_ranks(bamg_ctx* ctx, const double* coord, int64_t n, int32_t* rank, int64_t* nvalues_host) {
  ctx->arena.reset();
  if (nvalues_host) *nvalues_host = 0;
  if (n == 0) return 0;
  {
    unsigned int* probe;
    BAMG_TRY(arena_get(ctx, 2, &probe));
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(probe, 0, 2 * sizeof(unsigned int), ctx->stream));
    BAMG_LAUNCH(ctx, int_probe_kernel, grid_for(n, 256), 256, 0, coord, n, probe);
    unsigned int pr[2];
    BAMG_TRY(ctx_read_i32(ctx, reinterpret_cast<const int32_t*>(probe), 2, reinterpret_cast<int32_t*>(pr)));
    if (pr[0] == 0u) {
      const int64_t R = (int64_t)pr[1] + 1;  // values in [0, R)
      uint8_t* present;
      int32_t* pos;
      BAMG_TRY(arena_get(ctx, (size_t)R + 1, &present));
      BAMG_TRY(arena_get(ctx, (size_t)R + 1, &pos));
      BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(present, 0, (size_t)R + 1, ctx->stream));
      BAMG_LAUNCH(ctx, int_presence_kernel, grid_for(n, 256), 256, 0, coord, n, present);
      BAMG_TRY(scan_u8(ctx, present, pos, R, nvalues_host));
      BAMG_LAUNCH(ctx, int_rank_kernel, grid_for(n, 256), 256, 0, coord, n, (const int32_t*)pos, rank);
      return 0;
    }
  }
  unsigned long long *k1, *k2, *orand;
  int32_t *i1, *i2, *pos;
  uint8_t* flag;
  BAMG_TRY(arena_get(ctx, (size_t)n, &k1));
  BAMG_TRY(arena_get(ctx, (size_t)n, &k2));
  BAMG_TRY(arena_get(ctx, (size_t)n, &i1));
  BAMG_TRY(arena_get(ctx, (size_t)n, &i2));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &pos));
  BAMG_TRY(arena_get(ctx, (size_t)n, &flag));
  BAMG_TRY(arena_get(ctx, 2, &orand));
  unsigned long long init[2] = {0ull, ~0ull};
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(orand, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  BAMG_LAUNCH(ctx, keys_init_kernel, grid_for(n, 256), 256, 0, coord, n, k1, i1, orand);
  unsigned long long oa[2];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(orand), 2, reinterpret_cast<int64_t*>(oa)));
  unsigned long long vary = oa[0] ^ oa[1];
  for (int bit = 0; bit < 64; ++bit) {
    if (!((vary >> bit) & 1ull)) continue;
    BAMG_LAUNCH(ctx, bit_flags_kernel, grid_for(n, 256), 256, 0, k1, n, bit, flag);
    BAMG_TRY(scan_u8(ctx, flag, pos, n, nullptr));
    BAMG_LAUNCH(ctx, bit_scatter_kernel, grid_for(n, 256), 256, 0, k1, i1, n, bit, pos, k2, i2);
    std::swap(k1, k2);
    std::swap(i1, i2);
  }
  BAMG_LAUNCH(ctx, distinct_flags_kernel, grid_for(n, 256), 256, 0, k1, n, flag);
  int64_t ndistinct_minus_one = 0;
  BAMG_TRY(scan_u8(ctx, flag, pos, n, &ndistinct_minus_one));
  BAMG_LAUNCH(ctx, rank_scatter_kernel, grid_for(n, 256), 256, 0, i1, pos, flag, n, rank);
  if (nvalues_host) *nvalues_host = ndistinct_minus_one + 1;
  return 0;
}

__global__ void presence_kernel(const int32_t* __restrict__ prank, const int32_t* __restrict__ cidx, int64_t nc,
                                uint8_t* __restrict__ present) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) present[prank[cidx[i]]] = 1;
}

__global__ void rerank_kernel(const int32_t* __restrict__ prank, const int32_t* __restrict__ cidx, int64_t nc,
                              const int32_t* __restrict__ pos, int32_t* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nc) out[i] = pos[prank[cidx[i]]];
}

extern "C" int bamg_rerank(bamg_ctx* ctx, const int32_t* parent_rank, const int32_t* coarse_idx, int64_t nc,
                           int64_t nvalues_parent, int32_t* rank_out, int64_t* nvalues_host) {
  ctx->arena.reset();
  uint8_t* present;
  int32_t* pos;
  BAMG_TRY(arena_get(ctx, (size_t)nvalues_parent + 1, &present));
  BAMG_TRY(arena_get(ctx, (size_t)nvalues_parent + 1, &pos));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(present, 0, nvalues_parent + 1, ctx->stream));
  BAMG_LAUNCH(ctx, presence_kernel, grid_for(nc, 256), 256, 0, parent_rank, coarse_idx, nc, present);
  BAMG_TRY(scan_u8(ctx, present, pos, nvalues_parent, nvalues_host));
  BAMG_LAUNCH(ctx, rerank_kernel, grid_for(nc, 256), 256, 0, parent_rank, coarse_idx, nc, pos, rank_out);
  return 0;
}

struct RankPtrs {
  const int32_t* r[4];
};

__global__ void even_mask_kernel(RankPtrs rp, int ndim, int64_t n, uint8_t* __restrict__ mask) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ok = true;
  for (int a = 0; a < ndim; ++a) ok = ok && ((rp.r[a][i] & 1) == 0);
  mask[i] = ok;
}

extern "C" int bamg_even_mask(bamg_ctx* ctx, const int32_t* const* ranks_host, int ndim, int64_t n, uint8_t* mask) {
  BAMG_REQUIRE(ctx, ndim >= 1 && ndim <= 4, "1 to 4 axes supported");
  RankPtrs rp{};
  for (int a = 0; a < ndim; ++a) rp.r[a] = ranks_host[a];
  BAMG_LAUNCH(ctx, even_mask_kernel, grid_for(n, 256), 256, 0, rp, ndim, n, mask);
  return 0;
}

__global__ void split_scatter_kernel(const uint8_t* __restrict__ mask, const int32_t* __restrict__ pos, int64_t n,
                                     int32_t* __restrict__ coarse, int32_t* __restrict__ fine, int32_t* __restrict__ crank) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t p = pos[i];
  if (mask[i]) {
    coarse[p] = (int32_t)i;
    crank[i] = p;
  } else {
    fine[i - p] = (int32_t)i;
    crank[i] = -1;
  }
}

extern "C" int bamg_split_from_mask(bamg_ctx* ctx, const uint8_t* mask, int64_t n, int32_t* coarse, int32_t* fine,
                                    int32_t* coarse_rank, int64_t* nc_host) {
  ctx->arena.reset();
  int32_t* pos;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &pos));
  int64_t nc = 0;
  BAMG_TRY(scan_u8(ctx, mask, pos, n, &nc));
  if (nc_host) *nc_host = nc;
  BAMG_LAUNCH(ctx, split_scatter_kernel, grid_for(n, 256), 256, 0, mask, pos, n, coarse, fine, coarse_rank);
  return 0;
}

// ------------------------------------------------------ compatible relaxation
__global__ void count_mask_kernel(const uint8_t* __restrict__ m, int64_t n, unsigned long long* cnt) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int e = (i < n) && m[i];
  int t = __syncthreads_count(e);
  if (threadIdx.x == 0 && t) atomicAdd(cnt, (unsigned long long)t);
}

static int count_mask(bamg_ctx* ctx, const uint8_t* m, int64_t n, int64_t* out) {
  unsigned long long* c;
  BAMG_TRY(arena_get(ctx, 1, &c));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(c, 0, sizeof(*c), ctx->stream));
  BAMG_LAUNCH(ctx, count_mask_kernel, grid_for(n, 256), 256, 0, m, n, c);
  if (out) BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(c), 1, out));
  return 0;
}

__global__ void cr_start_kernel(const uint8_t* __restrict__ cmask, const int32_t* __restrict__ fpos,
                                const double* __restrict__ normals, int64_t n, double* __restrict__ x) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] = cmask[i] ? 0.0 : normals[i - fpos[i]];
}

// sum of x_f^2 over fine points (partials, fixed grid)
__global__ void cr_rms_partial(const double* __restrict__ x, const uint8_t* __restrict__ cmask, int64_t n,
                               double* __restrict__ partial) {
  BAMG_PDL_PROLOGUE();
  __shared__ double sh[RED_THREADS / 32];
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(r0 + per, n);
  double acc = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
    if (!cmask[i]) acc += x[i] * x[i];
  double v = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < RED_THREADS / 32; ++q) t += sh[q];
    partial[blockIdx.x] = t;
  }
}

__global__ void cr_rms_final(const double* __restrict__ partial, int nb, int64_t nf, double* scale) {
  BAMG_PDL_PROLOGUE();
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) v += partial[b];
  v = warp_sum(v);
  if (threadIdx.x == 0) scale[0] = fmax(sqrt(v / (double)nf), 1e-300);
}

__global__ void cr_scale_kernel(double* __restrict__ x, int64_t n, const double* __restrict__ scale) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] / scale[0];
}

__global__ void zero_where_kernel(double* __restrict__ x, const uint8_t* __restrict__ m, int64_t n) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && m[i]) x[i] = 0.0;
}

__global__ void dead_mask_kernel(const double* __restrict__ d, int64_t n, uint8_t* __restrict__ dead) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dead[i] = d[i] == 0.0;
}

// mu and candidate state; counts candidates
__global__ void cr_mu_kernel(const double* __restrict__ x, const uint8_t* __restrict__ cmask, int64_t n, double expo,
                             double thr, double* __restrict__ mu, uint8_t* __restrict__ state,
                             unsigned long long* __restrict__ ncand) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c = 0;
  if (i < n) {
    double m = cmask[i] ? 0.0 : pow(fmin(fabs(x[i]), 1e6), expo);
    mu[i] = m;
    c = (!cmask[i] && m > thr) ? 1 : 0;
    state[i] = c ? 0 : 3;  // 0 undecided candidate, 3 not a candidate
  }
  int tot = __syncthreads_count(c);
  if (threadIdx.x == 0 && tot) atomicAdd(ncand, (unsigned long long)tot);
}

// lexicographically-first MIS round.  Priority: larger mu first, then lower
// index (np.lexsort((candidates, -mu[candidates]))).
__global__ void mis_round_kernel(int64_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                 const double* __restrict__ mu, volatile uint8_t* state, int* __restrict__ changed,
                                 int* __restrict__ undecided) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (state[i] != 0) return;
  double mi = mu[i];
  bool all_out = true;
  bool any_in = false;
  for (int j = arp[i]; j < arp[i + 1]; ++j) {
    int p = acol[j];
    uint8_t sp = state[p];
    if (sp == 3) continue;
    double mp = mu[p];
    bool higher = (mp > mi) || (mp == mi && p < i);
    if (!higher) continue;
    if (sp == 1) {
      any_in = true;
      break;
    }
    if (sp == 0) all_out = false;
  }
  if (any_in) {
    state[i] = 2;
    *changed = 1;
  } else if (all_out) {
    state[i] = 1;
    *changed = 1;
  } else {
    *undecided = 1;
  }
}

__global__ void mis_commit_kernel(const uint8_t* __restrict__ state, int64_t n, uint8_t* __restrict__ cmask) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && state[i] == 1) cmask[i] = 1;
}

// fallback: coarse[argmax(where(fine, mu, -1))] = True
__global__ void cr_fallback_kernel(const double* __restrict__ mu, const uint8_t* __restrict__ cmask, int64_t n,
                                   uint8_t* __restrict__ cmask_out) {
  BAMG_PDL_PROLOGUE();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double best = -INFINITY;
  int64_t bi = 0;
  for (int64_t i = 0; i < n; ++i) {
    double v = cmask[i] ? -1.0 : mu[i];
    if (v > best) {
      best = v;
      bi = i;
    }
  }
  cmask_out[bi] = 1;
}

extern "C" int bamg_cr_pass(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* adj, const double* d, uint8_t* cmask,
                            const double* normals, int64_t n_fine, int sweeps, double omega, double threshold,
                            int coarse_empty, int64_t* ncand_host, int64_t* ncoarse_host) {
  ctx->arena.reset();
  const int64_t n = A->nrows;
  const int ns = sweeps > 1 ? sweeps : 1;
  double *x, *x2, *mu, *partial, *scale;
  int32_t* fpos;
  uint8_t *dead, *state;
  unsigned long long* ncand;
  int* flags;
  BAMG_TRY(arena_get(ctx, (size_t)n, &x));
  BAMG_TRY(arena_get(ctx, (size_t)n, &x2));
  BAMG_TRY(arena_get(ctx, (size_t)n, &mu));
  BAMG_TRY(arena_get(ctx, RED_BLOCKS, &partial));
  BAMG_TRY(arena_get(ctx, 1, &scale));
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &fpos));
  BAMG_TRY(arena_get(ctx, (size_t)n, &dead));
  BAMG_TRY(arena_get(ctx, (size_t)n, &state));
  BAMG_TRY(arena_get(ctx, 1, &ncand));
  BAMG_TRY(arena_get(ctx, 2, &flags));
  // fine positions = exclusive count of coarse points before i
  BAMG_TRY(scan_u8(ctx, cmask, fpos, n, nullptr));
  BAMG_LAUNCH(ctx, cr_start_kernel, grid_for(n, 256), 256, 0, cmask, fpos, normals, n, x);
  BAMG_LAUNCH(ctx, cr_rms_partial, RED_BLOCKS, RED_THREADS, 0, x, cmask, n, partial);
  BAMG_LAUNCH(ctx, cr_rms_final, 1, 32, 0, partial, RED_BLOCKS, n_fine, scale);
  BAMG_LAUNCH(ctx, cr_scale_kernel, grid_for(n, 256), 256, 0, x, n, scale);
  BAMG_LAUNCH(ctx, dead_mask_kernel, grid_for(n, 256), 256, 0, d, n, dead);
  for (int s = 0; s < ns; ++s) {
    // x + (omega * (0 - Bx)) / d, dead rows untouched, then C points zeroed
    BAMG_TRY(jacobi_dev(ctx, A, d, dead, nullptr, nullptr, x, x2, 1, omega, nullptr));
    BAMG_LAUNCH(ctx, zero_where_kernel, grid_for(n, 256), 256, 0, x2, cmask, n);
    std::swap(x, x2);
  }
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(ncand, 0, sizeof(*ncand), ctx->stream));
  BAMG_LAUNCH(ctx, cr_mu_kernel, grid_for(n, 256), 256, 0, x, cmask, n, 1.0 / ns, threshold, mu, state, ncand);
  int64_t nc = 0;
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(ncand), 1, &nc));
  *ncand_host = nc;
  if (nc == 0) {
    // no slow point left; on an empty coarse set promote argmax(mu) (coarsen.py:148-152)
    if (coarse_empty) BAMG_LAUNCH(ctx, cr_fallback_kernel, 1, 32, 0, mu, cmask, n, cmask);
    return count_mask(ctx, cmask, n, ncoarse_host);
  }
  for (int round = 0; round < 1 << 20; ++round) {
    BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx->stream));
    for (int r = 0; r < 4; ++r)
      BAMG_LAUNCH(ctx, mis_round_kernel, grid_for(n, 256), 256, 0, n, adj->rowptr, adj->col, mu, state, flags,
                  flags + 1);
    int fl[2];
    BAMG_TRY(ctx_read_i32(ctx, flags, 2, fl));
    if (!fl[1]) break;  // the last round saw no undecided candidate
  }
  BAMG_LAUNCH(ctx, mis_commit_kernel, grid_for(n, 256), 256, 0, state, n, cmask);
  return count_mask(ctx, cmask, n, ncoarse_host);
}

__global__ void empty_rows_kernel(const int32_t* __restrict__ rp, int64_t n, unsigned long long* cnt) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int e = (i < n) && (rp[i + 1] == rp[i]);
  int t = __syncthreads_count(e);
  if (threadIdx.x == 0 && t) atomicAdd(cnt, (unsigned long long)t);
}

extern "C" int bamg_count_empty_rows(bamg_ctx* ctx, const bamg_csr* A, int64_t* count_host) {
  ctx->arena.reset();
  unsigned long long* c;
  BAMG_TRY(arena_get(ctx, 1, &c));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(c, 0, sizeof(*c), ctx->stream));
  BAMG_LAUNCH(ctx, empty_rows_kernel, grid_for(A->nrows, 256), 256, 0, A->rowptr, A->nrows, c);
  return ctx_read_i64(ctx, reinterpret_cast<int64_t*>(c), 1, count_host);
}

