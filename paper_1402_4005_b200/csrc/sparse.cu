// sparse.cu -- bit-exact CSR SpMV / k-wide SpMM / fused weighted Jacobi,
// diagonal, degenerate-row mask, explicit transpose, symmetric pattern.
//
// Layout: CSR (int32 rowptr/col, fp64 val); k vectors interleaved n x k.
// Kernel shape ("CSR-stream"): one CTA owns a tile of TILE_ROWS consecutive
// rows, stages the tile's contiguous [rowptr[r0], rowptr[r0+R]) slice of
// col/val into shared memory with coalesced loads, then each thread walks
// one (row, vector) pair SEQUENTIALLY in ascending column order with
// __dmul_rn/__dadd_rn -- exactly scipy's csr_matvec(s) arithmetic
// (sparse.py:81-86 -> scipy _sparsetools csr_matvec: sum = 0; sum += a*x).
// The Jacobi epilogue reproduces relax.py:78-83 bit for bit:
//   r = b - Ax;  upd = (omega * r) / d;  upd = 0 on skipped rows;  x + upd.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

constexpr int TILE_ROWS = 256;
constexpr int TILE_THREADS = 256;
constexpr int TILE_NNZ = 2048;  // 24 KB of staged col/val per CTA

// EPI_JACOBI_M: Jacobi whose right-hand side is b_scale * (Mop bx)[row],
// the mass product formed in the same pass (the inhomogeneous bootstrap
// sweeps' sigma M u / sigma N v on the coarse levels)
enum { EPI_PLAIN = 0, EPI_JACOBI = 1, EPI_RESID = 2, EPI_ADD = 3, EPI_JACOBI_M = 4 };

struct EpiArgs {
  const double* d;        // diagonal
  const uint8_t* skip;    // rows left alone
  const double* b;        // rhs (may be null)
  const double* b_scale;  // per-vector scale of b (may be null)
  const double* xold;     // iterate being relaxed (EPI_JACOBI)
  const double* rd;       // RN(1/d) (may be null: plain IEEE division)
  double omega;
  double* peak;           // per-vector max |x'| (may be null)
  const int32_t* mrp;     // EPI_JACOBI_M: the mass operator's CSR ...
  const int32_t* mcol;
  const double* mval;
  const double* mx;       // ... and the block it multiplies
  int64_t mnnz;
};

template <int EPI>
__global__ void __launch_bounds__(TILE_THREADS)
csr_tile_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ X, int k,
                double* __restrict__ Y, EpiArgs ea) {
  BAMG_PDL_PROLOGUE();
  __shared__ int32_t s_rp[TILE_ROWS + 1];
  __shared__ int32_t s_col[TILE_NNZ];
  __shared__ double s_val[TILE_NNZ];
  __shared__ unsigned long long s_peak[32];

  const int r0 = blockIdx.x * TILE_ROWS;
  const int rows = min(TILE_ROWS, nrows - r0);
  for (int i = threadIdx.x; i <= rows; i += TILE_THREADS) s_rp[i] = rowptr[r0 + i];
  if (EPI == EPI_JACOBI && ea.peak && threadIdx.x < 32) s_peak[threadIdx.x] = 0ull;
  __syncthreads();
  const int nz0 = s_rp[0];
  const int tile_nnz = s_rp[rows] - nz0;
  const bool staged = tile_nnz <= TILE_NNZ;
  if (staged) {
    for (int j = threadIdx.x; j < tile_nnz; j += TILE_THREADS) {
      s_col[j] = col[nz0 + j];
      s_val[j] = val[nz0 + j];
    }
  }
  __syncthreads();

  const int pairs = rows * k;
  for (int p = threadIdx.x; p < pairs; p += TILE_THREADS) {
    const int lr = p / k;
    const int c = p - lr * k;
    const int row = r0 + lr;
    const int jb = s_rp[lr], je = s_rp[lr + 1];
    double sum = 0.0;
    if (staged) {
      for (int j = jb - nz0; j < je - nz0; ++j)
        sum = __dadd_rn(sum, __dmul_rn(s_val[j], X[(int64_t)s_col[j] * k + c]));
    } else {
      for (int j = jb; j < je; ++j)
        sum = __dadd_rn(sum, __dmul_rn(val[j], X[(int64_t)col[j] * k + c]));
    }
    const int64_t idx = (int64_t)row * k + c;
    if (EPI == EPI_PLAIN) {
      Y[idx] = sum;
    } else if (EPI == EPI_RESID) {
      Y[idx] = __dsub_rn(ea.b[idx], sum);
    } else if (EPI == EPI_ADD) {
      Y[idx] = __dadd_rn(ea.xold[idx], sum);
    } else {
      double bb = 0.0;
      if (ea.b) bb = ea.b_scale ? __dmul_rn(ea.b_scale[c], ea.b[idx]) : ea.b[idx];
      const double r = __dsub_rn(bb, sum);
      double upd = 0.0;
      if (!ea.skip[row]) {
        const double num = __dmul_rn(ea.omega, r);
        upd = ea.rd ? div_rn_recip(num, ea.d[row], ea.rd[row]) : __ddiv_rn(num, ea.d[row]);
      }
      const double xn = __dadd_rn(ea.xold[idx], upd);
      Y[idx] = xn;
      if (ea.peak) atomicMax(&s_peak[c], (unsigned long long)__double_as_longlong(fabs(xn)));
    }
  }
  if (EPI == EPI_JACOBI && ea.peak) {
    __syncthreads();
    if (threadIdx.x < k) atomic_max_nonneg(&ea.peak[threadIdx.x], __longlong_as_double((long long)s_peak[threadIdx.x]));
  }
}


// Row-per-thread variant for compile-time K (1, 2, 4, 8, 12, 16): a thread owns
// one row and all K vectors, so col/val/d/skip are read once per row, the K
// partial sums live in registers and each neighbour's K-value segment is read
// with 16-byte vector loads.  Per-vector sums stay sequential in ascending
// column order (bit-identical to the pair kernel and to scipy).
__device__ __forceinline__ void ldg_v4f64(const double* p, double* v) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void stg_v4f64(double* p, const double* v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

template <int K>
struct VecIO {
  static __device__ __forceinline__ void load(const double* __restrict__ p, double* v) {
    if constexpr (K % 4 == 0) {
      // 256-bit loads (sm_100): a thread owns 32-byte segments of a row of the block
#pragma unroll
      for (int i = 0; i < K / 4; ++i) ldg_v4f64(p + 4 * i, v + 4 * i);
    } else if constexpr (K % 2 == 0) {
      const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
      for (int i = 0; i < K / 2; ++i) {
        double2 t = __ldg(q + i);
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = __ldg(p + i);
    }
  }
  static __device__ __forceinline__ void store(double* __restrict__ p, const double* v) {
    if constexpr (K % 4 == 0) {
#pragma unroll
      for (int i = 0; i < K / 4; ++i) stg_v4f64(p + 4 * i, v + 4 * i);
    } else if constexpr (K % 2 == 0) {
      double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
      for (int i = 0; i < K / 2; ++i) q[i] = make_double2(v[2 * i], v[2 * i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) p[i] = v[i];
    }
  }
};

// slice [voff, voff + VV) of (Op X)[row], sequential ascending-column sums
template <int K, int VV, int U>
__device__ __forceinline__ void row_apply(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                          const double* __restrict__ val, const double* __restrict__ X, int row,
                                          int voff, double* acc) {
#pragma unroll
  for (int q = 0; q < VV; ++q) acc[q] = 0.0;
  const int jb = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
  for (int j = jb; j < je; j += U) {
    int cc[U];
    double aa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int jj = j + u < je ? j + u : je - 1;
      cc[u] = __ldg(col + jj);
      aa[u] = __ldg(val + jj);
    }
    double xv[U][VV];
#pragma unroll
    for (int u = 0; u < U; ++u) VecIO<VV>::load(X + (int64_t)cc[u] * K + voff, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < je) {
#pragma unroll
        for (int q = 0; q < VV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(aa[u], xv[u][q]));
      }
    }
  }
}

// G threads share a row, each owning V = K / G consecutive vectors (one
// 16-byte load per neighbour when V = 2), and the row's entries are consumed
// U at a time: all U neighbour segments are loaded before any is accumulated,
// so each thread keeps U independent loads in flight.  256 threads per CTA,
// 256 / G rows per CTA; col/val of the CTA's rows staged in shared memory.
template <int EPI, int K, int G, int U, bool STAGE, int MB = 0, bool EARLY = false>
// 8 resident CTAs per SM caps the row kernels at 32 registers (full
// occupancy): measured ~25% faster for k = 8 / 16 than the 40-72 registers
// ptxas picks otherwise (tools/csr_bench.py)
#ifndef BAMG_ROWS_MINB
#define BAMG_ROWS_MINB 8
#endif
__global__ void __launch_bounds__(TILE_THREADS, (MB > 0 ? MB : BAMG_ROWS_MINB))
csr_rows_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ X, double* __restrict__ Y, EpiArgs ea) {
  BAMG_PDL_PROLOGUE();
  constexpr int V = K / G;
  constexpr int RB = TILE_THREADS / G;  // rows per CTA
  constexpr int NNZ_CAP = STAGE ? RB * 12 : 1;  // staged when the tile averages <= 12 entries per row
  __shared__ int32_t s_col[NNZ_CAP];
  __shared__ double s_val[NNZ_CAP];
  __shared__ unsigned long long s_peak[K];
  const int r0 = blockIdx.x * RB;
  const int rows = min(RB, nrows - r0);
  if ((EPI == EPI_JACOBI || EPI == EPI_JACOBI_M) && ea.peak && threadIdx.x < K) s_peak[threadIdx.x] = 0ull;
  int nz0 = 0;
  bool staged = false;
  if constexpr (STAGE) {
    nz0 = rowptr[r0];
    const int tile_nnz = rowptr[r0 + rows] - nz0;
    staged = tile_nnz <= NNZ_CAP;
    if (staged) {
      for (int j = threadIdx.x; j < tile_nnz; j += TILE_THREADS) {
        s_col[j] = col[nz0 + j];
        s_val[j] = val[nz0 + j];
      }
    }
    __syncthreads();
  } else if ((EPI == EPI_JACOBI || EPI == EPI_JACOBI_M) && ea.peak) {
    __syncthreads();
  }
  const int lr = threadIdx.x / G;
  const int sub = threadIdx.x - lr * G;
  double pk[V];
#pragma unroll
  for (int q = 0; q < V; ++q) pk[q] = 0.0;
  if (lr < rows) {
    const int row = r0 + lr;
    const int voff = sub * V;
    double acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = 0.0;
    const int jb = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
    // EARLY: the Jacobi epilogue's operands depend on the row only -- issued with the row extents
    // instead of after the gathers (one memory latency less per row: the sweep is latency-bound)
    [[maybe_unused]] bool e_sk = false;
    [[maybe_unused]] double e_dd = 1.0, e_rdd = 0.0, e_xo[V], e_b[V];
    if constexpr (EARLY && EPI == EPI_ADD) VecIO<V>::load(ea.xold + (int64_t)row * K + voff, e_xo);
    if constexpr (EARLY && EPI == EPI_JACOBI) {
      e_sk = ea.skip[row] != 0;
      e_dd = ea.d[row];
      e_rdd = ea.rd ? ea.rd[row] : 0.0;
      VecIO<V>::load(ea.xold + (int64_t)row * K + voff, e_xo);
      if (ea.b) VecIO<V>::load(ea.b + (int64_t)row * K + voff, e_b);
    }
    for (int j = jb; j < je; j += U) {
      int cc[U];
      double aa[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j + u < je ? j + u : je - 1;
        if (STAGE && staged) {
          cc[u] = s_col[jj - nz0];
          aa[u] = s_val[jj - nz0];
        } else {
          cc[u] = __ldg(col + jj);
          aa[u] = __ldg(val + jj);
        }
      }
      double xv[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u) VecIO<V>::load(X + (int64_t)cc[u] * K + voff, xv[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j + u < je) {
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(aa[u], xv[u][q]));
        }
      }
    }
    const int64_t base = (int64_t)row * K + voff;
    double out[V];
    if (EPI == EPI_PLAIN) {
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = acc[q];
    } else if (EPI == EPI_RESID) {
      double bv[V];
      VecIO<V>::load(ea.b + base, bv);
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = __dsub_rn(bv[q], acc[q]);
    } else if (EPI == EPI_ADD) {
      double xo[V];
      if constexpr (EARLY) {
#pragma unroll
        for (int q = 0; q < V; ++q) xo[q] = e_xo[q];
      } else {
        VecIO<V>::load(ea.xold + base, xo);
      }
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = __dadd_rn(xo[q], acc[q]);
    } else {
      double bv[V];
      if (EPI == EPI_JACOBI_M) {
        row_apply<K, V, U>(ea.mrp, ea.mcol, ea.mval, ea.mx, row, voff, bv);
#pragma unroll
        for (int q = 0; q < V; ++q) bv[q] = __dmul_rn(ea.b_scale[voff + q], bv[q]);
      } else if (ea.b) {
        if constexpr (EARLY && EPI == EPI_JACOBI) {
#pragma unroll
          for (int q = 0; q < V; ++q) bv[q] = e_b[q];
        } else {
          VecIO<V>::load(ea.b + base, bv);
        }
        if (ea.b_scale) {
#pragma unroll
          for (int q = 0; q < V; ++q) bv[q] = __dmul_rn(ea.b_scale[voff + q], bv[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) bv[q] = 0.0;
      }
      double xo[V];
      bool sk;
      double dd, rdd;
      if constexpr (EARLY && EPI == EPI_JACOBI) {
#pragma unroll
        for (int q = 0; q < V; ++q) xo[q] = e_xo[q];
        sk = e_sk, dd = e_dd, rdd = e_rdd;
      } else {
        VecIO<V>::load(ea.xold + base, xo);
        sk = ea.skip[row] != 0;
        dd = ea.d[row];
        rdd = ea.rd ? ea.rd[row] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const double num = __dmul_rn(ea.omega, __dsub_rn(bv[q], acc[q]));
        double upd = sk ? 0.0 : (ea.rd ? div_rn_recip(num, dd, rdd) : __ddiv_rn(num, dd));
        out[q] = __dadd_rn(xo[q], upd);
        pk[q] = fabs(out[q]);
      }
    }
    VecIO<V>::store(Y + base, out);
  }
  if ((EPI == EPI_JACOBI || EPI == EPI_JACOBI_M) && ea.peak) {
    // max over the lanes that own the same vectors (lane % G), then one
    // shared atomic per (warp, vector) and one global atomic per (CTA, vector)
    constexpr bool POW2 = (G & (G - 1)) == 0;  // lane % G groups survive xor shuffles
    if constexpr (POW2) {
#pragma unroll
      for (int q = 0; q < V; ++q) {
        double m = pk[q];
        for (int o = G; o < 32; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        pk[q] = m;
      }
    }
    if (!POW2 || (threadIdx.x & 31) < G) {
#pragma unroll
      for (int q = 0; q < V; ++q)
        atomicMax(&s_peak[sub * V + q], (unsigned long long)__double_as_longlong(pk[q]));
    }
    __syncthreads();
    if (threadIdx.x < K) atomic_max_nonneg(&ea.peak[threadIdx.x], __longlong_as_double((long long)s_peak[threadIdx.x]));
  }
}

// Software-pipelined row kernel (persistent CTAs, same arithmetic).
// csr_rows_kernel's per-thread chain is rowptr -> col/val -> X gathers (one
// round per U entries) -> epilogue operands: four to five dependent memory
// latencies per row, with the wide gathers in flight only a fraction of the
// time (ncu at cfg4 level 0, k = 16: long-scoreboard bound, 40 % of HBM).
// Here every G-thread group walks its rows (tile blockIdx.x + i * gridDim.x)
// as a stream of chunks of <= U entries, and one step issues, before it
// consumes anything: the gathers and values of the current chunk, the column
// indices of the NEXT chunk (of this row or of the group's next row), the
// extents of the row after next, and the epilogue operands of a row that
// finishes.  A step therefore costs one memory latency and keeps
// U * 8V + 12U bytes per thread in flight.  Sums stay sequential in ascending
// column order per (row, vector): bit-identical to csr_rows_kernel.
template <int EPI, int K, int G, int U, int MINB, bool HASB = true>
__global__ void __launch_bounds__(TILE_THREADS, MINB)
csr_rows_pipe_kernel(int nrows, int ntiles, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                     const double* __restrict__ val, const double* __restrict__ X, double* __restrict__ Y,
                     EpiArgs ea) {
  BAMG_PDL_PROLOGUE();
  static_assert(EPI != EPI_JACOBI_M, "the mass-fused sweep stays on csr_rows_kernel");
  constexpr int V = K / G;
  constexpr int RB = TILE_THREADS / G;
  __shared__ unsigned long long s_peak[K];
  const bool want_peak = EPI == EPI_JACOBI && ea.peak != nullptr;
  if (want_peak) {
    if (threadIdx.x < K) s_peak[threadIdx.x] = 0ull;
    __syncthreads();
  }
  const int lr = threadIdx.x / G;
  const int sub = threadIdx.x - lr * G;
  const int voff = sub * V;
  const int stride = gridDim.x * RB;
  const int limit = lr < RB ? ntiles * RB : 0;  // threads past the last whole group idle (K = 12: 252 of 256)
  double pk[V], acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) pk[q] = 0.0, acc[q] = 0.0;

  int row = blockIdx.x * RB + lr;
  int j = 0, je = 0;
  if (row < limit && row < nrows) j = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
  int row_n = row + stride, jb_n = 0, je_n = 0;
  if (row_n < limit && row_n < nrows) jb_n = __ldg(rowptr + row_n), je_n = __ldg(rowptr + row_n + 1);
  int cc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cc[u] = j + u < je ? __ldg(col + j + u) : 0;

  while (row < limit) {
    const bool fin = j + U >= je;  // this chunk completes the row
    // (1) gathers and (2) values of the current chunk
    double xv[U][V], aa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < je) {
        VecIO<V>::load(X + (int64_t)cc[u] * K + voff, xv[u]);
        aa[u] = __ldg(val + j + u);
      } else {
        aa[u] = 0.0;
#pragma unroll
        for (int q = 0; q < V; ++q) xv[u][q] = 0.0;
      }
    }
    // (3) the next chunk's columns: the rest of this row, or the head of the group's next row
    const int rown = fin ? row_n : row;
    const int jn = fin ? jb_n : j + U;
    const int jen = fin ? je_n : je;
    int ccn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ccn[u] = jn + u < jen ? __ldg(col + jn + u) : 0;
    // (4) on a row change, the extents of the row after next
    int row_nn = row_n, jb_nn = jb_n, je_nn = je_n;
    if (fin) {
      row_nn = row_n + stride;
      jb_nn = je_nn = 0;
      if (row_nn < limit && row_nn < nrows) jb_nn = __ldg(rowptr + row_nn), je_nn = __ldg(rowptr + row_nn + 1);
    }
    // (5) epilogue operands of a finishing row
    const bool emit = fin && row < nrows;
    const int64_t base = (int64_t)row * K + voff;
    double e0[V], e1[V], dd = 1.0, rdd = 0.0;
    bool sk = false;
    if (emit) {
      if (EPI == EPI_RESID) VecIO<V>::load(ea.b + base, e0);
      if (EPI == EPI_ADD) VecIO<V>::load(ea.xold + base, e0);
      if (EPI == EPI_JACOBI) {
        VecIO<V>::load(ea.xold + base, e0);
        if constexpr (HASB) {
          if (ea.b) VecIO<V>::load(ea.b + base, e1);
        }
        sk = ea.skip[row] != 0;
        dd = ea.d[row];
        if (ea.rd) rdd = ea.rd[row];
      }
    }
    // (6) accumulate in column order
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < je) {
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(aa[u], xv[u][q]));
      }
    }
    // (7) finish the row
    if (emit) {
      double out[V];
      if (EPI == EPI_PLAIN) {
#pragma unroll
        for (int q = 0; q < V; ++q) out[q] = acc[q];
      } else if (EPI == EPI_RESID) {
#pragma unroll
        for (int q = 0; q < V; ++q) out[q] = __dsub_rn(e0[q], acc[q]);
      } else if (EPI == EPI_ADD) {
#pragma unroll
        for (int q = 0; q < V; ++q) out[q] = __dadd_rn(e0[q], acc[q]);
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          double bv = 0.0;
          if constexpr (HASB) {
            if (ea.b) bv = ea.b_scale ? __dmul_rn(ea.b_scale[voff + q], e1[q]) : e1[q];
          }
          const double num = __dmul_rn(ea.omega, __dsub_rn(bv, acc[q]));
          const double upd = sk ? 0.0 : (ea.rd ? div_rn_recip(num, dd, rdd) : __ddiv_rn(num, dd));
          out[q] = __dadd_rn(e0[q], upd);
          pk[q] = fmax(pk[q], fabs(out[q]));
        }
      }
      VecIO<V>::store(Y + base, out);
    }
    if (fin) {
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = 0.0;
      row_n = row_nn, jb_n = jb_nn, je_n = je_nn;
    }
    row = rown, j = jn, je = jen;
#pragma unroll
    for (int u = 0; u < U; ++u) cc[u] = ccn[u];
  }
  if (want_peak) {
    constexpr bool POW2 = (G & (G - 1)) == 0;
    if constexpr (POW2) {
#pragma unroll
      for (int q = 0; q < V; ++q) {
        double m = pk[q];
        for (int o = G; o < 32; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        pk[q] = m;
      }
    }
    if (lr < RB && (!POW2 || (threadIdx.x & 31) < G)) {
#pragma unroll
      for (int q = 0; q < V; ++q)
        atomicMax(&s_peak[sub * V + q], (unsigned long long)__double_as_longlong(pk[q]));
    }
    __syncthreads();
    if (threadIdx.x < K) atomic_max_nonneg(&ea.peak[threadIdx.x], __longlong_as_double((long long)s_peak[threadIdx.x]));
  }
}

// BAMG_G16 = "G:U": threads per row / unroll of the k = 16 kernels (G = 4: 256-bit segments)
static void g16_cfg(int* g, int* u, int* mb = nullptr, int* pg = nullptr) {
  static int gg = 0, uu = 0, mm = 0, pp = 0;
  if (!gg) {
    int a = 8, b = 4, c = 8;
    const char* e = getenv("BAMG_G16");
    if (!(e && sscanf(e, "%d:%d:%d", &a, &b, &c) == 3)) a = 8, b = 4, c = 8;
    const char* e2 = getenv("BAMG_PIPE_G16");
    pp = e2 ? atoi(e2) : 8;
    uu = b, mm = c, gg = a;
  }
  *g = gg, *u = uu;
  if (mb) *mb = mm;
  if (pg) *pg = pp;
}

// BAMG_ROWS_PIPE: "0" disables the pipelined kernel; "K:U:MINB[,K:U:MINB...]"
// overrides the per-K tuning (development: tools/csr_bench.py sweeps)
struct PipeCfg {
  int u, minb;
};
static PipeCfg pipe_cfg(int k) {
  static int init = 0;
  static PipeCfg tab[33];
  if (!init) {
    for (int i = 0; i <= 32; ++i) tab[i] = PipeCfg{0, 0};
    // measured at cfg4's level 0 (tools/pipe_sweep.sh): k = 16 sweeps with a right-hand side or the
    // per-column peak gain 7-13 % (one atomic per CTA and column instead of one per 32 rows)
    tab[16] = PipeCfg{4, 4};
    const char* e = getenv("BAMG_ROWS_PIPE");
    if (e && e[0] == '0' && e[1] == 0) {
      for (int i = 0; i <= 32; ++i) tab[i] = PipeCfg{0, 0};
    } else if (e) {
      int kk, uu, mm;
      const char* p = e;
      while (sscanf(p, "%d:%d:%d", &kk, &uu, &mm) == 3) {
        if (kk >= 1 && kk <= 32) tab[kk] = PipeCfg{uu, mm};
        p = strchr(p, ',');
        if (!p) break;
        ++p;
      }
    }
    init = 1;
  }
  return tab[k];
}

// returns 1 when (k, the configured U / MINB) has no pipelined instance
template <int EPI>
static int launch_rows_pipe(bamg_ctx* ctx, int k, double bytes, const bamg_csr* A, const double* X, double* Y,
                            const EpiArgs& ea) {
  const PipeCfg pc = pipe_cfg(k);
  if (pc.u == 0) return 1;
  int g16, u16;
  g16_cfg(&u16, &u16, nullptr, &g16);
  if (k == 16 && g16 != 8 &&
      ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(ea.b) |
        reinterpret_cast<uintptr_t>(ea.xold)) & 31) != 0)
    g16 = 8;
#define BAMG_PIPE_CASE(KK, GG, UU, MB)                                                                      \
  if (k == KK && pc.u == UU && pc.minb == MB && (KK != 16 || g16 == GG)) {                                  \
    const int rb = TILE_THREADS / GG;                                                                       \
    const int ntiles = (A->nrows + rb - 1) / rb;                                                            \
    const int g = ntiles < ctx->num_sms * MB ? ntiles : ctx->num_sms * MB;                                \
    if (EPI == EPI_JACOBI && !ea.b)                                                                         \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                          \
                      (csr_rows_pipe_kernel<EPI, KK, GG, UU, MB, false>), g, TILE_THREADS, 0, A->nrows,     \
                      ntiles, A->rowptr, A->col, A->val, X, Y, ea);                                         \
    else                                                                                                    \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                          \
                      (csr_rows_pipe_kernel<EPI, KK, GG, UU, MB>), g, TILE_THREADS, 0, A->nrows, ntiles,    \
                      A->rowptr, A->col, A->val, X, Y, ea);                                                 \
    return 0;                                                                                               \
  }
  BAMG_PIPE_CASE(16, 8, 4, 5)
  BAMG_PIPE_CASE(16, 8, 4, 4)
  BAMG_PIPE_CASE(16, 8, 5, 4)
  BAMG_PIPE_CASE(16, 8, 6, 4)
  BAMG_PIPE_CASE(16, 8, 6, 3)
  BAMG_PIPE_CASE(16, 8, 8, 3)
  BAMG_PIPE_CASE(16, 4, 2, 4)
  BAMG_PIPE_CASE(16, 4, 4, 3)
  BAMG_PIPE_CASE(12, 6, 6, 4)
  BAMG_PIPE_CASE(12, 6, 6, 3)
  BAMG_PIPE_CASE(8, 4, 6, 4)
  BAMG_PIPE_CASE(8, 4, 6, 3)
  BAMG_PIPE_CASE(8, 4, 8, 3)
  BAMG_PIPE_CASE(1, 1, 4, 8)
  BAMG_PIPE_CASE(1, 1, 4, 6)
  BAMG_PIPE_CASE(1, 1, 6, 5)
  BAMG_PIPE_CASE(1, 1, 6, 6)
  BAMG_PIPE_CASE(1, 1, 8, 6)
  BAMG_PIPE_CASE(1, 1, 8, 4)
#undef BAMG_PIPE_CASE
  return 1;
}

#ifndef BAMG_U1
#define BAMG_U1 4
#endif
#ifndef BAMG_G8
#define BAMG_G8 4
#endif
#ifndef BAMG_U8
#define BAMG_U8 6
#endif

static int rows_stage_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("BAMG_ROWS_STAGE");
    mode = (e && e[0] == '1') ? 1 : 0;
  }
  return mode;
}

template <int EPI>
static int launch_rows(bamg_ctx* ctx, int k, int /*grid*/, double bytes, const bamg_csr* A, const double* X, double* Y,
                       const EpiArgs& ea) {
  if (k == 16) {
    int g16, u16, m16;
    g16_cfg(&g16, &u16, &m16);
    const bool al32 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) |
                        reinterpret_cast<uintptr_t>(ea.b) | reinterpret_cast<uintptr_t>(ea.xold) |
                        reinterpret_cast<uintptr_t>(ea.mx)) & 31) == 0;
    static const bool early = getenv("BAMG_EARLY") && getenv("BAMG_EARLY")[0] == '1';
#define BAMG_ROWS16(GG, UU, MM)                                                                            \
  if (al32 && g16 == GG && u16 == UU && m16 == MM) {                                                       \
    int g = (A->nrows + TILE_THREADS / GG - 1) / (TILE_THREADS / GG);                                      \
    if (early && EPI == EPI_JACOBI) {                                                                      \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                        \
                      (csr_rows_kernel<EPI, 16, GG, UU, false, MM, true>), g, TILE_THREADS, 0, A->nrows,   \
                      A->rowptr, A->col, A->val, X, Y, ea);                                                \
      return 0;                                                                                            \
    }                                                                                                      \
    BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                          \
                    (csr_rows_kernel<EPI, 16, GG, UU, false, MM>), g, TILE_THREADS, 0, A->nrows, A->rowptr, \
                    A->col, A->val, X, Y, ea);                                                             \
    return 0;                                                                                              \
  }
    BAMG_ROWS16(8, 4, 8)
    BAMG_ROWS16(4, 4, 4)
    BAMG_ROWS16(4, 2, 5)
    BAMG_ROWS16(2, 2, 4)
#undef BAMG_ROWS16
  }
  if (k == 1 && (EPI == EPI_JACOBI || EPI == EPI_RESID || EPI == EPI_PLAIN) && A->nnz > 5 * (int64_t)A->nrows) {
    // Galerkin levels of the V-cycle (7-9 entries per row): the whole row in one round of U = 8
    // gathers and the Jacobi operands issued beside the row extents -- three dependent memory
    // latencies per row (extents -> col / val -> gathers) instead of five.
    // BAMG_K1W = "U:MB:EARLY" (development), "0" = off
    static int wu = -1, wmb = 0, wearly = 0;
    if (wu < 0) {
      int a = 8, b = 5, c = 1;
      const char* e = getenv("BAMG_K1W");
      if (e && e[0] == '0' && e[1] == 0) a = 0;
      else if (!(e && sscanf(e, "%d:%d:%d", &a, &b, &c) == 3)) a = 8, b = 5, c = 1;
      wu = a, wmb = b, wearly = c;
    }
    const int g = (A->nrows + TILE_THREADS - 1) / TILE_THREADS;
#define BAMG_K1W_CASE(UU, MM, EE)                                                                          \
  if (wu == UU && wmb == MM && wearly == EE) {                                                             \
    BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                          \
                    (csr_rows_kernel<EPI, 1, 1, UU, false, MM, EE != 0>), g, TILE_THREADS, 0, A->nrows,    \
                    A->rowptr, A->col, A->val, X, Y, ea);                                                  \
    return 0;                                                                                              \
  }
    BAMG_K1W_CASE(8, 5, 1)
    BAMG_K1W_CASE(8, 6, 1)
    BAMG_K1W_CASE(8, 6, 0)
#undef BAMG_K1W_CASE
  }
  if (k == 1 && EPI == EPI_ADD) {
    // the V-cycle's prolongation + correction (rows of 1-2 entries): the old iterate issued beside
    // the row extents (BAMG_K1W=0 disables)
    static const bool off = getenv("BAMG_K1W") && getenv("BAMG_K1W")[0] == '0' && getenv("BAMG_K1W")[1] == 0;
    if (!off) {
      const int g = (A->nrows + TILE_THREADS - 1) / TILE_THREADS;
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,
                      (csr_rows_kernel<EPI, 1, 1, 2, false, 8, true>), g, TILE_THREADS, 0, A->nrows, A->rowptr,
                      A->col, A->val, X, Y, ea);
      return 0;
    }
  }
  switch (k) {
#define BAMG_ROWS_CASE(KK, GG, UU)                                                                         \
  case KK: {                                                                                               \
    int g = (A->nrows + TILE_THREADS / GG - 1) / (TILE_THREADS / GG);                                      \
    if (rows_stage_mode())                                                                                 \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, (csr_rows_kernel<EPI, KK, GG, UU, true>), g, TILE_THREADS, 0,  \
                      A->nrows, A->rowptr, A->col, A->val, X, Y, ea);                                      \
    else                                                                                                   \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, (csr_rows_kernel<EPI, KK, GG, UU, false>), g, TILE_THREADS, 0, \
                      A->nrows, A->rowptr, A->col, A->val, X, Y, ea);                                      \
    return 0;                                                                                              \
  }
    BAMG_ROWS_CASE(1, 1, BAMG_U1)
    BAMG_ROWS_CASE(2, 1, 4)
    BAMG_ROWS_CASE(4, 2, 4)
    BAMG_ROWS_CASE(8, BAMG_G8, BAMG_U8)
    BAMG_ROWS_CASE(12, 6, 4)
    BAMG_ROWS_CASE(16, 8, 4)
#undef BAMG_ROWS_CASE
    default:
      return 1;  // not specialised
  }
}

static int check_csr(bamg_ctx* ctx, const bamg_csr* A);

// Fused Rayleigh quotient for identity masses (bootstrap.py:144-153 with
// M = N = I): one pass over A computes (A V)[row] per vector with the SpMM's
// sequential sums and folds it straight into u.(Av); the same pass sums u.u
// and v.v.  A fixed grid of RED_BLOCKS CTAs strides over row tiles, so the
// per-CTA partials -- and the last CTA's fixed-order final sum and sigma
// finish -- are bit-reproducible.  Saves the A V write + re-read and two
// launches per quotient.
// Masses M, N (nullable = identity): u.(M u) and v.(N v) from their rows in
// the same pass (the coarse levels' inhomogeneous sweeps), without writing
// M U, N V, A V.
// the stencil row in the kernel's parameter space (constant bank operands)
struct StencilArgs {
  const uint8_t* tiles;
  int w, diag;
  int delta[8];
  double val[8];
  double d, rd;
};

struct MassRows {
  const int32_t* mrp;
  const int32_t* mcol;
  const double* mval;
  const int32_t* nrp;
  const int32_t* ncol;
  const double* nval;
};

// MASS = false: identity masses (the finest levels) -- without the mass rows'
// code the kernel fits 40 registers, 6 CTAs per SM (62 registers otherwise)
#ifndef BAMG_RQ_MASS_MINB
#define BAMG_RQ_MASS_MINB 4
#endif
// identity masses: 4 CTAs per SM (64 registers) since the stencil path and the early u / v loads
#ifndef BAMG_RQ_MINB
#define BAMG_RQ_MINB 4
#endif
template <int K, int G, int U, bool MASS>
__global__ void __launch_bounds__(TILE_THREADS, MASS ? BAMG_RQ_MASS_MINB : BAMG_RQ_MINB)
rayleigh_fused_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                      const double* __restrict__ val, const double* __restrict__ Vv, const double* __restrict__ Uv,
                      double* __restrict__ partial, unsigned int* __restrict__ counter, double* __restrict__ dots,
                      double* __restrict__ sigma, double* __restrict__ flip, int mode, MassRows ms,
                      const __grid_constant__ StencilArgs st) {
  BAMG_PDL_PROLOGUE();
  constexpr int VV = K / G;
  constexpr int RB = TILE_THREADS / G;
  constexpr bool STENCIL_OK = 256 % RB == 0;  // a row tile lies inside one 256-row stencil tile
  __shared__ double sv[3][TILE_THREADS][VV];
  __shared__ bool last;
  const int lr = threadIdx.x / G;
  const int sub = threadIdx.x - lr * G;
  const int voff = sub * VV;
  double s0[VV], s1[VV], s2[VV];
#pragma unroll
  for (int q = 0; q < VV; ++q) s0[q] = s1[q] = s2[q] = 0.0;
  // stencil flag of a row tile, fetched one tile ahead (no load of the tile waits on it)
  unsigned char fnext = 0;
  if (STENCIL_OK && st.tiles && blockIdx.x * RB < nrows) fnext = st.tiles[(blockIdx.x * RB) >> 8];
  for (int tile = blockIdx.x; tile * RB < nrows; tile += gridDim.x) {
    const int row = tile * RB + lr;
    const unsigned char sten = fnext;
    if (STENCIL_OK && st.tiles && (tile + (int)gridDim.x) * RB < nrows)
      fnext = st.tiles[((tile + (int)gridDim.x) * RB) >> 8];
    if (row < nrows) {
      // the row's own u and v segments depend on the row only: issued before the gathers, so the
      // row costs one round of memory latency (they used to follow the sums: two rounds)
      // (identity masses only: the mass variant is short of registers and loads them after the sums)
      double uu[VV], vv[VV];
      if (!MASS) {
        VecIO<VV>::load(Uv + (int64_t)row * K + voff, uu);
        VecIO<VV>::load(Vv + (int64_t)row * K + voff, vv);
      }
      double acc[VV];
#pragma unroll
      for (int q = 0; q < VV; ++q) acc[q] = 0.0;
      if (STENCIL_OK && sten) {
        // stencil tile (bamg_csr_stencil): offsets and values from the parameter space, the
        // same products in the same order
        const double* xr = Vv + (int64_t)row * K + voff;
#pragma unroll
        for (int u0 = 0; u0 < 8; u0 += 4) {
          if (u0 < st.w) {
            double xv[4][VV];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u0 + u < st.w) VecIO<VV>::load(xr + (int64_t)st.delta[u0 + u] * K, xv[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (u0 + u < st.w) {
#pragma unroll
                for (int q = 0; q < VV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(st.val[u0 + u], xv[u][q]));
              }
            }
          }
        }
      } else {
        const int jb = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
        for (int j = jb; j < je; j += U) {
          int cc[U];
          double aa[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int jj = j + u < je ? j + u : je - 1;
            cc[u] = __ldg(col + jj);
            aa[u] = __ldg(val + jj);
          }
          double xv[U][VV];
#pragma unroll
          for (int u = 0; u < U; ++u) VecIO<VV>::load(Vv + (int64_t)cc[u] * K + voff, xv[u]);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (j + u < je) {
#pragma unroll
              for (int q = 0; q < VV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(aa[u], xv[u][q]));
            }
          }
        }
      }
      if (MASS) {
        VecIO<VV>::load(Uv + (int64_t)row * K + voff, uu);
        VecIO<VV>::load(Vv + (int64_t)row * K + voff, vv);
      }
      double mu[VV], nv[VV];
      if (MASS && ms.mrp) {
        row_apply<K, VV, U>(ms.mrp, ms.mcol, ms.mval, Uv, row, voff, mu);
      } else {
#pragma unroll
        for (int q = 0; q < VV; ++q) mu[q] = uu[q];
      }
      if (MASS && ms.nrp) {
        row_apply<K, VV, U>(ms.nrp, ms.ncol, ms.nval, Vv, row, voff, nv);
      } else {
#pragma unroll
        for (int q = 0; q < VV; ++q) nv[q] = vv[q];
      }
#pragma unroll
      for (int q = 0; q < VV; ++q) {
        s0[q] += uu[q] * acc[q];
        s1[q] += uu[q] * mu[q];
        s2[q] += vv[q] * nv[q];
      }
    }
  }
  // CTA sum per (quantity, vector): every thread parks its VV partials, then
  // thread t < 3K adds the RB threads that own vector (t % K) in row order
  // (G need not divide the warp: K = 12 runs G = 6)
  __syncthreads();
#pragma unroll
  for (int q = 0; q < VV; ++q) {
    sv[0][threadIdx.x][q] = s1[q];  // uMu
    sv[1][threadIdx.x][q] = s2[q];  // vNv
    sv[2][threadIdx.x][q] = s0[q];  // uBv
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < 3 * K) {
    const int qi = threadIdx.x / K, c = threadIdx.x % K, sb = c / VV, q = c % VV;
    double v = 0.0;
    for (int r = 0; r < RB; ++r) v += sv[qi][r * G + sb][q];
    partial[(int64_t)blockIdx.x * 3 * K + threadIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int m = 3 * K, nb = gridDim.x;
  for (int i = wid; i < m; i += TILE_THREADS / 32) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(partial + (int64_t)b * m + i);
    v = warp_sum(v);
    if (lane == 0) dots[i] = v;
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < K) {
    double du = sqrt(fmax(dots[c], 0.0));
    double dv = sqrt(fmax(dots[K + c], 0.0));
    double prev = sigma[c];
    double sg = (du < 1e-15 || dv < 1e-15) ? prev : dots[2 * K + c] / (du * dv);
    if (mode == 0) {
      sigma[c] = sg;
    } else {
      double f = 0.0;
      if (sg < -1e-13) {
        f = 1.0;
        sg = -sg;
      }
      flip[c] = f;
      sigma[c] = fabs(sg);
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// returns 1 when k has no specialisation (caller takes the general path)
int rayleigh_fused_dev(bamg_ctx* ctx, const bamg_csr* A, const double* U, const double* V, int k, double* sigma,
                       double* flip, int mode, double* dots, const bamg_csr* M, const bamg_csr* N) {
  BAMG_TRY(check_csr(ctx, A));
  if (((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(V)) & 15) != 0 && !(k & 1)) return 1;
  // grid: a fixed function of the row count (so the partial-sum tree is
  // reproducible), capped at exactly one wave of the identity-mass kernel
  // (6 CTAs per SM): 8 per SM left a third-occupied second wave (ncu: 24 % of
  // HBM bandwidth, long-scoreboard bound; 107 -> 84 us at cfg1's level 0).
  // Two row tiles in flight per thread (48 registers, 5 CTAs per SM) measured
  // no faster.
  constexpr int RQ_BLOCKS = BAMG_RQ_MINB * 148;
  const int rb_rows = TILE_THREADS / 8;  // rows per tile at the widest G
  int nblk = (A->nrows + 4 * rb_rows - 1) / (4 * rb_rows);
  // the mass variant holds BAMG_RQ_MASS_MINB CTAs per SM (76 registers): its own one-wave cap
  const int cap = (M || N) ? BAMG_RQ_MASS_MINB * 148 : RQ_BLOCKS;
  nblk = nblk < 1 ? 1 : (nblk > cap ? cap : nblk);
  double* partial;
  BAMG_TRY(arena_get(ctx, (size_t)RQ_BLOCKS * 3 * k, &partial));
  const double n = A->nrows;
  double bytes = 4.0 * (n + 1) + 12.0 * (double)A->nnz + 8.0 * k * A->ncols + 8.0 * k * n;
  StencilArgs st{};
  {
    const char* e = getenv("BAMG_NO_STENCIL");
    if (A->ptiles && A->st_w >= 1 && A->st_w <= 8 && !(e && e[0] == '1')) {
      st.tiles = A->ptiles;
      st.w = A->st_w;
      for (int u = 0; u < 8; ++u) st.delta[u] = A->st_delta[u], st.val[u] = A->st_val[u];
      st.d = A->st_d;
      st.rd = A->st_rd;
      // flagged tiles read no operator
      bytes -= (256.0 * (double)A->st_tiles / n) * (4.0 * (n + 1) + 12.0 * (double)A->nnz);
    }
  }
  MassRows ms{};
  if (M) {
    ms.mrp = M->rowptr, ms.mcol = M->col, ms.mval = M->val;
    bytes += 4.0 * (n + 1) + 12.0 * (double)M->nnz;
  }
  if (N) {
    ms.nrp = N->rowptr, ms.ncol = N->col, ms.nval = N->val;
    bytes += 4.0 * (n + 1) + 12.0 * (double)N->nnz;
  }
  switch (k) {
#define BAMG_RQ_CASE(KK, GG, UU)                                                                              \
  case KK:                                                                                                   \
    if (M || N)                                                                                              \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                           \
                      (rayleigh_fused_kernel<KK, GG, UU, true>), nblk, TILE_THREADS, 0, A->nrows, A->rowptr,  \
                      A->col, A->val, V, U, partial, ctx->counters + 2, dots, sigma, flip, mode, ms, st);     \
    else                                                                                                     \
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,                           \
                      (rayleigh_fused_kernel<KK, GG, UU, false>), nblk, TILE_THREADS, 0, A->nrows, A->rowptr, \
                      A->col, A->val, V, U, partial, ctx->counters + 2, dots, sigma, flip, mode, ms, st);     \
    return 0;
    BAMG_RQ_CASE(1, 1, BAMG_U1)
    BAMG_RQ_CASE(2, 1, 4)
    BAMG_RQ_CASE(4, 2, 4)
    BAMG_RQ_CASE(8, BAMG_G8, BAMG_U8)
    BAMG_RQ_CASE(12, 6, 4)
    BAMG_RQ_CASE(16, 8, 4)
#undef BAMG_RQ_CASE
    default:
      return 1;
  }
}

static bool rows_kernel_enabled() {
  const char* e = getenv("BAMG_PAIR_KERNEL");
  return !(e && e[0] == '1');
}

static int check_csr(bamg_ctx* ctx, const bamg_csr* A) {
  BAMG_REQUIRE(ctx, A && A->rowptr && (A->nnz == 0 || (A->col && A->val)), "null CSR");
  BAMG_REQUIRE(ctx, A->nrows >= 0 && A->ncols >= 0, "negative CSR shape");
  return 0;
}

static int launch_packed(bamg_ctx* ctx, int epi, const bamg_csr* A, const double* X, double* Y, const EpiArgs& ea);

// k-wide sweeps of a lattice operator with stencil tiles (bamg_csr_stencil).  csr_rows_kernel's
// per-row chain is rowptr -> col / val -> gathers -> epilogue operands; in a flagged 256-row tile
// every row's offsets and values are the kernel's constant-bank operands, so a row is ONE round of
// loads: its W gathers, its right-hand side and its skip flag, all issued together, and the tile
// reads neither rowptr / col / val nor d / 1/d (W = the stencil's entry count at compile time, 8 = any
// count up to 8; the tile flag is fetched one tile ahead).  Persistent CTAs stride over the tiles (one
// atomic per CTA and column for the peak); tiles that cross a lattice boundary take the CSR row
// code.  Sums in ascending column order per (row, vector): bit-identical to csr_rows_kernel.
template <int EPI, int V>
__device__ __forceinline__ void wide_epilogue(const EpiArgs& ea, int K, int row, int voff, const double* acc,
                                              const double* bv_in, bool hasb, bool sk, double dd, double rdd,
                                              double* pk, double* __restrict__ Y, const double* xo_in = nullptr) {
  const int64_t base = (int64_t)row * K + voff;
  double out[V];
  if (EPI == EPI_PLAIN) {
#pragma unroll
    for (int q = 0; q < V; ++q) out[q] = acc[q];
  } else if (EPI == EPI_RESID) {
#pragma unroll
    for (int q = 0; q < V; ++q) out[q] = __dsub_rn(bv_in[q], acc[q]);
  } else {
    double xo[V];
    if (xo_in) {  // the iterate's own row was one of the gathers (the stencil's diagonal entry)
#pragma unroll
      for (int q = 0; q < V; ++q) xo[q] = xo_in[q];
    } else {
      VecIO<V>::load(ea.xold + base, xo);
    }
#pragma unroll
    for (int q = 0; q < V; ++q) {
      double bv = 0.0;
      if (hasb) bv = ea.b_scale ? __dmul_rn(ea.b_scale[voff + q], bv_in[q]) : bv_in[q];
      const double num = __dmul_rn(ea.omega, __dsub_rn(bv, acc[q]));
      const double upd = sk ? 0.0 : div_rn_recip(num, dd, rdd);
      out[q] = __dadd_rn(xo[q], upd);
      pk[q] = fmax(pk[q], fabs(out[q]));
    }
  }
  VecIO<V>::store(Y + base, out);
}

// a tile that crosses a lattice boundary: the CSR row code, out of line (its registers are not the
// stencil path's)
template <int V>
struct PeakV {
  double v[V];
};

template <int EPI, int K, int G>
__device__ __noinline__ PeakV<K / G> stencil_generic_tile(int nrows, const int32_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val, const double* __restrict__ X,
                                                          double* __restrict__ Y, const EpiArgs& ea, int r0, int voff,
                                                          bool hasb) {
  constexpr int V = K / G;
  constexpr int RB = TILE_THREADS / G;
  double pk[V];
#pragma unroll
  for (int q = 0; q < V; ++q) pk[q] = 0.0;
  for (int p = 0; p < G; ++p) {
    const int row = r0 + p * RB;
    if (row >= nrows) break;
    double acc[V], bv[V];
    bool sk = false;
    double dd = 1.0, rdd = 0.0;
    if (hasb) VecIO<V>::load(ea.b + (int64_t)row * K + voff, bv);
    if (EPI == EPI_JACOBI) {
      sk = ea.skip[row] != 0;
      dd = ea.d[row];
      rdd = ea.rd ? ea.rd[row] : 0.0;
    }
    row_apply<K, V, 4>(rowptr, col, val, X, row, voff, acc);
    // without a stored reciprocal the IEEE division (div_rn_recip needs RN(1 / d))
    if (EPI == EPI_JACOBI && !ea.rd) {
      const int64_t base = (int64_t)row * K + voff;
      double xo[V], out[V];
      VecIO<V>::load(ea.xold + base, xo);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        double b1 = 0.0;
        if (hasb) b1 = ea.b_scale ? __dmul_rn(ea.b_scale[voff + q], bv[q]) : bv[q];
        const double num = __dmul_rn(ea.omega, __dsub_rn(b1, acc[q]));
        out[q] = __dadd_rn(xo[q], sk ? 0.0 : __ddiv_rn(num, dd));
        pk[q] = fmax(pk[q], fabs(out[q]));
      }
      VecIO<V>::store(Y + base, out);
    } else {
      wide_epilogue<EPI, V>(ea, K, row, voff, acc, bv, hasb, sk, dd, rdd, pk, Y);
    }
  }
  PeakV<V> r;
#pragma unroll
  for (int q = 0; q < V; ++q) r.v[q] = pk[q];
  return r;
}

template <int EPI, int K, int G, int W, int MINB, int UNR>
__global__ void __launch_bounds__(TILE_THREADS, MINB)
csr_rows_stencil_kernel(int nrows, int ntiles, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const double* __restrict__ X, double* __restrict__ Y,
                        EpiArgs ea, const __grid_constant__ StencilArgs st) {
  BAMG_PDL_PROLOGUE();
  static_assert(EPI == EPI_PLAIN || EPI == EPI_RESID || EPI == EPI_JACOBI, "epilogues of the B / B^T sweeps");
  constexpr int V = K / G;
  constexpr int RB = TILE_THREADS / G;  // rows per pass; a 256-row tile is G passes
  __shared__ unsigned long long s_peak[K];
  const bool want_peak = EPI == EPI_JACOBI && ea.peak != nullptr;
  if (want_peak) {
    if (threadIdx.x < K) s_peak[threadIdx.x] = 0ull;
    __syncthreads();
  }
  const int lr = threadIdx.x / G;
  const int sub = threadIdx.x - lr * G;
  const int voff = sub * V;
  const bool hasb = EPI == EPI_RESID || (EPI == EPI_JACOBI && ea.b != nullptr);
  double pk[V];
#pragma unroll
  for (int q = 0; q < V; ++q) pk[q] = 0.0;
  unsigned char fnext = blockIdx.x < ntiles ? st.tiles[blockIdx.x] : 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int r0 = tile * 256 + lr;
    // the flag was fetched one tile ahead: no load of this tile waits on it
    const unsigned char f = fnext;
    fnext = tile + (int)gridDim.x < ntiles ? st.tiles[tile + gridDim.x] : 0;
    if (f) {
#pragma unroll UNR
      for (int p = 0; p < G; ++p) {
        const int row = r0 + p * RB;
        const double* xr = X + (int64_t)row * K + voff;
        double xv[W][V], bv[V];
#pragma unroll
        for (int u = 0; u < W; ++u)
          if (W < 8 || u < st.w) VecIO<V>::load(xr + (int64_t)st.delta[u] * K, xv[u]);
        bool sk = false;
        if (hasb) VecIO<V>::load(ea.b + (int64_t)row * K + voff, bv);
        if (EPI == EPI_JACOBI) sk = ea.skip[row] != 0;
        double acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = 0.0;
#pragma unroll
        for (int u = 0; u < W; ++u) {
          if (W < 8 || u < st.w) {
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(st.val[u], xv[u][q]));
          }
        }
        wide_epilogue<EPI, V>(ea, K, row, voff, acc, bv, hasb, sk, st.d, st.rd, pk, Y);
      }
    } else {
      const PeakV<V> g = stencil_generic_tile<EPI, K, G>(nrows, rowptr, col, val, X, Y, ea, r0, voff, hasb);
#pragma unroll
      for (int q = 0; q < V; ++q) pk[q] = fmax(pk[q], g.v[q]);
    }
  }
  if (want_peak) {
#pragma unroll
    for (int q = 0; q < V; ++q) {
      double m = pk[q];
      for (int o = G; o < 32; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      pk[q] = m;
    }
    if ((threadIdx.x & 31) < G) {
#pragma unroll
      for (int q = 0; q < V; ++q)
        atomicMax(&s_peak[sub * V + q], (unsigned long long)__double_as_longlong(pk[q]));
    }
    __syncthreads();
    if (threadIdx.x < K) atomic_max_nonneg(&ea.peak[threadIdx.x], __longlong_as_double((long long)s_peak[threadIdx.x]));
  }
}

static bool stencil_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BAMG_NO_STENCIL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

// the bytes a k-wide stencil sweep moves: flagged tiles read no operator, no d / 1/d
static double stencil_bytes(int epi, const bamg_csr* A, int k, const EpiArgs& ea) {
  const double n = A->nrows, kk = k;
  const double generic = 1.0 - 256.0 * (double)A->st_tiles / n;
  double bytes = generic * (4.0 * (n + 1) + 12.0 * (double)A->nnz) + n / 256 + 8.0 * kk * A->ncols + 8.0 * kk * n;
  if (epi == EPI_RESID) bytes += 8.0 * kk * n;
  if (epi == EPI_JACOBI) bytes += (ea.b ? 8.0 * kk * n : 0.0) + n + generic * 16.0 * n;
  return bytes;
}

// returns 1 when the call is not covered (caller takes the CSR kernels)
static int launch_stencil(bamg_ctx* ctx, int epi, const bamg_csr* A, const double* X, int k, double* Y,
                          const EpiArgs& ea) {
  if (!A->ptiles || A->st_w < 1 || A->st_w > 8 || !stencil_enabled()) return 1;
  if (epi != EPI_PLAIN && epi != EPI_RESID && epi != EPI_JACOBI) return 1;
  if (epi == EPI_JACOBI && ea.xold != X) return 1;
  if (((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(ea.b) |
        reinterpret_cast<uintptr_t>(ea.xold)) & 31) != 0)
    return 1;
  StencilArgs st{};
  st.tiles = A->ptiles;
  st.w = A->st_w;
  st.diag = A->st_diag;
  for (int u = 0; u < 8; ++u) st.delta[u] = A->st_delta[u], st.val[u] = A->st_val[u];
  st.d = A->st_d;
  st.rd = A->st_rd;
  const int ntiles = (A->nrows + 255) / 256;
  const double bytes = stencil_bytes(epi, A, k, ea);
  const int fam = A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE;
  // BAMG_STENCIL_CFG = "MB:UNR" (development: CTAs per SM and passes in flight)
  static int cmb = 0, cun = 0;
  if (!cmb) {
    int a = 4, b = 2;
    const char* e = getenv("BAMG_STENCIL_CFG");
    if (!(e && sscanf(e, "%d:%d", &a, &b) == 2)) a = 4, b = 2;
    cmb = a, cun = b;
  }
#define BAMG_STENCIL_CASE(EE, KK, GG, WW, MB, UN)                                                              \
  if (epi == EE && k == KK && (WW == 8 ? A->st_w <= 8 : A->st_w == WW) && cmb == MB && cun == UN) {           \
    const int g = ntiles < ctx->num_sms * MB ? ntiles : ctx->num_sms * MB;                                    \
    BAMG_LAUNCH_FAM(ctx, fam, bytes, (csr_rows_stencil_kernel<EE, KK, GG, WW, MB, UN>), g, TILE_THREADS, 0,    \
                    A->nrows, ntiles, A->rowptr, A->col, A->val, X, Y, ea, st);                               \
    return 0;                                                                                                 \
  }
#define BAMG_STENCIL_K(KK, GG, MB, UN)                \
  BAMG_STENCIL_CASE(EPI_PLAIN, KK, GG, 4, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_RESID, KK, GG, 4, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_JACOBI, KK, GG, 4, MB, UN)    \
  BAMG_STENCIL_CASE(EPI_PLAIN, KK, GG, 5, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_PLAIN, KK, GG, 8, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_RESID, KK, GG, 5, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_RESID, KK, GG, 8, MB, UN)     \
  BAMG_STENCIL_CASE(EPI_JACOBI, KK, GG, 5, MB, UN)    \
  BAMG_STENCIL_CASE(EPI_JACOBI, KK, GG, 8, MB, UN)
  BAMG_STENCIL_K(16, 8, 4, 2)
  BAMG_STENCIL_K(16, 8, 4, 1)
  BAMG_STENCIL_K(8, 4, 4, 2)
  BAMG_STENCIL_K(8, 4, 4, 1)
#undef BAMG_STENCIL_K
#undef BAMG_STENCIL_CASE
  return 1;
}

// k = 16 with 32-byte-aligned blocks: 256-bit row segments (G = 4 threads per row).  Measured at
// cfg4's level 0 (tools/g16_sweep.sh, L2 flushed): plain SpMM 1143 -> 928 us through the pipelined
// kernel at U = 2 (0.85 of the HBM peak); the Jacobi sweep without a peak 1540 -> 1282 us through
// the row kernel with its epilogue operands issued beside the row extents (one memory latency less
// per row); the sweep with a peak stays on the G = 8 pipelined kernel (one atomic per CTA and column;
// the G = 4 pipelined sweep needs > 64 registers and loses more to occupancy or spills than it gains).
template <int EPI, int G, int U, int MB, bool HASB>
static int launch_pipe16(bamg_ctx* ctx, double bytes, const bamg_csr* A, const double* X, double* Y,
                         const EpiArgs& ea) {
  const int rb = TILE_THREADS / G;
  const int ntiles = (A->nrows + rb - 1) / rb;
  const int g = ntiles < ctx->num_sms * MB ? ntiles : ctx->num_sms * MB;
  BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,
                  (csr_rows_pipe_kernel<EPI, 16, G, U, MB, HASB>), g, TILE_THREADS, 0, A->nrows, ntiles, A->rowptr,
                  A->col, A->val, X, Y, ea);
  return 0;
}

static int k16_policy() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("BAMG_K16");
    mode = e ? atoi(e) : 1;
  }
  return mode;
}

static int launch_k16(bamg_ctx* ctx, int epi, double bytes, const bamg_csr* A, const double* X, double* Y,
                      const EpiArgs& ea) {
  const int mode = k16_policy();
  if (mode == 0) return 1;
  if (((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(ea.b) |
        reinterpret_cast<uintptr_t>(ea.xold)) & 31) != 0)
    return 1;
  switch (epi) {
    case EPI_PLAIN: return launch_pipe16<EPI_PLAIN, 4, 2, 4, true>(ctx, bytes, A, X, Y, ea);
    case EPI_RESID: return launch_pipe16<EPI_RESID, 4, 2, 4, true>(ctx, bytes, A, X, Y, ea);
    case EPI_ADD: return launch_pipe16<EPI_ADD, 4, 2, 4, true>(ctx, bytes, A, X, Y, ea);
    case EPI_JACOBI: {
      if (ea.peak) {
        if (mode == 2 && !ea.b) return launch_pipe16<EPI_JACOBI, 4, 2, 3, false>(ctx, bytes, A, X, Y, ea);
        return 1;  // G = 8 pipelined kernel
      }
      const int g = (A->nrows + TILE_THREADS / 4 - 1) / (TILE_THREADS / 4);
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes,
                      (csr_rows_kernel<EPI_JACOBI, 16, 4, 2, false, 5, true>), g, TILE_THREADS, 0, A->nrows,
                      A->rowptr, A->col, A->val, X, Y, ea);
      return 0;
    }
    default: return 1;
  }
}

static int launch_tile(bamg_ctx* ctx, int epi, const bamg_csr* A, const double* X, int k,
                       double* Y, const EpiArgs& ea) {
  BAMG_TRY(check_csr(ctx, A));
  BAMG_REQUIRE(ctx, k >= 1 && k <= 32, "k must lie in [1, 32]");
  int grid = (A->nrows + TILE_ROWS - 1) / TILE_ROWS;
  if (grid == 0) return 0;
  // algorithmic bytes: rowptr + col/val + each x once + y written (+ epilogue inputs)
  const double n = A->nrows, kk = k;
  double bytes = 4.0 * (n + 1) + 12.0 * (double)A->nnz + 8.0 * kk * A->ncols + 8.0 * kk * n;
  if (epi == EPI_RESID) bytes += 8.0 * n;                         // b
  if (epi == EPI_ADD) bytes += 8.0 * kk * n;                      // x_old
  if (epi == EPI_JACOBI) bytes += (ea.b ? 8.0 * kk * n : 0.0) + 9.0 * n;  // b, d, skip (x_old == X)
  if (epi == EPI_JACOBI_M) bytes += 4.0 * (n + 1) + 12.0 * (double)ea.mnnz + 8.0 * kk * n + 9.0 * n;
  // 16-byte vector loads need aligned blocks when K is even (K = 1 has none)
  bool aligned = (k & 1) || ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) |
                              reinterpret_cast<uintptr_t>(ea.b) | reinterpret_cast<uintptr_t>(ea.xold)) & 15) == 0;
  if (k == 1 && A->packed) {
    const int rc = launch_packed(ctx, epi, A, X, Y, ea);
    if (rc <= 0) return rc;
  }
  if (k > 1 && A->ptiles && rows_kernel_enabled()) {
    const int rc = launch_stencil(ctx, epi, A, X, k, Y, ea);
    if (rc <= 0) return rc;
  }
  static const bool pipe_forced = getenv("BAMG_ROWS_PIPE") != nullptr;
  if (k == 16 && rows_kernel_enabled() && !pipe_forced && !getenv("BAMG_G16")) {
    const int rc = launch_k16(ctx, epi, bytes, A, X, Y, ea);
    if (rc <= 0) return rc;
  }
  if (rows_kernel_enabled() && aligned && epi != EPI_JACOBI_M &&
      (pipe_forced || (epi == EPI_JACOBI && (ea.peak || ea.b)))) {
    int rc = 1;
    switch (epi) {
      case EPI_PLAIN: rc = launch_rows_pipe<EPI_PLAIN>(ctx, k, bytes, A, X, Y, ea); break;
      case EPI_RESID: rc = launch_rows_pipe<EPI_RESID>(ctx, k, bytes, A, X, Y, ea); break;
      case EPI_ADD: rc = launch_rows_pipe<EPI_ADD>(ctx, k, bytes, A, X, Y, ea); break;
      default: rc = launch_rows_pipe<EPI_JACOBI>(ctx, k, bytes, A, X, Y, ea);
    }
    if (rc <= 0) return rc;
  }
  if (rows_kernel_enabled() && aligned) {
    int rc = 1;
    switch (epi) {
      case EPI_PLAIN: rc = launch_rows<EPI_PLAIN>(ctx, k, grid, bytes, A, X, Y, ea); break;
      case EPI_RESID: rc = launch_rows<EPI_RESID>(ctx, k, grid, bytes, A, X, Y, ea); break;
      case EPI_ADD: rc = launch_rows<EPI_ADD>(ctx, k, grid, bytes, A, X, Y, ea); break;
      case EPI_JACOBI_M: rc = launch_rows<EPI_JACOBI_M>(ctx, k, grid, bytes, A, X, Y, ea); break;
      default: rc = launch_rows<EPI_JACOBI>(ctx, k, grid, bytes, A, X, Y, ea);
    }
    if (rc <= 0) return rc;
  }
  if (epi == EPI_JACOBI_M) return 1;  // rows kernel only: the caller forms the mass product separately
  switch (epi) {
    case EPI_PLAIN:
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, csr_tile_kernel<EPI_PLAIN>, grid, TILE_THREADS, 0, A->nrows,
                      A->rowptr, A->col, A->val, X, k, Y, ea);
      break;
    case EPI_RESID:
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, csr_tile_kernel<EPI_RESID>, grid, TILE_THREADS, 0, A->nrows,
                      A->rowptr, A->col, A->val, X, k, Y, ea);
      break;
    case EPI_ADD:
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, csr_tile_kernel<EPI_ADD>, grid, TILE_THREADS, 0, A->nrows,
                      A->rowptr, A->col, A->val, X, k, Y, ea);
      break;
    default:
      BAMG_LAUNCH_FAM(ctx, A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE, bytes, csr_tile_kernel<EPI_JACOBI>, grid, TILE_THREADS, 0, A->nrows,
                      A->rowptr, A->col, A->val, X, k, Y, ea);
  }
  return 0;
}

// ------------------------------------------------ packed operator (CSR-VI)
// The chain generators' B = I - A carries a handful of distinct values (the
// transition rates / 1/deg), and the lattice and mesh orderings keep
// |col - row| < 2^23.  Such an operator is stored a second time as one 32-bit
// word per entry -- (col - row) << 8 | value code, slice-major over 32-row
// slices (SELL-32: word u of the slice's 32 rows contiguous, short rows padded
// with code 255) -- plus a 256-entry value
// dictionary (with the correctly rounded reciprocals beside it): 4 instead of
// 12 bytes per entry on the k = 1 V-cycle sweeps, residuals and the GMRES
// SpMV, which are HBM-bound.  Decoding returns the original fp64 value, the
// sums keep the CSR order: bit-identical to csr_rows_kernel.  The Jacobi
// diagonal and its reciprocal come from the row's own delta = 0 entry (no d /
// rd streams).  Operators with more than 256 distinct values (every Galerkin
// level) or wider rows are simply not packed.
constexpr int PACK_DICT = 256;
constexpr int PACK_HASH = 1024;  // open addressing, power of two
constexpr unsigned long long PACK_EMPTY = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ unsigned int pack_hash(unsigned long long b) {
  b ^= b >> 33;
  b *= 0xff51afd7ed558ccdull;
  b ^= b >> 33;
  return (unsigned int)b & (PACK_HASH - 1);
}

// distinct value bit patterns -> global table (count[0] = distinct values, count[1] = failures)
__global__ void __launch_bounds__(256)
pack_collect_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                    const double* __restrict__ val, unsigned long long* __restrict__ table,
                    unsigned int* __restrict__ count) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned long long s_tab[PACK_HASH];
  __shared__ unsigned int s_n, s_bad;
  for (int i = threadIdx.x; i < PACK_HASH; i += blockDim.x) s_tab[i] = PACK_EMPTY;
  if (threadIdx.x == 0) s_n = 0u, s_bad = 0u;
  __syncthreads();
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrows; row += gridDim.x * blockDim.x) {
    const int jb = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
    for (int j = jb; j < je; ++j) {
      const int delta = __ldg(col + j) - row;
      if (delta >= (1 << 23) || delta < -(1 << 23)) s_bad = 1u;
      const unsigned long long b = (unsigned long long)__double_as_longlong(__ldg(val + j));
      if (b == PACK_EMPTY) {
        s_bad = 1u;
        continue;
      }
      unsigned int h = pack_hash(b);
      for (int probe = 0; probe < PACK_HASH; ++probe) {
        const unsigned long long cur = s_tab[h];
        if (cur == b) break;
        if (cur == PACK_EMPTY) {
          if (s_n > 2 * PACK_DICT) {  // hopeless: stop filling the table
            s_bad = 1u;
            break;
          }
          const unsigned long long old = atomicCAS(&s_tab[h], PACK_EMPTY, b);
          if (old == PACK_EMPTY) {
            atomicAdd(&s_n, 1u);
            break;
          }
          if (old == b) break;
        }
        h = (h + 1) & (PACK_HASH - 1);
      }
    }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicAdd(count + 1, 1u);
    return;
  }
  for (int i = threadIdx.x; i < PACK_HASH; i += blockDim.x) {
    const unsigned long long b = s_tab[i];
    if (b == PACK_EMPTY) continue;
    unsigned int h = pack_hash(b);
    for (int probe = 0; probe < PACK_HASH; ++probe) {
      const unsigned long long old = atomicCAS(table + h, PACK_EMPTY, b);
      if (old == PACK_EMPTY) {
        atomicAdd(count, 1u);
        break;
      }
      if (old == b) break;
      h = (h + 1) & (PACK_HASH - 1);
      if (probe == PACK_HASH - 1) atomicAdd(count + 1, 1u);
    }
  }
}

// one CTA: the table's values sorted by bit pattern (a fixed order whatever
// the insertion races were) -> dict[0..255], RN(1 / v) -> dict[256..511]
__global__ void __launch_bounds__(PACK_HASH)
pack_dict_kernel(const unsigned long long* __restrict__ table, unsigned int* __restrict__ count,
                 double* __restrict__ dict) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned long long s[PACK_HASH];
  const int t = threadIdx.x;
  s[t] = table[t];
  if (t < 2 * PACK_DICT) dict[t] = 0.0;
  __syncthreads();
  if (count[1] != 0u || count[0] > PACK_DICT) {
    if (t == 0) count[1] = 1u;
    return;
  }
  const unsigned long long mine = s[t];
  if (mine == PACK_EMPTY) return;
  int rank = 0;
  for (int i = 0; i < PACK_HASH; ++i) rank += (s[i] != PACK_EMPTY && s[i] < mine) ? 1 : 0;
  const double v = __longlong_as_double((long long)mine);
  dict[rank] = v;
  dict[PACK_DICT + rank] = __drcp_rn(v);
}

// words per 32-row slice: 32 x (longest row of the slice)
__global__ void __launch_bounds__(256)
pack_slice_width_kernel(int nrows, const int32_t* __restrict__ rowptr, int nslices, int32_t* __restrict__ w32) {
  BAMG_PDL_PROLOGUE();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  int len = row < nrows ? __ldg(rowptr + row + 1) - __ldg(rowptr + row) : 0;
  for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  if ((threadIdx.x & 31) == 0 && (row >> 5) < nslices) w32[row >> 5] = 32 * len;
}

constexpr uint32_t PACK_PAD = 255u;  // value code of a padding word (delta 0): loaded, never accumulated

// slice-major (SELL-32) fill: word u of row 32 s + l at pslice[s] + 32 u + l
__global__ void __launch_bounds__(256)
pack_fill_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                 const double* __restrict__ val, const double* __restrict__ dict, int nd,
                 const int32_t* __restrict__ pslice, uint32_t* __restrict__ packed) {
  BAMG_PDL_PROLOGUE();
  __shared__ unsigned long long s_key[PACK_DICT];
  for (int i = threadIdx.x; i < PACK_DICT; i += blockDim.x)
    s_key[i] = i < nd ? (unsigned long long)__double_as_longlong(dict[i]) : PACK_EMPTY;
  __syncthreads();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int slice = row >> 5, lane = threadIdx.x & 31;
  if (slice * 32 >= nrows) return;
  const int base = __ldg(pslice + slice);
  const int width = (__ldg(pslice + slice + 1) - base) >> 5;
  int jb = 0, je = 0;
  if (row < nrows) jb = __ldg(rowptr + row), je = __ldg(rowptr + row + 1);
  for (int u = 0; u < width; ++u) {
    uint32_t word = PACK_PAD;
    if (jb + u < je) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(__ldg(val + jb + u));
      int lo = 0, hi = nd - 1;  // the value is in the dictionary by construction
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_key[mid] < b) lo = mid + 1;
        else hi = mid;
      }
      const int delta = __ldg(col + jb + u) - row;
      word = ((uint32_t)delta << 8) | (uint32_t)lo;
    }
    packed[base + 32 * u + lane] = word;
  }
}

// Step 1: dictionary (dict[512]), slice offsets (pslice[nslices + 1], in words) and the
// verdict: *ok_host = number of dictionary entries (0: A does not qualify),
// *words_host = length of the packed array.
extern "C" int bamg_csr_pack_plan(bamg_ctx* ctx, const bamg_csr* A, int32_t* pslice, double* dict, int* ok_host,
                                  int64_t* words_host) {
  ctx->arena.reset();
  BAMG_TRY(check_csr(ctx, A));
  BAMG_REQUIRE(ctx, pslice && dict && ok_host && words_host, "null output");
  *ok_host = 0;
  *words_host = 0;
  if (A->nrows != A->ncols || A->nnz == 0) return 0;
  const int nslices = (A->nrows + 31) / 32;
  unsigned long long* table;
  int32_t* w32;
  BAMG_TRY(arena_get(ctx, (size_t)PACK_HASH + 2, &table));
  BAMG_TRY(arena_get(ctx, (size_t)nslices, &w32));
  unsigned int* count = reinterpret_cast<unsigned int*>(table + PACK_HASH);
  int64_t* total = reinterpret_cast<int64_t*>(table + PACK_HASH + 1);
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(table, 0xFF, sizeof(unsigned long long) * PACK_HASH, ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(count, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const int g = grid_for(A->nrows, 256);
  const int grid = g < ctx->num_sms * 8 ? g : ctx->num_sms * 8;
  BAMG_LAUNCH(ctx, pack_collect_kernel, grid, 256, 0, A->nrows, A->rowptr, A->col, A->val, table, count);
  BAMG_LAUNCH(ctx, pack_dict_kernel, 1, PACK_HASH, 0, table, count, dict);
  BAMG_LAUNCH(ctx, pack_slice_width_kernel, grid_for((int64_t)nslices * 32, 256), 256, 0, A->nrows, A->rowptr, nslices,
              w32);
  BAMG_TRY(scan_i32_dev(ctx, w32, pslice, nslices, total));
  int64_t res[2] = {0, 0};
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(count), 2, res));
  const uint64_t flags = (uint64_t)res[0];
  // count[1] == 0 (no failure), at most 255 values (code 255 pads), offsets fit int32
  if ((flags >> 32) == 0 && (flags & 0xffffffffu) < PACK_PAD && res[1] < (int64_t)1 << 31) {
    *ok_host = (int)(flags & 0xffffffffu);
    *words_host = res[1];
  }
  return 0;
}

// Step 2: the packed words (words_host of them) for a plan that said ok.
extern "C" int bamg_csr_pack_fill(bamg_ctx* ctx, const bamg_csr* A, const int32_t* pslice, const double* dict,
                                  int ndict, uint32_t* packed) {
  BAMG_TRY(check_csr(ctx, A));
  BAMG_REQUIRE(ctx, pslice && dict && packed && ndict >= 1 && ndict < (int)PACK_PAD, "bad packed plan");
  const int nslices = (A->nrows + 31) / 32;
  BAMG_LAUNCH(ctx, pack_fill_kernel, grid_for((int64_t)nslices * 32, 256), 256, 0, A->nrows, A->rowptr, A->col, A->val,
              dict, ndict, pslice, packed);
  return 0;
}

// ---- stencil tiles of a lattice operator
// record written by csr_stencil_kernel (device, 20 x 8 bytes): [0] w, [1] diag index,
// [2..9] col - row of entry u, [10..17] value bits of entry u, [18] matching tiles
__global__ void __launch_bounds__(256)
csr_stencil_kernel(int nrows, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                   const double* __restrict__ val, uint8_t* __restrict__ tiles, unsigned long long* __restrict__ rec) {
  BAMG_PDL_PROLOGUE();
  // the candidate: an interior point of the middle lattice line when the rows are a square
  // lattice (nrows / 2 itself starts a line for an even side, and is the centre for an odd one:
  // a quarter line further is interior for both)
  int ref = nrows / 2 + (int)sqrt((double)nrows) / 4;
  if (ref >= nrows) ref = nrows / 2;
  const int rb = __ldg(rowptr + ref), w = __ldg(rowptr + ref + 1) - rb;
  bool ok = w >= 1 && w <= 8;
  int rdelta[8];
  unsigned long long rbits[8];
  int diag = -1;
  if (ok) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      rdelta[u] = 0, rbits[u] = 0ull;
      if (u < w) {
        rdelta[u] = __ldg(col + rb + u) - ref;
        rbits[u] = (unsigned long long)__double_as_longlong(__ldg(val + rb + u));
        if (rdelta[u] == 0) diag = u;
      }
    }
  }
  ok = ok && diag >= 0;
  const int row = blockIdx.x * 256 + threadIdx.x;
  bool match = ok && row < nrows;
  if (match) {
    const int jb = __ldg(rowptr + row);
    match = __ldg(rowptr + row + 1) - jb == w;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (match && u < w)
        match = __ldg(col + jb + u) - row == rdelta[u] &&
                (unsigned long long)__double_as_longlong(__ldg(val + jb + u)) == rbits[u];
  }
  const int all = __syncthreads_and(match ? 1 : 0);
  if (threadIdx.x == 0) {
    tiles[blockIdx.x] = all ? 1 : 0;
    if (all) atomicAdd(rec + 18, 1ull);
    if (blockIdx.x == 0) {
      rec[0] = ok ? (unsigned long long)w : 0ull;
      rec[1] = (unsigned long long)(diag < 0 ? 0 : diag);
      for (int u = 0; u < 8; ++u) {
        rec[2 + u] = ok ? (unsigned long long)(long long)rdelta[u] : 0ull;
        rec[10 + u] = ok ? rbits[u] : 0ull;
      }
    }
  }
}

extern "C" int bamg_csr_stencil(bamg_ctx* ctx, const bamg_csr* A, uint8_t* tiles, bamg_csr* out) {
  ctx->arena.reset();
  BAMG_TRY(check_csr(ctx, A));
  BAMG_REQUIRE(ctx, out && tiles, "null output");
  *out = *A;
  out->ptiles = nullptr;
  out->st_w = 0;
  out->st_tiles = 0;
  if (A->nrows != A->ncols || A->nrows < 256 || A->nnz == 0) return 0;
  const int ntiles = (A->nrows + 255) / 256;
  unsigned long long* rec;
  BAMG_TRY(arena_get(ctx, 20, &rec));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(rec, 0, 20 * sizeof(unsigned long long), ctx->stream));
  BAMG_LAUNCH(ctx, csr_stencil_kernel, ntiles, 256, 0, A->nrows, A->rowptr, A->col, A->val, tiles, rec);
  int64_t h[19];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<int64_t*>(rec), 19, h));
  const int w = (int)h[0];
  if (w < 1 || w > 8 || 2 * h[18] < ntiles) return 0;
  out->st_w = w;
  out->st_diag = (int)h[1];
  for (int u = 0; u < 8; ++u) {
    out->st_delta[u] = u < w ? (int32_t)h[2 + u] : 0;
    double v = 0.0;
    if (u < w) memcpy(&v, &h[10 + u], sizeof(double));
    out->st_val[u] = v;
  }
  out->st_d = out->st_val[out->st_diag];
  out->st_rd = 1.0 / out->st_d;  // IEEE round-to-nearest: the value __drcp_rn gives the dictionary
  out->ptiles = tiles;
  out->st_tiles = h[18];
  return 0;
}

#ifndef BAMG_PACKED_U
#define BAMG_PACKED_U 4
#endif
constexpr int PACKED_U = BAMG_PACKED_U;
#ifndef BAMG_PACKED_MINB
#define BAMG_PACKED_MINB 8
#endif

// thread per row, k = 1, slice-major words: a warp's load of "entry u of my row" is one
// contiguous 128-byte line (row-major words cost 5-6 lines per load: the kernel sat at 69 % of
// the L1 pipe and 49 % of DRAM).  Same sums, in the same order, as csr_rows_kernel<EPI, 1, 1, U>.
template <int EPI, int U>
__device__ __forceinline__ void packed_row(int nrows, int row, int lane, const int32_t* __restrict__ pslice,
                                           const uint32_t* __restrict__ pk, const double* s_dict,
                                           const double* __restrict__ X, double* __restrict__ Y, const EpiArgs& ea) {
  const int slice = row >> 5;
  if (slice * 32 >= nrows) return;
  const bool valid = row < nrows;
  const int base = __ldg(pslice + slice);
  const int width = (__ldg(pslice + slice + 1) - base) >> 5;
  // epilogue operands depend on the row only: in flight with the row's first loads
  double eb = 0.0, exo = 0.0;
  bool sk = false;
  if (valid) {
    if (EPI == EPI_RESID) eb = __ldg(ea.b + row);
    if (EPI == EPI_JACOBI) {
      if (ea.b) eb = __ldg(ea.b + row);
      exo = __ldg(ea.xold + row);
      sk = ea.skip[row] != 0;
    }
  }
  double acc = 0.0;
  uint32_t dcode = PACK_PAD;  // value code of the row's diagonal entry (delta 0), if it has one
  const double* xr = X + (valid ? row : nrows - 1);  // rows past the end hold padding only (delta 0)
  const uint32_t* p = pk + base + lane;
  for (int u = 0; u < width; u += U) {
    uint32_t w[U];
#pragma unroll
    for (int i = 0; i < U; ++i) w[i] = u + i < width ? __ldg(p + 32 * (u + i)) : PACK_PAD;
    double xv[U];
#pragma unroll
    for (int i = 0; i < U; ++i) xv[i] = __ldg(xr + ((int32_t)w[i] >> 8));
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t code = w[i] & 255u;
      if (code != PACK_PAD) {
        acc = __dadd_rn(acc, __dmul_rn(s_dict[code], xv[i]));
        if (EPI == EPI_JACOBI && w[i] < 256u) dcode = code;
      }
    }
  }
  if (!valid) return;
  double out;
  if (EPI == EPI_PLAIN) {
    out = acc;
  } else if (EPI == EPI_RESID) {
    out = __dsub_rn(eb, acc);
  } else {
    // no diagonal entry: d = 0, 1/d = inf (such rows are skip rows)
    const double dd = dcode != PACK_PAD ? s_dict[dcode] : 0.0;
    const double rdd = dcode != PACK_PAD ? s_dict[PACK_DICT + dcode] : __longlong_as_double(0x7FF0000000000000ll);
    const double num = __dmul_rn(ea.omega, __dsub_rn(eb, acc));
    const double upd = sk ? 0.0 : div_rn_recip(num, dd, rdd);
    out = __dadd_rn(exo, upd);
  }
  Y[row] = out;
}

template <int EPI, int U>
__global__ void __launch_bounds__(TILE_THREADS, BAMG_PACKED_MINB)
csr_rows_packed_kernel(int nrows, const int32_t* __restrict__ pslice, const uint32_t* __restrict__ pk,
                       const double* __restrict__ dict, const double* __restrict__ X, double* __restrict__ Y,
                       EpiArgs ea) {
  BAMG_PDL_PROLOGUE();
  __shared__ double s_dict[2 * PACK_DICT];
  for (int i = threadIdx.x; i < 2 * PACK_DICT; i += TILE_THREADS) s_dict[i] = dict[i];
  __syncthreads();
  packed_row<EPI, U>(nrows, blockIdx.x * TILE_THREADS + threadIdx.x, threadIdx.x & 31, pslice, pk, s_dict, X, Y, ea);
}

// The packed operator of a lattice chain with stencil tiles (bamg_csr_stencil): persistent CTAs
// stride over the 256-row tiles.  A flagged tile reads no packed words and no dictionary: its
// rows' offsets and values are constant-bank operands, so a row is one round of loads (gathers,
// right-hand side, skip flag) and ~60 instructions; the next tile's flag is fetched one tile
// ahead, so no load waits on it.  (With one CTA per tile every CTA paid flag -> gathers -> store
// as a dependent chain, and the predicated 8-slot form issued 144 instructions per row: ncu had
// the sweep issue-bound at 31 % of the DRAM peak.)  Tiles that cross a lattice boundary take the
// packed words.  SW = the stencil's entry count at compile time (4, 5; 8 = any count up to 8).
template <int EPI, int U, int SW>
__global__ void __launch_bounds__(TILE_THREADS, BAMG_PACKED_MINB)
csr_rows_stencil1_kernel(int nrows, int ntiles, const int32_t* __restrict__ pslice, const uint32_t* __restrict__ pk,
                         const double* __restrict__ dict, const double* __restrict__ X, double* __restrict__ Y,
                         EpiArgs ea, const __grid_constant__ StencilArgs st) {
  BAMG_PDL_PROLOGUE();
  __shared__ double s_dict[2 * PACK_DICT];
  for (int i = threadIdx.x; i < 2 * PACK_DICT; i += TILE_THREADS) s_dict[i] = dict[i];
  __syncthreads();
  int tile = blockIdx.x;
  unsigned char f = tile < ntiles ? st.tiles[tile] : 0;
  while (tile < ntiles) {
    const int tn = tile + gridDim.x;
    const unsigned char fn = tn < ntiles ? st.tiles[tn] : 0;
    const int row = tile * TILE_THREADS + threadIdx.x;
    if (f) {
      double eb = 0.0, exo = 0.0;
      bool sk = false;
      if (EPI == EPI_RESID) eb = __ldg(ea.b + row);
      if (EPI == EPI_JACOBI) {
        if (ea.b) eb = __ldg(ea.b + row);
        exo = __ldg(ea.xold + row);
        sk = ea.skip[row] != 0;
      }
      const double* xr = X + row;
      double xv[SW];
#pragma unroll
      for (int u = 0; u < SW; ++u)
        if (SW < 8 || u < st.w) xv[u] = __ldg(xr + st.delta[u]);
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < SW; ++u)
        if (SW < 8 || u < st.w) acc = __dadd_rn(acc, __dmul_rn(st.val[u], xv[u]));
      double out;
      if (EPI == EPI_PLAIN) {
        out = acc;
      } else if (EPI == EPI_RESID) {
        out = __dsub_rn(eb, acc);
      } else {
        const double num = __dmul_rn(ea.omega, __dsub_rn(eb, acc));
        const double upd = sk ? 0.0 : div_rn_recip(num, st.d, st.rd);
        out = __dadd_rn(exo, upd);
      }
      Y[row] = out;
    } else {
      packed_row<EPI, U>(nrows, row, threadIdx.x & 31, pslice, pk, s_dict, X, Y, ea);
    }
    tile = tn;
    f = fn;
  }
}

// the bytes the packed kernels move (what the profiler's family figures use)
static double packed_bytes(int epi, const bamg_csr* A, const EpiArgs& ea) {
  const double n = A->nrows;
  // stencil tiles read neither their words nor the slice offsets
  const double generic = A->ptiles ? 1.0 - 256.0 * (double)A->st_tiles / n : 1.0;
  double bytes = generic * (4.0 * (n / 32 + 1) + 4.0 * (double)A->pwords) + 8.0 * A->ncols + 8.0 * n;
  if (A->ptiles) bytes += n / 256;
  if (epi == EPI_RESID) bytes += 8.0 * n;
  if (epi == EPI_JACOBI) bytes += (ea.b ? 8.0 * n : 0.0) + n;  // b, skip (d and 1/d come from the dictionary)
  return bytes;
}

static bool packed_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BAMG_NO_PACKED");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

// returns 1 when the call is not covered (caller takes the CSR kernels)
static int launch_packed(bamg_ctx* ctx, int epi, const bamg_csr* A, const double* X, double* Y, const EpiArgs& ea) {
  if (!A->packed || !A->dict || !A->pslice || !packed_enabled()) return 1;
  if (epi == EPI_JACOBI && (ea.peak || ea.b_scale || ea.xold != X)) return 1;
  if (epi != EPI_PLAIN && epi != EPI_RESID && epi != EPI_JACOBI) return 1;
  const int grid = (A->nrows + TILE_THREADS - 1) / TILE_THREADS;
  if (grid == 0) return 0;
  const double bytes = packed_bytes(epi, A, ea);
  const int fam = A->nrows >= FINE_ROWS ? FAM_TILE_FINE : FAM_TILE;
  StencilArgs st{};
  static const bool no_stencil = getenv("BAMG_NO_STENCIL") && getenv("BAMG_NO_STENCIL")[0] == '1';
  if (A->ptiles && A->st_w >= 1 && A->st_w <= 8 && !no_stencil) {
    static_assert(TILE_THREADS == 256, "stencil tiles are 256 rows");
    st.tiles = A->ptiles;
    st.w = A->st_w;
    for (int u = 0; u < 8; ++u) st.delta[u] = A->st_delta[u], st.val[u] = A->st_val[u];
    st.d = A->st_d;
    st.rd = A->st_rd;
  }
  const int ntiles = grid;
  const int pgrid = ntiles < ctx->num_sms * BAMG_PACKED_MINB ? ntiles : ctx->num_sms * BAMG_PACKED_MINB;
#define BAMG_STENCIL1_LAUNCH(EE, SWV)                                                                          \
  BAMG_LAUNCH_FAM(ctx, fam, bytes, (csr_rows_stencil1_kernel<EE, PACKED_U, SWV>), pgrid, TILE_THREADS, 0,       \
                  A->nrows, ntiles, A->pslice, A->packed, A->dict, X, Y, ea, st)
#define BAMG_PACKED_EPI(EE)                                                                                     \
  do {                                                                                                          \
    if (!st.tiles)                                                                                              \
      BAMG_LAUNCH_FAM(ctx, fam, bytes, (csr_rows_packed_kernel<EE, PACKED_U>), grid, TILE_THREADS, 0, A->nrows, \
                      A->pslice, A->packed, A->dict, X, Y, ea);                                                 \
    else if (st.w == 4) BAMG_STENCIL1_LAUNCH(EE, 4);                                                            \
    else if (st.w == 5) BAMG_STENCIL1_LAUNCH(EE, 5);                                                            \
    else BAMG_STENCIL1_LAUNCH(EE, 8);                                                                           \
  } while (0)
  switch (epi) {
    case EPI_PLAIN: BAMG_PACKED_EPI(EPI_PLAIN); break;
    case EPI_RESID: BAMG_PACKED_EPI(EPI_RESID); break;
    default: BAMG_PACKED_EPI(EPI_JACOBI);
  }
#undef BAMG_PACKED_EPI
#undef BAMG_STENCIL1_LAUNCH
  return 0;
}

// Internal entry points (used by the setup / solver translation units).
int spmm_dev(bamg_ctx* ctx, const bamg_csr* A, const double* X, double* Y, int k) {
  EpiArgs ea{};
  return launch_tile(ctx, EPI_PLAIN, A, X, k, Y, ea);
}

int resid_dev(bamg_ctx* ctx, const bamg_csr* A, const double* b, const double* X, double* R) {
  EpiArgs ea{};
  ea.b = b;
  return launch_tile(ctx, EPI_RESID, A, X, 1, R, ea);
}

// Y = Xold + A Xc (prolongation + correction, solver.py:116: x + P @ xc)
int addmv_dev(bamg_ctx* ctx, const bamg_csr* A, const double* Xc, const double* Xold, double* Y, int k) {
  EpiArgs ea{};
  ea.xold = Xold;
  return launch_tile(ctx, EPI_ADD, A, Xc, k, Y, ea);
}

int jacobi_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip,
               const double* b, const double* b_scale, const double* x, double* x_out, int k,
               double omega, double* peak, const double* rd) {
  EpiArgs ea{};
  ea.d = d;
  ea.rd = rd;
  ea.skip = skip;
  ea.b = b;
  ea.b_scale = b_scale;
  ea.xold = x;
  ea.omega = omega;
  ea.peak = peak;
  return launch_tile(ctx, EPI_JACOBI, A, x, k, x_out, ea);
}

// Jacobi sweep with right-hand side sigma * (M mx), the mass product formed
// row by row inside the sweep (bit-identical to spmm_dev(M, mx) followed by
// jacobi_dev with b_scale = sigma).  Returns 1 when k has no rows-kernel
// specialisation or the blocks are misaligned (caller takes the two-launch path).
int jacobi_mass_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip, const bamg_csr* M,
                    const double* mx, const double* sigma, const double* x, double* x_out, int k, double omega,
                    double* peak, const double* rd) {
  EpiArgs ea{};
  ea.d = d;
  ea.rd = rd;
  ea.skip = skip;
  ea.b_scale = sigma;
  ea.xold = x;
  ea.omega = omega;
  ea.peak = peak;
  ea.mrp = M->rowptr;
  ea.mcol = M->col;
  ea.mval = M->val;
  ea.mx = mx;
  ea.mnnz = M->nnz;
  if (!(k & 1) && (reinterpret_cast<uintptr_t>(mx) & 15) != 0) return 1;
  return launch_tile(ctx, EPI_JACOBI_M, A, x, k, x_out, ea);
}

// rd[i] = RN(1 / d[i]) (the reciprocal the Jacobi epilogue's exact division uses)
__global__ void recip_kernel(const double* __restrict__ d, int64_t n, double* __restrict__ rd) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rd[i] = __ddiv_rn(1.0, d[i]);
}

int recip_dev(bamg_ctx* ctx, const double* d, int64_t n, double* rd) {
  BAMG_LAUNCH(ctx, recip_kernel, grid_for(n, 256), 256, 0, d, n, rd);
  return 0;
}

// Self-test of div_rn_recip against __ddiv_rn on n pseudo-random operand
// pairs (counter-based hash, so every sample is reproducible from `seed`):
// mantissas uniform, exponents drawn from mode-dependent ranges
// (0: |e| <= 40, 1: the whole fast-path range, 2: all finite doubles incl.
// subnormals and zeros, 3: d within a few ulps of powers of two and
// all-ones mantissas).  Counts results whose bit patterns differ.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ double selftest_operand(unsigned long long h, unsigned long long h2, int mode, bool is_d) {
  unsigned long long mant = h & ((1ull << 52) - 1);
  int e;
  const unsigned long long r = h2 % 2001ull;
  switch (mode) {
    case 0: e = (int)(h2 % 81ull) - 40; break;
    case 1: e = is_d ? (int)(h2 % 801ull) - 400 : (int)(h2 % 1001ull) - 500; break;
    case 2: e = (int)(h2 % 2046ull) - 1022 - (int)(r % 2 ? 52 : 0); break;
    default: {
      e = (int)(h2 % 41ull) - 20;
      const int pick = (int)((h2 >> 20) % 4ull);
      if (pick == 0) mant = (1ull << 52) - 1 - (h2 >> 40) % 8ull;  // all-ones mantissa
      else if (pick == 1) mant = (h2 >> 40) % 8ull;               // just above a power of two
      break;
    }
  }
  const unsigned long long sign = (h >> 63) << 63;
  // signed zeros as numerators (every sixteenth x of modes 2 and 3): the zero fast path of div_rn_recip
  if (!is_d && mode >= 2 && ((h2 >> 50) % 16ull) == 0ull) return __longlong_as_double((long long)sign);
  if (e < -1022) {  // subnormal / zero
    int sh = -1022 - e;
    unsigned long long m = sh >= 53 ? 0ull : ((mant | (1ull << 52)) >> sh);
    return __longlong_as_double((long long)(sign | m));
  }
  unsigned long long bits = sign | ((unsigned long long)(e + 1023) << 52) | mant;
  return __longlong_as_double((long long)bits);
}

__global__ void selftest_div_kernel(int64_t n, unsigned long long seed, int mode,
                                    unsigned long long* __restrict__ mismatches) {
  BAMG_PDL_PROLOGUE();
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h0 = mix64(seed ^ (4ull * i)), h1 = mix64(seed ^ (4ull * i + 1));
    unsigned long long h2 = mix64(seed ^ (4ull * i + 2)), h3 = mix64(seed ^ (4ull * i + 3));
    double x = selftest_operand(h0, h1, mode, false);
    double d = selftest_operand(h2, h3, mode, true);
    double ref = __ddiv_rn(x, d);
    double got = div_rn_recip(x, d, __ddiv_rn(1.0, d));
    if (__double_as_longlong(ref) != __double_as_longlong(got) && !(ref != ref && got != got)) ++local;
  }
  local = (unsigned long long)warp_sum((double)local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(mismatches, local);
}

extern "C" int bamg_selftest_div(bamg_ctx* ctx, int64_t n, uint64_t seed, int mode, int64_t* mismatches_host) {
  ctx->arena.reset();
  BAMG_REQUIRE(ctx, mode >= 0 && mode <= 3, "mode must lie in [0, 3]");
  unsigned long long* cnt;
  BAMG_TRY(arena_get(ctx, 1, &cnt));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
  BAMG_LAUNCH(ctx, selftest_div_kernel, ctx->num_sms * 8, 256, 0, n, (unsigned long long)seed, mode, cnt);
  return ctx_read_i64(ctx, reinterpret_cast<int64_t*>(cnt), 1, mismatches_host);
}

extern "C" int bamg_spmv(bamg_ctx* ctx, const bamg_csr* A, const double* x, double* y) {
  return spmm_dev(ctx, A, x, y, 1);
}

extern "C" int bamg_spmm(bamg_ctx* ctx, const bamg_csr* A, const double* X, double* Y, int k) {
  return spmm_dev(ctx, A, X, Y, k);
}

extern "C" int bamg_jacobi(bamg_ctx* ctx, const bamg_csr* A, const double* d, const uint8_t* skip,
                           const double* b, const double* b_scale, const double* x,
                           double* x_out, int k, double omega, double* peak) {
  BAMG_REQUIRE(ctx, x != x_out, "Jacobi needs distinct input and output iterates");
  if (peak) BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(peak, 0, sizeof(double) * k, ctx->stream));
  return jacobi_dev(ctx, A, d, skip, b, b_scale, x, x_out, k, omega, peak, nullptr);
}

// ------------------------------------------------------------ diagonal
__global__ void diag_kernel(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, double* __restrict__ d) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = rp[i], hi = rp[i + 1] - 1;
  double v = 0.0;
  while (lo <= hi) {  // columns are sorted
    int mid = (lo + hi) >> 1;
    int c = col[mid];
    if (c == i) {
      v = val[mid];
      break;
    }
    if (c < i) lo = mid + 1;
    else hi = mid - 1;
  }
  d[i] = v;
}

int diag_dev(bamg_ctx* ctx, const bamg_csr* A, double* d) {
  int n = A->nrows < A->ncols ? A->nrows : A->ncols;
  BAMG_LAUNCH(ctx, diag_kernel, grid_for(n, 256), 256, 0, n, A->rowptr, A->col, A->val, d);
  return 0;
}

extern "C" int bamg_diag(bamg_ctx* ctx, const bamg_csr* A, double* d) {
  BAMG_TRY(check_csr(ctx, A));
  return diag_dev(ctx, A, d);
}

__global__ void count_nonpos_kernel(const double* __restrict__ d, int64_t n, unsigned long long* out) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int flag = (i < n) && (d[i] <= 0.0);
  int cnt = __syncthreads_count(flag);
  if (threadIdx.x == 0 && cnt) atomicAdd(out, (unsigned long long)cnt);
}

extern "C" int bamg_count_nonpositive(bamg_ctx* ctx, const double* d, int64_t n, int64_t* count_host) {
  ctx->arena.reset();
  unsigned long long* cnt = nullptr;
  BAMG_TRY(arena_get(ctx, 1, &cnt));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(*cnt), ctx->stream));
  BAMG_LAUNCH(ctx, count_nonpos_kernel, grid_for(n, 256), 256, 0, d, n, cnt);
  return ctx_read_i64(ctx, reinterpret_cast<int64_t*>(cnt), 1, count_host);
}

// ------------------------------------------------------ degenerate rows
// relax.py:47-63: off = (sum_j |a_ij|) - |d_i| (sequential row sum, as
// np.add.reduceat / the ones-vector product); skip = d <= 0 | off > 4 d.
__global__ void degenerate_kernel(int n, const int32_t* __restrict__ rp, const double* __restrict__ val,
                                  const double* __restrict__ d, uint8_t* __restrict__ skip) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double mass = 0.0;
  for (int j = rp[i]; j < rp[i + 1]; ++j) mass = __dadd_rn(mass, fabs(val[j]));
  double di = d[i];
  double off = __dsub_rn(mass, fabs(di));
  skip[i] = (di <= 0.0) || (off > __dmul_rn(4.0, di));
}

int degenerate_dev(bamg_ctx* ctx, const bamg_csr* A, const double* d, uint8_t* skip) {
  BAMG_LAUNCH(ctx, degenerate_kernel, grid_for(A->nrows, 256), 256, 0, A->nrows, A->rowptr, A->val, d, skip);
  return 0;
}

extern "C" int bamg_degenerate_rows(bamg_ctx* ctx, const bamg_csr* A, const double* d, uint8_t* skip) {
  BAMG_TRY(check_csr(ctx, A));
  return degenerate_dev(ctx, A, d, skip);
}

// ------------------------------------------------------------ transpose
// count per column -> exclusive scan -> scatter by (row-major) order using a
// per-column cursor, then sort each output row by source row (stable result
// independent of atomic order).  Output rows are short for every operator in
// scope; long rows fall back to a shell sort in the same thread.
__global__ void col_count_kernel(int64_t nnz, const int32_t* __restrict__ col, int32_t* __restrict__ cnt) {
  BAMG_PDL_PROLOGUE();
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nnz) atomicAdd(&cnt[col[j]], 1);
}

__global__ void transpose_scatter_kernel(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                         const double* __restrict__ val, int32_t* __restrict__ cursor,
                                         int32_t* __restrict__ col_t, double* __restrict__ val_t) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = rp[i]; j < rp[i + 1]; ++j) {
    int pos = atomicAdd(&cursor[col[j]], 1);
    col_t[pos] = i;
    val_t[pos] = val[j];
  }
}

__device__ void sort_segment(int32_t* key, double* val, int len) {
  // insertion sort (segments are short); shell gaps for long ones
  int gaps[] = {701, 301, 132, 57, 23, 10, 4, 1};
  for (int g = 0; g < 8; ++g) {
    int gap = gaps[g];
    if (gap >= len) continue;
    for (int i = gap; i < len; ++i) {
      int32_t kk = key[i];
      double vv = val ? val[i] : 0.0;
      int j = i;
      while (j >= gap && key[j - gap] > kk) {
        key[j] = key[j - gap];
        if (val) val[j] = val[j - gap];
        j -= gap;
      }
      key[j] = kk;
      if (val) val[j] = vv;
    }
  }
}

__global__ void sort_rows_kernel(int n, const int32_t* __restrict__ rp, int32_t* col, double* val) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int b = rp[i], e = rp[i + 1];
  sort_segment(col + b, val ? val + b : nullptr, e - b);
}

int transpose_dev(bamg_ctx* ctx, const bamg_csr* A, int32_t* rowptr_t, int32_t* col_t, double* val_t) {
  int32_t* cnt = nullptr;
  int32_t* cursor = nullptr;
  BAMG_TRY(arena_get(ctx, (size_t)A->ncols + 1, &cnt));
  BAMG_TRY(arena_get(ctx, (size_t)A->ncols + 1, &cursor));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (A->ncols + 1), ctx->stream));
  BAMG_LAUNCH(ctx, col_count_kernel, grid_for(A->nnz, 256), 256, 0, A->nnz, A->col, cnt);
  BAMG_TRY(scan_i32(ctx, cnt, rowptr_t, A->ncols, nullptr));
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(cursor, rowptr_t, sizeof(int32_t) * (A->ncols + 1),
                                       cudaMemcpyDeviceToDevice, ctx->stream));
  BAMG_LAUNCH(ctx, transpose_scatter_kernel, grid_for(A->nrows, 256), 256, 0, A->nrows, A->rowptr,
              A->col, A->val, cursor, col_t, val_t);
  BAMG_LAUNCH(ctx, sort_rows_kernel, grid_for(A->ncols, 256), 256, 0, A->ncols, rowptr_t, col_t, val_t);
  return 0;
}

extern "C" int bamg_csr_transpose(bamg_ctx* ctx, const bamg_csr* A, int32_t* rowptr_t, int32_t* col_t,
                                  double* val_t) {
  BAMG_TRY(check_csr(ctx, A));
  ctx->arena.reset();
  return transpose_dev(ctx, A, rowptr_t, col_t, val_t);
}

// ------------------------------------------------------ symmetric pattern
// pattern(A + A^T) minus the diagonal = sorted union of row i of A and row i
// of A^T (both sorted), without i.  (sparse.py:120-128)
template <bool FILL>
__global__ void sym_union_kernel(int n, const int32_t* __restrict__ ra, const int32_t* __restrict__ ca,
                                 const int32_t* __restrict__ rt, const int32_t* __restrict__ ct,
                                 int32_t* __restrict__ cnt_or_rp, int32_t* __restrict__ out) {
  BAMG_PDL_PROLOGUE();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int a = ra[i], ae = ra[i + 1], t = rt[i], te = rt[i + 1];
  int w = FILL ? cnt_or_rp[i] : 0;
  int count = 0;
  while (a < ae || t < te) {
    int x;
    if (t >= te || (a < ae && ca[a] < ct[t])) x = ca[a++];
    else if (a >= ae || ct[t] < ca[a]) x = ct[t++];
    else {
      x = ca[a];
      ++a;
      ++t;
    }
    if (x == i) continue;
    if (FILL) out[w + count] = x;
    ++count;
  }
  if (!FILL) cnt_or_rp[i] = count;
}

extern "C" int bamg_sym_pattern_count(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                                      int32_t* rowptr_s, int64_t* nnz_host) {
  BAMG_TRY(check_csr(ctx, A));
  BAMG_TRY(check_csr(ctx, A_t));
  BAMG_REQUIRE(ctx, A->nrows == A->ncols && A_t->nrows == A->nrows, "square matrix expected");
  ctx->arena.reset();
  int32_t* cnt = nullptr;
  BAMG_TRY(arena_get(ctx, (size_t)A->nrows + 1, &cnt));
  BAMG_LAUNCH(ctx, sym_union_kernel<false>, grid_for(A->nrows, 256), 256, 0, A->nrows, A->rowptr, A->col,
              A_t->rowptr, A_t->col, cnt, (int32_t*)nullptr);
  return scan_i32(ctx, cnt, rowptr_s, A->nrows, nnz_host);
}

extern "C" int bamg_sym_pattern_fill(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* A_t,
                                     const int32_t* rowptr_s, int32_t* col_s) {
  BAMG_LAUNCH(ctx, sym_union_kernel<true>, grid_for(A->nrows, 256), 256, 0, A->nrows, A->rowptr, A->col,
              A_t->rowptr, A_t->col, const_cast<int32_t*>(rowptr_s), col_s);
  return 0;
}
