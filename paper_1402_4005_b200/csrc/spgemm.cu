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
//
// Fast path: the list (<= LCAP distinct columns) and a 128-slot open-
// addressing index live in thread-local memory (L1-resident), so each product
// costs ~1 probe.  Rows with more distinct columns are flagged during the
// count and finished by the slow path, whose lists live in a global scratch
// slice sized by the structural upper bound sum_j nnz(B_j).  The flagged rows
// and their scratch offsets are memoised in the context between the count and
// fill calls, so a product costs two host synchronisations (row count, total).
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

constexpr int LCAP = 64;   // distinct columns per row on the fast path
constexpr int HSLOTS = 128;
constexpr int TSLOT = 32;  // kept entries per row parked by the count pass

constexpr int SPG_STORAGE = 1, SPG_REV_A = 2, SPG_REV_B = 4;

__device__ __forceinline__ bool keep_value(int order, double x) {
  return (order & SPG_STORAGE) == 0 ? !(fabs(x) < 1e-300) : (x != 0.0);
}

// write the row's kept entries in the requested order to (ocol, oval); the
// sorted order is produced by ranking (each kept entry counts the kept keys
// below it -- keys are distinct), so every output is stored exactly once
__device__ __forceinline__ void emit_row(int order, const int* key, const double* val, int len, int32_t* ocol,
                                         double* oval) {
  if (order & SPG_STORAGE) {  // reverse first touch
    int w = 0;
    for (int q = len - 1; q >= 0; --q)
      if (keep_value(order, val[q])) {
        ocol[w] = key[q];
        oval[w] = val[q];
        ++w;
      }
    return;
  }
  for (int q = 0; q < len; ++q) {  // sorted by column
    if (!keep_value(order, val[q])) continue;
    const int c = key[q];
    int r = 0;
    for (int p = 0; p < len; ++p) r += (key[p] < c && keep_value(order, val[p])) ? 1 : 0;
    ocol[r] = c;
    oval[r] = val[q];
  }
}

template <int PASS>
__global__ void __launch_bounds__(128)
spgemm_local_kernel(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                    const double* __restrict__ aval, const int32_t* __restrict__ brp,
                    const int32_t* __restrict__ bcol, const double* __restrict__ bval, int order,
                    int32_t* __restrict__ cnt, int32_t* __restrict__ big_list, unsigned int* __restrict__ nbig,
                    const int32_t* __restrict__ crp, int32_t* __restrict__ ccol, double* __restrict__ cval,
                    int32_t* __restrict__ tcol, double* __restrict__ tval, uint8_t* __restrict__ parked,
                    const int32_t* __restrict__ rows, const unsigned int* __restrict__ nrows) {
  BAMG_PDL_PROLOGUE();
  // rows (fill pass): grid-stride over the *nrows listed rows; else row = thread
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int tn = rows ? (int)*nrows : n;
  for (int t = t0; t < tn; t += rows ? gridDim.x * blockDim.x : tn) {
  const int i = rows ? rows[t] : t;
  int key[LCAP];
  double val[LCAP];
  unsigned int slotw[HSLOTS / 4];  // 1-byte list indices, 0xff = empty
#pragma unroll
  for (int h = 0; h < HSLOTS / 4; ++h) slotw[h] = 0xffffffffu;
  int len = 0;
  bool overflow = false;
  const bool rev_a = (order & SPG_REV_A) != 0, rev_b = (order & SPG_REV_B) != 0;
  const int a0 = arp[i], a1 = arp[i + 1];
  for (int ja = 0; ja < a1 - a0 && !overflow; ++ja) {
    const int jj = rev_a ? a1 - 1 - ja : a0 + ja;
    int j = acol[jj];
    double v = aval[jj];
    const int b0 = brp[j], b1 = brp[j + 1];
    for (int kb = 0; kb < b1 - b0; ++kb) {
      const int kk = rev_b ? b1 - 1 - kb : b0 + kb;
      int c = bcol[kk];
      double p = __dmul_rn(v, bval[kk]);
      unsigned h = ((unsigned)c * 2654435761u) >> 25;  // 7 bits
      while (true) {
        unsigned int s = (slotw[h >> 2] >> ((h & 3) * 8)) & 0xffu;
        if (s == 0xffu) {
          if (len >= LCAP) {
            overflow = true;
            break;
          }
          slotw[h >> 2] = (slotw[h >> 2] & ~(0xffu << ((h & 3) * 8))) | ((unsigned int)len << ((h & 3) * 8));
          key[len] = c;
          val[len] = __dadd_rn(0.0, p);
          ++len;
          break;
        }
        if (key[s] == c) {
          val[s] = __dadd_rn(val[s], p);
          break;
        }
        h = (h + 1) & (HSLOTS - 1);
      }
      if (overflow) break;
    }
  }
  if (PASS == 0) {
    if (overflow) {
      cnt[i] = 0;
      parked[i] = 0;
      big_list[atomicAdd(nbig, 1u)] = i;
      continue;
    }
    int c = 0;
    for (int q = 0; q < len; ++q) c += keep_value(order, val[q]) ? 1 : 0;
    cnt[i] = c;
    // park the finished row (<= TSLOT entries) so the fill pass only copies it
    const bool park = tcol != nullptr && c <= TSLOT;
    parked[i] = park ? 1 : 0;
    if (park) emit_row(order, key, val, len, tcol + (int64_t)i * TSLOT, tval + (int64_t)i * TSLOT);
    continue;
  }
  if (overflow) continue;  // slow path writes this row
  emit_row(order, key, val, len, ccol + crp[i], cval + crp[i]);
  }
}

// Count pass, shared-memory tier: the same walk, list and first-touch sums as
// spgemm_local_kernel, but the row's list (<= SCAP distinct columns) and its
// SHS-slot index live in shared memory, thread-interleaved (entry q of thread
// t at [q][t]: every access of a warp hits 32 distinct banks whatever the
// per-thread slot).  The local-memory tier's 64-entry lists spill out of L1
// at full occupancy (ncu, cfg1 level 0: 24M local sectors at 23% L1 hit, 1.4
// GB of DRAM reads for one product); here nothing leaves the SM.  Every row it
// finishes has <= SCAP <= TSLOT entries, so it is parked for the fill pass;
// longer rows go to `mid` for the local-memory tier (and from there to the
// slow path).
constexpr int SCAP = 32, SHS = 64, SPG_ST = 128;
constexpr size_t SPG_SMEM_BYTES = (size_t)SPG_ST * (SCAP * (sizeof(double) + sizeof(int32_t)) + SHS);
static_assert(SCAP <= TSLOT, "shared-tier rows are always parked");

__global__ void __launch_bounds__(SPG_ST)
spgemm_smem_count_kernel(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                         const double* __restrict__ aval, const int32_t* __restrict__ brp,
                         const int32_t* __restrict__ bcol, const double* __restrict__ bval, int order,
                         int32_t* __restrict__ cnt, int32_t* __restrict__ mid, unsigned int* __restrict__ nmid,
                         int32_t* __restrict__ tcol, double* __restrict__ tval, uint8_t* __restrict__ parked) {
  BAMG_PDL_PROLOGUE();
  extern __shared__ double spg_sm[];
  const int tid = threadIdx.x;
  double* sval = spg_sm + tid;                                                   // [SCAP][SPG_ST]
  int32_t* skey = reinterpret_cast<int32_t*>(spg_sm + SCAP * SPG_ST) + tid;      // [SCAP][SPG_ST]
  unsigned int* sslot = reinterpret_cast<unsigned int*>(spg_sm + SCAP * SPG_ST) + SCAP * SPG_ST + tid;  // [SHS/4][SPG_ST]
  const int i = blockIdx.x * SPG_ST + tid;
  if (i >= n) return;  // no block-wide synchronisation below
#pragma unroll
  for (int w = 0; w < SHS / 4; ++w) sslot[w * SPG_ST] = 0xffffffffu;
  int len = 0;
  bool overflow = false;
  const bool rev_a = (order & SPG_REV_A) != 0, rev_b = (order & SPG_REV_B) != 0;
  const int a0 = arp[i], a1 = arp[i + 1];
  // the insert of one product into the row's list (first-touch order)
  auto insert = [&](int c, double pr) {
    unsigned h = ((unsigned)c * 2654435761u) >> 26;  // 6 bits
    while (true) {
      unsigned int* wp = sslot + (h >> 2) * SPG_ST;
      const unsigned int sh = (h & 3) * 8;
      const unsigned int sl = (*wp >> sh) & 0xffu;
      if (sl == 0xffu) {
        if (len >= SCAP) {
          overflow = true;
          return;
        }
        *wp = (*wp & ~(0xffu << sh)) | ((unsigned int)len << sh);
        skey[len * SPG_ST] = c;
        sval[len * SPG_ST] = __dadd_rn(0.0, pr);
        ++len;
        return;
      }
      if (skey[sl * SPG_ST] == c) {
        sval[sl * SPG_ST] = __dadd_rn(sval[sl * SPG_ST], pr);
        return;
      }
      h = (h + 1) & (SHS - 1);
    }
  };
  // loads batched ahead of the (serial) inserts: four A entries' columns,
  // values and B row bounds, then each B row four entries at a time -- the
  // products are still inserted one by one in scipy's order
  constexpr int CA = 4, CB = 4;
  const int na = a1 - a0;
  for (int ja0 = 0; ja0 < na && !overflow; ja0 += CA) {
    int jb0[CA], jb1[CA];
    double av[CA];
#pragma unroll
    for (int u = 0; u < CA; ++u) {
      const int ja = ja0 + u < na ? ja0 + u : na - 1;
      const int jj = rev_a ? a1 - 1 - ja : a0 + ja;
      const int j = acol[jj];
      av[u] = aval[jj];
      jb0[u] = brp[j];
      jb1[u] = brp[j + 1];
    }
#pragma unroll
    for (int u = 0; u < CA; ++u) {
      if (ja0 + u >= na || overflow) break;
      const int b0 = jb0[u], b1 = jb1[u], nb = b1 - b0;
      const double v = av[u];
      for (int kb0 = 0; kb0 < nb && !overflow; kb0 += CB) {
        int cc[CB];
        double bv[CB];
#pragma unroll
        for (int w = 0; w < CB; ++w) {
          const int kb = kb0 + w < nb ? kb0 + w : nb - 1;
          const int kk = rev_b ? b1 - 1 - kb : b0 + kb;
          cc[w] = bcol[kk];
          bv[w] = bval[kk];
        }
#pragma unroll
        for (int w = 0; w < CB; ++w) {
          if (kb0 + w >= nb || overflow) break;
          insert(cc[w], __dmul_rn(v, bv[w]));
        }
      }
    }
  }
  if (overflow) {
    cnt[i] = 0;
    parked[i] = 0;
    mid[atomicAdd(nmid, 1u)] = i;
    return;
  }
  int kept = 0;
  for (int q = 0; q < len; ++q) kept += keep_value(order, sval[q * SPG_ST]) ? 1 : 0;
  cnt[i] = kept;
  const bool park = tcol != nullptr;
  parked[i] = park ? 1 : 0;
  if (!park) return;
  int32_t* ocol = tcol + (int64_t)i * TSLOT;
  double* oval = tval + (int64_t)i * TSLOT;
  if (order & SPG_STORAGE) {  // reverse first touch
    int w = 0;
    for (int q = len - 1; q >= 0; --q) {
      const double x = sval[q * SPG_ST];
      if (keep_value(order, x)) {
        ocol[w] = skey[q * SPG_ST];
        oval[w] = x;
        ++w;
      }
    }
    return;
  }
  for (int q = 0; q < len; ++q) {  // sorted by column (rank of each kept key)
    const double x = sval[q * SPG_ST];
    if (!keep_value(order, x)) continue;
    const int c = skey[q * SPG_ST];
    int r = 0;
    for (int p2 = 0; p2 < len; ++p2) r += (skey[p2 * SPG_ST] < c && keep_value(order, sval[p2 * SPG_ST])) ? 1 : 0;
    ocol[r] = c;
    oval[r] = x;
  }
}

static bool spgemm_smem_enabled() {
  const char* e = getenv("BAMG_SPGEMM_SMEM");  // development: 0 = local-memory tier only
  return !(e && e[0] == '0');
}

// fill pass for parked rows: one warp per row copies the parking slot
// (coalesced); rows that were not parked go to the redo list for the
// recomputing fill (or the slow path)
__global__ void spgemm_copy_parked_kernel(int n, const uint8_t* __restrict__ parked, const int32_t* __restrict__ crp,
                                          const int32_t* __restrict__ tcol, const double* __restrict__ tval,
                                          int32_t* __restrict__ ccol, double* __restrict__ cval,
                                          int32_t* __restrict__ redo, unsigned int* __restrict__ nredo) {
  BAMG_PDL_PROLOGUE();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int i = (int)w;
  const int b = crp[i], e = crp[i + 1];
  if (!parked[i]) {
    if (lane == 0 && e > b) redo[atomicAdd(nredo, 1u)] = i;
    return;
  }
  if (lane < e - b) {
    ccol[b + lane] = tcol[(int64_t)i * TSLOT + lane];
    cval[b + lane] = tval[(int64_t)i * TSLOT + lane];
  }
}

// slow path over the flagged rows: list in a global scratch slice
// Slow-path rows without a host round trip: the count pass's flagged rows are
// walked grid-stride over the device-resident count; in pass 0 each reserves
// its structural bound sum_j nnz(B_j) from a bump pointer over the context's
// scratch pool (soff[t] = start, or -1 when the pool is exhausted: the count
// call then grows the pool and recounts); pass 1 reuses the reservation.
__device__ __forceinline__ int32_t big_reserve(int i, const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                               const int32_t* __restrict__ brp, unsigned long long* pool_used,
                                               long long pool_cap) {
  long long s = 0;
  for (int jj = arp[i]; jj < arp[i + 1]; ++jj) {
    int j = acol[jj];
    s += brp[j + 1] - brp[j];
  }
  const unsigned long long at = atomicAdd(pool_used, (unsigned long long)s);
  return ((long long)at + s <= pool_cap) ? (int32_t)at : -1;
}

template <int PASS>
__global__ void spgemm_big_kernel(const unsigned int* __restrict__ nbig, const int32_t* __restrict__ list,
                                  const int32_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                  const double* __restrict__ aval, const int32_t* __restrict__ brp,
                                  const int32_t* __restrict__ bcol, const double* __restrict__ bval,
                                  int32_t* __restrict__ soff, int32_t* __restrict__ skey,
                                  double* __restrict__ sval, int order, int32_t* __restrict__ cnt,
                                  const int32_t* __restrict__ crp, int32_t* __restrict__ ccol,
                                  double* __restrict__ cval, unsigned long long* __restrict__ pool_used,
                                  long long pool_cap) {
  BAMG_PDL_PROLOGUE();
  const int nb = (int)*nbig;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
  int i = list[t];
  if (PASS == 0) soff[t] = big_reserve(i, arp, acol, brp, pool_used, pool_cap);
  if (soff[t] < 0) continue;  // pool exhausted: the count call recounts with a larger pool
  int32_t* key = skey + soff[t];
  double* val = sval + soff[t];
  int len = 0;
  const bool rev_a = (order & SPG_REV_A) != 0, rev_b = (order & SPG_REV_B) != 0;
  const int a0 = arp[i], a1 = arp[i + 1];
  for (int ja = 0; ja < a1 - a0; ++ja) {
    const int jj = rev_a ? a1 - 1 - ja : a0 + ja;
    int j = acol[jj];
    double v = aval[jj];
    const int b0 = brp[j], b1 = brp[j + 1];
    for (int kb = 0; kb < b1 - b0; ++kb) {
      const int kk = rev_b ? b1 - 1 - kb : b0 + kb;
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
  if (PASS == 0) {
    int c = 0;
    for (int q = 0; q < len; ++q) c += keep_value(order, val[q]) ? 1 : 0;
    cnt[i] = c;
    continue;
  }
  int w = crp[i];
  if (order & SPG_STORAGE) {
    for (int q = len - 1; q >= 0; --q)
      if (keep_value(order, val[q])) {
        ccol[w] = key[q];
        cval[w] = val[q];
        ++w;
      }
  } else {
    int start = w;
    for (int q = 0; q < len; ++q) {
      if (!keep_value(order, val[q])) continue;
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
  }  // grid-stride over the flagged rows
}

// Memo of the flagged rows between the count and the fill call (owned by the
// context; overwritten by the next count).
struct SpgemmMemo {
  const int32_t* arp = nullptr;
  const int32_t* brp = nullptr;
  int order = -1;
  int nbig = 0;
  unsigned int* nbig_dev = nullptr;  // device flagged-row counter (persistent, read by the fill)
  int32_t* list = nullptr;   // device, capacity cap
  int32_t* off = nullptr;    // device, capacity cap + 1 (per flagged row: scratch start or -1)
  int64_t cap = 0;
  // slow-path scratch pool (bump-allocated on device by spgemm_big_kernel<0>)
  int32_t* pkey = nullptr;
  double* pval = nullptr;
  int64_t pcap = 0;
  unsigned long long* stat = nullptr;  // [pool used, flagged rows, nnz(C)] read back in one sync
  bamg_csr a{}, b{};                   // operands of the pending count (async slots)
  int32_t* rowptr_c = nullptr;
  // parking slots of the count pass (TSLOT entries per row) + flags + redo list
  int32_t* tcol = nullptr;
  double* tval = nullptr;
  uint8_t* parked = nullptr;
  int32_t* redo = nullptr;
  unsigned int* nredo = nullptr;
  int64_t tcap = 0;
};

// SPG_SLOTS independent memos per context: products whose counts are issued
// together (bamg_spgemm_count_slot) and read back with one synchronisation
// (bamg_spgemm_count_wait) each keep their own parked rows and scratch.
constexpr int SPG_SLOTS = 4;

static SpgemmMemo& memo(bamg_ctx* ctx, int slot = 0) {
  if (!ctx->spgemm_memo) ctx->spgemm_memo = new SpgemmMemo[SPG_SLOTS]();
  return ctx->spgemm_memo[slot];
}

void spgemm_memo_release(bamg_ctx* ctx) {
  if (!ctx->spgemm_memo) return;
  for (int s = 0; s < SPG_SLOTS; ++s) {
    SpgemmMemo& m = ctx->spgemm_memo[s];
    for (void* p : {(void*)m.nbig_dev, (void*)m.list, (void*)m.off, (void*)m.pkey, (void*)m.pval, (void*)m.stat,
                    (void*)m.tcol, (void*)m.tval, (void*)m.parked, (void*)m.redo, (void*)m.nredo})
      if (p) cudaFree(p);
  }
  delete[] ctx->spgemm_memo;
  ctx->spgemm_memo = nullptr;
}

static int memo_reserve(bamg_ctx* ctx, SpgemmMemo& m, int64_t n) {
  if (m.tcap < n + 1) {
    cudaFree(m.tcol);
    cudaFree(m.tval);
    cudaFree(m.parked);
    cudaFree(m.redo);
    cudaFree(m.nredo);
    m.tcap = n + 1;
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.tcol, sizeof(int32_t) * TSLOT * m.tcap));
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.tval, sizeof(double) * TSLOT * m.tcap));
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.parked, m.tcap));
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.redo, sizeof(int32_t) * m.tcap));
    BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.nredo, sizeof(unsigned int)));
  }
  if (m.cap >= n + 1) return 0;
  if (m.list) cudaFree(m.list);
  if (m.off) cudaFree(m.off);
  m.cap = n + 1;
  BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.list, sizeof(int32_t) * m.cap));
  BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.off, sizeof(int32_t) * (m.cap + 1)));
  return 0;
}

static int pool_reserve(bamg_ctx* ctx, SpgemmMemo& m, int64_t want) {
  if (!m.stat) BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.stat, sizeof(unsigned long long) * 4));
  m.nbig_dev = reinterpret_cast<unsigned int*>(m.stat + 1);
  if (m.pcap >= want) return 0;
  cudaFree(m.pkey);
  cudaFree(m.pval);
  m.pcap = want;
  BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.pkey, sizeof(int32_t) * m.pcap));
  BAMG_CHECK_CUDA(ctx, cudaMalloc(&m.pval, sizeof(double) * m.pcap));
  return 0;
}

// Count pass in ONE host synchronisation: the flagged (slow-path) rows are
// handled without reading their number -- grid-stride kernels over the
// device-resident count, scratch bump-allocated from the memo's pool -- and
// the pool use, the flagged-row count and nnz(C) come back in one read.  A
// pool overflow (rows too long for the pool) grows it and recounts.
// Count pass of C = A B into memo `m` without reading anything back: the
// pool use, the flagged-row count and nnz(C) land in m.stat.
static int spgemm_count_launch(bamg_ctx* ctx, SpgemmMemo& m, const bamg_csr* A, const bamg_csr* B, int order,
                               int32_t* rowptr_c, bool recount = false) {
  BAMG_REQUIRE(ctx, A && B && A->ncols == B->nrows, "dimension mismatch in sparse product");
  BAMG_REQUIRE(ctx, order >= 0 && order <= 7,
               "order must be 0 (canonical) or 1 (scipy storage order), optionally | 2 (reverse A rows) | 4 (reverse B rows)");
  const int n = A->nrows;
  BAMG_TRY(memo_reserve(ctx, m, n));
  const char* e = recount ? nullptr : getenv("BAMG_SPGEMM_POOL");
  if (e) {  // tests: start from a tiny pool (exercises the regrowth)
    if (m.pcap > atoll(e)) {
      cudaFree(m.pkey);
      cudaFree(m.pval);
      m.pkey = nullptr;
      m.pval = nullptr;
      m.pcap = 0;
    }
    BAMG_TRY(pool_reserve(ctx, m, atoll(e) > 0 ? atoll(e) : 1));
  } else {
    BAMG_TRY(pool_reserve(ctx, m, (int64_t)1 << 20));
  }
  int32_t* cnt;
  // m.stat: [0] pool words used, [1] flagged rows (32-bit counter in the low
  // half), [2] nnz(C) from the scan -- one memset, one read
  unsigned int* nbig = m.nbig_dev;
  BAMG_TRY(arena_get(ctx, (size_t)n + 1, &cnt));
  const int bgrid = ctx->num_sms * 2;
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(m.stat, 0, sizeof(unsigned long long) * 4, ctx->stream));
  if (spgemm_smem_enabled()) {
    // shared-memory tier over every row; its overflow (> SCAP distinct
    // columns) through the local-memory tier (grid-stride over the device
    // count in stat[3]), whose overflow goes to the slow path
    BAMG_TRY(smem_optin(ctx, (const void*)spgemm_smem_count_kernel, SPG_SMEM_BYTES));
    unsigned int* nmid = reinterpret_cast<unsigned int*>(m.stat + 3);
    BAMG_LAUNCH_FAM(ctx, FAM_SPGEMM, 0.0, spgemm_smem_count_kernel, grid_for(n, SPG_ST), SPG_ST, SPG_SMEM_BYTES, n,
                    A->rowptr, A->col, A->val, B->rowptr, B->col, B->val, order, cnt, m.redo, nmid, m.tcol, m.tval,
                    m.parked);
    BAMG_LAUNCH_FAM(ctx, FAM_SPGEMM, 0.0, spgemm_local_kernel<0>, ctx->num_sms * 4, 128, 0, n, A->rowptr, A->col,
                    A->val, B->rowptr, B->col, B->val, order, cnt, m.list, nbig, (const int32_t*)nullptr,
                    (int32_t*)nullptr, (double*)nullptr, m.tcol, m.tval, m.parked, (const int32_t*)m.redo,
                    (const unsigned int*)nmid);
  } else {
    BAMG_LAUNCH_FAM(ctx, FAM_SPGEMM, 0.0, spgemm_local_kernel<0>, grid_for(n, 128), 128, 0, n, A->rowptr, A->col,
                    A->val, B->rowptr, B->col, B->val, order, cnt, m.list, nbig, (const int32_t*)nullptr,
                    (int32_t*)nullptr, (double*)nullptr, m.tcol, m.tval, m.parked, (const int32_t*)nullptr,
                    (const unsigned int*)nullptr);
  }
  BAMG_LAUNCH(ctx, spgemm_big_kernel<0>, bgrid, 128, 0, (const unsigned int*)nbig, m.list, A->rowptr, A->col,
              A->val, B->rowptr, B->col, B->val, m.off, m.pkey, m.pval, order, cnt, (const int32_t*)nullptr,
              (int32_t*)nullptr, (double*)nullptr, m.stat, (long long)m.pcap);
  BAMG_TRY(scan_i32_dev(ctx, cnt, rowptr_c, n, reinterpret_cast<int64_t*>(m.stat + 2)));
  m.a = *A;
  m.b = *B;
  m.rowptr_c = rowptr_c;
  m.arp = A->rowptr;
  m.brp = B->rowptr;
  m.order = order;
  return 0;
}

// Finish counts whose stats were copied to the host: a pool overflow grows
// the pool and recounts that product synchronously (rare).
static int spgemm_count_finish(bamg_ctx* ctx, SpgemmMemo& m, unsigned long long* st, int64_t* nnz_host) {
  st[1] &= 0xffffffffull;
  if ((int64_t)st[0] > m.pcap) {  // slow-path rows did not fit: grow the pool, recount
    BAMG_TRY(pool_reserve(ctx, m, (int64_t)st[0] + ((int64_t)st[0] >> 2)));
    bamg_csr a = m.a, b = m.b;
    ctx->arena.reset();
    BAMG_TRY(spgemm_count_launch(ctx, m, &a, &b, m.order, m.rowptr_c, true));
    BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<const int64_t*>(m.stat), 3, reinterpret_cast<int64_t*>(st)));
    st[1] &= 0xffffffffull;
    BAMG_REQUIRE(ctx, (int64_t)st[0] <= m.pcap, "SpGEMM scratch pool overflow after regrowth");
  }
  m.nbig = (int)st[1];
  *nnz_host = (int64_t)st[2];
  return 0;
}

// Count pass in ONE host synchronisation: the flagged (slow-path) rows are
// handled without reading their number -- grid-stride kernels over the
// device-resident count, scratch bump-allocated from the memo's pool -- and
// the pool use, the flagged-row count and nnz(C) come back in one read.  A
// pool overflow (rows too long for the pool) grows it and recounts.
extern "C" int bamg_spgemm_count(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order, int32_t* rowptr_c,
                                 int64_t* nnz_host) {
  ctx->arena.reset();
  SpgemmMemo& m = memo(ctx, 0);
  BAMG_TRY(spgemm_count_launch(ctx, m, A, B, order, rowptr_c));
  unsigned long long st[3];
  BAMG_TRY(ctx_read_i64(ctx, reinterpret_cast<const int64_t*>(m.stat), 3, reinterpret_cast<int64_t*>(st)));
  return spgemm_count_finish(ctx, m, st, nnz_host);
}

// Asynchronous count into slot `slot` (0..3): nothing is read back until
// bamg_spgemm_count_wait, so independent products share one synchronisation.
extern "C" int bamg_spgemm_count_slot(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                                      int32_t* rowptr_c, int slot) {
  BAMG_REQUIRE(ctx, slot >= 0 && slot < SPG_SLOTS, "slot must lie in [0, 4)");
  ctx->arena.reset();
  return spgemm_count_launch(ctx, memo(ctx, slot), A, B, order, rowptr_c);
}

extern "C" int bamg_spgemm_count_wait(bamg_ctx* ctx, int nslots, const int32_t* slots, int64_t* nnz_host) {
  BAMG_REQUIRE(ctx, nslots >= 1 && nslots <= SPG_SLOTS, "1..4 slots");
  BAMG_REQUIRE(ctx, ctx->pinned_doubles >= (size_t)(3 * SPG_SLOTS), "pinned staging too small");
  unsigned long long* host = reinterpret_cast<unsigned long long*>(ctx->pinned);
  for (int i = 0; i < nslots; ++i) {
    BAMG_REQUIRE(ctx, slots[i] >= 0 && slots[i] < SPG_SLOTS, "slot must lie in [0, 4)");
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(host + 3 * i, memo(ctx, slots[i]).stat, 3 * sizeof(unsigned long long),
                                         cudaMemcpyDeviceToHost, ctx->stream));
  }
  ctx->syncs++;
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  unsigned long long st[3 * SPG_SLOTS];
  memcpy(st, host, sizeof(unsigned long long) * 3 * nslots);
  for (int i = 0; i < nslots; ++i) BAMG_TRY(spgemm_count_finish(ctx, memo(ctx, slots[i]), st + 3 * i, nnz_host + i));
  return 0;
}

static int spgemm_fill_impl(bamg_ctx* ctx, SpgemmMemo& m, const bamg_csr* A, const bamg_csr* B, int order,
                            const int32_t* rowptr_c, int32_t* col_c, double* val_c);

extern "C" int bamg_spgemm_fill(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                                const int32_t* rowptr_c, int32_t* col_c, double* val_c) {
  ctx->arena.reset();
  return spgemm_fill_impl(ctx, memo(ctx, 0), A, B, order, rowptr_c, col_c, val_c);
}

extern "C" int bamg_spgemm_fill_slot(bamg_ctx* ctx, const bamg_csr* A, const bamg_csr* B, int order,
                                     const int32_t* rowptr_c, int32_t* col_c, double* val_c, int slot) {
  BAMG_REQUIRE(ctx, slot >= 0 && slot < SPG_SLOTS, "slot must lie in [0, 4)");
  ctx->arena.reset();
  return spgemm_fill_impl(ctx, memo(ctx, slot), A, B, order, rowptr_c, col_c, val_c);
}

static int spgemm_fill_impl(bamg_ctx* ctx, SpgemmMemo& m, const bamg_csr* A, const bamg_csr* B, int order,
                            const int32_t* rowptr_c, int32_t* col_c, double* val_c) {
  const int n = A->nrows;
  BAMG_REQUIRE(ctx, m.arp == A->rowptr && m.brp == B->rowptr && m.order == order,
               "bamg_spgemm_fill must follow bamg_spgemm_count on the same operands");
  // parked rows are copied; the others (more than TSLOT kept entries) are
  // recomputed by the local kernel over the redo list (slow-path rows return
  // there and are written below)
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(m.nredo, 0, sizeof(unsigned int), ctx->stream));
  static_assert(TSLOT == 32, "one lane per parked entry");
  BAMG_LAUNCH_FAM(ctx, FAM_SPGEMM, 0.0, spgemm_copy_parked_kernel, grid_for((int64_t)n * 32, 256), 256, 0, n, m.parked, rowptr_c,
                  m.tcol, m.tval, col_c, val_c, m.redo, m.nredo);
  {
    int g = grid_for(n, 128);
    if (g > ctx->num_sms * 4) g = ctx->num_sms * 4;
    BAMG_LAUNCH_FAM(ctx, FAM_SPGEMM, 0.0, spgemm_local_kernel<1>, g, 128, 0, n, A->rowptr, A->col, A->val,
                    B->rowptr, B->col, B->val, order, (int32_t*)nullptr, (int32_t*)nullptr, (unsigned int*)nullptr,
                    rowptr_c, col_c, val_c, (int32_t*)nullptr, (double*)nullptr, (uint8_t*)nullptr,
                    (const int32_t*)m.redo, (const unsigned int*)m.nredo);
  }
  if (m.nbig > 0) {
    BAMG_LAUNCH(ctx, spgemm_big_kernel<1>, grid_for(m.nbig, 128), 128, 0, (const unsigned int*)m.nbig_dev, m.list,
                A->rowptr, A->col, A->val, B->rowptr, B->col, B->val, m.off, m.pkey, m.pval, order, (int32_t*)nullptr,
                rowptr_c, col_c, val_c, (unsigned long long*)nullptr, (long long)0);
  }
  return 0;
}
