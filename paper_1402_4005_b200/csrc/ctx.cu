// ctx.cu -- context lifetime, pinned staging, device scans and deterministic
// column reductions shared by every other translation unit.
#include <mutex>

#include "common.cuh"

extern "C" int bamg_version(void) { return BAMG_VERSION; }

extern "C" int bamg_ctx_create(int device, void* cuda_stream, bamg_ctx** out) {
  if (!out) return -2;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return -1;
  bamg_ctx* ctx = new bamg_ctx();
  ctx->device = device;
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) ctx->num_sms = prop.multiProcessorCount;
  ctx->pinned_doubles = 1 << 16;
  if (cudaMallocHost(&ctx->pinned, ctx->pinned_doubles * sizeof(double)) != cudaSuccess) {
    delete ctx;
    return -1;
  }
  if (cudaMalloc(&ctx->counters, 64 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(ctx->counters, 0, 64 * sizeof(unsigned int)) != cudaSuccess) {
    cudaFreeHost(ctx->pinned);
    delete ctx;
    return -1;
  }
  *out = ctx;
  return 0;
}

extern "C" int bamg_ctx_destroy(bamg_ctx* ctx) {
  if (!ctx) return 0;
  cudaStreamSynchronize(ctx->stream);
  fit_slots_release(ctx);
  gmres_work_release(ctx);
  spgemm_memo_release(ctx);
  ctx->arena.release();
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->counters) cudaFree(ctx->counters);
  for (auto& b : ctx->buf_pool) cudaFree(b.first);
  for (auto e : ctx->exec_pool) cudaGraphExecDestroy(e);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  delete ctx;
  return 0;
}

constexpr size_t BUF_POOL_MAX = 16;

// smallest pooled buffer of at least `bytes`, else a fresh allocation
int pool_take(bamg_ctx* ctx, size_t bytes, char** out) {
  int best = -1;
  for (int i = 0; i < (int)ctx->buf_pool.size(); ++i)
    if (ctx->buf_pool[i].second >= bytes && (best < 0 || ctx->buf_pool[i].second < ctx->buf_pool[best].second))
      best = i;
  if (best >= 0) {
    *out = ctx->buf_pool[best].first;
    ctx->buf_pool.erase(ctx->buf_pool.begin() + best);
    return 0;
  }
  BAMG_CHECK_CUDA(ctx, cudaMalloc(out, bytes));
  return 0;
}

void pool_give(bamg_ctx* ctx, char* p, size_t bytes) {
  ctx->buf_pool.push_back({p, bytes});
  while (ctx->buf_pool.size() > BUF_POOL_MAX) {  // drop the smallest
    int s = 0;
    for (int i = 1; i < (int)ctx->buf_pool.size(); ++i)
      if (ctx->buf_pool[i].second < ctx->buf_pool[s].second) s = i;
    cudaFree(ctx->buf_pool[s].first);
    ctx->buf_pool.erase(ctx->buf_pool.begin() + s);
  }
}

int smem_optin(bamg_ctx* ctx, const void* fn, size_t bytes) {
  struct Rec {
    const void* fn;
    int device;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Rec> done;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& r : done)
    if (r.fn == fn && r.device == ctx->device && r.bytes >= bytes) return 0;
  BAMG_CHECK_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  for (auto& r : done)
    if (r.fn == fn && r.device == ctx->device) {
      r.bytes = bytes;
      return 0;
    }
  done.push_back({fn, ctx->device, bytes});
  return 0;
}

extern "C" const char* bamg_last_error(bamg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

extern "C" int64_t bamg_launch_count(bamg_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int64_t bamg_sync_count(bamg_ctx* ctx) { return ctx ? ctx->syncs : 0; }

extern "C" int bamg_sync(bamg_ctx* ctx) {
  ctx->syncs++;
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return 0;
}

static int ctx_read_bytes(bamg_ctx* ctx, const void* dev, size_t bytes, void* host) {
  if (bytes == 0) return 0;
  ctx->syncs++;
  if (ctx->trace.on) {  // zero-length marker: the host waits here
    trace_mark(ctx, "<host sync>");
    trace_mark(ctx, nullptr);
  }
  if (bytes > ctx->pinned_doubles * sizeof(double)) {
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return 0;
  }
  BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(host, ctx->pinned, bytes);
  return 0;
}

int ctx_read_doubles(bamg_ctx* ctx, const double* dev, size_t n, double* host) {
  return ctx_read_bytes(ctx, dev, n * sizeof(double), host);
}
int ctx_read_i64(bamg_ctx* ctx, const int64_t* dev, size_t n, int64_t* host) {
  return ctx_read_bytes(ctx, dev, n * sizeof(int64_t), host);
}
int ctx_read_i32(bamg_ctx* ctx, const int32_t* dev, size_t n, int32_t* host) {
  return ctx_read_bytes(ctx, dev, n * sizeof(int32_t), host);
}

// ------------------------------------------------------------------ scans
// Exclusive scans (CSR row pointers from counts).  Tiles of 4096 elements.
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// Single-pass exclusive scan with decoupled look-back: each CTA takes the
// next tile id from a counter (so predecessors are always running or done),
// publishes its aggregate, then walks back over the predecessors' published
// (flag, value) words until an inclusive prefix is found, and publishes its
// own inclusive prefix.  Integer sums: exact and deterministic.  One launch
// (plus a memset of the state words) instead of three.
constexpr unsigned long long LB_AGG = 1ull, LB_INC = 2ull;

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
scan_onepass_kernel(const T* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                    unsigned long long* __restrict__ state, unsigned int* __restrict__ counter,
                    int64_t* __restrict__ total) {
  BAMG_PDL_PROLOGUE();
  __shared__ int64_t warp_tot[32];
  __shared__ int tile_s;
  __shared__ int64_t excl_s;
  if (threadIdx.x == 0) tile_s = (int)atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = tile_s;
  const int64_t base = (int64_t)tile * SCAN_TILE;
  int64_t v[SCAN_ITEMS];
  int64_t local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    v[i] = idx < n ? (int64_t)in[idx] : 0;
    local += v[i];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc = local;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < (SCAN_THREADS / 32) ? warp_tot[lane] : 0;
    int64_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < (SCAN_THREADS / 32)) warp_tot[lane] = wi - w;
    if (lane == 31) {
      // wi on lane 31 is the tile aggregate
      const int64_t agg = wi;
      int64_t excl = 0;
      if (tile == 0) {
        atomicExch(state, ((unsigned long long)agg << 2) | LB_INC);
      } else {
        atomicExch(state + tile, ((unsigned long long)agg << 2) | LB_AGG);
        for (int p = tile - 1; p >= 0;) {
          unsigned long long wv = *(volatile unsigned long long*)(state + p);
          unsigned long long f = wv & 3ull;
          if (f == 0) continue;  // predecessor still computing its aggregate
          excl += (int64_t)(wv >> 2);
          if (f == LB_INC) break;
          --p;
        }
        atomicExch(state + tile, ((unsigned long long)(excl + agg) << 2) | LB_INC);
      }
      excl_s = excl;
      if (tile == (int)gridDim.x - 1) {
        out[n] = (int32_t)(excl + agg);
        *total = excl + agg;
      }
    }
  }
  __syncthreads();
  int64_t run = excl_s + warp_tot[wid] + inc - local;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    if (idx < n) out[idx] = (int32_t)run;
    run += v[i];
  }
}

template <typename T>
static int scan_impl(bamg_ctx* ctx, const T* in, int32_t* out, int64_t n, int64_t* total_host,
                     int64_t* total_dev = nullptr) {
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles < 1) tiles = 1;
  // state words (tiles) + tile counter + total, one memset
  unsigned long long* state = nullptr;
  BAMG_TRY(arena_get(ctx, (size_t)tiles + 2, &state));
  BAMG_CHECK_CUDA(ctx, cudaMemsetAsync(state, 0, sizeof(unsigned long long) * ((size_t)tiles + 2), ctx->stream));
  unsigned int* counter = reinterpret_cast<unsigned int*>(state + tiles);
  int64_t* total = total_dev ? total_dev : reinterpret_cast<int64_t*>(state + tiles + 1);
  BAMG_LAUNCH(ctx, scan_onepass_kernel<T>, (int)tiles, SCAN_THREADS, 0, in, n, out, state, counter, total);
  if (total_host) BAMG_TRY(ctx_read_i64(ctx, total, 1, total_host));
  return 0;
}

int scan_i32(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int64_t* total_host) {
  return scan_impl<int32_t>(ctx, in, out, n, total_host);
}
int scan_i32_dev(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int64_t* total_dev) {
  return scan_impl<int32_t>(ctx, in, out, n, nullptr, total_dev);
}
int scan_u8(bamg_ctx* ctx, const uint8_t* in, int32_t* out, int64_t n, int64_t* total_host) {
  return scan_impl<uint8_t>(ctx, in, out, n, total_host);
}

// ------------------------------------------------- deterministic colreduce
constexpr int KMAX = 32;

// Column sums of squares (kind 0) or of products (kind 1) of n x k blocks in
// ONE launch: RED_BLOCKS CTAs write per-CTA partials; the last CTA to arrive
// (arrival counter, self-resetting) reduces them in a fixed order -- per
// column, lanes stride over the CTAs, then a warp tree -- so the result is
// bit-reproducible run to run.
// KK > 0: k == KK at compile time, each thread loading UR rows before it
// accumulates them (in the same row order, so the sums are bit-identical to
// the generic form -- only more loads are in flight); KK == 0: any k <= KMAX.
template <int KK, int UR>
__global__ void __launch_bounds__(RED_THREADS)
colreduce_kernel(const double* __restrict__ X, const double* __restrict__ Y, int64_t n, int k_rt, int kind,
                 double* __restrict__ partial, unsigned int* __restrict__ counter, double* __restrict__ out,
                 int take_sqrt) {
  BAMG_PDL_PROLOGUE();
  constexpr int KA = KK > 0 ? KK : KMAX;  // accumulators
  const int k = KK > 0 ? KK : k_rt;
  __shared__ double sh[RED_THREADS / 32][KMAX];
  __shared__ bool last;
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = r0 + per < n ? r0 + per : n;
  double acc[KA];
#pragma unroll
  for (int c = 0; c < KA; ++c) acc[c] = 0.0;
  int64_t r = r0 + threadIdx.x;
  if constexpr (KK > 0) {
    const int64_t step = blockDim.x;
    for (; r + (UR - 1) * step < r1; r += UR * step) {
      double xv[UR][KK], yv[UR][KK];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const double* xr = X + (r + u * step) * KK;
#pragma unroll
        for (int c = 0; c < KK; ++c) xv[u][c] = xr[c];
        if (kind != 0) {
          const double* yr = Y + (r + u * step) * KK;
#pragma unroll
          for (int c = 0; c < KK; ++c) yv[u][c] = yr[c];
        }
      }
#pragma unroll
      for (int u = 0; u < UR; ++u)
#pragma unroll
        for (int c = 0; c < KK; ++c) acc[c] += xv[u][c] * (kind == 0 ? xv[u][c] : yv[u][c]);
    }
  }
  for (; r < r1; r += blockDim.x) {
    const double* xr = X + r * k;
    if (kind == 0) {
#pragma unroll
      for (int c = 0; c < KA; ++c)
        if (c < k) acc[c] += xr[c] * xr[c];
    } else {
      const double* yr = Y + r * k;
#pragma unroll
      for (int c = 0; c < KA; ++c)
        if (c < k) acc[c] += xr[c] * yr[c];
    }
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < KA; ++c) {
    if (c < k) {
      double v = warp_sum(acc[c]);
      if (lane == 0) sh[wid][c] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double v = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) v += sh[w][threadIdx.x];
    partial[(int64_t)blockIdx.x * k + threadIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nb = gridDim.x;
  for (int c = wid; c < k; c += RED_THREADS / 32) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(partial + (int64_t)b * k + c);
    v = warp_sum(v);
    if (lane == 0) out[c] = take_sqrt ? sqrt(v) : v;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// k = 8 / 16 with 16-byte aligned blocks: the CTA's row chunk read as one flat
// stream of double2 (fully coalesced; the row-per-thread form above touches 32
// lines per load instruction and ran at 2.1 TB/s on cfg4's level 0).  A
// thread's stride is a whole number of rows, so it always sees the same column
// pair; UR loads are in flight per thread.  Fixed order: thread partials, then
// per column the 256 / (KK / 2) owning threads in ascending order, then the
// last CTA's pass over the per-CTA partials as above.
template <int KK, int UR>
__global__ void __launch_bounds__(RED_THREADS)
colreduce_wide_kernel(const double* __restrict__ X, const double* __restrict__ Y, int64_t n, int kind,
                      double* __restrict__ partial, unsigned int* __restrict__ counter, double* __restrict__ out,
                      int take_sqrt) {
  BAMG_PDL_PROLOGUE();
  // KK == 1: one vector read as double2 (both halves belong to the column; an odd tail element
  // is added by the CTA that owns it)
  constexpr int PAIRS = KK == 1 ? 1 : KK / 2;
  static_assert(RED_THREADS % PAIRS == 0, "a thread must keep its column pair");
  __shared__ double sh[RED_THREADS][2];
  __shared__ bool last;
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  if (KK == 1) per = (per + 1) & ~(int64_t)1;  // even chunks keep the double2 loads aligned
  const int64_t r0 = min((int64_t)blockIdx.x * per, n);
  const int64_t r1 = r0 + per < n ? r0 + per : n;
  const double2* X2 = reinterpret_cast<const double2*>(X);
  const double2* Y2 = reinterpret_cast<const double2*>(Y);
  const int64_t u1 = KK == 1 ? r1 / 2 : r1 * PAIRS;
  double a0 = 0.0, a1 = 0.0;
  int64_t u = (KK == 1 ? r0 / 2 : r0 * PAIRS) + threadIdx.x;
  if (KK == 1 && (r1 & 1) && r1 == n && r0 < r1 && threadIdx.x == 0) {
    const double xl = X[n - 1];
    a0 = xl * (kind == 0 ? xl : Y[n - 1]);
  }
  for (; u + (int64_t)(UR - 1) * RED_THREADS < u1; u += (int64_t)UR * RED_THREADS) {
    double2 xv[UR], yv[UR];
#pragma unroll
    for (int i = 0; i < UR; ++i) {
      xv[i] = X2[u + (int64_t)i * RED_THREADS];
      if (kind != 0) yv[i] = Y2[u + (int64_t)i * RED_THREADS];
    }
#pragma unroll
    for (int i = 0; i < UR; ++i) {
      a0 += xv[i].x * (kind == 0 ? xv[i].x : yv[i].x);
      a1 += xv[i].y * (kind == 0 ? xv[i].y : yv[i].y);
    }
  }
  for (; u < u1; u += RED_THREADS) {
    const double2 xv = X2[u];
    const double2 yv = kind == 0 ? xv : Y2[u];
    a0 += xv.x * yv.x;
    a1 += xv.y * yv.y;
  }
  sh[threadIdx.x][0] = a0;
  sh[threadIdx.x][1] = a1;
  __syncthreads();
  if (KK == 1) {
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int t = 0; t < RED_THREADS; ++t) v += sh[t][0] + sh[t][1];
      partial[blockIdx.x] = v;
    }
  } else if (threadIdx.x < KK) {
    const int c = threadIdx.x;
    // the chunk starts on a row boundary: thread t owns columns 2 (t % PAIRS), + 1
    double v = 0.0;
    for (int t = c / 2; t < RED_THREADS; t += PAIRS) v += sh[t][c & 1];
    partial[(int64_t)blockIdx.x * KK + c] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nb = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c = wid; c < KK; c += RED_THREADS / 32) {
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += __ldcg(partial + (int64_t)b * KK + c);
    v = warp_sum(v);
    if (lane == 0) out[c] = take_sqrt ? sqrt(v) : v;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

int colreduce(bamg_ctx* ctx, const double* X, const double* Y, int64_t n, int k, int kind,
              double* out_dev, int take_sqrt) {
  BAMG_REQUIRE(ctx, k >= 1 && k <= KMAX, "k must lie in [1, 32]");
  double* partial = nullptr;
  BAMG_TRY(arena_get(ctx, (size_t)RED_BLOCKS * k, &partial));
  const int g = red_blocks_for(n);
  const bool al16 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) == 0;
  if (k == 16 && al16)
    BAMG_LAUNCH(ctx, (colreduce_wide_kernel<16, 8>), g, RED_THREADS, 0, X, Y, n, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else if (k == 1 && al16)
    BAMG_LAUNCH(ctx, (colreduce_wide_kernel<1, 8>), g, RED_THREADS, 0, X, Y, n, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else if (k == 8 && al16)
    BAMG_LAUNCH(ctx, (colreduce_wide_kernel<8, 8>), g, RED_THREADS, 0, X, Y, n, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else if (k == 8)
    BAMG_LAUNCH(ctx, (colreduce_kernel<8, 4>), g, RED_THREADS, 0, X, Y, n, k, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else if (k == 16)
    BAMG_LAUNCH(ctx, (colreduce_kernel<16, 2>), g, RED_THREADS, 0, X, Y, n, k, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else if (k == 1)
    BAMG_LAUNCH(ctx, (colreduce_kernel<1, 8>), g, RED_THREADS, 0, X, Y, n, k, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  else
    BAMG_LAUNCH(ctx, (colreduce_kernel<0, 1>), g, RED_THREADS, 0, X, Y, n, k, kind, partial, ctx->counters + 0,
                out_dev, take_sqrt);
  return 0;
}

extern "C" int bamg_col_norms(bamg_ctx* ctx, const double* X, int64_t n, int k, double* out) {
  ctx->arena.reset();
  return colreduce(ctx, X, nullptr, n, k, 0, out, 1);
}

extern "C" int bamg_col_dots(bamg_ctx* ctx, const double* X, const double* Y, int64_t n, int k,
                             double* out) {
  ctx->arena.reset();
  return colreduce(ctx, X, Y, n, k, 1, out, 0);
}

// n x k block kernels: one thread per row walking its k entries (no 64-bit
// div/mod per element; a row is one contiguous 8k-byte segment)
// x / d through the CTA's reciprocals of the k divisors (div_rn_recip:
// bit-identical to the IEEE quotient; a full fp64 division per element held
// this streaming kernel near 45 % of HBM bandwidth).  KK > 0: the row's k
// values are loaded before any is stored (X is read and written in place, so
// a rolled loop would serialise load -> divide -> store per element).
template <int KK>
__global__ void col_scale_div_kernel(double* X, int64_t n, int k_rt, const double* s, int fill_c, double fill_v) {
  BAMG_PDL_PROLOGUE();
  const int k = KK > 0 ? KK : k_rt;
  __shared__ double sd[KMAX], srd[KMAX];
  if (threadIdx.x < k) {
    double d = s[threadIdx.x];
    if (d == 0.0) d = 1.0;
    sd[threadIdx.x] = d;
    srd[threadIdx.x] = 1.0 / d;
  }
  __syncthreads();
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double* x = X + r * k;
  if constexpr (KK > 0) {
    double v[KK];
#pragma unroll
    for (int c = 0; c < KK; ++c) v[c] = x[c];
#pragma unroll
    for (int c = 0; c < KK; ++c) x[c] = c == fill_c ? fill_v : div_rn_recip(v[c], sd[c], srd[c]);
  } else {
    for (int c = 0; c < k; ++c) x[c] = c == fill_c ? fill_v : div_rn_recip(x[c], sd[c], srd[c]);
  }
}

// Flat form for k in {8, 16}: one double2 per thread, consecutive threads on
// consecutive 16-byte words (the row-per-thread form's loads and stores were
// 8 bytes at a 64-byte stride per lane).
template <int KK>
__global__ void col_scale_div_flat_kernel(double* X, int64_t total2, const double* s, int fill_c, double fill_v,
                                          const double* src) {
  BAMG_PDL_PROLOGUE();
  static_assert(KK % 2 == 0 && (KK & (KK - 1)) == 0, "power-of-two k");
  __shared__ double sd[KK], srd[KK];
  if (threadIdx.x < KK) {
    double d = s[threadIdx.x];
    if (d == 0.0) d = 1.0;
    sd[threadIdx.x] = d;
    srd[threadIdx.x] = 1.0 / d;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total2) return;
  double2* x2 = reinterpret_cast<double2*>(X);
  double2 v = src ? reinterpret_cast<const double2*>(src)[i] : x2[i];  // src: out-of-place (X = src / s)
  const int c = (int)((2 * i) & (KK - 1));
  v.x = c == fill_c ? fill_v : div_rn_recip(v.x, sd[c], srd[c]);
  v.y = c + 1 == fill_c ? fill_v : div_rn_recip(v.y, sd[c + 1], srd[c + 1]);
  x2[i] = v;
}

// X[:, c] /= s[c]; fill_c >= 0: column fill_c is set to fill_v instead (the
// refresh's normalise-then-overwrite of the first test vector in one pass)
int col_scale_div_dev(bamg_ctx* ctx, double* X, int64_t n, int k, const double* s, int fill_c, double fill_v,
                      const double* src) {
  const bool al16 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (src && src != X && !((k == 8 || k == 16) && al16)) {  // only the flat kernels divide out of place
    BAMG_CHECK_CUDA(ctx, cudaMemcpyAsync(X, src, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, ctx->stream));
    src = nullptr;
  }
  if (src == X) src = nullptr;
  if (k == 8 && al16)
    BAMG_LAUNCH(ctx, col_scale_div_flat_kernel<8>, grid_for(n * 4, 256), 256, 0, X, n * 4, s, fill_c, fill_v, src);
  else if (k == 16 && al16)
    BAMG_LAUNCH(ctx, col_scale_div_flat_kernel<16>, grid_for(n * 8, 256), 256, 0, X, n * 8, s, fill_c, fill_v, src);
  else if (k == 8)
    BAMG_LAUNCH(ctx, col_scale_div_kernel<8>, grid_for(n, 256), 256, 0, X, n, k, s, fill_c, fill_v);
  else if (k == 16)
    BAMG_LAUNCH(ctx, col_scale_div_kernel<16>, grid_for(n, 256), 256, 0, X, n, k, s, fill_c, fill_v);
  else
    BAMG_LAUNCH(ctx, col_scale_div_kernel<0>, grid_for(n, 256), 256, 0, X, n, k, s, fill_c, fill_v);
  return 0;
}

extern "C" int bamg_col_scale_div(bamg_ctx* ctx, double* X, int64_t n, int k, const double* s) {
  return col_scale_div_dev(ctx, X, n, k, s, -1, 0.0, nullptr);
}

__global__ void col_fill_kernel(double* X, int64_t n, int k, int c, double value) {
  BAMG_PDL_PROLOGUE();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) X[i * k + c] = value;
}

int col_fill_dev(bamg_ctx* ctx, double* X, int64_t n, int k, int c, double value) {
  BAMG_LAUNCH(ctx, col_fill_kernel, grid_for(n, 256), 256, 0, X, n, k, c, value);
  return 0;
}

extern "C" int bamg_col_fill(bamg_ctx* ctx, double* X, int64_t n, int k, int c, double value) {
  return col_fill_dev(ctx, X, n, k, c, value);
}

__global__ void gather_rows_kernel(const double* __restrict__ X, const int32_t* __restrict__ idx,
                                   int64_t m, int k, double* __restrict__ Y) {
  BAMG_PDL_PROLOGUE();
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double* x = X + (int64_t)idx[r] * k;
  double* y = Y + r * k;
  for (int c = 0; c < k; ++c) y[c] = x[c];
}

// k in {8, 16}: one double2 per thread (coalesced stores, 16-byte loads)
template <int KK>
__global__ void gather_rows_flat_kernel(const double* __restrict__ X, const int32_t* __restrict__ idx,
                                        int64_t total2, double* __restrict__ Y) {
  BAMG_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total2) return;
  constexpr int H = KK / 2;
  const int64_t r = i / H;
  const int c2 = (int)(i & (H - 1));
  reinterpret_cast<double2*>(Y)[i] = reinterpret_cast<const double2*>(X + (int64_t)idx[r] * KK)[c2];
}

extern "C" int bamg_gather_rows(bamg_ctx* ctx, const double* X, const int32_t* idx, int64_t m,
                                int k, double* Y) {
  const bool al16 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) == 0;
  if (al16 && k == 8)
    BAMG_LAUNCH(ctx, gather_rows_flat_kernel<8>, grid_for(m * 4, 256), 256, 0, X, idx, m * 4, Y);
  else if (al16 && k == 16)
    BAMG_LAUNCH(ctx, gather_rows_flat_kernel<16>, grid_for(m * 8, 256), 256, 0, X, idx, m * 8, Y);
  else
    BAMG_LAUNCH(ctx, gather_rows_kernel, grid_for(m, 256), 256, 0, X, idx, m, k, Y);
  return 0;
}

struct Perm32 {
  int32_t p[32];
};

__global__ void permute_cols_kernel(const double* __restrict__ X, int64_t n, int k, Perm32 perm, double* __restrict__ Y) {
  BAMG_PDL_PROLOGUE();
  __shared__ int sp[32];
  if (threadIdx.x < 32) sp[threadIdx.x] = perm.p[threadIdx.x];
  __syncthreads();
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double* x = X + r * k;
  double* y = Y + r * k;
  for (int c = 0; c < k; ++c) y[c] = x[sp[c]];
}

// k in {8, 16}: one output double2 per thread (coalesced stores; the two
// sources lie in the same 8k-byte row)
template <int KK>
__global__ void permute_cols_flat_kernel(const double* __restrict__ X, int64_t total2, Perm32 perm,
                                         double* __restrict__ Y) {
  BAMG_PDL_PROLOGUE();
  __shared__ int sp[32];
  if (threadIdx.x < 32) sp[threadIdx.x] = perm.p[threadIdx.x];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total2) return;
  const int64_t e = 2 * i;
  const int c = (int)(e & (KK - 1));
  const double* x = X + (e - c);
  reinterpret_cast<double2*>(Y)[i] = make_double2(x[sp[c]], x[sp[c + 1]]);
}

extern "C" int bamg_permute_cols(bamg_ctx* ctx, const double* X, int64_t n, int k, const int32_t* perm_host,
                                 double* Y) {
  BAMG_REQUIRE(ctx, k >= 1 && k <= 32 && X != Y, "k in [1, 32] and distinct buffers");
  Perm32 p{};
  for (int c = 0; c < k; ++c) p.p[c] = perm_host[c];
  const bool al16 = (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  if (al16 && k == 8)
    BAMG_LAUNCH(ctx, permute_cols_flat_kernel<8>, grid_for(n * 4, 256), 256, 0, X, n * 4, p, Y);
  else if (al16 && k == 16)
    BAMG_LAUNCH(ctx, permute_cols_flat_kernel<16>, grid_for(n * 8, 256), 256, 0, X, n * 8, p, Y);
  else
    BAMG_LAUNCH(ctx, permute_cols_kernel, grid_for(n, 256), 256, 0, X, n, k, p, Y);
  return 0;
}

extern "C" int bamg_prof_enable(bamg_ctx* ctx, unsigned mask) {
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->prof.mask = mask;
  for (int f = 0; f < NFAM; ++f) {
    ctx->prof.used[f] = 0;
    ctx->prof.bytes[f] = 0.0;
    ctx->prof.flops[f] = 0.0;
  }
  return 0;
}

// total device milliseconds, launch count and algorithmic bytes of family fam
extern "C" int bamg_prof_read(bamg_ctx* ctx, int fam, double* ms_host, int64_t* launches_host,
                              double* bytes_host) {
  BAMG_REQUIRE(ctx, fam >= 0 && fam < NFAM, "family out of range");
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  KProf& P = ctx->prof;
  double tot = 0.0;
  for (size_t i = 0; i + 1 < P.used[fam]; i += 2) {
    float ms = 0.f;
    BAMG_CHECK_CUDA(ctx, cudaEventElapsedTime(&ms, P.ev[fam][i], P.ev[fam][i + 1]));
    tot += ms;
  }
  *ms_host = tot;
  *launches_host = (int64_t)(P.used[fam] / 2);
  *bytes_host = P.bytes[fam];
  return 0;
}

#include <map>

extern "C" int bamg_trace_enable(bamg_ctx* ctx, int on) {
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->trace.on = on != 0;
  ctx->trace.used = 0;
  return 0;
}

// Writes "name total_ms count" lines (aggregated by kernel name) into buf.
// Per-launch timeline "name<TAB>start_us<TAB>end_us" (relative to the first
// traced event), in launch order: gaps between consecutive launches are
// pipeline bubbles (host syncs, host-side work, launch latency).
extern "C" int bamg_trace_timeline(bamg_ctx* ctx, char* buf, int64_t cap) {
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  KTrace& T = ctx->trace;
  std::string out;
  for (size_t i = 0; i + 1 < T.used; ++i) {
    if (!T.name[i] || T.name[i + 1]) continue;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, T.ev[0], T.ev[i]);
    cudaEventElapsedTime(&b, T.ev[0], T.ev[i + 1]);
    out += std::string(T.name[i]) + "\t" + std::to_string(a * 1e3) + "\t" + std::to_string(b * 1e3) + "\t" +
           std::to_string(i) + "\n";
  }
  int64_t len = (int64_t)out.size();
  if (len >= cap) len = cap - 1;
  memcpy(buf, out.data(), len);
  buf[len] = 0;
  return 0;
}

// Current trace position (events recorded so far): phase markers for the timeline.
extern "C" int64_t bamg_trace_position(bamg_ctx* ctx) { return ctx ? (int64_t)ctx->trace.used : 0; }

extern "C" int bamg_trace_dump(bamg_ctx* ctx, char* buf, int64_t cap) {
  BAMG_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::map<std::string, std::pair<double, int64_t>> agg;
  KTrace& T = ctx->trace;
  for (size_t i = 0; i + 1 < T.used; ++i) {
    if (!T.name[i] || T.name[i + 1]) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, T.ev[i], T.ev[i + 1]);
    auto& a = agg[T.name[i]];
    a.first += ms;
    a.second += 1;
  }
  std::string out;
  for (auto& kv : agg) out += kv.first + "\t" + std::to_string(kv.second.first) + "\t" + std::to_string(kv.second.second) + "\n";
  int64_t len = (int64_t)out.size();
  if (len >= cap) len = cap - 1;
  memcpy(buf, out.data(), len);
  buf[len] = 0;
  return 0;
}
