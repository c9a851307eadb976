// common.cuh -- shared plumbing for libbamg_sm100.so (context, arena, launch
// accounting, deterministic block reductions, device scan).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/bamg_sm100.h"

#define BAMG_VERSION 1

// Per-call scratch: one bump-allocated slab sized to the high-water mark of
// previous calls.  A call that outgrows the slab takes overflow blocks; the
// next reset (at API entry, all earlier users already enqueued on the same
// stream) frees them and regrows the slab once, so steady-state calls never
// touch cudaMalloc.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0, call_peak = 0, peak = 0;
  std::vector<char*> overflow;
  void reset() {
    if (!overflow.empty() || peak > cap) {
      cudaDeviceSynchronize();
      for (char* p : overflow) cudaFree(p);
      overflow.clear();
      if (peak > cap) {
        if (base) cudaFree(base);
        cap = peak + peak / 4 + (size_t(16) << 20);
        if (cudaMalloc(&base, cap) != cudaSuccess) {
          base = nullptr;
          cap = 0;
        }
      }
    }
    used = 0;
    call_peak = 0;
  }
  cudaError_t get(size_t bytes, void** out) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    call_peak += bytes;
    if (call_peak > peak) peak = call_peak;
    if (base && used + bytes <= cap) {
      *out = base + used;
      used += bytes;
      return cudaSuccess;
    }
    char* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return e;
    overflow.push_back(p);
    *out = p;
    return cudaSuccess;
  }
  void release() {
    for (char* p : overflow) cudaFree(p);
    overflow.clear();
    if (base) cudaFree(base);
    base = nullptr;
    cap = used = 0;
  }
};

// Per-family kernel timing with CUDA events on the launching stream
// (bench.py's live roofline).  Off unless bamg_prof_enable() set the family.
// FAM_TILE_FINE: the CSR row kernels on operators with >= 2^18 rows (the
// finest levels), reported beside the whole CSR family (FAM_TILE + FINE)
enum { FAM_TILE = 0, FAM_FIT = 1, FAM_SPGEMM = 2, FAM_ORTHO = 3, FAM_DENSE = 4, FAM_OTHER = 5, FAM_TILE_FINE = 6,
       NFAM = 7 };
constexpr int FINE_ROWS = 1 << 18;

struct KProf {
  unsigned mask = 0;
  std::vector<cudaEvent_t> ev[NFAM];  // start/stop pairs
  size_t used[NFAM] = {};
  double bytes[NFAM] = {};
  double flops[NFAM] = {};
  // batched[f]: launches of family f add their bytes but no event pair; the
  // caller times the whole batch with one pair on the context stream (the
  // LS-fit slots overlap on side streams: per-launch pairs would count the
  // overlapped time twice)
  bool batched[NFAM] = {};
};

// Whole-engine launch trace (development): every BAMG_LAUNCH brackets its
// kernel with an event pair tagged by the kernel's name.
struct KTrace {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> name;
  size_t used = 0;
};

struct bamg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t launches = 0;
  int64_t syncs = 0;  // host waits on the stream (small D2H reads, bamg_sync)
  std::string err;
  Arena arena;
  double* pinned = nullptr;  // small pinned host staging buffer
  size_t pinned_doubles = 0;
  KProf prof;
  KTrace trace;
  // V-cycle graph plumbing recycled across hierarchies (one hierarchy per
  // setup; a solve loop builds one per step): the capture stream, the level
  // buffers and the instantiated graphs (re-pointed by cudaGraphExecUpdate),
  // so steady-state steps make no cudaMalloc/cudaFree/instantiate calls.
  cudaStream_t cap_stream = nullptr;
  // zero-initialised arrival counters for single-launch ("last CTA finishes")
  // reductions; every user resets its counter to 0 before exiting
  unsigned int* counters = nullptr;
  std::vector<std::pair<char*, size_t>> buf_pool;
  std::vector<cudaGraphExec_t> exec_pool;
  // per-context state of the translation units, created on first use and
  // released by bamg_ctx_destroy (no process-wide tables keyed by address)
  struct FitSlots* fit_slots = nullptr;          // interp.cu
  // bamg_fit_set_row_range: the LS fits only produce rows [fit_lo, fit_hi) (multi-GPU setup:
  // every rank fits its row block, the blocks are all-gathered); fit_lo < 0 = every row
  int64_t fit_lo = -1, fit_hi = -1;
  struct GmresWork* gmres_work = nullptr;        // solver.cu
  struct SpgemmMemo* spgemm_memo = nullptr;      // spgemm.cu (SPG_SLOTS entries)
};

void fit_slots_release(bamg_ctx* ctx);
void gmres_work_release(bamg_ctx* ctx);
void spgemm_memo_release(bamg_ctx* ctx);

static inline void trace_mark(bamg_ctx* ctx, const char* name) {
  KTrace& T = ctx->trace;
  if (T.used >= T.ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    T.ev.push_back(e);
    T.name.push_back(nullptr);
  }
  T.name[T.used] = name;
  cudaEventRecord(T.ev[T.used++], ctx->stream);
}

// event pair around one launch of family `fam` (no-op unless profiled)
static inline cudaEvent_t prof_event(bamg_ctx* ctx, int fam) {
  KProf& P = ctx->prof;
  if (P.used[fam] >= P.ev[fam].size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    P.ev[fam].push_back(e);
  }
  return P.ev[fam][P.used[fam]++];
}

#define BAMG_LAUNCH_FAM(ctx, fam, nbytes, kernel, grid, block, smem, ...)       \
  do {                                                                          \
    bool _prof = ((ctx)->prof.mask >> (fam)) & 1u;                              \
    bool _ev = _prof && !(ctx)->prof.batched[fam];                              \
    if (_prof && (grid) > 0) (ctx)->prof.bytes[fam] += (double)(nbytes);        \
    if (_ev && (grid) > 0) cudaEventRecord(prof_event(ctx, fam), (ctx)->stream); \
    BAMG_LAUNCH(ctx, kernel, grid, block, smem, __VA_ARGS__);                   \
    if (_ev && (grid) > 0) cudaEventRecord(prof_event(ctx, fam), (ctx)->stream); \
  } while (0)

// ---------------------------------------------------------------- error glue
#define BAMG_CHECK_CUDA(ctx, expr)                                              \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(_e) +         \
                   " at " + __FILE__ + ":" + std::to_string(__LINE__);          \
      return -1;                                                                \
    }                                                                           \
  } while (0)

#define BAMG_REQUIRE(ctx, cond, msg)                                            \
  do {                                                                          \
    if (!(cond)) {                                                              \
      (ctx)->err = std::string("argument error: ") + (msg);                     \
      return -2;                                                                \
    }                                                                           \
  } while (0)

// Programmatic dependent launch (PDL).  Every engine kernel starts with
// BAMG_PDL_PROLOGUE: griddepcontrol.wait blocks until the preceding grid in
// the stream has completed and its writes are visible, so kernel bodies stay
// strictly stream-ordered; launch_dependents then lets the NEXT launch be
// scheduled while this grid runs.  With BAMG_LAUNCH's
// ProgrammaticStreamSerialization attribute the launch latency of kernel i+1
// (grid setup, CTA rasterisation) overlaps the tail of kernel i instead of
// sitting in the ~1,700 serial kernel boundaries of a setup + solve.  Both
// instructions are no-ops for kernels launched without the attribute.
#define BAMG_PDL_PROLOGUE() \
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

static inline bool bamg_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BAMG_NO_PDL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
static inline cudaError_t bamg_launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                          cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launch + accounting + immediate launch-error check.
#define BAMG_LAUNCH(ctx, kernel, grid, block, smem, ...)                        \
  do {                                                                          \
    if ((grid) > 0) {                                                           \
      if ((ctx)->trace.on) trace_mark(ctx, #kernel);                            \
      if (bamg_pdl_enabled()) {                                                 \
        BAMG_CHECK_CUDA(ctx, bamg_launch_pdl(kernel, dim3(grid), dim3(block), (size_t)(smem), \
                                             (ctx)->stream, __VA_ARGS__));     \
      } else {                                                                  \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);        \
      }                                                                         \
      (ctx)->launches++;                                                        \
      BAMG_CHECK_CUDA(ctx, cudaGetLastError());                                 \
      if ((ctx)->trace.on) trace_mark(ctx, nullptr);                            \
    }                                                                           \
  } while (0)

// Launch with a 3-D grid / 2-D block (no PDL attribute; accounting + error check).
#define BAMG_LAUNCH_GRID3(ctx, kernel, grid3, block3, smem, ...)                \
  do {                                                                          \
    if ((ctx)->trace.on) trace_mark(ctx, #kernel);                              \
    kernel<<<(grid3), (block3), (smem), (ctx)->stream>>>(__VA_ARGS__);          \
    (ctx)->launches++;                                                          \
    BAMG_CHECK_CUDA(ctx, cudaGetLastError());                                   \
    if ((ctx)->trace.on) trace_mark(ctx, nullptr);                              \
  } while (0)

#define BAMG_TRY(expr)                                                          \
  do {                                                                          \
    int _rc = (expr);                                                           \
    if (_rc != 0) return _rc;                                                   \
  } while (0)

template <typename T>
static inline int arena_get(bamg_ctx* ctx, size_t count, T** out) {
  void* p = nullptr;
  cudaError_t e = ctx->arena.get(count * sizeof(T), &p);
  if (e != cudaSuccess) {
    ctx->err = std::string("workspace allocation failed: ") + cudaGetErrorString(e);
    return -1;
  }
  *out = static_cast<T*>(p);
  return 0;
}

// Opt a kernel in to `bytes` of dynamic shared memory on the context's device.
// The attribute is per (function, device): recorded in a process-wide table so
// a second device in the same process gets its own cudaFuncSetAttribute.
int smem_optin(bamg_ctx* ctx, const void* fn, size_t bytes);

// Device buffers recycled across setups on the context's stream (V-cycle
// level slabs, the banded coarsest factor): take the smallest pooled buffer
// of at least `bytes` (else cudaMalloc); give one back (stream-ordered reuse:
// no synchronisation, later users are enqueued after earlier ones).
int pool_take(bamg_ctx* ctx, size_t bytes, char** out);
void pool_give(bamg_ctx* ctx, char* p, size_t bytes);

// Pinned staging for small device->host reads (synchronises the stream).
int ctx_read_doubles(bamg_ctx* ctx, const double* dev, size_t n, double* host);
int ctx_read_i64(bamg_ctx* ctx, const int64_t* dev, size_t n, int64_t* host);
int ctx_read_i32(bamg_ctx* ctx, const int32_t* dev, size_t n, int32_t* host);

static inline int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  return (int)(g < 1 ? 1 : g);
}

// ------------------------------------------------------- device-wide scans
// out[0..n] exclusive prefix sums of in[0..n-1] (out[n] = total).  Optional
// total read back to the host.
int scan_i32(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int64_t* total_host);
// Same, the total written to a caller-owned device word (no host read).
int scan_i32_dev(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int64_t* total_dev);
// Same for uint8 flags -> int32 offsets.
int scan_u8(bamg_ctx* ctx, const uint8_t* in, int32_t* out, int64_t n, int64_t* total_host);

// --------------------------------------------------- block reduce helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Correctly rounded x / d from rd = RN(1/d) (Markstein): q = RN(x rd) is within
// one ulp of x/d, r = x - d q is exact by FMA, and RN(q + r rd) = RN(x/d).
// The theorem needs x, d, q and r clear of under/overflow, so the fast path is
// taken only for 2^-500 <= |x| <= 2^500 and 2^-400 <= |d| <= 2^400 (then
// 2^-900 <= |q| <= 2^900); everything else (zeros, subnormals, inf, NaN)
// uses the IEEE division.  Bit-identical to __ddiv_rn (tests/test_gpu_kernels:
// bamg_selftest_div over 2^30+ operand pairs).
__device__ __forceinline__ double div_rn_recip(double x, double d, double rd) {
  const unsigned ex = (unsigned)((unsigned long long)__double_as_longlong(x) >> 52) & 0x7ffu;
  const unsigned ed = (unsigned)((unsigned long long)__double_as_longlong(d) >> 52) & 0x7ffu;
  if (ex - (1023u - 500u) <= 1000u && ed - (1023u - 400u) <= 800u) {
    const double q = __dmul_rn(x, rd);
    const double r = __fma_rn(-d, q, x);
    return __fma_rn(r, rd, q);
  }
  // an exact zero over a normal d is the signed zero (the pinned constant left test vector has
  // zero residual in every B^T sweep: one lane in eight took the slow IEEE path, ~25 % per sweep)
  if ((__double_as_longlong(x) & 0x7fffffffffffffffll) == 0 && ed - (1023u - 400u) <= 800u)
    return __longlong_as_double(__double_as_longlong(x) ^ (__double_as_longlong(d) & (long long)0x8000000000000000ull));
  return __ddiv_rn(x, d);
}

// max of non-negative doubles through their bit patterns (order-preserving,
// NaN propagates as the largest pattern).
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            (unsigned long long)__double_as_longlong(v));
}

// Deterministic column reductions over n x k interleaved blocks: a fixed grid
// of partial sums (rows chunked contiguously), then a fixed tree.
constexpr int RED_BLOCKS = 296;  // 2 x 148 SMs at most
constexpr int RED_THREADS = 256;
// CTAs of a deterministic column reduction over n rows: a fixed function of n
// (so the partial-sum tree is reproducible run to run), ~2,048 rows per CTA,
// so a coarse level's reduction is one or a few CTAs instead of 296 near-empty
// ones and a 296-way finish.
static inline int red_blocks_for(int64_t n) {
  const int64_t b = (n + 2047) / 2048;
  return b < 1 ? 1 : (b > RED_BLOCKS ? RED_BLOCKS : (int)b);
}

// compute partial[b * k + c] for op(x, y) summed over the rows of block b.
// kinds: 0 = x*x, 1 = x*y
int colreduce(bamg_ctx* ctx, const double* X, const double* Y, int64_t n, int k, int kind,
              double* out_dev /* k */, int take_sqrt);
