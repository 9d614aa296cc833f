// Hash tables and scatter plans (see plan.cuh).
#include <cstdarg>
#include <atomic>
#include <array>
#include <cstring>
#include <mutex>
#include <vector>

#include "plan.cuh"

namespace smm {

// ------------------------------------------------------------------ errors
static thread_local char g_err[512];

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char *last_error() { return g_err; }

int cuda_status(cudaError_t e, const char *what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return SMM_ERR_CUDA;
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launches() { return (int64_t)g_launches.load(std::memory_order_relaxed); }

// ------------------------------------------------------------------ kernel timing (evidence)
static std::atomic<int> g_timing{0};
static std::mutex g_tmx;
static std::vector<std::array<cudaEvent_t, 2>> g_tpool;                 // idle event pairs
static std::vector<std::pair<int, std::array<cudaEvent_t, 2>>> g_tdone;  // (channel, recorded pair)

KernelTimer::KernelTimer(int ch, cudaStream_t st) : s(st), channel(ch) {
  if (!g_timing.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> g(g_tmx);
  if (g_tpool.empty()) {
    std::array<cudaEvent_t, 2> e{};
    if (cudaEventCreate(&e[0]) != cudaSuccess || cudaEventCreate(&e[1]) != cudaSuccess) return;
    g_tpool.push_back(e);
  }
  ev[0] = g_tpool.back()[0];
  ev[1] = g_tpool.back()[1];
  g_tpool.pop_back();
  cudaEventRecord(ev[0], s);
}

KernelTimer::~KernelTimer() {
  if (!ev[0]) return;
  std::lock_guard<std::mutex> g(g_tmx);
  g_tpool.push_back({ev[0], ev[1]});
}

void KernelTimer::stop() {
  if (!ev[0]) return;
  cudaEventRecord(ev[1], s);
  std::lock_guard<std::mutex> g(g_tmx);
  g_tdone.push_back({channel, {ev[0], ev[1]}});
  ev[0] = ev[1] = nullptr;
}

void kernel_timing(int on) { g_timing.store(on ? 1 : 0, std::memory_order_relaxed); }

// sums and clears the recorded launches of `channel` (waits for their end events)
int kernel_timing_read(int channel, double *total_ms, int64_t *count) {
  std::lock_guard<std::mutex> g(g_tmx);
  double tot = 0.0;
  int64_t n = 0;
  std::vector<std::pair<int, std::array<cudaEvent_t, 2>>> keep;
  for (auto &r : g_tdone) {
    if (r.first != channel) {
      keep.push_back(r);
      continue;
    }
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.second[1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.second[0], r.second[1]);
    if (e != cudaSuccess) return cuda_status(e, "kernel timing");
    tot += ms;
    ++n;
    g_tpool.push_back(r.second);
  }
  g_tdone.swap(keep);
  *total_ms = tot;
  *count = n;
  return SMM_OK;
}

__global__ void l2_policy_kernel(uint64_t *out) {
  uint64_t a, b;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(a));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(b));
  out[0] = a;
  out[1] = b;
}

int l2_policies(uint64_t &evict_last, uint64_t &evict_first) {
  static uint64_t cache[64][2];
  static std::atomic<int> have[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!have[dev].load(std::memory_order_acquire)) {  // concurrent first calls compute the same values
    uint64_t *d = nullptr, h[2];
    SMM_CUDA_TRY(cudaMalloc(&d, 16), "policy alloc");
    l2_policy_kernel<<<1, 1>>>(d);
    const cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    SMM_CUDA_TRY(e, "policy readback");
    cache[dev][0] = h[0];
    cache[dev][1] = h[1];
    have[dev].store(1, std::memory_order_release);
  }
  evict_last = cache[dev][0];
  evict_first = cache[dev][1];
  return SMM_OK;
}

int num_sms() {
  static std::atomic<int> cached[64];  // per-device attribute cache (idempotent fill)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int c = cached[dev].load(std::memory_order_relaxed);
  if (!c) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    c = v > 0 ? v : 1;
    cached[dev].store(c, std::memory_order_relaxed);
  }
  return c;
}

void load_hashes(SketchHashes &h, const uint64_t *words, int d, int log2b) {
  memset(&h, 0, sizeof(h));
  h.d = d;
  h.log2b = log2b;
  for (int g = 0; g < 4; ++g)
    for (int t = 0; t < d; ++t) {
      h.f[g][t].a = words[g * 2 * d + 2 * t];
      h.f[g][t].c = words[g * 2 * d + 2 * t + 1];
    }
}

// ------------------------------------------------------------------ hash tables
__global__ void hash_table_kernel(SketchHashes h, int group, int64_t n, uint32_t *buckets, int8_t *signs) {
  int t = blockIdx.y;
  HashFn f = h.f[group][t];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    if (group < 2)
      buckets[t * n + x] = eval_bucket(f, (uint64_t)x, h.log2b);
    else
      signs[t * n + x] = eval_signbit(f, (uint64_t)x) ? (int8_t)-1 : (int8_t)1;
  }
}

int hash_tables(const SketchHashes &h, int group, int64_t n, uint32_t *buckets, int8_t *signs, cudaStream_t s) {
  if (n <= 0) return SMM_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 4096) blocks = 4096;
  hash_table_kernel<<<dim3((unsigned)blocks, h.d), 256, 0, s>>>(h, group, n, buckets, signs);
  SMM_LAUNCH_CHECK("hash_table_kernel");
  return SMM_OK;
}

// ------------------------------------------------------------------ plans
__host__ __device__ static inline int64_t pad256(int64_t x) { return ((x + 255) / 256) * 256; }

int64_t plan_bytes_per(int64_t nin_max, int L) {
  return pad256(nin_max * 4) + pad256((nin_max + 2) * 4) + pad256(((int64_t)1 << L) * 4) + 256 +
         pad256((nin_max + 2) * 4) + pad256(nin_max * 4);
}

int64_t plan_total_bytes(int d, int nops, int64_t n1, int64_t n2, int L) {
  int64_t nin_max = nops == 2 ? (n1 > n2 ? n1 : n2) : n1 + n2;
  return (int64_t)d * nops * plan_bytes_per(nin_max, L);
}

struct PlanArgs {
  SketchHashes h;
  char *base;
  int64_t per_bytes, nin_max, n1, n2;
  int nops, L;
  int smem_ints;
};

__device__ __forceinline__ uint32_t plan_bucket(const PlanArgs &p, int t, int op, int64_t q) {
  // full bucket of input q of operand op under repetition t
  if (p.nops == 2) return eval_bucket(p.h.f[op][t], (uint64_t)q, p.h.log2b);
  return q < p.n1 ? eval_bucket(p.h.f[0][t], (uint64_t)q, p.h.log2b)
                  : eval_bucket(p.h.f[1][t], (uint64_t)(q - p.n1), p.h.log2b);
}

constexpr int PLAN_THREADS = 512;

__global__ void __launch_bounds__(PLAN_THREADS) plan_kernel(PlanArgs p) {
  extern __shared__ int sm[];  // p.smem_ints ints
  __shared__ int s_red[32];
  __shared__ int s_scan[PLAN_THREADS / 32 + 1];
  const int t = blockIdx.x / p.nops, op = blockIdx.x % p.nops;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nin = p.nops == 2 ? (op == 0 ? p.n1 : p.n2) : p.n1 + p.n2;
  const int64_t ell = (int64_t)1 << p.L;
  const uint32_t cmask = (uint32_t)(ell - 1);
  char *blk = p.base + (int64_t)(t * p.nops + op) * p.per_bytes;
  uint32_t *list = (uint32_t *)blk;
  blk += pad256(p.nin_max * 4);
  int32_t *roff = (int32_t *)blk;
  blk += pad256((p.nin_max + 2) * 4);
  uint32_t *empty = (uint32_t *)blk;
  blk += pad256(ell * 4);
  int32_t *meta = (int32_t *)blk;
  blk += 256;
  int32_t *fill = (int32_t *)blk;
  blk += pad256((p.nin_max + 2) * 4);
  int32_t *rank = (int32_t *)blk;

  int *run = sm;  // ell ints
  for (int64_t c = tid; c < ell; c += PLAN_THREADS) run[c] = 0;
  for (int64_t r = tid; r < nin + 2; r += PLAN_THREADS) roff[r] = 0;
  __syncthreads();

  // 1. ranks: one warp walks the inputs in order (deterministic by construction)
  if (warp == 0) {
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = 0; base < nin; base += 32) {
      int64_t q = base + lane;
      bool valid = q < nin;
      uint32_t c = valid ? (plan_bucket(p, t, op, q) & cmask) : (0x80000000u | (uint32_t)lane);
      unsigned peers = __match_any_sync(0xffffffffu, c);
      int b0 = valid ? run[c] : 0;
      __syncwarp();
      int r = b0 + __popc(peers & lt);
      if (valid && lane == 31 - __clz(peers)) run[c] = b0 + __popc(peers);
      __syncwarp();
      if (valid) rank[q] = r;
    }
  }
  __syncthreads();

  // 2. nrounds = max bucket load; per-round sizes; empty buckets
  int mx = 0;
  for (int64_t c = tid; c < ell; c += PLAN_THREADS) mx = max(mx, run[c]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    int m = 0;
    for (int w = 0; w < PLAN_THREADS / 32; ++w) m = max(m, s_red[w]);
    meta[0] = m;
  }
  for (int64_t c = tid; c < ell; c += PLAN_THREADS)
    for (int r = 0; r < run[c]; ++r) atomicAdd(&roff[r + 1], 1);
  // ordered compaction of empty buckets
  int running = 0;
  for (int64_t c0 = 0; c0 < ell; c0 += PLAN_THREADS) {
    int64_t c = c0 + tid;
    bool e = c < ell && run[c] == 0;
    unsigned bal = __ballot_sync(0xffffffffu, e);
    if (lane == 0) s_scan[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < PLAN_THREADS / 32; ++w) {
        int v = s_scan[w];
        s_scan[w] = acc;
        acc += v;
      }
      s_scan[PLAN_THREADS / 32] = acc;
    }
    __syncthreads();
    if (e) empty[running + s_scan[warp] + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)c;
    running += s_scan[PLAN_THREADS / 32];
    __syncthreads();
  }
  if (tid == 0) meta[1] = running;
  __syncthreads();

  // 3. round offsets (exclusive scan of per-round sizes)
  const int nrounds = meta[0];
  if (tid == 0) {
    int acc = 0;
    for (int r = 0; r <= nrounds; ++r) {
      acc += roff[r];
      roff[r] = acc;  // roff[0] = 0, roff[r] = start of round r
    }
  }
  __syncthreads();

  // 4. placement: one warp, inputs in order; per-round fill pointers in smem when they fit
  const bool fill_in_smem = nrounds + 1 <= p.smem_ints;
  int *fs = sm;
  for (int r = tid; r <= nrounds; r += PLAN_THREADS) {
    if (fill_in_smem) fs[r] = roff[r];
    else fill[r] = roff[r];
  }
  __syncthreads();
  if (warp == 0) {
    const unsigned lt = (1u << lane) - 1u;
    int *fp = fill_in_smem ? fs : (int *)fill;
    for (int64_t base = 0; base < nin; base += 32) {
      int64_t q = base + lane;
      bool valid = q < nin;
      int r = valid ? rank[q] : (int)(0x80000000u | (uint32_t)lane);
      unsigned peers = __match_any_sync(0xffffffffu, r);
      int b0 = valid ? fp[r] : 0;
      __syncwarp();
      if (valid && lane == 31 - __clz(peers)) fp[r] = b0 + __popc(peers);
      __syncwarp();
      if (valid) list[b0 + __popc(peers & lt)] = (uint32_t)q;
    }
  }
}

int build_plans(const SketchHashes &h, int nops, int64_t n1, int64_t n2, int L, char *ws, cudaStream_t s) {
  PlanArgs p;
  p.h = h;
  p.base = ws;
  p.nin_max = nops == 2 ? (n1 > n2 ? n1 : n2) : n1 + n2;
  p.per_bytes = plan_bytes_per(p.nin_max, L);
  p.n1 = n1;
  p.n2 = n2;
  p.nops = nops;
  p.L = L;
  int64_t ell = (int64_t)1 << L;
  int ints = (int)(ell > 4096 ? ell : 4096);
  p.smem_ints = ints;
  size_t smem = (size_t)ints * 4;
  SMM_CUDA_TRY(cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "plan_kernel smem");
  plan_kernel<<<h.d * nops, PLAN_THREADS, smem, s>>>(p);
  SMM_LAUNCH_CHECK("plan_kernel");
  return SMM_OK;
}

// ------------------------------------------------------------------ CSR bucket sort
// The CSR fills (fwht2p / fft2p) place each bucket's entries with atomics, so their
// order inside a bucket is arbitrary; sorting every bucket segment by input index i
// (entry bits 0-25) restores the reference's serial order (sketch.py:166-172) and
// makes the plan deterministic.  Segments of <= 32 entries: one thread, insertion
// sort.  Longer ones (heavily loaded or degenerate hashes) are sorted by a whole CTA
// with a bitonic network: in shared memory up to 8192 entries, in place in global
// memory beyond (all-ascending network with virtual +inf padding, so any length).
namespace {
constexpr int SHORT_SEG = 32;
constexpr int SORT_THREADS = 1024;
constexpr int SMEM_SEG = 8192;
constexpr uint32_t IDX_MASK = 0x03ffffffu;

__device__ __forceinline__ void cmpswap(uint32_t *e, int64_t a, int64_t b) {
  const uint32_t x = e[a], y = e[b];
  if ((x & IDX_MASK) > (y & IDX_MASK)) {
    e[a] = y;
    e[b] = x;
  }
}

// ascending bitonic sort of e[0, L) by the index bits, virtual +inf past L; P = pow2 >= L
__device__ void bitonic_all_ascending(uint32_t *e, int64_t L, int64_t P) {
  for (int64_t k = 2; k <= P; k <<= 1) {
    // merge of two sorted runs of k/2 with the partner mirrored: every comparator ascending
    for (int64_t i = threadIdx.x; i < P / 2; i += blockDim.x) {
      const int64_t blk = i / (k / 2), pos = i % (k / 2);
      const int64_t a = blk * k + pos, b = blk * k + k - 1 - pos;
      if (b < L) cmpswap(e, a, b);
    }
    __syncthreads();
    for (int64_t j = k / 4; j >= 1; j >>= 1) {
      for (int64_t i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int64_t a = (i / j) * 2 * j + (i % j), b = a + j;
        if (b < L) cmpswap(e, a, b);
      }
      __syncthreads();
    }
  }
}
}  // namespace

__global__ void csr_sort_short_kernel(const int32_t *off, uint32_t *ent, int64_t nmax, int64_t b, int rows) {
  const int64_t total = (int64_t)rows * b;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = x / b, m = x % b;
    const int32_t e0 = off[row * (b + 1) + m], e1 = off[row * (b + 1) + m + 1];
    if (e1 - e0 > SHORT_SEG) continue;  // csr_sort_long_kernel
    uint32_t *e = ent + row * nmax;
    for (int32_t a = e0 + 1; a < e1; ++a) {
      const uint32_t key = e[a];
      int32_t q = a - 1;
      while (q >= e0 && (e[q] & IDX_MASK) > (key & IDX_MASK)) {
        e[q + 1] = e[q];
        --q;
      }
      e[q + 1] = key;
    }
  }
}

// every CTA scans a grid-strided share of the buckets; the long segments it finds
// are queued in shared memory and sorted one after the other by the whole CTA
__global__ void __launch_bounds__(SORT_THREADS) csr_sort_long_kernel(const int32_t *off, uint32_t *ent, int64_t nmax,
                                                                     int64_t b, int rows) {
  __shared__ uint32_t s_seg[SMEM_SEG];
  __shared__ int64_t s_q[SORT_THREADS];
  __shared__ int s_nq;
  const int64_t total = (int64_t)rows * b;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < total; base += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_nq = 0;
    __syncthreads();
    const int64_t x = base + threadIdx.x;
    if (x < total) {
      const int64_t row = x / b, m = x % b;
      if (off[row * (b + 1) + m + 1] - off[row * (b + 1) + m] > SHORT_SEG) s_q[atomicAdd(&s_nq, 1)] = x;
    }
    __syncthreads();
    const int nq = s_nq;
    for (int q = 0; q < nq; ++q) {
      const int64_t row = s_q[q] / b, m = s_q[q] % b;
      const int32_t e0 = off[row * (b + 1) + m], e1 = off[row * (b + 1) + m + 1];
      const int64_t L = e1 - e0;
      int64_t P = 1;
      while (P < L) P <<= 1;
      uint32_t *e = ent + row * nmax + e0;
      if (L <= SMEM_SEG) {
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) s_seg[i] = e[i];
        __syncthreads();
        bitonic_all_ascending(s_seg, L, P);
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) e[i] = s_seg[i];
      } else {
        bitonic_all_ascending(e, L, P);  // global memory, visible CTA-wide at each barrier
      }
      __syncthreads();
    }
  }
}

int csr_sort(const int32_t *off, uint32_t *ent, int64_t nmax, int64_t b, int rows, cudaStream_t s) {
  const int64_t total = (int64_t)rows * b;
  if (total <= 0) return SMM_OK;
  int64_t blocks = ceil_div(total, 256);
  if (blocks > 8192) blocks = 8192;
  csr_sort_short_kernel<<<(unsigned)blocks, 256, 0, s>>>(off, ent, nmax, b, rows);
  SMM_LAUNCH_CHECK("csr_sort_short_kernel");
  int64_t lb = ceil_div(total, SORT_THREADS);
  if (lb > 2 * num_sms()) lb = 2 * num_sms();
  csr_sort_long_kernel<<<(unsigned)lb, SORT_THREADS, 0, s>>>(off, ent, nmax, b, rows);
  SMM_LAUNCH_CHECK("csr_sort_long_kernel");
  return SMM_OK;
}

}  // namespace smm
