// Step 5: estimate extraction (gather + sign + median over d) fused with the
// heavy-hitter threshold.
//
// Reference: sketch.py:375-399 (`decompress_all`): idx = h1(i) ^ h2(j) (fwht)
// or (h1(i) + h2(j)) mod b (fft); vals = polys[t, idx] * s1 * s2; median over
// the d repetitions (odd d: the exact middle order statistic).  Threshold:
// experiments.py:136-168 (|est| >= thr, inclusive) or BASELINE cfg5 (> thr).
//
// One CTA covers a tile of rows x 256 columns; each thread owns one column,
// keeps its d (bucket, sign) pairs in registers and walks the rows, whose
// hashes are evaluated once per CTA into shared memory.  The gathered sketch
// values come from the L2-resident d x b polys.  Estimates are written with
// coalesced stores (or skipped in threshold-only mode); the threshold writes a
// bitmask + per-row counts so the pair list is emitted in row-major order by a
// second pass (deterministic, no atomics on positions).
#include "common.cuh"

namespace smm {

constexpr int XT = 256;
constexpr int XROWS = 64;

template <int D>
__device__ __forceinline__ double median_sorted(double (&v)[D]) {
#pragma unroll
  for (int i = 1; i < D; ++i) {
#pragma unroll
    for (int j = i; j > 0; --j) {
      const double a = v[j - 1], b = v[j];
      const bool sw = b < a;  // compare-exchange keeps the exact values
      v[j - 1] = sw ? b : a;
      v[j] = sw ? a : b;
    }
  }
  return v[(D - 1) / 2];
}

struct ExtractArgs {
  SketchHashes h;
  const double *polys;
  int64_t n1, n2, r0, r1;
  double *est;
  int64_t ld_est;
  double thr;
  int strict, xor_combine;
  uint32_t *mask;  // rows x ceil(n2/32)
  int64_t mask_ld;
  int64_t *rowcnt;  // rows
};

template <int D>
__global__ void __launch_bounds__(XT) extract_kernel(ExtractArgs p) {
  const int d = D > 0 ? D : p.h.d;
  constexpr int DM = D > 0 ? D : SMM_MAX_DEPTH;
  // rows per group whose gathers are in flight together (latency of the random
  // L2 gathers is the bound: d * RG independent 8-byte loads per thread)
  constexpr int RG = D > 0 ? 4 : 1;
  __shared__ uint32_t s_h1[XROWS][DM];
  __shared__ int8_t s_s1[XROWS][DM];
  const int log2b = p.h.log2b;
  const uint32_t bmask = (uint32_t)(((uint64_t)1 << log2b) - 1);
  const int64_t b = (int64_t)1 << log2b;
  const int64_t j = (int64_t)blockIdx.x * XT + threadIdx.x;
  const int64_t rbase = p.r0 + (int64_t)blockIdx.y * XROWS;
  const int nrows = (int)((p.r1 - rbase) < XROWS ? (p.r1 - rbase) : XROWS);
  for (int q = threadIdx.x; q < nrows * d; q += XT) {
    const int r = q / d, t = q % d;
    s_h1[r][t] = eval_bucket(p.h.f[0][t], (uint64_t)(rbase + r), log2b);
    s_s1[r][t] = eval_signbit(p.h.f[2][t], (uint64_t)(rbase + r)) ? -1 : 1;
  }
  __syncthreads();
  const bool colok = j < p.n2;
  uint32_t h2[DM];
  double s2[DM];
#pragma unroll
  for (int t = 0; t < DM; ++t) {
    if (t < d) {
      h2[t] = colok ? eval_bucket(p.h.f[1][t], (uint64_t)j, log2b) : 0u;
      s2[t] = (colok && eval_signbit(p.h.f[3][t], (uint64_t)j)) ? -1.0 : 1.0;
    }
  }
  const int lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < nrows; r0 += RG) {
    double v[RG][DM];
#pragma unroll
    for (int g = 0; g < RG; ++g) {
      const int r = r0 + g < nrows ? r0 + g : nrows - 1;  // clamped duplicate rows are not stored
#pragma unroll
      for (int t = 0; t < DM; ++t) {
        if (t < d) {
          const uint32_t a = s_h1[r][t];
          const uint32_t idx = p.xor_combine ? (a ^ h2[t]) : ((a + h2[t]) & bmask);
          v[g][t] = colok ? __ldg(p.polys + t * b + idx) : 0.0;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < RG; ++g) {
      const int r = r0 + g;
      if (r >= nrows) break;  // block-uniform
      const int64_t i = rbase + r;
#pragma unroll
      for (int t = 0; t < DM; ++t) {
        if (t < d) {
          v[g][t] *= (double)s_s1[r][t];  // vals *= s1 ; vals *= s2 (sketch.py:396-397)
          v[g][t] *= s2[t];
        }
      }
      // np.median semantics (sketch.py:398): any NaN among the d values gives NaN
      bool has_nan = false;
#pragma unroll
      for (int t = 0; t < DM; ++t)
        if (t < d) has_nan |= isnan(v[g][t]);
      double e;
      if (D > 0) {
        e = median_sorted<DM>(v[g]);
      } else {
        for (int a = 1; a < d; ++a) {
          double key = v[g][a];
          int q = a - 1;
          while (q >= 0 && v[g][q] > key) { v[g][q + 1] = v[g][q]; --q; }
          v[g][q + 1] = key;
        }
        e = v[g][(d - 1) / 2];
      }
      if (has_nan) e = __longlong_as_double(0x7ff8000000000000ll);
      if (colok && p.est) p.est[(i - p.r0) * p.ld_est + j] = e;
      const double ae = fabs(e);
      const bool hit = colok && (p.strict ? (ae > p.thr) : (ae >= p.thr));
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (lane == 0 && (j >> 5) < p.mask_ld) {
        p.mask[(i - p.r0) * p.mask_ld + (j >> 5)] = bal;
        if (bal) atomicAdd((unsigned long long *)&p.rowcnt[i - p.r0], (unsigned long long)__popc(bal));
      }
    }
  }
}

// exclusive scan of per-row counts (single block) -> offsets; total -> *count
__global__ void row_scan_kernel(const int64_t *rowcnt, int64_t rows, int64_t *offs, int64_t *count) {
  // exclusive scan of the per-row heavy-hitter counts: chunks of 1024 rows, warp-shuffle scans
  // and one block-wide combine per chunk, the running total carried across chunks
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < rows; base += 1024) {
    const int64_t r = base + threadIdx.x;
    const int64_t v = r < rows ? rowcnt[r] : 0;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int64_t c = carry;
    if (r < rows) offs[r] = c + inc - v + (warp > 0 ? wsum[warp - 1] : 0);
    __syncthreads();  // every thread has read wsum and carry
    if (threadIdx.x == 0) carry = c + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

// one warp per row: emit (i, j) pairs in column order
__global__ void hh_write_kernel(const uint32_t *mask, int64_t mask_ld, const int64_t *offs, int64_t rows, int64_t r0,
                                int64_t n2, int64_t *pairs, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool a16 = ((uintptr_t)pairs & 15) == 0;  // caller's buffer allows 16-byte stores
  for (int64_t r = warp; r < rows; r += nwarps) {
    int64_t pos = offs[r];
    const uint32_t *mrow = mask + r * mask_ld;
    for (int64_t w0 = 0; w0 < mask_ld; w0 += 32) {
      const int64_t w = w0 + lane;
      const uint32_t bits = w < mask_ld ? mrow[w] : 0u;
      const int cnt = __popc(bits);
      int incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int64_t p0 = pos + incl - cnt;
      uint32_t bb = bits;
      while (bb) {
        const int bit = __ffs(bb) - 1;
        bb &= bb - 1;
        const int64_t jj = w * 32 + bit;
        if (p0 < cap && jj < n2) {
          if (a16) {  // one 16-byte store per (i, j) pair
            *reinterpret_cast<longlong2 *>(pairs + 2 * p0) = make_longlong2(r0 + r, jj);
          } else {
            pairs[2 * p0] = r0 + r;
            pairs[2 * p0 + 1] = jj;
          }
        }
        ++p0;
      }
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// Per-entry queries (sketch.py:343-372 sketch_estimates / decompress_entry) for a batch
// of (i, j) pairs: one thread per query; est[q] = median, reps[q * d + t] (nullable) the
// d signed per-repetition estimates in repetition order.
__global__ void query_kernel(SketchHashes h, const double *polys, const int64_t *ij, int64_t count, int xor_combine,
                             double *est, double *reps) {
  const int d = h.d;
  const int log2b = h.log2b;
  const uint32_t bmask = (uint32_t)(((uint64_t)1 << log2b) - 1);
  const int64_t b = (int64_t)1 << log2b;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)ij[2 * q], j = (uint64_t)ij[2 * q + 1];
    double v[SMM_MAX_DEPTH];
    for (int t = 0; t < d; ++t) {
      const uint32_t a = eval_bucket(h.f[0][t], i, log2b), c = eval_bucket(h.f[1][t], j, log2b);
      const uint32_t idx = xor_combine ? (a ^ c) : ((a + c) & bmask);
      double x = polys[t * b + idx];
      x *= eval_signbit(h.f[2][t], i) ? -1.0 : 1.0;  // eval_sign(s1) * eval_sign(s2) * polys (sketch.py:364-366)
      x *= eval_signbit(h.f[3][t], j) ? -1.0 : 1.0;
      v[t] = x;
      if (reps) reps[q * d + t] = x;
    }
    bool has_nan = false;
    for (int t = 0; t < d; ++t) has_nan |= isnan(v[t]);
    for (int a2 = 1; a2 < d; ++a2) {  // insertion sort: the exact middle order statistic
      const double key = v[a2];
      int k = a2 - 1;
      while (k >= 0 && v[k] > key) { v[k + 1] = v[k]; --k; }
      v[k + 1] = key;
    }
    est[q] = has_nan ? __longlong_as_double(0x7ff8000000000000ll) : v[(d - 1) / 2];  // np.median: NaN in, NaN out
  }
}

// ---------------------------------------------------------------- depth > SMM_MAX_DEPTH
// The reference accepts any odd d (sketch.py:75-76).  Past the kernel-parameter
// hash block (63 repetitions) the hash functions come from a device array
// hf[4][d] and each thread keeps its d values in its own shared-memory column
// (stride = threads per CTA: conflict-free), sorted in place by insertion sort —
// the exact middle order statistic, NaN in -> NaN out, as np.median.
template <bool XOR>
__device__ __forceinline__ double big_entry(const HashFn *hf, int d, int log2b, const double *polys, uint64_t i,
                                            uint64_t j, double *col, int stride, double *reps) {
  const uint32_t bmask = (uint32_t)(((uint64_t)1 << log2b) - 1);
  const int64_t b = (int64_t)1 << log2b;
  bool has_nan = false;
  for (int t = 0; t < d; ++t) {
    const uint32_t a = eval_bucket(hf[t], i, log2b), c = eval_bucket(hf[d + t], j, log2b);
    const uint32_t idx = XOR ? (a ^ c) : ((a + c) & bmask);
    double x = __ldg(polys + t * b + idx);
    x *= eval_signbit(hf[2 * d + t], i) ? -1.0 : 1.0;  // vals *= s1 ; vals *= s2 (sketch.py:396-397)
    x *= eval_signbit(hf[3 * d + t], j) ? -1.0 : 1.0;
    if (reps) reps[t] = x;
    has_nan |= isnan(x);
    int k = t - 1;  // insertion into the sorted prefix
    while (k >= 0 && col[k * stride] > x) {
      col[(k + 1) * stride] = col[k * stride];
      --k;
    }
    col[(k + 1) * stride] = x;
  }
  return has_nan ? __longlong_as_double(0x7ff8000000000000ll) : col[((d - 1) / 2) * stride];
}

struct BigArgs {
  const HashFn *hf;
  int d, log2b, xor_combine;
  const double *polys;
  int64_t n2, r0, r1;
  double *est;
  int64_t ld_est;
  double thr;
  int strict;
  uint32_t *mask;
  int64_t mask_ld;
  int64_t *rowcnt;
};

// grid (ceil(n2 / blockDim), rows): one row per CTA row, one column per thread
__global__ void extract_big_kernel(BigArgs p) {
  extern __shared__ double sv[];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = p.r0 + blockIdx.y;
  const bool colok = j < p.n2;
  double e = 0.0;
  if (colok) {
    e = p.xor_combine ? big_entry<true>(p.hf, p.d, p.log2b, p.polys, (uint64_t)i, (uint64_t)j, sv + threadIdx.x,
                                        blockDim.x, nullptr)
                      : big_entry<false>(p.hf, p.d, p.log2b, p.polys, (uint64_t)i, (uint64_t)j, sv + threadIdx.x,
                                         blockDim.x, nullptr);
    if (p.est) p.est[(i - p.r0) * p.ld_est + j] = e;
  }
  const double ae = fabs(e);
  const bool hit = colok && (p.strict ? (ae > p.thr) : (ae >= p.thr));
  const unsigned bal = __ballot_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && (j >> 5) < p.mask_ld) {
    p.mask[(i - p.r0) * p.mask_ld + (j >> 5)] = bal;
    if (bal) atomicAdd((unsigned long long *)&p.rowcnt[i - p.r0], (unsigned long long)__popc(bal));
  }
}

__global__ void query_big_kernel(const HashFn *hf, int d, int log2b, const double *polys, const int64_t *ij,
                                 int64_t count, int xor_combine, double *est, double *reps) {
  extern __shared__ double sv[];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)ij[2 * q], j = (uint64_t)ij[2 * q + 1];
    double *r = reps ? reps + q * d : nullptr;
    est[q] = xor_combine ? big_entry<true>(hf, d, log2b, polys, i, j, sv + threadIdx.x, blockDim.x, r)
                         : big_entry<false>(hf, d, log2b, polys, i, j, sv + threadIdx.x, blockDim.x, r);
  }
}

// threads per CTA for the big-depth kernels: d doubles per thread in shared memory
static int big_threads(int d) {
  int th = 256;
  while (th > 32 && (int64_t)th * d * 8 > 200 * 1024) th /= 2;
  return th;
}

int64_t big_hash_bytes(int d) { return d > SMM_MAX_DEPTH ? (((int64_t)d * 4 * 16 + 255) / 256) * 256 : 0; }

// upload hf[4][d] (group-major draw order, hashing.py:146-152) into dev
static int upload_hashes(HashFn *dev, const uint64_t *words, int d, cudaStream_t s) {
  SMM_CUDA_TRY(cudaMemcpyAsync(dev, words, (size_t)d * 4 * 16, cudaMemcpyHostToDevice, s), "hash upload");
  return SMM_OK;
}

int extract_big(int variant, const uint64_t *words, int d, int log2b, const double *polys, int64_t n2, int64_t r0,
                int64_t r1, double *est, int64_t ld_est, double thr, int strict, int64_t *hh_pairs, int64_t hh_cap,
                int64_t *hh_count, char *ws, int64_t ws_bytes, cudaStream_t s);

int query(int variant, const SketchHashes &h, const double *polys, const int64_t *ij, int64_t count, double *est,
          double *reps, cudaStream_t s) {
  if (count <= 0) return SMM_OK;
  int64_t blocks = ceil_div(count, 128);
  if (blocks > 4096) blocks = 4096;
  query_kernel<<<(unsigned)blocks, 128, 0, s>>>(h, polys, ij, count, variant == SMM_VARIANT_FWHT ? 1 : 0, est, reps);
  SMM_LAUNCH_CHECK("query_kernel");
  return SMM_OK;
}

int hh_pairs(const void *ws, int64_t n2, int64_t r0, int64_t r1, int64_t *pairs, int64_t cap, cudaStream_t s);

int64_t extract_workspace(int64_t n2, int64_t r0, int64_t r1) {
  const int64_t rows = r1 - r0;
  const int64_t mask_ld = ceil_div(n2, 32);
  return ((rows * mask_ld * 4 + 255) / 256) * 256 + 2 * ((rows * 8 + 255) / 256) * 256 + 256;
}

int extract(int variant, const SketchHashes &h, const double *polys, int64_t n1, int64_t n2, int64_t r0, int64_t r1,
            double *est, int64_t ld_est, double thr, int strict, int64_t *hh_pairs, int64_t hh_cap,
            int64_t *hh_count, char *ws, int64_t ws_bytes, cudaStream_t s) {
  const int64_t rows = r1 - r0;
  if (ws_bytes < extract_workspace(n2, r0, r1)) {
    set_error("extract workspace too small");
    return SMM_ERR_WORKSPACE;
  }
  ExtractArgs p;
  p.h = h;
  p.polys = polys;
  p.n1 = n1;
  p.n2 = n2;
  p.r0 = r0;
  p.r1 = r1;
  p.est = est;
  p.ld_est = ld_est;
  p.thr = thr;
  p.strict = strict;
  p.xor_combine = variant == SMM_VARIANT_FWHT ? 1 : 0;
  p.mask_ld = ceil_div(n2, 32);
  p.mask = (uint32_t *)ws;
  char *q = ws + ((rows * p.mask_ld * 4 + 255) / 256) * 256;
  p.rowcnt = (int64_t *)q;
  int64_t *offs = (int64_t *)(q + ((rows * 8 + 255) / 256) * 256);
  if (rows <= 0 || n2 <= 0) {
    SMM_CUDA_TRY(cudaMemsetAsync(hh_count, 0, sizeof(int64_t), s), "extract memset");
    return SMM_OK;
  }
  SMM_CUDA_TRY(cudaMemsetAsync(p.rowcnt, 0, rows * 8, s), "extract memset");
  KernelTimer timer(1, s);
  const int64_t chunk = (int64_t)65535 * XROWS;  // grid.y limit: row chunks of 65535 tiles
  for (int64_t y0 = 0; y0 < rows; y0 += chunk) {
    ExtractArgs pc = p;
    pc.r0 = r0 + y0;
    pc.r1 = y0 + chunk < rows ? r0 + y0 + chunk : r1;
    pc.est = est ? est + y0 * ld_est : nullptr;
    pc.mask = p.mask + y0 * p.mask_ld;
    pc.rowcnt = p.rowcnt + y0;
    dim3 grid((unsigned)ceil_div(n2, XT), (unsigned)ceil_div(pc.r1 - pc.r0, XROWS));
    switch (h.d) {
      case 1: extract_kernel<1><<<grid, XT, 0, s>>>(pc); break;
      case 3: extract_kernel<3><<<grid, XT, 0, s>>>(pc); break;
      case 5: extract_kernel<5><<<grid, XT, 0, s>>>(pc); break;
      case 7: extract_kernel<7><<<grid, XT, 0, s>>>(pc); break;
      case 9: extract_kernel<9><<<grid, XT, 0, s>>>(pc); break;
      default: extract_kernel<0><<<grid, XT, 0, s>>>(pc); break;
    }
  }
  timer.stop();
  SMM_LAUNCH_CHECK("extract_kernel");
  row_scan_kernel<<<1, 1024, 0, s>>>(p.rowcnt, rows, offs, hh_count);
  SMM_LAUNCH_CHECK("row_scan_kernel");
  if (hh_pairs && hh_cap > 0) return smm::hh_pairs(ws, n2, r0, r1, hh_pairs, hh_cap, s);
  return SMM_OK;
}


int extract_big(int variant, const uint64_t *words, int d, int log2b, const double *polys, int64_t n2, int64_t r0,
                int64_t r1, double *est, int64_t ld_est, double thr, int strict, int64_t *hh_pairs, int64_t hh_cap,
                int64_t *hh_count, char *ws, int64_t ws_bytes, cudaStream_t s) {
  const int64_t rows = r1 - r0;
  const int64_t base = extract_workspace(n2, r0, r1);
  if (ws_bytes < base + big_hash_bytes(d)) {
    set_error("extract workspace too small");
    return SMM_ERR_WORKSPACE;
  }
  BigArgs p;
  p.hf = (const HashFn *)(ws + base);
  p.d = d;
  p.log2b = log2b;
  p.xor_combine = variant == SMM_VARIANT_FWHT ? 1 : 0;
  p.polys = polys;
  p.n2 = n2;
  p.r0 = r0;
  p.r1 = r1;
  p.est = est;
  p.ld_est = ld_est;
  p.thr = thr;
  p.strict = strict;
  p.mask_ld = ceil_div(n2, 32);
  p.mask = (uint32_t *)ws;
  char *q = ws + ((rows * p.mask_ld * 4 + 255) / 256) * 256;
  p.rowcnt = (int64_t *)q;
  int64_t *offs = (int64_t *)(q + ((rows * 8 + 255) / 256) * 256);
  if (rows <= 0 || n2 <= 0) {
    SMM_CUDA_TRY(cudaMemsetAsync(hh_count, 0, sizeof(int64_t), s), "extract memset");
    return SMM_OK;
  }
  int rc = upload_hashes((HashFn *)p.hf, words, d, s);
  if (rc) return rc;
  SMM_CUDA_TRY(cudaMemsetAsync(p.rowcnt, 0, rows * 8, s), "extract memset");
  const int th = big_threads(d);
  const size_t smem = (size_t)th * d * 8;
  SMM_CUDA_TRY(cudaFuncSetAttribute(extract_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "extract_big smem");
  KernelTimer timer(1, s);
  for (int64_t y0 = 0; y0 < rows; y0 += 65535) {  // grid.y limit
    BigArgs pc = p;
    pc.r0 = r0 + y0;
    pc.r1 = y0 + 65535 < rows ? r0 + y0 + 65535 : r1;
    pc.est = est ? est + y0 * ld_est : nullptr;
    pc.mask = p.mask + y0 * p.mask_ld;
    pc.rowcnt = p.rowcnt + y0;
    dim3 grid((unsigned)ceil_div(n2, th), (unsigned)(pc.r1 - pc.r0));
    extract_big_kernel<<<grid, th, smem, s>>>(pc);
  }
  timer.stop();
  SMM_LAUNCH_CHECK("extract_big_kernel");
  row_scan_kernel<<<1, 1024, 0, s>>>(p.rowcnt, rows, offs, hh_count);
  SMM_LAUNCH_CHECK("row_scan_kernel");
  if (hh_pairs && hh_cap > 0) return smm::hh_pairs(ws, n2, r0, r1, hh_pairs, hh_cap, s);
  return SMM_OK;
}

int query_big(int variant, const uint64_t *words, int d, int log2b, const double *polys, const int64_t *ij,
              int64_t count, double *est, double *reps, cudaStream_t s) {
  if (count <= 0) return SMM_OK;
  HashFn *hf = nullptr;
  keep_pool_memory();
  SMM_CUDA_TRY(cudaMallocAsync((void **)&hf, (size_t)d * 4 * 16, s), "query alloc");
  int rc = upload_hashes(hf, words, d, s);
  if (rc) return rc;
  const int th = big_threads(d);
  const size_t smem = (size_t)th * d * 8;
  SMM_CUDA_TRY(cudaFuncSetAttribute(query_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "query_big smem");
  int64_t blocks = ceil_div(count, th);
  if (blocks > 4096) blocks = 4096;
  query_big_kernel<<<(unsigned)blocks, th, smem, s>>>(hf, d, log2b, polys, ij, count,
                                                      variant == SMM_VARIANT_FWHT ? 1 : 0, est, reps);
  SMM_LAUNCH_CHECK("query_big_kernel");
  SMM_CUDA_TRY(cudaFreeAsync(hf, s), "query free");
  return SMM_OK;
}

int hh_pairs(const void *ws, int64_t n2, int64_t r0, int64_t r1, int64_t *pairs, int64_t cap, cudaStream_t s) {
  const int64_t rows = r1 - r0;
  if (rows <= 0 || n2 <= 0 || cap <= 0) return SMM_OK;
  const int64_t mask_ld = ceil_div(n2, 32);
  const uint32_t *mask = (const uint32_t *)ws;
  const char *q = (const char *)ws + ((rows * mask_ld * 4 + 255) / 256) * 256;
  const int64_t *offs = (const int64_t *)(q + ((rows * 8 + 255) / 256) * 256);
  int64_t blocks = ceil_div(rows * 32, 256);
  if (blocks > 8192) blocks = 8192;
  hh_write_kernel<<<(unsigned)blocks, 256, 0, s>>>(mask, mask_ld, offs, rows, r0, n2, pairs, cap);
  SMM_LAUNCH_CHECK("hh_write_kernel");
  return SMM_OK;
}

}  // namespace smm
