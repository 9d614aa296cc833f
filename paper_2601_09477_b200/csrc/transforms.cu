// Step 4 (single inverse transform per repetition, 1/b scale), the batched
// one-shot transforms behind the public transforms API, and the operand
// transpose.
//
// Reference: sketch.py:178-188 (FWHT inverse + 1/b), sketch.py:219-234 (FFT
// Hermitian fill + inverse + Re/b), transforms.py:37-175, sketch.py:305-307.
#include <atomic>

#include "common.cuh"

namespace smm {

int64_t twiddle_table_bytes(int log2b);
int twiddle_tables(int log2b, cplx *tlo, cplx *thi, int &s, cudaStream_t st);

constexpr int SMEM_FWHT_LOG = 11;  // low bits done in shared memory

// FWHT over the low `lb` bits of every length-2^log2n vector (blocks of 2^lb).
__global__ void fwht_low_kernel(double *x, int64_t nblocks, int lb, double scale, int apply_scale) {
  extern __shared__ double sm[];
  const int m = 1 << lb;
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    double *p = x + blk * m;
    for (int i = threadIdx.x; i < m; i += blockDim.x) sm[i] = p[i];
    __syncthreads();
    for (int h = 1; h < m; h <<= 1) {
      for (int q = threadIdx.x; q < m / 2; q += blockDim.x) {
        const int j = (q / h) * 2 * h + (q % h);
        const double u = sm[j], v = sm[j + h];
        sm[j] = u + v;
        sm[j + h] = u - v;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < m; i += blockDim.x) p[i] = apply_scale ? sm[i] * scale : sm[i];
    __syncthreads();
  }
}

// One radix-2 FWHT stage of half-width h on every vector (in place).
__global__ void fwht_stage_kernel(double *x, int64_t batch, int log2n, int64_t h, double scale, int apply_scale) {
  const int64_t n = (int64_t)1 << log2n;
  const int64_t pairs = batch * (n / 2);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < pairs; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = q / (n / 2), r = q % (n / 2);
    const int64_t j = v * n + (r / h) * 2 * h + (r % h);
    const double a = x[j], b = x[j + h];
    x[j] = apply_scale ? (a + b) * scale : a + b;
    x[j + h] = apply_scale ? (a - b) * scale : a - b;
  }
}

int fwht_batched(double *x, int64_t batch, int log2n, double scale, cudaStream_t s) {
  if (batch <= 0) return SMM_OK;
  const int lb = log2n < SMEM_FWHT_LOG ? log2n : SMEM_FWHT_LOG;
  const int64_t nblocks = batch * ((int64_t)1 << (log2n - lb));
  const bool scale_low = (lb == log2n);
  fwht_low_kernel<<<(unsigned)(nblocks < 4096 ? nblocks : 4096), 256, ((size_t)1 << lb) * sizeof(double), s>>>(
      x, nblocks, lb, scale, scale_low ? 1 : 0);
  SMM_LAUNCH_CHECK("fwht_low_kernel");
  for (int q = lb; q < log2n; ++q) {
    const int64_t pairs = batch * (((int64_t)1 << log2n) / 2);
    int64_t blocks = ceil_div(pairs, 256);
    if (blocks > 16384) blocks = 16384;
    const bool last = (q == log2n - 1);
    fwht_stage_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, batch, log2n, (int64_t)1 << q, scale, last ? 1 : 0);
    SMM_LAUNCH_CHECK("fwht_stage_kernel");
  }
  return SMM_OK;
}

// ---------------------------------------------------------------- complex FFT
__global__ void bitrev_kernel(cplx *z, int64_t batch, int log2n) {
  const int64_t n = (int64_t)1 << log2n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < batch * n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = q / n, i = q % n;
    const int64_t j = log2n == 0 ? 0 : (int64_t)(__brevll((unsigned long long)i) >> (64 - log2n));
    if (j > i) {
      cplx t = z[v * n + i];
      z[v * n + i] = z[v * n + j];
      z[v * n + j] = t;
    }
  }
}

__global__ void fft_stage_kernel(cplx *z, int64_t batch, int log2n, int64_t half, const cplx *tlo, const cplx *thi,
                                 int tws, int inverse, double scale, int apply_scale) {
  const int64_t n = (int64_t)1 << log2n;
  const int64_t pairs = batch * (n / 2);
  const int64_t step = n / (2 * half);
  const uint64_t mask = ((uint64_t)1 << tws) - 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < pairs; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = q / (n / 2), r = q % (n / 2);
    const int64_t j = r % half;
    const int64_t i0 = v * n + (r / half) * 2 * half + j;
    const uint64_t e = (uint64_t)(j * step);
    cplx w = cmul(thi[e >> tws], tlo[e & mask]);
    if (inverse) w.im = -w.im;
    const cplx u = z[i0];
    const cplx t = cmul(z[i0 + half], w);
    cplx o0 = {u.re + t.re, u.im + t.im}, o1 = {u.re - t.re, u.im - t.im};
    if (apply_scale) {
      o0.re *= scale; o0.im *= scale; o1.re *= scale; o1.im *= scale;
    }
    z[i0] = o0;
    z[i0 + half] = o1;
  }
}

__global__ void cscale_kernel(cplx *z, int64_t n, double scale) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    z[q].re *= scale;
    z[q].im *= scale;
  }
}

// The stream-ordered scratch below comes from the device's default memory pool;
// with its default release threshold (0) every synchronisation returns the memory
// to the driver and the next cudaMallocAsync maps it again (milliseconds of host
// time while the GPU idles).  Keep freed blocks in the pool.
void keep_pool_memory() {
  static std::atomic<bool> done[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64 || done[dev].load(std::memory_order_relaxed)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev].store(true, std::memory_order_relaxed);
}

int fft_batched(cplx *z, int64_t batch, int log2n, int inverse, double scale, cudaStream_t s) {
  if (batch <= 0) return SMM_OK;
  keep_pool_memory();
  const int64_t n = (int64_t)1 << log2n;
  cplx *tab = nullptr;
  SMM_CUDA_TRY(cudaMallocAsync((void **)&tab, twiddle_table_bytes(log2n) + 16, s), "fft twiddle alloc");
  int tws = 0;
  int rc = twiddle_tables(log2n, tab, tab + ((int64_t)1 << (log2n / 2)), tws, s);
  if (rc) return rc;
  const cplx *tlo = tab, *thi = tab + ((int64_t)1 << (log2n / 2));
  int64_t blocks = ceil_div(batch * n, 256);
  if (blocks > 16384) blocks = 16384;
  bitrev_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, batch, log2n);
  SMM_LAUNCH_CHECK("bitrev_kernel");
  for (int64_t half = 1; half < n; half <<= 1) {
    const bool last = (half * 2 == n);
    fft_stage_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, batch, log2n, half, tlo, thi, tws, inverse, scale,
                                                     last ? 1 : 0);
    SMM_LAUNCH_CHECK("fft_stage_kernel");
  }
  if (n == 1 && scale != 1.0) cscale_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, batch, scale);
  SMM_CUDA_TRY(cudaFreeAsync(tab, s), "fft twiddle free");
  return SMM_OK;
}

// ---------------------------------------------------------------- finalize
__global__ void copy_kernel(const double *src, double *dst, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[q] = src[q];
}

__global__ void add_kernel(double *dst, const double *src, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    dst[q] += src[q];
}

// dst += src (n doubles): accumulate mode of the kernels that reduce their partials at the end
int add_inplace(double *dst, const double *src, int64_t n, cudaStream_t s) {
  if (n <= 0) return SMM_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 4 * 148 * 8) blocks = 4 * 148 * 8;
  add_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, src, n);
  SMM_LAUNCH_CHECK("add_kernel");
  return SMM_OK;
}

// z[t][u] = acc[t][u] (u <= b/2), z[t][b-u] = conj(acc[t][u]) (1 <= u < b/2): sketch.py:227-231
__global__ void hermitian_fill_kernel(const cplx *acc, cplx *z, int d, int log2b) {
  const int64_t b = (int64_t)1 << log2b, half = b / 2 + 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)d * b; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / b, u = q % b;
    cplx v;
    if (u < half) v = acc[t * half + u];
    else {
      cplx w = acc[t * half + (b - u)];
      v = {w.re, -w.im};
    }
    z[q] = v;
  }
}

__global__ void real_part_kernel(const cplx *z, double *out, int64_t n, double inv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = z[q].re * inv;
}

int finalize(int variant, const void *acc, double *polys, int d, int log2b, cudaStream_t s) {
  const int64_t b = (int64_t)1 << log2b;
  const double inv = 1.0 / (double)b;
  int64_t blocks = ceil_div((int64_t)d * b, 256);
  if (blocks > 16384) blocks = 16384;
  if (variant == SMM_VARIANT_FWHT) {
    if ((const double *)acc != polys) {
      copy_kernel<<<(unsigned)blocks, 256, 0, s>>>((const double *)acc, polys, (int64_t)d * b);
      SMM_LAUNCH_CHECK("copy_kernel");
    }
    return fwht_batched(polys, d, log2b, inv, s);
  }
  cplx *z = nullptr;
  keep_pool_memory();
  SMM_CUDA_TRY(cudaMallocAsync((void **)&z, (size_t)d * b * sizeof(cplx), s), "finalize alloc");
  hermitian_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>((const cplx *)acc, z, d, log2b);
  SMM_LAUNCH_CHECK("hermitian_fill_kernel");
  int rc = fft_batched(z, d, log2b, 1, 1.0, s);
  if (rc) return rc;
  real_part_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, polys, (int64_t)d * b, inv);
  SMM_LAUNCH_CHECK("real_part_kernel");
  SMM_CUDA_TRY(cudaFreeAsync(z, s), "finalize free");
  return SMM_OK;
}

// ---------------------------------------------------------------- transpose
// 64 x 64 tiles, 256 threads: 16 loads in flight per thread before the tile is
// written back (the 32 x 32 version kept only 4 outstanding and reached ~75 % of HBM)
__global__ void __launch_bounds__(256) transpose_kernel(const double *in, int64_t rows, int64_t cols, int64_t ld_in,
                                                        double *out, int64_t ld_out) {
  __shared__ double tile[64][65];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (int64_t r0 = (int64_t)blockIdx.y * 64; r0 < rows; r0 += (int64_t)gridDim.y * 64)
    for (int64_t c0 = (int64_t)blockIdx.x * 64; c0 < cols; c0 += (int64_t)gridDim.x * 64) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t r = r0 + ty + 4 * q, c = c0 + tx;
        v[q] = (r < rows && c < cols) ? in[r * ld_in + c] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) tile[ty + 4 * q][tx] = v[q];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t c = c0 + ty + 4 * q, r = r0 + tx;
        if (r < rows && c < cols) out[c * ld_out + r] = tile[tx][ty + 4 * q];
      }
      __syncthreads();
    }
}

int transpose(const double *in, int64_t rows, int64_t cols, int64_t ld_in, double *out, int64_t ld_out,
              cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return SMM_OK;
  int64_t gx = ceil_div(cols, 64), gy = ceil_div(rows, 64);
  if (gx > 65535) gx = 65535;
  if (gy > 65535) gy = 65535;
  transpose_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, s>>>(in, rows, cols, ld_in, out, ld_out);
  SMM_LAUNCH_CHECK("transpose_kernel");
  return SMM_OK;
}

}  // namespace smm
