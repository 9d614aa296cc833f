/*
 * CPU ORACLE — test infrastructure only.
 *
 * Plain-C restatement of the reference `sketchmm` hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the CHECKER.  It is never linked into, loaded by, or called from the
 * product package (paper_2601_09477_b200/), which fails loudly when its CUDA
 * library is missing.
 *
 * Every function follows the reference loop order statement by statement, so
 * that with -ffp-contract=off (no FMA contraction, no fast-math — the same
 * as Numba's default @njit) it reproduces the reference's float64 results
 * bit for bit at the same chunk (thread) count.  Pinned against the reference
 * itself by tests/test_oracle_pins.py using fixtures from tools/make_golden.py.
 *
 * Reference citations (paths relative to /root/reference/pkg/src/sketchmm):
 *   fwht_serial            transforms.py:37-49
 *   fft_serial             transforms.py:52-74
 *   fft_tables             transforms.py:80-97   (tables are built by the
 *                          Python wrapper with numpy, exactly as the reference)
 *   _compress_fwht_kernel  sketch.py:152-189
 *   _compress_fft_kernel   sketch.py:192-235
 *   _chunk_bounds          sketch.py:117-120
 *   decompress_all         sketch.py:375-399
 *   heavy-hitter threshold experiments.py:136-168 (inclusive) / BASELINE cfg5
 *                          (strict) — comparator chosen by the caller
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* transforms.py:37-49 */
static void fwht_serial(double *x, int64_t n) {
  int64_t h = 1;
  while (h < n) {
    int64_t step = h << 1;
    for (int64_t start = 0; start < n; start += step) {
      for (int64_t j = start; j < start + h; ++j) {
        double u = x[j];
        double v = x[j + h];
        x[j] = u + v;
        x[j + h] = u - v;
      }
    }
    h = step;
  }
}

typedef struct { double re, im; } cplx;

static inline cplx cmul(cplx a, cplx b) {  /* numba complex_mul: ac-bd, ad+bc */
  cplx r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}

/* transforms.py:52-74 */
static void fft_serial(cplx *z, int64_t n, const cplx *tw, const int64_t *rev) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = rev[i];
    if (j > i) { cplx t = z[i]; z[i] = z[j]; z[j] = t; }
  }
  int64_t size = 2;
  while (size <= n) {
    int64_t half = size >> 1;
    int64_t step = n / size;
    for (int64_t start = 0; start < n; start += size) {
      int64_t idx = 0;
      for (int64_t j = start; j < start + half; ++j) {
        cplx w = tw[idx];
        cplx u = z[j];
        cplx v = cmul(z[j + half], w);
        z[j].re = u.re + v.re; z[j].im = u.im + v.im;
        z[j + half].re = u.re - v.re; z[j + half].im = u.im - v.im;
        idx += step;
      }
    }
    size <<= 1;
  }
}

void oracle_fwht_inplace(double *x, int64_t n) { fwht_serial(x, n); }
void oracle_fft_inplace(double *z, int64_t n, const double *tw, const int64_t *rev) {
  fft_serial((cplx *)z, n, (const cplx *)tw, rev);
}

/*
 * sketch.py:152-189.  at: (m, n1) row-major, bm: (m, n2) row-major.
 * h1/h2: (d, n1)/(d, n2) int64 buckets; s1/s2 float64 signs.
 * starts/ends: nchunks chunk bounds over m.  out: (d, b) float64.
 */
int oracle_compress_fwht(const double *at, const double *bm, int64_t m, int64_t n1, int64_t n2,
                         const int64_t *h1, const double *s1, const int64_t *h2, const double *s2,
                         int d, int64_t b, const int64_t *starts, const int64_t *ends, int nchunks,
                         int threads, double *out) {
  double *partial = (double *)calloc((size_t)nchunks * d * b, sizeof(double));
  if (!partial) return 1;
  (void)m;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int c = 0; c < nchunks; ++c) {
    double *pa = (double *)malloc((size_t)d * b * sizeof(double));
    double *pb = (double *)malloc((size_t)b * sizeof(double));
    for (int64_t k = starts[c]; k < ends[c]; ++k) {
      const double *ark = at + k * n1;
      const double *brk = bm + k * n2;
      for (int t = 0; t < d; ++t) {
        double *row = pa + (int64_t)t * b;
        memset(row, 0, (size_t)b * sizeof(double));
        const int64_t *ht = h1 + (int64_t)t * n1;
        const double *st = s1 + (int64_t)t * n1;
        for (int64_t i = 0; i < n1; ++i) row[ht[i]] += st[i] * ark[i];
        fwht_serial(row, b);
      }
      for (int t = 0; t < d; ++t) {
        memset(pb, 0, (size_t)b * sizeof(double));
        const int64_t *ht = h2 + (int64_t)t * n2;
        const double *st = s2 + (int64_t)t * n2;
        for (int64_t j = 0; j < n2; ++j) pb[ht[j]] += st[j] * brk[j];
        fwht_serial(pb, b);
        double *acc = partial + ((int64_t)c * d + t) * b;
        const double *row = pa + (int64_t)t * b;
        for (int64_t u = 0; u < b; ++u) acc[u] += row[u] * pb[u];
      }
    }
    free(pa);
    free(pb);
  }
  memset(out, 0, (size_t)d * b * sizeof(double));
  for (int c = 0; c < nchunks; ++c)
    for (int t = 0; t < d; ++t)
      for (int64_t u = 0; u < b; ++u) out[(int64_t)t * b + u] += partial[((int64_t)c * d + t) * b + u];
  free(partial);
  double inv = 1.0 / (double)b;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int t = 0; t < d; ++t) {
    double *row = out + (int64_t)t * b;
    fwht_serial(row, b);
    for (int64_t u = 0; u < b; ++u) row[u] *= inv;
  }
  return 0;
}

/* Accumulate-only FWHT variant over an arbitrary k-range with one chunk: used by
 * the CPU baseline (bounded k-slices) and the multi-GPU emulation checks.
 * acc (d, b) is ADDED to (pre-inverse accumulator). */
int oracle_accumulate_fwht(const double *at, const double *bm, int64_t n1, int64_t n2,
                           const int64_t *h1, const double *s1, const int64_t *h2, const double *s2,
                           int d, int64_t b, int64_t k0, int64_t k1, int threads, double *acc) {
  int nchunks = threads > 0 ? threads : 1;
  int64_t starts[1024], ends[1024];
  if (nchunks > 1024) nchunks = 1024;
  for (int c = 0; c <= nchunks - 1; ++c) {
    starts[c] = k0 + (k1 - k0) * c / nchunks;
    ends[c] = k0 + (k1 - k0) * (c + 1) / nchunks;
  }
  double *partial = (double *)calloc((size_t)nchunks * d * b, sizeof(double));
  if (!partial) return 1;
#ifdef _OPENMP
  omp_set_num_threads(nchunks);
#pragma omp parallel for schedule(static, 1)
#endif
  for (int c = 0; c < nchunks; ++c) {
    double *pa = (double *)malloc((size_t)d * b * sizeof(double));
    double *pb = (double *)malloc((size_t)b * sizeof(double));
    for (int64_t k = starts[c]; k < ends[c]; ++k) {
      const double *ark = at + k * n1;
      const double *brk = bm + k * n2;
      for (int t = 0; t < d; ++t) {
        double *row = pa + (int64_t)t * b;
        memset(row, 0, (size_t)b * sizeof(double));
        for (int64_t i = 0; i < n1; ++i) row[h1[(int64_t)t * n1 + i]] += s1[(int64_t)t * n1 + i] * ark[i];
        fwht_serial(row, b);
      }
      for (int t = 0; t < d; ++t) {
        memset(pb, 0, (size_t)b * sizeof(double));
        for (int64_t j = 0; j < n2; ++j) pb[h2[(int64_t)t * n2 + j]] += s2[(int64_t)t * n2 + j] * brk[j];
        fwht_serial(pb, b);
        double *a = partial + ((int64_t)c * d + t) * b;
        const double *row = pa + (int64_t)t * b;
        for (int64_t u = 0; u < b; ++u) a[u] += row[u] * pb[u];
      }
    }
    free(pa);
    free(pb);
  }
  for (int c = 0; c < nchunks; ++c)
    for (int64_t q = 0; q < (int64_t)d * b; ++q) acc[q] += partial[(int64_t)c * d * b + q];
  free(partial);
  return 0;
}

/*
 * sketch.py:192-235.  tw/twi: (b/2) complex128 as interleaved doubles,
 * rev: (b) int64 — both built by numpy in the wrapper exactly as
 * fft_tables (transforms.py:80-97).
 */
int oracle_compress_fft(const double *at, const double *bm, int64_t m, int64_t n1, int64_t n2,
                        const int64_t *h1, const double *s1, const int64_t *h2, const double *s2,
                        int d, int64_t b, const double *tw_, const double *twi_, const int64_t *rev,
                        const int64_t *starts, const int64_t *ends, int nchunks, int threads,
                        double *out) {
  const cplx *tw = (const cplx *)tw_;
  const cplx *twi = (const cplx *)twi_;
  int64_t half = (b >> 1) + 1;
  cplx *partial = (cplx *)calloc((size_t)nchunks * d * half, sizeof(cplx));
  if (!partial) return 1;
  (void)m;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int c = 0; c < nchunks; ++c) {
    cplx *z = (cplx *)malloc((size_t)b * sizeof(cplx));
    for (int64_t k = starts[c]; k < ends[c]; ++k) {
      const double *ark = at + k * n1;
      const double *brk = bm + k * n2;
      for (int t = 0; t < d; ++t) {
        memset(z, 0, (size_t)b * sizeof(cplx));
        for (int64_t i = 0; i < n1; ++i) {
          /* z[h1] += s1*at  (real added to complex: imag += 0.0) */
          int64_t h = h1[(int64_t)t * n1 + i];
          z[h].re += s1[(int64_t)t * n1 + i] * ark[i];
          z[h].im += 0.0;
        }
        for (int64_t j = 0; j < n2; ++j) {
          /* z[h2] += (s2*bm) * 1j  -> complex_mul((x,0),(0,1)) = (x*0 - 0*1, x*1 + 0*0) */
          int64_t h = h2[(int64_t)t * n2 + j];
          double x = s2[(int64_t)t * n2 + j] * brk[j];
          cplx p;
          p.re = x * 0.0 - 0.0 * 1.0;
          p.im = x * 1.0 + 0.0 * 0.0;
          z[h].re += p.re;
          z[h].im += p.im;
        }
        fft_serial(z, b, tw, rev);
        cplx *acc = partial + ((int64_t)c * d + t) * half;
        for (int64_t u = 0; u < half; ++u) {
          cplx zu = z[u];
          cplx zc = z[(b - u) & (b - 1)];
          cplx zv = {zc.re, -zc.im};
          cplx s = {zu.re + zv.re, zu.im + zv.im};
          cplx dd = {zu.re - zv.re, zu.im - zv.im};
          cplx half_c = {0.5, 0.0};
          cplx fa = cmul(half_c, s);               /* 0.5 * (zu + zv) */
          cplx mhj = {-0.0, -0.5};                  /* Python literal -0.5j */
          cplx fb = cmul(mhj, dd);                  /* -0.5j * (zu - zv) */
          cplx pr = cmul(fa, fb);
          acc[u].re += pr.re;
          acc[u].im += pr.im;
        }
      }
    }
    free(z);
  }
  cplx *total = (cplx *)calloc((size_t)d * half, sizeof(cplx));
  for (int c = 0; c < nchunks; ++c)
    for (int t = 0; t < d; ++t)
      for (int64_t u = 0; u < half; ++u) {
        total[(int64_t)t * half + u].re += partial[((int64_t)c * d + t) * half + u].re;
        total[(int64_t)t * half + u].im += partial[((int64_t)c * d + t) * half + u].im;
      }
  free(partial);
  double inv = 1.0 / (double)b;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int t = 0; t < d; ++t) {
    cplx *z = (cplx *)malloc((size_t)b * sizeof(cplx));
    for (int64_t u = 0; u < half; ++u) z[u] = total[(int64_t)t * half + u];
    for (int64_t u = 1; u < (b >> 1); ++u) {
      cplx v = total[(int64_t)t * half + u];
      z[b - u].re = v.re;
      z[b - u].im = -v.im;
    }
    fft_serial(z, b, twi, rev);
    for (int64_t u = 0; u < b; ++u) out[(int64_t)t * b + u] = z[u].re * inv;
    free(z);
  }
  free(total);
  return 0;
}

/* middle order statistic of d (odd) values — np.median for odd d */
static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x > y) - (x < y);
}

/*
 * sketch.py:375-399 plus the heavy-hitter threshold.  Rows [r0, r1) of the
 * n1 x n2 estimate; est_out may be NULL.  Heavy hitters (|est| > thr if strict,
 * >= thr otherwise) are counted into *hh_count and, if hh_out != NULL, written
 * as (i, j) pairs in row-major order up to hh_cap pairs.
 */
int oracle_decompress(const double *polys, int d, int64_t b, int xor_combine,
                      const int64_t *h1, const double *s1, const int64_t *h2, const double *s2,
                      int64_t n1, int64_t n2, int64_t r0, int64_t r1, double *est_out,
                      double thr, int strict, int64_t *hh_out, int64_t hh_cap, int64_t *hh_count,
                      int threads) {
  (void)n1;
  int64_t rows = r1 - r0;
  int64_t *row_counts = (int64_t *)calloc((size_t)(rows > 0 ? rows : 1), sizeof(int64_t));
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t r = 0; r < rows; ++r) {
    int64_t i = r0 + r;
    double vals[256];
    int64_t cnt = 0;
    for (int64_t j = 0; j < n2; ++j) {
      for (int t = 0; t < d; ++t) {
        int64_t a = h1[(int64_t)t * n1 + i], c = h2[(int64_t)t * n2 + j];
        int64_t idx = xor_combine ? (a ^ c) : ((a + c) % b);
        double v = polys[(int64_t)t * b + idx];
        v *= s1[(int64_t)t * n1 + i];
        v *= s2[(int64_t)t * n2 + j];
        vals[t] = v;
      }
      int has_nan = 0;
      for (int t = 0; t < d; ++t) has_nan |= isnan(vals[t]);
      qsort(vals, (size_t)d, sizeof(double), cmp_double);
      double e = has_nan ? NAN : vals[(d - 1) / 2];  /* np.median: any NaN gives NaN */
      if (est_out) est_out[r * n2 + j] = e;
      double ae = fabs(e);
      if (strict ? (ae > thr) : (ae >= thr)) cnt++;
    }
    row_counts[r] = cnt;
  }
  int64_t total = 0;
  for (int64_t r = 0; r < rows; ++r) total += row_counts[r];
  *hh_count = total;
  if (hh_out) {
    int64_t w = 0;
    for (int64_t r = 0; r < rows && w < hh_cap; ++r) {
      if (!row_counts[r]) continue;
      int64_t i = r0 + r;
      for (int64_t j = 0; j < n2 && w < hh_cap; ++j) {
        double vals[256];
        for (int t = 0; t < d; ++t) {
          int64_t a = h1[(int64_t)t * n1 + i], c = h2[(int64_t)t * n2 + j];
          int64_t idx = xor_combine ? (a ^ c) : ((a + c) % b);
          double v = polys[(int64_t)t * b + idx];
          v *= s1[(int64_t)t * n1 + i];
          v *= s2[(int64_t)t * n2 + j];
          vals[t] = v;
        }
        qsort(vals, (size_t)d, sizeof(double), cmp_double);
        double ae = fabs(vals[(d - 1) / 2]);
        if (strict ? (ae > thr) : (ae >= thr)) { hh_out[2 * w] = i; hh_out[2 * w + 1] = j; ++w; }
      }
    }
  }
  free(row_counts);
  return 0;
}
