// FFT compress (steps 1-3, cyclic-convolution variant).
//
// Reference: sketch.py:192-235 (`_compress_fft_kernel`), transforms.py:52-97.
// The reference packs A into the real and B into the imaginary part of one
// complex length-b signal z, runs one FFT, splits the spectra
//     FA[u] = (Z[u] + conj Z[-u]) / 2,   FB[u] = -i/2 (Z[u] - conj Z[-u])
// and accumulates FA*FB over k.  Here the b-point FFT is decimated in
// frequency into F = b/l slices (u = a + F*u'):
//     Z[a + F u'] = DFT_l(y_a)[u'],  y_a[m'] = sum_{m = m' mod l} z[m] w_b^(a*m)
// so one CTA owns the slice pair {a, -a mod F} of one repetition t (the pair
// needed by the split), folds the packed inputs directly into l buckets with
// the twiddle w_b^(a*h), runs two l-point FFTs in shared memory and keeps the
// product spectrum of both slices on chip across its k-range.
#include "plan.cuh"

namespace smm {

struct FftArgs {
  SketchHashes h;
  const double *at;
  int64_t ld_at;
  const double *bm;
  int64_t ld_bm;
  int64_t n1, n2, k0, K, W;
  int L, F, G, maxseg, nunits, tw_s;
  char *plans;
  int64_t plan_per, plan_nin_max;
  const cplx *tlo, *thi;  // w_b^q = thi[q >> tw_s] * tlo[q & ((1<<tw_s)-1)]
  cplx *partial;          // [G][maxseg][2][l]
};

constexpr int CT = 256;

__device__ __forceinline__ cplx twiddle_b(const FftArgs &p, uint64_t q) {
  const uint64_t mask = ((uint64_t)1 << p.tw_s) - 1;
  cplx lo = p.tlo[q & mask];
  cplx hi = p.thi[q >> p.tw_s];
  return cmul(hi, lo);
}

__device__ __forceinline__ void unit_slices(int F, int unit, int &a0, int &a1, int &nsl) {
  if (F == 1) { a0 = 0; a1 = 0; nsl = 1; return; }
  if (unit == 0) { a0 = 0; a1 = F / 2; nsl = 2; return; }
  a0 = unit; a1 = F - unit; nsl = 2;
}

__device__ void fold_scatter_fft(const FftArgs &p, int t, int a, int64_t k, cplx *Y) {
  const int tid = threadIdx.x;
  const double *rowa = p.at + k * p.ld_at;
  const double *rowb = p.bm + k * p.ld_bm;
  const int log2b = p.h.log2b;
  const uint64_t bmask = ((uint64_t)1 << log2b) - 1;
  const uint32_t cmask = (1u << p.L) - 1u;
  PlanView pv = plan_view_dev(p.plans, p.plan_per, p.plan_nin_max, p.L, 1, t, 0);
  const int nrounds = pv.meta[0];
  const int nempty = pv.meta[1];
  for (int e = tid; e < nempty; e += CT) Y[pv.empty[e]] = {0.0, 0.0};
  for (int r = 0; r < nrounds; ++r) {
    const int e0 = pv.roff[r], e1 = pv.roff[r + 1];
    for (int e = e0 + tid; e < e1; e += CT) {
      const int64_t q = pv.list[e];
      uint32_t m;
      double x;
      bool is_b = q >= p.n1;
      if (!is_b) {
        m = eval_bucket(p.h.f[0][t], (uint64_t)q, log2b);
        x = apply_sign(__ldg(rowa + q), eval_signbit(p.h.f[2][t], (uint64_t)q));
      } else {
        const int64_t j = q - p.n1;
        m = eval_bucket(p.h.f[1][t], (uint64_t)j, log2b);
        x = apply_sign(__ldg(rowb + j), eval_signbit(p.h.f[3][t], (uint64_t)j));
      }
      cplx w = twiddle_b(p, ((uint64_t)a * m) & bmask);
      cplx v = is_b ? cplx{-x * w.im, x * w.re} : cplx{x * w.re, x * w.im};
      const uint32_t c = m & cmask;
      if (r == 0) Y[c] = v;
      else { Y[c].re += v.re; Y[c].im += v.im; }
    }
    __syncthreads();
  }
  if (nrounds == 0) __syncthreads();
}

// In-place l-point forward DFT (natural order in and out): bit reversal + radix-2 DIT.
__device__ void block_fft(cplx *Y, const cplx *TW, int L) {
  const int ell = 1 << L;
  const int tid = threadIdx.x;
  for (int i = tid; i < ell; i += CT) {
    int j = (int)(__brev((unsigned)i) >> (32 - L));
    if (L == 0) j = 0;
    if (j > i) { cplx tmp = Y[i]; Y[i] = Y[j]; Y[j] = tmp; }
  }
  __syncthreads();
  for (int half = 1; half < ell; half <<= 1) {
    const int step = ell / (2 * half);
    for (int q = tid; q < ell / 2; q += CT) {
      const int grp = q / half, j = q % half;
      const int i0 = grp * 2 * half + j;
      cplx w = TW[j * step];
      cplx u = Y[i0];
      cplx v = cmul(Y[i0 + half], w);
      Y[i0] = {u.re + v.re, u.im + v.im};
      Y[i0 + half] = {u.re - v.re, u.im - v.im};
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(CT) fft_fold_kernel(FftArgs p) {
  extern __shared__ __align__(16) double smem_d[];
  cplx *smem = (cplx *)smem_d;
  const int ell = 1 << p.L;
  cplx *Y0 = smem, *Y1 = smem + ell, *A0 = smem + 2 * ell, *A1 = smem + 3 * ell, *TW = smem + 4 * ell;
  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  // l-point twiddles w_l^j = w_b^(F j)
  for (int j = tid; j < ell / 2; j += CT) TW[j] = twiddle_b(p, (uint64_t)p.F * j);
  __syncthreads();
  int64_t w0 = (p.W * g) / p.G, w1 = (p.W * (g + 1)) / p.G;
  int seg = 0;
  while (w0 < w1) {
    const int64_t item = w0 / p.K;
    const int64_t kk = w0 % p.K;
    const int64_t kend = (p.K < kk + (w1 - w0)) ? p.K : kk + (w1 - w0);
    const int t = (int)(item / p.nunits), unit = (int)(item % p.nunits);
    int a0, a1, nsl;
    unit_slices(p.F, unit, a0, a1, nsl);
    for (int c = tid; c < ell; c += CT) { A0[c] = {0.0, 0.0}; A1[c] = {0.0, 0.0}; }
    __syncthreads();
    for (int64_t k = p.k0 + kk; k < p.k0 + kend; ++k) {
      fold_scatter_fft(p, t, a0, k, Y0);
      block_fft(Y0, TW, p.L);
      if (nsl == 2) {
        fold_scatter_fft(p, t, a1, k, Y1);
        block_fft(Y1, TW, p.L);
      }
      for (int s = 0; s < nsl; ++s) {
        const int a = s == 0 ? a0 : a1;
        cplx *Ys = s == 0 ? Y0 : Y1;
        cplx *Acc = s == 0 ? A0 : A1;
        for (int u = tid; u < ell; u += CT) {
          cplx zu = Ys[u];
          cplx zm;
          if (a == 0) zm = Y0[(ell - u) & (ell - 1)];
          else {
            // partner slice F - a holds index l - 1 - u
            const int pa = p.F - a;
            cplx *Yp = (pa == a0) ? Y0 : Y1;
            zm = Yp[ell - 1 - u];
          }
          cplx zv = {zm.re, -zm.im};
          cplx sum = {zu.re + zv.re, zu.im + zv.im};
          cplx dif = {zu.re - zv.re, zu.im - zv.im};
          cplx fa = {0.5 * sum.re, 0.5 * sum.im};
          cplx fb = {0.5 * dif.im, -0.5 * dif.re};
          cplx pr = cmul(fa, fb);
          Acc[u].re += pr.re;
          Acc[u].im += pr.im;
        }
      }
      __syncthreads();
    }
    cplx *dst = p.partial + ((int64_t)g * p.maxseg + seg) * 2 * ell;
    for (int c = tid; c < ell; c += CT) { dst[c] = A0[c]; dst[ell + c] = A1[c]; }
    __syncthreads();
    ++seg;
    w0 += kend - kk;
  }
}

// acc[t][u] (u in [0, b/2]) from the slice partials, summed in CTA order.
__global__ void fft_reduce_kernel(const cplx *partial, cplx *acc, int64_t W, int G, int maxseg, int64_t K, int F,
                                  int L, int nunits, int d, int log2b) {
  const int64_t ell = (int64_t)1 << L;
  const int64_t half = ((int64_t)1 << log2b) / 2 + 1;
  const int64_t total = (int64_t)d * half;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / half);
    const int64_t u = x % half;
    const int a = (int)(u % F);
    const int64_t up = u / F;
    int unit, slot;
    if (F == 1) { unit = 0; slot = 0; }
    else if (a == 0) { unit = 0; slot = 0; }
    else if (2 * a == F) { unit = 0; slot = 1; }
    else if (2 * a < F) { unit = a; slot = 0; }
    else { unit = F - a; slot = 1; }
    const int64_t item = (int64_t)t * nunits + unit;
    cplx s = {0.0, 0.0};
    if (K > 0) {
      const int64_t lo = item * K, hi = (item + 1) * K;
      int64_t g = (lo * G) / W;
      if (g >= G) g = G - 1;
      while (g > 0 && (W * g) / G > lo) --g;
      while (g < G && (W * (g + 1)) / G <= lo) ++g;
      for (; g < G && (W * g) / G < hi; ++g) {
        const int64_t w0 = (W * g) / G, w1 = (W * (g + 1)) / G;
        if (w1 <= w0) continue;
        const int64_t segi = item - w0 / K;
        cplx v = partial[(((int64_t)g * maxseg + segi) * 2 + slot) * ell + up];
        s.re += v.re;
        s.im += v.im;
      }
    }
    acc[x] = s;
  }
}

__global__ void twiddle_tables_kernel(cplx *tlo, cplx *thi, int log2b, int s) {
  const int64_t nlo = (int64_t)1 << s, nhi = (int64_t)1 << (log2b - s);
  const double b = ldexp(1.0, log2b);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nlo + nhi; q += (int64_t)gridDim.x * blockDim.x) {
    const double e = q < nlo ? (double)q : (double)((q - nlo) << s);
    double sn, cs;
    sincospi(-2.0 * e / b, &sn, &cs);
    if (q < nlo) tlo[q] = {cs, sn};
    else thi[q - nlo] = {cs, sn};
  }
}

int twiddle_tables(int log2b, cplx *tlo, cplx *thi, int &s, cudaStream_t st) {
  s = log2b / 2;
  const int64_t n = ((int64_t)1 << s) + ((int64_t)1 << (log2b - s));
  int64_t blocks = ceil_div(n, 256);
  twiddle_tables_kernel<<<(unsigned)(blocks > 1024 ? 1024 : blocks), 256, 0, st>>>(tlo, thi, log2b, s);
  SMM_LAUNCH_CHECK("twiddle_tables_kernel");
  return SMM_OK;
}

int64_t twiddle_table_bytes(int log2b) {
  const int s = log2b / 2;
  return (((int64_t)1 << s) + ((int64_t)1 << (log2b - s))) * (int64_t)sizeof(cplx);
}

static int fft_L(int log2b) { return log2b < 11 ? log2b : 11; }

static void fft_geometry(int d, int log2b, int64_t K, int Gmax, int &L, int &F, int &nunits, int64_t &W, int &G,
                         int &maxseg) {
  L = fft_L(log2b);
  F = 1 << (log2b - L);
  nunits = F == 1 ? 1 : F / 2;
  W = (int64_t)d * nunits * K;
  G = Gmax;
  if (W > 0 && W < G) G = (int)W;
  if (W == 0) G = 1;
  const int64_t per = W > 0 ? ceil_div(W, G) : 1;
  maxseg = (int)(K > 0 ? ceil_div(per, K) + 1 : 1);
}

static inline int64_t pad(int64_t x) { return ((x + 255) / 256) * 256; }

int64_t fft_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int Gmax) {
  int L, F, nunits, G, maxseg;
  int64_t W;
  fft_geometry(d, log2b, K, Gmax, L, F, nunits, W, G, maxseg);
  const int64_t Gws = Gmax;  // upper bound on G
  return pad(plan_total_bytes(d, 1, n1, n2, L)) + pad(twiddle_table_bytes(log2b)) +
         Gws * (int64_t)maxseg * 2 * ((int64_t)1 << L) * (int64_t)sizeof(cplx);
}

int fft_accumulate(const SketchHashes &h, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm,
                   int64_t n1, int64_t n2, int64_t k0, int64_t k1, cplx *acc, char *ws, int64_t ws_bytes,
                   cudaStream_t s) {
  const int d = h.d, log2b = h.log2b;
  const int64_t K = k1 - k0;
  FftArgs p;
  int64_t W;
  fft_geometry(d, log2b, K, num_sms(), p.L, p.F, p.nunits, W, p.G, p.maxseg);
  const int64_t need = fft_workspace(d, log2b, n1, n2, K, num_sms());
  if (ws_bytes < need) {
    set_error("compress workspace too small: %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    return SMM_ERR_WORKSPACE;
  }
  p.h = h;
  p.at = at;
  p.ld_at = ld_at;
  p.bm = bm;
  p.ld_bm = ld_bm;
  p.n1 = n1;
  p.n2 = n2;
  p.k0 = k0;
  p.K = K;
  p.W = W;
  p.plans = ws;
  p.plan_nin_max = n1 + n2;
  p.plan_per = plan_bytes_per(p.plan_nin_max, p.L);
  char *q = ws + pad(plan_total_bytes(d, 1, n1, n2, p.L));
  cplx *tlo = (cplx *)q;
  int tws = 0;
  int rc = twiddle_tables(log2b, tlo, tlo + ((int64_t)1 << (log2b / 2)), tws, s);
  if (rc) return rc;
  p.tlo = tlo;
  p.thi = tlo + ((int64_t)1 << (log2b / 2));
  p.tw_s = tws;
  q += pad(twiddle_table_bytes(log2b));
  p.partial = (cplx *)q;
  const int64_t ell = (int64_t)1 << p.L;
  if (W > 0) {
    rc = build_plans(h, 1, n1, n2, p.L, ws, s);
    if (rc) return rc;
    size_t smem = (4 * ell + ell / 2 + 1) * sizeof(cplx);
    SMM_CUDA_TRY(cudaFuncSetAttribute(fft_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "fft_fold_kernel smem");
    fft_fold_kernel<<<p.G, CT, smem, s>>>(p);
    SMM_LAUNCH_CHECK("fft_fold_kernel");
  }
  const int64_t total = (int64_t)d * (((int64_t)1 << log2b) / 2 + 1);
  int64_t blocks = ceil_div(total, 256);
  if (blocks > 8192) blocks = 8192;
  fft_reduce_kernel<<<(unsigned)blocks, 256, 0, s>>>(p.partial, acc, W, p.G, p.maxseg, K, p.F, p.L, p.nunits, d,
                                                      log2b);
  SMM_LAUNCH_CHECK("fft_reduce_kernel");
  return SMM_OK;
}

}  // namespace smm
