// FWHT compress (steps 1-3): fused fold-scatter + on-chip Walsh-Hadamard
// transform + pointwise product accumulated over the inner dimension.
//
// Reference: sketch.py:152-189 (`_compress_fwht_kernel`), transforms.py:37-49.
//
// Decomposition: the length-b transform of each scattered
// column is never materialised.  With b = F * l (l <= 2^13 on chip), the
// outputs u = a*l + c of slice a satisfy
//     FWHT_b(x)[a*l + c] = FWHT_l(y_a)[c],
//     y_a[c] = sum_{i : h(i) mod l = c} s(i) * (-1)^popcount(a & (h(i) >> log2 l)) * x_i,
// so a CTA that owns (repetition t, slice a) folds the n inputs straight into
// l buckets (the "scatter" of the reference, with an extra sign) and runs an
// l-point FWHT entirely in registers + shared memory.  Both operands of the
// same (t, a, k) are transformed by the same CTA, so the product and its sum
// over k stay on chip: only one d x b accumulator ever leaves the SM.
//
// Work split: the d*F*K (item, k) steps are cut into G equal contiguous ranges
// (persistent grid, one CTA per SM); a CTA emits one partial slice per item it
// touches, and reduce_partials sums them in CTA order (deterministic).
#include "plan.cuh"

namespace smm {

struct FwhtArgs {
  SketchHashes h;
  const double *at;
  int64_t ld_at;
  const double *bm;
  int64_t ld_bm;
  int64_t n1, n2, k0, K, W;
  int L, F, G, maxseg;
  char *plans;
  int64_t plan_per, plan_nin_max;
  double *partial;  // [G][maxseg][l]
};

constexpr int FT = 256;  // threads per CTA in the fold kernels

__device__ __forceinline__ void cta_range(int64_t W, int G, int g, int64_t &w0, int64_t &w1) {
  w0 = (W * g) / G;
  w1 = (W * (g + 1)) / G;
}

// ---------------------------------------------------------------- scatter
// Fold-scatter of operand `op` (0: A via at row k, 1: B via bm row k) for
// repetition t and slice a into X (l doubles, swizzled by PHYS).
template <class Phys>
__device__ __forceinline__ void fold_scatter(const FwhtArgs &p, int op, int t, int a, int64_t k, double *X,
                                             Phys phys) {
  const int tid = threadIdx.x;
  const double *row = op == 0 ? p.at + k * p.ld_at : p.bm + k * p.ld_bm;
  const HashFn hb = p.h.f[op][t];
  const HashFn hs = p.h.f[2 + op][t];
  const int log2b = p.h.log2b;
  const int L = p.L;
  const uint32_t cmask = (1u << L) - 1u;
  PlanView pv = plan_view_dev(p.plans, p.plan_per, p.plan_nin_max, L, 2, t, op);
  const int nrounds = pv.meta[0];
  const int nempty = pv.meta[1];
  for (int e = tid; e < nempty; e += FT) X[phys(pv.empty[e])] = 0.0;
  for (int r = 0; r < nrounds; ++r) {
    const int e0 = pv.roff[r], e1 = pv.roff[r + 1];
    for (int e = e0 + tid; e < e1; e += 4 * FT) {
      uint32_t q[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = (e + u * FT < e1) ? pv.list[e + u * FT] : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (e + u * FT < e1) ? __ldg(row + q[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (e + u * FT < e1) {
          uint32_t m = eval_bucket(hb, (uint64_t)q[u], log2b);
          uint32_t sb = eval_signbit(hs, (uint64_t)q[u]) ^ (__popc((m >> L) & (uint32_t)a) & 1u);
          double x = apply_sign(v[u], sb);
          int pos = phys(m & cmask);
          if (r == 0) X[pos] = x;
          else X[pos] += x;
        }
      }
    }
    __syncthreads();
  }
  if (nrounds == 0) __syncthreads();
}

// ---------------------------------------------------------------- register/smem FWHT
template <int L>
struct Layout {
  static constexpr int RHO = L - 8;  // log2 registers per thread (FT = 256 = 2^8 threads)
  static constexpr int R = 1 << RHO;
  static constexpr int P = (L + RHO - 1) / RHO;  // phases
  static_assert(RHO >= 4 && RHO <= 5, "fold kernel supports l = 2^12 and 2^13");
  __device__ static constexpr int start(int p) { return p * RHO < L - RHO ? p * RHO : L - RHO; }
  __device__ static __forceinline__ int idx(int p, int tid, int j) {
    const int s = start(p);
    return (tid & ((1 << s) - 1)) | ((tid >> s) << (s + RHO)) | (j << s);
  }
  __device__ static __forceinline__ int phys(int i) { return i ^ ((i >> RHO) & 15); }
};

template <int L>
__device__ __forceinline__ void reg_stages(double (&v)[Layout<L>::R], int qlo, int qhi) {
  constexpr int R = Layout<L>::R;
#pragma unroll
  for (int q = 0; q < Layout<L>::RHO; ++q) {
    if (q >= qlo && q < qhi) {
      const int h = 1 << q;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (!(j & h)) {
          double x = v[j], y = v[j + h];
          v[j] = x + y;
          v[j + h] = x - y;
        }
      }
    }
  }
}

// X0 holds the folded vector (phys layout).  On return v holds the transform in
// the last phase's mapping.  Uses X1 as the ping-pong exchange buffer.
template <int L>
__device__ __forceinline__ void block_fwht(double (&v)[Layout<L>::R], double *X0, double *X1) {
  using Lo = Layout<L>;
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < Lo::R; ++j) v[j] = X0[Lo::phys(Lo::idx(0, tid, j))];
  reg_stages<L>(v, 0, Lo::RHO);
#pragma unroll
  for (int p = 1; p < Lo::P; ++p) {
    double *Xs = (p & 1) ? X1 : X0;
#pragma unroll
    for (int j = 0; j < Lo::R; ++j) Xs[Lo::phys(Lo::idx(p - 1, tid, j))] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < Lo::R; ++j) v[j] = Xs[Lo::phys(Lo::idx(p, tid, j))];
    const int s = Lo::start(p);
    const int hi = (p + 1) * Lo::RHO < L ? (p + 1) * Lo::RHO : L;
    reg_stages<L>(v, p * Lo::RHO - s, hi - s);
  }
}

template <int L>
__global__ void __launch_bounds__(FT, 1) fwht_fold_kernel(FwhtArgs p) {
  using Lo = Layout<L>;
  constexpr int ELL = 1 << L;
  extern __shared__ __align__(16) double smem[];
  double *X0 = smem, *X1 = smem + ELL, *FA = smem + 2 * ELL;
  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  int64_t w0, w1;
  cta_range(p.W, p.G, g, w0, w1);
  int seg = 0;
  auto phys = [](uint32_t c) { return Lo::phys((int)c); };
  while (w0 < w1) {
    const int64_t item = w0 / p.K;
    const int64_t kk = w0 % p.K;
    const int64_t kend = (p.K < kk + (w1 - w0)) ? p.K : kk + (w1 - w0);
    const int t = (int)(item / p.F), a = (int)(item % p.F);
    double acc[Lo::R];
#pragma unroll
    for (int j = 0; j < Lo::R; ++j) acc[j] = 0.0;
    for (int64_t k = p.k0 + kk; k < p.k0 + kend; ++k) {
      double v[Lo::R];
      fold_scatter(p, 0, t, a, k, X0, phys);
      block_fwht<L>(v, X0, X1);
#pragma unroll
      for (int j = 0; j < Lo::R; ++j) FA[j * FT + tid] = v[j];
      __syncthreads();
      fold_scatter(p, 1, t, a, k, X0, phys);
      block_fwht<L>(v, X0, X1);
#pragma unroll
      for (int j = 0; j < Lo::R; ++j) acc[j] = fma(FA[j * FT + tid], v[j], acc[j]);
      __syncthreads();
    }
    double *dst = p.partial + ((int64_t)g * p.maxseg + seg) * ELL;
#pragma unroll
    for (int j = 0; j < Lo::R; ++j) dst[Lo::idx(Lo::P - 1, tid, j)] = acc[j];
    ++seg;
    w0 += kend - kk;
  }
}

// Generic fold kernel for small l (any L <= 12): smem butterflies, smem accumulator.
__global__ void __launch_bounds__(FT) fwht_fold_small_kernel(FwhtArgs p) {
  extern __shared__ __align__(16) double smem[];
  const int ell = 1 << p.L;
  double *X = smem, *FA = smem + ell, *ACC = smem + 2 * ell;
  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  int64_t w0, w1;
  cta_range(p.W, p.G, g, w0, w1);
  int seg = 0;
  auto phys = [](uint32_t c) { return (int)c; };
  while (w0 < w1) {
    const int64_t item = w0 / p.K;
    const int64_t kk = w0 % p.K;
    const int64_t kend = (p.K < kk + (w1 - w0)) ? p.K : kk + (w1 - w0);
    const int t = (int)(item / p.F), a = (int)(item % p.F);
    for (int c = tid; c < ell; c += FT) ACC[c] = 0.0;
    __syncthreads();
    for (int64_t k = p.k0 + kk; k < p.k0 + kend; ++k) {
      for (int op = 0; op < 2; ++op) {
        fold_scatter(p, op, t, a, k, X, phys);
        for (int h = 1; h < ell; h <<= 1) {
          for (int q = tid; q < ell / 2; q += FT) {
            int j = ((q / h) * 2 * h) + (q % h);
            double x = X[j], y = X[j + h];
            X[j] = x + y;
            X[j + h] = x - y;
          }
          __syncthreads();
        }
        if (op == 0) {
          for (int c = tid; c < ell; c += FT) FA[c] = X[c];
        } else {
          for (int c = tid; c < ell; c += FT) ACC[c] = fma(FA[c], X[c], ACC[c]);
        }
        __syncthreads();
      }
    }
    double *dst = p.partial + ((int64_t)g * p.maxseg + seg) * ell;
    for (int c = tid; c < ell; c += FT) dst[c] = ACC[c];
    __syncthreads();
    ++seg;
    w0 += kend - kk;
  }
}

// Sum the CTA partial slices of every item in CTA order -> acc[t][a*l + c].
__global__ void reduce_partials_kernel(const double *partial, double *acc, int64_t W, int G, int maxseg,
                                       int64_t K, int F, int L, int64_t nitems) {
  const int64_t ell = (int64_t)1 << L;
  const int64_t total = nitems * ell;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = x / ell, c = x % ell;
    double s = 0.0;
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
        s += partial[((int64_t)g * maxseg + segi) * ell + c];
      }
    }
    const int64_t t = item / F, a = item % F;
    acc[(t * F + a) * ell + c] = s;
  }
}

// ---------------------------------------------------------------- host side
static int fold_L(int log2b) { return log2b < 13 ? log2b : 13; }

int64_t fwht_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int G) {
  const int L = fold_L(log2b);
  const int64_t F = (int64_t)1 << (log2b - L);
  const int64_t W = (int64_t)d * F * K;
  const int64_t per = W > 0 ? ceil_div(W, G) : 1;
  const int64_t maxseg = K > 0 ? ceil_div(per, K) + 1 : 1;
  const int64_t plans = plan_total_bytes(d, 2, n1, n2, L);
  return ((plans + 255) / 256) * 256 + (int64_t)G * maxseg * ((int64_t)1 << L) * 8;
}

int fwht_accumulate(const SketchHashes &h, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm,
                    int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc, char *ws, int64_t ws_bytes,
                    cudaStream_t s) {
  const int log2b = h.log2b;
  const int L = fold_L(log2b);
  const int F = 1 << (log2b - L);
  const int64_t K = k1 - k0;
  const int d = h.d;
  const int64_t nitems = (int64_t)d * F;
  const int64_t W = nitems * K;
  int G = num_sms();
  if (W > 0 && W < G) G = (int)W;
  if (W == 0) G = 1;
  const int64_t need = fwht_workspace(d, log2b, n1, n2, K, num_sms());
  if (ws_bytes < need) {
    set_error("compress workspace too small: %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    return SMM_ERR_WORKSPACE;
  }
  FwhtArgs p;
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
  p.L = L;
  p.F = F;
  p.G = G;
  const int64_t per = W > 0 ? ceil_div(W, G) : 1;
  p.maxseg = (int)(K > 0 ? ceil_div(per, K) + 1 : 1);
  p.plans = ws;
  p.plan_nin_max = n1 > n2 ? n1 : n2;
  p.plan_per = plan_bytes_per(p.plan_nin_max, L);
  const int64_t plans = plan_total_bytes(d, 2, n1, n2, L);
  p.partial = (double *)(ws + ((plans + 255) / 256) * 256);
  if (W > 0) {
    int rc = build_plans(h, 2, n1, n2, L, ws, s);
    if (rc) return rc;
    const int64_t ell = (int64_t)1 << L;
    if (L == 13) {
      size_t smem = 3 * ell * sizeof(double);
      SMM_CUDA_TRY(cudaFuncSetAttribute(fwht_fold_kernel<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "fwht_fold_kernel<13> smem");
      fwht_fold_kernel<13><<<G, FT, smem, s>>>(p);
      SMM_LAUNCH_CHECK("fwht_fold_kernel<13>");
    } else if (L == 12) {
      size_t smem = 3 * ell * sizeof(double);
      SMM_CUDA_TRY(cudaFuncSetAttribute(fwht_fold_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "fwht_fold_kernel<12> smem");
      fwht_fold_kernel<12><<<G, FT, smem, s>>>(p);
      SMM_LAUNCH_CHECK("fwht_fold_kernel<12>");
    } else {
      size_t smem = 3 * ell * sizeof(double);
      SMM_CUDA_TRY(cudaFuncSetAttribute(fwht_fold_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "fwht_fold_small_kernel smem");
      fwht_fold_small_kernel<<<G, FT, smem, s>>>(p);
      SMM_LAUNCH_CHECK("fwht_fold_small_kernel");
    }
  }
  const int64_t total = nitems * ((int64_t)1 << L);
  int64_t blocks = ceil_div(total, 256);
  if (blocks > 8192) blocks = 8192;
  if (blocks < 1) blocks = 1;
  reduce_partials_kernel<<<(unsigned)blocks, 256, 0, s>>>(p.partial, acc, W, G, p.maxseg, K, F, L, nitems);
  SMM_LAUNCH_CHECK("reduce_partials_kernel");
  return SMM_OK;
}

}  // namespace smm
