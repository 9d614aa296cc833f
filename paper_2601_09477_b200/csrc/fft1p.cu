// FFT compress (steps 1-3, cyclic-convolution variant) for b = 2^12 with small operands
// (n1 + n2 <= 16384): one pass, one inner index at a time per CTA, everything on chip —
// the FFT counterpart of fwht1p.cu.  Reference: sketch.py:192-235 (`_compress_fft_kernel`),
// transforms.py:52-97.
//
// Per (repetition t, inner index k) the reference packs z = pa + i*pb (A's signed column
// into the real part, B's signed row into the imaginary part), runs one complex b-point
// FFT and accumulates FA(u)*FB(u) for u in [0, b/2], with
//     FA = (Z[u] + conj Z[-u]) / 2,   FB = -i/2 (Z[u] - conj Z[-u]).
// Why a one-pass kernel: at b = 2^12 the two-pass fft2p has 32 pass-1 and 17 pass-2 items
// per unit, and every unit's pass 2 waits for all of its pass 1 (cfg5 b = 2^12 d = 5:
// 2.86 ms of kernel time at 18 % of the FP64 pipe).  Here one CTA of 512 threads per SM
// owns a share of the inner-dimension tiles and keeps one inner index on chip:
//   * A's column k and B's row k are staged in shared memory with cp.async (n1 + n2
//     doubles, <= 128 KB); the signed scatter reads them through a warp-interleaved CSR
//     (one coalesced word load per warp step, as fwht1p), into the thread's own 8 slots
//     of the exchange area (real part from A's entries, imaginary part from B's);
//   * the 4096-point FFT is decimation in frequency, radix 8 in four stages: thread n
//     holds the 8 elements b*L + j + (L/8)*r of one radix-8 butterfly per stage, the
//     8-point DFT runs in registers, the twiddles w_L^(j r') are powers of one table
//     value (two 64-entry shared tables), and the stages exchange through a padded
//     shared-memory array (index p + p/8: every access pattern is conflict-free);
//   * after the last stage thread n holds Z at positions 8n + r', i.e. frequencies
//     u = 512 r' + rev3(n) (digit reversal): r' < 4 are exactly the half spectrum
//     u < 2048 (u = 2048 is thread 0's r' = 4), so every thread accumulates 4 products,
//     reading the partner Z[-u] from shared memory; the d accumulators of the tile live
//     in TMEM (d <= 7 per launch; deeper sketches in balanced groups, one launch each).
//     (Accumulating Z^2 instead — FA FB = -i/4 (Z[u]^2 - conj Z[-u]^2) — needs no partner
//     read per (k, t), but 8 instead of 4 complex per thread in TMEM, i.e. launches of at
//     most 4 repetitions: measured slower at d = 5 and 9, 3.31 / 5.47 vs 3.02 / 5.22 ms);
//   * the columns of k + 1 are copied while the last repetition of k is transformed.
// The accumulator of every W-wide tile of inner indices (W | 32, relative to the call's
// k0) goes to a partial buffer that fft1p_reduce_kernel adds in k order, so results are
// deterministic and the host-streamed path (k-slabs on multiples of 32) reproduces one
// call's bits.  Against the reference's arithmetic order the results agree to rounding
// (the FFT variant's parity is the north star's 1e-10 * ||C||_F tolerance).
#include "plan.cuh"
#include "twopass.cuh"

namespace smm {

__global__ void csr_scan_kernel(const int32_t *cnt, int32_t *off, int64_t b);  // fwht2p.cu

namespace f1f {
using namespace tp;

constexpr int LB = 12;
constexpr int B = 1 << LB;
constexpr int HALF = B / 2;                 // u = 0 .. HALF (HALF + 1 accumulated frequencies)
constexpr int CT = 512;                     // threads: one radix-8 butterfly each per stage
constexpr int WARPS = CT / 32;
constexpr int MAXD = 7;                     // TMEM: 64 columns per repetition
constexpr int64_t MAX_COLS = 16384;         // n1 + n2 staged in shared memory
constexpr int ZS = B + B / 8;               // padded complex slots of the exchange area
// scatter word: byte offset of the input in its staged column (bits 0-16), slot r of the
// thread's 8 (bits 17-19), first / last entry of its bucket (bits 21 / 22), sign (bit 31)
constexpr uint32_t W_OFF = 0x1ffffu, W_FIRST = 1u << 21, W_LAST = 1u << 22, W_SIGN = 1u << 31;

// bucket m -> CSR key: thread n = m mod 512 owns keys 8n .. 8n + 7 (slot r = m / 512)
__device__ __forceinline__ uint32_t key_of(uint32_t m) { return ((m & 511u) << 3) | (m >> 9); }
__device__ __forceinline__ int zidx(int p) { return p + (p >> 3); }
// base-8 digit reversal of a 4-digit (12-bit) index
__device__ __forceinline__ int rev8x4(int p) {
  return ((p & 7) << 9) | (((p >> 3) & 7) << 6) | (((p >> 6) & 7) << 3) | (p >> 9);
}

struct Tab {
  int32_t base, maxcnt;
};

struct Args {
  const double *X[2];  // element (input i, inner index k) of operand op at X[op][k * ks[op] + i * is[op]]
  int64_t ks[2], is[2];
  int n[2];
  int64_t K;
  int d, W, ntiles;
  const uint32_t *ent2;  // [d][2][...] at row offsets roff[t * 2 + op]
  int64_t roff[2 * MAXD];
  const Tab *tab;        // [d][2][WARPS]
  const uint32_t *bmask;  // [d][2][CT]: slots of each thread's 8 that have an entry
  cplx *part;            // [ntiles][d][HALF + 1]
  int vec16;             // per operand: 16-byte async copies allowed
  int bulk;              // both columns are staged with TMA bulk copies (contiguous, 16-byte aligned)
};

__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx mul_mi(cplx a) { return {a.im, -a.re}; }  // * (-i)

// in-register forward 8-point DFT, natural order in and out: y[k] = sum_r x[r] w_8^(r k)
__device__ __forceinline__ void dft8(cplx (&x)[8]) {
  constexpr double R = 0.70710678118654752440;  // 1 / sqrt(2)
  // span 4: x[r] +- x[r + 4], the difference times w_8^r
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const cplx a = x[r], b = x[r + 4];
    x[r] = cadd(a, b);
    x[r + 4] = csub(a, b);
  }
  {
    const cplx t1 = x[5];
    x[5] = {R * (t1.re + t1.im), R * (t1.im - t1.re)};  // * (1 - i) / sqrt 2
    x[6] = mul_mi(x[6]);                                 // * -i
    const cplx t3 = x[7];
    x[7] = {R * (t3.im - t3.re), -R * (t3.re + t3.im)};  // * (-1 - i) / sqrt 2
  }
  // span 2 within each half: the difference times w_4^r
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const cplx a = x[h + r], b = x[h + r + 2];
      x[h + r] = cadd(a, b);
      x[h + r + 2] = r ? mul_mi(csub(a, b)) : csub(a, b);
    }
  }
  // span 1
#pragma unroll
  for (int q = 0; q < 8; q += 2) {
    const cplx a = x[q], b = x[q + 1];
    x[q] = cadd(a, b);
    x[q + 1] = csub(a, b);
  }
  // bit-reversed -> natural order: y[k] = x[brev3(k)]
  cplx t = x[1];
  x[1] = x[4];
  x[4] = t;
  t = x[3];
  x[3] = x[6];
  x[6] = t;
}

__device__ __forceinline__ void column_copy(const Args &p, int op, int64_t k, double *col) {
  const double *src = p.X[op] + k * p.ks[op];
  const int n = p.n[op];
  if (p.is[op] != 1) {
    const int64_t st = p.is[op];
    for (int i = threadIdx.x; i < n; i += CT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + i * st) : "memory");
    }
  } else if (p.vec16 & (1 << op)) {
    for (int i = 2 * threadIdx.x; i < n; i += 2 * CT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + i) : "memory");
    }
  } else {
    for (int i = threadIdx.x; i < n; i += CT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + i) : "memory");
    }
  }
}

__global__ void __launch_bounds__(CT, 1) fft1p_kernel(Args p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint32_t s_tmem;
  __shared__ cplx s_t0[64], s_t1[64];  // w_4096^e = s_t1[e >> 6] * s_t0[e & 63]
  __shared__ cplx s_acc_half[MAXD];    // the tile's u = 2048 accumulators (thread 0)
  __shared__ __align__(8) uint64_t s_colbar;  // bulk column copies landed
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  cplx *Z = (cplx *)sm;                                     // exchange area, ZS padded slots
  double *zd = sm;                                          // the same, as doubles
  double *colA = sm + 2 * ZS;                               // staged columns, each followed by a zero
  double *colB = colA + ((p.n[0] + 2) & ~1);
  if (tid == 0) {
    colA[p.n[0]] = 0.0;
    mbar_init(&s_colbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 1) colB[p.n[1]] = 0.0;
  uint32_t colpar = 0;  // phase parity of the next bulk copy pair
  // the inner index k's columns: one elected thread issues both bulk copies, or every thread
  // its cp.async share
  auto stage = [&](int64_t kk) {
    if (p.bulk) {
      if (tid == 0)
        bulk_copy2_g2s(colA, p.X[0] + kk * p.ks[0], (uint32_t)p.n[0] * 8u, colB, p.X[1] + kk * p.ks[1],
                       (uint32_t)p.n[1] * 8u, &s_colbar);
    } else {
      column_copy(p, 0, kk, colA);
      column_copy(p, 1, kk, colB);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  const uint32_t col_s[2] = {(uint32_t)__cvta_generic_to_shared(colA), (uint32_t)__cvta_generic_to_shared(colB)};
  if (tid < 64) {
    double sn, cs;
    sincospi(-2.0 * (double)tid / (double)B, &sn, &cs);
    s_t0[tid] = {cs, sn};
    sincospi(-2.0 * (double)(tid * 64) / (double)B, &sn, &cs);
    s_t1[tid] = {cs, sn};
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  auto col_acc = [&](int t) { return (uint32_t)(t * 64 + (warp >> 2) * 16); };  // 4 complex of repetition t
  const int d = p.d;
  // w_4096^(e * r') for r' = 1..7 as powers of w = w_4096^e (e < 4096)
  auto twiddles = [&](int e, cplx (&w)[8]) {
    const cplx a = s_t1[e >> 6], b0 = s_t0[e & 63];
    w[1] = cmul(a, b0);
#pragma unroll
    for (int r = 2; r < 8; ++r) w[r] = cmul(w[r - 1], w[1]);
  };
  // rev3(n): base-8 digit reversal of n < 512; position 8n + r' holds frequency 512 r' + rev3(n)
  const int rev_n = ((tid & 7) << 6) | (((tid >> 3) & 7) << 3) | (tid >> 6);
  // the thread's slot r of the exchange area: zidx(tid + 512 r) = zidx(tid) + 576 r
  const int zb = 2 * zidx(tid);
  int64_t tile = blockIdx.x;
  if (tile < p.ntiles) stage(tile * p.W);  // (the barrier above ordered the mbarrier's initialisation)
  for (; tile < p.ntiles; tile += gridDim.x) {
    const int64_t k_lo = tile * p.W;
    const int64_t k_hi = k_lo + p.W < p.K ? k_lo + p.W : p.K;
    for (int64_t k = k_lo; k < k_hi; ++k) {
      if (p.bulk) {
        mbar_wait(&s_colbar, colpar);
        colpar ^= 1u;
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();  // the columns are visible; the exchange area is free
      for (int t = 0; t < d; ++t) {
        // ---- signed scatter: real part from A's entries, imaginary part from B's, into this
        // thread's slots n + 512 r (entries in bucket order, increasing input index inside a
        // bucket, the reference's order; a bucket's sum starts from 0.0)
        uint32_t mask[2];
#pragma unroll
        for (int op = 0; op < 2; ++op) {
          const Tab tb = p.tab[(t * 2 + op) * WARPS + warp];
          const uint32_t *e2 = p.ent2 + p.roff[t * 2 + op] + tb.base + lane;
          mask[op] = __ldg(p.bmask + (t * 2 + op) * CT + tid);
          const uint32_t pad = (uint32_t)p.n[op] * 8u;
          double run = 0.0;
          uint32_t wn[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) wn[r] = r < tb.maxcnt ? __ldg(e2 + r * 32) : pad;
          for (int q0 = 0; q0 < tb.maxcnt; q0 += 8) {
            uint32_t w[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              w[r] = wn[r];
              wn[r] = q0 + 8 + r < tb.maxcnt ? __ldg(e2 + (q0 + 8 + r) * 32) : pad;
            }
            double x[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              double y;
              asm volatile("ld.shared.f64 %0, [%1];" : "=d"(y) : "r"(col_s[op] + (w[r] & W_OFF)));
              x[r] = __hiloint2double(__double2hiint(y) ^ (int)(w[r] & W_SIGN), __double2loint(y));
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              run = ((w[r] & W_FIRST) ? 0.0 : run) + x[r];
              if (w[r] & W_LAST) zd[zb + op + 1152 * (int)((w[r] >> 17) & 7u)] = run;
            }
          }
        }
        cplx v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int zi = zb + 1152 * r;
          v[r].re = ((mask[0] >> r) & 1u) ? zd[zi] : 0.0;
          v[r].im = ((mask[1] >> r) & 1u) ? zd[zi + 1] : 0.0;
        }
        if (t == d - 1) {
          // every read of column k is done: copy the next inner index's columns meanwhile
          __syncthreads();
          int64_t kn = k + 1;
          if (kn >= k_hi) {
            const int64_t tn = tile + gridDim.x;
            kn = tn < p.ntiles ? tn * p.W : -1;
          }
          if (kn >= 0) stage(kn);
        }
        // ---- 4096-point DFT: decimation in frequency, radix 8, four stages in place
        cplx w[8];
        // stage 0: L = 4096, j = n, elements n + 512 r
        dft8(v);
        twiddles(tid, w);
#pragma unroll
        for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], w[r]);
#pragma unroll
        for (int r = 0; r < 8; ++r) Z[zidx(tid + 512 * r)] = v[r];
        __syncthreads();
        // stage 1: L = 512, block tid >> 6, j = tid & 63, elements b*512 + j + 64 r
        {
          const int base = (tid >> 6) * 512 + (tid & 63);
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = Z[zidx(base + 64 * r)];
          dft8(v);
          twiddles(8 * (tid & 63), w);
#pragma unroll
          for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], w[r]);
#pragma unroll
          for (int r = 0; r < 8; ++r) Z[zidx(base + 64 * r)] = v[r];
        }
        __syncthreads();
        // stage 2: L = 64, block tid >> 3, j = tid & 7, elements b*64 + j + 8 r
        {
          const int base = (tid >> 3) * 64 + (tid & 7);
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = Z[zidx(base + 8 * r)];
          dft8(v);
          twiddles(64 * (tid & 7), w);
#pragma unroll
          for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], w[r]);
#pragma unroll
          for (int r = 0; r < 8; ++r) Z[zidx(base + 8 * r)] = v[r];
        }
        __syncthreads();
        // stage 3: L = 8, elements 8n + r; position 8n + r' holds Z[512 r' + rev3(n)]
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = Z[zidx(8 * tid + r)];
        dft8(v);
#pragma unroll
        for (int r = 0; r < 8; ++r) Z[zidx(8 * tid + r)] = v[r];
        __syncthreads();
        // ---- FA * FB for u = 512 r' + rev3(n), r' < 4 (and u = 2048 on thread 0)
        double pr[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int u = 512 * r + rev_n;
          const cplx zm = Z[zidx(rev8x4((B - u) & (B - 1)))];
          const cplx zu = v[r];
          const cplx sum = {zu.re + zm.re, zu.im - zm.im};  // Z[u] + conj Z[-u]
          const cplx dif = {zu.re - zm.re, zu.im + zm.im};  // Z[u] - conj Z[-u]
          const cplx fa = {0.5 * sum.re, 0.5 * sum.im};
          const cplx fb = {0.5 * dif.im, -0.5 * dif.re};
          const cplx q = cmul(fa, fb);
          pr[2 * r] = q.re;
          pr[2 * r + 1] = q.im;
        }
        if (tid == 0) {  // u = 2048 = -2048: its own partner (position 4)
          const cplx zu = v[4];
          const cplx fa = {zu.re, 0.0};  // (Z + conj Z) / 2
          const cplx fb = {zu.im, 0.0};  // -i/2 (Z - conj Z)
          const cplx q = cmul(fa, fb);
          s_acc_half[t] = k > k_lo ? cadd(s_acc_half[t], q) : q;
        }
        if (k > k_lo) {
          double acc[8];
          tmem_ld8(tq + col_acc(t), acc);
#pragma unroll
          for (int j = 0; j < 8; ++j) pr[j] = __dadd_rn(acc[j], pr[j]);
        }
        tmem_st8(tq + col_acc(t), pr);
        tmem_wait_st();
        __syncthreads();  // partner reads done: the exchange area is reused by the next scatter
      }
    }
    // ---- the tile's sums to the partial buffer
    for (int t = 0; t < d; ++t) {
      double acc[8];
      tmem_ld8(tq + col_acc(t), acc);
      cplx *dst = p.part + ((int64_t)tile * d + t) * (HALF + 1);
#pragma unroll
      for (int r = 0; r < 4; ++r) dst[512 * r + rev_n] = {acc[2 * r], acc[2 * r + 1]};
      if (tid == 0) dst[HALF] = s_acc_half[t];
    }
    __syncthreads();  // s_acc_half is rewritten by the next tile
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// acc[t][u] = ((acc_in + T0) + T1) + ... over the tiles in k order (acc_add), or from T0
__global__ void fft1p_reduce_kernel(const cplx *part, int ntiles, int d, cplx *acc, int acc_add) {
  const int64_t per = HALF + 1;
  const int64_t total = (int64_t)d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const cplx *pt = part + x;
    const int64_t stride = total;
    cplx s = acc_add ? cadd(acc[x], pt[0]) : pt[0];
    for (int q0 = 1; q0 < ntiles; q0 += 16) {
      cplx v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (q0 + r < ntiles) {
          const double2 y = __ldcg((const double2 *)(pt + (int64_t)(q0 + r) * stride));
          v[r] = {y.x, y.y};
        } else {
          v[r] = {0.0, 0.0};
        }
      }
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (q0 + r < ntiles) s = cadd(s, v[r]);
    }
    acc[x] = s;
  }
}

// CSR by key (per (t, op): off[B + 1], ent = i | slot << 26 | sign << 31), as fwht2p.cu's
// plan kernels with the bucket replaced by its key
__global__ void csr_count_key(SketchHashes h, int64_t n1, int64_t n2, int32_t *cnt) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const uint32_t m = eval_bucket(h.f[op][t], (uint64_t)i, LB);
    atomicAdd(&cnt[((int64_t)t * 2 + op) * B + key_of(m)], 1);
  }
}

__global__ void csr_fill_key(SketchHashes h, int64_t n1, int64_t n2, const int32_t *off, int32_t *fill, uint32_t *ent,
                             int64_t nmax) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const int64_t row = (int64_t)t * 2 + op;
    const uint32_t key = key_of(eval_bucket(h.f[op][t], (uint64_t)i, LB));
    const uint32_t sb = eval_signbit(h.f[2 + op][t], (uint64_t)i);
    const int32_t pos = off[row * (B + 1) + key] + atomicAdd(&fill[row * B + key], 1);
    ent[row * nmax + pos] = (uint32_t)i | ((key & 7u) << 26) | (sb << 31);
  }
}

struct RowOffsets {
  int64_t r[2 * MAXD];
};

// warp-interleaved scatter words of one (t, op) row per block (CT threads, 8 keys each)
__global__ void csr_interleave_key(const int32_t *off, const uint32_t *ent, int64_t nmax, uint32_t *ent2,
                                   RowOffsets roff, Tab *tab, uint32_t *bmask, int n0, int n1) {
  __shared__ int s_max[WARPS];
  const int row = blockIdx.x;
  const int nop = (row & 1) ? n1 : n0;
  const int n = threadIdx.x, w = n >> 5, lane = n & 31;
  const int32_t *o = off + (int64_t)row * (B + 1);
  const int lo = o[8 * n], hi = o[8 * n + 8];
  const int cnt = hi - lo;
  const int mx = __reduce_max_sync(0xffffffffu, cnt);
  if (lane == 0) s_max[w] = mx;
  __syncthreads();
  int base = 0;
  for (int x = 0; x < w; ++x) base += 32 * s_max[x];
  if (lane == 0) tab[row * WARPS + w] = Tab{base, mx};
  uint32_t *dst = ent2 + roff.r[row] + base + lane;
  const uint32_t *src = ent + (int64_t)row * nmax + lo;
  uint32_t mask = 0;
  for (int q = 0; q < mx; ++q) {
    uint32_t wd = (uint32_t)nop * 8u;  // padding: the zero double past the column
    if (q < cnt) {
      const uint32_t e = src[q];
      const uint32_t r = (e >> 26) & 7u;
      const bool first = q == 0 || ((src[q - 1] >> 26) & 7u) != r;
      const bool last = q == cnt - 1 || ((src[q + 1] >> 26) & 7u) != r;
      wd = ((e & 0x03ffffffu) * 8u) | (r << 17) | (first ? W_FIRST : 0u) | (last ? W_LAST : 0u) | (e & W_SIGN);
      mask |= 1u << r;
    }
    dst[q * 32] = wd;
  }
  bmask[row * CT + n] = mask;
}

static int64_t ent2_row_bound(int64_t nop) { return 32 * (nop > 0 ? nop : 1); }

}  // namespace f1f

static inline int64_t pad256f(int64_t x) { return ((x + 255) / 256) * 256; }

static int f1f_tile_width(int d, int64_t K) {
  // W | 32: the finest that keeps the partial buffer under 512 MB (load balance over the SMs)
  for (int W : {8, 16, 32}) {
    const int64_t nt = (K + W - 1) / W;
    if (nt * d * (f1f::HALF + 1) * 16 <= ((int64_t)512 << 20)) return W;
  }
  return 0;
}

// repetitions per launch: up to MAXD (the TMEM accumulators), deeper sketches in balanced groups
static int f1f_group(int d) {
  if (d <= f1f::MAXD) return d;
  const int ng = (d + f1f::MAXD - 1) / f1f::MAXD;
  return (d + ng - 1) / ng;
}

bool fft1p_supported(int log2b, int d, int64_t n1, int64_t n2, int64_t K) {
  static const bool off = getenv("SMM_NO_FFT1P") != nullptr;
  return !off && log2b == f1f::LB && d >= 1 && d <= SMM_MAX_DEPTH && n1 + n2 <= f1f::MAX_COLS &&
         n1 < f1f::MAX_COLS && n2 < f1f::MAX_COLS && (K == 0 || f1f_tile_width(f1f_group(d), K) > 0);
}

int64_t fft1p_workspace(int d, int64_t n1, int64_t n2, int64_t K) {
  using namespace f1f;
  d = f1f_group(d);  // one group's workspace, reused by the next group
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int W = f1f_tile_width(d, K > 0 ? K : 1);
  const int64_t nt = (K + (W ? W : 32) - 1) / (W ? W : 32);
  int64_t w = 0;
  w += pad256f((int64_t)d * 2 * (B + 1) * 4);  // off
  w += pad256f((int64_t)d * 2 * B * 4);        // cnt / fill
  w += pad256f((int64_t)d * 2 * nmax * 4);     // ent
  w += pad256f((int64_t)d * (ent2_row_bound(n1) + ent2_row_bound(n2)) * 4);  // ent2
  w += pad256f((int64_t)d * 2 * WARPS * sizeof(Tab));
  w += pad256f((int64_t)d * 2 * CT * 4);       // slot masks
  w += pad256f(nt * d * (HALF + 1) * 16);      // partial tile sums
  return w;
}

// k-major operand rows (A^T and B); inner range [k0, k1); acc: d x (b/2 + 1) complex
int fft1p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb, int64_t n1,
                     int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws, int64_t ws_bytes,
                     cudaStream_t s) {
  using namespace f1f;
  if (h.d > MAXD) {
    // repetition groups, one launch each, into rows [t0, t0 + dg) of acc (workspace reused)
    const int dg = f1f_group(h.d);
    for (int t0 = 0; t0 < h.d; t0 += dg) {
      SketchHashes hg;
      hg.d = t0 + dg <= h.d ? dg : h.d - t0;
      hg.log2b = h.log2b;
      for (int g = 0; g < 4; ++g)
        for (int t = 0; t < hg.d; ++t) hg.f[g][t] = h.f[g][t0 + t];
      const int rc = fft1p_accumulate(hg, xa, lda, xb, ldb, n1, n2, k0, k1, acc + (int64_t)t0 * (HALF + 1) * 2,
                                      acc_add, ws, ws_bytes, s);
      if (rc) return rc;
    }
    return SMM_OK;
  }
  const int d = h.d;
  const int64_t K = k1 - k0;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  if (ws_bytes < fft1p_workspace(d, n1, n2, K)) {
    set_error("compress workspace too small (one-pass fft)");
    return SMM_ERR_WORKSPACE;
  }
  if (K <= 0) {
    if (!acc_add) SMM_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)d * (HALF + 1) * 16, s), "acc memset");
    return SMM_OK;
  }
  const int W = f1f_tile_width(d, K);
  const int64_t nt = (K + W - 1) / W;
  char *q = ws;
  int32_t *off = (int32_t *)q;
  q += pad256f((int64_t)d * 2 * (B + 1) * 4);
  int32_t *cnt = (int32_t *)q;
  q += pad256f((int64_t)d * 2 * B * 4);
  uint32_t *ent = (uint32_t *)q;
  q += pad256f((int64_t)d * 2 * nmax * 4);
  uint32_t *ent2 = (uint32_t *)q;
  q += pad256f((int64_t)d * (ent2_row_bound(n1) + ent2_row_bound(n2)) * 4);
  Tab *tab = (Tab *)q;
  q += pad256f((int64_t)d * 2 * WARPS * sizeof(Tab));
  uint32_t *bmask = (uint32_t *)q;
  q += pad256f((int64_t)d * 2 * CT * 4);
  cplx *part = (cplx *)q;
  // CSR by key, deterministic order inside a key (increasing input index), interleaved copy
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * B * 4, s), "csr memset");
  const int64_t nin = (int64_t)d * (n1 + n2);
  int64_t blocks = ceil_div(nin, 256);
  if (blocks > 8192) blocks = 8192;
  if (nin > 0) {
    csr_count_key<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, cnt);
    SMM_LAUNCH_CHECK("csr_count_key");
  }
  csr_scan_kernel<<<d * 2, 1024, 0, s>>>(cnt, off, B);
  SMM_LAUNCH_CHECK("csr_scan_kernel");
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * B * 4, s), "csr memset");
  if (nin > 0) {
    csr_fill_key<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, off, cnt, ent, nmax);
    SMM_LAUNCH_CHECK("csr_fill_key");
    const int rc = csr_sort(off, ent, nmax, B, d * 2, s);
    if (rc) return rc;
  }
  RowOffsets ro;
  {
    int64_t pos = 0;
    for (int r = 0; r < 2 * d; ++r) {
      ro.r[r] = pos;
      pos += ent2_row_bound((r & 1) ? n2 : n1);
    }
  }
  csr_interleave_key<<<2 * d, CT, 0, s>>>(off, ent, nmax, ent2, ro, tab, bmask, (int)n1, (int)n2);
  SMM_LAUNCH_CHECK("csr_interleave_key");
  Args p;
  p.ks[0] = lda;
  p.is[0] = 1;
  p.ks[1] = ldb;
  p.is[1] = 1;
  p.X[0] = xa + k0 * lda;
  p.X[1] = xb + k0 * ldb;
  p.n[0] = (int)n1;
  p.n[1] = (int)n2;
  p.K = K;
  p.d = d;
  p.W = W;
  p.ntiles = (int)nt;
  p.ent2 = ent2;
  for (int r = 0; r < 2 * MAXD; ++r) p.roff[r] = r < 2 * d ? ro.r[r] : 0;
  p.tab = tab;
  p.bmask = bmask;
  p.part = part;
  p.vec16 = 0;
  if (p.ks[0] % 2 == 0 && n1 % 2 == 0 && (uintptr_t)p.X[0] % 16 == 0) p.vec16 |= 1;
  if (p.ks[1] % 2 == 0 && n2 % 2 == 0 && (uintptr_t)p.X[1] % 16 == 0) p.vec16 |= 2;
  static const bool no_bulk = getenv("SMM_NO_BULK_COLUMNS") != nullptr;
  p.bulk = (!no_bulk && p.vec16 == 3) ? 1 : 0;
  const size_t smem = (size_t)(2 * ZS + ((n1 + 2) & ~1) + n2 + 1) * 8;
  SMM_CUDA_TRY(cudaFuncSetAttribute(fft1p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "fft1p smem");
  int grid = num_sms();
  if (grid > nt) grid = (int)nt;
  {
    KernelTimer timer(0, s);
    fft1p_kernel<<<grid, CT, smem, s>>>(p);
    timer.stop();
  }
  SMM_LAUNCH_CHECK("fft1p_kernel");
  fft1p_reduce_kernel<<<(unsigned)ceil_div((int64_t)d * (HALF + 1), 64), 64, 0, s>>>(part, (int)nt, d, (cplx *)acc,
                                                                                      acc_add ? 1 : 0);
  SMM_LAUNCH_CHECK("fft1p_reduce_kernel");
  return SMM_OK;
}

}  // namespace smm
