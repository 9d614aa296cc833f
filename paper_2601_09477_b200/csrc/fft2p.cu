// FFT compress (steps 1-3, cyclic-convolution variant) for 2^8 <= b <= 2^14:
// two-pass, persistent, dependency-ordered — the FFT counterpart of fwht2p.cu.
// Reference: sketch.py:192-235 (`_compress_fft_kernel`), transforms.py:52-97.
//
// Per (repetition t, inner index k) the reference packs z = pa + i*pb, runs one
// complex b-point FFT and accumulates FA(u)*FB(u), u in [0, b/2], with
//   FA = (Z[u] + conj Z[-u]) / 2,   FB = -i/2 (Z[u] - conj Z[-u]).
// Here the FFT is a four-step split b = 128 * N2 (m = m1 + 128 m2, u = u2 + N2 u1):
//   pass 1 (gather item: 128 positions = 2^(7-S1) values of m1 x all m2):
//     T[m1][u2] = w_b^(m1 u2) * DFT_N2 over m2 of z[m1 + 128 m2]     (S1 = log2 N2)
//   pass 2 (slice item: one u2, or the pair {u2, N2-u2}):
//     Z[u2 + N2 u1] = DFT_128 over m1 of T[m1][u2]
// Both DFTs are radix-2 decimation in time with bit-reversed input, so the
// gather scatters entry m straight to its bit-reversed position (the CSR key)
// and every butterfly twiddle inside a pass depends only on the position inside
// the 128-point tile (a 64-entry constant table).  Lanes carry 32 consecutive
// inner indices k exactly as in fwht2p: each entry pulls one 256-byte row of the
// k-minor operand; 16 complex values per thread (4 bits in registers), one
// shared-memory exchange per pass (3 warp bits), T parked in L2 ((lag+2)-slot ring).
// Pass 2 transforms slice u2 (stashed in TMEM) and slice N2-u2 in the
// "complement" layout, where a thread's register holding Z[u] for slice u2 holds
// Z[-u] for the partner slice, so the FA/FB split is register-local; the two
// self-paired slices (u2 = 0, N2/2) exchange partners through shared memory.
// FA*FB is summed over the 32 lanes (k) in a fixed order and added to the
// d x (b/2+1) accumulator in k-tile order (flags), so runs are bit-reproducible.
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "plan.cuh"
#include "twopass.cuh"

namespace smm {

__global__ void csr_scan_kernel(const int32_t *cnt, int32_t *off, int64_t b);  // fwht2p.cu

namespace f2p {
using namespace tp;

constexpr int THREADS = 256;
constexpr int KT = 32;

__constant__ double2 c_w128[64];  // exp(-2 pi i j / 128), j < 64

// CSR key of bucket m: item * 128 + (m1 mod G) * N2 + rev_S1(m2)  (G = 128 / N2)
__device__ __forceinline__ uint32_t fft_key(uint32_t m, int S1) {
  const uint32_t m1 = m & 127u, m2 = m >> 7;
  const uint32_t r2 = __brev(m2) >> (32 - S1);
  const int gsh = 7 - S1;
  return ((m1 >> gsh) << 7) | ((m1 & ((1u << gsh) - 1u)) << S1) | r2;
}

// b here is the slice size 2^LBs: a bucket's key is its position within the slice
__global__ void csr_count_fft(SketchHashes h, int64_t n1, int64_t n2, int32_t *cnt, int64_t b, int S1) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const uint32_t key = fft_key(eval_bucket(h.f[op][t], (uint64_t)i, h.log2b) & (uint32_t)(b - 1), S1);
    atomicAdd(&cnt[((int64_t)t * 2 + op) * b + key], 1);
  }
}

__global__ void csr_fill_fft(SketchHashes h, int64_t n1, int64_t n2, const int32_t *off, int32_t *fill, uint32_t *ent,
                             int64_t nmax, int64_t b, int S1) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const int64_t row = (int64_t)t * 2 + op;
    const uint32_t key = fft_key(eval_bucket(h.f[op][t], (uint64_t)i, h.log2b) & (uint32_t)(b - 1), S1);
    const uint32_t sb = eval_signbit(h.f[2 + op][t], (uint64_t)i);
    const int32_t pos = off[row * (b + 1) + key] + atomicAdd(&fill[row * b + key], 1);
    // entry: i (26 bits) | register (4 bits) | sign (1 bit)
    ent[row * nmax + pos] = (uint32_t)i | ((key & 15u) << 26) | (sb << 31);
  }
}

__global__ void twiddle_b_kernel(double *tw, int log2b) {
  const int64_t b = (int64_t)1 << log2b;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < b; x += (int64_t)gridDim.x * blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)x / (double)b, &s, &c);  // exact argument: x / b is a dyadic rational
    tw[2 * x] = c;
    tw[2 * x + 1] = s;
  }
}

struct Args {
  SketchHashes h;
  const double *X[2];  // k-minor operands: element (i, k) at X[op][i * ld[op] + k]
  int64_t ld[2];
  int64_t k0, K;
  int B, N2, G1, G2, U, d, lag, nslot;  // P2(u) is dispensed lag groups after P1(u); nslot = lag + 2
  int F, NPU, halves;  // fold: F slices of 2^LBs frequencies; NPU slice-pair units per (k-tile, t)
  FastDiv div_dnpu, div_npu, div_slot, div_grp;
  const int32_t *off;
  const uint32_t *ent;
  int64_t nmax, bsz, bfull;  // bsz = slice size 2^LBs (CSR rows), bfull = b
  const double *twb;  // [b][2]: exp(-2 pi i x / b)
  double *Y;          // [nslot][halves][N2][128][KT][2]
  double *acc;        // [d][b/2 + 1][2]
  int *ctr;           // [0] ticket | done1[U] | done2[U] | acc_cnt[d * NPU * G2]
  int acc_add;
  int acc_slow;  // test knob (SMM_ACC_SLOWPATH): every P2 item takes the accumulator slow path
};

// CSR range of one warp's 16 tile positions of operand OP and its first 32 entry
// words (one per lane), fetched ahead of the pull
struct Head {
  int e_lo, e_hi;
  uint32_t win;
};

template <int OP>
__device__ __forceinline__ Head head(const Args &p, int t, int item) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)t * 2 + OP;
  const int32_t *off = p.off + row * (p.bsz + 1) + (int64_t)item * 128 + warp * 16;
  Head h;
  h.e_lo = __ldg(off);
  h.e_hi = __ldg(off + 16);
  h.win = h.e_lo + lane < h.e_hi ? __ldg(p.ent + row * p.nmax + h.e_lo + lane) : 0u;
  return h;
}

// signed gather of one operand into the real (op 0) or imaginary (op 1) parts of the
// warp's lane-private complex columns of the exchange area (S2[(16 w + j) * 32 + lane],
// j = tile position & 15) — a register target would need a jump per entry.  Entries
// are sorted by position: the first of a position stores, later ones add.  Returns the
// mask of positions written.
// fold character w_b^e of a gathered entry (e = a m mod b < 2^20): three shared tables,
// w_b^e = s_tf2[e >> 14] * s_tf1[(e >> 7) & 127] * s_tf0[e & 127], filled once per CTA (the
// global table's load sat on every batch's dependency chain: b = 2^20 d = 3 429 -> 366 ms; for
// pass 1's inter-pass twiddle, a warp-uniform broadcast load, the tables measured 2.5 % slower)
__shared__ double2 s_tf0[128], s_tf1[128], s_tf2[64];

__device__ __forceinline__ double2 fold_twiddle(uint32_t e) {
  const double2 a = s_tf2[e >> 14], b = s_tf1[(e >> 7) & 127u], c = s_tf0[e & 127u];
  const double2 ab = make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
  return make_double2(fma(ab.x, c.x, -ab.y * c.y), fma(ab.x, c.y, ab.y * c.x));
}

template <int OP, bool FOLD>
__device__ __forceinline__ void pull(const Args &p, int kappa, int t, const Head &hd, int a, double *S,
                                     uint32_t &mask) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)t * 2 + OP;
  const uint32_t *ent = p.ent + row * p.nmax;
  const int e_lo = hd.e_lo, e_hi = hd.e_hi;
  const int64_t kk = (int64_t)kappa * KT + lane;
  const char *Xb = (const char *)(p.X[OP] + p.k0 + (kk < p.K ? kk : p.K - 1));
  const uint32_t ldb = (uint32_t)(p.ld[OP] * 8);
  // fold (slice a): an entry of bucket m adds z * w_b^(a m) with z = x (A) or i x (B), so
  // both parts of its position; otherwise operand OP owns one part
  double *col = S + ((warp * 16) * 32 + lane) * 2 + (FOLD ? 0 : OP);
  const uint32_t bmask = (uint32_t)(p.bfull - 1);
  uint32_t win = hd.win;  // entry words [wbase, wbase + 32)
  int wbase = e_lo;
  for (int eb = e_lo; eb < e_hi; eb += 8) {
    if (eb - wbase == 32) {
      wbase = eb;
      win = eb + lane < e_hi ? __ldg(ent + eb + lane) : 0u;
    }
    uint32_t es[8];
    double x[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) es[s] = __shfl_sync(0xffffffffu, win, (eb - wbase) + s);
#pragma unroll
    for (int s = 0; s < 8; ++s)
      x[s] = eb + s < e_hi ? __ldg((const double *)(Xb + (uint64_t)(es[s] & 0x03ffffffu) * ldb)) : 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (eb + s < e_hi) {  // warp-uniform
        const int j = (int)((es[s] >> 26) & 15u);
        const double val = (es[s] >> 31) ? -x[s] : x[s];
        const bool have = (mask >> j) & 1u;
        if (FOLD) {
          const uint32_t m = eval_bucket(p.h.f[OP][t], (uint64_t)(es[s] & 0x03ffffffu), p.B);
          const double2 w = fold_twiddle(((uint32_t)a * m) & bmask);
          const double cr = OP ? -val * w.y : val * w.x;
          const double ci = OP ? val * w.x : val * w.y;
          col[j * 64] = (have ? col[j * 64] : 0.0) + cr;
          col[j * 64 + 1] = (have ? col[j * 64 + 1] : 0.0) + ci;
        } else {
          col[j * 64] = (have ? col[j * 64] : 0.0) + val;  // 0 + val == val, as a register sum
        }
        mask |= 1u << j;
      }
    }
  }
}

// x' = x + y w, y' = x - y w
__device__ __forceinline__ void bfly(double &xr, double &xi, double &yr, double &yi, double wr, double wi) {
  const double tr = fma(yr, wr, -yi * wi);
  const double ti = fma(yr, wi, yi * wr);
  const double ar = xr, ai = xi;
  xr = ar + tr;
  xi = ai + ti;
  yr = ar - tr;
  yi = ai - ti;
}
__device__ __forceinline__ void bfly1(double &xr, double &xi, double &yr, double &yi) {
  const double ar = xr, ai = xi;
  xr = ar + yr;
  xi = ai + yi;
  yr = ar - yr;
  yi = ai - yi;
}

// Radix-2 DIT stages s < NST (<= 4) over register bits (tile position L = (warp << 4) | r).
// CMP: the thread's registers hold actual position 127 - L ("complement" layout).
template <bool CMP, int NST>
__device__ __forceinline__ void reg_stages(double (&v)[32]) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < NST) {
      const int h = 1 << s;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (!(r & h)) {
          const int j = CMP ? (h - 1 - (r & (h - 1))) : (r & (h - 1));
          const int lo = CMP ? (r | h) : r, hi = CMP ? r : (r | h);  // lo: actual position bit s clear
          if (j == 0) {
            bfly1(v[2 * lo], v[2 * lo + 1], v[2 * hi], v[2 * hi + 1]);
          } else {
            const double2 w = c_w128[j << (6 - s)];
            bfly(v[2 * lo], v[2 * lo + 1], v[2 * hi], v[2 * hi + 1], w.x, w.y);
          }
        }
      }
    }
  }
}

// tile position of register r after the exchange: L bits 4-6 <- r bits 0-2, bit 3 <- r bit 3, bits 0-2 <- warp
__device__ __forceinline__ int post_pos(int warp, int r) { return ((r & 7) << 4) | (r & 8) | warp; }

// warp bits (L 4-6) <-> register bits 0-2 through shared memory (64 KB of complex values)
__device__ __forceinline__ void exchange(double (&v)[32], double *S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *S2 = (double2 *)S;
#pragma unroll
  for (int r = 0; r < 16; ++r) S2[((warp << 4) | r) * 32 + lane] = make_double2(v[2 * r], v[2 * r + 1]);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double2 q = S2[post_pos(warp, r) * 32 + lane];
    v[2 * r] = q.x;
    v[2 * r + 1] = q.y;
  }
}

// DIT stages 4 <= s < NST over register bits after the exchange
template <bool CMP, int NST>
__device__ __forceinline__ void post_stages(double (&v)[32]) {
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 4; s < 7; ++s) {
    if (s < NST) {
      const int bit = 1 << (s - 4), h = 1 << s;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (!(r & bit)) {
          const int jn = post_pos(warp, r) & (h - 1);
          const int j = CMP ? (h - 1 - jn) : jn;
          const int lo = CMP ? (r | bit) : r, hi = CMP ? r : (r | bit);
          const double2 w = c_w128[j << (6 - s)];
          bfly(v[2 * lo], v[2 * lo + 1], v[2 * hi], v[2 * hi + 1], w.x, w.y);
        }
      }
    }
  }
}

// Pass 1: gather both operands of tile `item`, DFT_N2 over m2, twiddle w_b^(m1 u2), park T in L2
// inter-pass twiddles w_b^e without a fold (b <= 2^14, so e < 2^14): w_b^e = s_tw_hi[e >> 7] *
// s_tw_lo[e & 127] from two shared tables filled once per CTA, instead of one global table load
// per value (cfg2 3.51 -> 3.40 ms; with a fold the same tables for the slice size measured 1 %
// slower, so the folded kernels keep the global table)
__shared__ double2 s_tw_lo[128], s_tw_hi[128];

template <int S1, bool FOLD>
__device__ __forceinline__ void p1_item(const Args &p, int kappa, int t, int pu, int slot, int idx, double *S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fold: tiles [0, 128) of slice pu, [128, 256) of its partner F - pu (none for the self-paired 0, F/2)
  int item = idx, half = 0, a = 0;
  if (FOLD) {
    half = idx >> 7;
    item = idx & 127;
    a = half ? (pu == 0 ? p.F / 2 : p.F - pu) : pu;  // unit 0 = the self-paired slices {0, F/2}
  }
  // both operands' CSR heads up front: operand 1's land while operand 0 pulls
  const Head h0 = head<0>(p, t, item);
  const Head h1 = head<1>(p, t, item);
  uint32_t m0 = 0, m1 = 0;
  pull<0, FOLD>(p, kappa, t, h0, a, S, m0);
  if (FOLD) {
    pull<1, true>(p, kappa, t, h1, a, S, m0);
    m1 = m0;
  } else {
    pull<1, false>(p, kappa, t, h1, a, S, m1);
  }
  double v[32];
  {
    const double *col = S + ((warp * 16) * 32 + lane) * 2;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[2 * j] = ((m0 >> j) & 1u) ? col[j * 64] : 0.0;
      v[2 * j + 1] = ((m1 >> j) & 1u) ? col[j * 64 + 1] : 0.0;
    }
  }
  if ((int64_t)kappa * KT + KT > p.K && (int64_t)kappa * KT + lane >= p.K) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.0;
  }
  reg_stages<false, (S1 < 4 ? S1 : 4)>(v);
  if (S1 > 4) {
    exchange(v, S);
    post_stages<false, S1>(v);
  }
  const uint64_t pol = policy_evict_last();
  constexpr int G = 128 >> S1;  // values of m1 per tile
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int L = S1 > 4 ? post_pos(warp, r) : ((warp << 4) | r);
    const int u2 = L & ((1 << S1) - 1);
    const int m1 = item * G + (L >> S1);
    // inter-pass twiddle of the slice's 2^LBs-point FFT: w_(b/F)^(m1 u2) = w_b^(F m1 u2)
    double2 w;
    if constexpr (FOLD) {
      w = __ldg((const double2 *)p.twb + (int64_t)m1 * u2 * p.F);
    } else {
      const int e = m1 * u2;
      const double2 hi = s_tw_hi[e >> 7], lo = s_tw_lo[e & 127];
      w = make_double2(fma(hi.x, lo.x, -hi.y * lo.y), fma(hi.x, lo.y, hi.y * lo.x));
    }
    const double re = fma(v[2 * r], w.x, -v[2 * r + 1] * w.y);
    const double im = fma(v[2 * r], w.y, v[2 * r + 1] * w.x);
    st2_hint(p.Y + (((((int64_t)slot * p.halves + half) * p.N2 + u2) * 128 + m1) * KT + lane) * 2, re, im, pol);
  }
}

// full 128-point DIT DFT of slice u2 (T[., u2] in L2) into registers; CMP = complement layout
template <bool CMP>
__device__ __forceinline__ void slice_dft(const Args &p, int slot, int half, int u2, double (&v)[32], double *S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  const double *Ys = p.Y + ((((int64_t)slot * p.halves + half) * p.N2 + u2) * 128) * KT * 2;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int pn = (warp << 4) | r;
    const int pa = CMP ? 127 - pn : pn;
    const int m1 = (int)(__brev((uint32_t)pa) >> 25);
    ld2_hint(Ys + ((int64_t)m1 * KT + lane) * 2, v[2 * r], v[2 * r + 1], pol);
  }
  reg_stages<CMP, 4>(v);
  exchange(v, S);  // its barrier also means every thread's loads of this slice completed
  {
    // last use of the slice's 64 KB: drop its L2 lines without write-back
    const char *base = (const char *)Ys;
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + (size_t)threadIdx.x * 256) : "memory");
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + (size_t)threadIdx.x * 256 + 128) : "memory");
  }
  post_stages<CMP, 7>(v);
  __syncthreads();  // shared memory is reused next
}

// FA * FB of Z[u] = (a, b) and Z[-u] = (c, e), in place of the second argument
__device__ __forceinline__ void split_product(double a, double b, double &c, double &e) {
  const double far = 0.5 * (a + c), fai = 0.5 * (b - e);   // FA = (Z[u] + conj Z[-u]) / 2
  const double fbr = 0.5 * (b + e), fbi = -0.5 * (a - c);  // FB = -i/2 (Z[u] - conj Z[-u])
  c = fma(far, fbr, -fai * fbi);
  e = fma(far, fbi, fai * fbr);
}

// Pass 2, item i2 of slice-pair unit pu (frequency u = a + F (u2 + N2 u1), u1 = tile position):
//   unit 0, i2 in [0, N2/2]: slice 0 (self-paired; the whole spectrum when F = 1) pairs rows
//     i2 and N2 - i2 (Z[-u] at row N2 - i2, position 127 - u1); rows 0 and N2/2 pair with
//     themselves (position -u1 / 127 - u1, through shared memory);
//   unit 0, i2 > N2/2 (fold only): slice F/2 (self-paired, the unit's second half) pairs rows
//     j = i2 - N2/2 - 1 and N2 - 1 - j;
//   unit pu > 0: row i2 of slice pu with row N2 - 1 - i2 of slice F - pu (the second half).
// The partner row is transformed in the complement layout, so Z[-u] is register-local.
// acc_ready (block-uniform): the scheduler thread already acquired this item's accumulator
// counter (the previous k-tile's update is visible); otherwise the update waits at the end.
__device__ __forceinline__ void p2_item(const Args &p, int kappa, int t, int pu, int slot, int i2, uint32_t tmem,
                                        const int *acc_flag, int acc_ready, double *S) {
  acc_ready |= kappa == 0;  // k-tile 0 adds to a previous launch's accumulator (stream order)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N2 = p.N2, F = p.F;
  bool pair = true;
  int halfA = 0, rowA = i2, halfB = 0, u2B = N2 - 1 - i2, baseA = pu, baseB = pu;
  if (pu == 0) {
    if (2 * i2 <= N2) {  // slice 0
      pair = i2 > 0 && 2 * i2 < N2;
      u2B = N2 - i2;
    } else {  // fold: slice F/2 in the unit's second half, rows j and N2 - 1 - j
      const int j = i2 - (N2 / 2 + 1);
      halfA = halfB = 1;
      rowA = j;
      u2B = N2 - 1 - j;
      baseA = baseB = F / 2;
    }
  } else {
    if (i2 >= N2) return;  // block-uniform: the spare item of a slice-pair unit
    halfB = 1;
    baseB = F - pu;
  }
  // after the lane reduction this lane owns double `lane` = (register lane >> 1, re/im lane & 1)
  const int u1 = post_pos(warp, lane >> 1);
  int entry = -1;
  bool conj = false;
  if (pair) {
    if (u1 < 64) entry = baseA + F * (rowA + N2 * u1);
    else { entry = baseB + F * (u2B + N2 * (127 - u1)); conj = true; }  // b - u holds conj(FA FB (u))
  } else if (i2 == 0) {
    if (u1 <= 64) entry = F * (N2 * u1);
  } else if (u1 <= 63) {
    entry = F * (i2 + N2 * u1);
  }
  double *a = entry >= 0 ? p.acc + (((int64_t)t * (p.bfull / 2 + 1) + entry) * 2 + (lane & 1)) : nullptr;
  const double acc_old = (a && (kappa > 0 || p.acc_add) && acc_ready) ? __ldcg(a) : 0.0;
  double v[32];
  slice_dft<false>(p, slot, halfA, rowA, v, S);
  if (pair) {
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st8(tq + 16 * c, v + 8 * c);
    tmem_wait_st();
    slice_dft<true>(p, slot, halfB, u2B, v, S);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double zu[8];
      tmem_ld8(tq + 16 * c, zu);
#pragma unroll
      for (int q = 0; q < 4; ++q) split_product(zu[2 * q], zu[2 * q + 1], v[8 * c + 2 * q], v[8 * c + 2 * q + 1]);
    }
  } else {
    // self-paired slice: Z[-u] sits at tile position -u1 (i2 = 0) or 127 - u1 (i2 = N2/2)
    double2 *S2 = (double2 *)S;
#pragma unroll
    for (int r = 0; r < 16; ++r) S2[post_pos(warp, r) * 32 + lane] = make_double2(v[2 * r], v[2 * r + 1]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int pu = post_pos(warp, r);
      const int pm = i2 == 0 ? ((128 - pu) & 127) : (127 - pu);
      const double2 zm = S2[pm * 32 + lane];
      double c = zm.x, e = zm.y;
      split_product(v[2 * r], v[2 * r + 1], c, e);
      v[2 * r] = c;
      v[2 * r + 1] = e;
    }
    __syncthreads();
  }
  // sum over the 32 inner indices (lanes) through this warp's 8 KB of shared memory
  double *W = S + warp * 1024;
#pragma unroll
  for (int r = 0; r < 32; ++r) W[r * 32 + (lane ^ r)] = v[r];
  __syncwarp();
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) sum += W[lane * 32 + (j ^ lane)];
  if (conj && (lane & 1)) sum = -sum;  // entry b - u holds conj(FA FB (u))
  if (a) {
    if (kappa == 0) {
      __stcg(a, p.acc_add ? acc_old + sum : sum);
    } else if (acc_ready) {
      __stcg(a, acc_old + sum);
    }
  }
  if (kappa > 0 && !acc_ready) {  // slow path: lane 0 acquires, __syncwarp orders the warp after it
    if (lane == 0)
      while (ld_acquire(acc_flag) < kappa) __nanosleep(32);
    __syncwarp();
    if (a) __stcg(a, __ldcg(a) + sum);
  }
}

struct Item {
  int64_t pos;
  int is_p1, u, idx;
};

// order: [P1(0 .. lag-1) x G1] then groups g: [P1(g+lag) x G1][P2(g) x G2]; once g + lag >= U
// the groups hold only [P2(g) x G2].  G1 = b / 128 is a power of two.
__device__ __forceinline__ Item decode_item(const Args &p, int64_t pos) {
  Item it;
  it.pos = pos;
  const int pro = p.U < p.lag ? p.U : p.lag;
  const int lg1 = 31 - __clz(p.G1);
  if (pos < (int64_t)pro * p.G1) {
    it.is_p1 = 1; it.u = (int)(pos >> lg1); it.idx = (int)(pos & (p.G1 - 1));
    return it;
  }
  const int q = (int)(pos - (int64_t)pro * p.G1);
  const int full = p.U - pro;  // groups with a P1 part
  const int regular = full * (p.G1 + p.G2);
  if (q < regular) {
    const int g = fdiv(q, p.div_grp);
    const int r = q - g * (p.G1 + p.G2);
    if (r < p.G1) { it.is_p1 = 1; it.u = g + p.lag; it.idx = r; }
    else { it.is_p1 = 0; it.u = g; it.idx = r - p.G1; }
  } else {
    const int q2 = q - regular;
    const int g2 = q2 / p.G2;
    it.is_p1 = 0; it.u = full + g2; it.idx = q2 - g2 * p.G2;
  }
  return it;
}

template <int S1, bool FOLD>
__global__ void __launch_bounds__(THREADS, 2) fft2p_kernel(Args p) {
  extern __shared__ __align__(16) double S[];  // 64 KB: exchanges, partner lookups, lane reduction
  __shared__ uint32_t s_tmem;
  __shared__ int s_item[8];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (FOLD) {  // w_b^e for e = l, 128 l (l < 128) and 16384 l (l < 64)
    for (int x = tid; x < 320; x += THREADS) {
      const int l = x < 128 ? x : (x < 256 ? x - 128 : x - 256);
      const double e = x < 128 ? (double)l : (x < 256 ? 128.0 * l : 16384.0 * l);
      double sn, cs;
      sincospi(-2.0 * e / (double)p.bfull, &sn, &cs);
      const double2 w = make_double2(cs, sn);
      if (x < 128) s_tf0[l] = w;
      else if (x < 256) s_tf1[l] = w;
      else s_tf2[l] = w;
    }
  }
  if (!FOLD) {  // w_b^l and w_b^(128 h), l, h < 128 (exact dyadic arguments, as twiddle_b_kernel)
    const double e = tid < 128 ? (double)tid : (double)(128 * (tid - 128));
    double sn, cs;
    sincospi(-2.0 * e / (double)p.bsz, &sn, &cs);
    if (tid < 128) s_tw_lo[tid] = make_double2(cs, sn);
    else s_tw_hi[tid - 128] = make_double2(cs, sn);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  int *ticket = p.ctr;
  int *done1 = p.ctr + 1;
  int *done2 = done1 + p.U;
  int *acc_cnt = done2 + p.U;
  const int64_t total = (int64_t)p.U * (p.G1 + p.G2);
  // Thread 0 schedules one item ahead (the ticket after next is claimed while the
  // current item computes).  Dependencies, as fwht2p: thread 0 issues RELAXED loads
  // of the next item's counters right before [B]; after [B] its fence.acquire
  // acquires them (an incomplete must-precede counter is polled with ld.acquire) and
  // [A] orders the CTA.  Thread 32 publishes the item after [B] (fence.release, then
  // the completion adds); warp 1 joins [A] through its own barrier with warp 0, so the
  // release's wait for the item's stores does not hold the other warps.
  // The accumulator counter (previous k-tile's P2 of the same rows) is only recorded:
  // if incomplete, the P2 item waits for it per warp at its end (acc_ready).
  __shared__ int64_t sh_nxt;
  __shared__ Item sh_itn;
  __shared__ int sh_ver[2];  // highest unit thread 0 acquired: done1 (P2 items), done2 (P1 slot reuse)
  __shared__ int s_acc_ok;
  int64_t &nxt = sh_nxt;
  Item &itn = sh_itn;
  struct Deps {
    const int *ptr[2];
    int tgt[2], val[2];
    int ver[2];
  };
  auto deps_of = [&](const Item &it, Deps &D) {
    D.ptr[0] = D.ptr[1] = nullptr;
    D.tgt[0] = D.tgt[1] = D.val[0] = D.val[1] = 0;
    D.ver[0] = sh_ver[0];
    D.ver[1] = sh_ver[1];
    if (it.pos >= total) return;
    if (it.is_p1) {
      const int need = it.u - p.nslot;
      if (need > sh_ver[1]) { D.ptr[0] = done2 + need; D.tgt[0] = p.G2; D.ver[1] = need; }
    } else {
      if (it.u > sh_ver[0]) { D.ptr[0] = done1 + it.u; D.tgt[0] = p.G1; D.ver[0] = it.u; }
      const int kap = fdiv(it.u, p.div_dnpu);
      if (kap > 0) {
        const int rem = it.u - kap * p.d * p.NPU;
        const int tt = fdiv(rem, p.div_npu);
        D.ptr[1] = acc_cnt + (tt * p.NPU + (rem - tt * p.NPU)) * p.G2 + it.idx;
        D.tgt[1] = kap;
      }
    }
  };
  auto deps_settle = [&](Deps &D) {
    if (D.ptr[0] && D.val[0] < D.tgt[0])
      while (ld_acquire(D.ptr[0]) < D.tgt[0]) __nanosleep(32);
    sh_ver[0] = D.ver[0];
    sh_ver[1] = D.ver[1];
    s_acc_ok = (!D.ptr[1] || D.val[1] >= D.tgt[1]) ? 1 : 0;
  };
  if (tid == 0) {
    const int64_t cur = atomicAdd(ticket, 1);
    nxt = atomicAdd(ticket, 1);
    itn = decode_item(p, cur);
    sh_ver[0] = sh_ver[1] = -1;
    Deps D;  // the first item's dependencies
    deps_of(itn, D);
    deps_settle(D);
    s_acc_ok = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  while (true) {
    if (tid == 0) {
      const Item it = itn;
      s_item[0] = it.pos < total ? 1 : 0;
      s_item[1] = it.is_p1;
      s_item[2] = it.u;
      s_item[3] = it.idx;
      const int kap = fdiv(it.u, p.div_dnpu);
      const int rem = it.u - kap * p.d * p.NPU;
      const int tt = fdiv(rem, p.div_npu);
      s_item[4] = kap;                             // kappa
      s_item[5] = tt;                              // t
      s_item[6] = fmod_(it.u, p.div_slot);         // Y slot
      s_item[7] = rem - tt * p.NPU;                // slice-pair unit
      itn = decode_item(p, nxt);
    }
    tc_fence_before();
    if (warp == 1) {  // [A] (warp 1 may still be publishing the previous item)
      asm volatile("bar.sync 2, 64;" ::: "memory");
    } else {
      if (warp == 0) asm volatile("bar.arrive 2, 64;" ::: "memory");
      asm volatile("bar.sync 1, 224;" ::: "memory");
    }
    tc_fence_after();
    const int go = s_item[0];
    const int is_p1 = s_item[1], u = s_item[2], idx = s_item[3];
    const int kappa = s_item[4], t = s_item[5], slot = s_item[6], pu = s_item[7];
    const int acc_ok = s_acc_ok && !p.acc_slow;
    if (tid == 0 && go) nxt = itn.pos < total ? (int64_t)atomicAdd(ticket, 1) : itn.pos;
    if (!go) break;
    int *acc_flag = acc_cnt + (t * p.NPU + pu) * p.G2 + idx;
    if (is_p1) p1_item<S1, FOLD>(p, kappa, t, pu, slot, idx, S);
    else p2_item(p, kappa, t, pu, slot, idx, tmem, acc_flag, acc_ok, S);
    Deps D;  // thread 0: relaxed probe of the next item's counters (acquired by the fence below)
    if (tid == 0) {
      const Item nx = itn;
      deps_of(nx, D);
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (D.ptr[j]) D.val[j] = ld_relaxed(D.ptr[j]);
    }
    tc_fence_before();
    __syncthreads();  // [B]
    tc_fence_after();
    if (tid == 32) {  // release this item (covered through [B]), then publish it
      asm volatile("fence.release.gpu;" ::: "memory");
      if (is_p1) red_add(done1 + u, 1);
      else {
        red_add(acc_flag, 1);
        red_add(done2 + u, 1);
      }
    }
    if (tid == 0) {  // acquire the probed counters (relaxed reads, then an acquire fence)
      asm volatile("fence.acquire.gpu;" ::: "memory");
      deps_settle(D);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

static inline int64_t pad256(int64_t x) { return ((x + 255) / 256) * 256; }

static int init_w128(cudaStream_t s) {
  static std::atomic<bool> done[64];  // idempotent: concurrent first calls copy the same table
  int dev = 0;
  SMM_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 64 && done[dev].load(std::memory_order_acquire)) return SMM_OK;
  double2 w[64];
  for (int j = 0; j < 64; ++j) {
    const double ang = M_PI * (double)j / 64.0;  // 2 pi j / 128
    w[j] = make_double2(std::cos(ang), -std::sin(ang));
  }
  SMM_CUDA_TRY(cudaMemcpyToSymbolAsync(c_w128, w, sizeof(w), 0, cudaMemcpyHostToDevice, s), "w128 table");
  SMM_CUDA_TRY(cudaStreamSynchronize(s), "w128 table");
  if (dev < 64) done[dev].store(true, std::memory_order_release);
  return SMM_OK;
}

}  // namespace f2p

bool fft2p_supported(int log2b, int64_t n1, int64_t n2) {
  return log2b >= 8 && log2b <= 20 && n1 < ((int64_t)1 << 26) && n2 < ((int64_t)1 << 26);
}

namespace f2p {
// Geometry: slices of 2^LBs frequencies (LBs <= 14: one 128 x N2 four-step FFT each);
// b > 2^14 is folded into F = b / 2^14 slices, grouped into NPU = F/2 + 1 slice-pair units.
struct Geom {
  int LBs, S1, N2, F, NPU, halves, G1, G2;
  int64_t bs;
};
static Geom geometry(int log2b) {
  Geom g;
  g.LBs = log2b < 14 ? log2b : 14;
  g.S1 = g.LBs - 7;
  g.N2 = 1 << g.S1;
  g.bs = (int64_t)1 << g.LBs;
  g.F = 1 << (log2b - g.LBs);
  if (g.F == 1) {
    g.NPU = 1; g.halves = 1; g.G1 = g.N2; g.G2 = g.N2 / 2 + 1;
  } else {  // fixed item counts per unit (empty items for the self-paired slices)
    // units: {0, F/2} and the pairs {a, F - a}; pass 2: N2 rows per pair unit (+1 spare),
    // N2/2 + 1 rows of slice 0 and N2/2 of slice F/2 in unit 0
    g.NPU = g.F / 2; g.halves = 2; g.G1 = 2 * 128; g.G2 = 128 + 1;
  }
  return g;
}

// Ring plan (as fwht2p.cu): lag for ~4 dispensable items per SM, slack up to 6 units
// between pass 2 and the pass-1 items that reuse its slots (pass-2 pair items weigh
// about two pass-1 items; at slack 2, 45 % of CTA time went into pass-1 slot waits),
// the T ring within ~96 MB of L2.
static void ring_plan(const Geom &g, int64_t U, int &lag, int &nslot) {
  const int grp = g.G1 + g.G2;
  const int64_t slot = (int64_t)g.halves * g.bs * KT * 16;
  int maxslots = (int)(((int64_t)96 << 20) / slot);
  if (maxslots < 3) maxslots = 3;
  lag = (4 * num_sms() + grp - 1) / grp;
  if (lag > maxslots - 2) lag = maxslots - 2;
  lag = lag < 1 ? 1 : (lag > 64 ? 64 : lag);
  int slack = maxslots - lag;  // whatever the L2 budget leaves (cfg5 b = 2^12: 4.2 -> 3.6 ms)
  slack = slack < 2 ? 2 : slack;
  nslot = lag + slack;
  if (nslot > U + 1) nslot = (int)(U + 1 > lag + 1 ? U + 1 : lag + 1);
}
}  // namespace f2p

int64_t fft2p_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K) {
  using f2p::pad256;
  const f2p::Geom g = f2p::geometry(log2b);
  const int64_t b = (int64_t)1 << log2b;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int64_t ntiles = (K + f2p::KT - 1) / f2p::KT;
  const int64_t U = ntiles * d * g.NPU;
  int64_t w = 0;
  w += pad256((int64_t)d * 2 * (g.bs + 1) * 4);                // off
  w += pad256((int64_t)d * 2 * g.bs * 4);                      // cnt / fill
  w += pad256((int64_t)d * 2 * nmax * 4);                      // ent
  w += pad256(b * 16);                                         // twiddles w_b^x
  int lag, nslot;
  f2p::ring_plan(g, U, lag, nslot);
  w += pad256((int64_t)nslot * g.halves * g.bs * f2p::KT * 16);  // T ring
  w += pad256((1 + 2 * U + (int64_t)d * g.NPU * g.G2) * 4);    // counters
  return w;
}

int fft2p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb, int64_t n1,
                     int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws, int64_t ws_bytes,
                     cudaStream_t s) {
  using namespace f2p;
  const int d = h.d, log2b = h.log2b;
  const Geom g = geometry(log2b);
  const int64_t b = (int64_t)1 << log2b;
  const int64_t bs = g.bs;
  const int64_t K = k1 - k0;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int S1 = g.S1;
  if (lda >= ((int64_t)1 << 28) || ldb >= ((int64_t)1 << 28)) {
    set_error("operand row stride too large for the two-pass kernel");
    return SMM_ERR_INVALID;
  }
  if (ws_bytes < fft2p_workspace(d, log2b, n1, n2, K)) {
    set_error("compress workspace too small (two-pass fft)");
    return SMM_ERR_WORKSPACE;
  }
  char *q = ws;
  int32_t *off = (int32_t *)q;
  q += pad256((int64_t)d * 2 * (bs + 1) * 4);
  int32_t *cnt = (int32_t *)q;
  q += pad256((int64_t)d * 2 * bs * 4);
  uint32_t *ent = (uint32_t *)q;
  q += pad256((int64_t)d * 2 * nmax * 4);
  double *twb = (double *)q;
  q += pad256(b * 16);
  double *Y = (double *)q;
  const int64_t ntiles = (K + KT - 1) / KT;
  const int64_t U = ntiles * d * g.NPU;
  int lag, nslot;
  ring_plan(g, U, lag, nslot);
  q += pad256((int64_t)nslot * g.halves * bs * KT * 16);
  int *ctr = (int *)q;
  const int N2 = g.N2, G1 = g.G1, G2 = g.G2;
  const size_t acc_bytes = (size_t)d * (size_t)(b / 2 + 1) * 16;
  if (K <= 0) {
    if (!acc_add) SMM_CUDA_TRY(cudaMemsetAsync(acc, 0, acc_bytes, s), "acc memset");
    return SMM_OK;
  }
  if (U * (G1 + G2) > ((int64_t)1 << 30)) {
    set_error("inner range too large for one call");
    return SMM_ERR_INVALID;
  }
  int rc = init_w128(s);
  if (rc) return rc;
  twiddle_b_kernel<<<(unsigned)ceil_div(b, 256) > 1024 ? 1024 : (unsigned)ceil_div(b, 256), 256, 0, s>>>(twb, log2b);
  SMM_LAUNCH_CHECK("twiddle_b_kernel");
  // plan: CSR by bit-reversed tile position
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * bs * 4, s), "csr memset");
  const int64_t nin = (int64_t)d * (n1 + n2);
  int64_t blocks = ceil_div(nin, 256);
  if (blocks > 8192) blocks = 8192;
  if (nin > 0) {
    csr_count_fft<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, cnt, bs, S1);
    SMM_LAUNCH_CHECK("csr_count_fft");
  }
  csr_scan_kernel<<<d * 2, 1024, 0, s>>>(cnt, off, bs);
  SMM_LAUNCH_CHECK("csr_scan_kernel");
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * bs * 4, s), "csr memset");
  if (nin > 0) {
    csr_fill_fft<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, off, cnt, ent, nmax, bs, S1);
    SMM_LAUNCH_CHECK("csr_fill_fft");
    const int rc = csr_sort(off, ent, nmax, bs, d * 2, s);  // deterministic: increasing i per bucket
    if (rc) return rc;
  }
  SMM_CUDA_TRY(cudaMemsetAsync(ctr, 0, (size_t)(1 + 2 * U + (int64_t)d * g.NPU * G2) * 4, s), "counter memset");
  Args p;
  p.h = h;
  p.X[0] = xa;
  p.X[1] = xb;
  p.ld[0] = lda;
  p.ld[1] = ldb;
  p.k0 = k0;
  p.K = K;
  p.B = log2b;
  p.N2 = N2;
  p.G1 = G1;
  p.G2 = G2;
  p.U = (int)U;
  p.d = d;
  p.F = g.F;
  p.NPU = g.NPU;
  p.halves = g.halves;
  p.div_dnpu = make_fastdiv((uint32_t)(d * g.NPU));
  p.div_npu = make_fastdiv((uint32_t)g.NPU);
  p.div_slot = make_fastdiv((uint32_t)nslot);
  p.lag = lag;
  p.nslot = nslot;
  p.div_grp = make_fastdiv((uint32_t)(G1 + G2));
  p.off = off;
  p.ent = ent;
  p.nmax = nmax;
  p.bsz = bs;
  p.bfull = b;
  p.twb = twb;
  p.Y = Y;
  p.acc = acc;
  p.ctr = ctr;
  p.acc_add = acc_add ? 1 : 0;
  static const bool acc_slow = getenv("SMM_ACC_SLOWPATH") != nullptr;
  p.acc_slow = acc_slow ? 1 : 0;
  const size_t smem = (size_t)8 * 32 * 32 * 8;
  const int G = 2 * num_sms();
#define F2P_LAUNCH(SS, FD)                                                                             \
  case SS + 8 * FD:                                                                                   \
    SMM_CUDA_TRY(cudaFuncSetAttribute(fft2p_kernel<SS, FD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), \
                 "fft2p smem");                                                                       \
    fft2p_kernel<SS, FD><<<G, THREADS, smem, s>>>(p);                                                 \
    break;
  KernelTimer timer(0, s);
  switch (S1 + 8 * (g.F > 1 ? 1 : 0)) {
    F2P_LAUNCH(1, 0) F2P_LAUNCH(2, 0) F2P_LAUNCH(3, 0) F2P_LAUNCH(4, 0) F2P_LAUNCH(5, 0) F2P_LAUNCH(6, 0)
    F2P_LAUNCH(7, 0) F2P_LAUNCH(7, 1)
#undef F2P_LAUNCH
    default:
      set_error("two-pass fft kernel: unsupported width");
      return SMM_ERR_INVALID;
  }
  timer.stop();
  SMM_LAUNCH_CHECK("fft2p_kernel");
  return SMM_OK;
}

}  // namespace smm
